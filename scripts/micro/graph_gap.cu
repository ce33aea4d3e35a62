// Kernel-to-kernel gap inside a CUDA graph on B200: chains of 1..4 small
// kernels (and a 190 KB-shared-memory kernel after a small one), timed with
// events around the replay and with globaltimer stamps at CTA entry/exit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o graph_gap graph_gap.cu && ./graph_gap
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_t[64];

__global__ void k_small(int slot, int work) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot] = t;
  float x = threadIdx.x;
  for (int i = 0; i < work; ++i) x = x * 1.0001f + 0.5f;
  if (x == 12345.f) g_t[63] = 1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot + 1] = t;
}

struct BigParams {
  float pad[580];  // ~2.3 KB, like RolloutArgs<float>
  int slot;
};

__global__ void k_params(const __grid_constant__ BigParams p, float* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * p.slot] = t;
  float x = threadIdx.x + p.pad[threadIdx.x % 580];
  for (int i = 0; i < 100; ++i) x = x * 1.0001f + 0.5f;
  if (out) {  // 8 KB of stores per CTA at the end (like the rollout's encodings)
    float4* o = reinterpret_cast<float4*>(out) + (size_t)blockIdx.x * 512;
    for (int i = threadIdx.x; i < 512; i += blockDim.x) o[i] = make_float4(x, x, x, x);
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * p.slot + 1] = t;
}

// ~64 KB of straight-line code (large kernels, like the rollout / MLP)
template <int U>
__global__ void k_code(int slot, float* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot] = t;
  float x = threadIdx.x, y = blockIdx.x;
#pragma unroll
  for (int i = 0; i < U; ++i) {
    x = __sinf(x) * y + 0.25f * i;
    y = __cosf(y) * x - 0.5f;
  }
  if (x == 12345.f) out[0] = y;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot + 1] = t;
}

__global__ void k_big(int slot) {
  extern __shared__ unsigned char sm[];
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot] = t;
  sm[threadIdx.x] = 1;
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot + 1] = t + sm[5];
}

// like k_big, plus a 512-column tensor-memory allocation (tcgen05)
__global__ void k_tmem(int slot) {
  extern __shared__ unsigned char sm[];
  __shared__ unsigned slot_addr;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot] = t;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&slot_addr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  sm[threadIdx.x] = 1;
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot_addr));
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot + 1] = t + sm[5];
}

// MLP-shaped launch: 544 threads, 88 registers in use, ~190 KB of dynamic
// shared memory, a TMEM allocation and a large body
__global__ void __launch_bounds__(544, 1) k_mlp_like(int slot, float* out) {
  extern __shared__ unsigned char sm[];
  __shared__ unsigned slot_addr;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot] = t;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&slot_addr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  float r[60];
#pragma unroll
  for (int i = 0; i < 60; ++i) r[i] = threadIdx.x * (i + 1) * 0.5f;
#pragma unroll
  for (int k = 0; k < 40; ++k)
#pragma unroll
    for (int i = 0; i < 60; ++i) r[i] = __sinf(r[i]) * r[(i + 7) % 60] + 0.25f;
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 60; ++i) acc += r[i];
  sm[threadIdx.x] = (unsigned char)acc;
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot_addr));
  if (acc == 1234.5f) out[0] = acc;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) g_t[2 * slot + 1] = t + sm[5];
}

int main(int argc, char**) {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 190 * 1024);
  cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 190 * 1024);
  cudaFuncSetAttribute(k_mlp_like, cudaFuncAttributeMaxDynamicSharedMemorySize, 193840);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float* buf;
  cudaMalloc(&buf, 125 * 8192);
  BigParams bp0 = {};
  bp0.slot = 0;
  unsigned char* flush;
  cudaMalloc(&flush, 256u << 20);
  const bool do_flush = argc > 1;
  for (int variant = 0; variant < 14; ++variant) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    int nk = 0;
    if (variant <= 3) {
      for (int i = 0; i <= variant; ++i) k_small<<<125, 128, 0, st>>>(nk++, 100);
    } else if (variant == 4) {
      k_small<<<125, 128, 0, st>>>(nk++, 100);
      k_big<<<118, 544, 190 * 1024, st>>>(nk++);
      k_small<<<16, 256, 0, st>>>(nk++, 100);
    } else if (variant == 5) {
      k_small<<<125, 128, 0, st>>>(nk++, 100);
      k_small<<<118, 544, 0, st>>>(nk++, 100);
      k_small<<<16, 256, 0, st>>>(nk++, 100);
    } else if (variant == 6) {  // 2.3 KB parameters, no stores
      k_params<<<125, 128, 0, st>>>(bp0, nullptr);
      k_big<<<118, 544, 190 * 1024, st>>>(1);
      nk = 2;
    } else if (variant == 12) {  // small kernel, then the MLP-shaped one, then small
      k_small<<<125, 128, 0, st>>>(nk++, 100);
      k_mlp_like<<<118, 544, 193840, st>>>(nk++, buf);
      k_small<<<16, 256, 0, st>>>(nk++, 100);
    } else if (variant == 13) {  // large-code 128-thread kernel (rollout-like), then the MLP-shaped one
      k_code<600><<<125, 128, 0, st>>>(nk++, buf);
      k_mlp_like<<<118, 544, 193840, st>>>(nk++, buf);
    } else if (variant == 10) {  // small kernel, then a TMEM-allocating 190 KB kernel, then small
      k_small<<<125, 128, 0, st>>>(nk++, 100);
      k_tmem<<<118, 544, 190 * 1024, st>>>(nk++);
      k_small<<<16, 256, 0, st>>>(nk++, 100);
    } else if (variant == 11) {  // TMEM kernel twice
      k_tmem<<<118, 544, 190 * 1024, st>>>(nk++);
      k_tmem<<<118, 544, 190 * 1024, st>>>(nk++);
    } else if (variant == 8) {  // two large-code kernels
      k_code<600><<<125, 128, 0, st>>>(0, buf);
      k_code<600><<<118, 544, 0, st>>>(1, buf);
      nk = 2;
    } else if (variant == 9) {  // large-code kernel, then the 190 KB one
      k_code<600><<<125, 128, 0, st>>>(0, buf);
      k_big<<<118, 544, 190 * 1024, st>>>(1);
      nk = 2;
    } else {  // 2.3 KB parameters + 8 KB of stores per CTA
      k_params<<<125, 128, 0, st>>>(bp0, buf);
      k_big<<<118, 544, 190 * 1024, st>>>(1);
      nk = 2;
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    float best = 1e9, sum = 0;
    unsigned long long ht[64];
    const int reps = 200;
    for (int r = 0; r < reps + 10; ++r) {
      if (do_flush) cudaMemsetAsync(flush, r & 255, 256u << 20, st);
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 10) {
        sum += ms;
        if (ms < best) best = ms;
      }
    }
    cudaMemcpyFromSymbol(ht, g_t, sizeof(ht));
    printf("variant %d (%d kernels): event mean %.2f us, min %.2f us; stamps:", variant, nk, 1e3 * sum / reps,
           1e3 * best);
    for (int i = 0; i < nk; ++i)
      printf(" [%.2f %.2f]", (ht[2 * i] - ht[0]) * 1e-3, (ht[2 * i + 1] - ht[0]) * 1e-3);
    printf("\n");
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  // the same chains launched directly into the stream (no graph), events around them
  for (int nk = 1; nk <= 3; ++nk) {
    float best = 1e9, sum = 0;
    const int reps = 200;
    for (int r = 0; r < reps + 10; ++r) {
      if (do_flush) cudaMemsetAsync(flush, r & 255, 256u << 20, st);
      cudaEventRecord(e0, st);
      for (int i = 0; i < nk; ++i) k_small<<<125, 128, 0, st>>>(i, 100);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 10) {
        sum += ms;
        if (ms < best) best = ms;
      }
    }
    printf("direct launches (%d kernels): event mean %.2f us, min %.2f us\n", nk, 1e3 * sum / reps, 1e3 * best);
  }
  return 0;
}
