// TMEM load/store throughput per SM on the B200 (sm_100a): W warps of one CTA
// per SM each read (or write) X columns of their lane quadrant with
// tcgen05.ld/st.32x32b.xX, R times; prints bytes per SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/tmem_bw scripts/micro/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int X>
__device__ __forceinline__ void ld(uint32_t a, uint32_t* r);
template <>
__device__ __forceinline__ void ld<8>(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a));
}
template <>
__device__ __forceinline__ void ld<16>(uint32_t a, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(a));
}
template <int X>
__device__ __forceinline__ void st(uint32_t a, const uint32_t* r);
template <>
__device__ __forceinline__ void st<8>(uint32_t a, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
template <>
__device__ __forceinline__ void st<16>(uint32_t a, const uint32_t* r) {
  st<8>(a, r);
  st<8>(a + 8, r + 8);
}

// mode 0: ld + wait per access; 1: two lds in flight; 2: st + wait::st; 3: ld, st back
template <int X, int MODE>
__global__ void tmem_bw(int reps, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const uint32_t base = tm + ((uint32_t)(32 * (warp & 3)) << 16);
  const int groups = nw / 4;  // column groups per quadrant
  const int g = warp >> 2;
  const int span = 512 / groups;  // columns per warp
  uint32_t acc = 0, r[2][X];
  for (int i = 0; i < X; ++i) r[0][i] = r[1][i] = threadIdx.x + i;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    const uint32_t col = (uint32_t)(g * span + (it * X) % span);
    if (MODE == 0) {
      ld<X>(base + col, r[0]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < X; ++i) acc ^= r[0][i];
    } else if (MODE == 1) {
      ld<X>(base + col, r[0]);
      ld<X>(base + ((col + X) % 512), r[1]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < X; ++i) acc ^= r[0][i] + r[1][i];
    } else if (MODE == 2) {
      st<X>(base + col, r[0]);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else {
      ld<X>(base + col, r[0]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < X; ++i) r[0][i] += 1u;
      st<X>(base + col, r[0]);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int X, int MODE>
void run(int warps, unsigned long long* d_cyc, uint32_t* sink) {
  const int reps = 4096;
  tmem_bw<X, MODE><<<148, warps * 32>>>(reps, d_cyc, sink);
  cudaDeviceSynchronize();
  tmem_bw<X, MODE><<<148, warps * 32>>>(reps, d_cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = (double)warps * reps * 32 * X * 4 * (MODE == 1 ? 2 : 1) * (MODE == 3 ? 2 : 1);
  const char* names[] = {"ld+wait", "2ld+wait", "st+wait", "ld,st"};
  printf("%-9s x%-2d warps %2d: %7.1f B/clk/SM  (%.1f clk per access per warp)\n", names[MODE], X, warps,
         bytes / mx, (double)mx / reps);
}

int main() {
  unsigned long long* d_cyc;
  uint32_t* sink;
  cudaMalloc(&d_cyc, 148 * sizeof(unsigned long long));
  cudaMalloc(&sink, 64);
  for (int w : {4, 8, 16, 32}) {
    run<8, 0>(w, d_cyc, sink);
    run<16, 0>(w, d_cyc, sink);
    run<8, 1>(w, d_cyc, sink);
    run<16, 1>(w, d_cyc, sink);
    run<8, 2>(w, d_cyc, sink);
    run<16, 2>(w, d_cyc, sink);
    run<8, 3>(w, d_cyc, sink);
  }
  return 0;
}
