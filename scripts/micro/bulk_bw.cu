// Microbenchmark: time for G CTAs (one per SM) to pull a 182 KB weight image
// into shared memory with cp.async.bulk (pieces of P bytes) or plain vector
// loads. nvcc -gencode arch=compute_100a,code=sm_100a -O3 bulk_bw.cu -o bulk_bw
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr uint32_t kBytes = 182400;
constexpr uint32_t kSmem = 190000;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const unsigned char* src, int replicas, uint32_t piece, int mode,
                            unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  src += (size_t)(blockIdx.x % replicas) * kBytes;
  const uint32_t b = su32(&bar);
  if (mode == 0) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kBytes) : "memory");
      for (uint32_t o = 0; o < kBytes; o += piece) {
        const uint32_t n = min(piece, kBytes - o);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sm) + o), "l"(src + o), "r"(n), "r"(b) : "memory");
      }
      asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}"
                   ::"r"(b) : "memory");
    }
  } else if (mode == 1) {  // many threads each issue pieces
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kBytes) : "memory");
    }
    __syncthreads();
    const uint32_t np = (kBytes + piece - 1) / piece;
    for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
      const uint32_t o = i * piece, n = min(piece, kBytes - o);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(sm) + o), "l"(src + o), "r"(n), "r"(b) : "memory");
    }
    if (threadIdx.x == 0)
      asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}"
                   ::"r"(b) : "memory");
  } else {  // plain 16-byte loads by all threads
    for (uint32_t o = threadIdx.x * 16; o < kBytes; o += blockDim.x * 16)
      *reinterpret_cast<uint4*>(sm + o) = __ldg(reinterpret_cast<const uint4*>(src + o));
  }
  __syncthreads();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = t0;
    out[2 * blockIdx.x + 1] = t1;
  }
}

int main() {
  const int G = 125, R = 32;
  unsigned char* src;
  cudaMalloc(&src, (size_t)kBytes * R);
  cudaMemset(src, 1, (size_t)kBytes * R);
  unsigned char* flush;
  cudaMalloc(&flush, 256 << 20);
  unsigned long long* out;
  cudaMalloc(&out, 2 * G * sizeof(unsigned long long));
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  std::vector<unsigned long long> h(2 * G);
  struct Cfg { int mode, rep; uint32_t piece; int threads; const char* name; };
  Cfg cfgs[] = {{0, 1, 32768, 128, "bulk 32K pieces, 1 thread, 1 replica"},
                {0, 1, 4096, 128, "bulk 4K pieces, 1 thread, 1 replica"},
                {0, 32, 32768, 128, "bulk 32K pieces, 1 thread, 32 replicas"},
                {1, 1, 4096, 128, "bulk 4K pieces, 128 threads, 1 replica"},
                {1, 1, 1024, 256, "bulk 1K pieces, 256 threads, 1 replica"},
                {2, 1, 16, 256, "ld.global.v4, 256 threads, 1 replica"},
                {2, 1, 16, 512, "ld.global.v4, 512 threads, 1 replica"}};
  for (int cold = 0; cold < 2; ++cold)
    for (auto& c : cfgs) {
      double best = 1e30, worst_sum = 0;
      for (int rep = 0; rep < 5; ++rep) {
        if (cold) cudaMemset(flush, rep, 256 << 20);
        else bulk_kernel<<<G, c.threads, kSmem>>>(src, c.rep, c.piece, c.mode, out);
        bulk_kernel<<<G, c.threads, kSmem>>>(src, c.rep, c.piece, c.mode, out);
        cudaDeviceSynchronize();
        cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull, t1 = 0;
        double sum = 0;
        for (int i = 0; i < G; ++i) {
          t0 = std::min(t0, h[2 * i]);
          t1 = std::max(t1, h[2 * i + 1]);
          sum += (double)(h[2 * i + 1] - h[2 * i]);
        }
        best = std::min(best, (double)(t1 - t0) * 1e-3);
        worst_sum += sum / G * 1e-3;
      }
      printf("%s %-44s span %.2f us  mean per-CTA %.2f us\n", cold ? "cold" : "warm", c.name, best, worst_sum / 5);
    }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
