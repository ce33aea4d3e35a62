// Latency of one all-to-all push round in a 16-CTA cluster, the statistics
// kernel's minimum exchange: every CTA st.async-pushes 8 bytes into slot
// [rank] of every peer (mbarrier complete_tx) and waits on its own barrier.
// Reports globaltimer ns from the push to the local barrier's completion,
// with mbarrier.try_wait vs test_wait polling.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/dsmem_push scripts/micro/dsmem_push.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}

template <bool TEST>
__global__ void __launch_bounds__(256, 1) push_round(long long* out, int rounds) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double slots[16];
  __shared__ __align__(8) unsigned long long bar;
  const int rank = (int)cl.block_rank(), n = (int)cl.num_blocks();
  const uint32_t b = smem_addr(&bar);
  long long acc = 0;
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(8u * n) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    cl.sync();
    const unsigned long long t0 = gt();
    if (threadIdx.x < n) {
      const double v = rank + 0.5;
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                       mapa(smem_addr(&slots[rank]), threadIdx.x)),
                   "l"(__double_as_longlong(v)), "r"(mapa(b, threadIdx.x))
                   : "memory");
    }
    uint32_t ok = 0;
    while (!ok) {
      if (TEST)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(b) : "memory");
      else
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(b) : "memory");
    }
    const unsigned long long t1 = gt();
    acc += (long long)(t1 - t0);
    cl.sync();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc / rounds;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  for (int test = 0; test < 2; ++test)
    for (int cs : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, 1, 1);
      cfg.blockDim = dim3(256, 1, 1);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      auto k = test ? push_round<true> : push_round<false>;
      if (cs > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k, d, 200);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("cluster %d: %s\n", cs, cudaGetErrorString(e));
        continue;
      }
      long long h[64];
      cudaMemcpy(h, d, cs * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0, s = 0;
      for (int i = 0; i < cs; ++i) {
        s += h[i];
        mx = h[i] > mx ? h[i] : mx;
      }
      printf("%s cluster %2d: push -> all %d pushes landed: mean %lld ns, max %lld ns\n",
             test ? "test_wait" : "try_wait ", cs, cs, s / cs, mx);
    }
  return 0;
}
