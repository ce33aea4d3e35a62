// tcgen05.mma issue/execution rate on one SM (all 148 SMs run the same CTA)
// for the MLP's shapes, alone and with 16 warps streaming TMEM loads/stores
// on a disjoint TMEM region (the epilogue's traffic):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -Iinclude -o scripts/micro/mma_rate scripts/micro/mma_rate.cu
#include <cstdio>

#include "../../paper_2104_13542_b200/csrc/mppi_mlp.cuh"

using namespace mppi;

// mode bit 0: A from TMEM (else smem); N in {64, 128, 256}; traffic 0 none, 1 ld x16, 2 ld+st x16, 3 st x16
__global__ void __launch_bounds__(17 * 32, 1) mma_rate(int N, int a_tmem, int traffic, int reps, long long* out, int nacc, int bvar) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ unsigned long long bar;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (warp == 16) {
    if (lane == 0) {
      const uint32_t sb = smem_u32(sm);
      const uint64_t dA = umma_desc(sb, 128, 256);            // 128 x 16 fp16 K-major
      const uint64_t dB = umma_desc(sb + 8192, 128, 256);      // N x 16
      const uint32_t id = umma_idesc((uint32_t)N);
      const long long t0 = clock64();
      if (a_tmem) {
        for (int r = 0; r < reps; ++r) {
          const uint32_t dcol = (uint32_t)((r % nacc) * N);
          const uint64_t b = dB + (uint64_t)((r % bvar) * (8192 >> 4));
          umma_f16_ts(tm + dcol, tm + 448 + 8 * (r & 1) * (bvar > 1), b, id, r >= nacc ? 1u : 0u);
        }
      } else {
        for (int r = 0; r < reps; ++r) {
          const uint32_t dcol = (uint32_t)((r % nacc) * N);
          umma_f16(tm + dcol, dA, dB + (uint64_t)((r % bvar) * (8192 >> 4)), id, r >= nacc ? 1u : 0u);
        }
      }
      const long long t1 = clock64();
      umma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), 0);
      const long long t2 = clock64();
      done = 1;
      if (blockIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t0;
      }
    }
  } else if (traffic) {
    const uint32_t base = tm + ((uint32_t)(32 * (warp & 3)) << 16) + 384 + 16 * (warp >> 2) % 64;
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = i;
    long long n = 0;
    while (!done) {
      if (traffic & 1) {
        tmem_ld16_async(base, r);
        tmem_wait_ld16(r);
      }
      if (traffic & 2) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
            "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(base),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
            "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      ++n;
    }
    if (blockIdx.x == 0 && tid == 0) out[2] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  struct C { int a, N, nacc, bvar; };
  const int reps = 2048;
  const C cs[] = {{1, 128, 1, 1}, {1, 128, 2, 1}, {1, 128, 3, 1}, {1, 128, 1, 2}, {1, 128, 2, 2},
                  {1, 64, 1, 1},  {1, 64, 2, 1},  {1, 64, 4, 1},  {1, 256, 1, 1}, {0, 128, 1, 1},
                  {0, 128, 2, 1}, {0, 128, 1, 2}, {0, 256, 1, 1}};
  for (const C& c : cs)
    for (int traffic : {0, 3}) {
      mma_rate<<<148, 17 * 32, 64 * 1024>>>(c.N, c.a, traffic, reps, d, c.nacc, c.bvar);
      mma_rate<<<148, 17 * 32, 64 * 1024>>>(c.N, c.a, traffic, reps, d, c.nacc, c.bvar);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      long long h[3] = {0, 0, 0};
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("A %-4s N=%3d accumulators %d B/A operands %d traffic %-9s: %6.1f clk/MMA issue, %6.1f done (%.0f MAC/clk)\n",
             c.a ? "tmem" : "smem", c.N, c.nacc, c.bvar, traffic ? "ld16+st16" : "none", (double)h[0] / reps,
             (double)h[1] / reps, 128.0 * c.N * 16 * reps / h[1]);
    }
  return 0;
}
