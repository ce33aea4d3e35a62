// mppi_fused.cuh — rollout + learned self-collision MLP in one kernel (latency path).
//
// For a single controller (config 2: 500 particles x H30) the step is latency
// bound: the MLP kernel's 176 KiB weight copy, its launch and the HBM round
// trip of the positional encodings sit between the rollout and the statistics.
// Here one CTA owns one 128-row MMA tile = 4 particles x 32 horizon lanes:
//   warps 0-3  roll out particle 4*blockIdx + w (lane = h, rollout_particle)
//              and write the lane's encoding [sin q, cos q] straight into the
//              fp16 hi/lo X tile (row 32w + h == TMEM lane of that warp's
//              quadrant, so the epilogue thread that reads the distance back is
//              the lane that computed the step);
//   warp 8     issues the weight TMA at entry (it lands under the rollout) and
//              then every tcgen05.mma of the three hidden layers;
//   warps 0-7  run the layer epilogues as mlp_tcgen05_kernel does with 16.
// Outputs are the two buffers the statistics kernel reads (step cost without
// the learned term, learned distance), so the statistics path is unchanged.
// The capsule staging area of the rollout aliases the activation buffers,
// which are first written after every rollout warp has passed the X barrier.
//
// Eligible when the particles of all instances fit one wave (ceil(B*N/4) CTAs
// <= SM count) and R = float; larger batches use the persistent MLP kernel.
// Opt-in (MPPI_FUSE=1): on B200 with the L2 flushed before every step it
// measured 1.5-2 us SLOWER than rollout_kernel + mlp_tcgen05_kernel (its
// layer-1 epilogue runs ~2 us longer than the standalone kernel's; see
// DESIGN.md §4.5), so the default path keeps the two kernels.
#pragma once

#include "mppi_kernels.cuh"
#include "mppi_mlp.cuh"

namespace mppi {

constexpr int kFusedParticles = 4;  // one particle per TMEM lane quadrant
// 16 epilogue warps (4 column groups) + the issuer = 544 threads, which caps
// the kernel at 96 registers per thread; the rollout warpgroup raises its own
// limit with setmaxnreg after the other warpgroups lower theirs.
constexpr int kFusedEpiWarps = 16;
constexpr int kFusedRegRollout = 168, kFusedRegEpi = 72, kFusedRegIssuer = 56;
constexpr int kFusedThreads = (kFusedEpiWarps + 1) * 32;
constexpr int kFusedCG = kFusedEpiWarps / 4;   // column groups
constexpr int kFusedCW = 32 / kFusedCG;        // accumulator columns per warp per 32-column chunk

__device__ __forceinline__ void fused_epi_barrier() {
  asm volatile("bar.sync 1, %0;" ::"n"(kFusedEpiWarps * 32) : "memory");
}

template <int CW>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float* y) {
  if constexpr (CW == 8) {
    tmem_ld8(taddr, y);
  } else {
    static_assert(CW % 16 == 0, "column count");
#pragma unroll
    for (int i = 0; i < CW / 16; ++i) tmem_ld16(taddr + 16 * i, y + 16 * i);
  }
}

// store CW activations of one row, columns k0..k0+CW of a 32-wide K-chunk
template <int CW>
__device__ __forceinline__ void store_cols(unsigned char* sm, uint32_t off_h, uint32_t off_l, uint32_t row,
                                           uint32_t k0, const float* y) {
#pragma unroll
  for (int i = 0; i < CW / 8; ++i) store_split8_act(sm, off_h, off_l, umma_off(row, k0 + 8 * i, kAChunkK), y + 8 * i);
}

template <typename R, int D>
__global__ void __launch_bounds__(kFusedThreads, 1)
    rollout_mlp_kernel(const __grid_constant__ RolloutArgs<R> a, const unsigned char* __restrict__ img,
                       float* __restrict__ out_d) {
  extern __shared__ __align__(1024) unsigned char fused_smem[];
  unsigned char* sm = fused_smem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sb = smem_u32(sm);
  const uint32_t barW0 = sb + OFF_BAR, barW1 = barW0 + 8, barW2 = barW0 + 16;
  // pairs of barriers, 8 bytes apart: [0] and [1] per buffer
  const uint32_t barL1[2] = {barW0 + 24, barW0 + 32};
  const uint32_t barL20 = barW0 + 40, barL30 = barW0 + 56, barA0 = barW0 + 72;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_TMEMPTR);
  const long long total = (long long)a.B * a.N;
  const long long g0 = (long long)blockIdx.x * kFusedParticles;
  unsigned long long* dbg = (a.dbg != nullptr && tid == 0 && blockIdx.x < 256) ? a.dbg + 16 * blockIdx.x : nullptr;
  unsigned long long* pdbg =  // issuer stamps: 8 W0, 9 W1, 10 W2, 11 last commit
      (a.dbg != nullptr && tid == kFusedEpiWarps * 32 && blockIdx.x < 256) ? a.dbg + 16 * blockIdx.x : nullptr;
  MPPI_TSTAMP(dbg, 0);

  if (tid == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(barW0 + 8 * i, 1);
    mbar_init(barA0, kFusedEpiWarps);
    mbar_init(barA0 + 8, kFusedEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
  }
  if (warp == kFusedEpiWarps) {  // the producer warp owns TMEM, so the rollout warps start at once
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc2 = tmem + 256, acc3 = tmem + 384;

  // ---- phase 1: weight TMA (issuer) under the rollout (warps 0-3) ----------
  // Everyone else sleeps in the block barrier: a spinning mbarrier wait here
  // would steal issue slots from the rollout warp sharing its SM sub-partition.
  const int quad = warp & 3, cg = warp >> 2;
  const int row_in_tile = quad * 32 + lane;
  const long long g = g0 + quad;
  auto issue_weights = [&]() {
    mbar_expect_tx(barW0, kSeg0);
    bulk_g2s(sb + 0, img, kSeg0, barW0);
    mbar_expect_tx(barW1, kSeg1);
    for (uint32_t o = 0; o < kSeg1; o += 32768)
      bulk_g2s(sb + OFF_W1H + o, img + OFF_W1H + o, min(32768u, kSeg1 - o), barW1);
    mbar_expect_tx(barW2, kSeg2);
    bulk_g2s(sb + OFF_W2H, img + OFF_W2H, kSeg2, barW2);
  };
  // register rebalance per warpgroup (warps 4w..4w+3): the epilogue and issuer
  // warpgroups release registers, the rollout warpgroup takes them
  if (warp == kFusedEpiWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kFusedRegIssuer));
    if (lane == 0) issue_weights();
  } else if (warp >= kFusedParticles) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kFusedRegEpi));
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kFusedRegRollout));
    float enc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) enc[k] = 0.f;
    if (g < total) {
      R* cap = reinterpret_cast<R*>(sm + OFF_A) + (size_t)warp * a.chain.n_caps * 6 * 32;
      rollout_particle<R, D>(a, g, lane, cap, enc);
    }
    MPPI_TSTAMP(dbg, 1);
    store_split8(sm, OFF_XH, OFF_XL, umma_off(row_in_tile, 0, 16), enc);
    store_split8(sm, OFF_XH, OFF_XL, umma_off(row_in_tile, 8, 16), enc + 8);
    fence_async_smem();  // X (generic proxy) -> the tensor cores (async proxy)
  }
  __syncthreads();  // X complete; every capsule read done, so the A buffers are free
  tc_fence_after();
  MPPI_TSTAMP(dbg, 2);

  if (warp == kFusedEpiWarps) {
    // ======================= MMA issuer (one tile) ==========================
    // the whole warp, MMAs/commits from one elect.sync-ed lane (mppi_mlp.cuh)
    {
      const uint32_t id32 = umma_idesc(32), id64 = umma_idesc(64), id128 = umma_idesc(128);
      const uint64_t dXH = umma_desc(sb + OFF_XH, 128, 256), dXL = umma_desc(sb + OFF_XL, 128, 256);
      const uint64_t dW0H = umma_desc(sb + OFF_W0H, 128, 256), dW0L = umma_desc(sb + OFF_W0L, 128, 256);
      const uint64_t dAH = umma_desc(sb + OFF_A, 128, 512), dAL = umma_desc(sb + OFF_A + kAHalf, 128, 512);
      const uint64_t dW1H = umma_desc(sb + OFF_W1H, 128, 4096), dW1L = umma_desc(sb + OFF_W1L, 128, 4096);
      const uint64_t dW2H = umma_desc(sb + OFF_W2H, 128, 2048), dW2L = umma_desc(sb + OFF_W2L, 128, 2048);
      mbar_wait(barW0, 0);
      MPPI_TSTAMP(pdbg, 8);
      tc_fence_after();
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {  // layer 1 as two N=128 halves
        const uint64_t wo = umma_off(128 * hf, 0, 16) >> 4;
        umma_f16_w(tmem + 128 * hf, dXH, dW0H + wo, id128, 0);
        umma_f16_w(tmem + 128 * hf, dXH, dW0L + wo, id128, 1);
        umma_f16_w(tmem + 128 * hf, dXL, dW0H + wo, id128, 1);
        umma_commit_w(barL1[hf]);
      }
      uint32_t phA = 0;  // parity bit per A buffer
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int bf = c & 1;
        mbar_wait(barA0 + 8 * bf, (phA >> bf) & 1u);
        phA ^= 1u << bf;
        if (c == 0) {
          mbar_wait(barW1, 0);
          MPPI_TSTAMP(pdbg, 9);
        }
        tc_fence_after();
        const uint64_t ao = (uint64_t)(bf * kABuf) >> 4;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint64_t aj = ao + (uint64_t)(j * 256 >> 4), wj = (uint64_t)((4 * c + 2 * j) * 128 >> 4);
          umma_f16_w(acc2, dAH + aj, dW1H + wj, id128, (c | j) ? 1u : 0u);
          umma_f16_w(acc2, dAH + aj, dW1L + wj, id128, 1);
          umma_f16_w(acc2, dAL + aj, dW1H + wj, id128, 1);
        }
        umma_commit_w(barL20 + 8 * bf);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int bf = c & 1;
        mbar_wait(barA0 + 8 * bf, (phA >> bf) & 1u);
        phA ^= 1u << bf;
        if (c == 0) {
          mbar_wait(barW2, 0);
          MPPI_TSTAMP(pdbg, 10);
        }
        tc_fence_after();
        const uint64_t ao = (uint64_t)(bf * kABuf) >> 4;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint64_t aj = ao + (uint64_t)(j * 256 >> 4), wj = (uint64_t)((4 * c + 2 * j) * 128 >> 4);
          umma_f16_w(acc3, dAH + aj, dW2H + wj, id128, (c | j) ? 1u : 0u);  // [W2 hi | W2 lo]
          umma_f16_w(acc3, dAL + aj, dW2H + wj, id64, 1);
        }
        umma_commit_w(barL30 + 8 * bf);
      }
      MPPI_TSTAMP(pdbg, 11);
    }
  } else {
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    auto publish = [&](uint32_t bar) {
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
    };
    mbar_wait(barW0, 0);  // biases live in the W0 segment
    MPPI_TSTAMP(dbg, 7);
    const float* par = reinterpret_cast<const float*>(sm + OFF_PAR);
    const float* b0 = par;
    const float* b1 = par + kMlpH0;
    const float* b2 = b1 + kMlpH1;
    const float* w3 = b2 + kMlpH2;
    const float s0 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 1];
    const float s1 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 2];
    const float s2 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 3];
    uint32_t phL2 = 0, phL3 = 0;  // parity bit per A buffer
    // ============================ layer epilogues ===========================
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int bf = c & 1;
      if ((c & 3) == 0) {
        mbar_wait(barL1[0] + 8 * (c >> 2), 0);
        tc_fence_after();
      }
      float y[kFusedCW];
      tmem_ld_cols<kFusedCW>(tmem + 32 * c + lane_base + kFusedCW * cg, y);
#pragma unroll
      for (int i = 0; i < kFusedCW; ++i) y[i] = fmaxf(fmaf(y[i], s0, b0[32 * c + kFusedCW * cg + i]), 0.f);
      if (c >= 2) {
        mbar_wait(barL20 + 8 * bf, (phL2 >> bf) & 1u);
        phL2 ^= 1u << bf;
      }
      store_cols<kFusedCW>(sm, OFF_A + bf * kABuf, OFF_A + bf * kABuf + kAHalf, row_in_tile, kFusedCW * cg, y);
      publish(barA0 + 8 * bf);
    }
    MPPI_TSTAMP(dbg, 3);
    mbar_wait(barL20, phL2 & 1u);
    mbar_wait(barL20 + 8, (phL2 >> 1) & 1u);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int bf = c & 1;
      float y[kFusedCW];
      tmem_ld_cols<kFusedCW>(acc2 + lane_base + 32 * c + kFusedCW * cg, y);
#pragma unroll
      for (int i = 0; i < kFusedCW; ++i) y[i] = fmaxf(fmaf(y[i], s1, b1[32 * c + kFusedCW * cg + i]), 0.f);
      if (c >= 2) {
        mbar_wait(barL30 + 8 * bf, (phL3 >> bf) & 1u);
        phL3 ^= 1u << bf;
      }
      store_cols<kFusedCW>(sm, OFF_A + bf * kABuf, OFF_A + bf * kABuf + kAHalf, row_in_tile, kFusedCW * cg, y);
      publish(barA0 + 8 * bf);
    }
    MPPI_TSTAMP(dbg, 4);
    mbar_wait(barL30, phL3 & 1u);
    mbar_wait(barL30 + 8, (phL3 >> 1) & 1u);
    tc_fence_after();
    MPPI_TSTAMP(dbg, 5);
    float part = 0.f;
    {
      constexpr int C3 = kMlpH2 / kFusedCG;  // layer-3 columns per warp
      float y[C3], z[C3];
      tmem_ld_cols<C3>(acc3 + lane_base + C3 * cg, y);
      tmem_ld_cols<C3>(acc3 + lane_base + 64 + C3 * cg, z);
      part = output_part<C3>(y, z, s2, b2 + C3 * cg, w3 + C3 * cg);
    }
    float* red = reinterpret_cast<float*>(sm + OFF_A);
    red[cg * 128 + row_in_tile] = part;
    fused_epi_barrier();
    if (cg == 0 && g < total && lane < a.H) {
      float o = par[kMlpH0 + kMlpH1 + 2 * kMlpH2];
#pragma unroll
      for (int k = 0; k < kFusedCG; ++k) o += red[128 * k + row_in_tile];
      out_d[(size_t)g * a.H + lane] = o;
    }
    MPPI_TSTAMP(dbg, 6);
    tc_fence_before();
  }
  __syncthreads();
  if (warp == kFusedEpiWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Staging bytes the rollout warps of one fused CTA need (must fit the A buffers).
template <typename R>
inline size_t fused_cap_bytes(const RolloutArgs<R>& a) {
  return rollout_needs_caps(a.cost) ? (size_t)kFusedParticles * a.chain.n_caps * 6 * 32 * sizeof(R) : 0;
}

template <typename R, int D>
cudaError_t launch_rollout_mlp_d(const RolloutArgs<R>& a, const unsigned char* img, float* out_d,
                                 cudaStream_t st) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(rollout_mlp_kernel<R, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kMlpSmem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  const long long total = (long long)a.B * a.N;
  const unsigned grid = (unsigned)((total + kFusedParticles - 1) / kFusedParticles);
  rollout_mlp_kernel<R, D><<<grid, kFusedThreads, kMlpSmem, st>>>(a, img, out_d);
  return cudaGetLastError();
}

}  // namespace mppi
