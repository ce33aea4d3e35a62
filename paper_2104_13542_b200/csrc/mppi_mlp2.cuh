// mppi_mlp2.cuh — learned-collision MLP, two tiles in flight per CTA,
// activations kept in tensor memory (opt-in: MPPI_MLP2=1; slower than the
// one-tile kernel as measured, see mlp_forward_auto).
//
// Same network, weights, FP16 hi/lo x3 products and accumulation order as
// mlp_tcgen05_kernel (mppi_mlp.cuh), so the outputs are bit-identical; the
// schedule differs. At scale (config 4: 61M rows) the one-tile kernel leaves
// the tensor pipe idle while its epilogue warps drain layers 2/3 of a tile and
// start layer 1 of the next (tensor pipe ~46% active). Here
//   * every layer's activations go back into TMEM in place (the epilogue warp
//     that read 16 fp32 accumulator columns overwrites them with 8 fp16-hi +
//     8 fp16-lo columns) and layers 2/3 read their A operand from TMEM
//     (tcgen05.mma ... [a_tmem]): no shared-memory activation buffers;
//   * layer 1 runs in two halves of 128 outputs through one 128-column
//     region, and layer 3 accumulates into that region once layer 2 is done,
//     so a tile needs 256 TMEM columns and two tiles fit the 512;
//   * two epilogue warp groups (8 warps each) own one tile slot each, and one
//     issuer thread polls both slots' barriers and feeds the tensor pipe from
//     whichever slot is ready — one slot's epilogue hides under the other's
//     MMAs.
// Per slot s: R1 = TMEM cols [256s, 256s+128) (layer-1 half accumulator ->
// layer-2 A operand -> layer-3 accumulator), R2 = [256s+128, 256s+256)
// (layer-2 accumulator -> layer-3 A operand).
#pragma once

#include "mppi_mlp.cuh"

namespace mppi {

constexpr uint32_t kXPart = 128 * 16 * 2;                     // X hi or lo of one tile, 4 KiB
constexpr uint32_t M2_OFF_X = kImgBytes;                      // 2 slots x (hi, lo)
constexpr uint32_t M2_OFF_RED = M2_OFF_X + 2 * 2 * kXPart;    // 2 slots x 4 partial sums x 128 rows, fp32
constexpr uint32_t M2_OFF_BAR = M2_OFF_RED + 2 * 4 * 128 * 4;
// per slot: X L1a L2a L1b L2 L3, then one "A ready" barrier per layer-2
// input chunk (8) and per layer-3 input chunk (4). The epilogue runs ahead of
// the issuer within a layer (no buffer to recycle), so every chunk gets its own
// barrier: each completes once per tile and a parity can never be skipped.
constexpr int kM2SlotBars = 6 + 8 + 4;
constexpr uint32_t M2_OFF_TMEMPTR = M2_OFF_BAR + (3 + 2 * kM2SlotBars) * 8;
constexpr uint32_t kMlp2Smem = M2_OFF_TMEMPTR + 16;
constexpr int kM2EpiWarps = 8;                                // per slot
constexpr int kM2Threads = (2 * kM2EpiWarps + 1) * 32;        // 544
static_assert(kMlp2Smem <= 232448, "two-slot MLP does not fit shared memory");
enum { SB_X = 0, SB_L1A, SB_L2A, SB_L1B, SB_L2, SB_L3, SB_A1 = 6, SB_A2 = 14 };

// A operand from tensor memory (kind::f16, K-major, M = 128)
__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 16 fp32 activations of one row -> 8 packed fp16-hi then 8 packed fp16-lo
// columns (element 2i in the low half), written over the same 16 columns.
__device__ __forceinline__ void tmem_store_split16(uint32_t taddr, const float* y) {
  uint32_t v[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const __half2 hh = __floats2half2_rn(y[2 * i], y[2 * i + 1]);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(y[2 * i] - hf.x, y[2 * i + 1] - hf.y);
    v[i] = *reinterpret_cast<const uint32_t*>(&hh);
    v[8 + i] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  tmem_st16(taddr, v);
}

__device__ __forceinline__ void slot_barrier(int s) {  // the 256 epilogue threads of one slot
  asm volatile("bar.sync %0, %1;" ::"r"(1 + s), "n"(kM2EpiWarps * 32) : "memory");
}

static __global__ void __launch_bounds__(kM2Threads, 1)
    mlp2_tcgen05_kernel(const float* __restrict__ x, long long M, const unsigned char* __restrict__ img,
                        float* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char mlp2_smem[];
  unsigned char* sm = mlp2_smem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sb = smem_u32(sm);
  const uint32_t barW0 = sb + M2_OFF_BAR, barW1 = barW0 + 8, barW2 = barW0 + 16;
  auto sbar = [&](int s, int k) -> uint32_t { return sb + M2_OFF_BAR + 24 + (uint32_t)(s * kM2SlotBars + k) * 8; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + M2_OFF_TMEMPTR);
  const int issuer_warp = 2 * kM2EpiWarps;

  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(barW0 + 8 * i, 1);
    for (int s = 0; s < 2; ++s)
      for (int k = 0; k < kM2SlotBars; ++k)
        mbar_init(sbar(s, k), (k == SB_X || k >= SB_A1) ? kM2EpiWarps : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
  }
  if (warp == issuer_warp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const long long ntiles = (M + 127) / 128;
  const long long G = gridDim.x;

  if (warp == issuer_warp) {
    // ============================== issuer ==================================
    if (lane == 0) {
      mbar_expect_tx(barW0, kSeg0);
      bulk_g2s(sb + 0, img, kSeg0, barW0);
      mbar_expect_tx(barW1, kSeg1);
      for (uint32_t o = 0; o < kSeg1; o += 32768)
        bulk_g2s(sb + OFF_W1H + o, img + OFF_W1H + o, min(32768u, kSeg1 - o), barW1);
      mbar_expect_tx(barW2, kSeg2);
      bulk_g2s(sb + OFF_W2H, img + OFF_W2H, kSeg2, barW2);
      const uint32_t id32 = umma_idesc(32), id64 = umma_idesc(64), id128 = umma_idesc(128);
      const uint64_t dW0H = umma_desc(sb + OFF_W0H, 128, 256), dW0L = umma_desc(sb + OFF_W0L, 128, 256);
      const uint64_t dW1H = umma_desc(sb + OFF_W1H, 128, 4096), dW1L = umma_desc(sb + OFF_W1L, 128, 4096);
      const uint64_t dW2H = umma_desc(sb + OFF_W2H, 128, 2048), dW2L = umma_desc(sb + OFF_W2L, 128, 2048);
      bool w0 = false, w1 = false, w2 = false;
      long long tile[2] = {blockIdx.x, blockIdx.x + G};
      int stage[2] = {0, 0}, chunk[2] = {0, 0};
      // every slot barrier completes once per tile: its parity is the slot's tile parity
      uint32_t ph[2] = {0, 0};
      auto ready = [&](int s, int k) { return mbar_test(sbar(s, k), ph[s]); };
      while (tile[0] < ntiles || tile[1] < ntiles) {
#pragma unroll  // compile-time slot index: the per-slot state stays in registers
        for (int s = 0; s < 2; ++s) {
          if (tile[s] >= ntiles) continue;
          const uint32_t R1 = tmem + 256 * s, R2 = R1 + 128;
          const uint64_t dXH = umma_desc(sb + M2_OFF_X + s * 2 * kXPart, 128, 256);
          const uint64_t dXL = umma_desc(sb + M2_OFF_X + s * 2 * kXPart + kXPart, 128, 256);
          switch (stage[s]) {
            case 0:    // layer 1, outputs 0-127, once the tile's X is in smem
            case 2: {  // layer 1, outputs 128-255, once layer 2 has consumed the first half
              const int k = stage[s] == 0 ? SB_X : SB_L2A;
              if (!ready(s, k)) break;
              if (!w0) {
                mbar_wait(barW0, 0);
                w0 = true;
              }
              tc_fence_after();
              const int h = stage[s] == 0 ? 0 : 1;
              {
                const uint64_t wo = umma_off(128 * h, 0, 16) >> 4;
                umma_f16(R1, dXH, dW0H + wo, id128, 0);
                umma_f16(R1, dXH, dW0L + wo, id128, 1);
                umma_f16(R1, dXL, dW0H + wo, id128, 1);
              }
              umma_commit(sbar(s, h == 0 ? SB_L1A : SB_L1B));
              stage[s] = 1;
              break;
            }
            case 1: {  // layer 2, K chunk c (32 of the 256 inputs), A from R1
              if (!ready(s, SB_A1 + chunk[s])) break;
              if (!w1) {
                mbar_wait(barW1, 0);
                w1 = true;
              }
              tc_fence_after();
              const int c = chunk[s], cl = c & 3;
#pragma unroll
              for (int g = 0; g < 2; ++g) {
                const uint32_t ah = R1 + 32 * cl + 16 * g, al = ah + 8;
                const uint64_t wj = (uint64_t)((4 * c + 2 * g) * 128 >> 4);
                umma_f16_ts(R2, ah, dW1H + wj, id128, (c | g) ? 1u : 0u);
                umma_f16_ts(R2, ah, dW1L + wj, id128, 1);
                umma_f16_ts(R2, al, dW1H + wj, id128, 1);
              }
              if (c == 3) {
                umma_commit(sbar(s, SB_L2A));
                stage[s] = 2;
              } else if (c == 7) {
                umma_commit(sbar(s, SB_L2));
                stage[s] = 3;
              }
              chunk[s] = c + 1;
              break;
            }
            case 3: {  // layer 3 accumulates into R1 once layer 2 (which read R1) is done
              if (!ready(s, SB_L2)) break;
              stage[s] = 4;
              chunk[s] = 0;
              break;
            }
            case 4: {  // layer 3, K chunk c (32 of the 128 inputs), A from R2
              if (!ready(s, SB_A2 + chunk[s])) break;
              if (!w2) {
                mbar_wait(barW2, 0);
                w2 = true;
              }
              tc_fence_after();
              const int c = chunk[s];
#pragma unroll
              for (int g = 0; g < 2; ++g) {
                const uint32_t ah = R2 + 32 * c + 16 * g, al = ah + 8;
                const uint64_t wj = (uint64_t)((4 * c + 2 * g) * 128 >> 4);
                umma_f16_ts(R1, ah, dW2H + wj, id128, (c | g) ? 1u : 0u);  // [W2 hi | W2 lo]
                umma_f16_ts(R1, al, dW2H + wj, id64, 1);
              }
              if (c == 3) {
                umma_commit(sbar(s, SB_L3));
                stage[s] = 0;
                chunk[s] = 0;
                tile[s] += 2 * G;
                ph[s] ^= 1u;
              } else {
                chunk[s] = c + 1;
              }
              break;
            }
          }
        }
      }
      // drain the weight copies of a CTA that had no tile
      if (!w0) mbar_wait(barW0, 0);
      if (!w1) mbar_wait(barW1, 0);
      if (!w2) mbar_wait(barW2, 0);
    }
  } else {
    // ============================ epilogue groups ===========================
    const int s = warp / kM2EpiWarps, wl = warp % kM2EpiWarps;
    const int quad = warp & 3, cg = wl >> 2;
    const int row_in_tile = quad * 32 + lane;
    const int gt = tid - s * kM2EpiWarps * 32;  // 0..255 within the slot group
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t R1 = tmem + 256 * s + lane_base, R2 = R1 + 128;
    const uint32_t offXH = M2_OFF_X + s * 2 * kXPart, offXL = offXH + kXPart;
    float* red = reinterpret_cast<float*>(sm + M2_OFF_RED) + s * 4 * 128;
    const float* par = reinterpret_cast<const float*>(sm + OFF_PAR);
    const float* b0 = par;
    const float* b1 = par + kMlpH0;
    const float* b2 = b1 + kMlpH1;
    const float* w3 = b2 + kMlpH2;
    auto arrive = [&](int k) {  // TMEM / smem writes of this warp -> the issuer
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(sbar(s, k));
    };
    bool have_bias = false;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, b3 = 0.f;
    uint32_t par_t = 0;  // parity of this slot's once-per-tile barriers
    auto load_x = [&](long long tile, float* xv) {  // thread = (row, half of the 16 encodings)
      const long long r = tile * 128 + (gt & 127);
      if (tile < ntiles && r < M) {
        const float4* src = reinterpret_cast<const float4*>(x + r * 16 + (gt >> 7) * 8);
        const float4 f0 = __ldg(src), f1 = __ldg(src + 1);
        xv[0] = f0.x; xv[1] = f0.y; xv[2] = f0.z; xv[3] = f0.w;
        xv[4] = f1.x; xv[5] = f1.y; xv[6] = f1.z; xv[7] = f1.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = 0.f;
      }
    };
    float xv[8];
    load_x(blockIdx.x + s * G, xv);
    for (long long tile = blockIdx.x + s * G; tile < ntiles; tile += 2 * G, par_t ^= 1u) {
      // ---- X of this tile into the slot's smem; the next tile's X is loaded
      // into registers now and lands while this tile runs
      store_split8(sm, offXH, offXL, umma_off(gt & 127, (gt >> 7) * 8, 16), xv);
      fence_async_smem();
      arrive(SB_X);
      load_x(tile + 2 * G, xv);
      if (!have_bias) {
        mbar_wait(barW0, 0);  // biases and scales live in the W0 segment
        s0 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 1];
        s1 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 2];
        s2 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 3];
        b3 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2];
        have_bias = true;
      }
      // ---- layer-1 epilogue, two halves of 4 chunks, in place in R1
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        mbar_wait(sbar(s, h == 0 ? SB_L1A : SB_L1B), par_t);
        tc_fence_after();
#pragma unroll 1
        for (int cl = 0; cl < 4; ++cl) {
          const int c = 4 * h + cl;
          float y[16];
          tmem_ld16(R1 + 32 * cl + 16 * cg, y);
#pragma unroll
          for (int i = 0; i < 16; ++i) y[i] = fmaxf(fmaf(y[i], s0, b0[32 * c + 16 * cg + i]), 0.f);
          tmem_store_split16(R1 + 32 * cl + 16 * cg, y);
          arrive(SB_A1 + c);
        }
      }
      // ---- layer-2 epilogue, in place in R2
      mbar_wait(sbar(s, SB_L2), par_t);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float y[16];
        tmem_ld16(R2 + 32 * c + 16 * cg, y);
#pragma unroll
        for (int i = 0; i < 16; ++i) y[i] = fmaxf(fmaf(y[i], s1, b1[32 * c + 16 * cg + i]), 0.f);
        tmem_store_split16(R2 + 32 * c + 16 * cg, y);
        arrive(SB_A2 + c);
      }
      // ---- layer-3 epilogue and the 64 -> 1 output layer
      mbar_wait(sbar(s, SB_L3), par_t);
      tc_fence_after();
      // four 16-column partial sums (A_hi W_hi + A_lo W_hi in cols 0-63, A_hi W_lo
      // in 64-127), combined in the one-tile kernel's order
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float y[16], z[16], part = 0.f;
        tmem_ld16(R1 + 32 * cg + 16 * q, y);
        tmem_ld16(R1 + 64 + 32 * cg + 16 * q, z);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = 32 * cg + 16 * q + i;
          part = fmaf(fmaxf(fmaf(y[i] + z[i], s2, b2[j]), 0.f), w3[j], part);
        }
        red[(2 * cg + q) * 128 + row_in_tile] = part;
      }
      tc_fence_before();
      slot_barrier(s);
      if (cg == 0) {
        const long long row = tile * 128 + row_in_tile;
        if (row < M)
          out[row] = b3 + red[row_in_tile] + red[128 + row_in_tile] + red[256 + row_in_tile] + red[384 + row_in_tile];
      }
      slot_barrier(s);  // red is rewritten by this slot's next tile
    }
  }
  __syncthreads();
  if (warp == issuer_warp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

inline cudaError_t mlp2_forward(const MlpWeights& m, const float* x, long long rows, float* out, cudaStream_t st) {
  static bool attr_set[64] = {};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(mlp2_tcgen05_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kMlp2Smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long tiles = (rows + 127) / 128;
  const long long want = (tiles + 1) / 2;  // two tiles per CTA at a time
  const unsigned grid = (unsigned)(want < sms ? want : sms);
  mlp2_tcgen05_kernel<<<grid, kM2Threads, kMlp2Smem, st>>>(x, rows, m.img, out);
  return cudaGetLastError();
}

}  // namespace mppi

namespace mppi {

// The one-tile kernel (mlp_tcgen05_kernel) everywhere; the two-slot kernel is
// opt-in (MPPI_MLP2=1) — bit-identical outputs, but measured SLOWER at config
// 4 (MLP 21.4 ms vs 16.2 ms, tensor pipe 34% vs 46% active): each slot's
// layer chain (L1 halves -> L2 -> L3 with in-place TMEM conversions by 8
// warps) is long enough that two slots do not keep the pipe busier than the
// one-tile kernel's 16-warp epilogue with smem double buffering.
inline cudaError_t mlp_forward_auto(const MlpWeights& m, const float* x, long long rows, float* out,
                                    cudaStream_t st, unsigned long long* dbg = nullptr) {
  const char* env = getenv("MPPI_MLP2");
  if (env && env[0] == '1') return mlp2_forward(m, x, rows, out, st);
  return mlp_forward(m, x, rows, out, st, dbg);
}

}  // namespace mppi
