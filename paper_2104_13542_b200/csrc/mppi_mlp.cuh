// mppi_mlp.cuh — learned self-collision MLP on the 5th-gen tensor cores.
//
// Reference: surrogate.py:42-52 (+ posenc :24-28): x = [sin q, cos q] (2d=14,
// padded to 16) -> 256 -> 128 -> 64 -> 1, ReLU between layers, float64 on
// the CPU. Here: one 128-row tile per CTA iteration, all three hidden layers
// on tcgen05.mma (kind::f16, FP32 accumulation in TMEM), the 64 -> 1 output
// layer fused into the last epilogue on the CUDA cores.
//
// Precision: every operand is split into an FP16 pair
// hi + lo (lo = fp16(x - hi)), and each product is computed as
// A_hi B_hi + A_hi B_lo + A_lo B_hi (three MMAs into the same accumulator):
// ~22 significant bits, within ~1e-6 m of the float64 reference distance,
// where a single bf16/tf32 pass is not parity safe. Weights are pre-scaled by
// a per-layer power of two so their lo parts stay clear of FP16 subnormals;
// the epilogue undoes the scale exactly.
//
// Data movement: the whole weight image (W0..W2 hi/lo in the UMMA canonical
// K-major no-swizzle layout, 176 KiB, + fp32 biases) is copied global -> smem
// once per CTA with cp.async.bulk (TMA bulk engine, three mbarriers so layer 1
// starts while W1/W2 are still in flight). The CTA is persistent over tiles.
//
// Pipeline per tile (one elected thread issues all MMAs; 128 threads = 128
// TMEM lanes run the epilogues, thread t owns row t of the tile):
//   L1 chunk c (64 of 256 outputs) -> TMEM acc1[c%2] ; epilogue (bias, ReLU,
//   split) -> smem A ; L2 K-chunk c accumulates into acc2 ; L1 chunk c+2 is
//   issued right behind it. Then layer 2's output goes back through smem in
//   two 64-wide K-chunks into L3 (acc3), and the final epilogue does the
//   64 -> 1 dot product.
#pragma once

#include <cuda_fp16.h>

#include "mppi_common.cuh"
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

namespace mppi {

constexpr int kMlpH0 = 256, kMlpH1 = 128, kMlpH2 = 64, kMlpIn = 16;

inline size_t mlp_padded_rows(size_t rows) { return (rows + 127) / 128 * 128; }

// ---- shared-memory image (byte offsets); identical in global memory so one
// bulk copy per segment lands every operand in place.
constexpr uint32_t kW0Bytes = kMlpH0 * kMlpIn * 2;   // 8 KiB per hi/lo
constexpr uint32_t kW1Bytes = kMlpH1 * kMlpH0 * 2;   // 64 KiB
constexpr uint32_t kW2Bytes = kMlpH2 * kMlpH1 * 2;   // 16 KiB
constexpr uint32_t OFF_W0H = 0;
constexpr uint32_t OFF_W0L = OFF_W0H + kW0Bytes;
constexpr uint32_t OFF_PAR = OFF_W0L + kW0Bytes;                  // fp32 params
constexpr uint32_t kParFloats = kMlpH0 + kMlpH1 + kMlpH2 + kMlpH2 + 4;  // b0 b1 b2 w3 | b3 s0 s1 s2
constexpr uint32_t kParBytes = kParFloats * 4;                    // 2064
constexpr uint32_t OFF_W1H = OFF_PAR + ((kParBytes + 127) / 128) * 128;
constexpr uint32_t OFF_W1L = OFF_W1H + kW1Bytes;
constexpr uint32_t OFF_W2H = OFF_W1L + kW1Bytes;
constexpr uint32_t OFF_W2L = OFF_W2H + kW2Bytes;
constexpr uint32_t kImgBytes = OFF_W2L + kW2Bytes;
constexpr uint32_t kSeg0 = OFF_W1H;                 // W0 + params
constexpr uint32_t kSeg1 = OFF_W2H - OFF_W1H;       // W1
constexpr uint32_t kSeg2 = kImgBytes - OFF_W2H;     // W2
constexpr uint32_t OFF_XH = kImgBytes;              // X tile 128 x 16 fp16
constexpr uint32_t OFF_XL = OFF_XH + 128 * 16 * 2;
// activations: two 32-wide K-chunk buffers (double buffering), each 128 x 32
// fp16 hi followed by 128 x 32 fp16 lo
constexpr uint32_t kAChunkK = 32;
constexpr uint32_t kAHalf = 128 * kAChunkK * 2;     // 8 KiB
constexpr uint32_t kABuf = 2 * kAHalf;              // hi + lo = 16 KiB
constexpr uint32_t OFF_A = OFF_XL + 128 * 16 * 2;
constexpr uint32_t OFF_BAR = OFF_A + 2 * kABuf;     // 16 mbarriers
constexpr uint32_t OFF_TMEMPTR = OFF_BAR + 16 * 8;  // 12 used
constexpr uint32_t OFF_RED = OFF_TMEMPTR + 16;      // output-layer partial sums, 4 x 128 fp32
constexpr uint32_t kMlpSmem = OFF_RED + 4 * 128 * 4;

static_assert(OFF_W2L == OFF_W2H + 64 * kMlpH1 * 2, "layer-3 N=128 MMA reads W2 hi and lo as one operand");
static_assert(kMlpSmem <= 232448, "MLP tile does not fit the 227 KiB of shared memory");
static_assert(kSeg0 % 16 == 0 && kSeg1 % 16 == 0 && kSeg2 % 16 == 0, "bulk copy sizes");

// byte offset of element (row, k) of a K-major, no-swizzle UMMA operand with
// K columns: 8x8 core matrices (8 rows x 16 B), K-chunks adjacent (LBO = 128 B),
// 8-row groups K*16 B apart (SBO).
__host__ __device__ constexpr uint32_t umma_off(uint32_t row, uint32_t k, uint32_t K) {
  return (row >> 3) * (K * 16) + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2;
}

struct MlpWeights {
  int in_dim = 0;
  unsigned char* img = nullptr;  // kImgBytes, device
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(phase)
      : "memory");
  return ok != 0;
}

// non-blocking probe of a phase (the two-slot issuer polls several barriers)
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(phase)
      : "memory");
  return ok != 0;
}

#ifdef MPPI_WATCHDOG
// development builds: a barrier that never completes traps instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  for (long long i = 0; !mbar_try(bar, phase); ++i)
    if (i > (1ll << 24)) __trap();
}
#else
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
#endif

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}

// kind::f16 instruction descriptor: F16 x F16 -> F32, both K-major, M=128.
__host__ __device__ constexpr uint32_t umma_idesc(uint32_t N) {
  return (1u << 4) | ((N >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Split 16 fp32 activations of one row into fp16 hi/lo (packed cvt.rn.f16x2)
// and store them as two 16-byte core-matrix rows each (k0 multiple of 16) of a
// K-wide K-major operand.
__device__ __forceinline__ void store_split16(unsigned char* sm, uint32_t off_h, uint32_t off_l,
                                              uint32_t row, uint32_t k0, uint32_t K, const float* y) {
  uint32_t h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const __half2 hh = __floats2half2_rn(y[2 * i], y[2 * i + 1]);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(y[2 * i] - hf.x, y[2 * i + 1] - hf.y);
    h[i] = *reinterpret_cast<const uint32_t*>(&hh);
    l[i] = *reinterpret_cast<const uint32_t*>(&ll);
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const uint32_t o = umma_off(row, k0 + 8 * c, K);
    *reinterpret_cast<uint4*>(sm + off_h + o) = make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
    *reinterpret_cast<uint4*>(sm + off_l + o) = make_uint4(l[4 * c], l[4 * c + 1], l[4 * c + 2], l[4 * c + 3]);
  }
}

// 8 fp32 -> one hi and one lo 16-byte core-matrix row.
__device__ __forceinline__ void store_split8(unsigned char* sm, uint32_t off_h, uint32_t off_l, uint32_t o,
                                             const float* y) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 hh = __floats2half2_rn(y[2 * i], y[2 * i + 1]);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(y[2 * i] - hf.x, y[2 * i + 1] - hf.y);
    h[i] = *reinterpret_cast<const uint32_t*>(&hh);
    l[i] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  *reinterpret_cast<uint4*>(sm + off_h + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(sm + off_l + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

// ------------------------------------------------------------------ the kernel
// Warp-specialised: warps 0-15 are the epilogue (warp w serves TMEM lane
// quadrant q = w % 4, i.e. rows 32q..32q+31 of the tile, and column group
// cg = w / 4: 8 of every 32 accumulator columns); warp 16 is the producer:
// it issues the weight TMA and every tcgen05.mma. Activations move through two
// 32-wide smem buffers; the hand-off is mbarrier-only:
//   epilogue --aready[b] (16 arrivals)--> issuer --tcgen05.commit--> epilogue
constexpr int kMlpEpiWarps = 16;
constexpr int kMlpThreads = (kMlpEpiWarps + 1) * 32;

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void epi_barrier() {  // named barrier over the 512 epilogue threads
  asm volatile("bar.sync 1, %0;" ::"n"(kMlpEpiWarps * 32) : "memory");
}

// x: (M_pad,16) fp32 positional encodings; out: (M) fp32 distances.
// 88 registers: 544 x 88 + a 128-thread rollout CTA (128 registers) fit one
// SM's 64K register file, so with programmatic dependent launch the MLP CTAs
// become resident next to the rollout and load their weights under it.
static __global__ void __maxnreg__(88)
    mlp_tcgen05_kernel(const float* __restrict__ x, long long M, const unsigned char* __restrict__ img,
                       float* __restrict__ out, int early, unsigned long long* dbg_base) {
  extern __shared__ __align__(1024) unsigned char mlp_smem[];
  unsigned char* sm = mlp_smem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // debug stamps (MPPI_DEBUG_TIMERS): 0 start, 1 X stored, 2 W0, 3 L1 epi, 4 L2 epi, 5 L3, 6 end
  unsigned long long* dbg = (dbg_base != nullptr && tid == 0 && blockIdx.x < 128) ? dbg_base + 16 * blockIdx.x : nullptr;
  MPPI_TSTAMP(dbg, 0);
  const uint32_t sb = smem_u32(sm);
  // barriers: 0-2 weights, 3-4 L1 done (per acc1 buffer), 5-6 L2 done (per A
  // buffer), 7-8 L3 done (per A buffer), 9-10 A ready (per A buffer), 11 X ready
  const uint32_t barW0 = sb + OFF_BAR, barW1 = barW0 + 8, barW2 = barW0 + 16;
  // barrier pairs 8 bytes apart, [0] and [1] per buffer
  const uint32_t barL10 = barW0 + 24, barL20 = barW0 + 40, barL30 = barW0 + 56, barA0 = barW0 + 72;
  const uint32_t barX = barW0 + 88;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_TMEMPTR);

  if (tid == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(barW0 + 8 * i, 1);
    mbar_init(barA0, kMlpEpiWarps);
    mbar_init(barA0 + 8, kMlpEpiWarps);
    mbar_init(barX, kMlpEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
  }
  if (warp == 0) {  // TMEM: acc1 8 x 32 (all of layer 1) | acc2 (128) | acc3 (2 x 64) -> all 512 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc2 = tmem + 256, acc3 = tmem + 384;  // acc1 chunk c at tmem + 32c
  const long long ntiles = (M + 127) / 128;

  if (warp == kMlpEpiWarps) {
    // ======================= producer / MMA issuer ==========================
    if (lane == 0) {
      mbar_expect_tx(barW0, kSeg0);
      bulk_g2s(sb + 0, img, kSeg0, barW0);
      mbar_expect_tx(barW1, kSeg1);
      for (uint32_t o = 0; o < kSeg1; o += 32768)
        bulk_g2s(sb + OFF_W1H + o, img + OFF_W1H + o, min(32768u, kSeg1 - o), barW1);
      mbar_expect_tx(barW2, kSeg2);
      bulk_g2s(sb + OFF_W2H, img + OFF_W2H, kSeg2, barW2);
      const uint32_t id32 = umma_idesc(32), id64 = umma_idesc(64), id128 = umma_idesc(128);
      // descriptors are built once; per-chunk operands differ only in the
      // start-address field (bits 0-13, 16-byte units, no carry: smem < 256 KiB)
      const uint64_t dXH = umma_desc(sb + OFF_XH, 128, 256), dXL = umma_desc(sb + OFF_XL, 128, 256);
      const uint64_t dW0H = umma_desc(sb + OFF_W0H, 128, 256), dW0L = umma_desc(sb + OFF_W0L, 128, 256);
      const uint64_t dAH = umma_desc(sb + OFF_A, 128, 512), dAL = umma_desc(sb + OFF_A + kAHalf, 128, 512);
      const uint64_t dW1H = umma_desc(sb + OFF_W1H, 128, 4096), dW1L = umma_desc(sb + OFF_W1L, 128, 4096);
      const uint64_t dW2H = umma_desc(sb + OFF_W2H, 128, 2048), dW2L = umma_desc(sb + OFF_W2L, 128, 2048);
      pdl_wait();  // sleep (rather than spin on barX) while the rollout still runs
      auto issue_l1_all = [&]() {  // the whole of layer 1: two halves of N=128, one commit each
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {  // (N=128 per instruction: small-N MMAs under-fill the tensor pipe)
          const uint64_t wo = umma_off(128 * hf, 0, 16) >> 4;
          umma_f16(tmem + 128 * hf, dXH, dW0H + wo, id128, 0);
          umma_f16(tmem + 128 * hf, dXH, dW0L + wo, id128, 1);
          umma_f16(tmem + 128 * hf, dXL, dW0H + wo, id128, 1);
          umma_commit(barL10 + 8 * hf);
        }
      };
      uint32_t phA = 0, phX = 0;  // parity bits
      bool first = true;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const bool has_next = tile + gridDim.x < ntiles;
        if (first) {
          mbar_wait(barX, phX);
          phX ^= 1;
          mbar_wait(barW0, 0);
          tc_fence_after();
          issue_l1_all();
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int bf = c & 1;
          mbar_wait(barA0 + 8 * bf, (phA >> bf) & 1u);
          phA ^= 1u << bf;
          if (first && c == 0) mbar_wait(barW1, 0);
          tc_fence_after();
          const uint64_t ao = (uint64_t)(bf * kABuf) >> 4;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint64_t aj = ao + (uint64_t)(j * 256 >> 4), wj = (uint64_t)((4 * c + 2 * j) * 128 >> 4);
            umma_f16(acc2, dAH + aj, dW1H + wj, id128, (c | j) ? 1u : 0u);
            umma_f16(acc2, dAH + aj, dW1L + wj, id128, 1);
            umma_f16(acc2, dAL + aj, dW1H + wj, id128, 1);
          }
          umma_commit(barL20 + 8 * bf);
          if (c == 7 && has_next) {  // every acc1 chunk consumed and the next X in smem
            mbar_wait(barX, phX);
            phX ^= 1;
            tc_fence_after();
            issue_l1_all();  // runs behind this tile's layer 2, under its layer-2/3 epilogues
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int bf = c & 1;
          mbar_wait(barA0 + 8 * bf, (phA >> bf) & 1u);
          phA ^= 1u << bf;
          if (first && c == 0) mbar_wait(barW2, 0);
          tc_fence_after();
          const uint64_t ao = (uint64_t)(bf * kABuf) >> 4;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint64_t aj = ao + (uint64_t)(j * 256 >> 4), wj = (uint64_t)((4 * c + 2 * j) * 128 >> 4);
            // W2 hi and lo are adjacent 64-row operands: one N=128 MMA gives
            // A_hi W_hi (cols 0-63) and A_hi W_lo (cols 64-127); A_lo W_hi adds to 0-63
            umma_f16(acc3, dAH + aj, dW2H + wj, id128, (c | j) ? 1u : 0u);
            umma_f16(acc3, dAL + aj, dW2H + wj, id64, 1);
          }
          umma_commit(barL30 + 8 * bf);
        }
        first = false;
      }
      if (first) {  // no tile for this CTA: drain the weight copies before exit
        mbar_wait(barW0, 0);
        mbar_wait(barW1, 0);
        mbar_wait(barW2, 0);
      }
    }
  } else {
    // ============================ epilogue warps ============================
    const int quad = warp & 3, cg = warp >> 2;
    const int row_in_tile = quad * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    float* red = reinterpret_cast<float*>(sm + OFF_RED);
    const float* par = reinterpret_cast<const float*>(sm + OFF_PAR);
    const float* b0 = par;
    const float* b1 = par + kMlpH0;
    const float* b2 = b1 + kMlpH1;
    const float* w3 = b2 + kMlpH2;
    uint32_t phL1 = 0, phL2 = 0, phL3 = 0;  // parity bits per buffer
    // (chunk loops fully unrolled: rolling them shrinks the cold-L2 code
    // fetch but costs 25% of the steady-state tile rate at scale)
    auto load_x = [&](long long tile, float* xv) {  // threads < 256: row tid % 128, 8 of 16 columns
      const long long r = tile * 128 + (tid & 127);
      if (tid < 256 && r < M) {
        const float4* src = reinterpret_cast<const float4*>(x + r * 16 + (tid >> 7) * 8);
        const float4 f0 = __ldg(src), f1 = __ldg(src + 1);
        xv[0] = f0.x; xv[1] = f0.y; xv[2] = f0.z; xv[3] = f0.w;
        xv[4] = f1.x; xv[5] = f1.y; xv[6] = f1.z; xv[7] = f1.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = 0.f;
      }
    };
    auto publish = [&](uint32_t bar) {  // generic-proxy smem writes -> async proxy, then arrive
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
    };
    float xnext[8];
    long long tile = blockIdx.x;
    if (early) pdl_trigger();
    pdl_wait();  // the rollout's positional encodings are complete past this point
    if (tile < ntiles) {
      load_x(tile, xnext);
      if (tid < 256) store_split8(sm, OFF_XH, OFF_XL, umma_off(tid & 127, (tid >> 7) * 8, 16), xnext);
      publish(barX);
      MPPI_TSTAMP(dbg, 1);
      mbar_wait(barW0, 0);  // biases live in the W0 segment
      MPPI_TSTAMP(dbg, 2);
    }
    const float s0 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 1];
    const float s1 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 2];
    const float s2 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 3];
    // Layer-1 epilogue of tile t (8 chunks into the two A buffers). `after_l3`:
    // the previous tile's layer 3 last read buffers 0/1 (its chunks 2/3), so
    // chunks 0/1 wait for those MMAs; also stages the X of tile t + G.
    auto epilogue_l1 = [&](long long t, bool after_l3) {
      const bool nxt = t + gridDim.x < ntiles;
      if (nxt) load_x(t + gridDim.x, xnext);  // in flight during layer 1
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int bf = c & 1;
        if ((c & 3) == 0) {  // layer-1 chunks 0-3 and 4-7 complete on separate barriers
          const int hb = c >> 2;
          mbar_wait(barL10 + 8 * hb, (phL1 >> hb) & 1u);
          phL1 ^= 1u << hb;
          tc_fence_after();
        }
        float y[8];
        tmem_ld8(tmem + 32 * c + lane_base + 8 * cg, y);
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = fmaxf(fmaf(y[i], s0, b0[32 * c + 8 * cg + i]), 0.f);
        if (c >= 2) {  // A[bf] was last read by the layer-2 MMAs of chunk c-2
          mbar_wait(barL20 + 8 * bf, (phL2 >> bf) & 1u);
          phL2 ^= 1u << bf;
        } else if (after_l3) {  // ... or by the previous tile's layer-3 chunk 2 + c
          mbar_wait(barL30 + 8 * bf, (phL3 >> bf) & 1u);
          phL3 ^= 1u << bf;
        }
        store_split8(sm, OFF_A + bf * kABuf, OFF_A + bf * kABuf + kAHalf,
                     umma_off(row_in_tile, 8 * cg, kAChunkK), y);
        publish(barA0 + 8 * bf);
        if (c == 7 && nxt) {  // every layer-1 MMA of this tile is complete: reuse X
          if (tid < 256) store_split8(sm, OFF_XH, OFF_XL, umma_off(tid & 127, (tid >> 7) * 8, 16), xnext);
          publish(barX);
        }
      }
    };
    // Per tile: layer-2 epilogue, then the NEXT tile's layer-1 epilogue, then
    // this tile's output layer. The next tile's layer 2 can start as soon as
    // this tile's layer 3 is done, instead of after the output layer too (the
    // output layer reads acc3, which only the next tile's layer 3 rewrites).
    if (tile < ntiles) epilogue_l1(tile, false);
#ifdef MPPI_DEBUG_TIMERS
    unsigned long long ts3 = 0, ts4 = 0, ts5 = 0, ts6 = 0, sum_a = 0, sum_b = 0, sum_c = 0, ntile = 0;
#define MLP_T(v) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v))
#else
#define MLP_T(v)
#endif
    for (; tile < ntiles; tile += gridDim.x) {
      const bool has_next = tile + gridDim.x < ntiles;
      MPPI_TSTAMP(dbg, 3);
      MLP_T(ts3);
      mbar_wait(barL20, phL2 & 1u);  // chunk 6's and chunk 7's layer-2 MMAs: all of layer 2
      mbar_wait(barL20 + 8, (phL2 >> 1) & 1u);
      phL2 ^= 3u;
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int bf = c & 1;
        float y[8];
        tmem_ld8(acc2 + lane_base + 32 * c + 8 * cg, y);
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = fmaxf(fmaf(y[i], s1, b1[32 * c + 8 * cg + i]), 0.f);
        if (c >= 2) {
          mbar_wait(barL30 + 8 * bf, (phL3 >> bf) & 1u);
          phL3 ^= 1u << bf;
        }
        store_split8(sm, OFF_A + bf * kABuf, OFF_A + bf * kABuf + kAHalf,
                     umma_off(row_in_tile, 8 * cg, kAChunkK), y);
        publish(barA0 + 8 * bf);
      }
      MPPI_TSTAMP(dbg, 4);
      MLP_T(ts4);
      if (has_next) {
        epilogue_l1(tile + gridDim.x, true);  // also waits for this tile's layer-3 chunks 2, 3
      } else {
        mbar_wait(barL30, phL3 & 1u);
        mbar_wait(barL30 + 8, (phL3 >> 1) & 1u);
        phL3 ^= 3u;
      }
      MPPI_TSTAMP(dbg, 5);
      MLP_T(ts5);
      tc_fence_after();
      float part = 0.f;
      {
        float y[16], z[16];
        tmem_ld16(acc3 + lane_base + 16 * cg, y);       // A_hi W_hi + A_lo W_hi
        tmem_ld16(acc3 + lane_base + 64 + 16 * cg, z);  // A_hi W_lo
#pragma unroll
        for (int i = 0; i < 16; ++i)
          part = fmaf(fmaxf(fmaf(y[i] + z[i], s2, b2[16 * cg + i]), 0.f), w3[16 * cg + i], part);
      }
      red[cg * 128 + row_in_tile] = part;
      epi_barrier();
      if (cg == 0) {
        const long long row = tile * 128 + row_in_tile;
        const float o = par[kMlpH0 + kMlpH1 + 2 * kMlpH2] + red[row_in_tile] + red[128 + row_in_tile] +
                        red[256 + row_in_tile] + red[384 + row_in_tile];
        if (row < M) out[row] = o;
      }
      tc_fence_before();
      epi_barrier();  // red is rewritten by the next tile's output layer
      MPPI_TSTAMP(dbg, 6);
#ifdef MPPI_DEBUG_TIMERS
      MLP_T(ts6);
      sum_a += ts4 - ts3;  // layer-2 wait + layer-2 epilogue
      sum_b += ts5 - ts4;  // next tile's layer-1 epilogue / layer-3 waits
      sum_c += ts6 - ts5;  // output layer
      ++ntile;
#endif
    }
#ifdef MPPI_DEBUG_TIMERS
    if (dbg) {
      dbg[8] = sum_a;
      dbg[9] = sum_b;
      dbg[10] = sum_c;
      dbg[11] = ntile;
    }
#endif
#undef MLP_T
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------------ host side
inline int pow2_scale(const double* w, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) m = std::fmax(m, std::fabs(w[i]));
  if (!(m > 0.0)) return 0;
  return 13 - (int)std::ceil(std::log2(m));  // max |w| * 2^s in (2^12, 2^13]
}

// Pack one layer W (in, out) row-major (the reference layout, surrogate.py:39)
// as Wt (out x K) hi/lo into the image.
inline void pack_layer(std::vector<unsigned char>& img, uint32_t off_h, uint32_t off_l, const double* W,
                       int in, int out, int K, int s) {
  const double sc = std::ldexp(1.0, s);
  for (int n = 0; n < out; ++n)
    for (int k = 0; k < K; ++k) {
      const double v = k < in ? W[(size_t)k * out + n] * sc : 0.0;
      const __half h = __float2half_rn((float)v);
      const __half l = __float2half_rn((float)(v - (double)__half2float(h)));
      const uint32_t o = umma_off(n, k, K);
      memcpy(&img[off_h + o], &h, 2);
      memcpy(&img[off_l + o], &l, 2);
    }
}

inline cudaError_t mlp_upload(MlpWeights& m, int in_dim, const double* W0, const double* b0,
                              const double* W1, const double* b1, const double* W2, const double* b2,
                              const double* W3, const double* b3, cudaStream_t st) {
  std::vector<unsigned char> img(kImgBytes, 0);
  const int s0 = pow2_scale(W0, (size_t)in_dim * kMlpH0), s1 = pow2_scale(W1, (size_t)kMlpH0 * kMlpH1),
            s2 = pow2_scale(W2, (size_t)kMlpH1 * kMlpH2);
  pack_layer(img, OFF_W0H, OFF_W0L, W0, in_dim, kMlpH0, kMlpIn, s0);
  pack_layer(img, OFF_W1H, OFF_W1L, W1, kMlpH0, kMlpH1, kMlpH0, s1);
  pack_layer(img, OFF_W2H, OFF_W2L, W2, kMlpH1, kMlpH2, kMlpH1, s2);
  float* par = reinterpret_cast<float*>(&img[OFF_PAR]);
  for (int i = 0; i < kMlpH0; ++i) par[i] = (float)b0[i];
  for (int i = 0; i < kMlpH1; ++i) par[kMlpH0 + i] = (float)b1[i];
  for (int i = 0; i < kMlpH2; ++i) par[kMlpH0 + kMlpH1 + i] = (float)b2[i];
  for (int i = 0; i < kMlpH2; ++i) par[kMlpH0 + kMlpH1 + kMlpH2 + i] = (float)W3[i];
  float* tail = par + kMlpH0 + kMlpH1 + 2 * kMlpH2;
  tail[0] = (float)b3[0];
  tail[1] = (float)std::ldexp(1.0, -s0);
  tail[2] = (float)std::ldexp(1.0, -s1);
  tail[3] = (float)std::ldexp(1.0, -s2);
  cudaError_t e = cudaSuccess;
  if (!m.img) e = cudaMalloc(&m.img, kImgBytes);
  if (e != cudaSuccess) return e;
  m.in_dim = in_dim;
  e = cudaMemcpyAsync(m.img, img.data(), kImgBytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);
}

inline cudaError_t mlp_forward(const MlpWeights& m, const float* x, long long rows, float* out,
                               cudaStream_t st, unsigned long long* dbg = nullptr) {
  static bool attr_set[64] = {};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(mlp_tcgen05_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kMlpSmem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long tiles = (rows + 127) / 128;
  const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kMlpThreads, 1, 1);
  cfg.dynamicSmemBytes = kMlpSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (pdl_mask() & PDL_MLP) != 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mlp_tcgen05_kernel, x, rows, (const unsigned char*)m.img, out,
                            (pdl_mask() & PDL_EARLY) ? 1 : 0, dbg);
}

inline void mlp_release(MlpWeights& m) {
  if (m.img) cudaFree(m.img);
  m.img = nullptr;
}

}  // namespace mppi
