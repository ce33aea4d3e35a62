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
// Pipeline: see the comment above mlp_tcgen05_kernel (activations stay in
// TMEM; layer 2 of tile t+1 overlaps the tail of tile t).
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
// fp16 hi followed by 128 x 32 fp16 lo — used by the opt-in fused rollout +
// MLP kernel (mppi_fused.cuh); mlp_tcgen05_kernel keeps activations in TMEM
// and uses the OFF_K* layout below.
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

// Warp-wide issue forms: the whole (converged) warp executes them and one
// elected lane issues, so the descriptors stay warp-uniform and ptxas keeps
// them in uniform registers — no per-MMA R2UR moves or divergent-issue loop.
// (The lane-0-only issuer spent ~8 instructions with dependent R2UR latency
// on each MMA and starved while 4 epilogue warps shared its scheduler:
// scripts/micro/mlp_trace.cu.) The same lane (the lowest, lane 0) issues
// every MMA and commit, as tcgen05.commit tracks the issuing thread's MMAs.
__device__ __forceinline__ void umma_f16_w(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_f16_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_w(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(bar)
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

// ReLU + hi/lo split of one activation pair (element 0 in the low half), in
// five SASS instructions per pair with the scale/bias FFMA2 in front of it
// (round 2 had eight: FMNMX x2, F2FP, HADD2.F32 x2, FFMA2, F2FP):
//   hi = fp16_rz(relu(v))          F2FP.RELU.RZ  (truncation keeps v - hi >= 0)
//   lo = fp16_rn(relu(v - hi))     FHFMA x2 (mixed f16 x f16 + f32), F2FP.RELU
// For v <= 0 both halves are 0; for v > 0, 0 <= v - hi < ulp16(v), so the
// relu on lo is a no-op and hi + lo carries ~21 significant bits (the
// round-to-nearest hi of store_split8 gives ~22; measured MLP error vs the
// float64 reference stays ~3e-7 m).
__device__ __forceinline__ void split_relu2(float v0, float v1, uint32_t& h, uint32_t& l) {
  asm("cvt.rz.relu.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(v1), "f"(v0));
  float d0, d1;
  const unsigned short m1 = 0xBC00u;  // fp16 -1.0
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d0) : "h"((unsigned short)(h & 0xffffu)), "h"(m1), "f"(v0));
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d1) : "h"((unsigned short)(h >> 16)), "h"(m1), "f"(v1));
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(d1), "f"(d0));
}

// 8 ReLU activations (already >= 0) -> one hi and one lo 16-byte core-matrix
// row with the split of split_relu2 (the fused kernel's A buffers).
__device__ __forceinline__ void store_split8_act(unsigned char* sm, uint32_t off_h, uint32_t off_l, uint32_t o,
                                                 const float* y) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_relu2(y[2 * i], y[2 * i + 1], h[i], l[i]);
  *reinterpret_cast<uint4*>(sm + off_h + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(sm + off_l + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

// 8 fp32 -> one hi and one lo 16-byte core-matrix row.
__device__ __forceinline__ void store_split8(unsigned char* sm, uint32_t off_h, uint32_t off_l, uint32_t o,
                                             const float* y) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 hh = __floats2half2_rn(y[2 * i], y[2 * i + 1]);
    const float2 hf = __half22float2(hh);
    // lo = y - hi for both elements in one packed FP32 op (FFMA2: hi * -1 + y)
    const float2 d = __ffma2_rn(hf, make_float2(-1.f, -1.f), make_float2(y[2 * i], y[2 * i + 1]));
    const __half2 ll = __floats2half2_rn(d.x, d.y);
    h[i] = *reinterpret_cast<const uint32_t*>(&hh);
    l[i] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  *reinterpret_cast<uint4*>(sm + off_h + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(sm + off_l + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

// ------------------------------------------------------------------ the kernel
// Warp-specialised: warps 0-15 are the epilogue (warp w serves TMEM lane
// quadrant q = w % 4, i.e. rows 32q..32q+31 of the tile, and column group
// cg = w / 4); warp 16 is the producer: it issues the weight copies and every
// tcgen05.mma. The hand-off is mbarrier-only:
//   epilogue --A1[c]/A2[c] (16 arrivals)--> issuer --tcgen05.commit--> epilogue
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

// Split form for software pipelining: the load is issued now, its registers
// are valid after tmem_wait_ld8 (which takes them as read-write operands, so
// no use can be scheduled ahead of the wait).
__device__ __forceinline__ void tmem_ld8_async(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld8(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
               :
               : "memory");
}

__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld16(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])
               :
               : "memory");
}
template <int X>
__device__ __forceinline__ void tmem_ld_async(uint32_t taddr, uint32_t* r) {
  if constexpr (X == 16) tmem_ld16_async(taddr, r);
  else tmem_ld8_async(taddr, r);
}
template <int X>
__device__ __forceinline__ void tmem_wait_ld(uint32_t* r) {
  if constexpr (X == 16) tmem_wait_ld16(r);
  else tmem_wait_ld8(r);
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void epi_barrier() {  // named barrier over the 512 epilogue threads
  asm volatile("bar.sync 1, %0;" ::"n"(kMlpEpiWarps * 32) : "memory");
}

// x: (M_pad,16) fp32 positional encodings; out: (M) fp32 distances.
// Warp-specialised: warps 0-15 run the epilogues (warp w serves TMEM lane
// quadrant q = w % 4 and column group cg = w / 4: 8 of every 32 accumulator
// columns), warp 16 issues the weight copies and every tcgen05.mma.
// Every activation stays in tensor memory: the epilogue converts each
// accumulator chunk IN PLACE into fp16-hi/lo columns and layers 2 and 3 read
// their A operand from TMEM (tcgen05.mma ... [a_tmem]); only the weights and
// the input encodings come from shared memory. (The first version sent the
// activations through two 16 KiB shared-memory buffers: that throttled the
// layer-1 epilogue to two chunks ahead of the MMAs and, with an N=128 MMA
// reading ~90 B/clk of the SM's ~128 B/clk, kept layer 2 near a shared-memory
// bound; config-4 MLP 13.2 -> 12.1 ms, bit-identical.)
//
// In-place layout: a 16-element K slice s of an activation occupies the 16
// TMEM columns [16s, 16s+16) of its accumulator: 8 columns of fp16-hi pairs,
// then 8 of fp16-lo pairs (element 2i in the low half). The two warps of a
// slice each write half of its hi and half of its lo columns, i.e. into each
// other's fp32 columns, so they meet at a 64-thread named barrier between
// reading and writing.
//
// Schedule per tile t: epilogue = [layer-2 epilogue (t)] -> [layer-1 epilogue
// (t+1)] -> [output layer (t)]; issuer = L2(t) -> (L2(t) done) L1(t+1) ->
// L3(t) -> (L3(t) done) L2(t+1). Layer 1 of the next tile runs while the
// layer-2 epilogue converts, and the next tile's layer-1 epilogue runs under
// layer 3. 88 registers (MPPI_MLP_MAXNREG). Note that no 4-warp CTA of
// another kernel fits beside this CTA even when the register total would:
// the register file is split by SM sub-partition and 17 warps put 5 on one
// (scripts/micro/coresident.cu).
// Epilogue geometry: each warp converts kEpiCols accumulator columns of its
// lane quadrant per chunk; a chunk (4 column groups) is what one A1/A2
// barrier hands to the issuer. 8 (default): two warps per 16-column K slice,
// meeting at a named barrier, 32-column chunks. 16: a warp owns whole slices
// (one 32x32b.x16 TMEM load and one x16 store per chunk, no pair barrier;
// x16 accesses move ~1.4x the bytes per clock of x8, scripts/micro/tmem_bw.cu)
// in 64-column chunks — measured equal at config 4 (4.20 vs 4.22e9
// particle-steps/s) and 1.5 us slower in the config-2 MLP, whose one tile
// per CTA streams into layer 2 at half the granularity (gpurun_out/ab_elect).
#ifndef MPPI_MLP_EPI_COLS
#define MPPI_MLP_EPI_COLS 8
#endif
// The layer-2 epilogue (which feeds layer 3) of the persistent many-tile
// kernel uses 16 columns per warp: its x16 TMEM accesses shorten the
// epilogue that layer 3 waits on (config-4 MLP 10.2 -> 10.0 ms,
// gpurun_out/ab_h16); the one-tile latency kernel keeps 8 (0.1 us faster at
// 500 x 30). MPPI_MLP_EPI_COLS_L2 overrides the many-tile value.
#ifndef MPPI_MLP_EPI_COLS_L2
#define MPPI_MLP_EPI_COLS_L2 16
#endif
constexpr int kEpiCols = MPPI_MLP_EPI_COLS;
static_assert((kEpiCols == 8 || kEpiCols == 16) && (MPPI_MLP_EPI_COLS_L2 == 8 || MPPI_MLP_EPI_COLS_L2 == 16),
              "epilogue columns per warp");
constexpr int kChunkCols = 4 * kEpiCols;
constexpr int kL1Chunks = kMlpH0 / kChunkCols;
constexpr int kSlicesPerChunk = kChunkCols / 16;
// layer-2 epilogue geometry of one kernel instantiation
template <bool ONE_TILE>
struct Epi2 {
  static constexpr int cols = ONE_TILE ? kEpiCols : MPPI_MLP_EPI_COLS_L2;
  static constexpr int chunk = 4 * cols, chunks = kMlpH1 / chunk, slices = chunk / 16;
};
// barriers: W0 W1 W2 | L1[2] | A1[8] | L2done | A2[4] | L3done | X
constexpr int kMlpBars = 3 + 2 + 8 + 1 + 4 + 1 + 1;
constexpr uint32_t OFF_KBAR = OFF_XL + 128 * 16 * 2;
constexpr uint32_t OFF_KTMEMPTR = OFF_KBAR + kMlpBars * 8;
constexpr uint32_t OFF_KRED = (OFF_KTMEMPTR + 16 + 15) / 16 * 16;
constexpr uint32_t kMlpKernelSmem = OFF_KRED + 2 * 4 * 128 * 4;  // output partial sums, double-buffered
static_assert(kMlpKernelSmem <= 232448, "MLP does not fit shared memory");

__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}

// Output layer share of C accumulator columns: relu((hi + lo products) * s +
// b) . w3, packed FP32 with two partial sums (shared by mlp_tcgen05_kernel and
// the fused kernel so both sum in the same order)
template <int C>
__device__ __forceinline__ float output_part(const float* y, const float* z, float s, const float* b,
                                             const float* w) {
  const float2 sc = make_float2(s, s);
  const float2* bb = reinterpret_cast<const float2*>(b);
  const float2* ww = reinterpret_cast<const float2*>(w);
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < C / 2; ++i) {
    float2 v = __fadd2_rn(make_float2(y[2 * i], y[2 * i + 1]), make_float2(z[2 * i], z[2 * i + 1]));
    v = __ffma2_rn(v, sc, bb[i]);
    v = make_float2(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f));
    acc = __ffma2_rn(v, ww[i], acc);
  }
  return acc.x + acc.y;
}

// 8 fp32 accumulator columns (columns 8cg..8cg+7 of a 32-column chunk at
// `chunk`) -> relu(y * s + b) -> 4 hi + 4 lo packed fp16 columns of the
// chunk's slice (cg >> 1) layout. `pair_bar`: named barrier of the two warps
// of the slice.
__device__ __forceinline__ void tmem_convert8(uint32_t chunk, int cg, const float* y, float s, const float* b,
                                              int pair_bar) {
  uint32_t h[4], l[4];
  const float2 s2 = make_float2(s, s);
  const float2* b2 = reinterpret_cast<const float2*>(b);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 v = __ffma2_rn(make_float2(y[2 * i], y[2 * i + 1]), s2, b2[i]);
    split_relu2(v.x, v.y, h[i], l[i]);
  }
  asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");  // both warps of the slice have read
  const uint32_t slice = chunk + 16 * (cg >> 1), half = 4 * (cg & 1);
  tmem_st4(slice + half, h);
  tmem_st4(slice + 8 + half, l);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 16 fp32 accumulator columns of one warp's own K slice (TMEM columns
// [slice, slice + 16)) -> relu(y * s + b) -> 8 hi then 8 lo packed fp16
// columns in the same 16 columns: one x16 store, no other warp involved.
__device__ __forceinline__ void tmem_convert16(uint32_t slice, const float* y, float s, const float* b) {
  uint32_t hl[16];
  const float2 s2 = make_float2(s, s);
  const float2* b2 = reinterpret_cast<const float2*>(b);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 v = __ffma2_rn(make_float2(y[2 * i], y[2 * i + 1]), s2, b2[i]);
    split_relu2(v.x, v.y, hl[i], hl[8 + i]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(slice),
      "r"(hl[0]), "r"(hl[1]), "r"(hl[2]), "r"(hl[3]), "r"(hl[4]), "r"(hl[5]), "r"(hl[6]), "r"(hl[7]), "r"(hl[8]),
      "r"(hl[9]), "r"(hl[10]), "r"(hl[11]), "r"(hl[12]), "r"(hl[13]), "r"(hl[14]), "r"(hl[15])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// one warp's share of an accumulator chunk starting at TMEM column `chunk`
template <int X>
__device__ __forceinline__ void tmem_convert(uint32_t chunk, int cg, const float* y, float s, const float* b,
                                             int pair_bar) {
  if constexpr (X == 16) tmem_convert16(chunk + 16 * cg, y, s, b);
  else tmem_convert8(chunk, cg, y, s, b, pair_bar);
}

#ifdef MPPI_DEBUG_TIMERS
// phase stamps (globaltimer) of CTAs < 256, 16 slots each: set by the host
static __device__ unsigned long long* mlp_dbg = nullptr;
#define MLP_STAMP(k)                                                         \
  do {                                                                       \
    if (mlp_dbg != nullptr && blockIdx.x < 256) {                            \
      unsigned long long t_;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      mlp_dbg[16 * blockIdx.x + (k)] = t_;                                   \
    }                                                                        \
  } while (0)
#else
#define MLP_STAMP(k) \
  do {               \
  } while (0)
#endif
#ifdef MPPI_MLP_TRACE
// per-tile event clocks of CTA 0 (scripts/micro/mlp_trace.cu): [local tile][event]
__device__ long long mlp_trace[32 * 32];
#define MLP_TRACE(k, e)                                                          \
  do {                                                                         \
    if (blockIdx.x == 0 && (k) < 32) mlp_trace[(k) * 32 + (e)] = clock64();    \
  } while (0)
#else
#define MLP_TRACE(k, e) \
  do {                  \
  } while (0)
#endif

// ONE_TILE: every CTA owns at most one tile (the latency path: rows <= 128 x
// SMs); the next-tile pipelining is compiled out, so the kernel's code holds
// only what such a launch executes (its instructions are fetched cold).
#ifndef MPPI_MLP_MAXNREG
#define MPPI_MLP_MAXNREG 88
#endif
template <bool ONE_TILE>
static __global__ void __maxnreg__(MPPI_MLP_MAXNREG)
    mlp_tcgen05_kernel(const float* __restrict__ x, long long M, const unsigned char* __restrict__ img,
                       float* __restrict__ out, int early, int x_q, int in_d) {
  extern __shared__ __align__(1024) unsigned char mlp_smem[];
  unsigned char* sm = mlp_smem;
  // the warp index broadcast from lane 0, so the compiler keeps the TMEM
  // addresses derived from it in uniform registers (fewer R2UR per access;
  // A/B: config 4 MLP -2 %, config-2 step -0.35 us)
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const uint32_t sb = smem_u32(sm);
  const uint32_t barW0 = sb + OFF_KBAR, barW1 = barW0 + 8, barW2 = barW0 + 16;
  const uint32_t barL10 = barW0 + 24, barA1 = barW0 + 40, barL2done = barW0 + 104, barA2 = barW0 + 112;
  const uint32_t barL3done = barW0 + 144, barX = barW0 + 152;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_KTMEMPTR);

  if (tid == 0) {
    MLP_STAMP(12);
    for (int i = 0; i < 5; ++i) mbar_init(barW0 + 8 * i, 1);  // W0 W1 W2 L1[2]
    for (int i = 0; i < 8; ++i) mbar_init(barA1 + 8 * i, kMlpEpiWarps);
    mbar_init(barL2done, 1);
    for (int i = 0; i < 4; ++i) mbar_init(barA2 + 8 * i, kMlpEpiWarps);
    mbar_init(barL3done, 1);
    mbar_init(barX, kMlpEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc2 = tmem + 256, acc3 = tmem + 384;  // acc1 at tmem
  const long long ntiles = (M + 127) / 128;
  const long long G = gridDim.x;
  constexpr int kEpiCols2 = Epi2<ONE_TILE>::cols, kChunkCols2 = Epi2<ONE_TILE>::chunk;
  constexpr int kL2Chunks = Epi2<ONE_TILE>::chunks, kSlicesPerChunk2 = Epi2<ONE_TILE>::slices;

  if (warp == kMlpEpiWarps) {
    // ============================== issuer ==================================
    if (lane == 0) {
      MLP_STAMP(11);
      mbar_expect_tx(barW0, kSeg0);
      bulk_g2s(sb + 0, img, kSeg0, barW0);
      mbar_expect_tx(barW1, kSeg1);
      for (uint32_t o = 0; o < kSeg1; o += 32768)
        bulk_g2s(sb + OFF_W1H + o, img + OFF_W1H + o, min(32768u, kSeg1 - o), barW1);
      mbar_expect_tx(barW2, kSeg2);
      bulk_g2s(sb + OFF_W2H, img + OFF_W2H, kSeg2, barW2);
    }
    __syncwarp();
    {  // the whole warp from here on: MMAs and commits issued by one elected lane
      const uint32_t id64 = umma_idesc(64), id128 = umma_idesc(128);
      const uint64_t dXH = umma_desc(sb + OFF_XH, 128, 256), dXL = umma_desc(sb + OFF_XL, 128, 256);
      const uint64_t dW0H = umma_desc(sb + OFF_W0H, 128, 256), dW0L = umma_desc(sb + OFF_W0L, 128, 256);
      const uint64_t dW1H = umma_desc(sb + OFF_W1H, 128, 4096), dW1L = umma_desc(sb + OFF_W1L, 128, 4096);
      const uint64_t dW2H = umma_desc(sb + OFF_W2H, 128, 2048);
      auto issue_l1 = [&]() {  // two halves of N=128 per product, one commit each
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const uint64_t wo = umma_off(128 * hf, 0, 16) >> 4;
          umma_f16_w(tmem + 128 * hf, dXH, dW0H + wo, id128, 0);
          umma_f16_w(tmem + 128 * hf, dXH, dW0L + wo, id128, 1);
          umma_f16_w(tmem + 128 * hf, dXL, dW0H + wo, id128, 1);
          umma_commit_w(barL10 + 8 * hf);
        }
      };
      uint32_t phX = 0, ph = 0;  // ph: parity of the once-per-tile barriers (A1[c], A2[c], L2done, L3done)
      bool first = true;
      int it = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += G, ph ^= 1u, ++it) {
        const bool has_next = !ONE_TILE && tile + G < ntiles;
        if (first) {
          mbar_wait(barX, phX);
          phX ^= 1;
          mbar_wait(barW0, 0);
          tc_fence_after();
          issue_l1();
        }
#pragma unroll
        for (int c = 0; c < kL1Chunks; ++c) {  // layer 2, K chunk c: its slices of acc1 (in place)
          mbar_wait(barA1 + 8 * c, ph);
          if (c == 0 && lane == 0) MLP_TRACE(it, 8);
          if (c == kL1Chunks - 1) if (lane == 0) MLP_TRACE(it, 9);
          if (first && c == 0) {
            mbar_wait(barW1, 0);
            if (lane == 0) MLP_STAMP(9);
          }
          if (!first && c == 0) {  // acc2 is rewritten: the previous tile's layer 3 (its A reader) is done
            mbar_wait(barL3done, ph ^ 1u);
            if (lane == 0) MLP_TRACE(it, 6);
          }
          tc_fence_after();
#pragma unroll
          for (int g = 0; g < kSlicesPerChunk; ++g) {
            const int s = kSlicesPerChunk * c + g;
            const uint32_t ah = tmem + 16 * s, al = ah + 8;
            const uint64_t wj = (uint64_t)((2 * s) * 128 >> 4);
            umma_f16_ts_w(acc2, ah, dW1H + wj, id128, s ? 1u : 0u);
            umma_f16_ts_w(acc2, ah, dW1L + wj, id128, 1);
            umma_f16_ts_w(acc2, al, dW1H + wj, id128, 1);
          }
        }
        umma_commit_w(barL2done);
        if (lane == 0) MLP_TRACE(it, 10);
        if (has_next) {  // acc1 is free once layer 2 has read it; X(t+1) staged by the epilogue
          mbar_wait(barL2done, ph);
          if (lane == 0) MLP_TRACE(it, 11);
          mbar_wait(barX, phX);
          if (lane == 0) MLP_TRACE(it, 16);
          phX ^= 1;
          tc_fence_after();
          issue_l1();
          if (lane == 0) MLP_TRACE(it, 17);
        }
#pragma unroll
        for (int c = 0; c < kL2Chunks; ++c) {  // layer 3, K chunk c: its slices of acc2 (in place)
          mbar_wait(barA2 + 8 * c, ph);
          if (c == 0 && lane == 0) MLP_TRACE(it, 12);
          if (c == kL2Chunks - 1) if (lane == 0) MLP_TRACE(it, 13);
          if (first && c == 0) {
            mbar_wait(barW2, 0);
            if (lane == 0) MLP_STAMP(10);
          }
          tc_fence_after();
#pragma unroll
          for (int g = 0; g < kSlicesPerChunk2; ++g) {
            const int s = kSlicesPerChunk2 * c + g;
            const uint32_t ah = acc2 + 16 * s, al = ah + 8;
            const uint64_t wj = (uint64_t)((2 * s) * 128 >> 4);
            // W2 hi and lo are adjacent 64-row operands: A_hi [W hi | W lo] in one N=128 MMA
            umma_f16_ts_w(acc3, ah, dW2H + wj, id128, s ? 1u : 0u);
            umma_f16_ts_w(acc3, al, dW2H + wj, id64, 1);
          }
        }
        umma_commit_w(barL3done);
        if (lane == 0) MLP_TRACE(it, 14);
        first = false;
      }
      if (first) {
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
    const int pair_bar = 2 + quad * 2 + (cg >> 1);  // named barriers 2..9
    float* red = reinterpret_cast<float*>(sm + OFF_KRED);
    const float* par = reinterpret_cast<const float*>(sm + OFF_PAR);
    const float* b0 = par;
    const float* b1 = par + kMlpH0;
    const float* b2 = b1 + kMlpH1;
    const float* w3 = b2 + kMlpH2;
    auto load_x = [&](long long t, float* xv) {  // threads < 256: row tid % 128, 8 of 16 columns
      const long long r = t * 128 + (tid & 127);
      if (x_q && tid < 256 && t < ntiles && r < M) {
        // joint positions (8 floats per row); encode_x turns them into the
        // row's encoding columns right before the shared-memory store, so the
        // load latency stays hidden behind the epilogue that follows
        const float4* src = reinterpret_cast<const float4*>(x + r * 8);
        const float4 f0 = __ldg(src), f1 = __ldg(src + 1);
        xv[0] = f0.x; xv[1] = f0.y; xv[2] = f0.z; xv[3] = f0.w;
        xv[4] = f1.x; xv[5] = f1.y; xv[6] = f1.z; xv[7] = f1.w;
      } else if (tid < 256 && t < ntiles && r < M) {
        const float4* src = reinterpret_cast<const float4*>(x + r * 16 + (tid >> 7) * 8);
        const float4 f0 = __ldg(src), f1 = __ldg(src + 1);
        xv[0] = f0.x; xv[1] = f0.y; xv[2] = f0.z; xv[3] = f0.w;
        xv[4] = f1.x; xv[5] = f1.y; xv[6] = f1.z; xv[7] = f1.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = 0.f;
      }
    };
    // x_q: joint positions in xv -> columns 8*(tid >> 7) .. +7 of [sin q,
    // cos q, 0...] (surrogate.py:24-28) with the rollout's own sincos_
    auto encode_x = [&](float* xv) {
      if (!x_q || tid >= 256) return;
      float q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = xv[j];
      const int c0 = (tid >> 7) * 8;
      if (in_d == 7) {  // arm7: [s0..s6 c0 | c1..c6 0 0]
        if (c0 == 0) {
          float cz;
#pragma unroll
          for (int j = 0; j < 7; ++j) {
            float cj;
            sincos_(q[j], &xv[j], &cj);
            if (j == 0) cz = cj;
          }
          xv[7] = cz;
        } else {
#pragma unroll
          for (int j = 0; j < 6; ++j) {
            float sj;
            sincos_(q[j + 1], &sj, &xv[j]);
          }
          xv[6] = xv[7] = 0.f;
        }
      } else {
        float sn[8], cs[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) sincos_(q[j], &sn[j], &cs[j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // register selects (no local-memory indexing)
          const int c = c0 + i;
          float v = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            v = (c == j && j < in_d) ? sn[j] : v;
            v = (c == in_d + j && j < in_d) ? cs[j] : v;
          }
          xv[i] = v;
        }
      }
    };
    auto arrive = [&](uint32_t bar) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
    };
    float xv[8];
    long long tile = blockIdx.x;
    if (tid == 0) MLP_STAMP(0);
    if (early) pdl_trigger();
    pdl_wait();  // the rollout's positional encodings are complete past this point
    if (tile < ntiles) {
      load_x(tile, xv);
      encode_x(xv);
      if (tid < 256) store_split8(sm, OFF_XH, OFF_XL, umma_off(tid & 127, (tid >> 7) * 8, 16), xv);
      fence_async_smem();
      arrive(barX);
      if (tid == 0) MLP_STAMP(1);
      mbar_wait(barW0, 0);
      if (tid == 0) MLP_STAMP(2);
    }
    const float s0 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 1];
    const float s1 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 2];
    const float s2 = par[kMlpH0 + kMlpH1 + 2 * kMlpH2 + 3];
    uint32_t phL1 = 0;
    // layer-1 epilogue of tile t, in place in acc1; stages X(t + G) on the way
    int eit = 0;  // local tile counter (trace)
    auto epilogue_l1 = [&](long long t) {
      const bool nxt = !ONE_TILE && t + G < ntiles;
      if (nxt) load_x(t + G, xv);
      // chunk c+1's TMEM load is in flight while chunk c is converted (within
      // one layer-1 half: the second half waits for its own MMA barrier)
      constexpr int HC = kL1Chunks / 2;  // chunks per layer-1 half (one MMA barrier each)
      uint32_t rb[2][kEpiCols];
#pragma unroll
      for (int c = 0; c < kL1Chunks; ++c) {
        if (c % HC == 0) {
          const int hb = c / HC;
          mbar_wait(barL10 + 8 * hb, (phL1 >> hb) & 1u);
          if (tid == 0 && hb == 0 && t == blockIdx.x) MLP_STAMP(3);
          if (tid == 0 && hb == 0) MLP_TRACE(eit, 2);
          phL1 ^= 1u << hb;
          tc_fence_after();
          tmem_ld_async<kEpiCols>(tmem + lane_base + kChunkCols * c + kEpiCols * cg, rb[c & 1]);
        }
        tmem_wait_ld<kEpiCols>(rb[c & 1]);
        if (c % HC != HC - 1)
          tmem_ld_async<kEpiCols>(tmem + lane_base + kChunkCols * (c + 1) + kEpiCols * cg, rb[(c + 1) & 1]);
        float y[kEpiCols];
#pragma unroll
        for (int i = 0; i < kEpiCols; ++i) y[i] = __uint_as_float(rb[c & 1][i]);
        tmem_convert<kEpiCols>(tmem + lane_base + kChunkCols * c, cg, y, s0, b0 + kChunkCols * c + kEpiCols * cg,
                               pair_bar);
        arrive(barA1 + 8 * c);
        if (tid == 0) MLP_TRACE(eit, 24 + c);
        if (tid == 0 && c == kL1Chunks - 1) MLP_TRACE(eit, 3);
        if (c == kL1Chunks - 1 && nxt) {  // both layer-1 halves done (barL1[1]): X can be rewritten
          encode_x(xv);
          if (tid < 256) store_split8(sm, OFF_XH, OFF_XL, umma_off(tid & 127, (tid >> 7) * 8, 16), xv);
          fence_async_smem();
          arrive(barX);
        }
      }
    };
    uint32_t ph = 0;
    if (tile < ntiles) epilogue_l1(tile);
    if (tid == 0) MLP_STAMP(4);
    for (; tile < ntiles; tile += G, ph ^= 1u) {
      const bool has_next = !ONE_TILE && tile + G < ntiles;
      // ---- layer-2 epilogue, in place in acc2
      mbar_wait(barL2done, ph);
      if (tid == 0 && tile == blockIdx.x) MLP_STAMP(5);
      if (tid == 0) MLP_TRACE(eit, 0);
      tc_fence_after();
      uint32_t r2[2][kEpiCols2];
      tmem_ld_async<kEpiCols2>(acc2 + lane_base + kEpiCols2 * cg, r2[0]);
#pragma unroll
      for (int c = 0; c < kL2Chunks; ++c) {  // chunk c+1's TMEM load in flight under chunk c
        tmem_wait_ld<kEpiCols2>(r2[c & 1]);
        if (c + 1 < kL2Chunks)
          tmem_ld_async<kEpiCols2>(acc2 + lane_base + kChunkCols2 * (c + 1) + kEpiCols2 * cg, r2[(c + 1) & 1]);
        float y[kEpiCols2];
#pragma unroll
        for (int i = 0; i < kEpiCols2; ++i) y[i] = __uint_as_float(r2[c & 1][i]);
        tmem_convert<kEpiCols2>(acc2 + lane_base + kChunkCols2 * c, cg, y, s1, b1 + kChunkCols2 * c + kEpiCols2 * cg,
                               pair_bar);
        arrive(barA2 + 8 * c);
        if (tid == 0) MLP_TRACE(eit, 20 + c);
      }
      if (tid == 0 && tile == blockIdx.x) MLP_STAMP(6);
      if (tid == 0) MLP_TRACE(eit, 1);
      ++eit;  // the next tile's layer-1 epilogue records under its own index
      // ---- the next tile's layer-1 epilogue runs under this tile's layer 3
      if (has_next) epilogue_l1(tile + G);
      --eit;
      // ---- output layer of this tile
      mbar_wait(barL3done, ph);
      if (tid == 0 && tile == blockIdx.x) MLP_STAMP(7);
      if (tid == 0) MLP_TRACE(eit, 4);
      tc_fence_after();
      float part = 0.f;
      {
        float y[16], z[16];
        tmem_ld16(acc3 + lane_base + 16 * cg, y);       // A_hi W_hi + A_lo W_hi
        tmem_ld16(acc3 + lane_base + 64 + 16 * cg, z);  // A_hi W_lo
        part = output_part<16>(y, z, s2, b2 + 16 * cg, w3 + 16 * cg);
      }
      // the four column-group warps of a lane quadrant combine their rows: a
      // 128-thread barrier per quadrant, partial sums double-buffered by tile
      // parity (the buffer is rewritten two tiles later, after the quadrant's
      // next barrier, which its reader has passed)
      float* rq = red + (ph & 1u) * 512;
      rq[cg * 128 + row_in_tile] = part;
      asm volatile("bar.sync %0, 128;" ::"r"(10 + quad) : "memory");
      if (cg == 0) {
        const long long row = tile * 128 + row_in_tile;
        const float o = par[kMlpH0 + kMlpH1 + 2 * kMlpH2] + rq[row_in_tile] + rq[128 + row_in_tile] +
                        rq[256 + row_in_tile] + rq[384 + row_in_tile];
        if (row < M) out[row] = o;
      }
      if (tid == 0 && tile == blockIdx.x) MLP_STAMP(8);
      if (tid == 0) MLP_TRACE(eit, 5);
      ++eit;
    }
  }
  tc_fence_before();  // every TMEM read of this CTA is ordered before the dealloc
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
#ifdef MPPI_DEBUG_TIMERS
  if (mlp_dbg != nullptr && tid == 0) {  // latest CTA end over the grid
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    atomicMax(&mlp_dbg[16 * 255 + 15], t_);
  }
#endif
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

// x_q = 0: x holds (rows,16) positional encodings; 1: (rows,8) joint positions
// (the d = in_dim/2 joints, zero padded), encoded inside the kernel.
inline cudaError_t mlp_forward(const MlpWeights& m, const float* x, long long rows, float* out,
                               cudaStream_t st, int x_q = 0) {
  static bool attr_set[64] = {};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    for (auto k : {mlp_tcgen05_kernel<false>, mlp_tcgen05_kernel<true>}) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMlpKernelSmem);
      if (e != cudaSuccess) return e;
    }
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long tiles = (rows + 127) / 128;
  const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
  auto kern = (tiles <= sms && getenv("MPPI_MLP_GENERAL") == nullptr) ? mlp_tcgen05_kernel<true>
                                                                       : mlp_tcgen05_kernel<false>;
  if (!(pdl_mask() & (PDL_MLP | PDL_EARLY))) {  // plain launch: no programmatic edge in a captured graph
    kern<<<grid, kMlpThreads, kMlpKernelSmem, st>>>(x, rows, (const unsigned char*)m.img, out, 0, x_q,
                                                    m.in_dim / 2);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kMlpThreads, 1, 1);
  cfg.dynamicSmemBytes = kMlpKernelSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (pdl_mask() & PDL_MLP) != 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, x, rows, (const unsigned char*)m.img, out,
                            (pdl_mask() & PDL_EARLY) ? 1 : 0, x_q, m.in_dim / 2);
}

inline void mlp_release(MlpWeights& m) {
  if (m.img) cudaFree(m.img);
  m.img = nullptr;
}

}  // namespace mppi
