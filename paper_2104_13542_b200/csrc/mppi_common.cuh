// mppi_common.cuh — shared device math and parameter blocks of the B200 MPPI path.
//
// Every routine here restates one numeric primitive of the reference's numba
// backend (pkg/src/jointmpc/kernels/jit.py) for the GPU, templated on the
// arithmetic type R (float for the fast fused path, double for the exact
// path and the float64 operator seam). Constants follow kernels/shared.py.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/mppi_b200.h"

namespace mppi {

constexpr int MAXD = MPPI_MAX_DOF;
constexpr int MAXH = MPPI_MAX_HORIZON;
constexpr int MAXC = MPPI_MAX_CAPSULES;
constexpr int MAXP = MPPI_MAX_PAIRS;
constexpr int REORTHO_EVERY = 8;    // shared.py:8
constexpr int POLAR_ITERS = 2;      // shared.py:11
constexpr int TERNARY_ITERS = 60;   // shared.py:15
constexpr double SEG_EPS = 1e-12;   // shared.py:18
constexpr double NO_CONTACT = -1.0e30;  // shared.py:21

// Term order of CostStack.term_names (costs.py:24).
enum Term { T_POSE = 0, T_STOP, T_JOINT, T_MANIP, T_SELF, T_ENV, N_TERMS };

// ---------------------------------------------------------------- params
// Chain in packed form (kinematics.py:53-114), converted once to R on the host.
template <typename R>
struct ChainT {
  int dof, task_dim, n_caps, n_pairs;
  int jtype[MAXD];
  int cap_link[MAXC];
  int pair_a[MAXP], pair_b[MAXP];
  R axes[MAXD][3];
  R orot[MAXD][9];
  R otrans[MAXD][3];
  R lo[MAXD], hi[MAXD];  // shrunken limits, costs.py:111-116 (host-computed in fp64)
  R accel[MAXD];         // accel_limits for the braking envelope, costs.py:98-102
  R cap_p0[MAXC][3], cap_p1[MAXC][3], cap_r[MAXC];
};

// CostWeights + active-term flags (costs.py:27-53, 222-240).
template <typename R>
struct CostT {
  R alpha_rot[3], alpha_trans[3];
  R a_stop, a_joint, a_manip, a_coll, k_m;
  int use_stop, use_joint, use_manip;  // weight > 0
  int selfcoll;                        // MPPI_SELFCOLL_* (0 when alpha_coll == 0)
  int use_env;                         // alpha_coll > 0 and world has obstacles
};

// World model on the device (simworld.py:30-49) + optional voxel broad phase.
template <typename R>
struct WorldT {
  const R* spheres;  // (ns,4)
  const R* boxes;    // (nb,6)
  int ns, nb;
  // voxel broad phase (config 3): exact distance-to-obstacle-set at voxel
  // centres; NULL when the world came as primitives only.
  const float* sdf;
  int nx, ny, nz;
  R ox, oy, oz, voxel;
};

// ---------------------------------------------------------------- small math
template <typename R>
__device__ __forceinline__ R rsqrt_(R x);
template <>
__device__ __forceinline__ float rsqrt_(float x) { return rsqrtf(x); }
template <>
__device__ __forceinline__ double rsqrt_(double x) { return rsqrt(x); }

// FP32 path: two-constant Cody-Waite reduction to [-pi, pi], then the SFU
// sine/cosine (|error| ~ 2^-21 there, ~5e-7 rad-equivalent overall for joint
// angles, far inside the FP32 parity tolerances) instead of the libm-accurate
// sincosf, whose slow-path argument reduction dominates the FK's instruction
// count.
__device__ __forceinline__ void sincos_(float x, float* s, float* c) {
  const float k = rintf(x * 0.159154943f);
  float r = fmaf(-k, 6.28318548f, x);
  r = fmaf(-k, -1.74845553e-7f, r);
  __sincosf(r, s, c);
}
__device__ __forceinline__ void sincos_(double x, double* s, double* c) { sincos(x, s, c); }

template <typename R>
__device__ __forceinline__ R clamp01(R x) {
  // min(max(x, 0), 1) with the numba operand order (jit.py:203-220)
  x = x > R(0) ? x : R(0);
  return x < R(1) ? x : R(1);
}

// ---------------------------------------------------------------- packed pairs
// Two configurations per lane in the paired throughput rollout
// (rollout_pair_kernel): every FP32 operation on a P2 is one packed
// instruction. mul/add/sub carry no rounding modifier, so ptxas contracts
// them into FFMA2 exactly where it contracts the scalar code into FFMA, and a
// P2 built from one float is a broadcast operand (FFMA2 takes it as a scalar
// register or a uniform register with no extra move).
struct P2 {
  unsigned long long v;
  __device__ __forceinline__ P2() {}
  __device__ __forceinline__ P2(float s) { asm("mov.b64 %0, {%1, %1};" : "=l"(v) : "f"(s)); }
  __device__ __forceinline__ P2(float a, float b) { asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(a), "f"(b)); }
  __device__ __forceinline__ float lo() const {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return a;
  }
  __device__ __forceinline__ float hi() const {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return b;
  }
};
__device__ __forceinline__ P2 operator*(P2 a, P2 b) {
  P2 r;
  asm("mul.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ P2 operator+(P2 a, P2 b) {
  P2 r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ P2 operator-(P2 a, P2 b) {
  P2 r;
  asm("sub.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ P2 operator-(P2 a) { return P2(0.f) - a; }
__device__ __forceinline__ P2 operator/(P2 a, P2 b) { return P2(a.lo() / b.lo(), a.hi() / b.hi()); }
__device__ __forceinline__ P2& operator+=(P2& a, P2 b) { return a = a + b; }
__device__ __forceinline__ P2 max0(P2 a) { return P2(fmaxf(a.lo(), 0.f), fmaxf(a.hi(), 0.f)); }
__device__ __forceinline__ P2 sqrt2(P2 a) { return P2(sqrtf(a.lo()), sqrtf(a.hi())); }
__device__ __forceinline__ P2 fabs2(P2 a) { return P2(fabsf(a.lo()), fabsf(a.hi())); }

// out = A(3x3, row-major) * B
template <typename R>
__device__ __forceinline__ void mat33_mul(const R* A, const R* B, R* out) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      out[i * 3 + j] = A[i * 3 + 0] * B[0 * 3 + j] + A[i * 3 + 1] * B[1 * 3 + j] +
                       A[i * 3 + 2] * B[2 * 3 + j];
}

// FP32: columns 0 and 1 of each output row as one packed FP32 pair (FFMA2
// with the row element of A broadcast), column 2 scalar; every element gets
// the same multiply-then-two-FMA sequence as the scalar form, so the result is
// bit-identical while the instruction count drops from 27 to 18.
template <>
__device__ __forceinline__ void mat33_mul<float>(const float* A, const float* B, float* out) {
  const float2 b0 = make_float2(B[0], B[1]), b1 = make_float2(B[3], B[4]), b2 = make_float2(B[6], B[7]);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float2 p = __fmul2_rn(make_float2(A[i * 3 + 0], A[i * 3 + 0]), b0);
    p = __ffma2_rn(make_float2(A[i * 3 + 1], A[i * 3 + 1]), b1, p);
    p = __ffma2_rn(make_float2(A[i * 3 + 2], A[i * 3 + 2]), b2, p);
    out[i * 3 + 0] = p.x;
    out[i * 3 + 1] = p.y;
    out[i * 3 + 2] = fmaf(A[i * 3 + 2], B[8], fmaf(A[i * 3 + 1], B[5], A[i * 3 + 0] * B[2]));
  }
}

template <typename R>
__device__ __forceinline__ void mat33_vec(const R* A, const R* v, R* out) {
#pragma unroll
  for (int i = 0; i < 3; ++i) out[i] = A[i * 3 + 0] * v[0] + A[i * 3 + 1] * v[1] + A[i * 3 + 2] * v[2];
}

// Rodrigues I + s K + (1-c) K^2 for a unit axis (jit.py:70-86).
template <typename R>
__device__ __forceinline__ void axis_rotation(const R* ax, R s, R c1, R* out) {
  const R x = ax[0], y = ax[1], z = ax[2];
  out[0] = R(1) + c1 * (-z * z - y * y);
  out[1] = -s * z + c1 * (x * y);
  out[2] = s * y + c1 * (x * z);
  out[3] = s * z + c1 * (x * y);
  out[4] = R(1) + c1 * (-z * z - x * x);
  out[5] = -s * x + c1 * (y * z);
  out[6] = -s * y + c1 * (x * z);
  out[7] = s * x + c1 * (y * z);
  out[8] = R(1) + c1 * (-y * y - x * x);
}

// Newton polar iteration R <- (R + R^-T)/2, POLAR_ITERS times (jit.py:38-67).
template <typename R>
__device__ __forceinline__ void orthonormalize(R* M) {
#pragma unroll
  for (int it = 0; it < POLAR_ITERS; ++it) {
    const R a = M[0], b = M[1], c = M[2], d = M[3], e = M[4], f = M[5], g = M[6], h = M[7],
            i = M[8];
    const R det = a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
    R inv[9];
    inv[0] = (e * i - f * h) / det;
    inv[1] = (c * h - b * i) / det;
    inv[2] = (b * f - c * e) / det;
    inv[3] = (f * g - d * i) / det;
    inv[4] = (a * i - c * g) / det;
    inv[5] = (c * d - a * f) / det;
    inv[6] = (d * h - e * g) / det;
    inv[7] = (b * g - a * h) / det;
    inv[8] = (a * e - b * d) / det;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int s = 0; s < 3; ++s) M[r * 3 + s] = R(0.5) * (M[r * 3 + s] + inv[s * 3 + r]);
  }
}

// Closest distance between segments [p0,p1] and [q0,q1] (jit.py:188-226).
template <typename R>
__device__ __forceinline__ R segseg_dist(const R* p0, const R* p1, const R* q0, const R* q1) {
  const R d1x = p1[0] - p0[0], d1y = p1[1] - p0[1], d1z = p1[2] - p0[2];
  const R d2x = q1[0] - q0[0], d2y = q1[1] - q0[1], d2z = q1[2] - q0[2];
  const R rx = p0[0] - q0[0], ry = p0[1] - q0[1], rz = p0[2] - q0[2];
  const R a = d1x * d1x + d1y * d1y + d1z * d1z;
  const R e = d2x * d2x + d2y * d2y + d2z * d2z;
  const R f = d2x * rx + d2y * ry + d2z * rz;
  const R c = d1x * rx + d1y * ry + d1z * rz;
  const R b = d1x * d2x + d1y * d2y + d1z * d2z;
  const R eps = R(SEG_EPS);
  R s, t;
  if (a <= eps && e <= eps) {
    s = R(0);
    t = R(0);
  } else if (a <= eps) {
    s = R(0);
    t = clamp01(f / e);
  } else if (e <= eps) {
    t = R(0);
    s = clamp01(-c / a);
  } else {
    const R denom = a * e - b * b;
    s = fabs(denom) > eps ? clamp01((b * f - c * e) / denom) : R(0);
    t = (b * s + f) / e;
    if (t < R(0)) {
      t = R(0);
      s = clamp01(-c / a);
    } else if (t > R(1)) {
      t = R(1);
      s = clamp01((b - c) / a);
    }
    t = clamp01(t);
  }
  const R cx = p0[0] + s * d1x - (q0[0] + t * d2x);
  const R cy = p0[1] + s * d1y - (q0[1] + t * d2y);
  const R cz = p0[2] + s * d1z - (q0[2] + t * d2z);
  return sqrt(cx * cx + cy * cy + cz * cz);
}

template <typename R>
__device__ __forceinline__ R point_box_dist(R px, R py, R pz, const R* bmin, const R* bmax) {
  // jit.py:263-268
  const R dx = fmax(bmin[0] - px, R(0)) + fmax(px - bmax[0], R(0));
  const R dy = fmax(bmin[1] - py, R(0)) + fmax(py - bmax[1], R(0));
  const R dz = fmax(bmin[2] - pz, R(0)) + fmax(pz - bmax[2], R(0));
  return sqrt(dx * dx + dy * dy + dz * dz);
}

// Segment/AABB distance by TERNARY_ITERS ternary-search steps (jit.py:271-286).
template <typename R>
__device__ __forceinline__ R seg_box_dist(const R* p0, const R* p1, const R* bmin, const R* bmax) {
  const R dx = p1[0] - p0[0], dy = p1[1] - p0[1], dz = p1[2] - p0[2];
  R lo = R(0), hi = R(1);
  for (int it = 0; it < TERNARY_ITERS; ++it) {
    const R m1 = lo + (hi - lo) / R(3);
    const R m2 = hi - (hi - lo) / R(3);
    const R f1 = point_box_dist(p0[0] + m1 * dx, p0[1] + m1 * dy, p0[2] + m1 * dz, bmin, bmax);
    const R f2 = point_box_dist(p0[0] + m2 * dx, p0[1] + m2 * dy, p0[2] + m2 * dz, bmin, bmax);
    if (f1 <= f2)
      hi = m2;
    else
      lo = m1;
  }
  const R mid = R(0.5) * (lo + hi);
  return point_box_dist(p0[0] + mid * dx, p0[1] + mid * dy, p0[2] + mid * dz, bmin, bmax);
}

// Capsule vs sphere, strict penetration (jit.py:306-322).
template <typename R>
__device__ __forceinline__ bool capsule_hits_sphere(const R* P0, const R* P1, R rcap, const R* sph) {
  const R dx = P1[0] - P0[0], dy = P1[1] - P0[1], dz = P1[2] - P0[2];
  const R dd = dx * dx + dy * dy + dz * dz;
  R t;
  if (dd <= R(SEG_EPS)) {
    t = R(0);
  } else {
    t = ((sph[0] - P0[0]) * dx + (sph[1] - P0[1]) * dy + (sph[2] - P0[2]) * dz) / dd;
    t = clamp01(t);
  }
  const R ex = P0[0] + t * dx - sph[0];
  const R ey = P0[1] + t * dy - sph[1];
  const R ez = P0[2] + t * dz - sph[2];
  return sqrt(ex * ex + ey * ey + ez * ez) < rcap + sph[3];
}

// ---------------------------------------------------------------- cluster push
// Distributed-shared-memory pushes that complete on the RECEIVER's mbarrier
// (st.async ... complete_tx): no cluster-wide fence, no L1 invalidation.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void push_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void push_f64x2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void cbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void cbar_arrive_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void cluster_init_fence_arrive() {
  asm volatile("fence.mbarrier_init.release.cluster;\n\tbarrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- programmatic dependent launch
// The step's kernels are chained with programmatic stream serialisation: a
// dependent grid may start (and run its prologue) while its predecessor
// drains, and blocks in pdl_wait() until the predecessor has completed and its
// writes are visible. pdl_trigger() lets the dependent grid be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// host side: which PDL features are on (MPPI_PDL bit mask, A/B switch):
// 1 = MLP after rollout, 2 = statistics after MLP/rollout, 4 = early triggers
enum { PDL_MLP = 1, PDL_STATS = 2, PDL_EARLY = 4 };
inline int pdl_mask() {
  static const int m = getenv("MPPI_PDL") ? atoi(getenv("MPPI_PDL")) : 0;
  return m;
}

// debug phase stamp (globaltimer ns) into dbg[k], compiled in with -DMPPI_DEBUG_TIMERS
#ifdef MPPI_DEBUG_TIMERS
#define MPPI_TSTAMP(ptr, k)                                      \
  do {                                                           \
    if ((ptr) != nullptr) {                                      \
      unsigned long long t_;                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));     \
      (ptr)[k] = t_;                                             \
    }                                                            \
  } while (0)
#else
#define MPPI_TSTAMP(ptr, k) \
  do {                      \
  } while (0)
#endif

// ---------------------------------------------------------------- warp helpers
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    T o = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v += o;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ bool finite_(double x) { return isfinite(x); }
__device__ __forceinline__ bool finite_(float x) { return isfinite(x); }

// ---------------------------------------------------------------- sampling math
// Acklam inverse-normal (sampling.py:146-202), float64.
__device__ __forceinline__ double acklam_icdf(double p) {
  const double a0 = -3.969683028665376e01, a1 = 2.209460984245205e02, a2 = -2.759285104469687e02,
               a3 = 1.383577518672690e02, a4 = -3.066479806614716e01, a5 = 2.506628277459239e00;
  const double b0 = -5.447609879822406e01, b1 = 1.615858368580409e02, b2 = -1.556989798598866e02,
               b3 = 6.680131188771972e01, b4 = -1.328068155288572e01;
  const double c0 = -7.784894002430293e-03, c1 = -3.223964580411365e-01, c2 = -2.400758277161838e00,
               c3 = -2.549732539343734e00, c4 = 4.374664141464968e00, c5 = 2.938163982698783e00;
  const double d0 = 7.784695709041462e-03, d1 = 3.224671290700398e-01, d2 = 2.445134137142996e00,
               d3 = 3.754408661907416e00;
  const double plow = 0.02425;
  if (p == 0.0) p = 4.9406564584124654e-324;  // np.nextafter(0, 1)
  if (p < plow) {
    const double q = sqrt(-2.0 * log(p));
    return (((((c0 * q + c1) * q + c2) * q + c3) * q + c4) * q + c5) /
           ((((d0 * q + d1) * q + d2) * q + d3) * q + 1.0);
  }
  if (p > 1.0 - plow) {
    const double q = sqrt(-2.0 * log(1.0 - p));
    return -(((((c0 * q + c1) * q + c2) * q + c3) * q + c4) * q + c5) /
           ((((d0 * q + d1) * q + d2) * q + d3) * q + 1.0);
  }
  const double q = p - 0.5, r = q * q;
  return (((((a0 * r + a1) * r + a2) * r + a3) * r + a4) * r + a5) * q /
         (((((b0 * r + b1) * r + b2) * r + b3) * r + b4) * r + 1.0);
}

// Base-p radical inverse of index in exact integer arithmetic followed by one
// correctly rounded divide — bit-identical to sampling.py:89-97 while
// num, denom < 2^53.
__device__ __forceinline__ double radical_inverse(uint64_t index, uint32_t base) {
  uint64_t num = 0, denom = 1;
  while (index > 0) {
    num = num * base + index % base;
    denom *= base;
    index /= base;
  }
  return (double)num / (double)denom;
}

__constant__ static const uint32_t kPrimes[40] = {
    2,  3,  5,  7,  11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71,
    73, 79, 83, 89, 97, 101, 103, 107, 109, 113, 127, 131, 137, 139, 149, 151, 157, 163, 167, 173};

// Philox4x32-10 (Salmon et al. 2011), used for the per-step pseudorandom set.
__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
    const uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += W0;
    key.y += W1;
  }
  return ctr;
}

// 53-bit uniform in [0,1) from two 32-bit words.
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  const uint64_t v = ((uint64_t)(a >> 5) << 26) | (uint64_t)(b >> 6);
  return (double)v * (1.0 / 9007199254740992.0);
}

}  // namespace mppi
