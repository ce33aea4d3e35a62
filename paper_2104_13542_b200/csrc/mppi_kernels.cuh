// mppi_kernels.cuh — the fused MPPI step kernels for sm_100a.
//
//   rollout_kernel  : policy shaping (sampling.py:268-290) + semi-implicit
//                     Euler (jit.py:335-349) + generic-chain FK (jit.py:89-111)
//                     + Jacobian/manipulability (jit.py:114-185) + capsule
//                     self collision (jit.py:241-260) + world collision
//                     (jit.py:289-332) + the cost stack (costs.py:76-187),
//                     one warp per particle, one lane per horizon step.
//   stats_kernel    : discounted totals + quarantine (rollout.py:111-171),
//                     exponentiated-utility weights (policy.py:103-121) and
//                     weighted sufficient statistics; the last block of each
//                     instance combines the block records and applies
//                     update_mean / update_covariance (policy.py:124-155),
//                     the shift (policy.py:158-167) and next_command
//                     (policy.py:170-177).
#pragma once

#include <cooperative_groups.h>
#include <type_traits>

#include "mppi_common.cuh"

namespace mppi {

constexpr int kRolloutWarps = 4;  // 128-thread blocks, one warp per particle
constexpr int kStatsThreads = 256;
constexpr int kRecHead = 6;       // m, S0, count, sum_finite, status, first bad row
// Statistics blocks of one instance combine their records in two levels when
// there are more than kStatsGroup of them: the last block of each group of
// kStatsGroup combines the group's records, the last group the group
// records (a single block combining ~300 records took 14-31 us). Records per
// instance: nblk block records + one per group; counters per instance: one
// for the instance + one per group.
constexpr int kStatsGroup = 16;
constexpr int kStatsMaxBlocks = 296;
constexpr int kStatsCounterStride = 1 + (kStatsMaxBlocks + kStatsGroup - 1) / kStatsGroup;
__host__ __device__ inline int stats_groups(int nblk) {
  return nblk > kStatsGroup ? (nblk + kStatsGroup - 1) / kStatsGroup : 0;
}
__host__ __device__ inline int stats_rec_stride(int nblk) { return nblk + stats_groups(nblk); }

// FP32 fast path of each revolute link: the joint rotation Rm(q) = I + s K +
// (1 - c) K^2 (Rodrigues, jit.py:70-86) enters the link transform only through
// Rm·orot and Rm·otrans, so those are folded on the host (float64) into
//   Rm·orot = O + s A + (1 - c) B,   Rm·otrans = t + s a + (1 - c) b
// with A = K orot, B = K^2 orot, a = K otrans, b = K^2 otrans: 12 instead of
// 45 FP32 operations per link for the rotation, generic over the chain data
// (no structural zeros assumed). Rows padded to 4 so column pairs load as one
// aligned 8-byte constant for FFMA2.
struct FkFold {
  float O[MAXD][3][4], A[MAXD][3][4], B[MAXD][3][4];
  float t[MAXD][4], a[MAXD][4], b[MAXD][4];
};

template <typename R>
struct RolloutArgs {
  FkFold fold;  // read by FP32 rollouts (see FkFold)
  ChainT<R> chain;
  CostT<R> cost;
  WorldT<R> world;
  R dts[MAXH];
  R remaining[MAXH];  // sum_{k>=h} dts[k] (costs.py:100), host fp64
  int H, N, B, null_count, particle_offset;
  int mode;       // 0: u = mu + sd*eps ; 1: u given (in0) ; 2: pos (in0) / vel (in1) given
  int shift;      // read the stored policy through the shift view
  int check_var;  // PolicyStateError check of build_control_batch (sampling.py:282)
  int skip_on_status;
  int pdl_early;  // trigger the dependent grid at entry
  int state_inline;  // single instance: theta, theta_dot travel in st0 (kernel parameter), not `state`,
  double st0[2 * MAXD];  // and the goal in g0, not `goal`
  double g0[16];
  double tail_mean, tail_sd;
  const double* eps;     // (N,H,d)
  const double* means;   // (B,H,d)
  const double* sd;      // (B,H,d)
  const double* state;   // (B,2d)
  const double* goal;    // (B,16): R(9) t(3) mode
  const double* in0;
  const double* in1;
  R* step;               // (B*N*H) step cost excluding the learned self-collision term
  float* mlp_x;          // (B*N*H,16) positional encoding (surrogate.py:24-28), or (B*N*H,8) joint
                         // positions when mlp_x_q (the MLP encodes them itself), or NULL
  int mlp_x_q;
  int* status;
  int* bad;
  double* out_pos;       // dumps, instance 0 only; (n,H,d)
  double* out_vel;
  double* out_acc;
  double* out_terms;     // (6,n,H)
  unsigned long long* dbg;  // debug phase stamps of the fused kernel (MPPI_DEBUG_TIMERS), else NULL
};

// Any capsule of this lane's configuration penetrates the world (costs.py:235-240).
// Capsule endpoints live in shared memory, [cap][6][32 lanes].
#ifdef MPPI_ENV_INLINE
#define MPPI_ENV_LINKAGE __forceinline__
#else  // out of line: config 1/2 rollouts never fetch the world code
#define MPPI_ENV_LINKAGE __noinline__
#endif
template <typename R>
__device__ MPPI_ENV_LINKAGE bool env_any_hit(const WorldT<R>& w, const ChainT<R>& ch, const R* cap,
                                            int lane, unsigned long long* dbg_counts = nullptr) {
  const int nc = ch.n_caps;
  // Capsule-level screen, one gather per capsule, all in flight together:
  // every point of a segment lies within len/2 of its midpoint, and the
  // midpoint's voxel clearance bounds the midpoint's distance to the boxes
  // (see the sampled broad phase below), so clearance - len/2 >= r + margin
  // clears the capsule of every box without sampling it.
  unsigned clear = 0;
  if (w.sdf != nullptr && w.nb > 0) {
    const R iv = R(1) / w.voxel;
    float f[MAXC];
    R hl[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      f[c] = 0.f;
      hl[c] = R(0);
      if (c < nc) {
        R m[3], d2 = R(0);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const R a0 = cap[(c * 6 + i) * 32 + lane], a1 = cap[(c * 6 + 3 + i) * 32 + lane];
          m[i] = R(0.5) * (a0 + a1);
          d2 += (a1 - a0) * (a1 - a0);
        }
        hl[c] = R(0.5) * sqrt(d2);
        int ix = (int)floor((m[0] - w.ox) * iv), iy = (int)floor((m[1] - w.oy) * iv),
            iz = (int)floor((m[2] - w.oz) * iv);
        ix = ix < 0 ? 0 : (ix >= w.nx ? w.nx - 1 : ix);
        iy = iy < 0 ? 0 : (iy >= w.ny ? w.ny - 1 : iy);
        iz = iz < 0 ? 0 : (iz >= w.nz ? w.nz - 1 : iz);
        f[c] = __ldg(w.sdf + (ix * w.ny + iy) * w.nz + iz);
      }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < nc && R(f[c]) - hl[c] >= ch.cap_r[c] + R(1e-5)) clear |= 1u << c;
  }
  for (int c = 0; c < nc; ++c) {
    R P0[3], P1[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      P0[i] = cap[(c * 6 + i) * 32 + lane];
      P1[i] = cap[(c * 6 + 3 + i) * 32 + lane];
    }
    const R rc = ch.cap_r[c];
    for (int o = 0; o < w.ns; ++o)
      if (capsule_hits_sphere(P0, P1, rc, w.spheres + 4 * o)) return true;
    if (w.nb == 0 || ((clear >> c) & 1u)) continue;
    if (w.sdf != nullptr) {
      // Conservative voxel broad phase. w.sdf holds, per voxel, the exact
      // distance from the voxel CUBE to the obstacle set (the union of the
      // boxes below), so every point of the cube is at least that far away.
      // A point outside the grid is no closer than its projection onto the
      // grid box (obstacles lie inside, projection onto a convex set).
      // Sample the segment every half voxel; every segment point is within
      // `half` of a sample, so min(clearance) - half >= r + margin proves no
      // strict penetration (jit.py:326) for every box and the exact narrow
      // phase is skipped. Anything else falls through to the exact test.
      const R dx = P1[0] - P0[0], dy = P1[1] - P0[1], dz = P1[2] - P0[2];
      const R len = sqrt(dx * dx + dy * dy + dz * dz);
      const int ns = 1 + (int)ceil(len / (R(0.5) * w.voxel));
      const R half = R(0.5) * len / R(ns > 1 ? ns - 1 : 1);
      // sample s sits at grid coordinate g0 + s * gs (voxel units): one FMA
      // per axis per sample instead of three divisions. Rounding moves a
      // sample by ~1e-7 voxel; a point on a voxel face may take either
      // neighbour, and both clearances bound it — the 1e-5 margin covers it.
      const R iv = R(1) / w.voxel, is = ns > 1 ? R(1) / R(ns - 1) : R(0);
      const R gx0 = (P0[0] - w.ox) * iv, gy0 = (P0[1] - w.oy) * iv, gz0 = (P0[2] - w.oz) * iv;
      const R gsx = dx * iv * is, gsy = dy * iv * is, gsz = dz * iv * is;
      // samples in batches of SB independent gathers
      constexpr int SB = 8;
      R lb = R(1e30);
      for (int s0 = 0; s0 < ns; s0 += SB) {
        float f[SB];
#pragma unroll
        for (int u = 0; u < SB; ++u) {
          const int s = s0 + u;
          f[u] = 1e30f;
          if (s < ns) {
            int ix = (int)floor(gx0 + R(s) * gsx);
            int iy = (int)floor(gy0 + R(s) * gsy);
            int iz = (int)floor(gz0 + R(s) * gsz);
            ix = ix < 0 ? 0 : (ix >= w.nx ? w.nx - 1 : ix);
            iy = iy < 0 ? 0 : (iy >= w.ny ? w.ny - 1 : iy);
            iz = iz < 0 ? 0 : (iz >= w.nz ? w.nz - 1 : iz);
            f[u] = __ldg(w.sdf + (ix * w.ny + iy) * w.nz + iz);
          }
        }
#pragma unroll
        for (int u = 0; u < SB; ++u) lb = R(f[u]) < lb ? R(f[u]) : lb;
      }
      if (lb - half >= rc + R(1e-5)) continue;
    }
#ifdef MPPI_DEBUG_TIMERS
    if (dbg_counts) atomicAdd(dbg_counts + c, 1ull);  // (configuration, capsule) pairs reaching the exact test
#endif
    // Exact narrow phase (60 ternary steps per box), skipped for boxes whose
    // gap to the segment's bounding box already exceeds the radius: every
    // point the ternary search evaluates lies in that bounding box, so its
    // distance cannot fall below the gap (margin as in the broad phase).
    const R rlim = rc + R(1e-5);
    for (int ob = 0; ob < w.nb; ++ob) {
      const R* bx = w.boxes + 6 * ob;
      R g2 = R(0);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const R smin = P0[i] < P1[i] ? P0[i] : P1[i], smax = P0[i] < P1[i] ? P1[i] : P0[i];
        const R gi = fmax(bx[i] - smax, R(0)) + fmax(smin - bx[3 + i], R(0));
        g2 += gi * gi;
      }
      if (g2 >= rlim * rlim) continue;
#ifdef MPPI_DEBUG_TIMERS
      if (dbg_counts) atomicAdd(dbg_counts + 15, 1ull);  // ternary searches run
#endif
      if (seg_box_dist(P0, P1, bx, bx + 3) < rc) return true;
    }
  }
  return false;
}

// Capsule endpoints are staged in shared memory only when a cost term reads
// them (world collision, capsule self-collision).
template <typename R>
__host__ __device__ __forceinline__ bool rollout_needs_caps(const CostT<R>& cs) {
  return cs.use_env || cs.selfcoll == MPPI_SELFCOLL_ORACLE;
}

// Rollout + cost stack of particle g (one warp, lane = horizon step h), the
// body of rollout_kernel and of the fused rollout + MLP kernel. `cap` is this
// warp's [cap][6][32] staging area; `enc` (16 floats, may be NULL) receives the
// lane's positional encoding [sin q, cos q, 0...] (surrogate.py:24-28).
// Returns false when the instance already failed (nothing written).
// LEAN: the control-step specialisation — sampled controls (mode 0), no
// capsule staging, no capsule self-collision oracle, no world — so the
// kernel's code holds only what a config-1/2 step executes (the latency
// build fetches its instructions cold after an L2 flush).
// FOLD: the FkFold link transform (FP32 only) — taken by the many-waves
// throughput build, where it saves issue slots (config 4 rollout -2 %); the
// latency build keeps the Rodrigues form, whose operands are already in
// registers (the fold's extra per-thread constant loads cost the cold
// 500 x 30 step ~0.5 us).
template <typename R, int D, bool LEAN = false, bool FOLD = false>
__device__ __forceinline__ bool rollout_particle(const RolloutArgs<R>& a, long long g, int lane, R* cap,
                                                 float* enc) {
  const int b = (int)(g / a.N);
  const int n = (int)(g - (long long)b * a.N);
  // Every global input of the warp is requested up front and the status word
  // is tested only once the control loads are in flight: after an L2 flush
  // each of these is an HBM round trip, and taken one after another they
  // were the largest part of the rollout's latency.
  const int status_b = a.skip_on_status ? a.status[b] : 0;
  const int H = a.H;
  const bool act = lane < H;
  const int h = act ? lane : H - 1;
  const ChainT<R>& ch = a.chain;
  const CostT<R>& cs = a.cost;
  const double* st = a.state_inline ? a.st0 : a.state + (size_t)b * 2 * D;
  R st_p[D], st_v[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    st_p[j] = (R)st[j];
    st_v[j] = (R)st[D + j];
  }
  const double* gl = a.state_inline ? a.g0 : a.goal + (size_t)b * 16;
  R Rg[9], tg[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) Rg[i] = (R)gl[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) tg[i] = (R)gl[9 + i];
  const int gmode = (int)gl[12];

  // ---- controls -> positions / velocities --------------------------------
  R p[D], v[D], u[D];
  const size_t row = ((size_t)n * H + h) * D;
  if (!LEAN && a.mode == 2) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      p[j] = (R)a.in0[row + j];
      v[j] = (R)a.in1[row + j];
      u[j] = R(0);
    }
    if (status_b != 0) return false;
  } else {
    bool bad = false, varbad = false;
    const int ng = n + a.particle_offset;
    if (LEAN || a.mode == 0) {
      const int hs = a.shift ? h + 1 : h;
      const double* mu = a.means + (size_t)b * H * D;
      const double* sdv = a.sd + (size_t)b * H * D;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double m = hs < H ? mu[hs * D + j] : a.tail_mean;
        const double s = hs < H ? sdv[hs * D + j] : a.tail_sd;
        varbad |= (s <= 0.0);
        double uu;
        if (ng < a.null_count)
          uu = 0.0;
        else if (ng == a.null_count)
          uu = m;
        else
          uu = m + s * a.eps[row + j];
        bad |= !isfinite(uu);
        u[j] = (R)uu;
      }
    } else {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double uu = a.in0[row + j];
        bad |= !isfinite(uu);
        u[j] = (R)uu;
      }
    }
    if (status_b != 0) return false;  // the instance already failed (an earlier iteration)
    const unsigned badm = __ballot_sync(0xffffffffu, act && bad);
    const unsigned varm = __ballot_sync(0xffffffffu, act && varbad);
#ifdef MPPI_DEBUG_TIMERS
    if (a.dbg != nullptr && threadIdx.x == 0 && blockIdx.x < 256) MPPI_TSTAMP(a.dbg + 16 * blockIdx.x, 5);  // controls formed
#endif
    if (lane == 0 && a.status != nullptr) {
      if (varm && a.check_var && n == 0) atomicMax(&a.status[b], (int)MPPI_E_NONPOSITIVE_VARIANCE);
      if (badm) {
        atomicMin(&a.bad[b], ng);
        atomicMax(&a.status[b], (int)MPPI_E_NONFINITE_CONTROL);
      }
    }
    // semi-implicit Euler as two inclusive warp scans over the horizon
    const R dt = act ? a.dts[h] : R(0);
#pragma unroll
    for (int j = 0; j < D; ++j) v[j] = st_v[j] + warp_inclusive_scan(dt * u[j], lane);
#ifdef MPPI_DEBUG_TIMERS
    if (a.dbg != nullptr && threadIdx.x == 0 && blockIdx.x < 256 && v[D - 1] != R(12345)) MPPI_TSTAMP(a.dbg + 16 * blockIdx.x, 6);
#endif
#pragma unroll
    for (int j = 0; j < D; ++j) p[j] = st_p[j] + warp_inclusive_scan(dt * v[j], lane);
  }

#ifdef MPPI_DEBUG_TIMERS
  unsigned long long* pdbg = (a.dbg != nullptr && threadIdx.x == 0 && blockIdx.x < 256) ? a.dbg + 16 * blockIdx.x
                                                                                         : nullptr;
#endif
  MPPI_TSTAMP(pdbg, 2);  // controls and integration issued
  // ---- forward kinematics, link by link in registers ----------------------
  R Rw[9] = {R(1), R(0), R(0), R(0), R(1), R(0), R(0), R(0), R(1)};
  R tw[3] = {R(0), R(0), R(0)};
  R ja[D][3], jp[D][3];  // Jacobian column data: world axis, joint origin
  R sq[D], cq[D];
  const int nc = (!LEAN && rollout_needs_caps(cs)) ? ch.n_caps : 0;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    ja[0][j] = ch.axes[0][j];
    jp[0][j] = R(0);
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    R Rmo[9], tmo[3];
    R s, c;
    sincos_(p[k], &s, &c);
    sq[k] = s;
    cq[k] = c;
    if (ch.jtype[k] == 0) {
      bool folded = false;
#ifndef MPPI_FK_UNFOLDED  // (A/B build: the Rodrigues form for FP32 too)
      if constexpr (FOLD && std::is_same<R, float>::value) {
        {  // FkFold: Rmo = O + s A + c1 B, tmo = t + s a + c1 b
          const FkFold& f = a.fold;
          const float c1 = 1.f - c;
          const float2 s2 = make_float2(s, s), c2 = make_float2(c1, c1);
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const float2 r = __ffma2_rn(c2, make_float2(f.B[k][i][0], f.B[k][i][1]),
                                        __ffma2_rn(s2, make_float2(f.A[k][i][0], f.A[k][i][1]),
                                                   make_float2(f.O[k][i][0], f.O[k][i][1])));
            Rmo[3 * i] = r.x;
            Rmo[3 * i + 1] = r.y;
            Rmo[3 * i + 2] = fmaf(c1, f.B[k][i][2], fmaf(s, f.A[k][i][2], f.O[k][i][2]));
          }
          const float2 tt = __ffma2_rn(c2, make_float2(f.b[k][0], f.b[k][1]),
                                       __ffma2_rn(s2, make_float2(f.a[k][0], f.a[k][1]),
                                                  make_float2(f.t[k][0], f.t[k][1])));
          tmo[0] = tt.x;
          tmo[1] = tt.y;
          tmo[2] = fmaf(c1, f.b[k][2], fmaf(s, f.a[k][2], f.t[k][2]));
          folded = true;
        }
      }
#endif
      if (!folded) {
        R Rm[9];
        axis_rotation(ch.axes[k], s, R(1) - c, Rm);
        mat33_mul(Rm, ch.orot[k], Rmo);
        mat33_vec(Rm, ch.otrans[k], tmo);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 9; ++i) Rmo[i] = ch.orot[k][i];
#pragma unroll
      for (int i = 0; i < 3; ++i) tmo[i] = p[k] * ch.axes[k][i] + ch.otrans[k][i];
    }
    R dtw[3];
    mat33_vec(Rw, tmo, dtw);
#pragma unroll
    for (int i = 0; i < 3; ++i) tw[i] = tw[i] + dtw[i];
    R Rn[9];
    mat33_mul(Rw, Rmo, Rn);
#pragma unroll
    for (int i = 0; i < 9; ++i) Rw[i] = Rn[i];
    if ((k + 1) % REORTHO_EVERY == 0) orthonormalize(Rw);
    if (k + 1 < D) {
      mat33_vec(Rw, ch.axes[k + 1], ja[k + 1]);
#pragma unroll
      for (int i = 0; i < 3; ++i) jp[k + 1][i] = tw[i];
    }
    for (int ci = 0; ci < nc; ++ci) {
      if (ch.cap_link[ci] != k) continue;
      R q0[3], q1[3];
      mat33_vec(Rw, ch.cap_p0[ci], q0);
      mat33_vec(Rw, ch.cap_p1[ci], q1);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        cap[(ci * 6 + i) * 32 + lane] = q0[i] + tw[i];
        cap[(ci * 6 + 3 + i) * 32 + lane] = q1[i] + tw[i];
      }
    }
  }
  __syncwarp();

  MPPI_TSTAMP(pdbg, 3);  // forward kinematics
  // ---- cost terms -----------------------------------------------------------
  // pose (costs.py:76-95)
  R pose;
  {
    const R e0 = tw[0] - tg[0], e1 = tw[1] - tg[1], e2 = tw[2] - tg[2];
    R acc = R(0);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const R di = Rg[0 * 3 + i] * e0 + Rg[1 * 3 + i] * e1 + Rg[2 * 3 + i] * e2;
      const R wi = cs.alpha_trans[i] * di;
      acc += wi * wi;
    }
    pose = sqrt(acc);
    if (gmode != MPPI_GOAL_POSITION_ONLY) {
      R racc = R(0);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const R rr = Rg[0 * 3 + i] * Rw[0 * 3 + kk] + Rg[1 * 3 + i] * Rw[1 * 3 + kk] +
                       Rg[2 * 3 + i] * Rw[2 * 3 + kk];
          const R res = cs.alpha_rot[i] * ((i == kk ? R(1) : R(0)) - rr);
          racc += res * res;
        }
      pose = pose + sqrt(racc);
    }
  }
  // stop (costs.py:98-108)
  R stop = R(0);
  if (cs.use_stop) {
    R acc = R(0);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const R lim = a.remaining[h] * ch.accel[j];
      R ex = fabs(v[j]) - lim;
      ex = ex > R(0) ? ex : R(0);
      acc += ex * ex;
    }
    stop = sqrt(acc);
  }
  // joint limits (costs.py:111-123)
  R joint = R(0);
  if (cs.use_joint) {
    R acc = R(0);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      R lo = ch.lo[j] - p[j];
      lo = lo > R(0) ? lo : R(0);
      R hi = p[j] - ch.hi[j];
      hi = hi > R(0) ? hi : R(0);
      const R dep = lo + hi;
      acc += dep * dep;
    }
    joint = sqrt(acc);
  }
  // manipulability (jit.py:114-185, costs.py:126-127)
  R manip = R(0);
  if (cs.use_manip) {
    R J[3][D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if (ch.jtype[k] == 0) {
        const R rx = tw[0] - jp[k][0], ry = tw[1] - jp[k][1], rz = tw[2] - jp[k][2];
        J[0][k] = ja[k][1] * rz - ja[k][2] * ry;
        J[1][k] = ja[k][2] * rx - ja[k][0] * rz;
        J[2][k] = ja[k][0] * ry - ja[k][1] * rx;
      } else {
        J[0][k] = ja[k][0];
        J[1][k] = ja[k][1];
        J[2][k] = ja[k][2];
      }
    }
    const int td = ch.task_dim;
    R m;
    if (D == td) {
      R det;
      if (td == 2)
        det = J[0][0] * J[1][1 % D] - J[0][1 % D] * J[1][0];
      else
        det = J[0][0] * (J[1][1 % D] * J[2][2 % D] - J[1][2 % D] * J[2][1 % D]) -
              J[0][1 % D] * (J[1][0] * J[2][2 % D] - J[1][2 % D] * J[2][0]) +
              J[0][2 % D] * (J[1][0] * J[2][1 % D] - J[1][1 % D] * J[2][0]);
      m = fabs(det);
    } else {
      R G[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          R acc = R(0);
#pragma unroll
          for (int k = 0; k < D; ++k) acc += J[i][k] * J[j][k];
          G[i][j] = acc;
        }
      R det;
      if (td == 2)
        det = G[0][0] * G[1][1] - G[0][1] * G[1][0];
      else
        det = G[0][0] * (G[1][1] * G[2][2] - G[1][2] * G[2][1]) -
              G[0][1] * (G[1][0] * G[2][2] - G[1][2] * G[2][0]) +
              G[0][2] * (G[1][0] * G[2][1] - G[1][1] * G[2][0]);
      m = sqrt(det > R(0) ? det : R(0));
    }
    manip = m < cs.k_m ? R(1) - m : R(0);
  }
  // capsule self collision oracle (jit.py:241-260, costs.py:234)
  R selfc = R(0);
  if (!LEAN && cs.selfcoll == MPPI_SELFCOLL_ORACLE) {
    R best = R(NO_CONTACT);
    for (int pi = 0; pi < ch.n_pairs; ++pi) {
      const int i = ch.pair_a[pi], j = ch.pair_b[pi];
      R a0[3], a1[3], b0[3], b1[3];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        a0[t] = cap[(i * 6 + t) * 32 + lane];
        a1[t] = cap[(i * 6 + 3 + t) * 32 + lane];
        b0[t] = cap[(j * 6 + t) * 32 + lane];
        b1[t] = cap[(j * 6 + 3 + t) * 32 + lane];
      }
      const R val = ch.cap_r[i] + ch.cap_r[j] - segseg_dist(a0, a1, b0, b1);
      if (val > best) best = val;
    }
    selfc = best > R(0) ? best : R(0);
  }
  // world collision, binary (jit.py:289-332, costs.py:235-240)
  R envc = R(0);
#ifdef MPPI_DEBUG_TIMERS
  if (!LEAN && cs.use_env)
    envc = env_any_hit(a.world, ch, cap, lane, a.dbg ? a.dbg + 16 * 253 : nullptr) ? R(1) : R(0);
#else
  if (!LEAN && cs.use_env) envc = env_any_hit(a.world, ch, cap, lane) ? R(1) : R(0);
#endif

  MPPI_TSTAMP(pdbg, 4);  // cost terms
  // total_cost (costs.py:176-187) minus the learned self-collision term
  const R stepc = pose + cs.a_stop * stop + cs.a_joint * joint + cs.a_manip * manip +
                  cs.a_coll * (selfc + envc);

  if (act) {
    const size_t m = (size_t)g * H + h;
    a.step[m] = stepc;
    if (a.mlp_x != nullptr && a.mlp_x_q) {  // one 32-byte row of positions: the MLP's X loader
      float xr[8];                           // computes [sin q, cos q] with the same sincos_
#pragma unroll
      for (int k = 0; k < 8; ++k) xr[k] = k < D ? (float)p[k] : 0.f;
      float4* x4 = reinterpret_cast<float4*>(a.mlp_x + m * 8);
      x4[0] = make_float4(xr[0], xr[1], xr[2], xr[3]);
      x4[1] = make_float4(xr[4], xr[5], xr[6], xr[7]);
    } else if (a.mlp_x != nullptr) {  // one 64-byte row, four 16-byte stores
      float xr[16];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        xr[k] = (float)sq[k];
        xr[D + k] = (float)cq[k];
      }
#pragma unroll
      for (int k = 2 * D; k < 16; ++k) xr[k] = 0.f;
      float4* x4 = reinterpret_cast<float4*>(a.mlp_x + m * 16);
#pragma unroll
      for (int q = 0; q < 4; ++q) x4[q] = make_float4(xr[4 * q], xr[4 * q + 1], xr[4 * q + 2], xr[4 * q + 3]);
    }
    if (enc != nullptr) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        enc[k] = (float)sq[k];
        enc[D + k] = (float)cq[k];
      }
    }
    if (a.out_pos != nullptr && b == 0) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        a.out_pos[row + j] = (double)p[j];
        a.out_vel[row + j] = (double)v[j];
        if (a.out_acc) a.out_acc[row + j] = (double)u[j];
      }
    }
    if (a.out_terms != nullptr && b == 0) {
      const size_t nh = (size_t)a.N * H, o = (size_t)n * H + h;
      a.out_terms[T_POSE * nh + o] = (double)pose;
      a.out_terms[T_STOP * nh + o] = (double)stop;
      a.out_terms[T_JOINT * nh + o] = (double)joint;
      a.out_terms[T_MANIP * nh + o] = (double)manip;
      a.out_terms[T_SELF * nh + o] = (double)selfc;
      a.out_terms[T_ENV * nh + o] = (double)envc;
    }
  }
  return true;
}

// Paired throughput rollout (FP32, control steps of configs 1/2, no bundle
// dumps): particles g and g+1 of one instance in one warp, lane = horizon
// step, both configurations of a lane in packed pairs (P2): every FMA of the
// integration, forward kinematics (FkFold link transform), Jacobian and cost
// stack is one FFMA2 for the two particles; sine/cosine, square roots and the
// branch decisions stay per particle. Same operations per configuration as
// rollout_particle<float, D, true, true> (step costs within FP32 rounding of
// it; the contraction pattern of each sum is the compiler's in both).
__device__ __forceinline__ P2 warp_inclusive_scan2(P2 v, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float a = __shfl_up_sync(0xffffffffu, v.lo(), off);
    const float b = __shfl_up_sync(0xffffffffu, v.hi(), off);
    if (lane >= off) v += P2(a, b);
  }
  return v;
}

template <int D>
__device__ __forceinline__ void rollout_pair(const RolloutArgs<float>& a, long long g, int lane) {
  const int b = (int)(g / a.N);
  const int n = (int)(g - (long long)b * a.N);  // particles n and n + 1 of instance b
  const int status_b = a.skip_on_status ? a.status[b] : 0;
  const int H = a.H;
  const bool act = lane < H;
  const int h = act ? lane : H - 1;
  const ChainT<float>& ch = a.chain;
  const CostT<float>& cs = a.cost;
  const double* st = a.state_inline ? a.st0 : a.state + (size_t)b * 2 * D;
  float st_p[D], st_v[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    st_p[j] = (float)st[j];
    st_v[j] = (float)st[D + j];
  }
  const double* gl = a.state_inline ? a.g0 : a.goal + (size_t)b * 16;
  float Rg[9], tg[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) Rg[i] = (float)gl[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) tg[i] = (float)gl[9 + i];
  const int gmode = (int)gl[12];

  // ---- controls (sampling.py:268-290) -> positions / velocities
  P2 u[D];
  bool bad0 = false, bad1 = false, varbad = false;
  const int ng = n + a.particle_offset;
  {
    const int hs = a.shift ? h + 1 : h;
    const double* mu = a.means + (size_t)b * H * D;
    const double* sdv = a.sd + (size_t)b * H * D;
    const size_t row0 = ((size_t)n * H + h) * D, row1 = row0 + (size_t)H * D;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double m = hs < H ? mu[hs * D + j] : a.tail_mean;
      const double s = hs < H ? sdv[hs * D + j] : a.tail_sd;
      varbad |= (s <= 0.0);
      const double e0 = a.eps[row0 + j], e1 = a.eps[row1 + j];
      const double u0 = ng < a.null_count ? 0.0 : (ng == a.null_count ? m : m + s * e0);
      const double u1 = ng + 1 < a.null_count ? 0.0 : (ng + 1 == a.null_count ? m : m + s * e1);
      bad0 |= !isfinite(u0);
      bad1 |= !isfinite(u1);
      u[j] = P2((float)u0, (float)u1);
    }
  }
  if (status_b != 0) return;  // the instance already failed (an earlier iteration)
  {
    const unsigned bm0 = __ballot_sync(0xffffffffu, act && bad0);
    const unsigned bm1 = __ballot_sync(0xffffffffu, act && bad1);
    const unsigned varm = __ballot_sync(0xffffffffu, act && varbad);
    if (lane == 0 && a.status != nullptr) {
      if (varm && a.check_var && n == 0) atomicMax(&a.status[b], (int)MPPI_E_NONPOSITIVE_VARIANCE);
      if (bm0 | bm1) {
        atomicMin(&a.bad[b], bm0 ? ng : ng + 1);
        atomicMax(&a.status[b], (int)MPPI_E_NONFINITE_CONTROL);
      }
    }
  }
  P2 v[D], p[D];
  {
    const P2 dt(act ? a.dts[h] : 0.f);
#pragma unroll
    for (int j = 0; j < D; ++j) v[j] = P2(st_v[j]) + warp_inclusive_scan2(dt * u[j], lane);
#pragma unroll
    for (int j = 0; j < D; ++j) p[j] = P2(st_p[j]) + warp_inclusive_scan2(dt * v[j], lane);
  }

  // ---- forward kinematics (FkFold for revolute links), Jacobian column data
  P2 Rw[9] = {P2(1.f), P2(0.f), P2(0.f), P2(0.f), P2(1.f), P2(0.f), P2(0.f), P2(0.f), P2(1.f)};
  P2 tw[3] = {P2(0.f), P2(0.f), P2(0.f)};
  P2 ja[D][3], jp[D][3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    ja[0][j] = P2(ch.axes[0][j]);
    jp[0][j] = P2(0.f);
  }
  const FkFold& f = a.fold;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    P2 Rmo[9], tmo[3];
    if (ch.jtype[k] == 0) {
      float s0, c0, s1, c1;
      sincos_(p[k].lo(), &s0, &c0);
      sincos_(p[k].hi(), &s1, &c1);
      const P2 s(s0, s1), cm(1.f - c0, 1.f - c1);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int jj = 0; jj < 3; ++jj)
          Rmo[3 * i + jj] = P2(f.O[k][i][jj]) + s * P2(f.A[k][i][jj]) + cm * P2(f.B[k][i][jj]);
#pragma unroll
      for (int i = 0; i < 3; ++i) tmo[i] = P2(f.t[k][i]) + s * P2(f.a[k][i]) + cm * P2(f.b[k][i]);
    } else {
#pragma unroll
      for (int i = 0; i < 9; ++i) Rmo[i] = P2(ch.orot[k][i]);
#pragma unroll
      for (int i = 0; i < 3; ++i) tmo[i] = p[k] * P2(ch.axes[k][i]) + P2(ch.otrans[k][i]);
    }
    P2 dtw[3];
    mat33_vec(Rw, tmo, dtw);
#pragma unroll
    for (int i = 0; i < 3; ++i) tw[i] = tw[i] + dtw[i];
    P2 Rn[9];
    mat33_mul(Rw, Rmo, Rn);
#pragma unroll
    for (int i = 0; i < 9; ++i) Rw[i] = Rn[i];
    if ((k + 1) % REORTHO_EVERY == 0) orthonormalize(Rw);
    if (k + 1 < D) {
      P2 axk[3] = {P2(ch.axes[k + 1][0]), P2(ch.axes[k + 1][1]), P2(ch.axes[k + 1][2])};
      mat33_vec(Rw, axk, ja[k + 1]);
#pragma unroll
      for (int i = 0; i < 3; ++i) jp[k + 1][i] = tw[i];
    }
  }

  // ---- cost terms (costs.py:76-187), as rollout_particle
  P2 pose;
  {
    const P2 e0 = tw[0] - P2(tg[0]), e1 = tw[1] - P2(tg[1]), e2 = tw[2] - P2(tg[2]);
    P2 acc(0.f);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const P2 di = P2(Rg[0 * 3 + i]) * e0 + P2(Rg[1 * 3 + i]) * e1 + P2(Rg[2 * 3 + i]) * e2;
      const P2 wi = P2(cs.alpha_trans[i]) * di;
      acc = acc + wi * wi;
    }
    pose = sqrt2(acc);
    if (gmode != MPPI_GOAL_POSITION_ONLY) {
      P2 racc(0.f);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const P2 rr = P2(Rg[0 * 3 + i]) * Rw[0 * 3 + kk] + P2(Rg[1 * 3 + i]) * Rw[1 * 3 + kk] +
                        P2(Rg[2 * 3 + i]) * Rw[2 * 3 + kk];
          const P2 res = P2(cs.alpha_rot[i]) * (P2(i == kk ? 1.f : 0.f) - rr);
          racc = racc + res * res;
        }
      pose = pose + sqrt2(racc);
    }
  }
  P2 stop(0.f);
  if (cs.use_stop) {
    P2 acc(0.f);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const P2 ex = max0(fabs2(v[j]) - P2(a.remaining[h] * ch.accel[j]));
      acc = acc + ex * ex;
    }
    stop = sqrt2(acc);
  }
  P2 joint(0.f);
  if (cs.use_joint) {
    P2 acc(0.f);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const P2 dep = max0(P2(ch.lo[j]) - p[j]) + max0(p[j] - P2(ch.hi[j]));
      acc = acc + dep * dep;
    }
    joint = sqrt2(acc);
  }
  P2 manip(0.f);
  if (cs.use_manip) {
    P2 J[3][D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if (ch.jtype[k] == 0) {
        const P2 rx = tw[0] - jp[k][0], ry = tw[1] - jp[k][1], rz = tw[2] - jp[k][2];
        J[0][k] = ja[k][1] * rz - ja[k][2] * ry;
        J[1][k] = ja[k][2] * rx - ja[k][0] * rz;
        J[2][k] = ja[k][0] * ry - ja[k][1] * rx;
      } else {
        J[0][k] = ja[k][0];
        J[1][k] = ja[k][1];
        J[2][k] = ja[k][2];
      }
    }
    const int td = ch.task_dim;
    P2 m;
    if (D == td) {
      P2 det;
      if (td == 2)
        det = J[0][0] * J[1][1 % D] - J[0][1 % D] * J[1][0];
      else
        det = J[0][0] * (J[1][1 % D] * J[2][2 % D] - J[1][2 % D] * J[2][1 % D]) -
              J[0][1 % D] * (J[1][0] * J[2][2 % D] - J[1][2 % D] * J[2][0]) +
              J[0][2 % D] * (J[1][0] * J[2][1 % D] - J[1][1 % D] * J[2][0]);
      m = fabs2(det);
    } else {
      P2 G[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          P2 acc(0.f);
#pragma unroll
          for (int k = 0; k < D; ++k) acc = acc + J[i][k] * J[j][k];
          G[i][j] = acc;
        }
      P2 det;
      if (td == 2)
        det = G[0][0] * G[1][1] - G[0][1] * G[1][0];
      else
        det = G[0][0] * (G[1][1] * G[2][2] - G[1][2] * G[2][1]) -
              G[0][1] * (G[1][0] * G[2][2] - G[1][2] * G[2][0]) +
              G[0][2] * (G[1][0] * G[2][1] - G[1][1] * G[2][0]);
      m = sqrt2(max0(det));
    }
    const float m0 = m.lo(), m1 = m.hi();
    manip = P2(m0 < cs.k_m ? 1.f - m0 : 0.f, m1 < cs.k_m ? 1.f - m1 : 0.f);
  }
  // total_cost (costs.py:176-187) minus the learned self-collision term
  const P2 stepc = pose + P2(cs.a_stop) * stop + P2(cs.a_joint) * joint + P2(cs.a_manip) * manip;
  if (act) {
    const size_t m0 = (size_t)g * H + h, m1 = m0 + H;
    a.step[m0] = stepc.lo();
    a.step[m1] = stepc.hi();
    if (a.mlp_x != nullptr) {  // 32-byte position rows of both particles (mlp_x_q)
      float4* x0 = reinterpret_cast<float4*>(a.mlp_x + m0 * 8);
      float4* x1 = reinterpret_cast<float4*>(a.mlp_x + m1 * 8);
      float q0[8], q1[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        q0[j] = j < D ? p[j].lo() : 0.f;
        q1[j] = j < D ? p[j].hi() : 0.f;
      }
      x0[0] = make_float4(q0[0], q0[1], q0[2], q0[3]);
      x0[1] = make_float4(q0[4], q0[5], q0[6], q0[7]);
      x1[0] = make_float4(q1[0], q1[1], q1[2], q1[3]);
      x1[1] = make_float4(q1[4], q1[5], q1[6], q1[7]);
    }
  }
}

#ifndef MPPI_PAIR_MINB
#define MPPI_PAIR_MINB 3
#endif
template <int D>
__global__ void __launch_bounds__(kRolloutWarps * 32, MPPI_PAIR_MINB)
    rollout_pair_kernel(const __grid_constant__ RolloutArgs<float> a) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long g = 2 * ((long long)blockIdx.x * kRolloutWarps + wib);
  if (g >= (long long)a.B * a.N) return;  // warp-uniform exit
  rollout_pair<D>(a, g, lane);
}

// MINB = 1: the latency build (128 registers, one warp per particle and at
// most one wave); MINB = 6: the throughput build for many waves (80
// registers, a few spills, 6 CTAs per SM to hide the FK dependency chains;
// config 4 rollout -6%).
template <typename R, int D, int MINB = 1, bool LEAN = false>
__global__ void __launch_bounds__(kRolloutWarps * 32, MINB)
    rollout_kernel(const __grid_constant__ RolloutArgs<R> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (a.pdl_early) pdl_trigger();  // the MLP / statistics grids may be scheduled as SMs free up
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long g = (long long)blockIdx.x * kRolloutWarps + wib;
  if (g >= (long long)a.B * a.N) return;  // warp-uniform exit
  unsigned long long* dbg =
      (a.dbg != nullptr && threadIdx.x == 0 && blockIdx.x < 256) ? a.dbg + 16 * blockIdx.x : nullptr;
  MPPI_TSTAMP(dbg, 0);
  R* cap = reinterpret_cast<R*>(smem_raw) + (size_t)wib * a.chain.n_caps * 6 * 32;
  rollout_particle<R, D, LEAN, (MINB > 1)>(a, g, lane, cap, nullptr);
  MPPI_TSTAMP(dbg, 1);
#ifdef MPPI_DEBUG_TIMERS
  if (a.dbg != nullptr && lane == 0) {  // latest warp end over the grid
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    atomicMax(&a.dbg[16 * 255 + 15], t_);
  }
#endif
}

// ============================================================== statistics
template <typename R>
struct StatsArgs {
  int H, N, B, D, null_count, particle_offset, ppb, nblk;
  int shift, learned, totals_only, finalize_inline, isotropic, raw_step;
  int reset_status;  // last iteration of a step: re-arm status/bad for the next step
  double beta, alpha_mu, alpha_sigma, smin, smax, a_coll;
  double tail_mean, tail_var, tail_sd;
  double disc[MAXH];   // gamma^h (numpy power), h < H-1
  double dlast;        // gamma^(H-1) * terminal_weight
  const R* step;       // (B*N*H)
  const float* mlp_d;  // (B*N*H) learned distance, or NULL
  const double* eps;   // (N,H,d)
  double* means;       // (B,H,d) policy storage, updated in place
  double* var;
  double* sd;
  double* prev_means;  // (B,H,d) the view used by this iteration
  double* prev_sd;
  double* totals;      // (B*N)
  double* records;     // (B,nblk,reclen)
  double* out_record;  // (B,reclen) when !finalize_inline
  unsigned* counters;  // (B)
  int* status;
  int* bad;
  double* cmd;         // (B,d)
  mppi_step_info* info;
  double* dump_step;   // (N,H) instance 0
  double* dump_terms;  // (6,N,H) instance 0 (selfcoll row written for learned)
  double* dump_weights;  // (N) instance 0
  unsigned long long* dbg;  // debug phase timers (globaltimer ns), NULL in production
  // Particle-sharded exchange over peer memory (config 5, mppi_step_exchange):
  // when peer_recv is set the rank record is not written to out_record but
  // pushed into slot [rank] of every rank's receive buffer (NVLink P2P
  // stores), published by a release store of `seq` into every rank's flag
  // [rank]; the block then waits for all `world` flags and applies the update
  // itself (exchange_and_finalize). Receive buffers are [2][world][reclen]
  // (parity of seq), flags [world] u64, monotonically increasing.
  double* const* peer_recv;               // [world] device pointers (peer mappings)
  unsigned long long* const* peer_flags;  // [world]
  const double* my_recv;
  const unsigned long long* my_flags;
  int world, rank;
  unsigned long long seq;
  unsigned long long peer_timeout_ns;  // bounded wait for the other ranks' flags
};

// Flag word of the peer exchange: the sequence number a rank has published,
// with kPeerAbort set when that rank gave up on the step (a host-side failure
// before its kernel ran, or its own wait timed out). A waiter for sequence s
// fails fast on an abort published for any s' >= s.
constexpr unsigned long long kPeerAbort = 1ull << 63;

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double block_min_d(double v, double* red) {
  for (int off = 16; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? red[l] : CUDART_INF;
    for (int off = 16; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

// Fixed-order combine of `count` statistics records (each relative to its own
// minimum) into one record relative to the global minimum. Deterministic:
// every sum runs in record order. (§8(e): rescale by exp(-(m_k - m)/beta).)
static __device__ void combine_records(const double* recs, int count, int reclen, int HD, double beta,
                                       double* out, double* scale_smem, double* red) {
  // Latency-oriented: ONE parallel load of every record head into shared
  // memory, the record columns are preloaded (16 in flight per thread) while
  // warp 0 derives the global minimum and the rescale factors.
  double* hs = scale_smem + max(count, 8);  // record heads follow the scales (host sizes both)
  for (int t = threadIdx.x; t < count * kRecHead; t += blockDim.x)
    hs[t] = recs[(size_t)(t / kRecHead) * reclen + (t % kRecHead)];
  constexpr int CB = 16;
  const int o0 = threadIdx.x, o1 = threadIdx.x + blockDim.x;
  double v0[CB], v1[CB];
#pragma unroll
  for (int u = 0; u < CB; ++u) {
    v0[u] = (u < count && o0 < 2 * HD) ? recs[(size_t)u * reclen + kRecHead + o0] : 0.0;
    v1[u] = (u < count && o1 < 2 * HD) ? recs[(size_t)u * reclen + kRecHead + o1] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double m = CUDART_INF;
    for (int k = lane; k < count; k += 32)
      if (hs[k * kRecHead + 2] > 0.0) m = fmin(m, hs[k * kRecHead + 0]);
    for (int off = 16; off > 0; off >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, off));
    double s0 = 0.0, cnt = 0.0, sf = 0.0, stt = 0.0, bad = 2147483647.0;
    for (int k = lane; k < count; k += 32) {
      const double* r = hs + k * kRecHead;
      const double sc = r[2] > 0.0 ? exp(-(r[0] - m) / beta) : 0.0;
      scale_smem[k] = sc;
      s0 += sc * r[1];
      cnt += r[2];
      sf += r[3];
      stt = fmax(stt, r[4]);
      bad = fmin(bad, r[5]);
    }
    s0 = warp_sum(s0);
    cnt = warp_sum(cnt);
    sf = warp_sum(sf);
    for (int off = 16; off > 0; off >>= 1) {
      stt = fmax(stt, __shfl_xor_sync(0xffffffffu, stt, off));
      bad = fmin(bad, __shfl_xor_sync(0xffffffffu, bad, off));
    }
    if (lane == 0) {
      out[0] = m;
      out[1] = s0;
      out[2] = cnt;
      out[3] = sf;
      out[4] = stt;
      out[5] = bad;
    }
  }
  __syncthreads();
  double s_0 = 0.0, s_1 = 0.0;
#pragma unroll
  for (int u = 0; u < CB; ++u)
    if (u < count) {
      s_0 += scale_smem[u] * v0[u];
      s_1 += scale_smem[u] * v1[u];
    }
  for (int k0 = CB; k0 < count; k0 += CB) {  // more than 16 records (large N): further batches
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      v0[u] = (k0 + u < count && o0 < 2 * HD) ? recs[(size_t)(k0 + u) * reclen + kRecHead + o0] : 0.0;
      v1[u] = (k0 + u < count && o1 < 2 * HD) ? recs[(size_t)(k0 + u) * reclen + kRecHead + o1] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < CB; ++u)
      if (k0 + u < count) {
        s_0 += scale_smem[k0 + u] * v0[u];
        s_1 += scale_smem[k0 + u] * v1[u];
      }
  }
  for (int o = 2 * blockDim.x; o < 2 * HD; o += blockDim.x) {  // only if 2HD > 2*blockDim
    double s = 0.0;
    for (int k = 0; k < count; ++k) s += scale_smem[k] * recs[(size_t)k * reclen + kRecHead + o];
    out[kRecHead + o] = s;
  }
  if (o0 < 2 * HD) out[kRecHead + o0] = s_0;
  if (o1 < 2 * HD) out[kRecHead + o1] = s_1;
  __syncthreads();
}

// Apply update_mean/update_covariance/shift/next_command from a combined record.
// One block per instance; thread o owns policy entry o = h*D + j (H*D <= 256).
template <typename R>
static __device__ void finalize_policy(const StatsArgs<R>& a, int b, const double* rec, double* emp_smem) {
  const int H = a.H, D = a.D, HD = H * D;
  const int o = threadIdx.x;
  double* means = a.means + (size_t)b * HD;
  double* var = a.var + (size_t)b * HD;
  double* sd = a.sd + (size_t)b * HD;
  __shared__ int s_status;
  __shared__ int s_varbad;
  if (threadIdx.x == 0) {
    int stt = max(a.status[b], (int)rec[4]);
    if ((int)rec[5] < a.bad[b]) a.bad[b] = (int)rec[5];
    if (stt == 0 && rec[2] <= 0.0) stt = MPPI_E_ALL_QUARANTINED;
    if (stt == 0 && !(rec[1] > 0.0)) stt = MPPI_E_WEIGHT_UNDERFLOW;
    s_status = stt;
    s_varbad = 0;
  }
  __syncthreads();
  // read the view this iteration used (shifted on the first iteration)
  double mo = 0.0, vo = 0.0, so = 0.0;
  const int h = o / D, j = o - (o / D) * D;
  if (o < HD) {
    const int hs = a.shift ? h + 1 : h;
    mo = hs < H ? means[hs * D + j] : a.tail_mean;
    vo = hs < H ? var[hs * D + j] : a.tail_var;
    so = hs < H ? sd[hs * D + j] : a.tail_sd;
  }
  double mu_new = mo, var_new = vo;
  if (s_status == 0 && o < HD) {
    const double S0 = rec[1], S1 = rec[kRecHead + o], S2 = rec[kRecHead + HD + o];
    const double avg = mo + S1 / S0;
    mu_new = (1.0 - a.alpha_mu) * mo + a.alpha_mu * avg;
    const double dl = mu_new - mo;
    double emp = S2 / S0 - 2.0 * dl * (S1 / S0) + dl * dl;
    emp_smem[o] = emp;
  }
  __syncthreads();
  if (s_status == 0 && o < HD) {
    double emp = emp_smem[o];
    if (a.isotropic) {
      double s = 0.0;
      for (int jj = 0; jj < D; ++jj) s += emp_smem[h * D + jj];
      emp = s / D;
    }
    double vn = (1.0 - a.alpha_sigma) * vo + a.alpha_sigma * emp;
    vn = vn < a.smin ? a.smin : (vn > a.smax ? a.smax : vn);  // np.clip keeps NaN
    var_new = vn;
    if (!(vn > 0.0) && !isnan(vn)) atomicOr(&s_varbad, 1);
  }
  __syncthreads();
  if (o < HD) {
    if (a.prev_means) {
      a.prev_means[(size_t)b * HD + o] = mo;
      a.prev_sd[(size_t)b * HD + o] = so;
    }
    if (s_status == 0) {
      means[o] = mu_new;
      if (!s_varbad) {
        var[o] = var_new;
        sd[o] = sqrt(var_new);
      } else {
        var[o] = vo;
        sd[o] = so;
      }
    } else if (a.shift && s_status != MPPI_E_SKIPPED) {  // failure: the shift of controller.py:200 still stands
      means[o] = mo;
      var[o] = vo;
      sd[o] = so;
    }
  }
  if (threadIdx.x == 0) {
    int stt = s_status;
    if (stt == 0 && s_varbad) stt = MPPI_E_NONPOSITIVE_VARIANCE;
    a.status[b] = stt;
    if (a.info) {
      mppi_step_info inf;
      inf.status = stt;
      inf.bad_particle = a.bad[b] >= 0x7f000000 ? -1 : a.bad[b];
      inf.finite_count = (int)rec[2];
      inf._pad = 0;
      inf.best_cost = rec[2] > 0.0 ? rec[0] : CUDART_NAN;
      inf.mean_cost = rec[2] > 0.0 ? rec[3] / rec[2] : CUDART_NAN;
      inf.device_ms = 0.0;
      inf.sample_ms = inf.rollout_ms = inf.mlp_ms = inf.update_ms = 0.0;
      a.info[b] = inf;
    }
  }
  if (s_status == 0 && o < D && a.cmd) a.cmd[(size_t)b * D + o] = mu_new;  // next_command "mean"
  if (a.reset_status) {
    __syncthreads();
    if (threadIdx.x == 0) {
      a.status[b] = 0;
      a.bad[b] = 0x7f7f7f7f;
    }
  }
}

// The rank record `rec` (reclen doubles, shared memory) -> every rank's
// receive slot [rank], release flag, wait for all ranks, fixed-order combine,
// update. One block, all threads. scratch: >= reclen + HD + 8 * (1 + kRecHead)
// + 32 doubles of shared memory not aliasing `rec`.
template <typename R>
static __device__ void exchange_and_finalize(const StatsArgs<R>& a, const double* rec, int HD, double* scratch) {
  const int reclen = kRecHead + 2 * HD;
  const int par = (int)(a.seq & 1ull);
  for (int k = 0; k < a.world; ++k) {  // NVLink P2P stores (local for k == rank)
    double* dst = a.peer_recv[k] + ((size_t)par * a.world + a.rank) * reclen;
    for (int i = threadIdx.x; i < reclen; i += blockDim.x) dst[i] = rec[i];
  }
  __threadfence_system();
  __shared__ int s_xfail;
  if (threadIdx.x == 0) s_xfail = a.status[0] == MPPI_E_EXCHANGE ? 4 : 0;  // an earlier iteration failed
  __syncthreads();
  if ((int)threadIdx.x < a.world) {
    unsigned long long* f = a.peer_flags[threadIdx.x] + a.rank;
    if (s_xfail) {  // do not make the others wait for an iteration this rank abandons
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(a.seq | kPeerAbort) : "memory");
    } else {
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(a.seq) : "memory");
      const unsigned long long* mine = a.my_flags + threadIdx.x;
      const unsigned long long t0 = global_ns();
      unsigned long long v = 0;
      for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
        const unsigned long long s = v & ~kPeerAbort;
        if ((v & kPeerAbort) && s >= a.seq) {  // that rank abandoned this step
          atomicOr(&s_xfail, 1);
          break;
        }
        if (!(v & kPeerAbort) && s >= a.seq) break;
        if (global_ns() - t0 > a.peer_timeout_ns) {  // a rank that never arrives
          atomicOr(&s_xfail, 2);
          break;
        }
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
  if (s_xfail) {
    // tell every rank (and keep this rank's status) so the others stop
    // waiting; the step keeps the shifted policy (controller.py:224-241)
    if ((int)threadIdx.x < a.world)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.peer_flags[threadIdx.x] + a.rank),
                   "l"(a.seq | kPeerAbort) : "memory");
    if (threadIdx.x == 0) a.status[0] = MPPI_E_EXCHANGE;
    __syncthreads();
    finalize_policy(a, 0, rec, scratch);
    return;
  }
  double* comb = scratch;
  double* emp = comb + reclen;
  double* red = emp + HD;
  double* scale = red + 32;
  combine_records(a.my_recv + (size_t)par * a.world * reclen, a.world, reclen, HD, a.beta, comb, scale, red);
  finalize_policy(a, 0, comb, emp);
}

template <typename R, int D>
__global__ void __launch_bounds__(kStatsThreads) stats_kernel(const __grid_constant__ StatsArgs<R> a) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.y, blk = blockIdx.x;
  const int H = a.H, HD = H * D, N = a.N;
  const int n0 = blk * a.ppb;
  const int n1 = min(N, n0 + a.ppb);
  const int cnt = max(0, n1 - n0);
  double* tot = sm;             // [ppb]
  double* wt = sm + a.ppb;      // [ppb]
  double* red = wt + a.ppb;     // [32]
  double* scale = red + 32;     // [max(nblk, 8)] scales + [max(nblk, 8) * kRecHead] heads
  const int reclen = kRecHead + 2 * HD;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kStatsThreads / 32;  // launched with kStatsThreads
  pdl_wait();  // rollout / MLP outputs and the status word are ready past this point
  const bool failed = (a.status[b] != 0);
#ifdef MPPI_DEBUG_TIMERS
#undef MPPI_STAMP
#define MPPI_STAMP(k)                                                                        \
  if (a.dbg && threadIdx.x == 0 && b == 0) {                                                  \
    unsigned long long t_;                                                                   \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
    a.dbg[blk * 16 + (k)] = t_;                                                              \
  }
#else
#define MPPI_STAMP(k)
#endif
  MPPI_STAMP(0);

  // ---- phase A: discounted totals, quarantine (rollout.py:111-171) ---------
  // Each warp takes PA particles at a time and issues all their loads before
  // the first reduction, so the HBM/L2 latency is paid once per batch.
  {  // runs even when the step already failed: cheap, and the status load overlaps it
    constexpr int PA = 4;
    // the lane's discount, read once: a lane-indexed parameter read inside the
    // loop is a serialised constant-cache load per row
    const double disc_l = lane < H ? (lane < H - 1 ? a.disc[lane] : a.dlast) : 0.0;
    for (int i0 = wid * PA; i0 < cnt; i0 += nw * PA) {
      double cv[PA], dv[PA];
#pragma unroll
      for (int u = 0; u < PA; ++u) {
        cv[u] = 0.0;
        dv[u] = 0.0;
        if (i0 + u < cnt && lane < H) {
          const size_t m = ((size_t)b * N + n0 + i0 + u) * H + lane;
          cv[u] = (double)a.step[m];
          if (a.learned) dv[u] = (double)a.mlp_d[m];
        }
      }
#pragma unroll
      for (int u = 0; u < PA; ++u) {
        const int i = i0 + u;
        if (i >= cnt) break;  // warp-uniform
        const int n = n0 + i;
        double c = 0.0, dself = 0.0;
        bool fin = true;
        if (lane < H) {
          c = cv[u];
          if (a.learned) {
            dself = dv[u] > 0.0 ? dv[u] : 0.0;
            c = c + a.a_coll * dself;
          }
          fin = isfinite(c);
        }
        const bool allfin = __all_sync(0xffffffffu, fin);
        double contrib = 0.0;
        if (lane < H) contrib = disc_l * c;
        double total = warp_sum(contrib);
        if (!allfin) total = CUDART_INF;
        if (lane == 0) {
          tot[i] = total;
          if (a.totals) a.totals[(size_t)b * N + n] = total;
        }
        if (b == 0 && lane < H) {
          if (a.dump_step) a.dump_step[(size_t)n * H + lane] = (allfin || a.raw_step) ? c : 0.0;
          if (a.dump_terms && a.learned) a.dump_terms[(size_t)T_SELF * N * H + (size_t)n * H + lane] = dself;
        }
      }
    }
  }
  if (a.totals_only) return;
  __syncthreads();
  MPPI_STAMP(1);

  // ---- phase B/C: block min, weights relative to it (policy.py:103-121) ----
  double mloc = CUDART_INF;
  if (!failed)
    for (int i = threadIdx.x; i < cnt; i += blockDim.x)
      if (isfinite(tot[i])) mloc = fmin(mloc, tot[i]);
  const double mb = block_min_d(mloc, red);
  if (!failed)
    for (int i = threadIdx.x; i < cnt; i += blockDim.x)
      wt[i] = isfinite(tot[i]) ? exp(-(tot[i] - mb) / a.beta) : 0.0;
  __syncthreads();

  // ---- phase D: weighted sufficient statistics around the old mean ---------
  double mo_pre = 0.0, so_pre = 0.0;  // this thread's policy entry, loaded before the barriers
  if (threadIdx.x < HD) {
    const int h = threadIdx.x / D, j = threadIdx.x - h * D;
    const int hs = a.shift ? h + 1 : h;
    mo_pre = hs < H ? a.means[(size_t)b * HD + hs * D + j] : a.tail_mean;
    so_pre = hs < H ? a.sd[(size_t)b * HD + hs * D + j] : a.tail_sd;
  }
  // Particles whose weight underflowed to exactly 0 contribute nothing; warp 0
  // compacts the others (ascending, so the summation order is fixed) and every
  // output then runs a branch-free loop with PD independent eps loads in flight.
  const int rstride = stats_rec_stride(a.nblk);
  double* rec = a.records + ((size_t)b * rstride + blk) * reclen;
  int* nz = reinterpret_cast<int*>(sm + 2 * a.ppb + 32 + max(a.nblk, 8) * (1 + kRecHead) + reclen + HD);
  __shared__ int s_nnz;
  if (wid == 0) {
    int base = 0;
    if (!failed)
      for (int c0 = 0; c0 < cnt; c0 += 32) {
        const int i = c0 + lane;
        const bool keep = i < cnt && wt[i] > 0.0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) nz[base + __popc(bal & ((1u << lane) - 1u))] = i;
        base += __popc(bal);
      }
    if (lane == 0) s_nnz = base;
  } else if (wid == 1) {
    double s0 = 0.0, c = 0.0, sf = 0.0;
    if (!failed)
      for (int i = lane; i < cnt; i += 32) {
        s0 += wt[i];
        if (isfinite(tot[i])) {
          c += 1.0;
          sf += tot[i];
        }
      }
    s0 = warp_sum(s0);
    c = warp_sum(c);
    sf = warp_sum(sf);
    if (lane == 0) {
      rec[0] = c > 0.0 ? mb : CUDART_INF;
      rec[1] = s0;
      rec[2] = c;
      rec[3] = sf;
      rec[4] = (double)a.status[b];
      rec[5] = (double)a.bad[b];
    }
  }
  __syncthreads();
  const int nnz = s_nnz;
  MPPI_STAMP(2);
  if (threadIdx.x < HD) {  // H*d <= 256 = blockDim: one policy entry per thread
    const int o = threadIdx.x;
    double s1 = 0.0, s2 = 0.0;
    if (!failed) {
      const double* ep = a.eps + (size_t)n0 * HD + o;
      constexpr int PD = 16;
      // null and mean rows (sampling.py:283-285) lead the ascending list:
      // summed first with their selects, the rest without (same order)
      int k1 = 0;
      while (k1 < nnz && n0 + nz[k1] + a.particle_offset <= a.null_count) {
        const int ng = n0 + nz[k1] + a.particle_offset;
        const double ev = __ldg(ep + (size_t)nz[k1] * HD);
        const double dv = ng < a.null_count ? 0.0 - mo_pre : (ng == a.null_count ? 0.0 : (mo_pre + so_pre * ev) - mo_pre);
        const double w = wt[nz[k1]];
        s1 += w * dv;
        s2 += w * dv * dv;
        ++k1;
      }
      for (int k0 = k1; k0 < nnz; k0 += PD) {
        double e[PD];
        int ii[PD];
#pragma unroll
        for (int u = 0; u < PD; ++u) {
          ii[u] = k0 + u < nnz ? nz[k0 + u] : -1;
          e[u] = ii[u] >= 0 ? __ldg(ep + (size_t)ii[u] * HD) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PD; ++u) {
          if (ii[u] < 0) break;
          const double dv = (mo_pre + so_pre * e[u]) - mo_pre;
          const double w = wt[ii[u]];
          s1 += w * dv;
          s2 += w * dv * dv;
        }
      }
    }
    rec[kRecHead + o] = s1;
    rec[kRecHead + HD + o] = s2;
  }

  // ---- last block of this instance combines + finalizes --------------------
  __shared__ bool s_last;
  MPPI_STAMP(3);
  unsigned* ctr = a.counters + (size_t)b * kStatsCounterStride;
  const int ngroups = stats_groups(a.nblk);
  const double* level = a.records + (size_t)b * rstride * reclen;  // records the final combine reads
  int nlevel = a.nblk;
  if (ngroups > 0) {  // first level: the last block of this group combines the group
    const int grp = blk / kStatsGroup, g0 = grp * kStatsGroup, gs = min(kStatsGroup, a.nblk - g0);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&ctr[1 + grp], 1u) == (unsigned)(gs - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) ctr[1 + grp] = 0u;
    double* grec = a.records + ((size_t)b * rstride + a.nblk + grp) * reclen;
    combine_records(a.records + ((size_t)b * rstride + g0) * reclen, gs, reclen, HD, a.beta, grec, scale, red);
    level = a.records + ((size_t)b * rstride + a.nblk) * reclen;
    nlevel = ngroups;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ctr[0], 1u) == (unsigned)((ngroups > 0 ? ngroups : a.nblk) - 1);
  __syncthreads();
  if (!s_last) return;
  MPPI_STAMP(4);
  __threadfence();
  if (threadIdx.x == 0) ctr[0] = 0u;
  MPPI_STAMP(7);
  const bool peer = a.peer_recv != nullptr;
  double* comb = (a.finalize_inline || peer) ? (sm + 2 * a.ppb + 32 + max(a.nblk, 8) * (1 + kRecHead))
                                             : a.out_record + (size_t)b * reclen;
  combine_records(level, nlevel, reclen, HD, a.beta, comb, scale, red);
  MPPI_STAMP(5);
  if (peer) {  // the rank record goes to every rank over peer memory; the update happens here
    __syncthreads();
    exchange_and_finalize(a, comb, HD, comb + reclen + HD);
    return;
  }
  if (!a.finalize_inline) return;
  double* emp = comb + reclen;
  finalize_policy(a, b, comb, emp);
  __syncthreads();
  MPPI_STAMP(6);
  if (b == 0 && a.dump_weights && a.status[0] == 0) {
    __syncthreads();
    const double m = comb[0];
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const double t = a.totals[n];
      a.dump_weights[n] = isfinite(t) ? exp(-(t - m) / a.beta) : 0.0;
    }
  }
}

// Cluster statistics (latency path, N <= 16 * kClusterMaxPPB): the nblk <= 16
// CTAs of one instance form one thread-block cluster. Every exchange is a
// PUSH into the receiver's shared memory (st.async) completing on the
// receiver's mbarrier, so no CTA ever waits on a cluster-wide fence:
//   1. each CTA's best finite total -> slot [blk] of every peer's `mins`;
//      after the barrier all CTAs hold the instance minimum, so weights are
//      exactly exp(-(c - min)/beta) (policy.py:113-114) with no rescaling;
//   2. each CTA's S0/count/sum and S1|S2 rows -> slot [blk] of rank 0;
//      after the barrier rank 0 reduces them in rank order from its own
//      shared memory and applies the update in registers (policy.py:124-177).
// The perturbation rows of the CTA's particles do not depend on this step's
// costs: they are loaded into registers before the totals, so the weighted
// sums are pure FMA chains once the weights exist. No global records,
// fences, atomics or last-block hand-off; the only cluster barrier publishes
// the mbarrier initialisation and is waited on after the totals.
constexpr int kClusterMax = 16;
#ifndef MPPI_CLUSTER_PPB
#define MPPI_CLUSTER_PPB 128  // A/B: 2048 particles 77 -> 71 us per step; 256 per CTA (N = 4096) is slower
#endif
constexpr int kClusterMaxPPB = MPPI_CLUSTER_PPB;
constexpr int kClusterEpsRegs = 32;  // perturbation rows held in registers per thread

inline size_t stats_cluster_smem_bytes(int ppb, int HD) {
  const size_t slots = ppb > kClusterEpsRegs ? (size_t)ppb : (size_t)kClusterEpsRegs;
  return sizeof(double) * (2 * slots + 32 + kClusterMax + kClusterMax * 4 + (size_t)kClusterMax * 2 * HD + HD) +
         2 * sizeof(unsigned long long);
}

// (kStatsThreads, 1): the full register budget — without the minimum-blocks
// hint ptxas caps this kernel at 128 registers and the step is 1.3 us slower
// LEAN: the control-step specialisation (update applied here, no bundle
// dumps, no rank record / peer exchange) — only the code a step executes.
template <typename R, int D, bool LEAN = false>
__global__ void __launch_bounds__(kStatsThreads, 1) stats_cluster_kernel(const __grid_constant__ StatsArgs<R> a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.y;
  const int blk = (int)cluster.block_rank();
  const int nblk = (int)cluster.num_blocks();
  // the CTA that reduces the weighted sums and applies the update (rank 0;
  // the last rank, which has the fewest particles, measured 0.2 us slower)
  const int root = 0;
  const int H = a.H, HD = H * D, N = a.N;
  // particles of this CTA: the instance's CTAs in grid order (several clusters
  // per instance in the multi-cluster layout, one record each)
  const int n0 = (int)blockIdx.x * a.ppb;
  const int cnt = max(0, min(N, n0 + a.ppb) - n0);
  const int slots = max(a.ppb, kClusterEpsRegs);
  double* tot = sm;                      // [slots]
  double* wt = tot + slots;              // [slots], 16-byte aligned
  double* red = wt + slots;              // [32]
  double* mins = red + 32;               // [kClusterMax] per-CTA best finite totals (pushed by peers)
  double* heads = mins + kClusterMax;    // [kClusterMax][4] S0, count, sum finite (rank 0)
  double* parts = heads + kClusterMax * 4;  // [kClusterMax][HD][2] S1, S2 pairs (rank 0)
  double* emp = parts + (size_t)kClusterMax * 2 * HD;  // [HD]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(emp + HD);  // [0] mins, [1] rank-0 sums
  const uint32_t bar_min = smem_addr(&bars[0]), bar_sum = smem_addr(&bars[1]);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kStatsThreads / 32;  // launched with kStatsThreads
  const int o = threadIdx.x;
  const bool owner = o < HD;  // H*d <= 256 = blockDim: one policy entry per thread
  MPPI_STAMP(6);  // (debug) CTA entry
  if (threadIdx.x == 0) {  // each receive barrier completes on bytes alone
    cbar_init(bar_min, 1);
    cbar_init(bar_sum, 1);
    cbar_arrive_expect(bar_min, 8u * nblk);
    if (blk == root) cbar_arrive_expect(bar_sum, (16u * HD + 32u) * nblk);
  }
  cluster_init_fence_arrive();  // waited on before the first push
  // ---- requests that do not depend on this step's costs ----------------------
  double mo = 0.0, so = 0.0, vo = 0.0;
  double e[kClusterEpsRegs];
  const double* ep = a.eps + (size_t)n0 * HD + o;
  if (owner) {
    const int h = o / D, j = o - h * D;
    const int hs = a.shift ? h + 1 : h;
    mo = hs < H ? a.means[(size_t)b * HD + hs * D + j] : a.tail_mean;
    so = hs < H ? a.sd[(size_t)b * HD + hs * D + j] : a.tail_sd;
    vo = hs < H ? a.var[(size_t)b * HD + hs * D + j] : a.tail_var;
#pragma unroll
    for (int i = 0; i < kClusterEpsRegs; ++i) e[i] = i < cnt ? __ldg(ep + (size_t)i * HD) : 0.0;
  }
  const double disc_l = lane < H - 1 ? a.disc[lane] : a.dlast;
  pdl_wait();
  const int status0 = a.status[b];
  const int bad0 = a.bad[b];  // (final once the rollout is complete) read here, off the update's path
  const bool failed = status0 != 0;
  MPPI_STAMP(0);

  // ---- totals (rollout.py:111-171), 4 particles per warp, loads batched -----
  {
    constexpr int PA = 4;
    for (int i0 = wid * PA; i0 < cnt; i0 += nw * PA) {
      double cv[PA], dv[PA];
#pragma unroll
      for (int u = 0; u < PA; ++u) {
        cv[u] = 0.0;
        dv[u] = 0.0;
        if (i0 + u < cnt && lane < H) {
          const size_t m = ((size_t)b * N + n0 + i0 + u) * H + lane;
          cv[u] = (double)a.step[m];
          if (a.learned) dv[u] = (double)a.mlp_d[m];
        }
      }
      // the PA horizon sums reduce side by side (independent shuffle chains)
      double ct[PA], ds[PA];
      bool allfin[PA];
#pragma unroll
      for (int u = 0; u < PA; ++u) {
        double c = 0.0, dself = 0.0;
        bool fin = true;
        if (lane < H) {
          c = cv[u];
          if (a.learned) {
            dself = dv[u] > 0.0 ? dv[u] : 0.0;
            c = c + a.a_coll * dself;
          }
          fin = isfinite(c);
        }
        allfin[u] = __all_sync(0xffffffffu, fin);
        ct[u] = c;
        ds[u] = dself;
        cv[u] = lane < H ? disc_l * c : 0.0;  // the discounted contribution
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int u = 0; u < PA; ++u) cv[u] += __shfl_xor_sync(0xffffffffu, cv[u], off);
#pragma unroll
      for (int u = 0; u < PA; ++u) {
        const int i = i0 + u;
        if (i >= cnt) break;
        const int n = n0 + i;
        const double total = allfin[u] ? cv[u] : CUDART_INF;
        if (lane == 0) {
          tot[i] = total;
          if (a.totals) a.totals[(size_t)b * N + n] = total;
        }
        if (b == 0 && lane < H) {
          if (!LEAN && a.dump_step) a.dump_step[(size_t)n * H + lane] = allfin[u] ? ct[u] : 0.0;
          if (!LEAN && a.dump_terms && a.learned)
            a.dump_terms[(size_t)T_SELF * N * H + (size_t)n * H + lane] = ds[u];
        }
      }
    }
  }
  __syncthreads();
  MPPI_STAMP(1);
  // ---- instance-wide best finite total: pushed to every peer -----------------
  // (Weighing against each CTA's own minimum and rescaling the sums at the
  // root instead — no round trip before the weights — measured 0.5 us slower:
  // the root's extra exp/shuffles cost more than the exchange it saves.)
  cluster_wait();  // every peer's receive barriers are initialised
  if (wid == 0) {
    double v = CUDART_INF;
    for (int i = lane; i < cnt; i += 32)
      if (isfinite(tot[i])) v = fmin(v, tot[i]);
    for (int off = 16; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane < nblk) push_f64(mapa_rank(smem_addr(&mins[blk]), lane), v, mapa_rank(bar_min, lane));
  }
  // deviations u - mu_old of the register rows (they do not depend on the
  // costs), computed while the minimum exchange is in flight, branch-free;
  // the null and mean rows (sampling.py:283-285) exist only in the CTA
  // holding global particles 0..null_count and are patched there (a
  // CTA-uniform branch), so the weighted sums below are one straight FMA
  // schedule (per-row selects inside the sums compiled to 32 branches that
  // serialised the chains: 1.05 -> 0.4 us)
  if (owner) {
    const int g0 = n0 + a.particle_offset;  // global index of this CTA's first particle
#pragma unroll
    for (int i = 0; i < kClusterEpsRegs; ++i) e[i] = (mo + so * e[i]) - mo;
    if (g0 <= a.null_count) {  // dv = k1 * dv + k0: (1, 0) sampled, (0, -mu) null, (0, 0) mean row
#pragma unroll
      for (int i = 0; i < kClusterEpsRegs; ++i) {
        const int ng = g0 + i;
        e[i] = fma(ng > a.null_count ? 1.0 : 0.0, e[i], ng < a.null_count ? 0.0 - mo : 0.0);
      }
    }
  }
  MPPI_STAMP(13);  // (debug) deviations formed: the perturbation rows have arrived
  cbar_wait(bar_min, 0);
  double m = CUDART_INF;
  for (int k = 0; k < nblk; ++k) m = mins[k] < m ? mins[k] : m;  // finite or +inf, never NaN
  MPPI_STAMP(2);
  // ---- weights (policy.py:103-121) ------------------------------------------
  // slots [cnt, 32) hold zero weights so the register loop below is branch-free
  for (int i = threadIdx.x; i < max(cnt, kClusterEpsRegs); i += blockDim.x)
    wt[i] = (i < cnt && !failed && isfinite(tot[i])) ? exp(-(tot[i] - m) / a.beta) : 0.0;
  if (!LEAN && b == 0 && a.dump_weights && !failed)
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) a.dump_weights[n0 + i] = wt[i];
  __syncthreads();
  MPPI_STAMP(3);
  // ---- weighted sufficient statistics around the old mean, pushed to rank 0 --
  // Zero weights add exact zeros. Four interleaved partial sums per entry
  // keep the FP64 dependency chains short (the reference's own reductions are
  // numpy pairwise sums, so no summation order is privileged).
  if (owner) {
    double s1[4] = {0.0, 0.0, 0.0, 0.0}, s2[4] = {0.0, 0.0, 0.0, 0.0};
    if (!failed) {
      const int g0 = n0 + a.particle_offset;  // global index of this CTA's first particle
      const double2* w2 = reinterpret_cast<const double2*>(wt);
#pragma unroll
      for (int i = 0; i < kClusterEpsRegs; i += 2) {
        const double2 w = w2[i / 2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const double dv = e[i + u];
          const double wu = u ? w.y : w.x;
          s1[(i + u) & 3] += wu * dv;
          s2[(i + u) & 3] += wu * dv * dv;
        }
      }
      for (int i = kClusterEpsRegs; i < cnt; ++i) {
        const int ng = g0 + i;
        const double ev = __ldg(ep + (size_t)i * HD);
        const double dv = ng < a.null_count ? 0.0 - mo : (ng == a.null_count ? 0.0 : (mo + so * ev) - mo);
        s1[0] += wt[i] * dv;  // (constant index: the partial sums stay in registers)
        s2[0] += wt[i] * dv * dv;
      }
    }
    MPPI_STAMP(8);
    push_f64x2(mapa_rank(smem_addr(parts + ((size_t)blk * HD + o) * 2), root), (s1[0] + s1[1]) + (s1[2] + s1[3]),
               (s2[0] + s2[1]) + (s2[2] + s2[3]), mapa_rank(bar_sum, root));
    MPPI_STAMP(9);
  }
  if (wid == nw - 1) {
    double s0 = 0.0, c = 0.0, sf = 0.0;
    if (!failed)
      for (int i = lane; i < cnt; i += 32) {
        s0 += wt[i];
        if (isfinite(tot[i])) {
          c += 1.0;
          sf += tot[i];
        }
      }
    s0 = warp_sum(s0);
    c = warp_sum(c);
    sf = warp_sum(sf);
    if (lane == 0) push_f64x2(mapa_rank(smem_addr(heads + blk * 4), root), s0, c, mapa_rank(bar_sum, root));
    if (lane == 1) push_f64x2(mapa_rank(smem_addr(heads + blk * 4 + 2), root), sf, 0.0, mapa_rank(bar_sum, root));
  }
  MPPI_STAMP(4);
  if (blk != root) return;  // peers are done: every push into them has landed
  cbar_wait(bar_sum, 0);
  MPPI_STAMP(5);
  // ---- rank 0: reduce in rank order, update in registers ---------------------
  double S0, cntf, sumf;
  {
    double x0 = 0.0, x1 = 0.0, x2 = 0.0;  // one lane per peer CTA, fixed-order warp tree
    if (lane < nblk) {
      x0 = heads[lane * 4 + 0];
      x1 = heads[lane * 4 + 1];
      x2 = heads[lane * 4 + 2];
    }
    S0 = warp_sum(x0);
    cntf = warp_sum(x1);
    sumf = warp_sum(x2);
  }
  double S1 = 0.0, S2 = 0.0;
  if (owner) {  // every peer row requested first, then summed in rank order
    double2 pr[kClusterMax];
#pragma unroll
    for (int k = 0; k < kClusterMax; ++k)
      pr[k] = k < nblk ? *reinterpret_cast<const double2*>(parts + ((size_t)k * HD + o) * 2) : make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < kClusterMax; ++k) {
      S1 += pr[k].x;
      S2 += pr[k].y;
    }
  }
  MPPI_STAMP(10);
  if (!LEAN && !a.finalize_inline) {  // rank record for the particle-sharded exchange
    const bool peer = a.peer_recv != nullptr;
    const int nclu = (int)gridDim.x / nblk;  // clusters per instance
    double* out = peer ? parts
                       : a.out_record + ((size_t)b * nclu + blockIdx.x / nblk) * (kRecHead + 2 * HD);
    if (peer) __syncthreads();  // every thread has read its partial sums out of `parts`
    if (owner) {
      out[kRecHead + o] = S1;
      out[kRecHead + HD + o] = S2;
    }
    if (o == 0) {
      out[0] = cntf > 0.0 ? m : CUDART_INF;
      out[1] = S0;
      out[2] = cntf;
      out[3] = sumf;
      out[4] = (double)status0;
      out[5] = (double)bad0;
    }
    if (peer) {
      __syncthreads();
      exchange_and_finalize(a, parts, HD, parts + kRecHead + 2 * HD);
    }
    return;
  }
  int stt = status0;
  if (stt == 0 && cntf <= 0.0) stt = MPPI_E_ALL_QUARANTINED;
  if (stt == 0 && !(S0 > 0.0)) stt = MPPI_E_WEIGHT_UNDERFLOW;
  double mu_new = mo, var_new = vo;
  int varbad = 0;
  if (stt == 0 && owner) {
    const double avg = mo + S1 / S0;
    mu_new = (1.0 - a.alpha_mu) * mo + a.alpha_mu * avg;
    const double dl = mu_new - mo;
    double em = S2 / S0 - 2.0 * dl * (S1 / S0) + dl * dl;
    if (a.isotropic) emp[o] = em;
    var_new = em;
  }
  if (a.isotropic) __syncthreads();
  if (stt == 0 && owner) {
    double em = var_new;
    if (a.isotropic) {
      const int h = o / D;
      double sacc = 0.0;
      for (int jj = 0; jj < D; ++jj) sacc += emp[h * D + jj];
      em = sacc / D;
    }
    double vn = (1.0 - a.alpha_sigma) * vo + a.alpha_sigma * em;
    vn = vn < a.smin ? a.smin : (vn > a.smax ? a.smax : vn);  // np.clip keeps NaN
    var_new = vn;
    varbad = (!(vn > 0.0) && !isnan(vn)) ? 1 : 0;
  }
  varbad = __syncthreads_or(varbad);
  MPPI_STAMP(11);
  double* means = a.means + (size_t)b * HD;
  double* var = a.var + (size_t)b * HD;
  double* sd = a.sd + (size_t)b * HD;
  if (owner) {
    if (a.prev_means) {
      a.prev_means[(size_t)b * HD + o] = mo;
      a.prev_sd[(size_t)b * HD + o] = so;
    }
    if (stt == 0) {
      means[o] = mu_new;
      if (!varbad) {
        var[o] = var_new;
        sd[o] = sqrt(var_new);
      } else {
        var[o] = vo;
        sd[o] = so;
      }
    } else if (a.shift && stt != MPPI_E_SKIPPED) {  // failure: the shift of controller.py:200 still stands
      means[o] = mo;
      var[o] = vo;
      sd[o] = so;
    }
  }
  MPPI_STAMP(12);
  if (stt == 0 && o < D && a.cmd) a.cmd[(size_t)b * D + o] = mu_new;  // next_command "mean"
  const int stt2 = (stt == 0 && varbad) ? MPPI_E_NONPOSITIVE_VARIANCE : stt;
  // mppi_step_info (mapped host memory) as nine 8-byte words, one per thread
  // of warp 2, so no single thread queues a chain of system-memory stores
  constexpr int kInfoWords = (int)(sizeof(mppi_step_info) / 8);
  static_assert(sizeof(mppi_step_info) % 8 == 0, "mppi_step_info words");
  if (a.info && threadIdx.x >= 64 && threadIdx.x < 64 + kInfoWords) {
    const int w = threadIdx.x - 64;
    unsigned long long word = 0ull;
    if (w == 0)
      word = (unsigned)stt2 | ((unsigned long long)(unsigned)(bad0 >= 0x7f000000 ? -1 : bad0) << 32);
    else if (w == 1)
      word = (unsigned)(int)cntf;
    else if (w == 2)
      word = (unsigned long long)__double_as_longlong(cntf > 0.0 ? m : CUDART_NAN);
    else if (w == 3)
      word = (unsigned long long)__double_as_longlong(cntf > 0.0 ? sumf / cntf : CUDART_NAN);
    reinterpret_cast<unsigned long long*>(a.info + b)[w] = word;  // words 4..8: the stage times, 0
  }
  if (threadIdx.x == 0) {
    if (a.reset_status) {
      a.status[b] = 0;
      a.bad[b] = 0x7f7f7f7f;
    } else {
      a.status[b] = stt2;
    }
  }
  MPPI_STAMP(7);
}

// Batched statistics, G instances per block (config 4: B >= 148, one block's
// worth of particles per instance, no bundle dumps, update applied here).
// stats_kernel with nblk == 1 re-reads the shared perturbation block
// (N*H*d doubles, 840 KB at 500 x 30 x 7) once per instance; here one load of
// eps[n][o] feeds the weighted sums of all G instances. Same arithmetic as
// stats_kernel + combine_records(count = 1) + finalize_policy, term by term:
//   totals      rollout.py:111-171 (rows of the G instances are contiguous)
//   weights     policy.py:103-121 (warp g reduces instance g in lane order)
//   S0/S1/S2    policy.py:124-155 around the pre-update mean; a particle in
//               the union of nonzero weights adds w*dv with w = 0 for the
//               instances where it underflowed, which leaves the sum unchanged
//   record      combine_records with one record: scale exp(-0/beta) = 1
template <typename R, int D, int G, int PD = 8, int MINB = 1>
__global__ void __launch_bounds__(kStatsThreads, MINB) stats_multi_kernel(const __grid_constant__ StatsArgs<R> a) {
  extern __shared__ __align__(16) double sm[];
  const int H = a.H, HD = H * D, N = a.N, cnt = N;
  const int b0 = blockIdx.x * G;
  const int gn = min(G, a.B - b0);
  const int reclen = kRecHead + 2 * HD;
  double* tot = sm;                  // [G][N]
  double* wt = tot + G * N;          // [G][N]
  double* recs = wt + G * N;         // [G][reclen]
  double* emp = recs + G * reclen;   // [HD]
  int* nz = reinterpret_cast<int*>(emp + HD);  // [N]
  __shared__ int s_failed[G];
  __shared__ int s_nnz;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kStatsThreads / 32;
  pdl_wait();
  if (threadIdx.x < G) s_failed[threadIdx.x] = threadIdx.x < gn ? (a.status[b0 + threadIdx.x] != 0) : 1;

  // ---- totals of the G*N contiguous rows -----------------------------------
  {
    constexpr int PA = 4;
    const int rows = gn * N;
    const double disc_l = lane < H ? (lane < H - 1 ? a.disc[lane] : a.dlast) : 0.0;
    for (int r0 = wid * PA; r0 < rows; r0 += nw * PA) {
      double cv[PA], dv[PA];
#pragma unroll
      for (int u = 0; u < PA; ++u) {
        cv[u] = 0.0;
        dv[u] = 0.0;
        if (r0 + u < rows && lane < H) {
          const size_t m = ((size_t)b0 * N + r0 + u) * H + lane;
          cv[u] = (double)a.step[m];
          if (a.learned) dv[u] = (double)a.mlp_d[m];
        }
      }
#pragma unroll
      for (int u = 0; u < PA; ++u) {
        const int r = r0 + u;
        if (r >= rows) break;  // warp-uniform
        double c = 0.0;
        bool fin = true;
        if (lane < H) {
          c = cv[u];
          if (a.learned) c = c + a.a_coll * (dv[u] > 0.0 ? dv[u] : 0.0);
          fin = isfinite(c);
        }
        const bool allfin = __all_sync(0xffffffffu, fin);
        double contrib = 0.0;
        if (lane < H) contrib = disc_l * c;
        double total = warp_sum(contrib);
        if (!allfin) total = CUDART_INF;
        if (lane == 0) {
          tot[r] = total;
          if (a.totals) a.totals[(size_t)b0 * N + r] = total;
        }
      }
    }
  }
  __syncthreads();

  // ---- per instance: minimum, weights, record head (warp g) ----------------
  if (wid < gn) {
    const int g = wid;
    const double* tg = tot + g * N;
    double* wg = wt + g * N;
    const bool failed = s_failed[g] != 0;
    double mloc = CUDART_INF;
    if (!failed)
      for (int i = lane; i < cnt; i += 32)
        if (isfinite(tg[i])) mloc = fmin(mloc, tg[i]);
    for (int off = 16; off > 0; off >>= 1) mloc = fmin(mloc, __shfl_xor_sync(0xffffffffu, mloc, off));
    const double mb = mloc;
    double s0 = 0.0, c = 0.0, sf = 0.0;
    for (int i = lane; i < cnt; i += 32) {
      const double w = (!failed && isfinite(tg[i])) ? exp(-(tg[i] - mb) / a.beta) : 0.0;
      wg[i] = w;
      if (!failed) {
        s0 += w;
        if (isfinite(tg[i])) {
          c += 1.0;
          sf += tg[i];
        }
      }
    }
    s0 = warp_sum(s0);
    c = warp_sum(c);
    sf = warp_sum(sf);
    if (lane == 0) {  // == combine_records over this single record
      const double sc = c > 0.0 ? 1.0 : 0.0;
      double* rec = recs + g * reclen;
      rec[0] = c > 0.0 ? mb : CUDART_INF;
      rec[1] = sc * s0 + 0.0;
      rec[2] = c + 0.0;
      rec[3] = sf + 0.0;
      rec[4] = fmax(0.0, (double)a.status[b0 + g]);
      rec[5] = fmin(2147483647.0, (double)a.bad[b0 + g]);
    }
  }
  __syncthreads();
  // union of the nonzero weights, ascending (the summation order of stats_kernel)
  if (wid == 0) {
    int base = 0;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int i = c0 + lane;
      bool keep = false;
      if (i < cnt)
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (g < gn) keep |= wt[g * N + i] > 0.0;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) nz[base + __popc(bal & ((1u << lane) - 1u))] = i;
      base += __popc(bal);
    }
    if (lane == 0) s_nnz = base;
  }
  double mo[G], so[G];
  if (threadIdx.x < HD) {
    const int h = threadIdx.x / D, j = threadIdx.x - h * D;
    const int hs = a.shift ? h + 1 : h;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int b = b0 + (g < gn ? g : 0);
      mo[g] = hs < H ? a.means[(size_t)b * HD + hs * D + j] : a.tail_mean;
      so[g] = hs < H ? a.sd[(size_t)b * HD + hs * D + j] : a.tail_sd;
    }
  }
  __syncthreads();
  const int nnz = s_nnz;

  // ---- weighted sums: one eps load feeds G instances ------------------------
  if (threadIdx.x < HD) {
    const int o = threadIdx.x;
    double s1[G], s2[G];
#pragma unroll
    for (int g = 0; g < G; ++g) s1[g] = s2[g] = 0.0;
    const double* ep = a.eps + o;
    // the null and mean rows (sampling.py:283-285) lead the ascending list:
    // summed first with their selects, then every other row without any
    // (same elements in the same order as before, so bit-identical)
    int k1 = 0;
    while (k1 < nnz && nz[k1] + a.particle_offset <= a.null_count) {
      const int ng = nz[k1] + a.particle_offset;
      const double ev = __ldg(ep + (size_t)nz[k1] * HD);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double dv = ng < a.null_count ? 0.0 - mo[g] : (ng == a.null_count ? 0.0 : (mo[g] + so[g] * ev) - mo[g]);
        const double w = wt[g * N + nz[k1]];
        s1[g] += w * dv;
        s2[g] += w * dv * dv;
      }
      ++k1;
    }
    for (int k0 = k1; k0 < nnz; k0 += PD) {
      double e[PD];
      int ii[PD];
#pragma unroll
      for (int u = 0; u < PD; ++u) {
        ii[u] = k0 + u < nnz ? nz[k0 + u] : -1;
        e[u] = ii[u] >= 0 ? __ldg(ep + (size_t)ii[u] * HD) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PD; ++u) {
        if (ii[u] < 0) break;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const double dv = (mo[g] + so[g] * e[u]) - mo[g];
          const double w = wt[g * N + ii[u]];
          s1[g] += w * dv;
          s2[g] += w * dv * dv;
        }
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (g < gn) {
        double* rec = recs + g * reclen;
        const double sc = rec[2] > 0.0 ? 1.0 : 0.0;
        rec[kRecHead + o] = sc * s1[g] + 0.0;
        rec[kRecHead + HD + o] = sc * s2[g] + 0.0;
      }
  }
  __syncthreads();
  for (int g = 0; g < gn; ++g) {
    finalize_policy(a, b0 + g, recs + g * reclen, emp);
    __syncthreads();
  }
}

// Finalize from R rank records (config 5, after the all-gather).
template <typename R>
__global__ void __launch_bounds__(kStatsThreads)
    finalize_kernel(const __grid_constant__ StatsArgs<R> a, const double* recs, int count) {
  extern __shared__ __align__(16) double sm[];
  const int HD = a.H * a.D, reclen = kRecHead + 2 * HD;
  double* red = sm;
  double* scale = sm + 32;
  double* comb = scale + max(count, 8) * (1 + kRecHead);
  double* emp = comb + reclen;
  combine_records(recs, count, reclen, HD, a.beta, comb, scale, red);
  finalize_policy(a, 0, comb, emp);
}

}  // namespace mppi
