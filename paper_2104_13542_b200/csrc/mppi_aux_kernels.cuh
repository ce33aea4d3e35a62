// mppi_aux_kernels.cuh — sampling, operator-seam and policy kernels.
//
//  * noise: Halton / Philox unit points -> Acklam ICDF -> B-spline / comb
//    smoothing -> batch centring (sampling.py:89-265, controller.py:166-176);
//  * the float64 operator seam of kernels/__init__.py (jit.py:89-349), one
//    thread per configuration;
//  * the stateless policy update (policy.py:103-155) behind the free
//    functions of the Python API.
#pragma once

#include "mppi_common.cuh"

namespace mppi {

// ------------------------------------------------------------------ noise
// z[(n*K + k)*d + j] for global particle rows [0, rows): Halton (gen 0) or
// Philox (gen 1; counter = (row*K+k, j, step, 0), key = seed).
static __global__ void knots_kernel(double* z, long long rows, int K, int d, int gen, uint64_t seed,
                             unsigned long long step, int* err) {
  const long long total = rows * K * d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % d);
    const long long idx = i / d;  // n*K + k: particle-major Halton index (sampling.py:136)
    double p;
    if (gen == MPPI_GEN_HALTON) {
      p = radical_inverse((uint64_t)idx + 1, kPrimes[j]);
    } else {
      const uint4 r = philox4x32_10(make_uint4((uint32_t)idx, (uint32_t)(idx >> 32), (uint32_t)j,
                                               (uint32_t)step),
                                    make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
      p = u53(r.x, r.y);
    }
    if (!(p >= 0.0 && p < 1.0)) atomicExch(err, 1);
    z[i] = acklam_icdf(p);
  }
}

// eps[n][h][j] from knot values (smooth_sequences, sampling.py:240-265).
// mode 0: sum_k basis[h][k] z[n][k][j]; 1: comb c1 x_h + c2 x_{h-1} + c3 x_{h-2}; 2: identity.
static __global__ void smooth_kernel(const double* z, double* eps, long long rows, int K, int H, int d,
                              int mode, const double* basis, double c1, double c2, double c3) {
  const long long total = rows * H * d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % d);
    const int h = (int)((i / d) % H);
    const long long n = i / ((long long)d * H);
    const double* zn = z + n * K * d;
    double out;
    if (mode == MPPI_SMOOTH_BSPLINE) {
      out = 0.0;
      for (int k = 0; k < K; ++k) out += basis[h * K + k] * zn[k * d + j];
    } else if (mode == MPPI_SMOOTH_COMB) {
      out = c1 * zn[h * d + j];
      if (h >= 1) out += c2 * zn[(h - 1) * d + j];
      if (h >= 2) out += c3 * zn[(h - 2) * d + j];
    } else {
      out = zn[h * d + j];
    }
    eps[i] = out;
  }
}

// Column means over `rows` particles of an (rows, cols) matrix, fixed-order
// tree per column (one block per column). controller.py:174.
static __global__ void column_mean_kernel(const double* x, long long rows, int cols, double* mean) {
  __shared__ double red[256];
  const int c = blockIdx.x;
  double s = 0.0;
  for (long long r = threadIdx.x; r < rows; r += blockDim.x) s += x[r * cols + c];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) mean[c] = red[0] / (double)rows;
}

// dst[r][c] = src[(r + row0)][c] - mean[c] for r < rows.
static __global__ void center_slice_kernel(const double* src, const double* mean, double* dst,
                                    long long row0, long long rows, int cols) {
  const long long total = rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % cols);
    dst[i] = src[i + row0 * cols] - (mean ? mean[c] : 0.0);
  }
}

// Clamped uniform B-spline design matrix (bspline_basis, sampling.py:205-237),
// one thread per horizon step, numpy linspace arithmetic reproduced exactly.
static __global__ void bspline_basis_kernel(int H, int K, int deg, double* basis) {
  const int hi = blockIdx.x * blockDim.x + threadIdx.x;
  if (hi >= H) return;
  double kv[64];
  const int nint = K - deg + 1;  // linspace(0,1,K-deg+1)
  int nk = 0;
  for (int i = 0; i <= deg; ++i) kv[nk++] = 0.0;
  for (int i = 1; i < nint - 1; ++i) kv[nk++] = (double)i * (1.0 / (double)(nint - 1));
  for (int i = 0; i <= deg; ++i) kv[nk++] = 1.0;
  const double t = H > 1 ? (hi == H - 1 ? 1.0 : (double)hi * (1.0 / (double)(H - 1))) : 0.0;
  int span;
  if (t >= 1.0) {
    span = K - 1;
  } else {
    int cnt = 0;  // searchsorted(kv, t, side="right")
    for (int i = 0; i < nk; ++i)
      if (kv[i] <= t) cnt = i + 1;
    span = cnt - 1;
  }
  double vals[16], left[16], right[16];
  for (int i = 0; i <= deg; ++i) vals[i] = 0.0;
  vals[0] = 1.0;
  for (int j = 1; j <= deg; ++j) {
    left[j] = t - kv[span + 1 - j];
    right[j] = kv[span + j] - t;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      const double tmp = vals[r] / (right[r + 1] + left[j - r]);
      vals[r] = saved + right[r + 1] * tmp;
      saved = left[j - r] * tmp;
    }
    vals[j] = saved;
  }
  for (int k = 0; k < K; ++k) basis[hi * K + k] = 0.0;
  for (int i = 0; i <= deg; ++i) basis[hi * K + span - deg + i] = vals[i];
}

// ------------------------------------------------------------------ seam (fp64)
struct SeamChain {
  const double* axes;
  const double* orot;
  const double* otrans;
  const long long* jtype;
};

static __global__ void fk_seam_kernel(const double* q, long long M, int d, SeamChain ch, double* rot,
                               double* trans) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (m >= M) return;
  double Rw[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, tw[3] = {0, 0, 0};
  for (int k = 0; k < d; ++k) {
    double Rmo[9], tmo[3];
    const double qk = q[m * d + k];
    if (ch.jtype[k] == 0) {
      double s, c, Rm[9];
      sincos(qk, &s, &c);
      axis_rotation(ch.axes + 3 * k, s, 1.0 - c, Rm);
      mat33_mul(Rm, ch.orot + 9 * k, Rmo);
      mat33_vec(Rm, ch.otrans + 3 * k, tmo);
    } else {
      for (int i = 0; i < 9; ++i) Rmo[i] = ch.orot[9 * k + i];
      for (int i = 0; i < 3; ++i) tmo[i] = qk * ch.axes[3 * k + i] + ch.otrans[3 * k + i];
    }
    double dtw[3], Rn[9];
    mat33_vec(Rw, tmo, dtw);
    for (int i = 0; i < 3; ++i) tw[i] = tw[i] + dtw[i];
    mat33_mul(Rw, Rmo, Rn);
    for (int i = 0; i < 9; ++i) Rw[i] = Rn[i];
    if ((k + 1) % REORTHO_EVERY == 0) orthonormalize(Rw);
    for (int i = 0; i < 9; ++i) rot[(m * d + k) * 9 + i] = Rw[i];
    for (int i = 0; i < 3; ++i) trans[(m * d + k) * 3 + i] = tw[i];
  }
}

static __global__ void jacobian_seam_kernel(long long M, int d, const double* rot, const double* trans,
                                     const double* axes, const long long* jtype, double* J) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (m >= M) return;
  double* Jm = J + m * 6 * d;
  for (int i = 0; i < 6 * d; ++i) Jm[i] = 0.0;
  const double* e = trans + (m * d + d - 1) * 3;
  for (int k = 0; k < d; ++k) {
    double a[3], p[3];
    if (k == 0) {
      for (int i = 0; i < 3; ++i) {
        a[i] = axes[i];
        p[i] = 0.0;
      }
    } else {
      mat33_vec(rot + (m * d + k - 1) * 9, axes + 3 * k, a);
      for (int i = 0; i < 3; ++i) p[i] = trans[(m * d + k - 1) * 3 + i];
    }
    if (jtype[k] == 0) {
      const double rx = e[0] - p[0], ry = e[1] - p[1], rz = e[2] - p[2];
      Jm[0 * d + k] = a[1] * rz - a[2] * ry;
      Jm[1 * d + k] = a[2] * rx - a[0] * rz;
      Jm[2 * d + k] = a[0] * ry - a[1] * rx;
      Jm[3 * d + k] = a[0];
      Jm[4 * d + k] = a[1];
      Jm[5 * d + k] = a[2];
    } else {
      Jm[0 * d + k] = a[0];
      Jm[1 * d + k] = a[1];
      Jm[2 * d + k] = a[2];
    }
  }
}

static __global__ void manip_seam_kernel(const double* J, long long M, int d, int td, double* out) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (m >= M) return;
  const double* Jm = J + m * 6 * d;
#define JJ(i, k) Jm[(i) * d + (k)]
  if (d == td) {
    double det;
    if (td == 2)
      det = JJ(0, 0) * JJ(1, 1) - JJ(0, 1) * JJ(1, 0);
    else
      det = JJ(0, 0) * (JJ(1, 1) * JJ(2, 2) - JJ(1, 2) * JJ(2, 1)) -
            JJ(0, 1) * (JJ(1, 0) * JJ(2, 2) - JJ(1, 2) * JJ(2, 0)) +
            JJ(0, 2) * (JJ(1, 0) * JJ(2, 1) - JJ(1, 1) * JJ(2, 0));
    out[m] = fabs(det);
    return;
  }
  double G[3][3];
  for (int i = 0; i < td; ++i)
    for (int j = 0; j < td; ++j) {
      double acc = 0.0;
      for (int k = 0; k < d; ++k) acc += JJ(i, k) * JJ(j, k);
      G[i][j] = acc;
    }
#undef JJ
  double det;
  if (td == 2)
    det = G[0][0] * G[1][1] - G[0][1] * G[1][0];
  else
    det = G[0][0] * (G[1][1] * G[2][2] - G[1][2] * G[2][1]) -
          G[0][1] * (G[1][0] * G[2][2] - G[1][2] * G[2][0]) +
          G[0][2] * (G[1][0] * G[2][1] - G[1][1] * G[2][0]);
  out[m] = sqrt(det > 0.0 ? det : 0.0);
}

struct SeamCaps {
  const double* p0;
  const double* p1;
  const double* r;
  const long long* link;
  int n;
};

__device__ __forceinline__ void seam_capsule(const double* rot, const double* trans, long long m,
                                             int d, const SeamCaps& c, int ci, double* P0,
                                             double* P1) {
  const long long lk = c.link[ci];
  const double* Rl = rot + (m * d + lk) * 9;
  const double* tl = trans + (m * d + lk) * 3;
  mat33_vec(Rl, c.p0 + 3 * ci, P0);
  mat33_vec(Rl, c.p1 + 3 * ci, P1);
  for (int i = 0; i < 3; ++i) {
    P0[i] += tl[i];
    P1[i] += tl[i];
  }
}

static __global__ void selfcoll_seam_kernel(const double* rot, const double* trans, long long M, int d,
                                     SeamCaps caps, const long long* pa, const long long* pb, int np,
                                     double* out) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (m >= M) return;
  double best = NO_CONTACT;
  for (int p = 0; p < np; ++p) {
    double a0[3], a1[3], b0[3], b1[3];
    seam_capsule(rot, trans, m, d, caps, (int)pa[p], a0, a1);
    seam_capsule(rot, trans, m, d, caps, (int)pb[p], b0, b1);
    const double val = caps.r[pa[p]] + caps.r[pb[p]] - segseg_dist(a0, a1, b0, b1);
    if (val > best) best = val;
  }
  out[m] = best;
}

// First colliding obstacle index, spheres first, -1 when clear (jit.py:289-332).
static __global__ void envcoll_seam_kernel(const double* rot, const double* trans, long long M, int d,
                                    SeamCaps caps, const double* spheres, int ns,
                                    const double* boxes, int nb, long long* hit) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (m >= M) return;
  long long found = -1;
  if (caps.n > 0 && (ns > 0 || nb > 0)) {
    for (int o = 0; o < ns && found < 0; ++o)
      for (int ci = 0; ci < caps.n; ++ci) {
        double P0[3], P1[3];
        seam_capsule(rot, trans, m, d, caps, ci, P0, P1);
        if (capsule_hits_sphere(P0, P1, caps.r[ci], spheres + 4 * o)) {
          found = o;
          break;
        }
      }
    for (int ob = 0; ob < nb && found < 0; ++ob)
      for (int ci = 0; ci < caps.n; ++ci) {
        double P0[3], P1[3];
        seam_capsule(rot, trans, m, d, caps, ci, P0, P1);
        if (seg_box_dist(P0, P1, boxes + 6 * ob, boxes + 6 * ob + 3) < caps.r[ci]) {
          found = ns + ob;
          break;
        }
      }
  }
  hit[m] = found;
}

// Sequential semi-implicit Euler per (n, j) (jit.py:335-349) — the seam keeps
// the reference's summation order exactly.
static __global__ void integrate_seam_kernel(const double* u, long long N, int H, int d, const double* dts,
                                      const double* th0, const double* thd0, double* pos,
                                      double* vel) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= N * d) return;
  const long long n = i / d;
  const int j = (int)(i % d);
  double v = thd0[j], p = th0[j];
  for (int h = 0; h < H; ++h) {
    const size_t o = ((size_t)n * H + h) * d + j;
    v = v + dts[h] * u[o];
    p = p + dts[h] * v;
    vel[o] = v;
    pos[o] = p;
  }
}

// ------------------------------------------------------------------ policy (stateless)
// particle_weights (policy.py:103-121); single block; status 2 = none finite, 3 = sum <= 0.
static __global__ void weights_kernel(const double* totals, long long n, double beta, double* w,
                               int* status) {
  __shared__ double red[32];
  double m = CUDART_INF;
  for (long long i = threadIdx.x; i < n; i += blockDim.x)
    if (isfinite(totals[i])) m = fmin(m, totals[i]);
  for (int off = 16; off > 0; off >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : CUDART_INF;
    for (int off = 16; off > 0; off >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  m = red[0];
  __syncthreads();
  if (!isfinite(m)) {
    if (threadIdx.x == 0) *status = MPPI_E_ALL_QUARANTINED;
    return;
  }
  for (long long i = threadIdx.x; i < n; i += blockDim.x)
    w[i] = isfinite(totals[i]) ? exp(-(totals[i] - m) / beta) : 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (long long i = 0; i < n; ++i) s += w[i];
    if (!(s > 0.0)) *status = MPPI_E_WEIGHT_UNDERFLOW;
  }
}

// update_mean then update_covariance (policy.py:124-155) with the reference's
// two-pass formulas; one thread per (h, j), single block (H*d <= 1024).
static __global__ void update_policy_kernel(const double* u, const double* w, long long n, int H, int d,
                                     int iso, double alpha_mu, double alpha_sigma, double smin,
                                     double smax, int do_mean, int do_cov, double* means,
                                     double* var, int* status) {
  __shared__ double emp_s[1024];
  __shared__ double wsum_s;
  const int o = threadIdx.x, HD = H * d;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (long long i = 0; i < n; ++i) s += w[i];
    wsum_s = s;
    if (!(s > 0.0)) *status = MPPI_E_WEIGHT_UNDERFLOW;
  }
  __syncthreads();
  const double ws = wsum_s;
  if (!(ws > 0.0)) return;
  double mu = o < HD ? means[o] : 0.0;
  if (do_mean && o < HD) {
    double acc = 0.0;
    for (long long i = 0; i < n; ++i) acc += w[i] * u[i * HD + o];
    mu = (1.0 - alpha_mu) * mu + alpha_mu * (acc / ws);
  }
  if (do_cov && o < HD) {
    double acc = 0.0;
    for (long long i = 0; i < n; ++i) {
      const double dv = u[i * HD + o] - mu;
      acc += w[i] * (dv * dv);
    }
    emp_s[o] = acc / ws;
  }
  __syncthreads();
  if (do_mean && o < HD) means[o] = mu;
  if (do_cov) {
    if (iso) {
      if (o < H) {
        double s = 0.0;
        for (int j = 0; j < d; ++j) s += emp_s[o * d + j];
        double v = (1.0 - alpha_sigma) * var[o] + alpha_sigma * (s / d);
        v = v < smin ? smin : (v > smax ? smax : v);
        var[o] = v;
      }
    } else if (o < HD) {
      double v = (1.0 - alpha_sigma) * var[o] + alpha_sigma * emp_s[o];
      v = v < smin ? smin : (v > smax ? smax : v);
      var[o] = v;
    }
  }
}

// build_control_batch (sampling.py:268-290).
static __global__ void build_controls_kernel(const double* eps, const double* means, const double* sd,
                                      long long n, int H, int d, int null_count, double* out,
                                      int* bad) {
  const long long total = n * H * d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ((long long)H * d);
    const int o = (int)(i % ((long long)H * d));
    double u;
    if (r < null_count)
      u = 0.0;
    else if (r == null_count)
      u = means[o];
    else
      u = means[o] + sd[o] * eps[i];
    out[i] = u;
    if (!isfinite(u)) atomicExch(bad, 1);
  }
}


// Pseudorandom knots for a captured graph: the step number is read from the
// device copy of the host input block. Row index is global (row + offset) so a
// particle-sharded plan draws exactly the rows an unsharded plan would.
static __global__ void knots_ptr_kernel(double* z, long long rows, int K, int d, uint64_t seed,
                                 const unsigned long long* stepctr, unsigned long long iters, int it,
                                 int offset, int* err) {
  const unsigned long long step = stepctr[0] * iters + (unsigned long long)it;
  const long long total = rows * K * d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % d);
    const long long idx = i / d + (long long)offset * K;
    const uint4 r = philox4x32_10(
        make_uint4((uint32_t)idx, (uint32_t)(idx >> 32), (uint32_t)j, (uint32_t)step),
        make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    z[i] = acklam_icdf(u53(r.x, r.y));
  }
  (void)err;
}

static __global__ void halton_points_kernel(double* out, long long count, int dims) {
  const long long total = count * dims;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % dims);
    out[i] = radical_inverse((uint64_t)(i / dims) + 1, kPrimes[j]);
  }
}

static __global__ void gaussianize_kernel(const double* p, long long n, double* out, int* err) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double x = p[i];
    if (!(x >= 0.0 && x < 1.0)) {
      atomicExch(err, 1);
      out[i] = CUDART_NAN;
    } else {
      out[i] = acklam_icdf(x);
    }
  }
}

// Exact distance from every voxel cube to the union of boxes (the broad-phase
// clearance field of env_any_hit).
static __global__ void clearance_kernel(const double* boxes, int nb, int nx, int ny, int nz, double ox,
                                 double oy, double oz, double vox, float* clr) {
  const long long total = (long long)nx * ny * nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int iz = (int)(i % nz), iy = (int)((i / nz) % ny), ix = (int)(i / ((long long)ny * nz));
    const double lo[3] = {ox + ix * vox, oy + iy * vox, oz + iz * vox};
    const double hi[3] = {lo[0] + vox, lo[1] + vox, lo[2] + vox};
    double best = 1e30;
    for (int b = 0; b < nb; ++b) {
      const double* bx = boxes + 6 * b;
      double s = 0.0;
      for (int t = 0; t < 3; ++t) {
        const double g = fmax(fmax(bx[t] - hi[t], lo[t] - bx[3 + t]), 0.0);
        s += g * g;
      }
      best = fmin(best, sqrt(s));
    }
    // round down so the float field never overstates the clearance
    float f = (float)best;
    if ((double)f > best) f = nextafterf(f, 0.0f);
    clr[i] = f;
  }
}

static __global__ void posenc_kernel(const double* q, long long m, int d, float* x) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    for (int k = 0; k < d; ++k) {
      float s, c;
      sincosf((float)q[i * d + k], &s, &c);
      x[i * 16 + k] = s;
      x[i * 16 + d + k] = c;
    }
  }
}

static __global__ void float_to_double_kernel(const float* a, long long n, double* b) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    b[i] = (double)a[i];
}

}  // namespace mppi
