// mppi_seam.cu — the stateless float64 functions of the C ABI: the sampling /
// policy free functions of the Python API (sampling.py, policy.py), the
// reference's six-function operator seam (kernels/__init__.py:50-66,
// jit.py:89-349) and the cost-term free functions (costs.py:76-173). Each
// call copies its host inputs to scratch device buffers on a private stream,
// runs one kernel, copies the result back and synchronises; outputs are
// caller-owned, as the reference's kernels return fresh arrays.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "mppi_abi_util.cuh"
#include "mppi_aux_kernels.cuh"

using namespace mppi;

namespace {

// ---------------------------------------------------------------- cost terms
// One thread per configuration; the small per-call constants travel by value.
struct PoseArgs {
  double rg[9], tg[3], arot[3], atrans[3];
  int full;  // 0: position_only
};

__global__ void pose_cost_kernel(const double* __restrict__ rot, const double* __restrict__ trans, long long M,
                                 const PoseArgs a, double* __restrict__ out) {
  for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < M; m += (long long)gridDim.x * blockDim.x) {
    const double* t = trans + 3 * m;
    const double dx = t[0] - a.tg[0], dy = t[1] - a.tg[1], dz = t[2] - a.tg[2];
    double acc = 0.0;
    for (int i = 0; i < 3; ++i) {  // (R_g^T (t - t_g))_i, weighted
      const double e = a.atrans[i] * (a.rg[i] * dx + a.rg[3 + i] * dy + a.rg[6 + i] * dz);
      acc += e * e;
    }
    double c = sqrt(acc);
    if (a.full) {
      const double* R = rot + 9 * m;
      double fro = 0.0;
      for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) {  // alpha_rot[i] (I - R_g^T R_ee)_ik
          const double g = a.rg[i] * R[k] + a.rg[3 + i] * R[3 + k] + a.rg[6 + i] * R[6 + k];
          const double r = a.arot[i] * ((i == k ? 1.0 : 0.0) - g);
          fro += r * r;
        }
      c += sqrt(fro);
    }
    out[m] = c;
  }
}

__global__ void stop_cost_kernel(const double* __restrict__ vel, long long rows, int H, int d,
                                 const double* __restrict__ lim, double* __restrict__ out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
    const int h = (int)(r % H);
    double acc = 0.0;
    for (int j = 0; j < d; ++j) {
      const double e = fmax(fabs(vel[r * d + j]) - lim[h * d + j], 0.0);
      acc += e * e;
    }
    out[r] = sqrt(acc);
  }
}

__global__ void joint_limit_cost_kernel(const double* __restrict__ pos, long long M, int d,
                                        const double* __restrict__ lo, const double* __restrict__ hi,
                                        double* __restrict__ out) {
  for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < M; m += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < d; ++j) {
      const double q = pos[m * d + j];
      const double e = fmax(lo[j] - q, 0.0) + fmax(q - hi[j], 0.0);
      acc += e * e;
    }
    out[m] = sqrt(acc);
  }
}

__global__ void manip_cost_kernel(const double* __restrict__ mv, long long M, double k_m, double* __restrict__ out) {
  for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < M; m += (long long)gridDim.x * blockDim.x)
    out[m] = mv[m] < k_m ? 1.0 - mv[m] : 0.0;  // NaN compares false -> 0, as np.where
}

}  // namespace

extern "C" {

int mppi_halton_points(int64_t count, int32_t dims, double* out) {
  if (count < 1) return fail(MPPI_E_BAD_ARGUMENT, "count must be >= 1");
  if (dims > 40) return fail(MPPI_E_CONFIG, "halton supports at most 40 dims, got " + std::to_string(dims));
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, d, (size_t)count * dims, (const double*)nullptr);
  halton_points_kernel<<<grid_for(count * dims, 256), 256, 0, S.st>>>(d, count, dims);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d, sizeof(double) * count * dims, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_gaussianize(const double* p, int64_t n, double* out) {
  if (n < 0) return fail(MPPI_E_BAD_ARGUMENT, "negative size");
  if (n == 0) return MPPI_OK;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, dp, n, p);
  DEVPTR(S, double, dout, n, (const double*)nullptr);
  DEVPTR(S, int, err, 1, (const int*)nullptr);
  CK(cudaMemsetAsync(err, 0, sizeof(int), S.st));
  gaussianize_kernel<<<grid_for(n, 256), 256, 0, S.st>>>(dp, n, dout, err);
  CK(cudaGetLastError());
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, S.st));
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  if (herr) return fail(MPPI_E_BAD_ARGUMENT, "unit samples must lie in [0, 1)");
  return MPPI_OK;
}

int mppi_smooth_sequences(const double* knots, int64_t n, int32_t k, int32_t d, int32_t mode,
                          const double* basis, const double* comb, int32_t horizon, double* out) {
  if (n < 0 || k < 1 || d < 1 || horizon < 1) return fail(MPPI_E_BAD_ARGUMENT, "bad shape");
  if (n == 0) return MPPI_OK;
  if (mode == MPPI_SMOOTH_BSPLINE && !basis) return fail(MPPI_E_BAD_ARGUMENT, "basis missing");
  if (mode != MPPI_SMOOTH_BSPLINE && k != horizon) return fail(MPPI_E_BAD_ARGUMENT, "K != H");
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, dz, (size_t)n * k * d, knots);
  DEVPTR(S, double, db, (size_t)horizon * k, mode == MPPI_SMOOTH_BSPLINE ? basis : nullptr);
  DEVPTR(S, double, dout, (size_t)n * horizon * d, (const double*)nullptr);
  const double c1 = comb ? comb[0] : 0.3, c2 = comb ? comb[1] : 0.4, c3 = comb ? comb[2] : 0.3;
  smooth_kernel<<<grid_for(n * horizon * d, 256), 256, 0, S.st>>>(dz, dout, n, k, horizon, d, mode, db, c1, c2, c3);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * n * horizon * d, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_bspline_basis(int32_t horizon, int32_t k, int32_t degree, double* out) {
  if (k < degree + 1) return fail(MPPI_E_CONFIG, "bspline of degree " + std::to_string(degree) +
                                                     " needs at least " + std::to_string(degree + 1) +
                                                     " control points");
  if (horizon < 1 || k + degree + 1 > 64 || degree > 15) return fail(MPPI_E_BAD_ARGUMENT, "bad basis shape");
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, db, (size_t)horizon * k, (const double*)nullptr);
  bspline_basis_kernel<<<(horizon + 63) / 64, 64, 0, S.st>>>(horizon, k, degree, db);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, db, sizeof(double) * horizon * k, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_build_controls(const double* eps, const double* means, const double* stddev, int64_t n,
                        int32_t h, int32_t d, int32_t null_count, double* out) {
  if (n < 1 || h < 1 || d < 1) return fail(MPPI_E_BAD_ARGUMENT, "bad shape");
  SCRATCH_OR_FAIL(S);
  const size_t nhd = (size_t)n * h * d;
  DEVPTR(S, double, de, nhd, eps);
  DEVPTR(S, double, dm, (size_t)h * d, means);
  DEVPTR(S, double, ds, (size_t)h * d, stddev);
  DEVPTR(S, double, dout, nhd, (const double*)nullptr);
  DEVPTR(S, int, bad, 1, (const int*)nullptr);
  CK(cudaMemsetAsync(bad, 0, sizeof(int), S.st));
  build_controls_kernel<<<grid_for(nhd, 256), 256, 0, S.st>>>(de, dm, ds, n, h, d, null_count, dout, bad);
  CK(cudaGetLastError());
  int hb = 0;
  CK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, S.st));
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * nhd, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  if (hb) return fail(MPPI_E_NONFINITE_CONTROL, "control batch contains non-finite entries");
  return MPPI_OK;
}

int mppi_particle_weights(const double* totals, int64_t n, double beta, double* weights) {
  if (n < 1) return fail(MPPI_E_ALL_QUARANTINED, "all particles quarantined; no finite costs");
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, dt, n, totals);
  DEVPTR(S, double, dw, n, (const double*)nullptr);
  DEVPTR(S, int, stt, 1, (const int*)nullptr);
  CK(cudaMemsetAsync(stt, 0, sizeof(int), S.st));
  weights_kernel<<<1, 1024, 0, S.st>>>(dt, n, beta, dw, stt);
  CK(cudaGetLastError());
  int hs = 0;
  CK(cudaMemcpyAsync(&hs, stt, sizeof(int), cudaMemcpyDeviceToHost, S.st));
  CK(cudaMemcpyAsync(weights, dw, sizeof(double) * n, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  if (hs == MPPI_E_ALL_QUARANTINED) return fail(hs, "all particles quarantined; no finite costs");
  if (hs == MPPI_E_WEIGHT_UNDERFLOW) return fail(hs, "all particle weights underflowed to zero; increase beta");
  return MPPI_OK;
}

int mppi_update_policy(const double* controls, const double* weights, int64_t n, int32_t h, int32_t d,
                       int32_t policy_mode, double alpha_mu, double alpha_sigma, double smin, double smax,
                       int32_t do_mean, int32_t do_cov, double* means, double* variances) {
  if (n < 1 || h < 1 || d < 1 || h * d > 1024) return fail(MPPI_E_BAD_ARGUMENT, "bad shape");
  SCRATCH_OR_FAIL(S);
  const size_t nhd = (size_t)n * h * d;
  const size_t nv = policy_mode == MPPI_POLICY_ISOTROPIC ? (size_t)h : (size_t)h * d;
  DEVPTR(S, double, du, nhd, controls);
  DEVPTR(S, double, dw, n, weights);
  DEVPTR(S, double, dm, (size_t)h * d, means);
  DEVPTR(S, double, dv, nv, variances);
  DEVPTR(S, int, stt, 1, (const int*)nullptr);
  CK(cudaMemsetAsync(stt, 0, sizeof(int), S.st));
  update_policy_kernel<<<1, 1024, 0, S.st>>>(du, dw, n, h, d, policy_mode == MPPI_POLICY_ISOTROPIC,
                                             alpha_mu, alpha_sigma, smin, smax, do_mean, do_cov, dm, dv, stt);
  CK(cudaGetLastError());
  int hs = 0;
  CK(cudaMemcpyAsync(&hs, stt, sizeof(int), cudaMemcpyDeviceToHost, S.st));
  CK(cudaMemcpyAsync(means, dm, sizeof(double) * h * d, cudaMemcpyDeviceToHost, S.st));
  CK(cudaMemcpyAsync(variances, dv, sizeof(double) * nv, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  if (hs) return fail(hs, "weight sum must be positive");
  return MPPI_OK;
}

// ---------------------------------------------------------------- operator seam
int mppi_fk_batch(const double* q, int64_t m, int32_t d, const double* axes, const double* orot,
                  const double* otrans, const int64_t* jtype, double* rot_out, double* trans_out) {
  if (m < 0 || d < 1) return fail(MPPI_E_BAD_ARGUMENT, "bad shape");
  if (m == 0) return MPPI_OK;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, dq, (size_t)m * d, q);
  DEVPTR(S, double, da, (size_t)3 * d, axes);
  DEVPTR(S, double, dr, (size_t)9 * d, orot);
  DEVPTR(S, double, dt, (size_t)3 * d, otrans);
  DEVPTR(S, long long, dj, (size_t)d, (const long long*)jtype);
  DEVPTR(S, double, rot, (size_t)m * d * 9, (const double*)nullptr);
  DEVPTR(S, double, tr, (size_t)m * d * 3, (const double*)nullptr);
  SeamChain ch{da, dr, dt, dj};
  fk_seam_kernel<<<(unsigned)((m + 127) / 128), 128, 0, S.st>>>(dq, m, d, ch, rot, tr);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(rot_out, rot, sizeof(double) * m * d * 9, cudaMemcpyDeviceToHost, S.st));
  CK(cudaMemcpyAsync(trans_out, tr, sizeof(double) * m * d * 3, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_jacobian_batch(const double* q, int64_t m, int32_t d, const double* rot, const double* trans,
                        const double* axes, const int64_t* jtype, double* jac_out) {
  (void)q;
  if (m < 0 || d < 1) return fail(MPPI_E_BAD_ARGUMENT, "bad shape");
  if (m == 0) return MPPI_OK;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, drot, (size_t)m * d * 9, rot);
  DEVPTR(S, double, dtr, (size_t)m * d * 3, trans);
  DEVPTR(S, double, da, (size_t)3 * d, axes);
  DEVPTR(S, long long, dj, (size_t)d, (const long long*)jtype);
  DEVPTR(S, double, J, (size_t)m * 6 * d, (const double*)nullptr);
  jacobian_seam_kernel<<<(unsigned)((m + 127) / 128), 128, 0, S.st>>>(m, d, drot, dtr, da, dj, J);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(jac_out, J, sizeof(double) * m * 6 * d, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_manip_batch(const double* jac, int64_t m, int32_t d, int32_t task_dim, double* out) {
  if (m < 0 || d < 1 || (task_dim != 2 && task_dim != 3)) return fail(MPPI_E_BAD_ARGUMENT, "bad shape");
  if (m == 0) return MPPI_OK;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, dj, (size_t)m * 6 * d, jac);
  DEVPTR(S, double, dout, (size_t)m, (const double*)nullptr);
  manip_seam_kernel<<<(unsigned)((m + 127) / 128), 128, 0, S.st>>>(dj, m, d, task_dim, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * m, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_self_collision_batch(const double* rot, const double* trans, int64_t m, int32_t d,
                              const double* cap_p0, const double* cap_p1, const double* cap_r,
                              const int64_t* cap_link, int32_t n_caps, const int64_t* pair_a,
                              const int64_t* pair_b, int32_t n_pairs, double* out) {
  if (m < 0 || d < 1) return fail(MPPI_E_BAD_ARGUMENT, "bad shape");
  if (m == 0) return MPPI_OK;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, drot, (size_t)m * d * 9, rot);
  DEVPTR(S, double, dtr, (size_t)m * d * 3, trans);
  DEVPTR(S, double, p0, (size_t)3 * n_caps, cap_p0);
  DEVPTR(S, double, p1, (size_t)3 * n_caps, cap_p1);
  DEVPTR(S, double, r, (size_t)n_caps, cap_r);
  DEVPTR(S, long long, lk, (size_t)n_caps, (const long long*)cap_link);
  DEVPTR(S, long long, pa, (size_t)n_pairs, (const long long*)pair_a);
  DEVPTR(S, long long, pb, (size_t)n_pairs, (const long long*)pair_b);
  DEVPTR(S, double, dout, (size_t)m, (const double*)nullptr);
  SeamCaps caps{p0, p1, r, lk, n_caps};
  selfcoll_seam_kernel<<<(unsigned)((m + 127) / 128), 128, 0, S.st>>>(drot, dtr, m, d, caps, pa, pb, n_pairs, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * m, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_env_collision_batch(const double* rot, const double* trans, int64_t m, int32_t d,
                             const double* cap_p0, const double* cap_p1, const double* cap_r,
                             const int64_t* cap_link, int32_t n_caps, const double* spheres,
                             int32_t n_spheres, const double* boxes, int32_t n_boxes, int64_t* hit_out) {
  if (m < 0 || d < 1) return fail(MPPI_E_BAD_ARGUMENT, "bad shape");
  if (m == 0) return MPPI_OK;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, drot, (size_t)m * d * 9, rot);
  DEVPTR(S, double, dtr, (size_t)m * d * 3, trans);
  DEVPTR(S, double, p0, (size_t)3 * n_caps, cap_p0);
  DEVPTR(S, double, p1, (size_t)3 * n_caps, cap_p1);
  DEVPTR(S, double, r, (size_t)n_caps, cap_r);
  DEVPTR(S, long long, lk, (size_t)n_caps, (const long long*)cap_link);
  DEVPTR(S, double, sp, (size_t)4 * n_spheres, spheres);
  DEVPTR(S, double, bx, (size_t)6 * n_boxes, boxes);
  DEVPTR(S, long long, hit, (size_t)m, (const long long*)nullptr);
  SeamCaps caps{p0, p1, r, lk, n_caps};
  envcoll_seam_kernel<<<(unsigned)((m + 127) / 128), 128, 0, S.st>>>(drot, dtr, m, d, caps, sp, n_spheres, bx,
                                                                      n_boxes, hit);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(hit_out, hit, sizeof(long long) * m, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_integrate_batch(const double* u, int64_t n, int32_t h, int32_t d, const double* dts,
                         const double* th0, const double* thd0, double* pos_out, double* vel_out) {
  if (n < 0 || h < 1 || d < 1) return fail(MPPI_E_BAD_ARGUMENT, "bad shape");
  if (n == 0) return MPPI_OK;
  SCRATCH_OR_FAIL(S);
  const size_t nhd = (size_t)n * h * d;
  DEVPTR(S, double, du, nhd, u);
  DEVPTR(S, double, ddt, (size_t)h, dts);
  DEVPTR(S, double, t0, (size_t)d, th0);
  DEVPTR(S, double, v0, (size_t)d, thd0);
  DEVPTR(S, double, pos, nhd, (const double*)nullptr);
  DEVPTR(S, double, vel, nhd, (const double*)nullptr);
  integrate_seam_kernel<<<(unsigned)((n * d + 127) / 128), 128, 0, S.st>>>(du, n, h, d, ddt, t0, v0, pos, vel);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(pos_out, pos, sizeof(double) * nhd, cudaMemcpyDeviceToHost, S.st));
  CK(cudaMemcpyAsync(vel_out, vel, sizeof(double) * nhd, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

// ---------------------------------------------------------------- cost terms
int mppi_pose_cost(const double* rot_ee, const double* trans_ee, int64_t m, const double* goal_rot,
                   const double* goal_trans, int32_t mode, const double* alpha_rot, const double* alpha_trans,
                   double* out) {
  if (m < 0 || !trans_ee || !goal_rot || !goal_trans || !alpha_rot || !alpha_trans || !out)
    return fail(MPPI_E_BAD_ARGUMENT, "bad pose_cost arguments");
  if (mode != MPPI_GOAL_POSITION_ONLY && mode != MPPI_GOAL_FULL_POSE)
    return fail(MPPI_E_BAD_ARGUMENT, "unknown goal mode");
  const int full = mode == MPPI_GOAL_FULL_POSE;
  if (full && !rot_ee) return fail(MPPI_E_BAD_ARGUMENT, "rotations required for a full-pose goal");
  if (m == 0) return MPPI_OK;
  PoseArgs a;
  memcpy(a.rg, goal_rot, sizeof a.rg);
  memcpy(a.tg, goal_trans, sizeof a.tg);
  memcpy(a.arot, alpha_rot, sizeof a.arot);
  memcpy(a.atrans, alpha_trans, sizeof a.atrans);
  a.full = full;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, dr, full ? (size_t)m * 9 : 1, full ? rot_ee : nullptr);
  DEVPTR(S, double, dt, (size_t)m * 3, trans_ee);
  DEVPTR(S, double, dout, (size_t)m, (const double*)nullptr);
  pose_cost_kernel<<<grid_for(m, 128), 128, 0, S.st>>>(dr, dt, m, a, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * m, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_stop_cost(const double* vel, int64_t n, int32_t h, int32_t d, const double* limits, double* out) {
  if (n < 0 || h < 1 || d < 1 || !vel || !limits || !out) return fail(MPPI_E_BAD_ARGUMENT, "bad stop_cost arguments");
  if (n == 0) return MPPI_OK;
  const long long rows = (long long)n * h;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, dv, (size_t)rows * d, vel);
  DEVPTR(S, double, dl, (size_t)h * d, limits);
  DEVPTR(S, double, dout, (size_t)rows, (const double*)nullptr);
  stop_cost_kernel<<<grid_for(rows, 128), 128, 0, S.st>>>(dv, rows, h, d, dl, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * rows, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_joint_limit_cost(const double* pos, int64_t m, int32_t d, const double* lo, const double* hi,
                          double* out) {
  if (m < 0 || d < 1 || !pos || !lo || !hi || !out) return fail(MPPI_E_BAD_ARGUMENT, "bad joint_limit_cost arguments");
  if (m == 0) return MPPI_OK;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, dp, (size_t)m * d, pos);
  DEVPTR(S, double, dlo, (size_t)d, lo);
  DEVPTR(S, double, dhi, (size_t)d, hi);
  DEVPTR(S, double, dout, (size_t)m, (const double*)nullptr);
  joint_limit_cost_kernel<<<grid_for(m, 128), 128, 0, S.st>>>(dp, m, d, dlo, dhi, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * m, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

int mppi_manipulability_cost(const double* manip, int64_t m, double k_m, double* out) {
  if (m < 0 || !manip || !out) return fail(MPPI_E_BAD_ARGUMENT, "bad manipulability_cost arguments");
  if (m == 0) return MPPI_OK;
  SCRATCH_OR_FAIL(S);
  DEVPTR(S, double, dm, (size_t)m, manip);
  DEVPTR(S, double, dout, (size_t)m, (const double*)nullptr);
  manip_cost_kernel<<<grid_for(m, 256), 256, 0, S.st>>>(dm, m, k_m, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * m, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

}  // extern "C"
