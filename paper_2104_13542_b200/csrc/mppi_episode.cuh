// mppi_episode.cuh — closed-loop episode on the device.
//
// run_episode (controller.py:331-416) alternates control and plant steps.
// Here every step is a section of a CUDA graph
//   episode_pre_kernel   target_at (simworld.py:175-197, 182-197), filter_state
//                        (controller.py:63-78), state + step counter into the
//                        plan, the plant state into the cost evaluation
//   then two branches that run concurrently:
//   [the control step]   the same rollout / MLP / statistics kernels as mppi_step,
//                        command and step info written to device buffers
//   [instantaneous costs] rollout in "positions given" mode with H = 1 and the
//                        whole-horizon braking time (controller.py:262-269) + MLP
//                        + totals, i.e. CostStack.evaluate of the plant state
//   episode_post_kernel  fallback ladder (controller.py:224-248), filter command,
//                        EE pose (fk_batch), log row, sim_step (simworld.py:108-127)
// One graph holds several steps; the host launches it back to back with no
// synchronisation, and sections past the last step do nothing.
// The step index, filter, fallback and plant state live in EpisodeDev. After a
// non-finite plant state (JointState's finiteness check, rollout.py:34-40) the
// episode is over: later replays mark the plan status MPPI_E_SKIPPED, so the
// control step runs nothing and the policy is left as it was.
#pragma once

#include "mppi_common.cuh"

namespace mppi {

// numpy evaluates a*b + c as two rounded operations; keep the compiler from
// contracting them into an FMA so the host-side formulas hold bit for bit
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }

struct EpisodeDev {
  int i;        // rows logged so far
  int aborted;  // plant state went non-finite
  int armed;    // Controller._fallback_armed
  int pad;
  unsigned long long ctr_base;  // pseudorandom step counter of the first step
  double plant[2 * MAXD];  // plant theta, theta_dot
  double est[2 * MAXD];    // FilterState.last_estimate
  double last_cmd[MAXD];   // FilterState.last_command
  double prev_cmd[MAXD];   // Controller._prev_command
  double cmd[MAXD];        // this step's command
};

struct EpisodeArgs {
  EpisodeDev* ep;
  int S, D, goal_source, interp, script_mode, W, has_noise;
  double dt, lam;
  const double* times;          // (W)
  const double* positions;      // (W,3)
  const double* noise;          // (S,2D) or NULL
  double* state;                // plan state block (2D + counter)
  double* goal;                 // plan goal, instance 0: R(9) t(3) mode
  int* status;                  // plan status word, instance 0
  const double* step_cmd;       // finalize output (D)
  const mppi_step_info* step_info;
  double* ev_pos;               // (D) inputs of the instantaneous-cost evaluation
  double* ev_vel;
  int* ev_status;               // its status word (skip marker when aborted)
  const double* ev_step;        // (1) raw step cost
  const double* ev_terms;       // (6) term rows
  ChainT<double> chain;
  // log, S rows each
  double *t, *theta, *theta_dot, *command, *goalp, *goal_rot, *ee, *ee_rot, *cost_total, *cost_terms;
  int *collision, *fallback, *stat;
};

// target_position_at (simworld.py:182-197): held outside [t_0, t_W-1], stepped
// or linearly interpolated between the bracketing waypoints (searchsorted
// side="right").
__device__ inline void target_position(const EpisodeArgs& a, double t, double* p) {
  const int W = a.W;
  if (t <= a.times[0]) {
    for (int k = 0; k < 3; ++k) p[k] = a.positions[k];
    return;
  }
  if (t >= a.times[W - 1]) {
    for (int k = 0; k < 3; ++k) p[k] = a.positions[3 * (W - 1) + k];
    return;
  }
  int hi = 0;
  while (hi < W && a.times[hi] <= t) ++hi;
  const int lo = hi - 1;
  if (a.interp == MPPI_INTERP_HOLD) {
    for (int k = 0; k < 3; ++k) p[k] = a.positions[3 * lo + k];
    return;
  }
  const double frac = (t - a.times[lo]) / (a.times[hi] - a.times[lo]);
  for (int k = 0; k < 3; ++k)
    p[k] = add_(mul_(1.0 - frac, a.positions[3 * lo + k]), mul_(frac, a.positions[3 * hi + k]));
}

// End-effector frame of one configuration (the last link of fk_batch,
// jit.py:89-111), float64.
__device__ inline void ee_frame(const ChainT<double>& ch, const double* q, int D, double* Rw, double* tw) {
  for (int r = 0; r < 9; ++r) Rw[r] = (r % 4 == 0) ? 1.0 : 0.0;
  for (int r = 0; r < 3; ++r) tw[r] = 0.0;
  for (int k = 0; k < D; ++k) {
    double Rmo[9], tmo[3];
    if (ch.jtype[k] == 0) {
      double s, c, Rm[9];
      sincos(q[k], &s, &c);
      axis_rotation(ch.axes[k], s, 1.0 - c, Rm);
      mat33_mul(Rm, ch.orot[k], Rmo);
      mat33_vec(Rm, ch.otrans[k], tmo);
    } else {
      for (int r = 0; r < 9; ++r) Rmo[r] = ch.orot[k][r];
      for (int r = 0; r < 3; ++r) tmo[r] = q[k] * ch.axes[k][r] + ch.otrans[k][r];
    }
    double dtw[3], Rn[9];
    mat33_vec(Rw, tmo, dtw);
    for (int r = 0; r < 3; ++r) tw[r] = tw[r] + dtw[r];
    mat33_mul(Rw, Rmo, Rn);
    for (int r = 0; r < 9; ++r) Rw[r] = Rn[r];
    if ((k + 1) % REORTHO_EVERY == 0) orthonormalize(Rw);
  }
}

// Top-k rollouts for telemetry (bridge.py:196-203): the k lowest totals of
// instance 0 (ties to the lower particle index; +inf quarantined rows last),
// then the end-effector path of each selected particle from the bundle dump.
// One block: k rounds of a block-wide (total, index) argmin, then k x H FKs.
__global__ void topk_rollouts_kernel(const double* __restrict__ totals, int N, int k, const double* __restrict__ pos,
                                     int H, int D, const ChainT<double> ch, int* __restrict__ idx_out,
                                     double* __restrict__ tot_out, double* __restrict__ ee_out,
                                     unsigned char* __restrict__ taken) {
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ int chosen[64];
  for (int n = threadIdx.x; n < N; n += blockDim.x) taken[n] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = 0; r < k; ++r) {
    double bv = CUDART_INF;
    int bi = 0x7fffffff;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      if (taken[n]) continue;
      double v = totals[n];
      if (isnan(v)) v = CUDART_INF;  // argsort puts NaN last as well
      if (v < bv || (v == bv && n < bi)) {
        bv = v;
        bi = n;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      sv[w] = bv;
      si[w] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = sv[0];
      int b = si[0];
      for (int q = 1; q < nw; ++q)
        if (sv[q] < v || (sv[q] == v && si[q] < b)) {
          v = sv[q];
          b = si[q];
        }
      chosen[r] = b;
      idx_out[r] = b;
      tot_out[r] = totals[b];
      taken[b] = 1;
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < k * H; t += blockDim.x) {
    const int r = t / H, h = t - r * H;
    double Rw[9], tw[3];
    ee_frame(ch, pos + ((size_t)chosen[r] * H + h) * D, D, Rw, tw);
    for (int c = 0; c < 3; ++c) ee_out[(size_t)t * 3 + c] = tw[c];
  }
}

// aborted, or the section is past the episode's last step
__device__ __forceinline__ bool episode_over(const EpisodeArgs& a) { return a.ep->aborted || a.ep->i >= a.S; }

__global__ void episode_pre_kernel(const __grid_constant__ EpisodeArgs a) {
  if (threadIdx.x != 0) return;
  EpisodeDev* ep = a.ep;
  if (episode_over(a)) {  // the control step and the cost evaluation run nothing
    *a.status = MPPI_E_SKIPPED;
    *a.ev_status = MPPI_E_SKIPPED;
    return;
  }
  const int i = ep->i, D = a.D;
  const double t = mul_((double)i, a.dt);
  if (a.goal_source == MPPI_GOAL_SCRIPT) {  // goal_at_position: identity orientation
    double p[3];
    target_position(a, t, p);
    for (int k = 0; k < 9; ++k) a.goal[k] = (k % 4 == 0) ? 1.0 : 0.0;
    for (int k = 0; k < 3; ++k) a.goal[9 + k] = p[k];
    a.goal[12] = (double)a.script_mode;
  }
  for (int k = 0; k < 3; ++k) a.goalp[3 * i + k] = a.goal[9 + k];
  for (int k = 0; k < 9; ++k) a.goal_rot[9 * i + k] = a.goal[k];
  // filter_state for i > 0, the raw plant state at i = 0
  double est[2 * MAXD];
  if (i > 0) {
    for (int j = 0; j < D; ++j) {
      const double pv = add_(ep->est[D + j], mul_(a.dt, ep->last_cmd[j]));
      const double pp = add_(ep->est[j], mul_(a.dt, pv));
      est[j] = add_(mul_(1.0 - a.lam, pp), mul_(a.lam, ep->plant[j]));
      est[D + j] = add_(mul_(1.0 - a.lam, pv), mul_(a.lam, ep->plant[D + j]));
    }
    for (int j = 0; j < 2 * D; ++j) ep->est[j] = est[j];
  } else {
    for (int j = 0; j < 2 * D; ++j) est[j] = ep->plant[j];
  }
  for (int j = 0; j < 2 * D; ++j) a.state[j] = est[j];
  const unsigned long long ctr = ep->ctr_base + (unsigned long long)i;
  reinterpret_cast<unsigned long long*>(a.state)[2 * D] = ctr;
  a.t[i] = t;
  for (int j = 0; j < D; ++j) {
    a.theta[D * i + j] = ep->plant[j];
    a.theta_dot[D * i + j] = ep->plant[D + j];
    a.ev_pos[j] = ep->plant[j];  // instantaneous_costs(state) of the plant state
    a.ev_vel[j] = ep->plant[D + j];
  }
  *a.ev_status = 0;
}

__global__ void episode_post_kernel(const __grid_constant__ EpisodeArgs a) {
  if (threadIdx.x != 0) return;
  EpisodeDev* ep = a.ep;
  if (episode_over(a)) return;
  const int i = ep->i, D = a.D, S = a.S;
  // ---- command: the step's, or the fallback ladder
  const int st = a.step_info->status;
  int fb = MPPI_FALLBACK_NONE;
  if (st == MPPI_OK) {
    ep->armed = 0;
    for (int j = 0; j < D; ++j) {
      ep->cmd[j] = a.step_cmd[j];
      ep->prev_cmd[j] = a.step_cmd[j];
    }
  } else if (!ep->armed) {  // previous command once ...
    ep->armed = 1;
    fb = MPPI_FALLBACK_REISSUE;
    for (int j = 0; j < D; ++j) ep->cmd[j] = ep->prev_cmd[j];
  } else {  // ... then brake
    fb = MPPI_FALLBACK_BRAKE;
    for (int j = 0; j < D; ++j) ep->cmd[j] = 0.0;
  }
  for (int j = 0; j < D; ++j) {
    ep->last_cmd[j] = ep->cmd[j];
    a.command[D * i + j] = ep->cmd[j];
  }
  a.fallback[i] = fb;
  a.stat[i] = st;
  // ---- instantaneous_costs of the plant state
  a.cost_total[i] = a.ev_step[0];
  for (int k = 0; k < N_TERMS; ++k) a.cost_terms[(size_t)k * S + i] = a.ev_terms[k];
  a.collision[i] = a.ev_terms[T_ENV] > 0.0 ? 1 : 0;
  // end-effector frame: fk_batch(chain, theta)[.., -1] (jit.py:89-111)
  double Rw[9], tw[3];
  ee_frame(a.chain, ep->plant, D, Rw, tw);
  for (int r = 0; r < 3; ++r) a.ee[3 * i + r] = tw[r];
  for (int r = 0; r < 9; ++r) a.ee_rot[9 * i + r] = Rw[r];
  // sim_step: semi-implicit Euler + the caller's noise draws
  double nx[2 * MAXD];
  bool fin = true;
  for (int j = 0; j < D; ++j) {
    const double u = ep->cmd[j];
    double v = add_(ep->plant[D + j], mul_(a.dt, u));
    double p = add_(ep->plant[j], mul_(a.dt, v));
    if (a.has_noise) {
      p = add_(p, a.noise[(size_t)2 * D * i + j]);
      v = add_(v, a.noise[(size_t)2 * D * i + D + j]);
    }
    nx[j] = p;
    nx[D + j] = v;
    fin = fin && isfinite(p) && isfinite(v) && isfinite(u);
  }
  if (fin) {
    for (int j = 0; j < 2 * D; ++j) ep->plant[j] = nx[j];
  } else {
    ep->aborted = 1;  // "plant diverged at step i": this row is kept
  }
  ep->i = i + 1;
}

}  // namespace mppi
