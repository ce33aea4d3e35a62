// mppi_abi.cu — the C ABI (include/mppi_b200.h): plans, CUDA-graph step,
// evaluation, the particle-sharded update and the stateless seam functions.
//
// Build (see __graft_entry__.build):
//   nvcc -shared -Xcompiler -fPIC -O3 -lineinfo -std=c++17
//        -gencode arch=compute_100a,code=sm_100a csrc/*.cu -o _mppi_b200.so
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "mppi_abi_util.cuh"
#include "mppi_aux_kernels.cuh"
#include "mppi_launch.cuh"
#include "mppi_mlp.cuh"
#include "mppi_episode.cuh"

using namespace mppi;

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

namespace {

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  int alloc(size_t count) {
    if (count <= n && p) return MPPI_OK;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (count == 0) return MPPI_OK;
    CK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
    return MPPI_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct HostChain {
  int dof = 0, task_dim = 3, n_caps = 0, n_pairs = 0;
  std::vector<double> axes, orot, otrans, limits, vel, acc, p0, p1, r;
  std::vector<long long> jtype, link, pa, pb;
};

template <typename R>
void fill_chain(const HostChain& c, double k_jl, ChainT<R>& o) {
  memset(&o, 0, sizeof(o));
  o.dof = c.dof;
  o.task_dim = c.task_dim;
  o.n_caps = c.n_caps;
  o.n_pairs = c.n_pairs;
  for (int k = 0; k < c.dof; ++k) {
    o.jtype[k] = (int)c.jtype[k];
    for (int i = 0; i < 3; ++i) o.axes[k][i] = (R)c.axes[3 * k + i];
    for (int i = 0; i < 9; ++i) o.orot[k][i] = (R)c.orot[9 * k + i];
    for (int i = 0; i < 3; ++i) o.otrans[k][i] = (R)c.otrans[3 * k + i];
    const double lo = c.limits[2 * k], hi = c.limits[2 * k + 1], span = hi - lo;
    o.lo[k] = (R)(lo + k_jl * span);  // shrunken_limits, costs.py:111-116
    o.hi[k] = (R)(hi - k_jl * span);
    o.accel[k] = (R)c.acc[k];
  }
  for (int i = 0; i < c.n_caps; ++i) {
    o.cap_link[i] = (int)c.link[i];
    o.cap_r[i] = (R)c.r[i];
    for (int t = 0; t < 3; ++t) {
      o.cap_p0[i][t] = (R)c.p0[3 * i + t];
      o.cap_p1[i][t] = (R)c.p1[3 * i + t];
    }
  }
  for (int i = 0; i < c.n_pairs; ++i) {
    o.pair_a[i] = (int)c.pa[i];
    o.pair_b[i] = (int)c.pb[i];
  }
}

template <typename R>
void fill_cost(const mppi_cost_desc& w, int has_pairs, int has_world, CostT<R>& o) {
  memset(&o, 0, sizeof(o));
  for (int i = 0; i < 3; ++i) {
    o.alpha_rot[i] = (R)w.alpha_rot[i];
    o.alpha_trans[i] = (R)w.alpha_trans[i];
  }
  o.a_stop = (R)w.alpha_stop;
  o.a_joint = (R)w.alpha_joint;
  o.a_manip = (R)w.alpha_manip;
  o.a_coll = (R)w.alpha_coll;
  o.k_m = (R)w.k_m;
  o.use_stop = w.alpha_stop > 0.0;
  o.use_joint = w.alpha_joint > 0.0;
  o.use_manip = w.alpha_manip > 0.0;
  int sc = w.self_collision;
  if (sc == MPPI_SELFCOLL_ORACLE && !has_pairs) sc = MPPI_SELFCOLL_ORACLE;  // NO_CONTACT -> 0
  o.selfcoll = w.alpha_coll > 0.0 ? sc : MPPI_SELFCOLL_NONE;
  o.use_env = (w.alpha_coll > 0.0) && has_world;
}

}  // namespace

// ------------------------------------------------------------------ the plan
struct mppi_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  int D = 0, H = 0, N = 0, B = 1, Kn = 0, iters = 1, null_count = 0, policy_mode = 0;
  int precision = 0, generator = 0, smoothing = 0, degree = 3, offset = 0, Ntot = 0;
  uint64_t seed = 0;
  double comb[3] = {0.3, 0.4, 0.3};
  double gamma = 0.99, tw = 1.0, beta = 0.5, alpha_mu = 0.9, alpha_sigma = 0.5, sigma0_sq = 1.0,
         smin = 1e-4, smax = 1.0, tail = 0.0;
  std::vector<double> dts;
  HostChain chain;
  mppi_cost_desc costs{};
  ChainT<float> chf;
  ChainT<double> chd;
  // world
  int ns = 0, nb = 0;
  DevBuf<double> sph_d, box_d;
  DevBuf<float> sph_f, box_f;
  DevBuf<float> clearance;
  int gx = 0, gy = 0, gz = 0;
  double gorigin[3] = {0, 0, 0}, gvoxel = 0.0;
  // learned collision
  bool mlp_ready = false;
  MlpWeights mlp;
  // device state
  DevBuf<double> eps, z, basis, colmean;
  DevBuf<double> means, var, sd, prev_means, prev_sd, goal, state;
  DevBuf<unsigned char> stepbuf;  // R-typed step costs
  DevBuf<float> mlp_x, mlp_d;
  DevBuf<double> totals, records, out_record, cmd, counters_pad;
  DevBuf<unsigned> counters;
  DevBuf<unsigned long long> dbg;  // MPPI_DEBUG_TIMERS=1: stats-kernel phase stamps
  DevBuf<int> status, bad;
  DevBuf<mppi_step_info> info;
  int nblk = 1, ppb = 64;
  int dump = 0;  // bundle dumps for instance 0
  DevBuf<double> d_pos, d_vel, d_acc, d_terms, d_step, d_w;
  // pinned staging
  // pinned host staging: one H2D node copies h_state (+ step counter) into the
  // graph; h_cmd / h_info are mapped and written directly by the finalize
  double* h_state = nullptr;          // (B,2D)
  double* h_cmd = nullptr;            // (B,D)
  mppi_step_info* h_info = nullptr;   // (B)
  double* m_state = nullptr;          // device aliases of the above
  double* m_cmd = nullptr;
  mppi_step_info* m_info = nullptr;
  std::vector<double> goal_host;
  bool goal_dirty = false;  // goal_host newer than the device copy (uploaded lazily: flush_goal)
  // graph
  cudaGraphExec_t graph = nullptr;       // lean step graph (production)
  cudaGraphExec_t graph_prof = nullptr;  // same step + event-record nodes between the stages
  // Single-instance plans pass the joint state as a rollout kernel PARAMETER:
  // each step rewrites the captured rollout nodes' arguments
  // (cudaGraphExecKernelNodeSetParams) instead of replaying an H2D copy node,
  // whose copy-engine hand-off cost ~4 us of device time per step.
  struct InlineNode {
    cudaGraphNode_t node;
    cudaKernelNodeParams kp;
    std::vector<unsigned char> args;  // RolloutArgs<R> image
    size_t st_off;                    // offsetof(RolloutArgs<R>, st0)
    size_t g_off;                     // offsetof(RolloutArgs<R>, g0)
    void* argv[1];
  };
  std::vector<InlineNode> inl, inl_prof;
  std::vector<InlineNode>* capture_inl = nullptr;  // set while capturing a graph with inline state
  cudaGraph_t graph_tmpl = nullptr, graph_tmpl_prof = nullptr;  // kept alive: node handles index them
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaEvent_t> stage_ev;
  int profile_level = 0;  // 0 none, 1 device time of the lean graph, 2 instrumented graph (stage times)
  unsigned long long step_counter = 0;
  int sharded_iter = 0;
  // particle-sharded exchange over peer memory (mppi_step_exchange)
  DevBuf<double> peer_recv_buf;             // [2][world][reclen] this rank's receive slots
  DevBuf<unsigned long long> peer_flag_buf;  // [world]
  DevBuf<double*> peer_recv_tab;            // [world] pointers (peer mappings), device
  DevBuf<unsigned long long*> peer_flag_tab;
  int peer_world = 0, peer_rank = 0;
  bool peer_active = false;                 // set while enqueuing an exchange step
  unsigned long long peer_seq = 0;
  double peer_timeout_s = 5.0;                         // mppi_set_exchange_timeout
  std::vector<unsigned long long*> peer_flag_host;     // every rank's flag array (this rank's view)
  // eval scratch
  DevBuf<double> e_in0, e_in1, e_pos, e_vel, e_acc, e_terms, e_step, e_tot, e_state, e_dts;
  DevBuf<unsigned char> e_stepbuf;
  DevBuf<float> e_x, e_d;
  DevBuf<int> e_status;
  DevBuf<double> e_w;  // mppi_replay_bundle: weights of the replayed iteration
  DevBuf<double> e_records;
  DevBuf<unsigned> e_counters;
  // closed-loop episode (mppi_episode): device state, log, script, noise,
  // the step's command/info (device instead of mapped host) and the
  // instantaneous-cost evaluation of the plant state (n = 1, H = 1)
  DevBuf<double> ep_state, ep_log, ep_script, ep_noise, ep_cmd;
  DevBuf<int> ep_ilog;
  DevBuf<mppi_step_info> ep_info;
  DevBuf<double> ev_in, ev_out, ev_records;
  DevBuf<unsigned char> ev_stepbuf;
  DevBuf<float> ev_x, ev_d;
  DevBuf<int> ev_status;
  DevBuf<unsigned> ev_counters;
  double* cmd_dst = nullptr;             // finalize outputs while capturing an episode
  mppi_step_info* info_dst = nullptr;
  cudaStream_t stream2 = nullptr;        // the episode's cost-evaluation branch
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaGraphExec_t ep_graph = nullptr;    // last episode graph, reused while its arguments match
  std::vector<unsigned char> ep_key;

  bool learned() const {
    return costs.self_collision == MPPI_SELFCOLL_LEARNED && costs.alpha_coll > 0.0;
  }
};

namespace {

int set_device(mppi_plan* p) {
  CK(cudaSetDevice(p->device));
  return MPPI_OK;
}

// The device copy of the goals, brought up to date before any work that
// reads it (the inline-state step graph carries the goal in its parameters
// and does not need it). From pageable memory: the copy has read goal_host
// when cudaMemcpyAsync returns, so the host may edit it right away.
// The copy is queued on the stream the reading work is queued on (`st`, the
// plan's stream unless the caller passed its own), so it is ordered before it.
int flush_goal(mppi_plan* p, cudaStream_t st = nullptr) {
  if (!p->goal_dirty) return MPPI_OK;
  CK(cudaMemcpyAsync(p->goal.p, p->goal_host.data(), sizeof(double) * 16 * p->B, cudaMemcpyHostToDevice,
                     st ? st : p->stream));
  p->goal_dirty = false;
  return MPPI_OK;
}

void invalidate_graph(mppi_plan* p) {
  if (p->graph) cudaGraphExecDestroy(p->graph);
  if (p->graph_prof) cudaGraphExecDestroy(p->graph_prof);
  if (p->graph_tmpl) cudaGraphDestroy(p->graph_tmpl);
  if (p->graph_tmpl_prof) cudaGraphDestroy(p->graph_tmpl_prof);
  p->graph_tmpl = p->graph_tmpl_prof = nullptr;
  p->inl.clear();
  p->inl_prof.clear();
  if (p->ep_graph) cudaGraphExecDestroy(p->ep_graph);
  p->ep_graph = nullptr;
  p->graph = nullptr;
  p->graph_prof = nullptr;
}

template <typename R>
WorldT<R> world_of(mppi_plan* p) {
  WorldT<R> w{};
  if constexpr (sizeof(R) == 4) {
    w.spheres = p->sph_f.p;
    w.boxes = p->box_f.p;
  } else {
    w.spheres = p->sph_d.p;
    w.boxes = p->box_d.p;
  }
  w.ns = p->ns;
  w.nb = p->nb;
  w.sdf = p->clearance.p;
  w.nx = p->gx;
  w.ny = p->gy;
  w.nz = p->gz;
  w.ox = (R)p->gorigin[0];
  w.oy = (R)p->gorigin[1];
  w.oz = (R)p->gorigin[2];
  w.voxel = (R)p->gvoxel;
  return w;
}

// FkFold of the chain (float64 on the host): K = skew(axis), K^2 = a a^T - I.
void fill_fold(const HostChain& c, FkFold& f) {
  memset(&f, 0, sizeof(f));
  for (int k = 0; k < c.dof; ++k) {
    const double* ax = &c.axes[3 * k];
    const double K[3][3] = {{0.0, -ax[2], ax[1]}, {ax[2], 0.0, -ax[0]}, {-ax[1], ax[0], 0.0}};
    double K2[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int m = 0; m < 3; ++m) s += K[i][m] * K[m][j];
        K2[i][j] = s;
      }
    const double* O = &c.orot[9 * k];
    const double* t = &c.otrans[3 * k];
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) {
        double sa = 0.0, sb = 0.0;
        for (int m = 0; m < 3; ++m) {
          sa += K[i][m] * O[3 * m + j];
          sb += K2[i][m] * O[3 * m + j];
        }
        f.O[k][i][j] = (float)O[3 * i + j];
        f.A[k][i][j] = (float)sa;
        f.B[k][i][j] = (float)sb;
      }
      double ta = 0.0, tb = 0.0;
      for (int m = 0; m < 3; ++m) {
        ta += K[i][m] * t[m];
        tb += K2[i][m] * t[m];
      }
      f.t[k][i] = (float)t[i];
      f.a[k][i] = (float)ta;
      f.b[k][i] = (float)tb;
    }
  }
}

// Build the static part of the rollout arguments for horizon H and dt schedule.
template <typename R>
void rollout_static(mppi_plan* p, int H, const double* dts, RolloutArgs<R>& a) {
  memset(&a, 0, sizeof(a));
  if (std::is_same<R, float>::value) fill_fold(p->chain, a.fold);
  fill_chain(p->chain, p->costs.k_jl, a.chain);
  fill_cost(p->costs, p->chain.n_pairs > 0, (p->ns + p->nb) > 0, a.cost);
  a.world = world_of<R>(p);
  double rem = 0.0;
  std::vector<double> remaining(H);
  for (int h = H - 1; h >= 0; --h) {  // np.cumsum(dts[::-1])[::-1]
    rem += dts[h];
    remaining[h] = rem;
  }
  for (int h = 0; h < H; ++h) {
    a.dts[h] = (R)dts[h];
    a.remaining[h] = (R)remaining[h];
  }
  a.H = H;
}

template <typename R>
void stats_static(mppi_plan* p, int H, double gamma, double tw, StatsArgs<R>& s) {
  memset(&s, 0, sizeof(s));
  s.H = H;
  s.D = p->D;
  s.beta = p->beta;
  s.alpha_mu = p->alpha_mu;
  s.alpha_sigma = p->alpha_sigma;
  s.smin = p->smin;
  s.smax = p->smax;
  s.a_coll = p->costs.alpha_coll;
  s.isotropic = p->policy_mode == MPPI_POLICY_ISOTROPIC;
  s.tail_mean = p->tail;
  s.tail_var = p->sigma0_sq;
  s.tail_sd = std::sqrt(p->sigma0_sq);
  for (int h = 0; h < H; ++h) s.disc[h] = std::pow(gamma, (double)h);  // gamma ** arange(H)
  s.dlast = s.disc[H - 1] * tw;
  s.learned = p->learned() ? 1 : 0;
}

void choose_blocks(int N, int B, int& ppb, int& nblk) {
  // Enough instances to fill the GPU on their own (>= one per SM; config 4):
  // one block per instance, no record combine (4096 x 500: statistics 2.22
  // -> 1.59 ms; at 64 instances it would halve the parallelism). Otherwise 32
  // particles per block (latency: more blocks pull eps/step costs in
  // parallel); up to 16 * kClusterMaxPPB = 2048 particles grow the block to
  // keep one <= 16-CTA cluster per instance (stats_cluster_kernel); beyond
  // that at most 296 blocks per instance (the record combine is linear in it)
  if (B >= 148 && N <= 2048) {
    ppb = N;
    nblk = 1;
    return;
  }
  ppb = 32;
  if (N > 16 * 32 && N <= 16 * kClusterMaxPPB) ppb = (N + 15) / 16;
  // A/B knob, clamped to a layout the plan can launch: [1, min(N, 1024)]
  // particles per block (statistics shared memory stays < 64 KB at H*D <= 512)
  if (const char* ev = getenv("MPPI_STATS_PPB")) ppb = std::min(std::max(1, atoi(ev)), std::min(N, 1024));
  nblk = (N + ppb - 1) / ppb;
  if (nblk > kStatsMaxBlocks) {
    nblk = kStatsMaxBlocks;
    ppb = (N + nblk - 1) / nblk;
    nblk = (N + ppb - 1) / ppb;
  }
}

// Enqueue one optimisation iteration (rollout -> [MLP] -> statistics) for all
// B instances. `inline_final` false writes the rank record instead.
template <typename R>
int enqueue_iteration(mppi_plan* p, int it, bool inline_final, double* out_record, cudaStream_t st,
                      unsigned stages = 7u) {
  RolloutArgs<R> a;
  rollout_static<R>(p, p->H, p->dts.data(), a);
  a.N = p->N;
  a.B = p->B;
  a.null_count = p->null_count;
  a.particle_offset = p->offset;
  a.mode = 0;
  a.shift = it == 0;
  a.check_var = 1;
  a.skip_on_status = 1;
  a.pdl_early = (pdl_mask() & PDL_EARLY) ? 1 : 0;
  a.dbg = p->dbg.p ? p->dbg.p + 16 * p->nblk : nullptr;
  a.tail_mean = p->tail;
  a.tail_sd = std::sqrt(p->sigma0_sq);
  a.eps = p->eps.p;
  a.means = p->means.p;
  a.sd = p->sd.p;
  a.state = p->state.p;
  a.goal = p->goal.p;
  a.step = reinterpret_cast<R*>(p->stepbuf.p);
  a.mlp_x = p->learned() ? p->mlp_x.p : nullptr;
  // float plans hand the MLP 32-byte position rows instead of 64-byte encodings
  // (it recomputes the same fp32 sincos_); float64 plans keep the encodings of
  // their float64 positions
  a.mlp_x_q = std::is_same<R, float>::value && getenv("MPPI_MLP_POSENC") == nullptr ? 1 : 0;
  a.status = p->status.p;
  a.bad = p->bad.p;
  if (p->dump) {
    a.out_pos = p->d_pos.p;
    a.out_vel = p->d_vel.p;
    a.out_acc = p->d_acc.p;
    a.out_terms = p->d_terms.p;
  }
  // Rollout + MLP in one kernel (mppi_fused.cuh) when the particles fit one
  // wave. Opt-in (MPPI_FUSE=1): measured 1.5-2 us slower per cold-L2 step than
  // the two kernels on B200.
  bool fused = false;
  if constexpr (std::is_same<R, float>::value) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    fused = p->learned() && getenv("MPPI_FUSE") != nullptr &&
            ((long long)p->B * p->N + 3) / 4 <= sms && fused_cap_bytes_f32(a) <= 2 * kABuf;
    if (fused) {
      a.mlp_x = nullptr;
      if (stages & 1u) CK(launch_rollout_mlp_any(a, p->D, p->mlp.img, p->mlp_d.p, st));
    }
  }
  if (!fused) {
    if (p->capture_inl && (stages & 1u)) {
      a.state_inline = 1;
      for (int j = 0; j < 2 * p->D; ++j) a.st0[j] = p->h_state[j];
      for (int j = 0; j < 16; ++j) a.g0[j] = p->goal_host[j];
    }
    if (stages & 1u) CK(launch_rollout_any<R>(a, p->D, (long long)p->B * p->N, st));
    if (p->capture_inl && (stages & 1u)) {  // remember the node and its argument image
      cudaStreamCaptureStatus cs;
      const cudaGraphNode_t* deps = nullptr;
      size_t ndeps = 0;
      CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &ndeps));
      if (cs != cudaStreamCaptureStatusActive || ndeps != 1) return fail(MPPI_E_CUDA, "rollout node not found");
      mppi_plan::InlineNode n;
      n.node = deps[0];
      CK(cudaGraphKernelNodeGetParams(n.node, &n.kp));
      n.args.assign(reinterpret_cast<const unsigned char*>(&a), reinterpret_cast<const unsigned char*>(&a) + sizeof(a));
      n.st_off = offsetof(RolloutArgs<R>, st0);
      n.g_off = offsetof(RolloutArgs<R>, g0);
      p->capture_inl->push_back(std::move(n));
    }
    if ((stages & 2u) && p->learned())
      CK(mlp_forward(p->mlp, p->mlp_x.p, (long long)p->B * p->N * p->H, p->mlp_d.p, st, a.mlp_x_q));
  }
  StatsArgs<R> s;
  stats_static<R>(p, p->H, p->gamma, p->tw, s);
  s.N = p->N;
  s.B = p->B;
  s.null_count = p->null_count;
  s.particle_offset = p->offset;
  s.ppb = p->ppb;
  s.nblk = p->nblk;
  s.shift = it == 0;
  s.finalize_inline = inline_final;
  s.reset_status = inline_final && it == p->iters - 1;
  s.step = reinterpret_cast<const R*>(p->stepbuf.p);
  s.mlp_d = p->learned() ? p->mlp_d.p : nullptr;
  s.eps = p->eps.p;
  s.means = p->means.p;
  s.var = p->var.p;
  s.sd = p->sd.p;
  s.prev_means = p->prev_means.p;
  s.prev_sd = p->prev_sd.p;
  s.totals = p->totals.p;
  s.records = p->records.p;
  s.out_record = out_record;
  s.counters = p->counters.p;
  s.status = p->status.p;
  s.bad = p->bad.p;
  s.dbg = p->dbg.p;
  if (p->peer_active && !inline_final) {
    s.peer_recv = p->peer_recv_tab.p;
    s.peer_flags = p->peer_flag_tab.p;
    s.my_recv = p->peer_recv_buf.p;
    s.my_flags = p->peer_flag_buf.p;
    s.world = p->peer_world;
    s.rank = p->peer_rank;
    s.seq = p->peer_seq;
    s.peer_timeout_ns = (unsigned long long)(p->peer_timeout_s * 1e9);
    s.reset_status = it == p->iters - 1;
  }
  s.cmd = p->cmd_dst ? p->cmd_dst : p->m_cmd;  // mapped host memory: no D2H copy node
  s.info = p->info_dst ? p->info_dst : p->m_info;
  if (p->dump) {
    s.dump_step = p->d_step.p;
    s.dump_terms = p->d_terms.p;
    s.dump_weights = inline_final ? p->d_w.p : nullptr;
  }
  if (stages & 4u) CK(launch_stats_any<R>(s, p->D, st));
  return MPPI_OK;
}

int enqueue_sampling(mppi_plan* p, int it, cudaStream_t st) {
  if (p->generator != MPPI_GEN_PSEUDORANDOM) return MPPI_OK;
  // Philox counter = step * iterations + it; the step number is read from the
  // device copy of the input block so the captured graph stays valid.
  const long long rows = p->N;  // pseudorandom rows are local (no centring)
  const long long nz = rows * p->Kn * p->D;
  knots_ptr_kernel<<<grid_for(nz, 256), 256, 0, st>>>(p->z.p, rows, p->Kn, p->D, p->seed,
                                                      reinterpret_cast<const unsigned long long*>(
                                                          p->state.p + (size_t)p->B * 2 * p->D),
                                                      (unsigned long long)p->iters, it, p->offset,
                                                      p->status.p);
  CK(cudaGetLastError());
  const long long ne = rows * p->H * p->D;
  smooth_kernel<<<grid_for(ne, 256), 256, 0, st>>>(p->z.p, p->eps.p, rows, p->Kn, p->H, p->D,
                                                   p->smoothing, p->basis.p, p->comb[0], p->comb[1],
                                                   p->comb[2]);
  CK(cudaGetLastError());
  return MPPI_OK;
}

int enqueue_step_body(mppi_plan* p, cudaStream_t st, bool stage_events, bool h2d = true) {
  const int B = p->B, D = p->D;
  // one H2D node: the (B,2d) state followed by the step counter (pseudorandom
  // generator). Status words were re-armed by the previous step's finalize.
  // (The episode graph writes the state on the device instead.)
  if (h2d && !p->capture_inl)
    CK(cudaMemcpyAsync(p->state.p, p->h_state, sizeof(double) * (B * 2 * D + 1), cudaMemcpyHostToDevice, st));
  // event-record nodes between the stages give per-kernel device times of
  // every replayed step (mppi_step_info.*_ms)
  // event-record nodes between the stages (instrumented graph only: each node
  // serialises the replay, ~3.5 us apiece on B200)
  auto mark = [&](int i) -> int {
    if (stage_events) CK(cudaEventRecordWithFlags(p->stage_ev[i], st, cudaEventRecordExternal));
    return MPPI_OK;
  };
  for (int it = 0; it < p->iters; ++it) {
    CKR(mark(4 * it + 0));
    CKR(enqueue_sampling(p, it, st));  // no-op (and a zero-length stage) unless pseudorandom
    for (int sg = 0; sg < 3; ++sg) {
      CKR(mark(4 * it + 1 + sg));
      if (p->precision == MPPI_FP64)
        CKR(enqueue_iteration<double>(p, it, true, nullptr, st, 1u << sg));
      else
        CKR(enqueue_iteration<float>(p, it, true, nullptr, st, 1u << sg));
    }
  }
  CKR(mark(4 * p->iters));
  return MPPI_OK;
}

int ensure_graph(mppi_plan* p, bool prof = false) {
  cudaGraphExec_t* slot = prof ? &p->graph_prof : &p->graph;
  if (*slot) return MPPI_OK;
  if (p->learned() && !p->mlp_ready)
    return fail(MPPI_E_CONFIG, "learned self-collision selected but mppi_set_mlp was not called");
  cudaGraph_t g = nullptr;
  // the state as a kernel parameter: one instance, no device-side step counter
  // (Philox), the two-kernel path (MPPI_INLINE_STATE=0 restores the H2D node)
  const char* env = getenv("MPPI_INLINE_STATE");
  std::vector<mppi_plan::InlineNode>& nodes = prof ? p->inl_prof : p->inl;
  nodes.clear();
  const bool inl = p->B == 1 && p->generator != MPPI_GEN_PSEUDORANDOM && !(env && env[0] == '0') &&
                   getenv("MPPI_FUSE") == nullptr;
  p->capture_inl = inl ? &nodes : nullptr;
  CK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_step_body(p, p->stream, prof);
  p->capture_inl = nullptr;
  cudaError_t e = cudaStreamEndCapture(p->stream, &g);
  if (rc != MPPI_OK) {
    if (g) cudaGraphDestroy(g);
    nodes.clear();
    return rc;
  }
  if (e != cudaSuccess) return fail(MPPI_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(slot, g, 0);
  if (nodes.empty()) {
    cudaGraphDestroy(g);
  } else {
    (prof ? p->graph_tmpl_prof : p->graph_tmpl) = g;
    for (auto& n : nodes) {
      n.argv[0] = n.args.data();
      n.kp.kernelParams = n.argv;
      n.kp.extra = nullptr;
    }
  }
  if (e != cudaSuccess) return fail(MPPI_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  return MPPI_OK;
}

int copy_chain(const mppi_chain_desc* c, HostChain& h) {
  if (!c || c->dof < 1 || c->dof > MPPI_MAX_DOF)
    return fail(MPPI_E_CONFIG, "chain dof must lie in [1, " + std::to_string(MPPI_MAX_DOF) + "]");
  if (c->n_caps < 0 || c->n_caps > MPPI_MAX_CAPSULES) return fail(MPPI_E_CONFIG, "too many capsules");
  if (c->n_pairs < 0 || c->n_pairs > MPPI_MAX_PAIRS) return fail(MPPI_E_CONFIG, "too many pairs");
  const int d = c->dof;
  h.dof = d;
  h.task_dim = c->task_dim;
  h.n_caps = c->n_caps;
  h.n_pairs = c->n_pairs;
  h.axes.assign(c->axes, c->axes + 3 * d);
  h.orot.assign(c->origin_rot, c->origin_rot + 9 * d);
  h.otrans.assign(c->origin_trans, c->origin_trans + 3 * d);
  h.jtype.assign(c->jtype, c->jtype + d);
  h.limits.assign(c->joint_limits, c->joint_limits + 2 * d);
  h.vel.assign(c->velocity_limits, c->velocity_limits + d);
  h.acc.assign(c->accel_limits, c->accel_limits + d);
  if (c->n_caps) {
    h.p0.assign(c->cap_p0, c->cap_p0 + 3 * c->n_caps);
    h.p1.assign(c->cap_p1, c->cap_p1 + 3 * c->n_caps);
    h.r.assign(c->cap_r, c->cap_r + c->n_caps);
    h.link.assign(c->cap_link, c->cap_link + c->n_caps);
  }
  if (c->n_pairs) {
    h.pa.assign(c->pair_a, c->pair_a + c->n_pairs);
    h.pb.assign(c->pair_b, c->pair_b + c->n_pairs);
    for (int i = 0; i < c->n_pairs; ++i)
      if (h.pa[i] < 0 || h.pa[i] >= c->n_caps || h.pb[i] < 0 || h.pb[i] >= c->n_caps)
        return fail(MPPI_E_CONFIG, "self-collision pair indexes a missing capsule");
  }
  for (int i = 0; i < c->n_caps; ++i)
    if (h.link[i] < 0 || h.link[i] >= d) return fail(MPPI_E_CONFIG, "capsule link out of range");
  return MPPI_OK;
}

}  // namespace

// ================================================================== C ABI
// ---------------------------------------------------------------- episode
namespace {

constexpr int kEpisodeUnroll = 16;  // episode steps per captured graph

// instantaneous_costs (controller.py:262-269) of the plant state in ev_in:
// CostStack.evaluate with one step whose braking time is the whole horizon.
template <typename R>
int enqueue_instant_costs(mppi_plan* p, cudaStream_t st) {
  const int D = p->D;
  double horizon_time = 0.0;
  for (double x : p->dts) horizon_time += x;
  RolloutArgs<R> a;
  rollout_static<R>(p, 1, &horizon_time, a);
  a.N = 1;
  a.B = 1;
  a.mode = 2;  // positions (in0) and velocities (in1) given
  a.skip_on_status = 1;
  a.state = p->ev_in.p;
  a.goal = p->goal.p;
  a.in0 = p->ev_in.p;
  a.in1 = p->ev_in.p + D;
  a.step = reinterpret_cast<R*>(p->ev_stepbuf.p);
  a.mlp_x = p->learned() ? p->ev_x.p : nullptr;
  a.status = p->ev_status.p;
  a.bad = p->ev_status.p + 1;
  a.out_terms = p->ev_out.p + 1;
  CK(launch_rollout_any<R>(a, D, 1, st));
  if (p->learned()) CK(mlp_forward(p->mlp, p->ev_x.p, 1, p->ev_d.p, st));
  StatsArgs<R> s;
  stats_static<R>(p, 1, p->gamma, 1.0, s);
  s.N = 1;
  s.B = 1;
  s.ppb = 1;
  s.nblk = 1;
  s.totals_only = 1;
  s.raw_step = 1;
  s.step = reinterpret_cast<const R*>(p->ev_stepbuf.p);
  s.mlp_d = p->learned() ? p->ev_d.p : nullptr;
  s.totals = p->ev_out.p + 7;
  s.records = p->ev_records.p;
  s.counters = p->ev_counters.p;
  s.status = p->ev_status.p;
  s.bad = p->ev_status.p + 1;
  s.dump_step = p->ev_out.p;       // raw step cost (total_cost incl. the learned term)
  s.dump_terms = p->ev_out.p + 1;  // selfcoll row rewritten for the learned provider
  CK(launch_stats_any<R>(s, D, st));
  return MPPI_OK;
}

// `unroll` episode steps in one graph: pre -> {control step || cost
// evaluation} -> post, per step. Sections past the last step do nothing.
int capture_episode_graph(mppi_plan* p, const EpisodeArgs& ea, int unroll, cudaGraphExec_t* exec) {
  cudaStream_t st = p->stream;
  if (!p->stream2) {
    CK(cudaStreamCreateWithFlags(&p->stream2, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
  }
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  int rc = MPPI_OK;
  auto launched = [&](const char* what) {
    if (rc == MPPI_OK && cudaGetLastError() != cudaSuccess) rc = fail(MPPI_E_CUDA, std::string(what) + " launch");
  };
  for (int u = 0; u < unroll && rc == MPPI_OK; ++u) {
    episode_pre_kernel<<<1, 32, 0, st>>>(ea);
    launched("episode_pre_kernel");
    // fork: the plant-state cost evaluation runs beside the control step
    if (rc == MPPI_OK && (cudaEventRecord(p->ev_fork, st) != cudaSuccess ||
                          cudaStreamWaitEvent(p->stream2, p->ev_fork, 0) != cudaSuccess))
      rc = fail(MPPI_E_CUDA, "episode fork");
    if (rc == MPPI_OK)
      rc = p->precision == MPPI_FP64 ? enqueue_instant_costs<double>(p, p->stream2)
                                     : enqueue_instant_costs<float>(p, p->stream2);
    if (rc == MPPI_OK && cudaEventRecord(p->ev_join, p->stream2) != cudaSuccess)
      rc = fail(MPPI_E_CUDA, "episode join");
    p->cmd_dst = p->ep_cmd.p;
    p->info_dst = p->ep_info.p;
    if (rc == MPPI_OK) rc = enqueue_step_body(p, st, false, false);
    p->cmd_dst = nullptr;
    p->info_dst = nullptr;
    if (rc == MPPI_OK && cudaStreamWaitEvent(st, p->ev_join, 0) != cudaSuccess) rc = fail(MPPI_E_CUDA, "episode join");
    if (rc == MPPI_OK) {
      episode_post_kernel<<<1, 32, 0, st>>>(ea);
      launched("episode_post_kernel");
    }
  }
  cudaError_t e = cudaStreamEndCapture(st, &g);
  if (rc != MPPI_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return fail(MPPI_E_CUDA, std::string("episode capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(MPPI_E_CUDA, std::string("episode instantiate: ") + cudaGetErrorString(e));
  return MPPI_OK;
}

}  // namespace

extern "C" {

int32_t mppi_abi_version(void) { return MPPI_ABI_VERSION; }

const char* mppi_last_error(void) { return g_last_error.c_str(); }

// error hand-off from the other translation units (mppi_train.cu); not part of the public header
int mppi_internal_fail(int code, const char* msg) {
  g_last_error = msg;
  return code;
}

const char* mppi_build_info(void) {
#define MPPI_STR2(x) #x
#define MPPI_STR(x) MPPI_STR2(x)
  return "mppi_b200 sm_100a (fused rollout, CUDA graph step); nvcc " MPPI_STR(__CUDACC_VER_MAJOR__) "." MPPI_STR(
      __CUDACC_VER_MINOR__) "." MPPI_STR(__CUDACC_VER_BUILD__);
}

int mppi_device_count(int32_t* count) {
  int c = 0;
  CK(cudaGetDeviceCount(&c));
  *count = c;
  return MPPI_OK;
}

int mppi_plan_create(const mppi_chain_desc* chain, const mppi_cost_desc* costs,
                     const mppi_plan_desc* desc, mppi_plan** out) {
  if (!out || !desc || !costs) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  *out = nullptr;
  mppi_plan* p = new mppi_plan();
  int rc = [&]() -> int {
    CKR(copy_chain(chain, p->chain));
    const mppi_plan_desc& d = *desc;
    if (d.horizon < 2 || d.horizon > MPPI_MAX_HORIZON)
      return fail(MPPI_E_CONFIG, "horizon must lie in [2, " + std::to_string(MPPI_MAX_HORIZON) + "]");
    if (d.particles < 1) return fail(MPPI_E_CONFIG, "particles must be positive");
    if (d.instances < 1) return fail(MPPI_E_CONFIG, "instances must be positive");
    if (!d.dts) return fail(MPPI_E_BAD_ARGUMENT, "dts is null");
    p->device = d.device;
    CKR(set_device(p));
    p->D = p->chain.dof;
    p->H = d.horizon;
    p->N = d.particles;
    p->B = d.instances;
    p->iters = std::max(1, d.iterations);
    p->null_count = d.null_count;
    p->policy_mode = d.policy_mode;
    p->precision = d.precision;
    p->generator = d.generator;
    p->smoothing = d.smoothing;
    p->degree = d.spline_degree;
    p->Kn = d.knots > 0 ? d.knots : d.horizon;
    p->offset = d.particle_offset;
    p->Ntot = d.particles_total > 0 ? d.particles_total : d.particles;
    p->seed = d.seed;
    for (int i = 0; i < 3; ++i) p->comb[i] = d.comb[i];
    p->gamma = d.gamma;
    p->tw = d.terminal_weight;
    p->beta = d.beta;
    p->alpha_mu = d.alpha_mu;
    p->alpha_sigma = d.alpha_sigma;
    p->sigma0_sq = d.sigma0_sq;
    p->smin = d.sigma_sq_min;
    p->smax = d.sigma_sq_max;
    p->tail = d.default_tail;
    p->dts.assign(d.dts, d.dts + d.horizon);
    p->costs = *costs;
    p->dump = d.dump;
    if (p->offset < 0 || p->offset + p->N > p->Ntot)
      return fail(MPPI_E_CONFIG, "particle shard out of range");
    CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&p->ev0));
    CK(cudaEventCreate(&p->ev1));
    p->stage_ev.assign(4 * p->iters + 1, nullptr);
    for (auto& e : p->stage_ev) CK(cudaEventCreate(&e));
    const int B = p->B, D = p->D, H = p->H, N = p->N;
    const size_t HD = (size_t)H * D;
    choose_blocks(N, B, p->ppb, p->nblk);
    const size_t rsz = p->precision == MPPI_FP64 ? sizeof(double) : sizeof(float);
    const int reclen = kRecHead + 2 * (int)HD;
    CKR(p->eps.alloc((size_t)N * HD));
    CK(cudaMemset(p->eps.p, 0, sizeof(double) * N * HD));
    CKR(p->means.alloc(B * HD));
    CKR(p->var.alloc(B * HD));
    CKR(p->sd.alloc(B * HD));
    CKR(p->prev_means.alloc(B * HD));
    CKR(p->prev_sd.alloc(B * HD));
    CKR(p->goal.alloc((size_t)B * 16));
    CKR(p->state.alloc((size_t)B * 2 * D + 1));  // + step counter slot
    CKR(p->stepbuf.alloc((size_t)B * N * H * rsz));
    CKR(p->totals.alloc((size_t)B * N));
    CKR(p->records.alloc((size_t)B * stats_rec_stride(p->nblk) * reclen));
    CKR(p->out_record.alloc(reclen));
    CKR(p->cmd.alloc((size_t)B * D));
    CKR(p->counters.alloc((size_t)B * kStatsCounterStride));
    CK(cudaMemset(p->counters.p, 0, sizeof(unsigned) * B * kStatsCounterStride));
    CKR(p->status.alloc(B));
    CKR(p->bad.alloc(B));
    CK(cudaMemset(p->status.p, 0, sizeof(int) * B));
    CK(cudaMemset(p->bad.p, 0x7f, sizeof(int) * B));
    CKR(p->info.alloc(B));
    if (getenv("MPPI_DEBUG_TIMERS")) {
      // stats phases (16 per stats block) + fused rollout/MLP phases (8 per CTA, <= 256 CTAs)
      CKR(p->dbg.alloc((size_t)16 * p->nblk + 2 * 16 * 256));
      CK(cudaMemset(p->dbg.p, 0, sizeof(unsigned long long) * (16 * p->nblk + 2 * 16 * 256)));
#ifdef MPPI_DEBUG_TIMERS
      unsigned long long* mdbg = p->dbg.p + 16 * p->nblk + 16 * 256;
      CK(cudaMemcpyToSymbol(mlp_dbg, &mdbg, sizeof(mdbg)));
#endif
    }
    if (p->dump) {
      CKR(p->d_pos.alloc((size_t)N * HD));
      CKR(p->d_vel.alloc((size_t)N * HD));
      CKR(p->d_acc.alloc((size_t)N * HD));
      CKR(p->d_terms.alloc((size_t)6 * N * H));
      CK(cudaMemset(p->d_terms.p, 0, sizeof(double) * 6 * N * H));
      CKR(p->d_step.alloc((size_t)N * H));
      CKR(p->d_w.alloc((size_t)N));
    }
    if (p->learned()) {
      const size_t rows = (size_t)B * N * H;
      CKR(p->mlp_x.alloc(mlp_padded_rows(rows) * 16));
      CK(cudaMemset(p->mlp_x.p, 0, sizeof(float) * mlp_padded_rows(rows) * 16));
      CKR(p->mlp_d.alloc(mlp_padded_rows(rows)));
    }
    // policy: zero mean, sigma0^2 variance (make_policy, policy.py:88-95)
    std::vector<double> z(B * HD, 0.0), v(B * HD, p->sigma0_sq), s(B * HD, std::sqrt(p->sigma0_sq));
    CK(cudaMemcpy(p->means.p, z.data(), sizeof(double) * B * HD, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p->var.p, v.data(), sizeof(double) * B * HD, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p->sd.p, s.data(), sizeof(double) * B * HD, cudaMemcpyHostToDevice));
    // identity goal at the origin, position_only
    p->goal_host.assign((size_t)B * 16, 0.0);
    for (int b = 0; b < B; ++b) {
      p->goal_host[b * 16 + 0] = p->goal_host[b * 16 + 4] = p->goal_host[b * 16 + 8] = 1.0;
    }
    CK(cudaMemcpy(p->goal.p, p->goal_host.data(), sizeof(double) * B * 16, cudaMemcpyHostToDevice));
    CK(cudaHostAlloc(&p->h_state, sizeof(double) * (B * 2 * D + 1), cudaHostAllocMapped));
    CK(cudaHostAlloc(&p->h_cmd, sizeof(double) * B * D, cudaHostAllocMapped));
    CK(cudaHostAlloc(&p->h_info, sizeof(mppi_step_info) * B, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&p->m_state, p->h_state, 0));
    CK(cudaHostGetDevicePointer((void**)&p->m_cmd, p->h_cmd, 0));
    CK(cudaHostGetDevicePointer((void**)&p->m_info, p->h_info, 0));
    memset(p->h_state, 0, sizeof(double) * B * 2 * D);
    if (p->generator == MPPI_GEN_PSEUDORANDOM) {
      CKR(p->z.alloc((size_t)N * p->Kn * D));
      if (p->smoothing == MPPI_SMOOTH_BSPLINE) {
        CKR(p->basis.alloc((size_t)H * p->Kn));
        bspline_basis_kernel<<<1, 64, 0, p->stream>>>(H, p->Kn, p->degree, p->basis.p);
        CK(cudaGetLastError());
      }
    }
    CK(cudaStreamSynchronize(p->stream));
    return MPPI_OK;
  }();
  if (rc != MPPI_OK) {
    mppi_plan_destroy(p);
    return rc;
  }
  *out = p;
  return MPPI_OK;
}

int mppi_plan_destroy(mppi_plan* p) {
  if (!p) return MPPI_OK;
  cudaSetDevice(p->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  invalidate_graph(p);
  DevBuf<double>* dbl[] = {&p->sph_d, &p->box_d, &p->eps, &p->z, &p->basis, &p->colmean, &p->means,
                           &p->var, &p->sd, &p->prev_means, &p->prev_sd, &p->goal, &p->state,
                           &p->totals, &p->records, &p->out_record, &p->cmd, &p->counters_pad,
                           &p->e_in0, &p->e_in1, &p->e_pos, &p->e_vel, &p->e_acc, &p->e_terms,
                           &p->e_step, &p->e_tot, &p->e_state, &p->e_dts, &p->e_records,
                           &p->d_pos, &p->d_vel, &p->d_acc, &p->d_terms, &p->d_step, &p->d_w,
                           &p->ep_state, &p->ep_log, &p->ep_script, &p->ep_noise, &p->ep_cmd,
                           &p->ev_in, &p->ev_out, &p->ev_records};
  for (auto* b : dbl) b->release();
  p->sph_f.release();
  p->box_f.release();
  p->clearance.release();
  p->mlp_x.release();
  p->mlp_d.release();
  p->e_x.release();
  p->e_d.release();
  p->stepbuf.release();
  p->e_stepbuf.release();
  p->counters.release();
  p->dbg.release();
  p->e_counters.release();
  p->status.release();
  p->bad.release();
  p->e_status.release();
  p->e_w.release();
  p->info.release();
  p->ep_ilog.release();
  p->ep_info.release();
  p->ev_stepbuf.release();
  p->ev_x.release();
  p->ev_d.release();
  p->ev_status.release();
  p->ev_counters.release();
  mlp_release(p->mlp);
  if (p->h_state) cudaFreeHost(p->h_state);
  if (p->h_cmd) cudaFreeHost(p->h_cmd);
  if (p->h_info) cudaFreeHost(p->h_info);
  if (p->ev0) cudaEventDestroy(p->ev0);
  if (p->ev1) cudaEventDestroy(p->ev1);
  for (auto e : p->stage_ev) cudaEventDestroy(e);
  if (p->stream) cudaStreamDestroy(p->stream);
  p->peer_recv_buf.release();
  p->peer_flag_buf.release();
  p->peer_recv_tab.release();
  p->peer_flag_tab.release();
  if (p->stream2) cudaStreamDestroy(p->stream2);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  delete p;
  return MPPI_OK;
}

int mppi_init_noise(mppi_plan* p, const double* basis_host) {
  if (!p) return fail(MPPI_E_BAD_ARGUMENT, "null plan");
  CKR(set_device(p));
  if (p->generator != MPPI_GEN_HALTON) return MPPI_OK;
  if (p->D > 40) return fail(MPPI_E_CONFIG, "halton supports at most 40 dims");
  const long long rows = p->Ntot;
  const int K = p->Kn, H = p->H, D = p->D;
  DevBuf<double> zt, full, bas;
  CKR(zt.alloc((size_t)rows * K * D));
  CKR(full.alloc((size_t)rows * H * D));
  const double* bptr = nullptr;
  if (p->smoothing == MPPI_SMOOTH_BSPLINE) {
    CKR(bas.alloc((size_t)H * K));
    if (basis_host) {
      CK(cudaMemcpyAsync(bas.p, basis_host, sizeof(double) * H * K, cudaMemcpyHostToDevice, p->stream));
    } else {
      bspline_basis_kernel<<<1, 64, 0, p->stream>>>(H, K, p->degree, bas.p);
    }
    bptr = bas.p;
  }
  if (p->smoothing != MPPI_SMOOTH_BSPLINE && K != H) {
    zt.release();
    full.release();
    return fail(MPPI_E_BAD_ARGUMENT, "smoothing expects K == H");
  }
  DevBuf<int> err;
  CKR(err.alloc(1));
  CK(cudaMemsetAsync(err.p, 0, sizeof(int), p->stream));
  knots_kernel<<<grid_for(rows * K * D, 256), 256, 0, p->stream>>>(zt.p, rows, K, D, MPPI_GEN_HALTON, 0, 0, err.p);
  smooth_kernel<<<grid_for(rows * H * D, 256), 256, 0, p->stream>>>(zt.p, full.p, rows, K, H, D, p->smoothing,
                                                                    bptr, p->comb[0], p->comb[1], p->comb[2]);
  CKR(p->colmean.alloc((size_t)H * D));
  column_mean_kernel<<<H * D, 256, 0, p->stream>>>(full.p, rows, H * D, p->colmean.p);
  center_slice_kernel<<<grid_for((long long)p->N * H * D, 256), 256, 0, p->stream>>>(
      full.p, p->colmean.p, p->eps.p, p->offset, p->N, H * D);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(p->stream));
  zt.release();
  full.release();
  bas.release();
  err.release();
  return MPPI_OK;
}

int mppi_set_noise(mppi_plan* p, const double* eps) {
  if (!p || !eps) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  CKR(set_device(p));
  CK(cudaMemcpyAsync(p->eps.p, eps, sizeof(double) * p->N * p->H * p->D, cudaMemcpyHostToDevice, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return MPPI_OK;
}

int mppi_get_step_inputs(mppi_plan* p, int32_t inst, double* theta, double* theta_dot, double* means,
                         double* stddev) {
  if (!p || !theta || !theta_dot || !means || !stddev) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (inst < 0 || inst >= p->B) return fail(MPPI_E_BAD_ARGUMENT, "instance out of range");
  if (p->step_counter == 0) return fail(MPPI_E_CONFIG, "no step has run on this plan");
  CKR(set_device(p));
  const int D = p->D, HD = p->H * p->D;
  CK(cudaStreamSynchronize(p->stream));
  memcpy(theta, p->h_state + (size_t)inst * 2 * D, sizeof(double) * D);
  memcpy(theta_dot, p->h_state + (size_t)inst * 2 * D + D, sizeof(double) * D);
  CK(cudaMemcpyAsync(means, p->prev_means.p + (size_t)inst * HD, sizeof(double) * HD, cudaMemcpyDeviceToHost,
                     p->stream));
  CK(cudaMemcpyAsync(stddev, p->prev_sd.p + (size_t)inst * HD, sizeof(double) * HD, cudaMemcpyDeviceToHost,
                     p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return MPPI_OK;
}

int mppi_get_noise(mppi_plan* p, double* eps) {
  if (!p || !eps) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  CKR(set_device(p));
  CK(cudaMemcpyAsync(eps, p->eps.p, sizeof(double) * p->N * p->H * p->D, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return MPPI_OK;
}

int mppi_set_goal(mppi_plan* p, int32_t inst, const double* R, const double* t, int32_t mode) {
  if (!p || !R || !t) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (inst < -1 || inst >= p->B) return fail(MPPI_E_BAD_ARGUMENT, "instance out of range");
  CKR(set_device(p));
  const int b0 = inst < 0 ? 0 : inst, b1 = inst < 0 ? p->B : inst + 1;
  for (int b = b0; b < b1; ++b) {
    double* g = &p->goal_host[(size_t)b * 16];
    for (int i = 0; i < 9; ++i) g[i] = R[i];
    for (int i = 0; i < 3; ++i) g[9 + i] = t[i];
    g[12] = (double)mode;
  }
  p->goal_dirty = true;  // uploaded with the next step (flush_goal / the step graph's parameters)
  return MPPI_OK;
}

int mppi_set_goals(mppi_plan* p, int32_t first, int32_t count, const double* R, const double* t,
                   const int32_t* modes) {
  if (!p || !R || !t || !modes) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (first < 0 || count < 1 || first + count > p->B) return fail(MPPI_E_BAD_ARGUMENT, "instance range");
  CKR(set_device(p));
  for (int i = 0; i < count; ++i) {
    double* g = &p->goal_host[(size_t)(first + i) * 16];
    for (int k = 0; k < 9; ++k) g[k] = R[(size_t)i * 9 + k];
    for (int k = 0; k < 3; ++k) g[9 + k] = t[(size_t)i * 3 + k];
    g[12] = (double)modes[i];
  }
  p->goal_dirty = true;
  return MPPI_OK;
}

int mppi_set_world(mppi_plan* p, const double* spheres, int32_t ns, const double* boxes, int32_t nb) {
  if (!p || ns < 0 || nb < 0) return fail(MPPI_E_BAD_ARGUMENT, "bad world arguments");
  CKR(set_device(p));
  CK(cudaStreamSynchronize(p->stream));
  p->ns = ns;
  p->nb = nb;
  std::vector<float> sf(std::max(1, 4 * ns)), bf(std::max(1, 6 * nb));
  for (int i = 0; i < 4 * ns; ++i) sf[i] = (float)spheres[i];
  for (int i = 0; i < 6 * nb; ++i) bf[i] = (float)boxes[i];
  CKR(p->sph_d.alloc(std::max(1, 4 * ns)));
  CKR(p->box_d.alloc(std::max(1, 6 * nb)));
  CKR(p->sph_f.alloc(std::max(1, 4 * ns)));
  CKR(p->box_f.alloc(std::max(1, 6 * nb)));
  if (ns) CK(cudaMemcpy(p->sph_d.p, spheres, sizeof(double) * 4 * ns, cudaMemcpyHostToDevice));
  if (nb) CK(cudaMemcpy(p->box_d.p, boxes, sizeof(double) * 6 * nb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(p->sph_f.p, sf.data(), sizeof(float) * sf.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(p->box_f.p, bf.data(), sizeof(float) * bf.size(), cudaMemcpyHostToDevice));
  p->clearance.release();
  p->gx = p->gy = p->gz = 0;
  invalidate_graph(p);
  return MPPI_OK;
}

int mppi_set_voxel_world(mppi_plan* p, const uint8_t* occ, int32_t nx, int32_t ny, int32_t nz,
                         const double* origin, double voxel, const double* spheres, int32_t ns) {
  if (!p || !occ || nx < 1 || ny < 1 || nz < 1 || !(voxel > 0.0))
    return fail(MPPI_E_BAD_ARGUMENT, "bad voxel world arguments");
  // Greedy box decomposition of the occupied set on the host (init-time
  // geometry preprocessing): grow x-runs, then y, then z. The union of the
  // boxes is exactly the occupied voxel set, so the narrow phase keeps the
  // reference's box semantics (simworld.py:30-49, jit.py:325-331).
  std::vector<uint8_t> left(occ, occ + (size_t)nx * ny * nz);
  auto at = [&](int i, int j, int k) -> uint8_t& { return left[((size_t)i * ny + j) * nz + k]; };
  std::vector<double> boxes;
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j)
      for (int k = 0; k < nz; ++k) {
        if (!at(i, j, k)) continue;
        int k1 = k;
        while (k1 + 1 < nz && at(i, j, k1 + 1)) ++k1;
        int j1 = j;
        for (;;) {
          if (j1 + 1 >= ny) break;
          bool ok = true;
          for (int kk = k; kk <= k1 && ok; ++kk) ok = at(i, j1 + 1, kk);
          if (!ok) break;
          ++j1;
        }
        int i1 = i;
        for (;;) {
          if (i1 + 1 >= nx) break;
          bool ok = true;
          for (int jj = j; jj <= j1 && ok; ++jj)
            for (int kk = k; kk <= k1 && ok; ++kk) ok = at(i1 + 1, jj, kk);
          if (!ok) break;
          ++i1;
        }
        for (int ii = i; ii <= i1; ++ii)
          for (int jj = j; jj <= j1; ++jj)
            for (int kk = k; kk <= k1; ++kk) at(ii, jj, kk) = 0;
        boxes.push_back(origin[0] + i * voxel);
        boxes.push_back(origin[1] + j * voxel);
        boxes.push_back(origin[2] + k * voxel);
        boxes.push_back(origin[0] + (i1 + 1) * voxel);
        boxes.push_back(origin[1] + (j1 + 1) * voxel);
        boxes.push_back(origin[2] + (k1 + 1) * voxel);
      }
  const int nb = (int)(boxes.size() / 6);
  CKR(mppi_set_world(p, spheres, ns, boxes.data(), nb));
  p->gx = nx;
  p->gy = ny;
  p->gz = nz;
  for (int i = 0; i < 3; ++i) p->gorigin[i] = origin[i];
  p->gvoxel = voxel;
  CKR(p->clearance.alloc((size_t)nx * ny * nz));
  clearance_kernel<<<grid_for((long long)nx * ny * nz, 256, 1 << 20), 256, 0, p->stream>>>(
      p->box_d.p, nb, nx, ny, nz, origin[0], origin[1], origin[2], voxel, p->clearance.p);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(p->stream));
  invalidate_graph(p);
  return MPPI_OK;
}

int mppi_set_mlp(mppi_plan* p, int32_t in_dim, const double* W0, const double* b0, const double* W1,
                 const double* b1, const double* W2, const double* b2, const double* W3,
                 const double* b3) {
  if (!p) return fail(MPPI_E_BAD_ARGUMENT, "null plan");
  if (in_dim != 2 * p->D || in_dim > MPPI_MLP_IN_MAX)
    return fail(MPPI_E_CONFIG, "surrogate input dim must be 2*dof <= 16");
  CKR(set_device(p));
  CK(mlp_upload(p->mlp, in_dim, W0, b0, W1, b1, W2, b2, W3, b3, p->stream));
  p->mlp_ready = true;
  invalidate_graph(p);
  return MPPI_OK;
}

int mppi_set_policy(mppi_plan* p, int32_t inst, const double* means, const double* variances) {
  if (!p || !means || !variances) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (inst < 0 || inst >= p->B) return fail(MPPI_E_BAD_ARGUMENT, "instance out of range");
  CKR(set_device(p));
  const size_t HD = (size_t)p->H * p->D;
  std::vector<double> s(HD);
  for (size_t i = 0; i < HD; ++i) s[i] = std::sqrt(variances[i]);
  CK(cudaMemcpyAsync(p->means.p + inst * HD, means, sizeof(double) * HD, cudaMemcpyHostToDevice, p->stream));
  CK(cudaMemcpyAsync(p->var.p + inst * HD, variances, sizeof(double) * HD, cudaMemcpyHostToDevice, p->stream));
  CK(cudaMemcpyAsync(p->sd.p + inst * HD, s.data(), sizeof(double) * HD, cudaMemcpyHostToDevice, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return MPPI_OK;
}

int mppi_get_policy(mppi_plan* p, int32_t inst, double* means, double* variances) {
  if (!p) return fail(MPPI_E_BAD_ARGUMENT, "null plan");
  if (inst < 0 || inst >= p->B) return fail(MPPI_E_BAD_ARGUMENT, "instance out of range");
  CKR(set_device(p));
  const size_t HD = (size_t)p->H * p->D;
  if (means)
    CK(cudaMemcpyAsync(means, p->means.p + inst * HD, sizeof(double) * HD, cudaMemcpyDeviceToHost, p->stream));
  if (variances)
    CK(cudaMemcpyAsync(variances, p->var.p + inst * HD, sizeof(double) * HD, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return MPPI_OK;
}

int mppi_step(mppi_plan* p, const double* theta, const double* theta_dot, double* command_out,
              mppi_step_info* info) {
  if (!p || !theta || !theta_dot || !command_out) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  CKR(set_device(p));
  CKR(ensure_graph(p));
  const int B = p->B, D = p->D;
  for (int b = 0; b < B; ++b) {
    memcpy(p->h_state + (size_t)b * 2 * D, theta + (size_t)b * D, sizeof(double) * D);
    memcpy(p->h_state + (size_t)b * 2 * D + D, theta_dot + (size_t)b * D, sizeof(double) * D);
  }
  {
    const unsigned long long ctr = p->step_counter++;
    memcpy(p->h_state + (size_t)B * 2 * D, &ctr, sizeof(ctr));
  }
  // device timing of the replay only when profiling: on the latency path every
  // extra runtime call is host time between the state and the command
  const bool prof = p->profile_level >= 2;
  if (prof) CKR(ensure_graph(p, true));
#ifdef MPPI_DEBUG_TIMERS
  using clk = std::chrono::steady_clock;
  const auto h0 = clk::now();
#endif
  auto& inl_nodes = prof ? p->inl_prof : p->inl;
  if (inl_nodes.empty()) CKR(flush_goal(p));  // the graph reads the device goals
  for (auto& n : inl_nodes) {
    memcpy(n.args.data() + n.st_off, p->h_state, sizeof(double) * 2 * D);
    memcpy(n.args.data() + n.g_off, p->goal_host.data(), sizeof(double) * 16);
    CK(cudaGraphExecKernelNodeSetParams(prof ? p->graph_prof : p->graph, n.node, &n.kp));
  }
#ifdef MPPI_DEBUG_TIMERS
  const auto h1 = clk::now();
#endif
  if (p->profile_level) CK(cudaEventRecord(p->ev0, p->stream));
  CK(cudaGraphLaunch(prof ? p->graph_prof : p->graph, p->stream));
  if (p->profile_level) CK(cudaEventRecord(p->ev1, p->stream));
#ifdef MPPI_DEBUG_TIMERS
  const auto h2 = clk::now();
#endif
  CK(cudaStreamSynchronize(p->stream));
#ifdef MPPI_DEBUG_TIMERS
  if (getenv("MPPI_HOST_TIMING")) {  // host-side split of one step: set params | launch | wait
    static double acc[3] = {0, 0, 0};
    static long cnt = 0;
    const auto h3 = clk::now();
    acc[0] += std::chrono::duration<double, std::micro>(h1 - h0).count();
    acc[1] += std::chrono::duration<double, std::micro>(h2 - h1).count();
    acc[2] += std::chrono::duration<double, std::micro>(h3 - h2).count();
    if (++cnt % 1000 == 0) {
      fprintf(stderr, "host us/step: set params %.2f  graph launch %.2f  wait %.2f\n", acc[0] / cnt, acc[1] / cnt,
              acc[2] / cnt);
    }
  }
#endif
  float ms = 0.f;
  if (p->profile_level) CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
  memcpy(command_out, p->h_cmd, sizeof(double) * B * D);
  if (p->dbg.p) {  // debug: stats-kernel phase timeline of instance 0, relative to block 0 start
    std::vector<unsigned long long> t((size_t)16 * p->nblk + 2 * 16 * 256);
    CK(cudaMemcpy(t.data(), p->dbg.p, sizeof(unsigned long long) * t.size(), cudaMemcpyDeviceToHost));
    const unsigned long long* f = t.data() + 16 * p->nblk;
    unsigned long long t0 = t[0];
    if (f[0]) {  // fused rollout + MLP: phase stamps relative to the earliest CTA start
      for (int k = 0; k < 256; ++k)
        if (f[16 * k] && f[16 * k] < t0) t0 = f[16 * k];
      double mx[12] = {0};
      for (int k = 0; k < 256; ++k)
        for (int j = 0; j < 12; ++j)
          if (f[16 * k + j]) mx[j] = std::max(mx[j], (double)(long long)(f[16 * k + j] - t0) * 1e-3);
      for (int k : {0, 1, 2, 3, 64, 124}) {
        fprintf(stderr, "fused blk %3d:", k);
        for (int j = 0; j < 12; ++j)
          fprintf(stderr, " %7.2f", f[16 * k + j] ? (double)(long long)(f[16 * k + j] - t0) * 1e-3 : -1.0);
        fprintf(stderr, "\n");
      }
      fprintf(stderr, "fused max    :");
      for (int j = 0; j < 12; ++j) fprintf(stderr, " %7.2f", mx[j]);
      fprintf(stderr, "\n");
    }
    {  // MLP phase stamps: min / max over CTAs, relative to the same origin
      const unsigned long long* g = t.data() + 16 * p->nblk + 16 * 256;
      double lo[16], hi[16];
      for (int j = 0; j < 16; ++j) lo[j] = 1e30, hi[j] = -1e30;
      for (int k = 0; k < 255; ++k)
        for (int j = 0; j < 16; ++j)
          if (g[16 * k + j]) {
            const double v = (double)(long long)(g[16 * k + j] - t0) * 1e-3;
            lo[j] = std::min(lo[j], v);
            hi[j] = std::max(hi[j], v);
          }
      const unsigned long long re = t[16 * p->nblk + 16 * 255 + 15], me = g[16 * 255 + 15];
      const unsigned long long* ec = t.data() + 16 * p->nblk + 16 * 253;
      if (ec[15] || ec[0] || ec[1]) {
        fprintf(stderr, "world exact tests (cumulative) per capsule:");
        for (int c = 0; c < 8; ++c) fprintf(stderr, " %llu", ec[c]);
        fprintf(stderr, " | ternary searches %llu\n", ec[15]);
      }
      fprintf(stderr, "rollout last warp end %.2f, mlp last CTA end %.2f\n",
              re ? (double)(long long)(re - t0) * 1e-3 : -1.0, me ? (double)(long long)(me - t0) * 1e-3 : -1.0);
      fprintf(stderr, "mlp min     :");
      for (int j = 0; j < 13; ++j) fprintf(stderr, " %7.2f", lo[j] < 1e29 ? lo[j] : -1.0);
      fprintf(stderr, "\nmlp max     :");
      for (int j = 0; j < 13; ++j) fprintf(stderr, " %7.2f", hi[j] > -1e29 ? hi[j] : -1.0);
      fprintf(stderr, "\n");
    }
    for (int k = 0; k < p->nblk; ++k) {
      fprintf(stderr, "stats blk %2d:", k);
      for (int j = 0; j < 14; ++j)
        fprintf(stderr, " %8.2f", t[k * 16 + j] ? (double)(long long)(t[k * 16 + j] - t0) * 1e-3 : -1.0);
      fprintf(stderr, "\n");
    }
  }
  if (info) {
    memcpy(info, p->h_info, sizeof(mppi_step_info) * B);
    double stg[4] = {0, 0, 0, 0};
    for (int it = 0; it < (prof ? p->iters : 0); ++it)
      for (int sg = 0; sg < 4; ++sg) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, p->stage_ev[4 * it + sg], p->stage_ev[4 * it + sg + 1]));
        stg[sg] += t;
      }
    for (int b = 0; b < B; ++b) {
      info[b].device_ms = ms;
      info[b].sample_ms = stg[0];
      info[b].rollout_ms = stg[1];
      info[b].mlp_ms = stg[2];
      info[b].update_ms = stg[3];
    }
  }
  return MPPI_OK;
}

int mppi_evaluate(mppi_plan* p, int32_t mode, int32_t n, int32_t H, const double* dts, double gamma,
                  double tw, const double* theta0, const double* theta_dot0, const double* in0,
                  const double* in1, mppi_eval_out* out) {
  if (!p || !dts || !in0 || !out) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (mode != 0 && mode != 1) return fail(MPPI_E_BAD_ARGUMENT, "mode must be 0 or 1");
  if (mode == 1 && !in1) return fail(MPPI_E_BAD_ARGUMENT, "velocities missing");
  if (mode == 0 && (!theta0 || !theta_dot0)) return fail(MPPI_E_BAD_ARGUMENT, "initial state missing");
  if (H < 1 || H > MPPI_MAX_HORIZON) return fail(MPPI_E_CONFIG, "horizon out of range");
  if (n < 1) return fail(MPPI_E_BAD_ARGUMENT, "empty batch");
  if (p->learned() && !p->mlp_ready) return fail(MPPI_E_CONFIG, "learned provider without weights");
  CKR(set_device(p));
  CKR(flush_goal(p));
  cudaStream_t st = p->stream;
  const int D = p->D;
  const size_t nhd = (size_t)n * H * D, nh = (size_t)n * H;
  CKR(p->e_in0.alloc(nhd));
  CKR(p->e_in1.alloc(nhd));
  CKR(p->e_pos.alloc(nhd));
  CKR(p->e_vel.alloc(nhd));
  CKR(p->e_acc.alloc(nhd));
  CKR(p->e_terms.alloc(6 * nh));
  CKR(p->e_step.alloc(nh));
  CKR(p->e_tot.alloc(n));
  CKR(p->e_state.alloc(2 * D));
  CKR(p->e_stepbuf.alloc(nh * sizeof(double)));
  CKR(p->e_status.alloc(2));
  int ppb, nblk;
  choose_blocks(n, 1, ppb, nblk);
  CKR(p->e_records.alloc((size_t)nblk * (kRecHead + 2 * H * D)));
  CKR(p->e_counters.alloc(1));
  if (p->learned()) {
    CKR(p->e_x.alloc(mlp_padded_rows(nh) * 16));
    CKR(p->e_d.alloc(mlp_padded_rows(nh)));
    CK(cudaMemsetAsync(p->e_x.p, 0, sizeof(float) * mlp_padded_rows(nh) * 16, st));
  }
  if (in0 != p->e_in0.p)  // (mppi_replay_bundle builds the controls in e_in0 itself)
    CK(cudaMemcpyAsync(p->e_in0.p, in0, sizeof(double) * nhd, cudaMemcpyHostToDevice, st));
  if (mode == 1) CK(cudaMemcpyAsync(p->e_in1.p, in1, sizeof(double) * nhd, cudaMemcpyHostToDevice, st));
  std::vector<double> s0(2 * D, 0.0);
  if (mode == 0) {
    memcpy(s0.data(), theta0, sizeof(double) * D);
    memcpy(s0.data() + D, theta_dot0, sizeof(double) * D);
  }
  CK(cudaMemcpyAsync(p->e_state.p, s0.data(), sizeof(double) * 2 * D, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(p->e_status.p, 0, sizeof(int), st));
  CK(cudaMemsetAsync(p->e_status.p + 1, 0x7f, sizeof(int), st));
  CK(cudaMemsetAsync(p->e_counters.p, 0, sizeof(unsigned), st));
  auto run = [&](auto tag) -> int {
    using R = decltype(tag);
    RolloutArgs<R> a;
    rollout_static<R>(p, H, dts, a);
    a.N = n;
    a.B = 1;
    a.mode = mode == 0 ? 1 : 2;
    a.state = p->e_state.p;
    a.goal = p->goal.p;
    a.in0 = p->e_in0.p;
    a.in1 = p->e_in1.p;
    a.step = reinterpret_cast<R*>(p->e_stepbuf.p);
    a.mlp_x = p->learned() ? p->e_x.p : nullptr;
    a.status = p->e_status.p;
    a.bad = p->e_status.p + 1;
    a.out_pos = p->e_pos.p;
    a.out_vel = p->e_vel.p;
    a.out_acc = p->e_acc.p;
    a.out_terms = p->e_terms.p;
    CK(launch_rollout_any<R>(a, D, n, st));
    if (p->learned()) CK(mlp_forward(p->mlp, p->e_x.p, (long long)nh, p->e_d.p, st));
    StatsArgs<R> s;
    stats_static<R>(p, H, gamma, tw, s);
    s.N = n;
    s.B = 1;
    s.ppb = ppb;
    s.nblk = nblk;
    s.totals_only = 1;
    s.raw_step = mode == 1;
    s.step = reinterpret_cast<const R*>(p->e_stepbuf.p);
    s.mlp_d = p->learned() ? p->e_d.p : nullptr;
    s.totals = p->e_tot.p;
    s.records = p->e_records.p;
    s.counters = p->e_counters.p;
    s.status = p->e_status.p + 0;
    s.bad = p->e_status.p + 1;
    s.dump_step = p->e_step.p;
    s.dump_terms = p->e_terms.p;
    // phase A ignores the status word when totals_only; use a zero status
    CK(launch_stats_any<R>(s, D, st));
    return MPPI_OK;
  };
  if (p->precision == MPPI_FP64)
    CKR(run(double{}));
  else
    CKR(run(float{}));
  int hst[2];
  CK(cudaMemcpyAsync(hst, p->e_status.p, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
  std::vector<double> tot(n);
  CK(cudaMemcpyAsync(tot.data(), p->e_tot.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  if (out->positions) CK(cudaMemcpyAsync(out->positions, p->e_pos.p, sizeof(double) * nhd, cudaMemcpyDeviceToHost, st));
  if (out->velocities) CK(cudaMemcpyAsync(out->velocities, p->e_vel.p, sizeof(double) * nhd, cudaMemcpyDeviceToHost, st));
  if (out->accelerations) CK(cudaMemcpyAsync(out->accelerations, p->e_acc.p, sizeof(double) * nhd, cudaMemcpyDeviceToHost, st));
  if (out->step_costs) CK(cudaMemcpyAsync(out->step_costs, p->e_step.p, sizeof(double) * nh, cudaMemcpyDeviceToHost, st));
  if (out->terms) CK(cudaMemcpyAsync(out->terms, p->e_terms.p, sizeof(double) * 6 * nh, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (out->totals) memcpy(out->totals, tot.data(), sizeof(double) * n);
  out->bad_particle = hst[1] >= 0x7f000000 ? -1 : hst[1];
  int q = 0;
  for (int i = 0; i < n; ++i) q += std::isfinite(tot[i]) ? 0 : 1;
  out->quarantined = q;
  if (hst[0] == MPPI_E_NONFINITE_CONTROL)
    return fail(MPPI_E_NONFINITE_CONTROL, "non-finite control in particle " + std::to_string(out->bad_particle));
  return MPPI_OK;
}

int mppi_replay_bundle(mppi_plan* p, mppi_eval_out* out, double* weights) {
  if (!p || !out) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (p->step_counter == 0) return fail(MPPI_E_CONFIG, "no step has run on this plan");
  CKR(set_device(p));
  cudaStream_t st = p->stream;
  const int n = p->N, H = p->H, D = p->D;
  const size_t nhd = (size_t)n * H * D;
  CK(cudaStreamSynchronize(st));
  // u = mu + sd * eps of instance 0's last iteration (sampling.py:268-290),
  // straight into the evaluation's control buffer
  CKR(p->e_in0.alloc(nhd));
  CKR(p->e_status.alloc(2));
  CK(cudaMemsetAsync(p->e_status.p, 0, sizeof(int), st));
  build_controls_kernel<<<grid_for((long long)nhd, 256), 256, 0, st>>>(p->eps.p, p->prev_means.p, p->prev_sd.p, n, H,
                                                                        D, p->null_count, p->e_in0.p,
                                                                        p->e_status.p);
  CK(cudaGetLastError());
  std::vector<double> th(p->h_state, p->h_state + D), thd(p->h_state + D, p->h_state + 2 * D);
  double* totals = out->totals;
  std::vector<double> tot_tmp;
  if (weights && !totals) {
    tot_tmp.resize(n);
    out->totals = tot_tmp.data();
  }
  const int rc = mppi_evaluate(p, 0, n, H, p->dts.data(), p->gamma, p->tw, th.data(), thd.data(), p->e_in0.p,
                               nullptr, out);
  out->totals = totals;
  if (rc != MPPI_OK) return rc;
  if (weights) {  // particle_weights (policy.py:103-121) of the replayed totals
    CKR(p->e_w.alloc(n));
    CK(cudaMemsetAsync(p->e_status.p, 0, sizeof(int), st));
    weights_kernel<<<1, 1024, 0, st>>>(p->e_tot.p, n, p->beta, p->e_w.p, p->e_status.p);
    CK(cudaGetLastError());
    int wst = 0;
    CK(cudaMemcpyAsync(weights, p->e_w.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&wst, p->e_status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (wst) for (int i = 0; i < n; ++i) weights[i] = NAN;  // the step itself failed: no weights
  }
  return MPPI_OK;
}

int mppi_get_bundle(mppi_plan* p, mppi_eval_out* out, double* weights) {
  if (!p || !out) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (!p->dump) return fail(MPPI_E_CONFIG, "plan was created without dump = 1");
  CKR(set_device(p));
  cudaStream_t st = p->stream;
  const size_t nhd = (size_t)p->N * p->H * p->D, nh = (size_t)p->N * p->H;
  if (out->positions) CK(cudaMemcpyAsync(out->positions, p->d_pos.p, sizeof(double) * nhd, cudaMemcpyDeviceToHost, st));
  if (out->velocities) CK(cudaMemcpyAsync(out->velocities, p->d_vel.p, sizeof(double) * nhd, cudaMemcpyDeviceToHost, st));
  if (out->accelerations) CK(cudaMemcpyAsync(out->accelerations, p->d_acc.p, sizeof(double) * nhd, cudaMemcpyDeviceToHost, st));
  if (out->step_costs) CK(cudaMemcpyAsync(out->step_costs, p->d_step.p, sizeof(double) * nh, cudaMemcpyDeviceToHost, st));
  if (out->terms) CK(cudaMemcpyAsync(out->terms, p->d_terms.p, sizeof(double) * 6 * nh, cudaMemcpyDeviceToHost, st));
  if (out->totals) CK(cudaMemcpyAsync(out->totals, p->totals.p, sizeof(double) * p->N, cudaMemcpyDeviceToHost, st));
  if (weights) CK(cudaMemcpyAsync(weights, p->d_w.p, sizeof(double) * p->N, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  out->bad_particle = -1;
  out->quarantined = 0;
  return MPPI_OK;
}


int mppi_episode(mppi_plan* p, const mppi_episode_desc* d, const double* theta0, const double* theta_dot0,
                 mppi_episode_state* es, mppi_episode_log* lg, int32_t* steps_done, double* device_ms) {
  if (!p || !d || !theta0 || !theta_dot0 || !es || !lg) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (p->B != 1) return fail(MPPI_E_CONFIG, "an episode drives a single-instance plan");
  if (d->steps < 0) return fail(MPPI_E_BAD_ARGUMENT, "negative episode length");
  if (!(d->dt > 0.0)) return fail(MPPI_E_BAD_ARGUMENT, "dt must be positive");
  if (!(d->filter_lambda >= 0.0 && d->filter_lambda <= 1.0))
    return fail(MPPI_E_BAD_ARGUMENT, "filter blend must lie in [0, 1]");
  const bool script = d->goal_source == MPPI_GOAL_SCRIPT;
  if (d->goal_source != MPPI_GOAL_FIXED && !script) return fail(MPPI_E_BAD_ARGUMENT, "unknown goal source");
  if (script) {
    if (d->waypoints < 1 || !d->times || !d->positions)
      return fail(MPPI_E_BAD_ARGUMENT, "target script needs at least one waypoint");
    for (int w = 1; w < d->waypoints; ++w)
      if (!(d->times[w] > d->times[w - 1])) return fail(MPPI_E_BAD_ARGUMENT, "waypoint times must increase");
    if (d->interpolation != MPPI_INTERP_HOLD && d->interpolation != MPPI_INTERP_LINEAR)
      return fail(MPPI_E_BAD_ARGUMENT, "unknown interpolation");
  }
  if (p->learned() && !p->mlp_ready) return fail(MPPI_E_CONFIG, "learned provider without weights");
  if (steps_done) *steps_done = 0;
  if (device_ms) *device_ms = 0.0;
  const int S = d->steps, D = p->D;
  if (S == 0) return MPPI_OK;
  CKR(set_device(p));
  CKR(flush_goal(p));
  cudaStream_t st = p->stream;
  // ---- buffers
  const size_t flog = (size_t)S * (1 + 3 * D + 3 + 9 + 3 + 9 + 1 + N_TERMS);
  CKR(p->ep_state.alloc((sizeof(EpisodeDev) + 7) / 8));
  CKR(p->ep_log.alloc(flog));
  CKR(p->ep_ilog.alloc((size_t)3 * S));
  CKR(p->ep_cmd.alloc(MPPI_MAX_DOF));
  CKR(p->ep_info.alloc(1));
  CKR(p->ev_in.alloc(2 * MPPI_MAX_DOF));
  CKR(p->ev_out.alloc(8));
  CKR(p->ev_records.alloc(kRecHead + 2 * D));
  CKR(p->ev_stepbuf.alloc(sizeof(double)));
  CKR(p->ev_status.alloc(2));
  CKR(p->ev_counters.alloc(1));
  if (p->learned()) {
    CKR(p->ev_x.alloc(128 * 16));
    CKR(p->ev_d.alloc(128));
    CK(cudaMemsetAsync(p->ev_x.p, 0, sizeof(float) * 128 * 16, st));
  }
  CK(cudaMemsetAsync(p->ev_status.p, 0, sizeof(int), st));
  CK(cudaMemsetAsync(p->ev_status.p + 1, 0x7f, sizeof(int), st));
  CK(cudaMemsetAsync(p->ev_counters.p, 0, sizeof(unsigned), st));
  if (script) {
    CKR(p->ep_script.alloc((size_t)4 * d->waypoints));
    CK(cudaMemcpyAsync(p->ep_script.p, d->times, sizeof(double) * d->waypoints, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(p->ep_script.p + d->waypoints, d->positions, sizeof(double) * 3 * d->waypoints,
                       cudaMemcpyHostToDevice, st));
  }
  if (d->noise) {
    CKR(p->ep_noise.alloc((size_t)2 * D * S));
    CK(cudaMemcpyAsync(p->ep_noise.p, d->noise, sizeof(double) * 2 * D * S, cudaMemcpyHostToDevice, st));
  }
  EpisodeDev h;
  memset(&h, 0, sizeof(h));
  h.armed = es->fallback_armed;
  h.ctr_base = p->step_counter;
  for (int j = 0; j < D; ++j) {
    h.plant[j] = h.est[j] = theta0[j];
    h.plant[D + j] = h.est[D + j] = theta_dot0[j];
    h.prev_cmd[j] = es->prev_command[j];
  }
  CK(cudaMemcpyAsync(p->ep_state.p, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  // ---- graph of one episode step
  EpisodeArgs ea;
  memset(&ea, 0, sizeof(ea));
  ea.ep = reinterpret_cast<EpisodeDev*>(p->ep_state.p);
  ea.S = S;
  ea.D = D;
  ea.goal_source = d->goal_source;
  ea.interp = d->interpolation;
  ea.script_mode = d->script_mode;
  ea.W = d->waypoints;
  ea.has_noise = d->noise != nullptr;
  ea.dt = d->dt;
  ea.lam = d->filter_lambda;
  ea.times = script ? p->ep_script.p : nullptr;
  ea.positions = script ? p->ep_script.p + d->waypoints : nullptr;
  ea.noise = d->noise ? p->ep_noise.p : nullptr;
  ea.state = p->state.p;
  ea.goal = p->goal.p;
  ea.status = p->status.p;
  ea.step_cmd = p->ep_cmd.p;
  ea.step_info = p->ep_info.p;
  ea.ev_pos = p->ev_in.p;
  ea.ev_vel = p->ev_in.p + D;
  ea.ev_status = p->ev_status.p;
  ea.ev_step = p->ev_out.p;
  ea.ev_terms = p->ev_out.p + 1;
  fill_chain(p->chain, p->costs.k_jl, ea.chain);
  double* L = p->ep_log.p;
  ea.t = L;
  ea.theta = ea.t + S;
  ea.theta_dot = ea.theta + (size_t)S * D;
  ea.command = ea.theta_dot + (size_t)S * D;
  ea.goalp = ea.command + (size_t)S * D;
  ea.goal_rot = ea.goalp + (size_t)3 * S;
  ea.ee = ea.goal_rot + (size_t)9 * S;
  ea.ee_rot = ea.ee + (size_t)3 * S;
  ea.cost_total = ea.ee_rot + (size_t)9 * S;
  ea.cost_terms = ea.cost_total + S;
  ea.collision = p->ep_ilog.p;
  ea.fallback = p->ep_ilog.p + S;
  ea.stat = p->ep_ilog.p + 2 * S;
  const int unroll = std::min(S, kEpisodeUnroll);
  // the graph bakes in the arguments (buffer pointers, sizes, dt, ...): reuse
  // the previous one when they are the same, recapture otherwise
  std::vector<unsigned char> key(sizeof(ea) + sizeof(int));
  memcpy(key.data(), &ea, sizeof(ea));
  memcpy(key.data() + sizeof(ea), &unroll, sizeof(int));
  if (!p->ep_graph || key != p->ep_key) {
    if (p->ep_graph) cudaGraphExecDestroy(p->ep_graph);
    p->ep_graph = nullptr;
    CKR(capture_episode_graph(p, ea, unroll, &p->ep_graph));
    p->ep_key = key;
  }
  cudaGraphExec_t exec = p->ep_graph;
  // ---- ceil(S / unroll) replays back to back, one synchronisation
  cudaError_t e = cudaEventRecord(p->ev0, st);
  for (int i = 0; i < S && e == cudaSuccess; i += unroll) e = cudaGraphLaunch(exec, st);
  if (e == cudaSuccess) e = cudaEventRecord(p->ev1, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(MPPI_E_CUDA, std::string("episode: ") + cudaGetErrorString(e));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
  CK(cudaMemcpy(&h, p->ep_state.p, sizeof(h), cudaMemcpyDeviceToHost));
  const int done = h.i;
  // ---- log and state back to the caller
  std::vector<double> fl(flog);
  std::vector<int> il((size_t)3 * S);
  CK(cudaMemcpy(fl.data(), L, sizeof(double) * flog, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(il.data(), p->ep_ilog.p, sizeof(int) * 3 * S, cudaMemcpyDeviceToHost));
  auto col = [&](double* dst, const double* src, size_t width) {
    if (dst) memcpy(dst, src, sizeof(double) * width * done);
  };
  const double* F = fl.data();
  col(lg->t, F, 1);
  col(lg->theta, F + S, D);
  col(lg->theta_dot, F + (size_t)S * (1 + D), D);
  col(lg->command, F + (size_t)S * (1 + 2 * D), D);
  col(lg->goal, F + (size_t)S * (1 + 3 * D), 3);
  col(lg->goal_rot, F + (size_t)S * (4 + 3 * D), 9);
  col(lg->ee, F + (size_t)S * (13 + 3 * D), 3);
  col(lg->ee_rot, F + (size_t)S * (16 + 3 * D), 9);
  col(lg->cost_total, F + (size_t)S * (25 + 3 * D), 1);
  if (lg->cost_terms)
    for (int k = 0; k < N_TERMS; ++k)
      memcpy(lg->cost_terms + (size_t)k * S, F + (size_t)S * (26 + 3 * D + k), sizeof(double) * done);
  if (lg->collision) memcpy(lg->collision, il.data(), sizeof(int) * done);
  if (lg->fallback) memcpy(lg->fallback, il.data() + S, sizeof(int) * done);
  if (lg->status) memcpy(lg->status, il.data() + 2 * S, sizeof(int) * done);
  for (int j = 0; j < 2 * D; ++j) {
    es->last_estimate[j] = h.est[j];
    es->plant[j] = h.plant[j];
  }
  for (int j = 0; j < D; ++j) {
    es->last_command[j] = h.last_cmd[j];
    es->prev_command[j] = h.prev_cmd[j];
  }
  es->fallback_armed = h.armed;
  es->aborted = h.aborted;
  p->step_counter += (unsigned long long)done;
  if (script && done > 0) {  // the plan goal is the last script goal; keep goal_host in step
    CK(cudaMemcpy(p->goal_host.data(), p->goal.p, sizeof(double) * 16, cudaMemcpyDeviceToHost));
  }
  if (steps_done) *steps_done = done;
  if (device_ms) *device_ms = ms;
  return MPPI_OK;
}

int mppi_top_rollouts(mppi_plan* p, int32_t k, int32_t* index_out, double* totals_out, double* ee_out) {
  if (!p || !index_out || !totals_out || !ee_out) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (k < 1 || k > 64 || k > p->N) return fail(MPPI_E_BAD_ARGUMENT, "k must lie in [1, min(64, particles)]");
  if (!p->dump) return fail(MPPI_E_CONFIG, "top rollouts need the bundle dump (plan created with dump = 1)");
  CKR(set_device(p));
  cudaStream_t st = p->stream;
  const int N = p->N, H = p->H, D = p->D;
  DevBuf<int> idx;
  DevBuf<double> out;
  DevBuf<unsigned char> taken;
  CKR(idx.alloc(k));
  CKR(out.alloc((size_t)k + (size_t)k * H * 3));
  CKR(taken.alloc(N));
  ChainT<double> ch;
  fill_chain(p->chain, p->costs.k_jl, ch);
  topk_rollouts_kernel<<<1, 512, 0, st>>>(p->totals.p, N, k, p->d_pos.p, H, D, ch, idx.p, out.p, out.p + k,
                                          taken.p);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(index_out, idx.p, sizeof(int) * k, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(totals_out, out.p, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ee_out, out.p + k, sizeof(double) * k * H * 3, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  idx.release();
  out.release();
  taken.release();
  return MPPI_OK;
}

int mppi_profile_stages(mppi_plan* p, int32_t enable) {
  if (!p) return fail(MPPI_E_BAD_ARGUMENT, "null plan");
  p->profile_level = enable < 0 ? 0 : (enable > 2 ? 2 : enable);
  return MPPI_OK;
}

int mppi_time_stage(mppi_plan* p, int32_t stage, int32_t reps, double* ms_per_launch) {
  if (!p || !ms_per_launch || reps < 1 || stage < 0 || stage > 3) return fail(MPPI_E_BAD_ARGUMENT, "bad arguments");
  CKR(set_device(p));
  CKR(flush_goal(p));
  CKR(ensure_graph(p));
  cudaStream_t st = p->stream;
  const unsigned mask = stage == 3 ? 7u : (1u << stage);
  CK(cudaStreamSynchronize(st));
  CK(cudaEventRecord(p->ev0, st));
  for (int r = 0; r < reps; ++r) {
    if (stage == 3) {
      CK(cudaGraphLaunch(p->graph, st));
    } else if (p->precision == MPPI_FP64) {
      CKR(enqueue_iteration<double>(p, 0, true, nullptr, st, mask));
    } else {
      CKR(enqueue_iteration<float>(p, 0, true, nullptr, st, mask));
    }
  }
  CK(cudaEventRecord(p->ev1, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
  *ms_per_launch = (double)ms / reps;
  return MPPI_OK;
}

// ---------------------------------------------------------------- sharded update
int mppi_stats_record_len(mppi_plan* p, int32_t* len) {
  if (!p || !len) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  *len = kRecHead + 2 * p->H * p->D;
  return MPPI_OK;
}

int mppi_stats_dev(mppi_plan* p, const double* theta, const double* theta_dot, void* record_dev,
                   void* stream) {
  if (!p || !record_dev) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (p->B != 1) return fail(MPPI_E_CONFIG, "particle sharding is for single-instance plans");
  if (p->learned() && !p->mlp_ready) return fail(MPPI_E_CONFIG, "learned provider without weights");
  CKR(set_device(p));
  cudaStream_t st = stream ? (cudaStream_t)stream : p->stream;
  CKR(flush_goal(p, st));
  const int D = p->D, it = p->sharded_iter;
  if (it == 0) {
    if (!theta || !theta_dot) return fail(MPPI_E_BAD_ARGUMENT, "state missing");
    memcpy(p->h_state, theta, sizeof(double) * D);
    memcpy(p->h_state + D, theta_dot, sizeof(double) * D);
    const unsigned long long ctr = p->step_counter++;
    memcpy(p->h_state + 2 * D, &ctr, sizeof(ctr));
    CK(cudaMemcpyAsync(p->state.p, p->h_state, sizeof(double) * (2 * D + 1), cudaMemcpyHostToDevice, st));
  }
  CKR(enqueue_sampling(p, it, st));
  double* rec = reinterpret_cast<double*>(record_dev);
  if (p->precision == MPPI_FP64)
    CKR(enqueue_iteration<double>(p, it, false, rec, st));
  else
    CKR(enqueue_iteration<float>(p, it, false, rec, st));
  return MPPI_OK;
}

int mppi_finalize_dev(mppi_plan* p, const void* records_dev, int32_t n_records, double* command_out,
                      mppi_step_info* info, void* stream) {
  if (!p || !records_dev || n_records < 1) return fail(MPPI_E_BAD_ARGUMENT, "bad records");
  CKR(set_device(p));
  cudaStream_t st = stream ? (cudaStream_t)stream : p->stream;
  const int it = p->sharded_iter;
  auto run = [&](auto tag) -> int {
    using R = decltype(tag);
    StatsArgs<R> s;
    stats_static<R>(p, p->H, p->gamma, p->tw, s);
    s.N = p->N;
    s.B = 1;
    s.shift = it == 0;
    s.means = p->means.p;
    s.var = p->var.p;
    s.sd = p->sd.p;
    s.prev_means = p->prev_means.p;
    s.prev_sd = p->prev_sd.p;
    s.status = p->status.p;
    s.bad = p->bad.p;
    s.cmd = p->m_cmd;
    s.info = p->m_info;
    s.reset_status = it == p->iters - 1;
    CK(launch_finalize<R>(s, (const double*)records_dev, n_records, st));
    return MPPI_OK;
  };
  if (p->precision == MPPI_FP64)
    CKR(run(double{}));
  else
    CKR(run(float{}));
  p->sharded_iter = (it + 1) % p->iters;
  if (command_out || info) {
    CK(cudaStreamSynchronize(st));
    if (command_out) memcpy(command_out, p->h_cmd, sizeof(double) * p->D);
    if (info) memcpy(info, p->h_info, sizeof(mppi_step_info));
  }
  return MPPI_OK;
}

// ---------------------------------------------------------------- exchange over peer memory
int mppi_peer_buffers(mppi_plan* p, int32_t world, void** recv_dev, void** flags_dev) {
  if (!p || !recv_dev || !flags_dev || world < 1 || world > MPPI_MAX_PEERS)
    return fail(MPPI_E_BAD_ARGUMENT, "world size out of range");
  if (p->B != 1) return fail(MPPI_E_CONFIG, "particle sharding is for single-instance plans");
  CKR(set_device(p));
  const size_t reclen = kRecHead + 2 * (size_t)p->H * p->D;
  if (p->peer_world != world) {
    p->peer_recv_buf.release();
    p->peer_flag_buf.release();
    CKR(p->peer_recv_buf.alloc(2 * (size_t)world * reclen));
    CKR(p->peer_flag_buf.alloc(world));
    CK(cudaMemset(p->peer_flag_buf.p, 0, sizeof(unsigned long long) * world));
    p->peer_world = world;
    p->peer_seq = 0;
  }
  *recv_dev = p->peer_recv_buf.p;
  *flags_dev = p->peer_flag_buf.p;
  return MPPI_OK;
}

int mppi_set_peers(mppi_plan* p, int32_t world, int32_t rank, void* const* recv_ptrs, void* const* flag_ptrs) {
  if (!p || !recv_ptrs || !flag_ptrs) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (world != p->peer_world || rank < 0 || rank >= world)
    return fail(MPPI_E_BAD_ARGUMENT, "mppi_peer_buffers(world) first; rank out of range");
  if (recv_ptrs[rank] != p->peer_recv_buf.p || flag_ptrs[rank] != p->peer_flag_buf.p)
    return fail(MPPI_E_BAD_ARGUMENT, "slot [rank] must hold this plan's own buffers");
  CKR(set_device(p));
  p->peer_recv_tab.release();
  p->peer_flag_tab.release();
  CKR(p->peer_recv_tab.alloc(world));
  CKR(p->peer_flag_tab.alloc(world));
  CK(cudaMemcpy(p->peer_recv_tab.p, recv_ptrs, sizeof(double*) * world, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(p->peer_flag_tab.p, flag_ptrs, sizeof(unsigned long long*) * world, cudaMemcpyHostToDevice));
  p->peer_rank = rank;
  p->peer_flag_host.assign((unsigned long long* const*)flag_ptrs, (unsigned long long* const*)flag_ptrs + world);
  return MPPI_OK;
}

int mppi_set_exchange_timeout(mppi_plan* p, double seconds) {
  if (!p || !(seconds > 0.0)) return fail(MPPI_E_BAD_ARGUMENT, "timeout must be positive");
  p->peer_timeout_s = seconds;
  return MPPI_OK;
}

// host-side abort of the next step: flag[rank] = (last seq of that step) | abort in every rank
static int publish_abort(mppi_plan* p, unsigned long long seq) {
  const unsigned long long v = seq | kPeerAbort;
  for (auto* f : p->peer_flag_host)
    CK(cudaMemcpy(f + p->peer_rank, &v, sizeof(v), cudaMemcpyHostToDevice));
  return MPPI_OK;
}

int mppi_exchange_abort(mppi_plan* p) {
  if (!p) return fail(MPPI_E_BAD_ARGUMENT, "null plan");
  if (p->peer_flag_host.empty()) return fail(MPPI_E_CONFIG, "mppi_set_peers first");
  CKR(set_device(p));
  p->peer_seq += (unsigned long long)p->iters;  // the abandoned step's sequence numbers
  return publish_abort(p, p->peer_seq);
}

int mppi_step_exchange(mppi_plan* p, const double* theta, const double* theta_dot, double* command_out,
                       mppi_step_info* info) {
  if (!p || !theta || !theta_dot || !command_out) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (!p->peer_recv_tab.p) return fail(MPPI_E_CONFIG, "mppi_set_peers first");
  if (p->learned() && !p->mlp_ready) return fail(MPPI_E_CONFIG, "learned provider without weights");
  CKR(set_device(p));
  CKR(flush_goal(p));
  cudaStream_t st = p->stream;
  const int D = p->D;
  memcpy(p->h_state, theta, sizeof(double) * D);
  memcpy(p->h_state + D, theta_dot, sizeof(double) * D);
  const unsigned long long ctr = p->step_counter++;
  memcpy(p->h_state + 2 * D, &ctr, sizeof(ctr));
  CK(cudaMemcpyAsync(p->state.p, p->h_state, sizeof(double) * (2 * D + 1), cudaMemcpyHostToDevice, st));
  p->peer_active = true;
  const unsigned long long seq0 = p->peer_seq;
  int rc = MPPI_OK;
  for (int it = 0; it < p->iters && rc == MPPI_OK; ++it) {
    ++p->peer_seq;  // one exchange per iteration, the same count on every rank
    rc = enqueue_sampling(p, it, st);
    if (rc == MPPI_OK)
      rc = p->precision == MPPI_FP64 ? enqueue_iteration<double>(p, it, false, nullptr, st)
                                     : enqueue_iteration<float>(p, it, false, nullptr, st);
  }
  p->peer_active = false;
  if (rc != MPPI_OK) {  // some iterations never launched: release the ranks waiting on them
    const std::string why = mppi_last_error();
    cudaStreamSynchronize(st);
    const unsigned long long last = seq0 + (unsigned long long)p->iters;  // the step's final sequence number
    p->peer_seq = last;
    publish_abort(p, last);
    return fail(rc, why);
  }
  CK(cudaStreamSynchronize(st));
  memcpy(command_out, p->h_cmd, sizeof(double) * D);
  if (info) memcpy(info, p->h_info, sizeof(mppi_step_info));
  if (p->h_info[0].status == MPPI_E_EXCHANGE)
    return fail(MPPI_E_EXCHANGE, "particle-sharded exchange: a rank aborted this step or did not publish its "
                                 "record within " + std::to_string(p->peer_timeout_s) + " s (policy kept shifted)");
  return MPPI_OK;
}

int mppi_ipc_get_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle_out, &h, sizeof(h));
  return MPPI_OK;
}

int mppi_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CK(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return MPPI_OK;
}

int mppi_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  CK(cudaIpcCloseMemHandle(dev_ptr));
  return MPPI_OK;
}

// ---------------------------------------------------------------- parity: the plan's MLP
int mppi_mlp_forward(mppi_plan* p, const double* q, int64_t m, double* out) {
  if (!p || !q || !out) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (!p->mlp_ready) return fail(MPPI_E_CONFIG, "mppi_set_mlp was not called");
  if (m < 1) return MPPI_OK;
  CKR(set_device(p));
  SCRATCH_OR_FAIL(S);
  const size_t rows = mlp_padded_rows(m);
  DEVPTR(S, double, dq, (size_t)m * p->D, q);
  DEVPTR(S, float, dx, rows * 16, (const float*)nullptr);
  DEVPTR(S, float, dd, rows, (const float*)nullptr);
  DEVPTR(S, double, dout, m, (const double*)nullptr);
  CK(cudaMemsetAsync(dx, 0, sizeof(float) * rows * 16, S.st));
  posenc_kernel<<<grid_for(m, 256), 256, 0, S.st>>>(dq, m, p->D, dx);
  CK(mlp_forward(p->mlp, dx, m, dd, S.st));
  float_to_double_kernel<<<grid_for(m, 256), 256, 0, S.st>>>(dd, m, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, sizeof(double) * m, cudaMemcpyDeviceToHost, S.st));
  CK(cudaStreamSynchronize(S.st));
  return MPPI_OK;
}

}  // extern "C"
