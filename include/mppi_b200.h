/*
 * mppi_b200.h — C ABI of the B200-native joint-space MPPI step.
 *
 * This is the drop-in boundary for the reference's hot path
 * (jointmpc, arXiv 2104.13542). Everything below is
 * plain C: pointers, sizes, int status codes. No torch or CUDA types appear
 * in a signature; device pointers are passed as `void*`/`uint64_t` only in the
 * *_dev entry points, and a CUDA stream as an opaque `void*` (NULL = the
 * plan's own stream).
 *
 * Reference interfaces each entry point replaces (file:line are relative to
 * /root/reference/pkg/src/jointmpc/):
 *
 *   mppi_plan_create        Controller.__init__            controller.py:98-187
 *                           (+ CostStack.__post_init__      costs.py:205-207,
 *                              make_dt_schedule             rollout.py:67-81,
 *                              make_policy                  policy.py:88-95)
 *   mppi_init_noise         Halton fixed set               controller.py:166-176
 *                           <- unit_samples/gaussianize/smooth_sequences
 *                                                           sampling.py:118-265
 *   mppi_set_noise          Controller._perturbations       controller.py:192-196
 *                           (injected perturbations, the parity hook of
 *                            SURVEY §3.4)
 *   mppi_set_goal           Controller.set_goal             controller.py:189-190
 *   mppi_set_world          CostStack.world / WorldModel    simworld.py:30-49
 *   mppi_set_voxel_world    (new: 64^3 occupancy grid, config 3 bridge §8c)
 *   mppi_set_mlp            LearnedSelfCollision.load       surrogate.py:134-143
 *   mppi_get/set_policy     Controller.policy               controller.py:157,200,216
 *   mppi_step               Controller.control_step         controller.py:198-260
 *   mppi_evaluate           evaluate_rollouts               rollout.py:124-180
 *                           CostStack.evaluate              costs.py:209-242
 *   mppi_update_policy      particle_weights + update_mean + update_covariance
 *                                                           policy.py:103-155
 *   mppi_stats_dev /        (new: particle-sharded update, §8(e) config 5 —
 *   mppi_finalize_dev         per-rank weighted sufficient statistics, one
 *                             all-gather, fixed-order combine)
 *   mppi_step_exchange      (new: the same with the exchange fused into the
 *                             statistics kernel over NVLink peer memory)
 *
 *   The reference's fine-grained operator seam (kernels/__init__.py:50-66),
 *   float64 in / float64 out, caller-owned outputs:
 *   mppi_fk_batch           kernels.fk_batch                jit.py:89-111
 *   mppi_jacobian_batch     kernels.jacobian_batch          jit.py:114-148
 *   mppi_manip_batch        kernels.manip_batch             jit.py:151-185
 *   mppi_self_collision_batch kernels.self_collision_batch  jit.py:241-260
 *   mppi_env_collision_batch  kernels.env_collision_batch   jit.py:289-332
 *   mppi_integrate_batch    kernels.integrate_batch         jit.py:335-349
 *
 *   Sampling / policy free functions (sampling.py, policy.py):
 *   mppi_halton_points      halton_points                   sampling.py:100-115
 *   mppi_gaussianize        gaussianize                     sampling.py:167-202
 *   mppi_smooth_sequences   smooth_sequences                sampling.py:240-265
 *   mppi_build_controls     build_control_batch             sampling.py:268-290
 *   mppi_particle_weights   particle_weights                policy.py:103-121
 *   mppi_mlp_forward        MLP.forward (inference)         surrogate.py:42-52
 *
 * Error convention: every function returns an int status (MPPI_OK = 0). The
 * message of the last failure on the calling thread is in mppi_last_error().
 * The Python layer maps codes to the reference exceptions (errors.py):
 *   NONFINITE_CONTROL, BAD_ARGUMENT      -> ContractError
 *   ALL_QUARANTINED, WEIGHT_UNDERFLOW,
 *   NONPOSITIVE_VARIANCE                 -> PolicyStateError
 *   CONFIG                               -> ConfigError
 *   CUDA                                 -> DeviceError (not caught by the
 *                                           controller's fallback ladder)
 *
 * Threading: a plan is single-threaded (Controller is, controller.py:93-96);
 * distinct plans may be used from distinct threads / devices. The stateless
 * seam functions are re-entrant.
 */
#ifndef MPPI_B200_H
#define MPPI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPPI_ABI_VERSION 2

/* Compile-time capacity of the fused kernels. */
#define MPPI_MAX_DOF      8   /* kernels are instantiated for dof 1..8      */
#define MPPI_MAX_HORIZON  32  /* one warp per particle, one lane per step   */
#define MPPI_MAX_CAPSULES 16
#define MPPI_MAX_PAIRS    64
#define MPPI_MAX_PEERS    8   /* ranks of one node in the peer-memory exchange */
#define MPPI_MLP_IN_MAX   16  /* 2*dof positional encoding, padded          */

enum mppi_status {
  MPPI_OK = 0,
  MPPI_E_NONFINITE_CONTROL = 1,
  MPPI_E_ALL_QUARANTINED = 2,
  MPPI_E_WEIGHT_UNDERFLOW = 3,
  MPPI_E_BAD_ARGUMENT = 4,
  MPPI_E_CUDA = 5,
  MPPI_E_NONPOSITIVE_VARIANCE = 6,
  MPPI_E_CONFIG = 7,
  MPPI_E_SKIPPED = 8,          /* step not run: the on-device episode aborted */
  MPPI_E_EXCHANGE = 9          /* particle-sharded exchange: a rank aborted the step or did not
                                  publish its record within the exchange timeout (DeviceError) */
};

enum mppi_goal_mode {          /* costs.py:20-22 */
  MPPI_GOAL_POSITION_ONLY = 0,
  MPPI_GOAL_FULL_POSE = 1,     /* full_pose and orientation_constrained */
};

enum mppi_self_collision {     /* CostStack.self_collision provider kind */
  MPPI_SELFCOLL_NONE = 0,
  MPPI_SELFCOLL_ORACLE = 1,    /* capsule pairs, costs.py:136-156        */
  MPPI_SELFCOLL_LEARNED = 2    /* MLP on tcgen05, surrogate.py:120-125   */
};

enum mppi_generator {
  MPPI_GEN_HALTON = 0,         /* fixed, centred set drawn once           */
  MPPI_GEN_PSEUDORANDOM = 1,   /* Philox4x32-10 on device, every step     */
  MPPI_GEN_EXTERNAL = 2        /* caller injects eps via mppi_set_noise   */
};

enum mppi_smoothing { MPPI_SMOOTH_BSPLINE = 0, MPPI_SMOOTH_COMB = 1, MPPI_SMOOTH_NONE = 2 };
enum mppi_goal_source { MPPI_GOAL_FIXED = 0, MPPI_GOAL_SCRIPT = 1 };  /* run_episode goal_source */
enum mppi_interp { MPPI_INTERP_HOLD = 0, MPPI_INTERP_LINEAR = 1 };    /* TargetScript.interpolation */
enum mppi_fallback { MPPI_FALLBACK_NONE = 0, MPPI_FALLBACK_REISSUE = 1, MPPI_FALLBACK_BRAKE = 2 };
enum mppi_policy_mode { MPPI_POLICY_PER_JOINT = 0, MPPI_POLICY_ISOTROPIC = 1 };
enum mppi_precision { MPPI_FP32 = 0, MPPI_FP64 = 1 };

/* Packed chain, the layout of KinematicChain (kinematics.py:53-114).
 * All arrays row-major float64 / int64, exactly the numpy arrays. */
typedef struct mppi_chain_desc {
  int32_t dof;
  int32_t task_dim;          /* 2 or 3 */
  int32_t n_caps;
  int32_t n_pairs;
  const double* axes;         /* (dof,3)   */
  const double* origin_rot;   /* (dof,3,3) */
  const double* origin_trans; /* (dof,3)   */
  const int64_t* jtype;       /* (dof,) 0 revolute, 1 prismatic */
  const double* joint_limits; /* (dof,2)   */
  const double* velocity_limits; /* (dof,) */
  const double* accel_limits; /* (dof,)    */
  const double* cap_p0;       /* (n_caps,3) */
  const double* cap_p1;       /* (n_caps,3) */
  const double* cap_r;        /* (n_caps,)  */
  const int64_t* cap_link;    /* (n_caps,)  */
  const int64_t* pair_a;      /* (n_pairs,) */
  const int64_t* pair_b;      /* (n_pairs,) */
} mppi_chain_desc;

/* CostWeights (costs.py:27-53) + the provider kind. */
typedef struct mppi_cost_desc {
  double alpha_rot[3];
  double alpha_trans[3];
  double alpha_stop;
  double alpha_joint;
  double alpha_manip;
  double alpha_coll;
  double k_jl;
  double k_m;
  int32_t self_collision;     /* enum mppi_self_collision */
  int32_t _pad;
} mppi_cost_desc;

/* Controller kwargs (controller.py:98-129) in resolved form. */
typedef struct mppi_plan_desc {
  int32_t horizon;            /* H <= MPPI_MAX_HORIZON                      */
  int32_t particles;          /* particles held by THIS plan (per instance) */
  int32_t null_count;
  int32_t instances;          /* B independent controllers (config 4)       */
  int32_t iterations;         /* K optimisation iterations per step         */
  int32_t policy_mode;        /* enum mppi_policy_mode                      */
  int32_t precision;          /* enum mppi_precision (fused rollout)        */
  int32_t generator;          /* enum mppi_generator                        */
  int32_t smoothing;          /* enum mppi_smoothing                        */
  int32_t spline_degree;
  int32_t knots;              /* K knot slots (SmoothingSpec.knot_count)    */
  int32_t device;             /* CUDA ordinal                               */
  int32_t particle_offset;    /* particle sharding (config 5): this plan     */
  int32_t particles_total;    /*   holds global rows [offset, offset+N)     */
  int32_t dump;               /* 1: every step also writes instance 0's
                                 rollout bundle to device (mppi_get_bundle) */
  int32_t _pad0;
  uint64_t seed;             /* Philox key for the pseudorandom generator  */
  double comb[3];
  double gamma;
  double terminal_weight;
  double beta;
  double alpha_mu;
  double alpha_sigma;
  double sigma0_sq;           /* initial + tail variance                   */
  double sigma_sq_min;
  double sigma_sq_max;        /* already resolved: 0 in the kwargs -> sigma0_sq */
  double default_tail;
  const double* dts;          /* (horizon,) DtSchedule.dts                  */
} mppi_plan_desc;

/* Per-instance result of one control step (StepDiagnostics, controller.py:81-90). */
typedef struct mppi_step_info {
  int32_t status;             /* enum mppi_status of this instance           */
  int32_t bad_particle;       /* first non-finite particle, or -1            */
  int32_t finite_count;
  int32_t _pad;
  double best_cost;           /* min finite total                            */
  double mean_cost;           /* mean finite total                           */
  double device_ms;           /* CUDA-event time of the step on the stream   */
  /* per-stage device times inside the captured graph (event-record nodes),
   * summed over the K iterations */
  double sample_ms;
  double rollout_ms;
  double mlp_ms;
  double update_ms;
} mppi_step_info;

/* Outputs of mppi_evaluate (RolloutBundle, rollout.py:84-91). Any pointer may
 * be NULL to skip that output. Shapes use n particles x H steps x dof. */
typedef struct mppi_eval_out {
  double* positions;          /* (n,H,d) */
  double* velocities;         /* (n,H,d) */
  double* accelerations;      /* (n,H,d) the controls as integrated         */
  double* step_costs;         /* (n,H)   quarantined rows zeroed            */
  double* terms;              /* (6,n,H) pose, stop, joint, manip, selfcoll, envcoll */
  double* totals;             /* (n,)    +inf for quarantined rows          */
  int32_t bad_particle;       /* out: first non-finite control row, or -1   */
  int32_t quarantined;        /* out: number of quarantined rows            */
} mppi_eval_out;

typedef struct mppi_plan mppi_plan;

/* ---- library ---------------------------------------------------------- */
int32_t mppi_abi_version(void);
const char* mppi_last_error(void);
const char* mppi_build_info(void);          /* arch, nvcc, flags             */
int mppi_device_count(int32_t* count);

/* ---- plan lifecycle --------------------------------------------------- */
int mppi_plan_create(const mppi_chain_desc* chain, const mppi_cost_desc* costs,
                     const mppi_plan_desc* desc, mppi_plan** out);
int mppi_plan_destroy(mppi_plan* plan);

/* Build the Halton set on the device (FP64, bit-exact radical inverse),
 * Acklam ICDF, smoothing with the given (H,K) basis, then subtract the batch
 * mean over particles_total rows. basis may be NULL for comb / none. */
int mppi_init_noise(mppi_plan* plan, const double* basis /* (H,K) */);
int mppi_set_noise(mppi_plan* plan, const double* eps /* (N,H,d) host */);
int mppi_get_noise(mppi_plan* plan, double* eps /* (N,H,d) host */);

int mppi_set_goal(mppi_plan* plan, int32_t instance /* -1: all */,
                  const double* rotation /* (3,3) */, const double* translation /* (3,) */,
                  int32_t mode);
/* All instances at once (config 4): rotations (count,3,3), translations
 * (count,3), modes (count,) for instances [first, first+count). */
int mppi_set_goals(mppi_plan* plan, int32_t first, int32_t count, const double* rotations,
                   const double* translations, const int32_t* modes);
int mppi_set_world(mppi_plan* plan,const double* spheres, int32_t n_spheres,
                   const double* boxes, int32_t n_boxes);
/* Occupancy grid (nx,ny,nz) uint8, voxel (i,j,k) covers
 * origin + [i,i+1)*voxel ... ; narrow phase against boxes (nb,6) that tile
 * exactly the occupied set (NULL: decomposed on the host from the grid). */
int mppi_set_voxel_world(mppi_plan* plan, const uint8_t* occupancy, int32_t nx, int32_t ny,
                         int32_t nz, const double* origin /* (3,) */, double voxel,
                         const double* spheres, int32_t n_spheres);
int mppi_set_mlp(mppi_plan* plan, int32_t in_dim,
                 const double* W0, const double* b0, const double* W1, const double* b1,
                 const double* W2, const double* b2, const double* W3, const double* b3);

int mppi_set_policy(mppi_plan* plan, int32_t instance, const double* means /* (H,d) */,
                    const double* variances /* (H,d) */);
int mppi_get_policy(mppi_plan* plan, int32_t instance, double* means, double* variances);

/* ---- the hot path ----------------------------------------------------- */
/* One control step for all B instances: shift, K x (sample, rollout, costs,
 * learned collision, weights, mean/covariance update), command = means[0].
 * Host buffers; one H2D, one CUDA-graph replay, one D2H. theta/theta_dot are
 * (B,d); command_out (B,d); info (B) or NULL. On a per-instance failure the
 * policy of that instance is left shifted-but-not-updated (controller.py:200,
 * 224) and info[b].status says why; the function itself returns MPPI_OK. */
int mppi_step(mppi_plan* plan, const double* theta, const double* theta_dot,
              double* command_out, mppi_step_info* info);

/* Generic evaluation (evaluate_rollouts / CostStack.evaluate) on instance 0's
 * goal/world. mode 0: integrate `controls` (n,H,d) from theta0/theta_dot0;
 * mode 1: `controls` holds positions and `controls2` velocities (n,H,d), no
 * integration (CostStack.evaluate). dts (H,), gamma, terminal weight as in
 * rollout.py:111-121. Always FP64-exact inputs; arithmetic in the plan's
 * precision. */
int mppi_evaluate(mppi_plan* plan, int32_t mode, int32_t n, int32_t horizon,
                  const double* dts, double gamma, double terminal_weight,
                  const double* theta0, const double* theta_dot0,
                  const double* controls, const double* controls2, mppi_eval_out* out);

/* The inputs of the last iteration of the last mppi_step for one instance:
 * the joint state it started from and the (shifted) policy view its controls
 * were built from, u = means + stddev * eps (sampling.py:268-290). Replaying
 * them through mppi_evaluate (mode 0) reproduces that iteration's
 * RolloutBundle on a lean plan (dump = 0): Controller's lazily built
 * StepDiagnostics.bundle (controller.py:250-259).                            */
int mppi_get_step_inputs(mppi_plan* plan, int32_t instance, double* theta /* (d,) */,
                         double* theta_dot /* (d,) */, double* means /* (H,d) */,
                         double* stddev /* (H,d) */);

/* Instance 0's RolloutBundle of the last iteration of the last mppi_step on
 * a plan without dumps (the lean latency graph), recomputed on the device from
 * the iteration's recorded inputs: controls from the perturbation block and
 * the policy view of that iteration, one evaluation pass (mppi_evaluate mode
 * 0), the particle weights (NaN if that step failed). StepDiagnostics.bundle
 * (controller.py:250-259) of Controller(keep_bundle=False).                 */
int mppi_replay_bundle(mppi_plan* plan, mppi_eval_out* out, double* weights);

/* Instance 0's RolloutBundle of the last iteration of the last mppi_step
 * (plan created with dump = 1), plus the particle weights (N,). */
int mppi_get_bundle(mppi_plan* plan, mppi_eval_out* out, double* weights);

/* ---- closed-loop episode on the device -------------
 * run_episode (controller.py:331-416) without a host round trip per step: for
 * i < steps, on the plan stream,
 *   goal  = target_at(script, i*dt) (simworld.py:175-197) or the plan goal,
 *   est   = i > 0 ? filter_state(plant, filter, dt) : plant (controller.py:63-78),
 *   cmd   = control_step(est) with the fallback ladder (controller.py:224-241),
 *   costs = instantaneous_costs(plant) (controller.py:262-269), EE pose = FK,
 *   plant = sim_step(plant, cmd, dt, noise) (simworld.py:108-127);
 * a non-finite plant state ends the episode after logging that row (the
 * remaining replays leave the policy untouched, status MPPI_E_SKIPPED).
 * Plant noise is not drawn on the device: pass the reference's draws
 * (rng.normal(0, sigma, d) for the position, then for the velocity, per step)
 * as `noise` so the episode is the reference's bit-for-bit input. Requires
 * instances == 1 and command_mode "mean". */
typedef struct mppi_episode_desc {
  int32_t steps;              /* S                                          */
  int32_t goal_source;        /* enum mppi_goal_source                      */
  int32_t interpolation;      /* enum mppi_interp (script goals)            */
  int32_t script_mode;        /* enum mppi_goal_mode of the script goals    */
  int32_t waypoints;          /* W (script goals)                           */
  int32_t _pad;
  double dt;                  /* Controller.control_period                  */
  double filter_lambda;       /* FilterState.lam                            */
  const double* times;        /* (W,) strictly increasing                   */
  const double* positions;    /* (W,3)                                      */
  const double* noise;        /* (S,2d) or NULL                             */
} mppi_episode_desc;

/* EpisodeLog columns (controller.py:273-291), caller-owned host arrays of
 * `steps` rows; rows past *steps_done are left untouched. */
typedef struct mppi_episode_log {
  double* t;                  /* (S,)   */
  double* theta;              /* (S,d)  plant state at the start of the step */
  double* theta_dot;          /* (S,d)  */
  double* command;            /* (S,d)  */
  double* goal;               /* (S,3)  */
  double* goal_rot;           /* (S,9)  */
  double* ee;                 /* (S,3)  */
  double* ee_rot;             /* (S,9)  */
  double* cost_total;         /* (S,)   */
  double* cost_terms;         /* (6,S)  pose stop joint manip selfcoll envcoll */
  int32_t* collision;         /* (S,)   envcoll > 0                         */
  int32_t* fallback;          /* (S,)   enum mppi_fallback                  */
  int32_t* status;            /* (S,)   enum mppi_status of the control step */
} mppi_episode_log;

/* The filter / fallback state a host-side Controller mirrors. */
typedef struct mppi_episode_state {
  double last_estimate[2 * MPPI_MAX_DOF]; /* theta, theta_dot              */
  double last_command[MPPI_MAX_DOF];
  double prev_command[MPPI_MAX_DOF];      /* Controller._prev_command      */
  double plant[2 * MPPI_MAX_DOF];         /* plant state after the last step */
  int32_t fallback_armed;
  int32_t aborted;
} mppi_episode_state;

/* The filter starts from last_estimate = x0, last_command = 0 as run_episode
 * sets it (controller.py:354-355); prev_command and fallback_armed are read
 * from `state` (the Controller's); every field is written back at the end. */
int mppi_episode(mppi_plan* plan, const mppi_episode_desc* desc, const double* theta0,
                 const double* theta_dot0, mppi_episode_state* state, mppi_episode_log* log,
                 int32_t* steps_done, double* device_ms);

/* ---- surrogate training on the device --------------
 * train_collision_surrogate (surrogate.py:146-206) in float64: mini-batch MSE
 * on the (2d -> 256 -> 128 -> 64 -> 1) ReLU MLP, Adam (0.9, 0.999, 1e-8) with
 * the per-epoch step size lr[e], then the holdout MAE and sign agreement.
 * The caller supplies what the reference draws from its numpy generator —
 * the encoded samples, the labels, the per-epoch permutations, the He
 * initialisation (in weights / biases, overwritten with the trained values)
 * — and the Adam bias corrections 1 - beta^t per step, so the device trains
 * on the reference's inputs bit for bit. */
typedef struct mppi_train_desc {
  int32_t in_dim;             /* 2d                                         */
  int32_t n_train;
  int32_t n_hold;
  int32_t epochs;
  int32_t batch_size;         /* <= 1024                                    */
  int32_t _pad;
  const double* x_train;      /* (n_train, in_dim) positional encodings     */
  const double* y_train;      /* (n_train,) oracle distances                */
  const double* x_hold;       /* (n_hold, in_dim)                           */
  const double* y_hold;       /* (n_hold,)                                  */
  const int64_t* order;       /* (epochs, n_train) rng.permutation per epoch */
  const double* lr;           /* (epochs,) step size of each epoch          */
  const double* bias_corr1;   /* (epochs * ceil(n_train / batch)) 1 - 0.9^t   */
  const double* bias_corr2;   /* same, 1 - 0.999^t                          */
} mppi_train_desc;

typedef struct mppi_train_result {
  int64_t steps;              /* optimiser steps taken                      */
  int32_t diverged_epoch;     /* epoch of the first non-finite loss, or -1  */
  int32_t _pad;
  double last_finite_loss;
  double holdout_mae;
  double sign_agreement;
  double device_ms;           /* the training loop on the device            */
  double* losses;             /* optional out (epochs * batches) or NULL    */
} mppi_train_result;

/* weights[l] (dims[l], dims[l+1]) and biases[l] (dims[l+1]), l = 0..3. */
int mppi_train_mlp(const mppi_train_desc* desc, double* const* weights, double* const* biases,
                   mppi_train_result* result);

/* Telemetry: the k (<= 64) best rollouts of instance 0's last iteration
 * (bridge.py:196-203 — argsort of the totals, then the end-effector path of
 * each): particle indices (k), their totals (k) and end-effector positions
 * (k, H, 3). Ties go to the lower index. Needs a plan created with dump = 1. */
int mppi_top_rollouts(mppi_plan* plan, int32_t k, int32_t* index_out, double* totals_out, double* ee_out);

/* Step timing level. 0 (default): the lean step graph, no timing calls on the
 * latency path. 1: two stream events around the lean graph fill
 * mppi_step_info.device_ms. 2: an instrumented copy of the graph with
 * event-record nodes between the stages fills sample/rollout/mlp/update_ms
 * (the nodes serialise the replay and cost ~3.5 us each, so level 2 is for
 * attributing time to kernels, not for measuring the step). */
int mppi_profile_stages(mppi_plan* plan, int32_t level);

/* Benchmark hook: launch one stage of the step `reps` times back to back on
 * the plan stream between two CUDA events and report the mean device time per
 * launch. stage 0 = rollout kernel, 1 = learned-collision MLP, 2 = statistics
 * + update, 3 = the whole captured step graph. Perturbs the plan's policy
 * (the update runs `reps` times); call it after the steps you care about. */
int mppi_time_stage(mppi_plan* plan, int32_t stage, int32_t reps, double* ms_per_launch);

/* ---- particle-sharded update (config 5) -------------------------------- */
/* Size in doubles of one rank's statistics record for this plan. */
int mppi_stats_record_len(mppi_plan* plan, int32_t* len);
/* Run shift + sample + rollout + costs + local statistics for instance 0 into
 * the device buffer `record_dev` (record_len doubles); theta/theta_dot host. */
int mppi_stats_dev(mppi_plan* plan, const double* theta, const double* theta_dot,
                   void* record_dev, void* stream);
/* Combine `n_records` records (device, contiguous, rank order) and apply the
 * update; command/info as in mppi_step (instance 0). */
int mppi_finalize_dev(mppi_plan* plan, const void* records_dev, int32_t n_records,
                      double* command_out, mppi_step_info* info, void* stream);

/* ---- particle-sharded update over peer memory (config 5) ---------------
 * The same algebra as mppi_stats_dev + all-gather + mppi_finalize_dev, with
 * the collective fused into the statistics kernel: the kernel pushes the
 * rank record into slot [rank] of every rank's receive buffer with NVLink
 * P2P stores, publishes it with a release store of a sequence number into
 * every rank's flag [rank], waits for all ranks' flags and applies the update
 * (replaces sharded.py's NCCL all-gather; reference: controller.py:198-260
 * run on one controller's particles split over the ranks).
 * Setup, once per rank: mppi_peer_buffers -> mppi_ipc_get_handle on both
 * buffers -> exchange handles (any host collective) -> mppi_ipc_open_handle
 * for the peers' -> mppi_set_peers (slot [rank] = this plan's own buffers). */
int mppi_peer_buffers(mppi_plan* plan, int32_t world, void** recv_dev, void** flags_dev);
int mppi_set_peers(mppi_plan* plan, int32_t world, int32_t rank, void* const* recv_ptrs,
                   void* const* flag_ptrs);
/* One control step (all iterations) of this rank's particle shard; every rank
 * calls it with the same state and receives the same command. */
/* Bounded wait of the fused exchange (default 5 s): a rank whose flags do not
 * all arrive in time fails the step with MPPI_E_EXCHANGE, keeps the shifted
 * policy and publishes an abort so the other ranks stop waiting too.        */
int mppi_set_exchange_timeout(mppi_plan* plan, double seconds);
/* Abandon this rank's next exchange step (a host-side failure before its
 * kernels ran): publishes an abort for every iteration of that step into
 * every rank's flags and advances this rank's sequence past it.             */
int mppi_exchange_abort(mppi_plan* plan);
int mppi_step_exchange(mppi_plan* plan, const double* theta, const double* theta_dot,
                       double* command_out, mppi_step_info* info);
/* CUDA IPC of device buffers (handle: 64 bytes). */
int mppi_ipc_get_handle(void* dev_ptr, void* handle_out);
int mppi_ipc_open_handle(const void* handle, void** dev_ptr_out);
int mppi_ipc_close(void* dev_ptr);

/* ---- stateless free functions (host in, host out) ---------------------- */
int mppi_halton_points(int64_t count, int32_t dims, double* out /* (count,dims) */);
int mppi_gaussianize(const double* p, int64_t n, double* out);
/* Clamped uniform B-spline design matrix (bspline_basis, sampling.py:205-237). */
int mppi_bspline_basis(int32_t horizon, int32_t k, int32_t degree, double* out /* (H,K) */);
int mppi_smooth_sequences(const double* knots /* (N,K,d) */, int64_t n, int32_t k, int32_t d,
                          int32_t mode, const double* basis /* (H,K) or NULL */,
                          const double* comb /* (3,) */, int32_t horizon, double* out);
int mppi_build_controls(const double* eps /* (N,H,d) */, const double* means /* (H,d) */,
                        const double* stddev /* (H,d) */, int64_t n, int32_t h, int32_t d,
                        int32_t null_count, double* out /* (N,H,d) */);
int mppi_particle_weights(const double* totals, int64_t n, double beta, double* weights);
/* weights + mean + covariance update (policy.py:103-155), one call.
 * controls (N,H,d), weights (N,) ; means/variances in: the policy, out: updated.
 * isotropic: variances are (H,). */
int mppi_update_policy(const double* controls, const double* weights, int64_t n, int32_t h,
                       int32_t d, int32_t policy_mode, double alpha_mu, double alpha_sigma,
                       double sigma_sq_min, double sigma_sq_max, int32_t do_mean,
                       int32_t do_cov, double* means, double* variances);
int mppi_mlp_forward(mppi_plan* plan, const double* q /* (M,d) */, int64_t m,
                     double* out /* (M,) */);

/* ---- the reference operator seam (kernels/__init__.py) ------------------ */
int mppi_fk_batch(const double* q, int64_t m, int32_t d, const double* axes,
                  const double* origin_rot, const double* origin_trans, const int64_t* jtype,
                  double* rot_out /* (m,d,3,3) */, double* trans_out /* (m,d,3) */);
int mppi_jacobian_batch(const double* q, int64_t m, int32_t d, const double* rot,
                        const double* trans, const double* axes, const int64_t* jtype,
                        double* jac_out /* (m,6,d) */);
int mppi_manip_batch(const double* jac, int64_t m, int32_t d, int32_t task_dim,
                     double* out /* (m,) */);
int mppi_self_collision_batch(const double* rot, const double* trans, int64_t m, int32_t d,
                              const double* cap_p0, const double* cap_p1, const double* cap_r,
                              const int64_t* cap_link, int32_t n_caps, const int64_t* pair_a,
                              const int64_t* pair_b, int32_t n_pairs, double* out /* (m,) */);
int mppi_env_collision_batch(const double* rot, const double* trans, int64_t m, int32_t d,
                             const double* cap_p0, const double* cap_p1, const double* cap_r,
                             const int64_t* cap_link, int32_t n_caps, const double* spheres,
                             int32_t n_spheres, const double* boxes, int32_t n_boxes,
                             int64_t* hit_out /* (m,) */);
int mppi_integrate_batch(const double* u, int64_t n, int32_t h, int32_t d, const double* dts,
                         const double* th0, const double* thd0, double* pos_out,
                         double* vel_out);

/* ---- cost-term free functions (costs.py:76-133) ---------------------------
 * float64, stateless, caller-owned outputs, like the seam above. They replace
 * the reference's numpy bodies of the same names; the fused rollout computes
 * the same terms in-register and does not call these.                       */
/* pose_cost (costs.py:76-95): ||alpha_trans . R_g^T (t_ee - t_g)||_2, plus
 * ||diag(alpha_rot) (I - R_g^T R_ee)||_F unless mode = MPPI_GOAL_POSITION_ONLY */
int mppi_pose_cost(const double* rot_ee /* (m,3,3) */, const double* trans_ee /* (m,3) */, int64_t m,
                   const double* goal_rot /* (3,3) */, const double* goal_trans /* (3,) */, int32_t mode,
                   const double* alpha_rot /* (3,) */, const double* alpha_trans /* (3,) */,
                   double* out /* (m,) */);
/* stop_cost (costs.py:104-108): ||max(|v| - limits[h], 0)||_2 over joints;
 * limits = braking_limits (costs.py:98-101), (h,d)                          */
int mppi_stop_cost(const double* vel /* (n,h,d) */, int64_t n, int32_t h, int32_t d,
                   const double* limits /* (h,d) */, double* out /* (n,h) */);
/* joint_limit_cost (costs.py:118-123) against shrunken limits lo/hi (d,)   */
int mppi_joint_limit_cost(const double* pos /* (m,d) */, int64_t m, int32_t d, const double* lo,
                          const double* hi, double* out /* (m,) */);
/* manipulability_cost_from_values (costs.py:126-127): 1 - m if m < k_m else 0 */
int mppi_manipulability_cost(const double* manip /* (m,) */, int64_t m, double k_m,
                             double* out /* (m,) */);

#ifdef __cplusplus
}
#endif
#endif /* MPPI_B200_H */
