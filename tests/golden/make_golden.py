"""Generate the golden fixtures by running the REFERENCE itself.

Build container only (needs /root/reference; the GPU box never runs this):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz. Every array is the reference's own output on the
named inputs (numba backend, the reference default), so the oracle and the CUDA
path are both pinned to the reference, not to each other.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
OUT = Path(__file__).resolve().parent

import jointmpc  # noqa: E402  (the reference)
from jointmpc import kernels as rk  # noqa: E402
from jointmpc.controller import Controller  # noqa: E402
from jointmpc.costs import FULL_POSE, CostWeights, GoalSpec, goal_at_position  # noqa: E402
from jointmpc.kinematics import Pose, _rpy_matrix, load_chain  # noqa: E402
from jointmpc.policy import (UpdateConfig, make_policy, particle_weights, shift,  # noqa: E402
                             update_covariance, update_mean)
from jointmpc.rollout import JointState, evaluate_rollouts, make_dt_schedule  # noqa: E402
from jointmpc.sampling import (HALTON, SmoothingSpec, bspline_basis, gaussianize,  # noqa: E402
                               halton_points, smooth_sequences)
from jointmpc.controller import FilterState, filter_state, run_episode  # noqa: E402
from jointmpc.simworld import TargetScript, WorldModel, sim_step, target_position_at  # noqa: E402
from jointmpc.surrogate import LearnedSelfCollision  # noqa: E402

from paper_2104_13542_b200 import configs  # noqa: E402  (numbers only)

SURR = ROOT / "paper_2104_13542_b200" / "data" / "arm7_surrogate.npz"
print("reference backend:", rk.BACKEND_NAME, file=sys.stderr)


def random_q(chain, rng, n, margin=0.05):
    lo, hi = chain.joint_limits[:, 0], chain.joint_limits[:, 1]
    span = hi - lo
    return rng.uniform(lo + margin * span, hi - margin * span, size=(n, chain.dof))


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print("wrote", name, {k: np.shape(v) for k, v in arrays.items()}, file=sys.stderr)


def sampling_fixtures():
    rng = np.random.default_rng(1234)
    p = np.concatenate([rng.random(200), [0.0, 1e-12, 0.01, 0.02424, 0.02426, 0.5, 0.97574, 0.97576,
                                          0.99, 1.0 - 1e-12]])
    comb_in = rng.standard_normal((5, 12, 2))
    spline_knots = rng.standard_normal((6, 5, 3))
    arm7 = load_chain("arm7.chain")
    c = Controller(arm7, goal_at_position([0.4, 0.2, 0.5]), horizon=30, particles=48, seed=0)
    save("sampling",
         halton=halton_points(600, 7), gauss_p=p, gauss=gaussianize(p),
         basis_30_5=bspline_basis(30, 5, 3), basis_24_6=bspline_basis(24, 6, 3),
         basis_7_4_2=bspline_basis(7, 4, 2),
         comb_in=comb_in, comb_out=smooth_sequences(comb_in, SmoothingSpec(mode="comb"), 12),
         spline_knots=spline_knots,
         spline_out=smooth_sequences(spline_knots, SmoothingSpec(mode="bspline", knots_per_horizon=5), 30),
         fixed_eps_arm7_48=c._fixed_eps)


def kinematics_fixtures():
    rng = np.random.default_rng(7)
    out = {}
    for name, n in (("arm7", 96), ("planar2", 64), ("slider1", 16)):
        ch = load_chain(f"{name}.chain")
        q = random_q(ch, rng, n)
        rot, trans = rk.fk_batch(q, ch.axes, ch.origin_rot, ch.origin_trans, ch.jtype)
        J = rk.jacobian_batch(q, rot, trans, ch.axes, ch.jtype)
        out[f"{name}_q"] = q
        out[f"{name}_rot"] = rot
        out[f"{name}_trans"] = trans
        out[f"{name}_J"] = J
        out[f"{name}_manip"] = rk.manip_batch(J, ch.task_dim)
        out[f"{name}_self"] = rk.self_collision_batch(rot, trans, ch.cap_p0, ch.cap_p1, ch.cap_r,
                                                      ch.cap_link, ch.pair_a, ch.pair_b)
    # env collision: arm7 against spheres + boxes placed around its workspace
    ch = load_chain("arm7.chain")
    q = random_q(ch, rng, 256)
    rot, trans = rk.fk_batch(q, ch.axes, ch.origin_rot, ch.origin_trans, ch.jtype)
    spheres = np.array([[0.3, 0.0, 0.5, 0.15], [-0.2, 0.3, 0.8, 0.1], [0.0, -0.4, 0.3, 0.2]])
    boxes = np.array([[0.2, -0.2, 0.0, 0.6, 0.2, 0.3], [-0.6, -0.6, 0.6, -0.2, -0.1, 1.0],
                      [0.1, 0.3, 0.7, 0.5, 0.6, 1.1]])
    out["env_q"] = q
    out["env_spheres"] = spheres
    out["env_boxes"] = boxes
    out["env_hit"] = rk.env_collision_batch(rot, trans, ch.cap_p0, ch.cap_p1, ch.cap_r, ch.cap_link,
                                            spheres, boxes)
    out["env_hit_boxes_only"] = rk.env_collision_batch(rot, trans, ch.cap_p0, ch.cap_p1, ch.cap_r,
                                                       ch.cap_link, np.zeros((0, 4)), boxes)
    # integration
    u = rng.standard_normal((9, 11, 3)) * 3.0
    dts = make_dt_schedule(11, 0.05, "two_phase").dts
    th0, thd0 = rng.standard_normal(3), rng.standard_normal(3)
    pos, vel = rk.integrate_batch(u, dts, th0, thd0)
    out.update(int_u=u, int_dts=dts, int_th0=th0, int_thd0=thd0, int_pos=pos, int_vel=vel)
    save("kinematics", **out)


def mlp_fixtures():
    surr = LearnedSelfCollision.load(SURR)
    arm7 = load_chain("arm7.chain")
    q = random_q(arm7, np.random.default_rng(11), 512, margin=0.0)
    save("mlp", q=q, dist=surr.distance(q))


def policy_fixtures():
    rng = np.random.default_rng(5)
    totals = np.concatenate([rng.random(60) * 50 + 1000, [np.inf, np.inf]])
    w = particle_weights(totals, beta=0.7)
    pol = make_policy(6, 3, 0.8)
    pol.means[:] = rng.standard_normal((6, 3))
    u = rng.standard_normal((62, 6, 3))
    cfg = UpdateConfig(sigma_sq_min=0.05, sigma_sq_max=2.0)
    m1 = update_mean(pol, u, w, 0.9)
    c1 = update_covariance(m1, u, w, 0.5, cfg)
    iso = make_policy(6, 3, 0.8, mode="isotropic")
    iso_m = update_mean(iso, u, w, 0.7)
    iso_c = update_covariance(iso_m, u, w, 0.4, cfg)
    sh = shift(c1, 0.25)
    save("policy", totals=totals, weights=w, means0=pol.means, var0=pol.variances, controls=u,
         means1=m1.means, var1=c1.variances, iso_means=iso_m.means, iso_var=iso_c.variances,
         shift_means=sh.means, shift_var=sh.variances)


def reach_controller(config, particles=500, world=None, **kw):
    arm7 = load_chain("arm7.chain")
    wts = configs.WEIGHTS[config]
    weights = CostWeights(**wts)
    goal = GoalSpec(target_pose=Pose(rotation=_rpy_matrix(*configs.REACH_GOAL_RPY),
                                     translation=configs.REACH_GOAL_POS.copy()), mode=FULL_POSE)
    ckw = dict(configs.CONTROLLER_KW)
    ckw["particles"] = particles
    ckw.update(kw)
    provider = LearnedSelfCollision.load(SURR) if config == 2 else None
    return Controller(arm7, goal, weights=weights, self_collision=provider, world=world, **ckw)


def step_fixture(name, config, particles=500, steps=3, world=None, **kw):
    """Reference control steps from the reach start; step 0's full outputs plus
    the command / policy sequence of `steps` closed-loop steps (plant = sim_step)."""
    c = reach_controller(config, particles, world=world, **kw)
    state = JointState(theta=configs.REACH_START.copy(), theta_dot=np.zeros(7), theta_ddot=np.zeros(7))
    rec = {"eps": c._fixed_eps}
    cmds, means, variances, thetas, thetadots, best, mean = [], [], [], [], [], [], []
    for i in range(steps):
        thetas.append(state.theta.copy())
        thetadots.append(state.theta_dot.copy())
        cmd, diag = c.control_step(state)
        assert diag.fallback == "", diag.fallback
        cmds.append(cmd)
        means.append(c.policy.means.copy())
        variances.append(c.policy.variances.copy())
        best.append(diag.best_cost)
        mean.append(diag.mean_cost)
        if i == 0:
            b = diag.bundle
            rec.update(step_costs=b.step_costs, totals=b.total_per_particle,
                       weights=particle_weights(b.total_per_particle, c.update_cfg.beta),
                       positions_head=b.positions[:16], velocities_head=b.velocities[:16],
                       controls_head=b.accelerations[:16])
            for k, v in b.term_breakdown.items():
                rec[f"term_{k}"] = v
        state = sim_step(state, cmd, 0.05)
    rec.update(theta=np.array(thetas), theta_dot=np.array(thetadots), command=np.array(cmds),
               means=np.array(means), variances=np.array(variances), best_cost=np.array(best),
               mean_cost=np.array(mean))
    save(name, **rec)


def world_fixture():
    """Config-3-like world: boxes from a seeded voxel grid (the same boxes the
    GPU gets as a grid), position-only goal, N=128."""
    from paper_2104_13542_b200.simworld import seeded_box_grid

    grid_world = seeded_box_grid(n_boxes=8, dims=64, seed=3, max_extent=10)
    world = WorldModel(spheres=np.array([[0.35, 0.25, 0.55, 0.08]]), boxes=grid_world.boxes,
                       bounds_min=np.full(3, -1.0), bounds_max=np.full(3, 1.0))
    c = reach_controller(3, particles=128, world=world)
    c.cost_stack.goal = goal_at_position([0.45, 0.1, 0.55])
    state = JointState(theta=configs.REACH_START.copy(), theta_dot=np.zeros(7), theta_ddot=np.zeros(7))
    cmd, diag = c.control_step(state)
    b = diag.bundle
    save("step_world", occupancy=grid_world.voxel_grid.occupancy, boxes=grid_world.boxes,
         spheres=world.spheres, goal=np.array([0.45, 0.1, 0.55]), command=cmd,
         means=c.policy.means, variances=c.policy.variances, totals=b.total_per_particle,
         step_costs=b.step_costs, term_envcoll=b.term_breakdown["envcoll"],
         term_stop=b.term_breakdown["stop"], term_pose=b.term_breakdown["pose"])


def episode_parts():
    """Small known answers of the episode driver's pieces: target_position_at
    (hold / linear, before / inside / after the script), filter_state, sim_step
    with noise."""
    times = np.array([0.0, 0.3, 0.5, 1.2])
    pos = np.array([[0.1, 0.2, 0.3], [0.4, -0.2, 0.6], [0.0, 0.0, 0.9], [-0.3, 0.5, 0.2]])
    ts = np.array([0.0, 0.05, 0.3, 0.31, 0.499, 0.5, 0.9, 1.2, 1.5, 7.0])
    hold = np.array([target_position_at(TargetScript(times, pos, "hold"), t) for t in ts])
    lin = np.array([target_position_at(TargetScript(times, pos, "linear"), t) for t in ts])
    rng = np.random.default_rng(11)
    raw = JointState(theta=rng.normal(size=7), theta_dot=rng.normal(size=7), theta_ddot=np.zeros(7))
    filt = FilterState(lam=0.3, last_command=rng.normal(size=7),
                       last_estimate=JointState(theta=rng.normal(size=7), theta_dot=rng.normal(size=7),
                                                theta_ddot=np.zeros(7)))
    le_th, le_thd, lc = filt.last_estimate.theta.copy(), filt.last_estimate.theta_dot.copy(), filt.last_command.copy()
    est = filter_state(raw, filt, 0.05)
    u = rng.normal(size=7)
    nxt = sim_step(raw, u, 0.05, noise_sigma=0.01, rng=np.random.default_rng(5))
    save("episode_parts", times=times, positions=pos, ts=ts, hold=hold, linear=lin,
         raw_theta=raw.theta, raw_theta_dot=raw.theta_dot, le_theta=le_th, le_theta_dot=le_thd,
         last_command=lc, est_theta=est.theta, est_theta_dot=est.theta_dot, u=u,
         sim_theta=nxt.theta, sim_theta_dot=nxt.theta_dot)


def episode_fixture(name, config, steps, particles=500, script=None, goal=None, noise_sigma=0.0,
                    sim_seed=0, world=None):
    """Reference run_episode (controller.py:331-416): every EpisodeLog column
    plus the controller state it leaves behind."""
    c = reach_controller(config, particles, world=world)
    x0 = JointState(theta=configs.REACH_START.copy(), theta_dot=np.zeros(7), theta_ddot=np.zeros(7))
    lg = run_episode(c, x0, script if script is not None else goal, steps, noise_sigma=noise_sigma,
                     sim_seed=sim_seed)
    rec = dict(t=lg.t, theta=lg.theta, theta_dot=lg.theta_dot, command=lg.command, goal=lg.goal, ee=lg.ee,
               cost_total=lg.cost_total, collision=lg.collision, aborted=np.array(lg.aborted),
               goal_rotations=lg.goal_rotations, ee_rotations=lg.ee_rotations,
               final_means=c.policy.means, final_variances=c.policy.variances,
               filt_last_command=c.filter.last_command, filt_theta=c.filter.last_estimate.theta,
               filt_theta_dot=c.filter.last_estimate.theta_dot, noise_sigma=np.array(noise_sigma),
               sim_seed=np.array(sim_seed), steps=np.array(steps), particles=np.array(particles),
               csv=np.array(lg.to_csv()))
    for k, v in lg.cost_terms.items():
        rec[f"term_{k}"] = v
    if script is not None:
        rec.update(script_times=script.times, script_positions=script.positions,
                   script_interp=np.array(script.interpolation), script_mode=np.array(script.mode))
    if world is not None:
        rec.update(boxes=world.boxes, spheres=world.spheres)
    save(name, **rec)


def episode_fixtures():
    lin = TargetScript(times=np.array([0.0, 0.2, 0.45]),
                       positions=np.array([[0.45, 0.1, 0.55], [0.35, -0.2, 0.6], [0.5, 0.05, 0.4]]),
                       interpolation="linear", mode="position_only")
    episode_fixture("episode_c1", 1, steps=12, script=lin, noise_sigma=0.002, sim_seed=7)
    goal = GoalSpec(target_pose=Pose(rotation=_rpy_matrix(*configs.REACH_GOAL_RPY),
                                     translation=configs.REACH_GOAL_POS.copy()), mode=FULL_POSE)
    episode_fixture("episode_c2", 2, steps=6, goal=goal)
    from paper_2104_13542_b200.simworld import seeded_box_grid

    grid_world = seeded_box_grid(n_boxes=8, dims=64, seed=3, max_extent=10)
    world = WorldModel(spheres=np.array([[0.35, 0.25, 0.55, 0.08]]), boxes=grid_world.boxes,
                       bounds_min=np.full(3, -1.0), bounds_max=np.full(3, 1.0))
    hold = TargetScript(times=np.array([0.0, 0.1]), positions=np.array([[0.45, 0.1, 0.55], [0.4, 0.2, 0.5]]),
                        interpolation="hold", mode="position_only")
    episode_fixture("episode_c3", 3, steps=5, particles=128, script=hold, world=world)


def cost_term_fixtures():
    """The reference's cost-term free functions (costs.py:76-173) and
    jacobian_dot_times_qdot (kinematics.py:235-245) on seeded inputs, with
    manipulability values straddling k_m and states outside the limits."""
    from jointmpc import costs as rc
    from jointmpc.kinematics import fk_batch as rfk, jacobian_dot_times_qdot
    from jointmpc.rollout import make_dt_schedule

    rng = np.random.default_rng(21)
    arm7 = load_chain("arm7.chain")
    q = random_q(arm7, rng, 6 * 5, margin=-0.15).reshape(6, 5, 7)  # some beyond the limits
    rot, trans = rfk(arm7, q)  # (6,5,7,3,3), (6,5,7,3)
    goal_full = GoalSpec(target_pose=Pose(rotation=_rpy_matrix(0.3, -0.2, 1.1),
                                          translation=np.array([0.3, -0.1, 0.6])), mode=FULL_POSE)
    goal_pos = goal_at_position([0.45, 0.1, 0.55])
    a_rot, a_trans = np.array([30.0, 20.0, 10.0]), np.array([150.0, 120.0, 90.0])
    sched = make_dt_schedule(30, 0.05, "two_phase")
    vel = rng.normal(scale=2.0, size=(4, 30, 7))
    manip_vals = np.concatenate([rng.uniform(0.0, 0.1, 40), [0.05, 0.05 - 1e-9, 0.05 + 1e-9, 0.0, 1.0]])
    world = WorldModel(spheres=np.array([[0.35, 0.25, 0.55, 0.08], [0.1, -0.3, 0.4, 0.12]]),
                       boxes=np.array([[0.2, -0.1, 0.3, 0.45, 0.15, 0.5], [-0.5, -0.5, 0.0, -0.2, -0.2, 0.3]]),
                       bounds_min=np.full(3, -1.0), bounds_max=np.full(3, 1.0))
    qd = rng.normal(size=(3, 7))
    save("cost_terms", q=q, ee_rot=rot[..., -1, :, :], ee_trans=trans[..., -1, :],
         goal_full_R=goal_full.target_pose.rotation, goal_full_t=goal_full.target_pose.translation,
         goal_pos_t=goal_pos.target_pose.translation, a_rot=a_rot, a_trans=a_trans,
         pose_full=rc.pose_cost(rot[..., -1, :, :], trans[..., -1, :], goal_full, a_rot, a_trans),
         pose_pos=rc.pose_cost(rot[..., -1, :, :], trans[..., -1, :], goal_pos, a_rot, a_trans),
         dts=sched.dts, braking=rc.braking_limits(arm7.accel_limits, sched), vel=vel,
         stop=rc.stop_cost(vel, arm7.accel_limits, sched),
         shrunk_lo=rc.shrunken_limits(arm7, 0.1)[0], shrunk_hi=rc.shrunken_limits(arm7, 0.1)[1],
         joint=rc.joint_limit_cost(q, arm7, 0.1), joint_k02=rc.joint_limit_cost(q, arm7, 0.2),
         manip_vals=manip_vals, manip_from_values=rc.manipulability_cost_from_values(manip_vals, 0.05),
         manip=rc.manipulability_cost(arm7, q, 0.05),
         spheres=world.spheres, boxes=world.boxes, envcoll=rc.env_collision_cost(rot, trans, arm7, world),
         qd=qd, jdot_qd=np.stack([jacobian_dot_times_qdot(arm7, q[0, i], qd[i]) for i in range(3)]),
         jdot_zero=jacobian_dot_times_qdot(arm7, q[0, 0], np.zeros(7)))


def topk_fixture():
    """The reference bridge's telemetry selection (bridge.py:196-203) on its own
    bundle: config 2, N=500, the second closed-loop step."""
    from jointmpc.kinematics import fk_batch as rfk

    c = reach_controller(2)
    state = JointState(theta=configs.REACH_START.copy(), theta_dot=np.zeros(7), theta_ddot=np.zeros(7))
    cmd, _ = c.control_step(state)
    state = sim_step(state, cmd, 0.05)
    means_in, variances_in = c.policy.means.copy(), c.policy.variances.copy()
    cmd, diag = c.control_step(state)
    k = 8
    order = np.argsort(diag.bundle.total_per_particle)[:k]
    q_paths = diag.bundle.positions[order]
    _, path_trans = rfk(c.chain, q_paths.reshape(-1, 7))
    save("topk", theta=np.stack([configs.REACH_START, state.theta]),
         theta_dot=np.stack([np.zeros(7), state.theta_dot]), order=order, means_in=means_in,
         variances_in=variances_in,
         totals=diag.bundle.total_per_particle, ee_paths=path_trans[:, -1, :3].reshape(k, 30, 3))


def tracking_fixture(particles=500, steps=3):
    """Config 3 at the benched shape: configs.tracking_problem()'s
    script and box world (built with the reference's FK), N=500, 3 closed-loop
    steps, goal = the script's target at t = i*dt. Every step's inputs (state,
    goal, the policy it starts from) and outputs (terms, totals, weights,
    command, updated policy), so each GPU step can start from the reference's
    own inputs and the decision-band rule can be applied per step."""
    from jointmpc.kinematics import fk_batch as rfk
    from jointmpc.simworld import target_at as rtarget_at

    script, world = configs.tracking_problem(fk=rfk)
    rworld = WorldModel(spheres=np.zeros((0, 4)), boxes=world.boxes, bounds_min=np.full(3, -1.0),
                        bounds_max=np.full(3, 1.0))
    rscript = TargetScript(times=script.times, positions=script.positions, interpolation="linear",
                           mode="position_only")
    c = reach_controller(3, particles, world=rworld)
    state = JointState(theta=configs.REACH_START.copy(), theta_dot=np.zeros(7), theta_ddot=np.zeros(7))
    rec = {"eps": c._fixed_eps, "boxes": world.boxes, "occupancy": world.voxel_grid.occupancy,
           "script_times": script.times, "script_positions": script.positions}
    cols = {k: [] for k in ("theta", "theta_dot", "goal", "means_in", "variances_in", "command", "means",
                            "variances", "totals", "weights", "step_costs", "best_cost")}
    terms = {k: [] for k in ("pose", "stop", "joint", "manip", "selfcoll", "envcoll")}
    for i in range(steps):
        goal = rtarget_at(rscript, i * 0.05)
        c.set_goal(goal)
        cols["theta"].append(state.theta.copy())
        cols["theta_dot"].append(state.theta_dot.copy())
        cols["goal"].append(goal.target_pose.translation.copy())
        cols["means_in"].append(c.policy.means.copy())
        cols["variances_in"].append(c.policy.variances.copy())
        cmd, diag = c.control_step(state)
        assert diag.fallback == "", diag.fallback
        b = diag.bundle
        cols["command"].append(cmd)
        cols["means"].append(c.policy.means.copy())
        cols["variances"].append(c.policy.variances.copy())
        cols["totals"].append(b.total_per_particle)
        cols["weights"].append(particle_weights(b.total_per_particle, c.update_cfg.beta))
        cols["step_costs"].append(b.step_costs)
        cols["best_cost"].append(diag.best_cost)
        for k in terms:
            terms[k].append(b.term_breakdown[k])
        state = sim_step(state, cmd, 0.05)
    rec.update({k: np.array(v) for k, v in cols.items()})
    rec.update({f"term_{k}": np.array(v) for k, v in terms.items()})
    save("step_c3", **rec)


def training_fixtures():
    """Reference train_collision_surrogate runs (surrogate.py:146-206): a short
    one (3 epochs) for weight-level parity, one through both step-size halvings
    (80 epochs), and the acceptance configuration's metrics (50k samples, 100
    epochs, seed 0; test_acceptance.py:267-279)."""
    import time

    from jointmpc.surrogate import train_collision_surrogate

    arm7 = load_chain("arm7.chain")
    for name, samples, seed, epochs in (("train_short", 2000, 3, 3), ("train_sched", 3000, 5, 80)):
        m = train_collision_surrogate(arm7, samples, seed, epochs=epochs)
        rec = {f"W{i}": w for i, w in enumerate(m.net.weights)}
        rec.update({f"b{i}": v for i, v in enumerate(m.net.biases)})
        save(name, samples=np.array(samples), seed=np.array(seed), epochs=np.array(epochs),
             holdout_mae=np.array(m.holdout_mae), sign_agreement=np.array(m.sign_agreement), **rec)
    t0 = time.perf_counter()
    m = train_collision_surrogate(arm7, 50_000, 0)
    save("train_accept", samples=np.array(50_000), seed=np.array(0), epochs=np.array(100),
         holdout_mae=np.array(m.holdout_mae), sign_agreement=np.array(m.sign_agreement),
         cpu_seconds=np.array(time.perf_counter() - t0))


if __name__ == "__main__":
    which = set(sys.argv[1:])
    jobs = {"sampling": sampling_fixtures, "kinematics": kinematics_fixtures, "mlp": mlp_fixtures,
            "policy": policy_fixtures,
            "step_c1": lambda: step_fixture("step_c1", 1),
            "step_c2": lambda: step_fixture("step_c2", 2),
            "step_c2_iso_k2": lambda: step_fixture("step_c2_iso_k2", 2, particles=256, steps=2,
                                                   policy_mode="isotropic", iterations=2),
            "step_world": world_fixture, "episode_parts": episode_parts, "episodes": episode_fixtures,
            "cost_terms": cost_term_fixtures, "topk": topk_fixture, "step_c3": tracking_fixture,
            "training": training_fixtures}
    for name, fn in jobs.items():
        if not which or name in which:
            fn()
