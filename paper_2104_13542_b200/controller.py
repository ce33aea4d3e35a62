"""Receding-horizon control loop on the B200 (jointmpc/controller.py:93-269).

``Controller.control_step`` is the drop-in for the reference's hot path. One
call = one H2D of the joint state, one CUDA-graph replay of
[shift, K x (sample, rollout + cost stack, learned collision, weights,
mean/covariance update)], one D2H of the command and status. The policy lives
on the device; ``controller.policy`` reads it back on access.

The episode driver around it (controller.py:53-78, 273-416: FilterState,
filter_state, EpisodeLog, run_episode) is here too; run_episode runs the whole
closed loop on the device (mppi_episode) when the controller's command mode
allows it.

Differences from the reference, by design:
  * ``workers`` is accepted and ignored (particles map to warps, not threads);
  * ``diag.bundle`` is always set, as in the reference (controller.py:250-259),
    but lazily: with ``keep_bundle=True`` the step graph dumps the last
    iteration and the bundle reads that dump back; by default (the lean
    latency graph) first access replays the last iteration on the device from
    its recorded inputs (state, policy view, perturbations) — one evaluation
    pass, paid only by callers that read the bundle;
  * per-stage times are device event times (event-record nodes in the step graph).
"""

from __future__ import annotations

import csv
import io
import logging
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .costs import CostStack, CostWeights, GoalSpec
from .engine import Plan, PlanSpec
from .errors import ContractError, PolicyStateError
from .kinematics import KinematicChain
from .policy import ISOTROPIC, PER_JOINT, PolicyParams, UpdateConfig
from .rollout import DtSchedule, JointState, RolloutBundle, make_dt_schedule
from .sampling import HALTON, PSEUDORANDOM, SmoothingSpec, smoothing_code
from .simworld import HOLD, LINEAR, TargetScript, sim_step, target_at

log = logging.getLogger(__name__)


@dataclass
class FilterState:
    """Measurement/prediction blend state (controller.py:53-60)."""

    lam: float
    last_command: np.ndarray
    last_estimate: JointState

    def __post_init__(self):
        if not 0.0 <= self.lam <= 1.0:
            raise ContractError("filter blend must lie in [0, 1]")


def filter_state(raw: JointState, filt: FilterState, dt: float) -> JointState:
    """Blend the measurement with the model prediction from the last command
    (controller.py:63-78); updates filt.last_estimate."""
    if dt <= 0.0:
        raise ContractError("dt must be positive")
    pv = filt.last_estimate.theta_dot + dt * filt.last_command
    pp = filt.last_estimate.theta + dt * pv
    lam = filt.lam
    est = JointState(theta=(1.0 - lam) * pp + lam * raw.theta, theta_dot=(1.0 - lam) * pv + lam * raw.theta_dot,
                     theta_ddot=filt.last_command.copy(), stamp=raw.stamp)
    filt.last_estimate = est
    return est


@dataclass(slots=True)  # built once per control step: slots make that ~2x cheaper
class StepDiagnostics:
    latency_ms: float
    sample_ms: float
    rollout_ms: float
    update_ms: float
    best_cost: float
    mean_cost: float
    fallback: str = ""  # "", "reissue", "brake"
    bundle: object = None


class Controller:
    """Owns the device policy, the perturbation block and the cost stack.
    Single-threaded by contract (controller.py:93-96)."""

    def __init__(
        self,
        chain: KinematicChain,
        goal: GoalSpec,
        *,
        horizon: int = 30,
        particles: int = 200,
        dt_base: float = 0.05,
        dt_ramp: str = "two_phase",
        gamma: float = 0.99,
        workers: int = 1,
        terminal_weight: float = 1.0,
        generator: str = HALTON,
        smoothing: SmoothingSpec | None = None,
        null_count: int = 2,
        weights: CostWeights | None = None,
        world=None,
        self_collision=None,
        beta: float = 0.5,
        alpha_mu: float = 0.9,
        alpha_sigma: float = 0.5,
        sigma0_sq: float = 1.0,
        sigma_sq_min: float = 1e-4,
        sigma_sq_max: float = 0.0,
        policy_mode: str = PER_JOINT,
        command_mode: str = "mean",
        iterations: int = 1,
        control_period: float = 0.05,
        latency_budget: float = 0.05,
        filter_lambda: float = 0.3,
        seed: int = 0,
        precision: str = "fp32",
        device: int = 0,
        keep_bundle: bool = False,
    ):
        if particles <= null_count + 1:
            raise ContractError("need more particles than reserved sequences")
        if generator not in (HALTON, PSEUDORANDOM):
            raise ContractError(f"unknown generator {generator!r}")
        if control_period <= 0.0:
            raise ContractError("control_period must be positive")
        if command_mode not in ("mean", "sample"):
            raise ContractError(f"unknown command mode {command_mode!r}")
        if policy_mode not in (ISOTROPIC, PER_JOINT):
            raise ContractError(f"unknown policy mode {policy_mode!r}")
        if precision not in ("fp32", "fp64"):
            raise ContractError(f"unknown precision {precision!r}")
        self.chain = chain
        self.generator = generator
        self.smoothing = smoothing or SmoothingSpec()
        self.particles = particles
        self.null_count = null_count
        self.horizon = horizon
        self.workers = workers
        self.terminal_weight = terminal_weight
        self.command_mode = command_mode
        self.iterations = max(1, iterations)
        self.control_period = control_period
        self.latency_budget = latency_budget
        self.filter_lambda = filter_lambda
        self.policy_mode = policy_mode
        self.sched = make_dt_schedule(horizon, dt_base, dt_ramp)
        self.update_cfg = UpdateConfig(
            beta=beta, alpha_mu=alpha_mu, alpha_sigma=alpha_sigma, gamma=gamma,
            sigma_sq_min=sigma_sq_min,
            sigma_sq_max=sigma_sq_max if sigma_sq_max > 0.0 else sigma0_sq,
        )
        self.sigma0_sq = sigma0_sq
        self.cost_stack = CostStack(chain=chain, weights=weights or CostWeights(), goal=goal,
                                    world=world, self_collision=self_collision)
        self.rng = np.random.default_rng(seed)
        self._knots = self.smoothing.knot_count(horizon)
        spec = PlanSpec(
            horizon=horizon, particles=particles, dts=self.sched.dts, null_count=null_count,
            instances=1, iterations=self.iterations,
            policy_mode=N.POLICY_ISOTROPIC if policy_mode == ISOTROPIC else N.POLICY_PER_JOINT,
            precision=N.FP64 if precision == "fp64" else N.FP32,
            generator=N.GEN_HALTON if generator == HALTON else N.GEN_PSEUDORANDOM,
            smoothing=smoothing_code(self.smoothing), spline_degree=self.smoothing.spline_degree,
            knots=self._knots, device=device, particles_total=particles, seed=seed,
            comb=tuple(self.smoothing.comb_coeffs), gamma=gamma, terminal_weight=terminal_weight,
            beta=beta, alpha_mu=alpha_mu, alpha_sigma=alpha_sigma, sigma0_sq=sigma0_sq,
            sigma_sq_min=self.update_cfg.sigma_sq_min, sigma_sq_max=self.update_cfg.sigma_sq_max,
            default_tail=self.update_cfg.default_tail, dump=int(keep_bundle),
        )
        world_arg = world if (world is not None and getattr(world, "obstacle_count", 0)) else None
        self._plan = Plan(chain, self.cost_stack.weights, spec, provider=self.cost_stack.self_collision,
                          world=world_arg)
        if generator == HALTON:
            self._plan.init_noise()
        self._goal_uploaded = None
        self._sync_goal()
        self._prev_command = np.zeros(chain.dof)
        self._fallback_armed = False
        self._step_serial = 0
        self.keep_bundle = keep_bundle
        z = np.zeros(chain.dof)
        self.filter = FilterState(lam=filter_lambda, last_command=z.copy(),
                                  last_estimate=JointState(theta=z.copy(), theta_dot=z.copy(), theta_ddot=z.copy()))

    # ---------------------------------------------------------------- state
    @property
    def plan(self) -> Plan:
        return self._plan

    @property
    def policy(self) -> PolicyParams:
        means, var = self._plan.get_policy(0)
        if self.policy_mode == ISOTROPIC:
            var = var[:, 0].copy()
        return PolicyParams(means=means, variances=var, mode=self.policy_mode, tail_variance=self.sigma0_sq)

    @policy.setter
    def policy(self, pol: PolicyParams):
        self._plan.set_policy(pol.means, pol.variances, 0)

    @property
    def _fixed_eps(self):
        """The centred Halton block (controller.py:166-176), read back from the device."""
        return self._plan.get_noise() if self.generator == HALTON else None

    def set_goal(self, goal: GoalSpec):
        self.cost_stack.goal = goal
        self._sync_goal()
        self._step_serial += 1  # a replayed bundle would see the new goal: expire it

    def set_perturbations(self, eps):
        """Overwrite the device perturbation block (the parity hook for
        Controller._perturbations, controller.py:192-196)."""
        self._plan.set_noise(eps)

    def _sync_goal(self):
        """Upload cost_stack.goal when it changed (a new GoalSpec, or its arrays
        edited in place — both are compared, as bytes, against the uploaded copy)."""
        g = self.cost_stack.goal
        pose = g.target_pose
        up = self._goal_uploaded
        if up is not None and up[0] is g and up[1] == g.mode and up[2] == pose.translation.tobytes() and \
                up[3] == pose.rotation.tobytes():
            return
        R = np.ascontiguousarray(pose.rotation, dtype=np.float64)
        t = np.ascontiguousarray(pose.translation, dtype=np.float64)
        self._plan.set_goal(R, t, g.mode_code, 0)
        self._goal_uploaded = (g, g.mode, pose.translation.tobytes(), pose.rotation.tobytes())

    def profile_stages(self, level: int = 2):
        """Fill StepDiagnostics.sample_ms / rollout_ms / update_ms from device
        events (level 2: instrumented graph with per-stage events; 1: whole-step
        device time; 0: off, the default)."""
        self._plan.profile_stages(int(level))

    # ---------------------------------------------------------------- hot path
    def control_step(self, state: JointState) -> tuple[np.ndarray, StepDiagnostics]:
        t_start = time.perf_counter()
        self._sync_goal()
        cmd_view, info = self._plan.step_single(state.theta, state.theta_dot)
        self._step_serial += 1
        if info.status != N.OK:
            exc = N.status_exception(info.status, info.bad_particle)
            if not isinstance(exc, (PolicyStateError, ContractError)):
                raise exc
            if not self._fallback_armed:
                self._fallback_armed = True
                command, mode = self._prev_command.copy(), "reissue"
            else:
                command, mode = np.zeros(self.chain.dof), "brake"
            log.warning("control step failed (%s); falling back to %s", exc, mode)
            self.filter.last_command = command.copy()
            latency = (time.perf_counter() - t_start) * 1e3
            return command, StepDiagnostics(latency_ms=latency, sample_ms=0.0, rollout_ms=info.device_ms,
                                            update_ms=0.0, best_cost=float("nan"),
                                            mean_cost=float("nan"), fallback=mode)
        self._fallback_armed = False
        if self.command_mode == "mean":
            command = cmd_view.copy()
        else:  # host rng, as next_command(policy, "sample", rng) (policy.py:174-176)
            pol = self.policy
            command = self.rng.normal(pol.means[0], pol.stddev()[0])
        # one private copy shared by the fallback ladder and the filter (both
        # only ever rebind it); the caller owns `command`
        kept = command.copy()
        self._prev_command = kept
        self.filter.last_command = kept
        latency = (time.perf_counter() - t_start) * 1e3
        if latency > self.latency_budget * 1e3:
            log.debug("control step overran budget: %.2f ms", latency)
        bundle = LazyBundle(self, self._step_serial)
        # positional: latency, sample, rollout, update, best, mean, fallback, bundle
        if not self._plan.profile_level:  # no device timing: the stage fields are zero (4 ctypes reads saved)
            return command, StepDiagnostics(latency, 0.0, latency, 0.0, info.best_cost, info.mean_cost, "", bundle)
        # without per-stage events the whole fused step is reported as rollout time
        roll = info.rollout_ms + info.mlp_ms
        return command, StepDiagnostics(latency, info.sample_ms, roll if roll > 0.0 else latency, info.update_ms,
                                        info.best_cost, info.mean_cost, "", bundle)

    def top_rollouts(self, k: int):
        """The k best rollouts of the last step for telemetry (bridge.py:196-203):
        (particle indices (k,), totals (k,), end-effector paths (k, H, coords)),
        selected and run through FK on the device. Needs keep_bundle=True."""
        import ctypes as C

        if not self.keep_bundle:
            raise ContractError("top_rollouts needs keep_bundle=True")
        k = int(k)
        idx = np.empty(k, dtype=np.int32)
        tot = np.empty(k)
        ee = np.empty((k, self.horizon, 3))
        N.check(self._plan.lib.mppi_top_rollouts(self._plan.handle, k, idx.ctypes.data_as(C.POINTER(C.c_int32)),
                                                 N.dptr(tot), N.dptr(ee)))
        coords = 2 if self.chain.task_dim == 2 else 3
        return idx.astype(np.int64), tot, ee[:, :, :coords]

    def instantaneous_costs(self, state: JointState):
        """Per-term costs of one plant state with the h=0 braking limit (controller.py:262-269)."""
        one = DtSchedule(dts=np.array([self.sched.dts.sum()]))
        step, terms = self.cost_stack.evaluate(state.theta[None, None, :], state.theta_dot[None, None, :], one)
        return float(step[0, 0]), {k: float(v[0, 0]) for k, v in terms.items()}


class LazyBundle:
    """RolloutBundle of the last iteration of one step, fetched from the device
    on first attribute access (the graph's dump with keep_bundle=True, else a
    device replay of that iteration). Valid until the controller's next step
    or goal change."""

    _FIELDS = ("positions", "velocities", "accelerations", "step_costs", "term_breakdown",
               "total_per_particle", "weights")

    def __init__(self, ctrl: Controller, serial: int):
        self._ctrl = ctrl
        self._serial = serial
        self._data = None

    def _load(self):
        if self._data is None:
            if self._ctrl._step_serial != self._serial:
                raise ContractError("bundle expired: the controller has stepped since")
            c = self._ctrl
            if c.keep_bundle:
                self._data = c._plan.get_bundle()
            else:
                self._data = c._plan.replay_bundle()
        return self._data

    def __getattr__(self, name):
        if name.startswith("_") or name not in self._FIELDS:
            raise AttributeError(name)
        return self._load()[name]

    def materialize(self) -> RolloutBundle:
        d = self._load()
        return RolloutBundle(**{k: d[k] for k in self._FIELDS if k != "weights"})


# ---------------------------------------------------------------- episodes
@dataclass
class EpisodeLog:
    """Step-indexed record of one simulated episode (controller.py:273-328);
    the CSV rendering is the external interface."""

    chain: KinematicChain
    t: np.ndarray
    theta: np.ndarray
    theta_dot: np.ndarray
    command: np.ndarray
    goal: np.ndarray
    ee: np.ndarray
    cost_total: np.ndarray
    cost_terms: dict
    collision: np.ndarray
    latency_ms: np.ndarray
    aborted: bool = False
    goal_rotations: np.ndarray | None = None
    ee_rotations: np.ndarray | None = None

    @property
    def steps(self) -> int:
        return self.t.shape[0]

    def header(self) -> list:
        d = self.chain.dof
        return (["t"] + [f"theta_{k}" for k in range(d)] + [f"thetadot_{k}" for k in range(d)]
                + [f"u_{k}" for k in range(d)] + [f"goal_{k}" for k in range(3)]
                + ["cost_total"] + [f"cost_{k}" for k in TERMS] + ["collision", "latency_ms"])

    def to_csv(self, path=None) -> str:
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(self.header())
        g = lambda v: f"{v:.17g}"  # noqa: E731
        for i in range(self.steps):
            w.writerow([g(self.t[i])] + [g(v) for v in self.theta[i]] + [g(v) for v in self.theta_dot[i]]
                       + [g(v) for v in self.command[i]] + [g(v) for v in self.goal[i]]
                       + [g(self.cost_total[i])] + [g(self.cost_terms[k][i]) for k in TERMS]
                       + [str(int(self.collision[i])), g(self.latency_ms[i])])
        text = buf.getvalue()
        if path is not None:
            with open(path, "w") as fh:
                fh.write(text)
        return text


TERMS = ("pose", "stop", "joint", "manip", "selfcoll", "envcoll")


def run_episode(controller: Controller, x0: JointState, goal_source, steps: int, noise_sigma: float = 0.0,
                sim_seed: int = 0, *, device_loop: bool | None = None) -> EpisodeLog:
    """Alternate control and plant steps (controller.py:331-416).

    goal_source is a GoalSpec or a TargetScript; a non-finite plant state
    ends the episode after logging that step. By default the whole loop runs
    on the device (mppi_episode: one graph replay per step, no host round
    trip; latency_ms is then the device time per step), with the plant noise
    drawn here from default_rng(sim_seed) in the reference's order so the
    inputs are the reference's. command_mode "sample" draws commands from the
    host rng and so runs the host loop (device_loop=False forces it)."""
    if device_loop is None:
        device_loop = controller.command_mode == "mean"
    if device_loop and controller.command_mode != "mean":
        raise ContractError("the device episode loop issues mean commands only")
    if device_loop:
        return _run_episode_device(controller, x0, goal_source, steps, noise_sigma, sim_seed)
    return _run_episode_host(controller, x0, goal_source, steps, noise_sigma, sim_seed)


def _episode_log(chain, cols: dict, aborted: bool) -> EpisodeLog:
    n = len(cols["t"])
    return EpisodeLog(
        chain=chain, t=np.asarray(cols["t"], dtype=np.float64),
        theta=np.asarray(cols["theta"]).reshape(n, chain.dof),
        theta_dot=np.asarray(cols["theta_dot"]).reshape(n, chain.dof),
        command=np.asarray(cols["command"]).reshape(n, chain.dof),
        goal=np.asarray(cols["goal"]).reshape(n, 3), ee=np.asarray(cols["ee"]).reshape(n, 3),
        cost_total=np.asarray(cols["cost_total"], dtype=np.float64),
        cost_terms={k: np.asarray(v, dtype=np.float64) for k, v in cols["terms"].items()},
        collision=np.asarray(cols["collision"], dtype=bool),
        latency_ms=np.asarray(cols["latency_ms"], dtype=np.float64), aborted=aborted,
        goal_rotations=np.asarray(cols["goal_rot"]).reshape(n, 3, 3),
        ee_rotations=np.asarray(cols["ee_rot"]).reshape(n, 3, 3))


def _run_episode_host(controller, x0, goal_source, steps, noise_sigma, sim_seed) -> EpisodeLog:
    """The reference's loop over this package's Controller (one control_step
    per plant step, each a host round trip)."""
    from .kinematics import fk_batch

    chain, dt = controller.chain, controller.control_period
    rng = np.random.default_rng(sim_seed) if noise_sigma > 0.0 else None
    cols = {k: [] for k in ("t", "theta", "theta_dot", "command", "goal", "goal_rot", "ee", "ee_rot",
                            "cost_total", "collision", "latency_ms")}
    cols["terms"] = {k: [] for k in TERMS}
    controller.filter.last_estimate = x0
    controller.filter.last_command = np.zeros(chain.dof)
    state, aborted = x0, False
    for i in range(steps):
        t_now = i * dt
        goal = target_at(goal_source, t_now) if isinstance(goal_source, TargetScript) else goal_source
        controller.set_goal(goal)
        est = filter_state(state, controller.filter, dt) if i > 0 else state
        command, diag = controller.control_step(est)
        total, terms = controller.instantaneous_costs(state)
        rot, trans = fk_batch(chain, state.theta[None, :])
        for k, v in (("t", t_now), ("theta", state.theta.copy()), ("theta_dot", state.theta_dot.copy()),
                     ("command", command.copy()), ("goal", goal.target_pose.translation.copy()),
                     ("goal_rot", goal.target_pose.rotation.copy()), ("ee", trans[0, -1].copy()),
                     ("ee_rot", rot[0, -1].copy()), ("cost_total", total),
                     ("collision", bool(terms["envcoll"] > 0.0)), ("latency_ms", diag.latency_ms)):
            cols[k].append(v)
        for k in TERMS:
            cols["terms"][k].append(terms[k])
        try:
            state = sim_step(state, command, dt, noise_sigma=noise_sigma, rng=rng)
        except ContractError:
            log.error("plant diverged at step %d; aborting episode", i)
            aborted = True
            break
    return _episode_log(chain, cols, aborted)


def _run_episode_device(controller, x0, goal_source, steps, noise_sigma, sim_seed) -> EpisodeLog:
    from .costs import goal_at_position

    chain, dt, d = controller.chain, controller.control_period, controller.chain.dof
    if steps < 0:
        raise ContractError("negative episode length")
    noise = None
    if noise_sigma > 0.0 and steps > 0:
        rng = np.random.default_rng(sim_seed)
        noise = np.empty((steps, 2 * d))
        for i in range(steps):  # sim_step's draw order: positions, then velocities
            noise[i, :d] = rng.normal(0.0, noise_sigma, size=d)
            noise[i, d:] = rng.normal(0.0, noise_sigma, size=d)
    script = None
    if isinstance(goal_source, TargetScript):
        mode_code = goal_at_position(goal_source.positions[0], mode=goal_source.mode).mode_code
        script = (goal_source.times, goal_source.positions,
                  N.INTERP_LINEAR if goal_source.interpolation == LINEAR else N.INTERP_HOLD, mode_code)
    else:
        controller.set_goal(goal_source)
    r = controller.plan.episode(steps, dt, controller.filter.lam, x0.theta, x0.theta_dot,
                                prev_command=controller._prev_command, fallback_armed=controller._fallback_armed,
                                script=script, noise=noise)
    n = r["steps_done"]
    # the Controller's host-side state as the reference loop leaves it
    controller._step_serial += n
    controller._prev_command = r["prev_command"].copy()
    controller._fallback_armed = r["fallback_armed"]
    controller.filter.last_command = r["last_command"].copy()
    if n > 1:
        est = r["last_estimate"]
        controller.filter.last_estimate = JointState(theta=est[:d].copy(), theta_dot=est[d:].copy(),
                                                     theta_ddot=r["command"][n - 2].copy(),
                                                     stamp=x0.stamp + (n - 1) * dt)
    else:
        controller.filter.last_estimate = x0
    if script is not None and n > 0:
        goal = target_at(goal_source, (n - 1) * dt)
        controller.cost_stack.goal = goal
        controller._goal_uploaded = (goal, goal.mode, goal.target_pose.translation.tobytes(),
                                     goal.target_pose.rotation.tobytes())
    for i in np.flatnonzero(r["fallback"] != N.FALLBACK_NONE):
        mode = "reissue" if r["fallback"][i] == N.FALLBACK_REISSUE else "brake"
        log.warning("control step %d failed (%s); fell back to %s", i,
                    N.status_exception(int(r["status"][i])), mode)
    if r["aborted"]:
        log.error("plant diverged at step %d; aborting episode", n - 1)
    per_step = r["device_ms"] / max(n, 1)
    cols = {"t": r["t"], "theta": r["theta"], "theta_dot": r["theta_dot"], "command": r["command"],
            "goal": r["goal"], "goal_rot": r["goal_rot"], "ee": r["ee"], "ee_rot": r["ee_rot"],
            "cost_total": r["cost_total"], "collision": r["collision"] != 0,
            "latency_ms": np.full(n, per_step), "terms": {k: r["cost_terms"][i] for i, k in enumerate(TERMS)}}
    return _episode_log(chain, cols, r["aborted"])
