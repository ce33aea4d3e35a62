"""Cost-term library and the fused cost stack (jointmpc/costs.py).

CostStack.evaluate runs the same fused rollout kernel as the controller in
"given positions/velocities" mode (one FK per configuration shared by all
terms, zero-weight terms skipped, costs.py:209-242) and returns
(step_costs, term breakdown) exactly like the reference.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as N
from . import kernels
from .errors import ContractError
from .kinematics import KinematicChain, Pose

FULL_POSE = "full_pose"
POSITION_ONLY = "position_only"
ORIENTATION_CONSTRAINED = "orientation_constrained"

TERM_NAMES = ("pose", "stop", "joint", "manip", "selfcoll", "envcoll")
NO_CONTACT = -1.0e30


@dataclass(frozen=True)
class CostWeights:
    """Directional pose weights + scalar term weights (costs.py:27-53)."""

    alpha_rot: np.ndarray = field(default_factory=lambda: np.full(3, 150.0))
    alpha_trans: np.ndarray = field(default_factory=lambda: np.full(3, 20.0))
    alpha_stop: float = 50.0
    alpha_joint: float = 100.0
    alpha_manip: float = 30.0
    alpha_coll: float = 1000.0
    k_jl: float = 0.1
    k_m: float = 0.05

    def __post_init__(self):
        for name in ("alpha_rot", "alpha_trans"):
            object.__setattr__(self, name, np.broadcast_to(
                np.asarray(getattr(self, name), dtype=np.float64), (3,)).copy())
        scalars = (self.alpha_stop, self.alpha_joint, self.alpha_manip, self.alpha_coll)
        if any(s < 0 for s in scalars) or np.any(self.alpha_rot < 0) or np.any(self.alpha_trans < 0):
            raise ContractError("cost weights must be non-negative")
        if not 0.0 <= self.k_jl < 0.5:
            raise ContractError("k_jl must lie in [0, 0.5)")
        if self.k_m <= 0.0:
            raise ContractError("k_m must be positive")


@dataclass
class GoalSpec:
    target_pose: Pose
    mode: str = POSITION_ONLY

    def __post_init__(self):
        if self.mode not in (FULL_POSE, POSITION_ONLY, ORIENTATION_CONSTRAINED):
            raise ContractError(f"unknown goal mode {self.mode!r}")
        R = np.asarray(self.target_pose.rotation, dtype=np.float64)
        if np.abs(R @ R.T - np.eye(3)).max() > 1e-9 or np.linalg.det(R) < 0.0:
            raise ContractError("goal rotation is not a proper rotation matrix")

    @property
    def mode_code(self) -> int:
        return N.GOAL_POSITION_ONLY if self.mode == POSITION_ONLY else N.GOAL_FULL_POSE


def goal_at_position(position, mode: str = POSITION_ONLY) -> GoalSpec:
    p = np.asarray(position, dtype=np.float64).ravel()
    if p.size == 2:
        p = np.array([p[0], p[1], 0.0])
    return GoalSpec(target_pose=Pose(rotation=np.eye(3), translation=p), mode=mode)


# ---------------------------------------------------------------- cost-term free functions
# The reference's per-term functions (costs.py:76-173), same signatures and
# broadcasting; the per-state arithmetic runs in the float64 cost-term kernels
# of the native library (csrc/mppi_seam.cu). braking_limits and
# shrunken_limits are O(H*d) configuration constants and stay on the host, as
# the plan builder computes them.

def pose_cost(rot_ee, trans_ee, goal: GoalSpec, alpha_rot, alpha_trans) -> np.ndarray:
    """Weighted pose distance for (..., 3, 3)/(..., 3) end-effector poses
    (costs.py:76-95): translation residual in the goal frame, plus the
    row-weighted Frobenius norm of I - R_g^T R_ee unless position_only."""
    trans_ee = N.f64(trans_ee)
    lead = trans_ee.shape[:-1]
    if trans_ee.shape[-1:] != (3,):
        raise ContractError("end-effector translations must be (..., 3)")
    m = int(np.prod(lead, dtype=np.int64))
    full = goal.mode != POSITION_ONLY
    rot = N.f64(rot_ee).reshape(m, 3, 3) if full else None
    out = np.empty(m)
    N.check(kernels._lib().mppi_pose_cost(
        N.dptr(rot), N.dptr(trans_ee.reshape(m, 3)), m, N.dptr(N.f64(goal.target_pose.rotation, (3, 3))),
        N.dptr(N.f64(goal.target_pose.translation, (3,))), N.GOAL_FULL_POSE if full else N.GOAL_POSITION_ONLY,
        N.dptr(np.broadcast_to(N.f64(alpha_rot), (3,)).copy()),
        N.dptr(np.broadcast_to(N.f64(alpha_trans), (3,)).copy()), N.dptr(out)))
    return out.reshape(lead)


def braking_limits(accel_max: np.ndarray, sched) -> np.ndarray:
    """(H, d) speeds still stoppable at maximum deceleration over the rest of
    the horizon (costs.py:98-101): suffix sums of dt times accel_max."""
    remaining = np.cumsum(np.asarray(sched.dts, dtype=np.float64)[::-1])[::-1]
    return np.multiply.outer(remaining, np.asarray(accel_max, dtype=np.float64))


def stop_cost(velocities: np.ndarray, accel_max: np.ndarray, sched) -> np.ndarray:
    """||max(|v| - braking limit, 0)||_2 per state (costs.py:104-108);
    velocities (..., H, d) -> (..., H)."""
    limits = N.f64(braking_limits(accel_max, sched))
    vel = N.f64(velocities)
    H, d = limits.shape
    if vel.shape[-2:] != (H, d):
        raise ContractError(f"velocities must be (..., {H}, {d}), got {vel.shape}")
    lead = vel.shape[:-2] if vel.ndim > 2 else (1,)  # (H, d) broadcasts to one batch row
    n = int(np.prod(lead, dtype=np.int64))
    out = np.empty((n, H))
    N.check(kernels._lib().mppi_stop_cost(N.dptr(vel.reshape(n, H, d)), n, H, d, N.dptr(limits), N.dptr(out)))
    return out.reshape(*lead, H)


def shrunken_limits(chain: KinematicChain, k_jl: float):
    """Joint range pulled in by k_jl of its span at both ends (costs.py:111-115)."""
    lo, hi = chain.joint_limits[:, 0], chain.joint_limits[:, 1]
    margin = k_jl * (hi - lo)
    return lo + margin, hi - margin


def joint_limit_cost(positions: np.ndarray, chain: KinematicChain, k_jl: float) -> np.ndarray:
    """Euclidean depth outside the shrunken limits (costs.py:118-123); (..., d) -> (...)."""
    lo, hi = shrunken_limits(chain, k_jl)
    pos = N.f64(positions)
    d = chain.dof
    if pos.shape[-1] != d:
        raise ContractError(f"expected {d} joint values, got shape {pos.shape}")
    lead = pos.shape[:-1]
    m = int(np.prod(lead, dtype=np.int64))
    out = np.empty(m)
    N.check(kernels._lib().mppi_joint_limit_cost(N.dptr(pos.reshape(m, d)), m, d, N.dptr(N.f64(lo)),
                                                 N.dptr(N.f64(hi)), N.dptr(out)))
    return out.reshape(lead)


def manipulability_cost_from_values(manip: np.ndarray, k_m: float) -> np.ndarray:
    """1 - m below the threshold k_m, else 0 (costs.py:126-127; discontinuous at k_m)."""
    mv = N.f64(manip)
    out = np.empty(mv.size)
    N.check(kernels._lib().mppi_manipulability_cost(N.dptr(mv.reshape(-1)), mv.size, float(k_m), N.dptr(out)))
    return out.reshape(mv.shape)


def manipulability_cost(chain: KinematicChain, q: np.ndarray, k_m: float) -> np.ndarray:
    """manipulability_cost_from_values of the chain's manipulability at q (costs.py:130-133)."""
    from .kinematics import manipulability_batch

    return manipulability_cost_from_values(manipulability_batch(chain, q), k_m)


def env_collision_cost(rot, trans, chain: KinematicChain, world) -> np.ndarray:
    """1.0 where any capsule hits an obstacle, else 0.0, for (..., d, 3, 3)/(..., d, 3)
    link poses (costs.py:164-173; deliberately discrete)."""
    trans = N.f64(trans)
    lead = trans.shape[:-2]
    hit = kernels.env_collision_batch(N.f64(rot).reshape(-1, chain.dof, 3, 3), trans.reshape(-1, chain.dof, 3),
                                      chain.cap_p0, chain.cap_p1, chain.cap_r, chain.cap_link,
                                      world.spheres, world.boxes)
    return (hit >= 0).astype(np.float64).reshape(lead)


class OracleSelfCollision:
    """Exact capsule-pair penetration (costs.py:136-156), on the GPU seam."""

    kind = "oracle"

    def __init__(self, chain: KinematicChain):
        self.chain = chain

    def distance(self, q: np.ndarray, poses=None) -> np.ndarray:
        ch = self.chain
        q = np.asarray(q, dtype=np.float64)
        if poses is None:
            rot, trans = kernels.fk_batch(q.reshape(-1, ch.dof), ch.axes, ch.origin_rot,
                                          ch.origin_trans, ch.jtype)
        else:
            rot = np.asarray(poses[0]).reshape(-1, ch.dof, 3, 3)
            trans = np.asarray(poses[1]).reshape(-1, ch.dof, 3)
        dist = kernels.self_collision_batch(rot, trans, ch.cap_p0, ch.cap_p1, ch.cap_r, ch.cap_link,
                                            ch.pair_a, ch.pair_b)
        return dist.reshape(q.shape[:-1])


def self_collision_cost(q: np.ndarray, provider) -> np.ndarray:
    return np.maximum(provider.distance(q), 0.0)


def total_cost(terms: dict, weights: CostWeights) -> np.ndarray:
    """Weighted sum of term arrays (costs.py:176-187). The fused kernels compute
    the same sum in-register; this helper only combines user-held arrays."""
    shapes = {np.shape(t) for t in terms.values()}
    if len(shapes) != 1:
        raise ContractError(f"cost term shapes differ: {sorted(shapes)}")
    return (terms["pose"] + weights.alpha_stop * terms["stop"] + weights.alpha_joint * terms["joint"]
            + weights.alpha_manip * terms["manip"]
            + weights.alpha_coll * (terms["selfcoll"] + terms["envcoll"]))


@dataclass
class CostStack:
    """Bound evaluation context (costs.py:190-245): chain, weights, goal,
    world and self-collision provider."""

    chain: KinematicChain
    weights: CostWeights
    goal: GoalSpec
    world: object = None
    self_collision: object = None

    term_names = TERM_NAMES

    def __post_init__(self):
        if self.self_collision is None and self.chain.pair_a.size:
            self.self_collision = OracleSelfCollision(self.chain)
        self._engine = None
        self._engine_key = None

    # one native plan per (weights, provider, world) combination, built lazily
    def engine(self, precision: int = N.FP32):
        from .engine import Plan, PlanSpec

        key = (id(self.weights), id(self.self_collision), id(self.world), precision)
        if self._engine is None or self._engine_key != key:
            spec = PlanSpec(horizon=2, particles=1, dts=np.full(2, 0.05), null_count=0,
                            generator=N.GEN_EXTERNAL, precision=precision, sigma_sq_max=1.0)
            world = self.world if (self.world is not None and getattr(self.world, "obstacle_count", 0)) else None
            self._engine = Plan(self.chain, self.weights, spec, provider=self.self_collision, world=world)
            self._engine_key = key
        g = self.goal
        self._engine.set_goal(g.target_pose.rotation, g.target_pose.translation, g.mode_code)
        return self._engine

    def evaluate(self, positions: np.ndarray, velocities: np.ndarray, sched, precision: int = N.FP64):
        """(step_costs, breakdown) for (n, H, d) position/velocity slices."""
        pos = N.f64(positions)
        vel = N.f64(velocities)
        if pos.ndim != 3 or pos.shape != vel.shape or pos.shape[2] != self.chain.dof:
            raise ContractError("positions/velocities must be matching (n, H, d) arrays")
        if pos.shape[1] != sched.horizon:
            raise ContractError("schedule horizon does not match the batch")
        eng = self.engine(precision)
        # mode 1: positions/velocities given, raw (un-quarantined) step costs
        r = eng.evaluate(1, pos, vel, sched.dts, 1.0, 1.0, want=("terms", "step_costs"))
        terms = {name: r["terms"][i] for i, name in enumerate(TERM_NAMES)}
        return r["step_costs"], terms

    def with_goal(self, goal: GoalSpec) -> "CostStack":
        return replace(self, goal=goal)
