"""The BASELINE.json workloads as plain data.

Config 1/2 are reach_arm7.toml (fixtures/reach_arm7.toml:1-49) at N=500:
full-pose goal, alpha_p = [[30]*3, [150]*3] (rotation, translation — the
harness mapping, harness.py:66), beta 1, alpha_mu 0.9, alpha_sigma 0.5,
sigma0^2 0.5, sigma_min^2 0.01, Halton + cubic B-spline, 2 null rows,
H = 30, dt 0.05 two_phase, gamma 0.99.
"""

from __future__ import annotations

import numpy as np

REACH_START = np.array([0.0, -0.5, 0.0, -1.8, 0.0, 1.4, 0.0])
REACH_GOAL_POS = np.array([-0.13, -0.109, 0.864])
REACH_GOAL_RPY = (0.108, 0.489, 0.927)

CONTROLLER_KW = dict(
    horizon=30, particles=500, dt_base=0.05, dt_ramp="two_phase", gamma=0.99, terminal_weight=1.0,
    null_count=2, beta=1.0, alpha_mu=0.9, alpha_sigma=0.5, sigma0_sq=0.5, sigma_sq_min=0.01,
    sigma_sq_max=0.0, seed=0,
)

WEIGHTS = {
    # config 1: goal pose + joint limits only
    1: dict(alpha_rot=30.0, alpha_trans=150.0, alpha_stop=0.0, alpha_joint=100.0, alpha_manip=0.0,
            alpha_coll=0.0),
    # config 2: full stack with the learned self-collision MLP
    2: dict(alpha_rot=30.0, alpha_trans=150.0, alpha_stop=50.0, alpha_joint=100.0, alpha_manip=30.0,
            alpha_coll=1000.0),
    # config 3: pose (position only, moving target) + joint + stop + world collision
    3: dict(alpha_rot=30.0, alpha_trans=150.0, alpha_stop=50.0, alpha_joint=100.0, alpha_manip=0.0,
            alpha_coll=1000.0),
}


def reach_goal_rotation() -> np.ndarray:
    from .kinematics import rpy_matrix

    return rpy_matrix(*REACH_GOAL_RPY)


def make_weights(config: int):
    from .costs import CostWeights

    return CostWeights(**WEIGHTS[config])


def make_goal(config: int):
    from .costs import FULL_POSE, GoalSpec
    from .kinematics import Pose

    return GoalSpec(target_pose=Pose(rotation=reach_goal_rotation(), translation=REACH_GOAL_POS.copy()),
                    mode=FULL_POSE)


def make_controller(config: int = 2, **overrides):
    """A Controller for BASELINE config 1 or 2 (arm7, 500 x 30)."""
    from .controller import Controller
    from .kinematics import load_chain
    from .surrogate import load_arm7_surrogate

    kw = dict(CONTROLLER_KW)
    kw.update(overrides)
    provider = load_arm7_surrogate() if config == 2 else None
    return Controller(load_chain("arm7.chain"), make_goal(config), weights=make_weights(config),
                      self_collision=provider, **kw)


def batched_problem(instances: int, first: int = 0, chain=None):
    """Config 4 goals and start states for instances [first, first+instances):
    goal_i = FK(q_i) (full pose), q_i ~ U(k_jl-shrunk limits) from default_rng(i);
    theta0_i ~ U(shrunk limits) from default_rng(10000 + i)."""
    from .costs import FULL_POSE, GoalSpec
    from .kinematics import Pose, fk_batch, load_chain

    chain = chain or load_chain("arm7.chain")
    lo, hi = chain.joint_limits[:, 0], chain.joint_limits[:, 1]
    k = WEIGHTS[2].get("k_jl", 0.1)
    lo_s, hi_s = lo + k * (hi - lo), hi - k * (hi - lo)
    idx = range(first, first + instances)
    q = np.stack([np.random.default_rng(i).uniform(lo_s, hi_s) for i in idx])
    th0 = np.stack([np.random.default_rng(10000 + i).uniform(lo_s, hi_s) for i in idx])
    rot, trans = fk_batch(chain, q)
    goals = [GoalSpec(target_pose=Pose(rotation=rot[i, -1], translation=trans[i, -1]), mode=FULL_POSE)
             for i in range(instances)]
    return goals, th0


def tracking_problem(seed: int = 0, n_boxes: int = 8, dims: int = 64, fk=None):
    """Config 3: moving target (TargetScript, linear, 5 waypoints = FK of seeded
    in-limit q, one every 3 s, position_only) and a 64^3 grid over [-1,1]^3
    built from 8 seeded voxel-aligned boxes that do not touch the start pose's
    capsules. ``fk(chain, q)`` defaults to the device seam;
    tests/golden/make_golden.py passes the reference's own FK."""
    from .kinematics import load_chain
    from .simworld import TargetScript, seeded_box_grid

    if fk is None:
        from .kinematics import fk_batch as fk
    fk_batch = fk

    chain = load_chain("arm7.chain")
    rng = np.random.default_rng(seed)
    lo, hi = chain.joint_limits[:, 0], chain.joint_limits[:, 1]
    q = rng.uniform(lo + 0.1 * (hi - lo), hi - 0.1 * (hi - lo), size=(5, 7))
    _, trans = fk_batch(chain, q)
    script = TargetScript(times=np.arange(5) * 3.0, positions=trans[:, -1], interpolation="linear",
                          mode="position_only")
    rot0, tr0 = fk_batch(chain, REACH_START[None])
    caps0 = [(rot0[0, l] @ p0 + tr0[0, l], rot0[0, l] @ p1 + tr0[0, l], r)
             for p0, p1, r, l in zip(chain.cap_p0, chain.cap_p1, chain.cap_r, chain.cap_link)]

    def keep_clear(box):
        lo_b, hi_b = box[:3], box[3:]
        for a, b, r in caps0:
            for t in np.linspace(0.0, 1.0, 9):
                p = a + t * (b - a)
                gap = np.maximum(lo_b - p, 0.0) + np.maximum(p - hi_b, 0.0)
                if np.sqrt((gap * gap).sum()) < r + 0.05:
                    return False
        return True

    world = seeded_box_grid(n_boxes=n_boxes, dims=dims, seed=seed, keep_clear=keep_clear)
    return script, world


def start_state():
    from .rollout import JointState

    return JointState(theta=REACH_START.copy(), theta_dot=np.zeros(7), theta_ddot=np.zeros(7))
