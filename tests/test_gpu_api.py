"""The drop-in Python API above the seam (SURVEY §8(b) "what the new drop-in
must keep") on the GPU: the cost-term free functions, jacobian_dot_times_qdot,
use_backend, StepDiagnostics.bundle on the lean graph, and the telemetry top-k
against the reference's own selection. Every expected value comes from the
reference itself (tests/golden/make_golden.py: cost_terms, topk)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _native():
    from paper_2104_13542_b200 import _native as N

    N.load_library()
    N.require_device()


def test_cost_term_free_functions_match_reference(arm7):
    from paper_2104_13542_b200 import costs as C
    from paper_2104_13542_b200.costs import FULL_POSE, GoalSpec, goal_at_position
    from paper_2104_13542_b200.kinematics import Pose
    from paper_2104_13542_b200.rollout import DtSchedule
    from paper_2104_13542_b200.simworld import WorldModel

    g = golden("cost_terms")
    full = GoalSpec(target_pose=Pose(rotation=g["goal_full_R"], translation=g["goal_full_t"]), mode=FULL_POSE)
    pos = goal_at_position(g["goal_pos_t"])
    np.testing.assert_allclose(C.pose_cost(g["ee_rot"], g["ee_trans"], full, g["a_rot"], g["a_trans"]),
                               g["pose_full"], rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(C.pose_cost(g["ee_rot"], g["ee_trans"], pos, g["a_rot"], g["a_trans"]),
                               g["pose_pos"], rtol=1e-13, atol=1e-12)
    # position-only goals never read the rotations (costs.py:91)
    np.testing.assert_allclose(C.pose_cost(None, g["ee_trans"], pos, g["a_rot"], g["a_trans"]), g["pose_pos"],
                               rtol=1e-13, atol=1e-12)
    sched = DtSchedule(dts=g["dts"])
    np.testing.assert_array_equal(C.braking_limits(arm7.accel_limits, sched), g["braking"])
    np.testing.assert_allclose(C.stop_cost(g["vel"], arm7.accel_limits, sched), g["stop"], rtol=1e-13, atol=1e-13)
    lo, hi = C.shrunken_limits(arm7, 0.1)
    np.testing.assert_array_equal(lo, g["shrunk_lo"])
    np.testing.assert_array_equal(hi, g["shrunk_hi"])
    np.testing.assert_allclose(C.joint_limit_cost(g["q"], arm7, 0.1), g["joint"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(C.joint_limit_cost(g["q"], arm7, 0.2), g["joint_k02"], rtol=1e-13, atol=1e-13)
    assert (g["joint"] > 0).any()  # the fixture leaves the limits
    # the branch at k_m is decided exactly as the reference decides it
    np.testing.assert_array_equal(C.manipulability_cost_from_values(g["manip_vals"], 0.05), g["manip_from_values"])
    np.testing.assert_allclose(C.manipulability_cost(arm7, g["q"], 0.05), g["manip"], atol=1e-12)
    world = WorldModel(spheres=g["spheres"], boxes=g["boxes"], bounds_min=np.full(3, -1.0),
                       bounds_max=np.full(3, 1.0))
    from paper_2104_13542_b200.kinematics import fk_batch

    rot, trans = fk_batch(arm7, g["q"])
    np.testing.assert_array_equal(C.env_collision_cost(rot, trans, arm7, world), g["envcoll"])
    # shapes and empty batches, as numpy would give them
    assert C.pose_cost(np.zeros((0, 3, 3)), np.zeros((0, 3)), full, g["a_rot"], g["a_trans"]).shape == (0,)
    assert C.joint_limit_cost(np.zeros((2, 0, 7)), arm7, 0.1).shape == (2, 0)
    assert C.stop_cost(g["vel"][0], arm7.accel_limits, sched).shape == (1, 30)


def test_jacobian_dot_times_qdot_matches_reference(arm7):
    from paper_2104_13542_b200.kinematics import jacobian_dot_times_qdot

    g = golden("cost_terms")
    for i in range(3):
        got = jacobian_dot_times_qdot(arm7, g["q"][0, i], g["qd"][i])
        # a central difference with step 1e-6: the float64 J agrees to ~1e-15,
        # amplified by 1/(2e-6)
        np.testing.assert_allclose(got, g["jdot_qd"][i], atol=5e-8)
    np.testing.assert_array_equal(jacobian_dot_times_qdot(arm7, g["q"][0, 0], np.zeros(7)), g["jdot_zero"])


def test_use_backend_rebinds_the_seam_table(arm7):
    from paper_2104_13542_b200 import kernels as K
    from paper_2104_13542_b200.kinematics import fk_batch

    seen = []
    real = K.fk_batch

    class Spy:
        BACKEND_NAME = K.BACKEND_NAME

    for fn in K._EXPORTED:
        setattr(Spy, fn, staticmethod(getattr(K, fn)))
    Spy.fk_batch = staticmethod(lambda *a: seen.append(1) or real(*a))
    orig_get = K.get_backend
    K.get_backend = lambda name: Spy if name == "spy" else orig_get(name)
    try:
        with K.use_backend("spy"):
            fk_batch(arm7, np.zeros(7))  # consumers resolve kernels.fk_batch at call time
        assert seen == [1]
        fk_batch(arm7, np.zeros(7))
        assert seen == [1] and K.fk_batch is real  # restored on exit
    finally:
        K.get_backend = orig_get
    with K.use_backend("cuda") as mod:
        assert mod.BACKEND_NAME == "cuda-sm100a"
    with pytest.raises(ValueError):
        with K.use_backend("numba"):
            pass


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_bundle_on_the_lean_graph_replays_the_step(precision):
    """diag.bundle is always set (controller.py:250-259). On the lean graph it
    is recomputed on first access from the step's recorded inputs; it must
    equal the dump of a keep_bundle=True controller fed the same states."""
    from paper_2104_13542_b200 import configs

    lean = configs.make_controller(2, precision=precision)
    dump = configs.make_controller(2, precision=precision, keep_bundle=True)
    st = configs.start_state()
    for i in range(3):
        st.theta = configs.start_state().theta + 0.01 * i
        c1, d1 = lean.control_step(st)
        c2, d2 = dump.control_step(st)
        np.testing.assert_array_equal(c1, c2)
        a, b = d1.bundle, d2.bundle
        assert a is not None
        rt = 1e-12 if precision == "fp64" else 2e-6
        np.testing.assert_allclose(a.total_per_particle, b.total_per_particle, rtol=rt)
        np.testing.assert_allclose(a.positions, b.positions, rtol=rt, atol=1e-12)
        np.testing.assert_allclose(a.accelerations, b.accelerations, rtol=1e-15, atol=1e-15)
        for k in b.term_breakdown:
            np.testing.assert_allclose(a.term_breakdown[k], b.term_breakdown[k], rtol=max(rt, 1e-9), atol=1e-9,
                                       err_msg=k)
        np.testing.assert_allclose(a.weights, b.weights, atol=1e-6)
    # a bundle expires with the next step
    _, d3 = lean.control_step(st)
    lean.control_step(st)
    from paper_2104_13542_b200.errors import ContractError

    with pytest.raises(ContractError):
        d3.bundle.total_per_particle


def test_top_rollouts_match_reference_selection(arm7):
    """Telemetry top-k against the reference bridge's own selection
    (bridge.py:196-203 on the reference's bundle): same particle indices, same
    totals and end-effector paths, at the second closed-loop step of config 2."""
    from paper_2104_13542_b200 import configs

    g = golden("topk")
    from paper_2104_13542_b200.policy import PER_JOINT, PolicyParams

    c = configs.make_controller(2, particles=500, keep_bundle=True, precision="fp64")
    # the second step starts from the reference's own policy and state
    c.policy = PolicyParams(means=g["means_in"], variances=g["variances_in"], mode=PER_JOINT, tail_variance=0.5)
    st = configs.start_state()
    st.theta = g["theta"][1].copy()
    st.theta_dot = g["theta_dot"][1].copy()
    c.control_step(st)
    idx, tot, ee = c.top_rollouts(8)
    np.testing.assert_array_equal(idx, g["order"])
    np.testing.assert_allclose(tot, g["totals"][g["order"]], rtol=1e-6)  # tensor-core MLP in the totals
    np.testing.assert_allclose(ee, g["ee_paths"], atol=1e-9)
