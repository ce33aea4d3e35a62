"""FP32 parity at the benched shapes of configs 3 and 5 under the SURVEY §8(c)
decision-band rule (tests/band.py).

* Config 3: configs.tracking_problem() (the world and target script
  `bench.py --workload c3` times), N=500, against the reference's own three
  closed-loop steps (tests/golden/step_c3.npz). Each device step starts from
  the reference's inputs (state, goal, policy), so every difference is the
  device's arithmetic. The device sees the 64^3 voxel grid, the reference the
  union of boxes it was built from (the config-3 bridge).
* Config 5: config-2 costs (learned self-collision MLP), FP32, N = 65,536 and
  262,144, against the chunked float64 oracle (oracle.rollout_scores with
  `chunk`: per-slice evaluation, then the full-N update), which is pinned to
  the reference at N=500 by tests/test_oracle_golden.py. The Halton block is
  the device's (bit-exact Halton + FP64 centring, pinned separately).
"""

import numpy as np
import pytest

from band import apply_bands, corrected_command, weight_safe
from conftest import golden
from oracle import mppi_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _native():
    from paper_2104_13542_b200 import _native as N

    N.load_library()
    N.require_device()


def _check_step(report, cmd, bundle, ref, margins, weights, cfg, means_in, variances_in, precision, null_count=2):
    """Band rule on one step; returns the band report."""
    _, dtot, rep = apply_bands(bundle.term_breakdown, ref["terms"], margins, weights, cfg["gamma"], 1.0)
    tot = bundle.total_per_particle + dtot
    tol = 1e-3 if precision == "fp32" else 1e-6
    rep["weight_safe_err"] = weight_safe(tot, ref["totals"], ref["weights"], cfg["beta"], tol)
    ms, vs = O.shifted(means_in, variances_in, 0.0, cfg["sigma0_sq"])
    kw = dict(beta=cfg["beta"], alpha_mu=cfg["alpha_mu"], alpha_sigma=cfg["alpha_sigma"],
              smin=cfg["sigma_sq_min"], smax=cfg["sigma0_sq"])
    u = bundle.accelerations  # the device's own controls
    np.testing.assert_allclose(u, O.shape_controls(ref["eps"], ms, vs, null_count), atol=1e-6)
    # the device's command is the update of its own totals ...
    own, _, _, _ = corrected_command(u, bundle.total_per_particle, ms, vs, **kw)
    np.testing.assert_allclose(cmd, own, atol=1e-3)
    # ... and, with band hits substituted, the reference's command
    fixed, _, _, _ = corrected_command(u, tot, ms, vs, **kw)
    np.testing.assert_allclose(fixed, ref["command"], atol=1e-3)
    if rep["manip_band_hits"] == 0 and rep["envcoll_band_hits"] == 0:
        np.testing.assert_allclose(cmd, ref["command"], atol=1e-3)
    report.append(rep)
    return rep


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_config3_benched_world_matches_reference(arm7, precision):
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.controller import Controller
    from paper_2104_13542_b200.costs import goal_at_position
    from paper_2104_13542_b200.policy import PER_JOINT, PolicyParams
    from paper_2104_13542_b200.simworld import target_at

    g = golden("step_c3")
    script, world = configs.tracking_problem()  # built on this box with the device FK
    np.testing.assert_array_equal(world.voxel_grid.occupancy, g["occupancy"])
    np.testing.assert_array_equal(world.boxes, g["boxes"])
    np.testing.assert_allclose(script.positions, g["script_positions"], atol=1e-12)
    kw = dict(configs.CONTROLLER_KW)
    c = Controller(arm7, target_at(script, 0.0), weights=configs.make_weights(3), world=world, keep_bundle=True,
                   precision=precision, **kw)
    np.testing.assert_allclose(c._fixed_eps, g["eps"], atol=1e-12)
    cfg = dict(kw)
    w3 = configs.make_weights(3)
    report = []
    for i in range(g["command"].shape[0]):
        c.policy = PolicyParams(means=g["means_in"][i], variances=g["variances_in"][i], mode=PER_JOINT,
                                tail_variance=cfg["sigma0_sq"])
        c.set_goal(goal_at_position(g["goal"][i]))
        st = configs.start_state()
        st.theta, st.theta_dot = g["theta"][i].copy(), g["theta_dot"][i].copy()
        cmd, diag = c.control_step(st)
        assert diag.fallback == ""
        # oracle margins on the reference's inputs
        ms, vs = O.shifted(g["means_in"][i], g["variances_in"][i], 0.0, cfg["sigma0_sq"])
        u = O.shape_controls(g["eps"], ms, vs, 2)
        res = O.rollout_scores(st.theta, st.theta_dot, u, c.sched.dts, arm7, w3, np.eye(3), g["goal"][i], False,
                               cfg["gamma"], 1.0, provider="oracle", spheres=np.zeros((0, 4)), boxes=g["boxes"],
                               keep=("terms", "decisions"))
        ref_terms = {k: g[f"term_{k}"][i] for k in O.TERMS}
        # the oracle reproduces the reference's decisions on these inputs
        np.testing.assert_array_equal(res["terms"]["envcoll"], ref_terms["envcoll"])
        ref = {"terms": ref_terms, "totals": g["totals"][i], "weights": g["weights"][i], "eps": g["eps"],
               "command": g["command"][i]}
        rep = _check_step(report, cmd, diag.bundle, ref, res["decisions"], w3, cfg, g["means_in"][i],
                          g["variances_in"][i], precision)
        if precision == "fp64":
            assert rep["envcoll_band_hits"] == 0
            np.testing.assert_allclose(c.policy.means, g["means"][i], atol=1e-6)
    print("config-3 band report:", report)


@pytest.mark.parametrize("n", [65536, 262144])
def test_config5_large_n_vs_chunked_oracle(arm7, surrogate_state, n):
    from paper_2104_13542_b200 import configs

    c = configs.make_controller(2, particles=n, keep_bundle=True)  # FP32, as `bench.py --workload c5`
    eps = c._fixed_eps
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = n
    w2 = configs.make_weights(2)
    oc = O.OracleController(arm7, w2, configs.reach_goal_rotation(), configs.REACH_GOAL_POS, True,
                            provider="learned", mlp_state=surrogate_state, eps_source=lambda: eps, chunk=8192,
                            keep=("terms", "decisions"), **kw)
    st = configs.start_state()
    report = []
    for step in range(2):
        means_in, var_in = oc.means.copy(), oc.variances.copy()
        cmd, diag = c.control_step(st)
        assert diag.fallback == ""
        ocmd = oc.step(st.theta, st.theta_dot)
        r = oc.last
        ref = {"terms": r["terms"], "totals": r["totals"], "weights": r["weights"], "eps": eps, "command": ocmd}
        _check_step(report, cmd, diag.bundle, ref, r["decisions"], w2, kw, means_in, var_in, "fp32")
        # the next step from the oracle's policy: every step compares arithmetic, not drift
        from paper_2104_13542_b200.policy import PER_JOINT, PolicyParams

        c.policy = PolicyParams(means=oc.means, variances=oc.variances, mode=PER_JOINT,
                                tail_variance=kw["sigma0_sq"])
        st.theta_dot = st.theta_dot + 0.05 * ocmd
        st.theta = st.theta + 0.05 * st.theta_dot
    print(f"config-5 N={n} band report:", report)
