"""Pin the CPU oracle (oracle/mppi_oracle.py) to the reference's own outputs.

The golden fixtures were produced by running jointmpc itself
(tests/golden/make_golden.py). If these pass, the oracle is a faithful
restatement and can be trusted as the checker of the CUDA path.
"""

from fractions import Fraction

import numpy as np
import pytest

from conftest import golden
from oracle import mppi_oracle as O
from paper_2104_13542_b200 import configs


def test_halton_bit_exact():
    g = golden("sampling")
    np.testing.assert_array_equal(O.halton(600, 7), g["halton"])


def test_halton_known_answers():
    # sampling.py docstring / test_sampling.py:36-48
    base2 = [Fraction(v).limit_denominator(1 << 30) for v in O.halton(8, 1)[:, 0]]
    assert base2 == [Fraction(1, 2), Fraction(1, 4), Fraction(3, 4), Fraction(1, 8),
                     Fraction(5, 8), Fraction(3, 8), Fraction(7, 8), Fraction(1, 16)]
    base3 = [Fraction(v).limit_denominator(1 << 30) for v in O.halton(8, 2)[:, 1]]
    assert base3 == [Fraction(1, 3), Fraction(2, 3), Fraction(1, 9), Fraction(4, 9),
                     Fraction(7, 9), Fraction(2, 9), Fraction(5, 9), Fraction(8, 9)]


def test_acklam_matches_reference():
    g = golden("sampling")
    np.testing.assert_allclose(O.acklam(g["gauss_p"]), g["gauss"], rtol=0, atol=1e-15)


def test_bspline_basis_matches_reference():
    g = golden("sampling")
    np.testing.assert_allclose(O.bspline_design(30, 5, 3), g["basis_30_5"], atol=1e-15)
    np.testing.assert_allclose(O.bspline_design(24, 6, 3), g["basis_24_6"], atol=1e-15)
    np.testing.assert_allclose(O.bspline_design(7, 4, 2), g["basis_7_4_2"], atol=1e-15)
    assert O.knot_count(30) == 5 and O.knot_count(8) == 4


def test_smoothing_matches_reference():
    g = golden("sampling")
    np.testing.assert_allclose(O.smooth(g["comb_in"], "comb", 12), g["comb_out"], atol=1e-15)
    np.testing.assert_allclose(O.smooth(g["spline_knots"], "bspline", 30), g["spline_out"], atol=1e-14)


def test_fixed_halton_block_matches_controller():
    g = golden("sampling")
    eps = O.fixed_halton_block(48, 30, 7)
    np.testing.assert_allclose(eps, g["fixed_eps_arm7_48"], atol=1e-13)
    np.testing.assert_allclose(eps.mean(axis=0), 0.0, atol=1e-12)


@pytest.mark.parametrize("name", ["arm7", "planar2", "slider1"])
def test_kinematics_match_reference(name, request):
    g = golden("kinematics")
    ch = request.getfixturevalue(name)
    q = g[f"{name}_q"]
    rot, trans = O.link_poses(q, ch)
    np.testing.assert_allclose(rot, g[f"{name}_rot"], atol=1e-13)
    np.testing.assert_allclose(trans, g[f"{name}_trans"], atol=1e-13)
    J = O.geometric_jacobian(rot, trans, ch)
    np.testing.assert_allclose(J, g[f"{name}_J"], atol=1e-13)
    np.testing.assert_allclose(O.manipulability(J, ch.task_dim), g[f"{name}_manip"], atol=1e-12)
    np.testing.assert_allclose(O.capsule_self_collision(rot, trans, ch), g[f"{name}_self"], atol=1e-12)


def test_env_collision_matches_reference(arm7):
    g = golden("kinematics")
    rot, trans = O.link_poses(g["env_q"], arm7)
    hit = O.first_obstacle_hit(rot, trans, arm7, g["env_spheres"], g["env_boxes"])
    np.testing.assert_array_equal(hit, g["env_hit"])
    hit_b = O.first_obstacle_hit(rot, trans, arm7, np.zeros((0, 4)), g["env_boxes"])
    np.testing.assert_array_equal(hit_b, g["env_hit_boxes_only"])
    assert (g["env_hit"] >= 0).any() and (g["env_hit"] < 0).any()  # both branches exercised


def test_integration_matches_reference():
    g = golden("kinematics")
    pos, vel = O.euler(g["int_u"], g["int_dts"], g["int_th0"], g["int_thd0"])
    np.testing.assert_array_equal(pos, g["int_pos"])
    np.testing.assert_array_equal(vel, g["int_vel"])


def test_mlp_matches_reference(surrogate_state):
    g = golden("mlp")
    np.testing.assert_allclose(O.mlp_distance(g["q"], surrogate_state), g["dist"], atol=1e-12)


def test_policy_updates_match_reference():
    g = golden("policy")
    w = O.weights_from_totals(g["totals"], 0.7)
    np.testing.assert_allclose(w, g["weights"], atol=1e-15)
    mu, var = O.blend_policy(g["means0"], g["var0"], g["controls"], w, 0.9, 0.5, 0.05, 2.0)
    np.testing.assert_allclose(mu, g["means1"], atol=1e-13)
    np.testing.assert_allclose(var, g["var1"], atol=1e-13)
    mu_i, var_i = O.blend_policy(np.zeros((6, 3)), np.full(6, 0.8), g["controls"], w, 0.7, 0.4, 0.05, 2.0,
                                 isotropic=True)
    np.testing.assert_allclose(mu_i, g["iso_means"], atol=1e-13)
    np.testing.assert_allclose(var_i, g["iso_var"], atol=1e-13)
    sm, sv = O.shifted(g["means1"], g["var1"], 0.25, 0.8)
    np.testing.assert_array_equal(sm, g["shift_means"])
    np.testing.assert_array_equal(sv, g["shift_var"])


def _oracle_controller(arm7, config, particles=500, **kw):
    w = configs.make_weights(config)
    provider = "learned" if config == 2 else None
    mlp_state = None
    if config == 2:
        from paper_2104_13542_b200.surrogate import ARM7_SURROGATE

        with np.load(ARM7_SURROGATE) as z:
            mlp_state = {k: z[k] for k in z.files if k.startswith(("W", "b"))}
    ckw = dict(configs.CONTROLLER_KW)
    ckw.pop("seed")
    ckw["particles"] = particles
    ckw.update(kw)
    return O.OracleController(arm7, w, configs.reach_goal_rotation(), configs.REACH_GOAL_POS, True,
                              provider=provider, mlp_state=mlp_state, **ckw)


@pytest.mark.parametrize("fixture,config,kw", [
    ("step_c1", 1, {}),
    ("step_c2", 2, {}),
    ("step_c2_iso_k2", 2, dict(particles=256, isotropic=True, iterations=2)),
])
def test_control_steps_match_reference(arm7, fixture, config, kw):
    g = golden(fixture)
    c = _oracle_controller(arm7, config, **kw)
    first = None
    for i in range(g["command"].shape[0]):
        cmd = c.step(g["theta"][i], g["theta_dot"][i])
        if i == 0:
            first = c.last
            np.testing.assert_allclose(first["eps"], g["eps"], atol=1e-12)
        np.testing.assert_allclose(cmd, g["command"][i], atol=1e-9)
        np.testing.assert_allclose(c.means, g["means"][i], atol=1e-9)
        np.testing.assert_allclose(c.variances, g["variances"][i], atol=1e-9)
        assert c.last["best_cost"] == pytest.approx(g["best_cost"][i], rel=1e-12)
        assert c.last["mean_cost"] == pytest.approx(g["mean_cost"][i], rel=1e-12)
    if "iterations" not in kw:  # the bundle is the first step's only iteration
        np.testing.assert_allclose(first["totals"], g["totals"], rtol=1e-12)
        np.testing.assert_allclose(first["weights"], g["weights"], atol=1e-12)
        np.testing.assert_allclose(first["step_costs"], g["step_costs"], rtol=1e-11, atol=1e-11)
        for name in O.TERMS:
            np.testing.assert_allclose(first["terms"][name], g[f"term_{name}"], rtol=1e-11, atol=1e-11)
        np.testing.assert_allclose(first["positions"][:16], g["positions_head"], atol=1e-13)
        np.testing.assert_allclose(first["accelerations"][:16], g["controls_head"], atol=1e-13)


def test_world_step_matches_reference(arm7):
    g = golden("step_world")
    w = configs.make_weights(3)
    ckw = dict(configs.CONTROLLER_KW)
    ckw.pop("seed")
    ckw["particles"] = 128
    c = O.OracleController(arm7, w, np.eye(3), g["goal"], False, spheres=g["spheres"], boxes=g["boxes"],
                           provider="oracle", **ckw)
    cmd = c.step(configs.REACH_START, np.zeros(7))
    np.testing.assert_array_equal(c.last["terms"]["envcoll"], g["term_envcoll"])
    np.testing.assert_allclose(c.last["totals"], g["totals"], rtol=1e-12)
    np.testing.assert_allclose(cmd, g["command"], atol=1e-9)
    np.testing.assert_allclose(c.variances, g["variances"], atol=1e-9)
    assert g["term_envcoll"].any()  # the world is actually hit


def test_obstacle_margin_decides_like_first_hit(arm7):
    """The decision-band margin (tests/band.py) is < 0 exactly where the
    reference reports a hit (kinematics golden: its own hit indices)."""
    g = golden("kinematics")
    rot, trans = O.link_poses(g["env_q"], arm7)
    m = O.obstacle_margin(rot, trans, arm7, g["env_spheres"], g["env_boxes"])
    np.testing.assert_array_equal(m < 0, g["env_hit"] >= 0)
    m = O.obstacle_margin(rot, trans, arm7, np.zeros((0, 4)), g["env_boxes"])
    np.testing.assert_array_equal(m < 0, g["env_hit_boxes_only"] >= 0)


def test_chunked_rollout_scores_equal_unchunked(arm7, surrogate_state):
    """The chunked oracle driver for N >= 65k (SURVEY §8(c) scale limits):
    rows are independent, so per-chunk evaluation + one full-N update equals
    the one-shot evaluation."""
    rng = np.random.default_rng(3)
    u = rng.normal(scale=0.7, size=(300, 30, 7))
    dts = O.dt_schedule(30, 0.05, "two_phase")
    args = (configs.REACH_START, np.zeros(7), u, dts, arm7, configs.make_weights(2), configs.reach_goal_rotation(),
            configs.REACH_GOAL_POS, True, 0.99, 1.0)
    kw = dict(provider="learned", mlp_state=surrogate_state)
    one = O.rollout_scores(*args, keep=("terms", "decisions"), **kw)
    chunked = O.rollout_scores(*args, chunk=128, keep=("terms", "decisions"), **kw)
    np.testing.assert_allclose(chunked["totals"], one["totals"], rtol=1e-14)
    for k in O.TERMS:
        np.testing.assert_allclose(chunked["terms"][k], one["terms"][k], rtol=1e-14, atol=0)
    np.testing.assert_array_equal(chunked["decisions"]["manip"], one["decisions"]["manip"])


def test_tracking_step_matches_reference(arm7):
    """Config 3 at the benched shape (configs.tracking_problem boxes, N=500):
    the oracle's rollout of the reference's first step equals the reference's
    terms and totals (tests/golden/step_c3.npz)."""
    g = golden("step_c3")
    kw = configs.CONTROLLER_KW
    ms, vs = O.shifted(g["means_in"][0], g["variances_in"][0], 0.0, kw["sigma0_sq"])
    u = O.shape_controls(g["eps"], ms, vs, 2)
    dts = O.dt_schedule(30, 0.05, "two_phase")
    res = O.rollout_scores(g["theta"][0], g["theta_dot"][0], u, dts, arm7, configs.make_weights(3), np.eye(3),
                           g["goal"][0], False, kw["gamma"], 1.0, provider="oracle", spheres=np.zeros((0, 4)),
                           boxes=g["boxes"], keep=("terms", "decisions"))
    for k in O.TERMS:
        np.testing.assert_allclose(res["terms"][k], g[f"term_{k}"][0], rtol=1e-10, atol=1e-10, err_msg=k)
    np.testing.assert_allclose(res["totals"], g["totals"][0], rtol=1e-11)
    env = res["decisions"]["env"]
    np.testing.assert_array_equal(env < 0, g["term_envcoll"][0] > 0)
    w = O.weights_from_totals(res["totals"], kw["beta"])
    mu, _ = O.blend_policy(ms, vs, u, w, kw["alpha_mu"], kw["alpha_sigma"], kw["sigma_sq_min"], kw["sigma0_sq"])
    np.testing.assert_allclose(mu[0], g["command"][0], atol=1e-10)
