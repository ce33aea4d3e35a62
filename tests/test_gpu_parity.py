"""CUDA path vs the reference (golden fixtures) and the pinned oracle.

Tolerances (stated per north_star):
  * float64 seam / FP64 plans: 1e-9 absolute or tighter;
  * FP32 fused path: controls 1e-6, positions/velocities 1e-5 abs, step costs
    1e-4 relative, totals such that |d(c_i - c_min)| <= 1e-3*beta for every
    particle with weight > 1e-6, weights 1e-3 abs, policy / command 1e-3 abs.
"""

import numpy as np
import pytest

from conftest import golden, random_q
from oracle import mppi_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _native():
    from paper_2104_13542_b200 import _native as N

    N.load_library()
    N.require_device()


# ---------------------------------------------------------------- operator seam (float64)
@pytest.mark.parametrize("name", ["arm7", "planar2", "slider1"])
def test_seam_kinematics(name, request):
    from paper_2104_13542_b200 import kernels as K

    g = golden("kinematics")
    ch = request.getfixturevalue(name)
    q = g[f"{name}_q"]
    rot, trans = K.fk_batch(q, ch.axes, ch.origin_rot, ch.origin_trans, ch.jtype)
    np.testing.assert_allclose(rot, g[f"{name}_rot"], atol=1e-12)
    np.testing.assert_allclose(trans, g[f"{name}_trans"], atol=1e-12)
    J = K.jacobian_batch(q, rot, trans, ch.axes, ch.jtype)
    np.testing.assert_allclose(J, g[f"{name}_J"], atol=1e-12)
    np.testing.assert_allclose(K.manip_batch(J, ch.task_dim), g[f"{name}_manip"], atol=1e-11)
    s = K.self_collision_batch(rot, trans, ch.cap_p0, ch.cap_p1, ch.cap_r, ch.cap_link, ch.pair_a, ch.pair_b)
    np.testing.assert_allclose(s, g[f"{name}_self"], atol=1e-11)


def test_seam_env_collision(arm7):
    from paper_2104_13542_b200 import kernels as K

    g = golden("kinematics")
    rot, trans = K.fk_batch(g["env_q"], arm7.axes, arm7.origin_rot, arm7.origin_trans, arm7.jtype)
    hit = K.env_collision_batch(rot, trans, arm7.cap_p0, arm7.cap_p1, arm7.cap_r, arm7.cap_link,
                                g["env_spheres"], g["env_boxes"])
    np.testing.assert_array_equal(hit, g["env_hit"])
    hit = K.env_collision_batch(rot, trans, arm7.cap_p0, arm7.cap_p1, arm7.cap_r, arm7.cap_link,
                                np.zeros((0, 4)), g["env_boxes"])
    np.testing.assert_array_equal(hit, g["env_hit_boxes_only"])


def test_seam_integrate():
    from paper_2104_13542_b200 import kernels as K

    g = golden("kinematics")
    pos, vel = K.integrate_batch(g["int_u"], g["int_dts"], g["int_th0"], g["int_thd0"])
    np.testing.assert_allclose(pos, g["int_pos"], atol=1e-14)
    np.testing.assert_allclose(vel, g["int_vel"], atol=1e-14)


def test_seam_empty_batch(arm7):
    from paper_2104_13542_b200 import kernels as K

    rot, trans = K.fk_batch(np.zeros((0, 7)), arm7.axes, arm7.origin_rot, arm7.origin_trans, arm7.jtype)
    assert rot.shape == (0, 7, 3, 3) and trans.shape == (0, 7, 3)


# ---------------------------------------------------------------- sampling / policy free functions
def test_sampling_functions():
    from paper_2104_13542_b200 import sampling as S

    g = golden("sampling")
    np.testing.assert_array_equal(S.halton_points(600, 7), g["halton"])  # bit-exact
    np.testing.assert_allclose(S.gaussianize(g["gauss_p"]), g["gauss"], rtol=1e-12, atol=1e-12)  # CUDA log vs glibc: ulps
    np.testing.assert_allclose(S.bspline_basis(30, 5, 3), g["basis_30_5"], atol=1e-15)
    np.testing.assert_allclose(S.bspline_basis(24, 6, 3), g["basis_24_6"], atol=1e-15)
    np.testing.assert_allclose(S.bspline_basis(7, 4, 2), g["basis_7_4_2"], atol=1e-15)
    np.testing.assert_allclose(S.smooth_sequences(g["comb_in"], S.SmoothingSpec(mode="comb"), 12),
                               g["comb_out"], atol=1e-14)
    np.testing.assert_allclose(
        S.smooth_sequences(g["spline_knots"], S.SmoothingSpec(mode="bspline", knots_per_horizon=5), 30),
        g["spline_out"], atol=1e-14)
    with pytest.raises(S.ContractError):
        S.gaussianize(np.array([1.0]))


def test_build_control_batch_rows(rng):
    from paper_2104_13542_b200.policy import make_policy
    from paper_2104_13542_b200.sampling import build_control_batch

    pol = make_policy(8, 3, 4.0)
    pol.means[:] = rng.standard_normal((8, 3))
    eps = rng.standard_normal((6, 8, 3))
    b = build_control_batch(eps, pol, null_count=2)
    np.testing.assert_array_equal(b.controls[:2], 0.0)
    np.testing.assert_array_equal(b.controls[2], pol.means)
    np.testing.assert_allclose(b.controls[3:], pol.means[None] + 2.0 * eps[3:], atol=1e-14)


def test_policy_functions():
    from paper_2104_13542_b200.policy import (PolicyParams, UpdateConfig, make_policy, particle_weights,
                                              update_covariance, update_mean)

    g = golden("policy")
    w = particle_weights(g["totals"], 0.7)
    np.testing.assert_allclose(w, g["weights"], atol=1e-15)
    pol = PolicyParams(means=g["means0"], variances=g["var0"], mode="per_joint_diagonal", tail_variance=0.8)
    cfg = UpdateConfig(sigma_sq_min=0.05, sigma_sq_max=2.0)
    m1 = update_mean(pol, g["controls"], w, 0.9)
    c1 = update_covariance(m1, g["controls"], w, 0.5, cfg)
    np.testing.assert_allclose(m1.means, g["means1"], atol=1e-13)
    np.testing.assert_allclose(c1.variances, g["var1"], atol=1e-13)
    iso = make_policy(6, 3, 0.8, mode="isotropic")
    im = update_mean(iso, g["controls"], w, 0.7)
    ic = update_covariance(im, g["controls"], w, 0.4, cfg)
    np.testing.assert_allclose(ic.variances, g["iso_var"], atol=1e-13)
    with pytest.raises(Exception):
        particle_weights(np.full(4, np.inf), 1.0)


# ---------------------------------------------------------------- learned collision
def test_mlp_forward_matches_reference():
    from paper_2104_13542_b200.surrogate import load_arm7_surrogate

    g = golden("mlp")
    d = load_arm7_surrogate().distance(g["q"])
    # FP16-split x3 tensor-core product, FP32 accumulate (~3.5e-7 m)
    err = np.abs(d - g["dist"]).max()
    print(f"mlp max |d - ref| = {err:.3e}")
    assert err < 2e-6, err
    assert np.array_equal(d > 0, g["dist"] > 0) or np.abs(g["dist"][(d > 0) != (g["dist"] > 0)]).max() < 2e-6


# ---------------------------------------------------------------- fused controller
def _weight_safe(tot, ref_tot, ref_w, beta, tol):
    """|d(c_i - c_min)| <= tol*beta for every particle with ref weight > 1e-6."""
    ok = np.isfinite(ref_tot)
    assert np.array_equal(np.isfinite(tot), ok)
    rel_gpu = tot[ok] - tot[ok].min()
    rel_ref = ref_tot[ok] - ref_tot[ok].min()
    sel = ref_w[ok] > 1e-6
    err = np.abs(rel_gpu - rel_ref)[sel].max()
    assert err <= tol * beta, err


@pytest.mark.parametrize("config", [1, 2])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_control_step_matches_reference(config, precision):
    from paper_2104_13542_b200 import configs

    g = golden(f"step_c{config}")
    c = configs.make_controller(config, precision=precision, keep_bundle=True)
    np.testing.assert_allclose(c._fixed_eps, g["eps"], atol=1e-12)  # FP64 device init
    exact = precision == "fp64"
    for i in range(g["command"].shape[0]):
        st = configs.start_state()
        st.theta[:] = g["theta"][i]
        st.theta_dot[:] = g["theta_dot"][i]
        cmd, diag = c.control_step(st)
        assert diag.fallback == ""
        tol = 1e-7 if exact else 1e-3
        if config == 2:
            tol = 1e-4 if exact else 1e-3  # tensor-core MLP
        np.testing.assert_allclose(cmd, g["command"][i], atol=tol)
        pol = c.policy
        np.testing.assert_allclose(pol.means, g["means"][i], atol=tol)
        np.testing.assert_allclose(pol.variances, g["variances"][i], atol=tol)
        assert diag.best_cost == pytest.approx(g["best_cost"][i], rel=1e-5)
        if i == 0:
            b = diag.bundle
            np.testing.assert_allclose(b.accelerations[:16], g["controls_head"], atol=1e-6)
            np.testing.assert_allclose(b.positions[:16], g["positions_head"], atol=1e-5)
            np.testing.assert_allclose(b.velocities[:16], g["velocities_head"], atol=1e-5)
            np.testing.assert_allclose(b.step_costs, g["step_costs"], rtol=1e-4, atol=1e-3)
            for name in ("pose", "stop", "joint", "manip", "selfcoll", "envcoll"):
                np.testing.assert_allclose(b.term_breakdown[name], g[f"term_{name}"], rtol=1e-4, atol=2e-4,
                                           err_msg=name)
            _weight_safe(b.total_per_particle, g["totals"], g["weights"], 1.0, 1e-3 if not exact else 1e-6)
            np.testing.assert_allclose(b.weights, g["weights"], atol=1e-3)


def test_isotropic_two_iterations_matches_reference():
    from paper_2104_13542_b200 import configs

    g = golden("step_c2_iso_k2")
    c = configs.make_controller(2, particles=256, policy_mode="isotropic", iterations=2, precision="fp64")
    for i in range(g["command"].shape[0]):
        st = configs.start_state()
        st.theta[:] = g["theta"][i]
        st.theta_dot[:] = g["theta_dot"][i]
        cmd, _ = c.control_step(st)
        np.testing.assert_allclose(cmd, g["command"][i], atol=1e-4)
        np.testing.assert_allclose(c.policy.variances, g["variances"][i], atol=1e-4)


def test_evaluate_rollouts_vs_oracle(arm7, rng):
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.costs import CostStack
    from paper_2104_13542_b200.rollout import evaluate_rollouts, make_dt_schedule, zero_state

    w = configs.make_weights(2)
    w = type(w)(**{**configs.WEIGHTS[2], "alpha_coll": 1000.0})
    stack = CostStack(chain=arm7, weights=w, goal=configs.make_goal(2))  # oracle self collision
    sched = make_dt_schedule(30, 0.05, "two_phase")
    u = rng.standard_normal((300, 30, 7)) * 2.0
    x0 = zero_state(7)
    x0.theta[:] = configs.REACH_START
    ref = O.rollout_scores(x0.theta, x0.theta_dot, u, sched.dts, arm7, w, configs.reach_goal_rotation(),
                           configs.REACH_GOAL_POS, True, 0.99, 1.0, provider="oracle")
    for precision, tol in ((1, 1e-9), (0, 1e-4)):
        b = evaluate_rollouts(x0, u, arm7, stack, sched, gamma=0.99, precision=precision)
        np.testing.assert_allclose(b.positions, ref["positions"], atol=1e-5 if precision == 0 else 1e-12)
        np.testing.assert_allclose(b.step_costs, ref["step_costs"], rtol=tol, atol=tol)
        for name in O.TERMS:
            np.testing.assert_allclose(b.term_breakdown[name], ref["terms"][name], rtol=tol, atol=tol,
                                       err_msg=name)
        np.testing.assert_allclose(b.total_per_particle, ref["totals"], rtol=tol)


def test_evaluate_rollouts_quarantine_and_contract(arm7, rng):
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.costs import CostStack
    from paper_2104_13542_b200.errors import ContractError
    from paper_2104_13542_b200.rollout import evaluate_rollouts, make_dt_schedule, zero_state

    stack = CostStack(chain=arm7, weights=configs.make_weights(1), goal=configs.make_goal(1))
    sched = make_dt_schedule(12, 0.05, "uniform")
    u = rng.standard_normal((40, 12, 7))
    u[5, 3, 2] = np.nan
    with pytest.raises(ContractError, match="particle 5"):
        evaluate_rollouts(zero_state(7), u, arm7, stack, sched)
    u[5, 3, 2] = 1e200  # finite control, overflowing state -> quarantined row
    b = evaluate_rollouts(zero_state(7), u, arm7, stack, sched)
    assert not np.isfinite(b.total_per_particle[5])
    np.testing.assert_array_equal(b.step_costs[5], 0.0)
    assert np.isfinite(np.delete(b.total_per_particle, 5)).all()


def test_cost_stack_evaluate_planar(planar2):
    from paper_2104_13542_b200.costs import CostStack, CostWeights, goal_at_position
    from paper_2104_13542_b200.rollout import make_dt_schedule
    from paper_2104_13542_b200.simworld import world_from_dict

    world = world_from_dict({"obstacles": [{"type": "disc", "center": [2.0, 0.0], "radius": 0.3}],
                             "bounds": {"min": [-3, -3], "max": [3, 3]}})
    stack = CostStack(chain=planar2, weights=CostWeights(), goal=goal_at_position(np.zeros(3)), world=world)
    sched = make_dt_schedule(2, 0.05, "uniform")
    hit_q = np.zeros((1, 2, 2))
    free_q = np.full((1, 2, 2), 1.5)
    _, t_hit = stack.evaluate(hit_q, np.zeros_like(hit_q), sched)
    _, t_free = stack.evaluate(free_q, np.zeros_like(free_q), sched)
    assert t_hit["envcoll"].max() == 1.0 and t_free["envcoll"].max() == 0.0
    # manipulability closed form |sin q2| (test_costs.py:111-130)
    qs = np.array([[[0.0, q2] for q2 in np.linspace(0.01, 0.4, 20)]])
    stack2 = CostStack(chain=planar2, weights=CostWeights(k_m=0.5, alpha_coll=0.0), goal=goal_at_position(np.zeros(3)))
    _, terms = stack2.evaluate(qs, np.zeros_like(qs), __import__(
        "paper_2104_13542_b200.rollout", fromlist=["x"]).make_dt_schedule(20, 0.05, "uniform"))
    np.testing.assert_allclose(terms["manip"][0], 1.0 - np.abs(np.sin(qs[0, :, 1])), atol=1e-9)


def test_fallback_ladder():
    from paper_2104_13542_b200 import configs

    c = configs.make_controller(1, particles=64)
    st = configs.start_state()
    cmd0, d0 = c.control_step(st)
    assert d0.fallback == ""
    pol = c.policy
    pol.means[:] = np.nan  # poisons every shaped control -> ContractError on the device
    c.policy = pol
    cmd1, d1 = c.control_step(st)
    assert d1.fallback == "reissue"
    np.testing.assert_array_equal(cmd1, cmd0)
    cmd2, d2 = c.control_step(st)
    assert d2.fallback == "brake"
    np.testing.assert_array_equal(cmd2, np.zeros(7))


def test_world_step_voxel_grid(arm7):
    """A seed-3 voxel world plus a sphere, N=128, FP64 and FP32, under the
    decision-band rule (tests/band.py): out-of-band env-collision flips fail,
    band hits are substituted and counted."""
    from band import apply_bands, corrected_command, weight_safe
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.controller import Controller
    from paper_2104_13542_b200.costs import goal_at_position
    from paper_2104_13542_b200.simworld import voxel_world

    g = golden("step_world")
    world = voxel_world(g["occupancy"], origin=np.full(3, -1.0), voxel=2.0 / 64, spheres=g["spheres"])
    np.testing.assert_allclose(np.sort(world.boxes, axis=0), np.sort(g["boxes"], axis=0), atol=1e-12)
    kw = dict(configs.CONTROLLER_KW)
    kw["particles"] = 128
    w3 = configs.make_weights(3)
    for precision in ("fp64", "fp32"):
        c = Controller(arm7, goal_at_position(g["goal"]), weights=w3, world=world,
                       keep_bundle=True, precision=precision, **kw)
        cmd, diag = c.control_step(configs.start_state())
        b = diag.bundle
        st = configs.start_state()
        ms, vs = O.shifted(np.zeros((30, 7)), np.full((30, 7), kw["sigma0_sq"]), 0.0, kw["sigma0_sq"])
        u = O.shape_controls(c._fixed_eps, ms, vs, 2)
        res = O.rollout_scores(st.theta, st.theta_dot, u, c.sched.dts, arm7, w3, np.eye(3), g["goal"], False,
                               kw["gamma"], 1.0, provider="oracle", spheres=g["spheres"], boxes=g["boxes"],
                               keep=("terms", "decisions"))
        np.testing.assert_array_equal(res["terms"]["envcoll"], g["term_envcoll"])
        ref_terms = {k: g[f"term_{k}"] for k in ("envcoll", "stop", "pose")}
        _, dtot, rep = apply_bands(b.term_breakdown, ref_terms, res["decisions"], w3, kw["gamma"], 1.0)
        if precision == "fp64":
            assert rep["envcoll_band_hits"] == 0
        tot = b.total_per_particle + dtot
        ref_w = O.weights_from_totals(g["totals"], kw["beta"])
        weight_safe(tot, g["totals"], ref_w, kw["beta"], 1e-3 if precision == "fp32" else 1e-6)
        fixed, _, _, _ = corrected_command(b.accelerations, tot, ms, vs, beta=kw["beta"], alpha_mu=kw["alpha_mu"],
                                           alpha_sigma=kw["alpha_sigma"], smin=kw["sigma_sq_min"],
                                           smax=kw["sigma0_sq"])
        np.testing.assert_allclose(fixed, g["command"], atol=1e-3)
        if rep["envcoll_band_hits"] == 0:
            np.testing.assert_allclose(cmd, g["command"], atol=1e-3)
        print(precision, "band report:", rep)


def test_pseudorandom_injected_noise_vs_oracle(arm7, rng):
    """Pseudorandom parity: the same eps injected into the device plan and the oracle."""
    from paper_2104_13542_b200 import configs

    c = configs.make_controller(1, particles=200, precision="fp64")
    eps = rng.standard_normal((200, 30, 7))
    c.set_perturbations(eps)
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = 200
    oc = O.OracleController(arm7, configs.make_weights(1), configs.reach_goal_rotation(), configs.REACH_GOAL_POS,
                            True, eps_source=lambda: eps, **kw)
    st = configs.start_state()
    for _ in range(3):
        cmd, _ = c.control_step(st)
        ocmd = oc.step(st.theta, st.theta_dot)
        np.testing.assert_allclose(cmd, ocmd, atol=1e-7)


@pytest.mark.parametrize("particles", [1500, 2048, 2100, 8192, 9000])
def test_many_statistics_blocks_vs_oracle(arm7, rng, particles):
    """Up to 2048 particles one 16-CTA cluster holds the instance (94 and 128
    particles per CTA here, beyond the 32 rows each thread preloads); up to
    8192, clusters of 16 CTAs of 32 particles each reduce to one record and a
    finalize kernel combines them (5 and 16 clusters here); beyond, 32
    particles per block with a record combine in two levels (282 blocks here:
    18 groups)."""
    from paper_2104_13542_b200 import configs

    c = configs.make_controller(1, particles=particles, precision="fp64")
    eps = rng.standard_normal((particles, 30, 7))
    c.set_perturbations(eps)
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = particles
    oc = O.OracleController(arm7, configs.make_weights(1), configs.reach_goal_rotation(), configs.REACH_GOAL_POS,
                            True, eps_source=lambda: eps, **kw)
    st = configs.start_state()
    for _ in range(2):
        cmd, diag = c.control_step(st)
        ocmd = oc.step(st.theta, st.theta_dot)
        np.testing.assert_allclose(cmd, ocmd, atol=1e-7)
        np.testing.assert_allclose(c.policy.variances, oc.variances, atol=1e-7)


def test_pseudorandom_generator_runs_and_is_seeded():
    from paper_2104_13542_b200 import configs

    outs = []
    for seed in (3, 3, 4):
        c = configs.make_controller(1, particles=128, generator="pseudorandom", seed=seed)
        cmd, d = c.control_step(configs.start_state())
        assert d.fallback == ""
        outs.append(cmd)
    np.testing.assert_array_equal(outs[0], outs[1])
    assert not np.array_equal(outs[0], outs[2])


def test_cuda_backend_in_unmodified_reference():
    """INTEGRATION.md tier 2: install the six seam kernels into the reference's
    own kernel table (oracle/_ref, unmodified) and run ITS Controller."""
    import sys
    from pathlib import Path

    ref_root = Path(__file__).resolve().parents[1] / "oracle" / "_ref"
    if not (ref_root / "jointmpc").exists():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, str(ref_root))
    import jointmpc.kernels as RK
    from jointmpc.controller import Controller as RefController
    from jointmpc.costs import CostWeights as RefWeights
    from jointmpc.costs import goal_at_position as ref_goal
    from jointmpc.kinematics import load_chain as ref_load
    from jointmpc.rollout import JointState as RefState

    from paper_2104_13542_b200 import kernels as cuda_backend

    saved = cuda_backend.install_into(RK)
    try:
        chain = ref_load("arm7.chain")
        c = RefController(chain, ref_goal([0.4, 0.2, 0.5]), particles=64, horizon=20, weights=RefWeights(), seed=0)
        st = RefState(theta=np.array([0.0, -0.5, 0.0, -1.8, 0.0, 1.4, 0.0]), theta_dot=np.zeros(7),
                      theta_ddot=np.zeros(7))
        cmd, diag = c.control_step(st)
        assert RK.BACKEND_NAME in ("numba", "numpy")  # the table was rebound, not the module swapped
        assert RK.fk_batch is cuda_backend.fk_batch
    finally:
        for k, fn in saved.items():
            setattr(RK, k, fn)
    # the same step with the oracle (float64, same kwargs) — defaults of Controller / CostWeights
    from paper_2104_13542_b200.costs import CostWeights
    from paper_2104_13542_b200.kinematics import load_chain

    oc = O.OracleController(load_chain("arm7.chain"), CostWeights(), np.eye(3), np.array([0.4, 0.2, 0.5]), False,
                            particles=64, horizon=20, provider="oracle")
    ocmd = oc.step(st.theta, st.theta_dot)
    np.testing.assert_allclose(cmd, ocmd, atol=1e-9)


def _random_chain(d, seed):
    from paper_2104_13542_b200.kinematics import chain_from_dict

    rng = np.random.default_rng(seed)
    joints = []
    for k in range(d):
        ax = rng.standard_normal(3)
        ax /= np.linalg.norm(ax)
        joints.append({"type": "prismatic" if (k % 3 == 2) else "revolute", "axis": ax.tolist(),
                       "origin": {"xyz": (rng.standard_normal(3) * 0.2).tolist(),
                                  "rpy": (rng.standard_normal(3) * 0.5).tolist()}})
    caps = [{"link": int(l), "p0": (rng.standard_normal(3) * 0.05).tolist(),
             "p1": (rng.standard_normal(3) * 0.1).tolist(), "radius": 0.04} for l in range(d)]
    pairs = [[i, j] for i in range(d) for j in range(i + 2, d)][:8]
    return chain_from_dict({"name": f"rand{d}", "task_dim": 3, "joints": joints,
                            "limits": {"position": [[-2.0, 2.0]] * d, "velocity": [3.0] * d,
                                       "acceleration": [10.0] * d},
                            "capsules": caps, "self_collision_pairs": pairs})


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6, 7, 8])
def test_fused_rollout_generic_chains(d):
    """Every dof instantiation of the fused kernel (d = 8 exercises the
    re-orthonormalisation of jit.py:190), prismatic joints, non-identity origin
    rotations, all cost terms incl. capsules and a world, vs the oracle."""
    from paper_2104_13542_b200.costs import CostStack, CostWeights, goal_at_position
    from paper_2104_13542_b200.kinematics import Pose
    from paper_2104_13542_b200.costs import GoalSpec, FULL_POSE
    from paper_2104_13542_b200.rollout import evaluate_rollouts, make_dt_schedule, zero_state
    from paper_2104_13542_b200.simworld import world_from_dict
    from paper_2104_13542_b200 import kernels as K

    chain = _random_chain(d, 100 + d)
    rng = np.random.default_rng(d)
    q = rng.uniform(-1, 1, size=(64, d))
    rot, trans = K.fk_batch(q, chain.axes, chain.origin_rot, chain.origin_trans, chain.jtype)
    orot, otrans = O.link_poses(q, chain)
    np.testing.assert_allclose(rot, orot, atol=1e-12)
    np.testing.assert_allclose(trans, otrans, atol=1e-12)
    world = world_from_dict({"obstacles": [{"type": "sphere", "center": [0.2, 0.1, 0.3], "radius": 0.15},
                                           {"type": "box", "min": [-0.4, -0.3, 0.0], "max": [-0.1, 0.2, 0.4]}]})
    Rg = O._rodrigues(np.array([0.0, 0.0, 1.0]), np.array([0.3]))[0]
    goal = GoalSpec(target_pose=Pose(rotation=Rg, translation=np.array([0.2, -0.1, 0.3])), mode=FULL_POSE)
    w = CostWeights(alpha_stop=5.0, alpha_joint=10.0, alpha_manip=3.0, alpha_coll=10.0, k_m=0.02)
    stack = CostStack(chain=chain, weights=w, goal=goal, world=world)
    sched = make_dt_schedule(12, 0.05, "linear")
    u = rng.standard_normal((96, 12, d)) * 2.0
    x0 = zero_state(d)
    ref = O.rollout_scores(x0.theta, x0.theta_dot, u, sched.dts, chain, w, Rg, goal.target_pose.translation, True,
                           0.97, 2.0, provider="oracle" if chain.pair_a.size else None, spheres=world.spheres,
                           boxes=world.boxes)
    b = evaluate_rollouts(x0, u, chain, stack, sched, gamma=0.97, terminal_weight=2.0)  # FP64 plan
    np.testing.assert_allclose(b.positions, ref["positions"], atol=1e-12)
    for name in O.TERMS:
        np.testing.assert_allclose(b.term_breakdown[name], ref["terms"][name], rtol=1e-9, atol=1e-9, err_msg=name)
    np.testing.assert_allclose(b.total_per_particle, ref["totals"], rtol=1e-10)


@pytest.mark.parametrize("mode,horizon,iso", [("comb", 12, False), ("none", 8, True), ("bspline", 8, False)])
def test_controller_smoothing_modes_vs_oracle(planar2, mode, horizon, iso):
    """Halton set built on the device for every smoothing mode (sampling.py:240-265)
    and short horizons, planar2 (the reference's controller test chain)."""
    from paper_2104_13542_b200.controller import Controller
    from paper_2104_13542_b200.costs import CostWeights, goal_at_position
    from paper_2104_13542_b200.rollout import JointState
    from paper_2104_13542_b200.sampling import SmoothingSpec

    spec = SmoothingSpec(mode=mode)
    kw = dict(horizon=horizon, particles=24, beta=0.5, sigma0_sq=1.0, alpha_mu=0.9, alpha_sigma=0.5,
              policy_mode="isotropic" if iso else "per_joint_diagonal")
    c = Controller(planar2, goal_at_position([1.2, 0.8]), smoothing=spec, precision="fp64", seed=7, **kw)
    oc = O.OracleController(planar2, CostWeights(), np.eye(3), np.array([1.2, 0.8, 0.0]), False,
                            provider="oracle", smoothing=mode, isotropic=iso, **{k: v for k, v in kw.items()
                                                                                 if k != "policy_mode"})
    np.testing.assert_allclose(c._fixed_eps, oc.eps_source(), atol=1e-12)
    st = JointState(theta=np.array([0.3, -0.2]), theta_dot=np.zeros(2), theta_ddot=np.zeros(2))
    for _ in range(4):
        cmd, d = c.control_step(st)
        ocmd = oc.step(st.theta, st.theta_dot)
        np.testing.assert_allclose(cmd, ocmd, atol=1e-8)
        st = JointState(theta=st.theta + 0.05 * (st.theta_dot + 0.05 * cmd), theta_dot=st.theta_dot + 0.05 * cmd,
                        theta_ddot=cmd)


def test_failure_in_second_iteration_keeps_first_update():
    """iterations=2: a poisoned policy makes iteration 1 fail -> the shifted
    policy stands (controller.py:200, 224); status is re-armed for the next step."""
    from paper_2104_13542_b200 import configs

    c = configs.make_controller(1, particles=64, iterations=2, precision="fp64")
    st = configs.start_state()
    cmd0, d0 = c.control_step(st)
    assert d0.fallback == ""
    pol = c.policy
    pol.variances[3, 2] = np.nan  # NaN variance: finite-check fails on the shaped controls
    c.policy = pol
    before = c.policy
    _, d1 = c.control_step(st)
    assert d1.fallback == "reissue"
    after = c.policy
    # the failed step still shifted the policy (and changed nothing else)
    np.testing.assert_array_equal(after.means[:-1], before.means[1:])
    np.testing.assert_array_equal(after.means[-1], 0.0)
    # recovery: a healthy policy steps normally again
    from paper_2104_13542_b200.policy import make_policy

    c.policy = make_policy(30, 7, 0.5)
    _, d2 = c.control_step(st)
    assert d2.fallback == ""


@pytest.mark.gpu
def test_fused_rollout_mlp_matches_two_kernel_path(monkeypatch):
    """The opt-in fused rollout + MLP kernel (MPPI_FUSE=1, mppi_fused.cuh)
    computes exactly what rollout_kernel + mlp_tcgen05_kernel compute."""
    from paper_2104_13542_b200 import configs

    st = configs.start_state()
    outs = []
    for fuse in (False, True):
        if fuse:
            monkeypatch.setenv("MPPI_FUSE", "1")
        else:
            monkeypatch.delenv("MPPI_FUSE", raising=False)
        c = configs.make_controller(2, particles=500)
        seq = []
        for _ in range(3):
            cmd, d = c.control_step(st)
            seq.append((cmd.copy(), d.best_cost, d.mean_cost))
        outs.append((seq, c.policy.means.copy(), c.policy.variances.copy()))
    (s0, m0, v0), (s1, m1, v1) = outs
    for (c0, b0, mc0), (c1, b1, mc1) in zip(s0, s1):
        np.testing.assert_array_equal(c0, c1)
        assert b0 == b1 and mc0 == mc1
    np.testing.assert_array_equal(m0, m1)
    np.testing.assert_array_equal(v0, v1)


def test_state_parameter_reaches_both_step_graphs():
    """The joint state travels as a rollout kernel parameter of the captured
    step graph; the instrumented copy (profile_stages(2)) is a second graph
    with its own nodes. Alternating between them over a moving state must give
    the commands of a controller that only ever used the lean graph."""
    from paper_2104_13542_b200 import configs

    a = configs.make_controller(2, particles=256)
    b = configs.make_controller(2, particles=256)
    st = configs.start_state()
    for i in range(6):
        st.theta = configs.start_state().theta + 0.02 * i
        st.theta_dot = np.full(7, 0.01 * i)
        a.profile_stages(2 if i % 2 else 0)
        ca, _ = a.control_step(st)
        cb, _ = b.control_step(st)
        np.testing.assert_array_equal(ca, cb)


@pytest.mark.gpu
@pytest.mark.parametrize("null_count", [0, 1, 5, 40])
@pytest.mark.parametrize("keep_bundle", [False, True])
def test_null_rows_any_count_vs_oracle(null_count, keep_bundle):
    """The null (u = 0) and mean (u = mu) rows of sampling.py:283-285 at
    counts other than the default 2, including 40 (they span two statistics
    CTAs of 32 particles): the lean cluster kernel patches their deviations
    in the CTAs that hold them (mppi_kernels.cuh), the bundle path selects
    per row. FP64 plan, config 1, three closed-loop steps vs the oracle."""
    from oracle import mppi_oracle as O
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.kinematics import load_chain

    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["null_count"] = null_count
    c = configs.make_controller(1, precision="fp64", keep_bundle=keep_bundle, null_count=null_count)
    oc = O.OracleController(load_chain("arm7.chain"), configs.make_weights(1), configs.reach_goal_rotation(),
                            configs.REACH_GOAL_POS, True, **kw)
    st = configs.start_state()
    for _ in range(3):
        cmd, diag = c.control_step(st)
        ocmd = oc.step(st.theta, st.theta_dot)
        assert diag.fallback == ""
        np.testing.assert_allclose(cmd, ocmd, atol=1e-7)
        np.testing.assert_allclose(c.policy.means, oc.means, atol=1e-7)
        np.testing.assert_allclose(c.policy.variances, oc.variances, atol=1e-7)
        assert diag.best_cost == pytest.approx(oc.last["best_cost"], rel=1e-9)
