"""The closed-loop episode on the device (mppi_episode, controller.run_episode)
against the reference's own run_episode (tests/golden/episode_*.npz) and
against this package's host loop (same kernels, one round trip per step).

Closed loops amplify per-step differences, so the reference comparisons use
short episodes: FP64 plans must track the reference to 1e-6 on states and
commands over 12 steps; the FP32 plan of config 2 to 2e-3 over 6 steps.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

TERMS = ("pose", "stop", "joint", "manip", "selfcoll", "envcoll")


def _script(g):
    from paper_2104_13542_b200.simworld import TargetScript

    return TargetScript(times=g["script_times"], positions=g["script_positions"],
                        interpolation=str(g["script_interp"]), mode=str(g["script_mode"]))


def _check_log(lg, g, tol_state, tol_cmd, tol_cost):
    n = int(g["steps"])
    assert lg.steps == n and lg.aborted == bool(g["aborted"])
    np.testing.assert_array_equal(lg.t, g["t"])
    np.testing.assert_allclose(lg.goal, g["goal"], atol=1e-15)
    np.testing.assert_allclose(lg.goal_rotations, g["goal_rotations"], atol=1e-15)
    np.testing.assert_allclose(lg.theta, g["theta"], atol=tol_state)
    np.testing.assert_allclose(lg.theta_dot, g["theta_dot"], atol=tol_state)
    np.testing.assert_allclose(lg.command, g["command"], atol=tol_cmd)
    np.testing.assert_allclose(lg.ee, g["ee"], atol=tol_state)
    np.testing.assert_allclose(lg.ee_rotations, g["ee_rotations"], atol=tol_state)
    np.testing.assert_allclose(lg.cost_total, g["cost_total"], rtol=tol_cost, atol=tol_cost)
    for k in TERMS:
        np.testing.assert_allclose(lg.cost_terms[k], g[f"term_{k}"], rtol=tol_cost, atol=tol_cost)
    np.testing.assert_array_equal(lg.collision, g["collision"])


def test_episode_fp64_script_noise_matches_reference():
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.controller import run_episode

    g = golden("episode_c1")
    c = configs.make_controller(1, particles=int(g["particles"]), precision="fp64")
    lg = run_episode(c, configs.start_state(), _script(g), int(g["steps"]), noise_sigma=float(g["noise_sigma"]),
                     sim_seed=int(g["sim_seed"]))
    _check_log(lg, g, 1e-6, 1e-6, 1e-6)
    np.testing.assert_allclose(c.policy.means, g["final_means"], atol=1e-6)
    np.testing.assert_allclose(c.policy.variances, g["final_variances"], atol=1e-6)
    np.testing.assert_allclose(c.filter.last_command, g["filt_last_command"], atol=1e-6)
    np.testing.assert_allclose(c.filter.last_estimate.theta, g["filt_theta"], atol=1e-6)
    np.testing.assert_allclose(c.filter.last_estimate.theta_dot, g["filt_theta_dot"], atol=1e-6)
    assert (lg.latency_ms > 0).all()


def test_episode_fp32_learned_collision_matches_reference():
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.controller import run_episode

    g = golden("episode_c2")
    c = configs.make_controller(2, particles=int(g["particles"]))
    lg = run_episode(c, configs.start_state(), configs.make_goal(2), int(g["steps"]))
    _check_log(lg, g, 2e-3, 2e-3, 2e-3)


def test_episode_world_collision_column_matches_reference():
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.controller import run_episode
    from paper_2104_13542_b200.simworld import voxel_world

    g = golden("episode_c3")
    w = voxel_world(golden("step_world")["occupancy"], origin=np.full(3, -1.0), voxel=2.0 / 64,
                    spheres=g["spheres"])
    np.testing.assert_allclose(np.sort(w.boxes, axis=0), np.sort(g["boxes"], axis=0), atol=1e-12)
    c = configs.make_controller(3, particles=int(g["particles"]), precision="fp64", world=w)
    lg = run_episode(c, configs.start_state(), _script(g), int(g["steps"]))
    _check_log(lg, g, 1e-6, 1e-6, 1e-6)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_device_loop_equals_host_loop(precision):
    """Same kernels, same inputs: the device episode and the host loop of
    control_step calls agree to rounding (the filter blend runs in fp64 in
    both; only FMA contraction can differ)."""
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.controller import run_episode
    from paper_2104_13542_b200.simworld import TargetScript

    script = TargetScript(times=[0.0, 0.15, 0.3], positions=[[0.45, 0.1, 0.55], [0.3, -0.2, 0.6],
                                                            [0.5, 0.1, 0.4]], interpolation="linear")
    logs, ctrls = [], []
    for dev in (True, False):
        c = configs.make_controller(2, particles=500, precision=precision)
        logs.append(run_episode(c, configs.start_state(), script, 10, noise_sigma=0.001, sim_seed=3,
                                device_loop=dev))
        ctrls.append(c)
    a, b = logs
    tol = 1e-9 if precision == "fp64" else 1e-4
    for k in ("theta", "theta_dot", "command", "ee", "cost_total"):
        np.testing.assert_allclose(getattr(a, k), getattr(b, k), atol=tol, rtol=tol, err_msg=k)
    np.testing.assert_array_equal(a.goal, b.goal)
    ca, cb = ctrls
    np.testing.assert_allclose(ca.policy.means, cb.policy.means, atol=tol)
    np.testing.assert_allclose(ca.filter.last_command, cb.filter.last_command, atol=tol)
    np.testing.assert_allclose(ca.filter.last_estimate.theta, cb.filter.last_estimate.theta, atol=tol)
    np.testing.assert_allclose(ca._prev_command, cb._prev_command, atol=tol)
    # the controller keeps working after the episode, from the same state
    st = configs.start_state()
    np.testing.assert_allclose(ca.control_step(st)[0], cb.control_step(st)[0], atol=10 * tol)


def test_abort_on_non_finite_plant_keeps_row_and_freezes_policy():
    """A non-finite plant state ends the episode after that row; the replays
    that follow leave the policy untouched (status MPPI_E_SKIPPED)."""
    from paper_2104_13542_b200 import configs

    noise = np.zeros((6, 14))
    noise[2, 3] = np.inf
    outs = []
    for steps, nz in ((6, noise), (3, np.zeros((3, 14)))):
        c = configs.make_controller(1, particles=256, precision="fp64")
        c.set_goal(configs.make_goal(1))
        r = c.plan.episode(steps, 0.05, 0.3, configs.REACH_START, np.zeros(7), noise=nz)
        outs.append((r, c.plan.get_policy(0)))
    (ra, pa), (rb, pb) = outs
    assert ra["aborted"] and ra["steps_done"] == 3
    assert not rb["aborted"] and rb["steps_done"] == 3
    np.testing.assert_array_equal(ra["command"], rb["command"])
    np.testing.assert_array_equal(ra["theta"], rb["theta"])
    np.testing.assert_array_equal(pa[0], pb[0])
    np.testing.assert_array_equal(pa[1], pb[1])


def test_fallback_ladder_on_device_matches_host():
    """Non-finite policy means make every control step fail (non-finite
    controls): previous command once, then brake (controller.py:224-241), on
    the device as on the host."""
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.controller import run_episode

    logs = []
    for dev in (True, False):
        c = configs.make_controller(1, particles=256, precision="fp64")
        c._prev_command = np.full(7, 0.25)
        means, var = c.plan.get_policy(0)
        c.plan.set_policy(np.full_like(means, np.nan), var, 0)
        logs.append((run_episode(c, configs.start_state(), configs.make_goal(1), 4, device_loop=dev), c))
    (a, ca), (b, cb) = logs
    np.testing.assert_array_equal(a.command, b.command)
    np.testing.assert_array_equal(a.command[0], np.full(7, 0.25))
    np.testing.assert_array_equal(a.command[1:], 0.0)
    assert ca._fallback_armed and cb._fallback_armed
    np.testing.assert_allclose(a.theta, b.theta, atol=1e-12)


def test_episode_graph_reuse_and_counter():
    """A second episode of the same shape replays the cached graph and gives
    the same log from the same start; the pseudorandom step counter advances
    by the steps run, exactly as S host control_steps would advance it."""
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.controller import run_episode

    logs = []
    for _ in range(2):
        c = configs.make_controller(1, particles=256, precision="fp64")
        run_episode(c, configs.start_state(), configs.make_goal(1), 5)  # capture
        logs.append(run_episode(c, configs.start_state(), configs.make_goal(1), 5))  # cached graph
    np.testing.assert_array_equal(logs[0].command, logs[1].command)
    # pseudorandom: an episode of S steps, then one host step == S + 1 host steps
    cmds = []
    for dev in (True, False):
        c = configs.make_controller(1, particles=256, precision="fp64", generator="pseudorandom")
        run_episode(c, configs.start_state(), configs.make_goal(1), 4, device_loop=dev)
        cmds.append(c.control_step(configs.start_state())[0])
    np.testing.assert_allclose(cmds[0], cmds[1], atol=1e-9)
