"""CPU checks of the episode driver's host pieces against the reference's own
outputs (tests/golden/episode_parts.npz, episode_*.npz): target_position_at,
filter_state, sim_step with noise, EpisodeLog's CSV rendering."""

import numpy as np
import pytest

from conftest import golden


def test_target_position_hold_and_linear():
    from paper_2104_13542_b200.simworld import TargetScript, target_position_at

    g = golden("episode_parts")
    for interp in ("hold", "linear"):
        script = TargetScript(g["times"], g["positions"], interp)
        got = np.array([target_position_at(script, t) for t in g["ts"]])
        np.testing.assert_array_equal(got, g[interp])


def test_filter_state_and_sim_step():
    from paper_2104_13542_b200.controller import FilterState, filter_state
    from paper_2104_13542_b200.rollout import JointState
    from paper_2104_13542_b200.simworld import sim_step

    g = golden("episode_parts")
    raw = JointState(theta=g["raw_theta"], theta_dot=g["raw_theta_dot"], theta_ddot=np.zeros(7))
    filt = FilterState(lam=0.3, last_command=g["last_command"].copy(),
                       last_estimate=JointState(theta=g["le_theta"], theta_dot=g["le_theta_dot"],
                                                theta_ddot=np.zeros(7)))
    est = filter_state(raw, filt, 0.05)
    np.testing.assert_array_equal(est.theta, g["est_theta"])
    np.testing.assert_array_equal(est.theta_dot, g["est_theta_dot"])
    assert filt.last_estimate is est
    nxt = sim_step(raw, g["u"], 0.05, noise_sigma=0.01, rng=np.random.default_rng(5))
    np.testing.assert_array_equal(nxt.theta, g["sim_theta"])
    np.testing.assert_array_equal(nxt.theta_dot, g["sim_theta_dot"])


def test_filter_rejects_bad_blend():
    from paper_2104_13542_b200.controller import FilterState
    from paper_2104_13542_b200.errors import ContractError
    from paper_2104_13542_b200.rollout import zero_state

    with pytest.raises(ContractError):
        FilterState(lam=1.5, last_command=np.zeros(7), last_estimate=zero_state(7))


def test_episode_log_csv_matches_reference_rendering(arm7):
    """EpisodeLog.to_csv is the external interface: the same columns and number
    formatting as the reference's, byte for byte."""
    from paper_2104_13542_b200.controller import EpisodeLog

    g = golden("episode_c1")
    ref_csv = str(g["csv"])
    lat = np.array([float(r.split(",")[-1]) for r in ref_csv.strip().split("\n")[1:]])
    lg = EpisodeLog(chain=arm7, t=g["t"], theta=g["theta"], theta_dot=g["theta_dot"], command=g["command"],
                    goal=g["goal"], ee=g["ee"], cost_total=g["cost_total"],
                    cost_terms={k: g[f"term_{k}"] for k in ("pose", "stop", "joint", "manip", "selfcoll",
                                                            "envcoll")},
                    collision=g["collision"], latency_ms=lat)
    assert lg.steps == 12
    assert lg.to_csv() == ref_csv
