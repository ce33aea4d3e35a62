"""Config 4 (batched independent controllers) and config 5 (particle-sharded
single controller) on the GPU, against independent oracle controllers and the
unsharded device controller."""

import numpy as np
import pytest

from oracle import mppi_oracle as O

pytestmark = pytest.mark.gpu


def _oracle_for(goal, theta0, config=2, particles=128, **extra):
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import ARM7_SURROGATE

    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = particles
    kw.update(extra)
    mlp = None
    if config == 2:
        with np.load(ARM7_SURROGATE) as z:
            mlp = {k: z[k] for k in z.files if k.startswith(("W", "b"))}
    return O.OracleController(load_chain("arm7.chain"), configs.make_weights(config), goal.target_pose.rotation,
                              goal.target_pose.translation, goal.mode != "position_only",
                              provider="learned" if config == 2 else None, mlp_state=mlp, **kw)


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-4), ("fp32", 1e-3)])  # MLP-limited (config-2 costs)
def test_batched_instances_match_independent_controllers(precision, tol):
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.batched import BatchedController
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import load_arm7_surrogate

    B, n = 5, 128
    goals, th0 = configs.batched_problem(B)
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = n
    bc = BatchedController(load_chain("arm7.chain"), goals, weights=configs.make_weights(2),
                           self_collision=load_arm7_surrogate(), precision=precision, **kw)
    oracles = [_oracle_for(goals[b], th0[b], particles=n) for b in range(B)]
    theta = th0.copy()
    thetad = np.zeros_like(theta)
    for _ in range(2):
        cmds, diag = bc.control_step(theta, thetad)
        assert (diag.status == 0).all()
        for b in range(B):
            ref = oracles[b].step(theta[b], thetad[b])
            np.testing.assert_allclose(cmds[b], ref, atol=tol, err_msg=f"instance {b}")
            np.testing.assert_allclose(bc.policy(b).means, oracles[b].means, atol=tol)
        thetad = thetad + 0.05 * cmds
        theta = theta + 0.05 * thetad


@pytest.mark.parametrize("total,R", [(600, 3), (262144, 2)])  # config 5's largest N at full size
def test_emulated_particle_shards_match_unsharded(total, R):
    """R plans holding disjoint particle shards on one GPU; their records are
    concatenated on the device exactly as the all-gather would, and every
    shard's finalize must reproduce the unsharded controller."""
    import torch

    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.engine import Plan, PlanSpec
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.sharded import particle_shard
    from paper_2104_13542_b200 import _native as N

    ref = configs.make_controller(1, particles=total, precision="fp64")
    chain = load_chain("arm7.chain")
    goal = configs.make_goal(1)
    plans = []
    for r in range(R):
        off, cnt = particle_shard(total, R, r)
        spec = PlanSpec(horizon=30, particles=cnt, dts=ref.sched.dts, null_count=2, precision=N.FP64,
                        particle_offset=off, particles_total=total, gamma=0.99, beta=1.0, alpha_mu=0.9,
                        alpha_sigma=0.5, sigma0_sq=0.5, sigma_sq_min=0.01, sigma_sq_max=0.5, knots=5)
        p = Plan(chain, configs.make_weights(1), spec)
        p.init_noise()
        p.set_goal(goal.target_pose.rotation, goal.target_pose.translation, goal.mode_code, 0)
        plans.append(p)
    # the shards' noise rows are exactly the unsharded block's rows
    full = ref.plan.get_noise()
    for r, p in enumerate(plans):
        off, cnt = particle_shard(total, R, r)
        np.testing.assert_array_equal(p.get_noise(), full[off:off + cnt])
    L = plans[0].record_len()
    recs = torch.zeros(R * L, dtype=torch.float64, device="cuda:0")
    st = configs.start_state()
    for _ in range(3):
        cmd_ref, _ = ref.control_step(st)
        for r, p in enumerate(plans):
            p.stats_dev(st.theta, st.theta_dot, recs.data_ptr() + r * L * 8)
        torch.cuda.synchronize()
        outs = [p.finalize_dev(recs.data_ptr(), R)[0] for p in plans]
        for c in outs:
            np.testing.assert_allclose(c, cmd_ref, atol=1e-9)
        np.testing.assert_array_equal(outs[0], outs[1])
        np.testing.assert_allclose(plans[0].get_policy(0)[1], ref.plan.get_policy(0)[1], atol=1e-9)


@pytest.mark.parametrize("B", [12, 150])  # multi-block statistics with a record combine / one block per instance
def test_batched_statistics_layouts_match_oracle(B):
    """Batches between 9 and 147 instances use 32-particle statistics blocks
    and the last-block record combine; from 148 instances on, one block per
    instance (choose_blocks). Both must match independent oracles."""
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.batched import BatchedController
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import load_arm7_surrogate

    n = 128
    goals, th0 = configs.batched_problem(B)
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = n
    bc = BatchedController(load_chain("arm7.chain"), goals, weights=configs.make_weights(2),
                           self_collision=load_arm7_surrogate(), precision="fp64", **kw)
    picks = [0, B // 2, B - 1]
    oracles = {b: _oracle_for(goals[b], th0[b], particles=n) for b in picks}
    cmds, diag = bc.control_step(th0, np.zeros_like(th0))
    assert (diag.status == 0).all()
    for b in picks:
        ref = oracles[b].step(th0[b], np.zeros(7))
        np.testing.assert_allclose(cmds[b], ref, atol=1e-4, err_msg=f"instance {b}")
        np.testing.assert_allclose(bc.policy(b).means, oracles[b].means, atol=1e-4)


def test_peer_exchange_step_matches_allgather_path():
    """mppi_step_exchange (the record pushed over peer memory and the update
    applied inside the statistics kernel) against mppi_stats_dev + all-gather
    + mppi_finalize_dev on a one-rank world: identical commands and policies,
    both within tolerance of the unsharded controller. (Ranks whose kernels
    wait on one another need one GPU each; the multi-rank wiring is covered by
    tests/test_sharding_gloo.py.)"""
    import torch

    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200 import _native as N
    from paper_2104_13542_b200.engine import Plan, PlanSpec
    from paper_2104_13542_b200.kinematics import load_chain

    total = 600  # > 512 particles: the multi-block statistics kernel with its record combine
    for n, precision in ((total, N.FP64), (300, N.FP32)):
        ref = configs.make_controller(1, particles=n, precision="fp64" if precision == N.FP64 else "fp32")
        chain = load_chain("arm7.chain")
        goal = configs.make_goal(1)
        plans = []
        for _ in range(2):
            spec = PlanSpec(horizon=30, particles=n, dts=ref.sched.dts, null_count=2, precision=precision,
                            particle_offset=0, particles_total=n, gamma=0.99, beta=1.0, alpha_mu=0.9,
                            alpha_sigma=0.5, sigma0_sq=0.5, sigma_sq_min=0.01, sigma_sq_max=0.5, knots=5)
            p = Plan(chain, configs.make_weights(1), spec)
            p.init_noise()
            p.set_goal(goal.target_pose.rotation, goal.target_pose.translation, goal.mode_code, 0)
            plans.append(p)
        peer, gather = plans
        recv, flags = peer.peer_buffers(1)
        peer.set_peers(0, [recv], [flags])
        rec = torch.zeros(gather.record_len(), dtype=torch.float64, device="cuda:0")
        st = configs.start_state()
        for step in range(4):
            st.theta[:] = configs.start_state().theta + 0.01 * step
            cmd_ref, _ = ref.control_step(st)
            cmd_p, info_p = peer.step_exchange(st.theta, st.theta_dot)
            gather.stats_dev(st.theta, st.theta_dot, rec.data_ptr())
            torch.cuda.synchronize()
            cmd_g, info_g = gather.finalize_dev(rec.data_ptr(), 1)
            assert info_p.status == 0 and info_g.status == 0
            np.testing.assert_array_equal(cmd_p, cmd_g)
            np.testing.assert_array_equal(peer.get_policy(0)[0], gather.get_policy(0)[0])
            np.testing.assert_array_equal(peer.get_policy(0)[1], gather.get_policy(0)[1])
            assert info_p.best_cost == info_g.best_cost
            np.testing.assert_allclose(cmd_p, cmd_ref, atol=1e-9 if precision == N.FP64 else 1e-3)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_multi_instance_statistics_bit_identical(precision, monkeypatch):
    """stats_multi_kernel (G instances per block sharing the perturbation
    loads; mppi_kernels.cuh) against stats_kernel with one block per instance
    (MPPI_STATS_G=1): identical commands, policies, best and mean costs over
    several steps, with a ragged last block (150 = 37 x 4 + 2, 75 x 2)."""
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.batched import BatchedController
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import load_arm7_surrogate

    B, n = 150, 128
    goals, th0 = configs.batched_problem(B)
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = n
    runs = {}
    for g in ("1", "2", "4", "22"):  # 22: the default, two instances at 5 blocks per SM
        monkeypatch.setenv("MPPI_STATS_G", g)  # read when the step is launched / captured
        bc = BatchedController(load_chain("arm7.chain"), goals, weights=configs.make_weights(2),
                               self_collision=load_arm7_surrogate(), precision=precision, **kw)
        th, thd = th0.copy(), np.zeros_like(th0)
        out = []
        for step in range(3):
            cmds, diag = bc.control_step(th + 0.01 * step, thd)
            assert (diag.status == 0).all()
            out.append((cmds.copy(), diag.best_cost.copy(), diag.mean_cost.copy()))
        out.append(tuple(np.stack([getattr(bc.policy(b), f) for b in range(B)])
                         for f in ("means", "variances")))
        runs[g] = out
    for g in ("2", "4", "22"):
        for a, b in zip(runs["1"], runs[g]):
            for x, y in zip(a, b):
                np.testing.assert_array_equal(x, y, err_msg=f"G={g}")
