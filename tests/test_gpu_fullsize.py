"""Config 4 at the bench's full size (4096 controllers x 500 particles x H30,
fp32, config-2 costs): spot instances against independent oracle controllers
and a size-independent property — reversing the instance order reverses the
commands bit for bit (every instance's rollout rows, MLP rows and statistics
are independent of its slot; cf. the reference's worker / permutation
invariance tests, test_rollout.py:134-156)."""

import numpy as np
import pytest

from oracle import mppi_oracle as O

pytestmark = pytest.mark.gpu


def _controller(goals):
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.batched import BatchedController
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import load_arm7_surrogate

    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = 500
    return BatchedController(load_chain("arm7.chain"), goals, weights=configs.make_weights(2),
                             self_collision=load_arm7_surrogate(), precision="fp32", **kw)


def test_config4_full_size_matches_oracle_and_is_permutation_invariant():
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import ARM7_SURROGATE

    B = 4096
    goals, th0 = configs.batched_problem(B)
    bc = _controller(goals)
    cmds, diag = bc.control_step(th0, np.zeros_like(th0))
    assert (diag.status == 0).all() and np.isfinite(cmds).all()

    with np.load(ARM7_SURROGATE) as z:
        mlp = {k: z[k] for k in z.files if k.startswith(("W", "b"))}
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = 500
    for b in (0, 2047, 4095):
        g = goals[b]
        oc = O.OracleController(load_chain("arm7.chain"), configs.make_weights(2), g.target_pose.rotation,
                                g.target_pose.translation, g.mode != "position_only", provider="learned",
                                mlp_state=mlp, **kw)
        ref = oc.step(th0[b], np.zeros(7))
        np.testing.assert_allclose(cmds[b], ref, atol=1e-3, err_msg=f"instance {b}")  # fp32, MLP-limited
        np.testing.assert_allclose(diag.best_cost[b], oc.last["totals"][np.isfinite(oc.last["totals"])].min(),
                                   rtol=1e-4)

    rev = _controller(goals[::-1])
    cmds_r, diag_r = rev.control_step(th0[::-1].copy(), np.zeros_like(th0))
    np.testing.assert_array_equal(cmds_r[::-1], cmds)
    np.testing.assert_array_equal(diag_r.best_cost[::-1], diag.best_cost)
