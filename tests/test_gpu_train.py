"""Surrogate training on the device (mppi_train_mlp) against the reference's
own train_collision_surrogate runs (tests/golden/train_*.npz).

The device trains in float64 on the reference's samples, He initialisation,
permutations and Adam bias corrections; only the summation order of the
matrix products differs (and the oracle labels, computed by the GPU capsule
seam instead of numba), so short runs must land on the reference's weights
to ~1e-9 and long runs on its holdout metrics.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _weights(m):
    return [np.asarray(w) for w in m.net.weights] + [np.asarray(b) for b in m.net.biases]


@pytest.mark.parametrize("name,tol", [("train_short", 1e-9), ("train_sched", 1e-6)])
def test_training_matches_reference(arm7, name, tol):
    from paper_2104_13542_b200.surrogate import train_collision_surrogate

    g = golden(name)
    m, losses, ms = train_collision_surrogate(arm7, int(g["samples"]), int(g["seed"]), epochs=int(g["epochs"]),
                                              return_losses=True)
    ref = [g[f"W{i}"] for i in range(4)] + [g[f"b{i}"] for i in range(4)]
    for got, want in zip(_weights(m), ref):
        np.testing.assert_allclose(got, want, rtol=tol, atol=tol)
    assert abs(m.holdout_mae - float(g["holdout_mae"])) < 10 * tol
    assert m.sign_agreement == pytest.approx(float(g["sign_agreement"]), abs=1e-3)
    assert np.isfinite(losses).all() and ms > 0.0


def test_training_acceptance_quality(arm7):
    """The reference's acceptance configuration (50k samples, 100 epochs,
    seed 0): the model meets the acceptance bar (sign >= 0.95, MAE < 0.02 m,
    test_acceptance.py:267-279) and lands on the reference's own metrics."""
    from paper_2104_13542_b200.surrogate import train_collision_surrogate

    g = golden("train_accept")
    m, losses, ms = train_collision_surrogate(arm7, 50_000, 0, return_losses=True)
    assert m.sign_agreement >= 0.95 and m.holdout_mae < 0.02
    assert m.holdout_mae == pytest.approx(float(g["holdout_mae"]), rel=1e-3)
    assert m.sign_agreement == pytest.approx(float(g["sign_agreement"]), abs=2e-3)
    print(f"device training: {ms:.1f} ms for {losses.size} steps "
          f"(reference {float(g['cpu_seconds']):.1f} s on the CPU)")


def test_trained_model_runs_on_the_tensor_core_path(arm7):
    """The trained weights feed the tcgen05 MLP like the bundled ones."""
    from paper_2104_13542_b200.surrogate import train_collision_surrogate

    m = train_collision_surrogate(arm7, 2000, 1, epochs=2)
    q = np.random.default_rng(0).uniform(arm7.joint_limits[:, 0], arm7.joint_limits[:, 1], size=(300, 7))
    x = np.concatenate([np.sin(q), np.cos(q)], axis=1)
    h = x
    for i, (W, b) in enumerate(zip(m.net.weights, m.net.biases)):
        h = h @ W + b
        if i < 3:
            h = np.maximum(h, 0.0)
    np.testing.assert_allclose(m.distance(q), h[:, 0], atol=1e-5)


def test_training_rejects_small_sample_counts(arm7):
    from paper_2104_13542_b200.errors import ContractError
    from paper_2104_13542_b200.surrogate import train_collision_surrogate

    with pytest.raises(ContractError):
        train_collision_surrogate(arm7, 500, 0)
