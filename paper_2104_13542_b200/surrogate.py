"""Learned self-collision distance (jointmpc/surrogate.py), inference only.

The net is the reference's posenc(14) -> 256 -> 128 -> 64 -> 1 ReLU MLP
(surrogate.py:21-52); weights load from the reference's ``.npz`` layout
(surrogate.py:127-143). Inference runs on the GPU (csrc/mppi_mlp.cuh).
Training (Adam, backprop, surrogate.py:54-206) is offline and out of scope —
the bundled weights were produced by the reference's trainer
(scripts/make_surrogate.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ContractError

HIDDEN = (256, 128, 64)
DATA = Path(__file__).resolve().parent / "data"
ARM7_SURROGATE = DATA / "arm7_surrogate.npz"


def positional_encoding(q: np.ndarray) -> np.ndarray:
    """[sin q, cos q] on the last axis (surrogate.py:24-28). The fused rollout
    computes this in-register; this helper is for host-side inspection."""
    q = np.asarray(q, dtype=np.float64)
    return np.concatenate([np.sin(q), np.cos(q)], axis=-1)


class MLP:
    """Weight container with the reference's state-dict layout (W_i stored (in, out))."""

    def __init__(self, in_dim: int, rng: np.random.Generator):
        dims = [in_dim, *HIDDEN, 1]
        self.weights, self.biases = [], []
        for a, b in zip(dims[:-1], dims[1:]):
            self.weights.append(rng.normal(0.0, np.sqrt(2.0 / a), size=(a, b)))
            self.biases.append(np.zeros(b))

    def state_dict(self) -> dict:
        out = {}
        for i, (W, b) in enumerate(zip(self.weights, self.biases)):
            out[f"W{i}"] = W
            out[f"b{i}"] = b
        return out

    @classmethod
    def from_state(cls, state: dict) -> "MLP":
        net = cls.__new__(cls)
        net.weights, net.biases = [], []
        i = 0
        while f"W{i}" in state:
            net.weights.append(np.asarray(state[f"W{i}"], dtype=np.float64))
            net.biases.append(np.asarray(state[f"b{i}"], dtype=np.float64))
            i += 1
        if not net.weights:
            raise ContractError("empty surrogate state")
        return net


@dataclass
class LearnedSelfCollision:
    """Self-collision provider backed by the MLP (surrogate.py:108-143)."""

    net: MLP
    dof: int
    holdout_mae: float
    sign_agreement: float

    kind = "learned"

    def distance(self, q: np.ndarray, poses=None) -> np.ndarray:
        """Predicted penetration depth for q (..., d), evaluated on the GPU."""
        q = np.asarray(q, dtype=np.float64)
        if q.shape[-1] != self.dof:
            raise ContractError(f"expected {self.dof} joints, got shape {q.shape}")
        return self._engine().mlp_forward(q.reshape(-1, self.dof)).reshape(q.shape[:-1])

    def _engine(self):
        eng = getattr(self, "_plan", None)
        if eng is None:
            from .costs import CostWeights
            from .engine import Plan, PlanSpec
            from .kinematics import chain_from_dict

            # a bare revolute chain of the right length carries the weights
            chain = chain_from_dict({
                "joints": [{"type": "revolute", "axis": [0, 0, 1]} for _ in range(self.dof)],
                "limits": {"position": [[-3.2, 3.2]] * self.dof, "velocity": [1.0] * self.dof,
                           "acceleration": [1.0] * self.dof},
            })
            spec = PlanSpec(horizon=2, particles=1, dts=np.full(2, 0.05), null_count=0, sigma_sq_max=1.0)
            eng = Plan(chain, CostWeights(), spec, provider=self)
            object.__setattr__(self, "_plan", eng)
        return eng

    def save(self, path):
        state = self.net.state_dict()
        state["dof"] = np.array(self.dof)
        state["holdout_mae"] = np.array(self.holdout_mae)
        state["sign_agreement"] = np.array(self.sign_agreement)
        np.savez(path, **state)

    @classmethod
    def load(cls, path) -> "LearnedSelfCollision":
        with np.load(path) as data:
            state = {k: data[k] for k in data.files}
        return cls(net=MLP.from_state(state), dof=int(state["dof"]),
                   holdout_mae=float(state["holdout_mae"]),
                   sign_agreement=float(state["sign_agreement"]))


def load_arm7_surrogate() -> LearnedSelfCollision:
    """The bundled arm7 weights (train_collision_surrogate(arm7, 50000, seed=0))."""
    return LearnedSelfCollision.load(ARM7_SURROGATE)
