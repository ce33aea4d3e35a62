"""Learned self-collision distance (jointmpc/surrogate.py).

The net is the reference's posenc(14) -> 256 -> 128 -> 64 -> 1 ReLU MLP
(surrogate.py:21-52); weights load from the reference's ``.npz`` layout
(surrogate.py:127-143). Inference runs on the tensor cores
(csrc/mppi_mlp.cuh); ``train_collision_surrogate`` (surrogate.py:146-206)
trains on the device in float64 (csrc/mppi_train.cu) from the reference's own
random draws. The bundled weights were produced by the reference's trainer
(scripts/make_surrogate.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ContractError, TrainingError

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


def train_collision_surrogate(chain, samples: int, seed: int, epochs: int = 100, batch_size: int = 256,
                              lr: float = 1e-3, *, return_losses: bool = False):
    """Fit the net to oracle distances on uniform in-limit configurations
    (surrogate.py:146-206): 90/10 split, mini-batch MSE, Adam with the step
    size halved at epochs 50 and 75, holdout MAE and sign agreement.

    The random draws happen here with the reference's generator and order —
    samples, He initialisation, one permutation per epoch — and the oracle
    labels come from the GPU capsule seam, so the device loop (mppi_train_mlp,
    float64) trains on the reference's data, initialisation and batch order.
    A non-finite loss raises TrainingError with the last finite loss, after
    the loop (the device does not stop early)."""
    import ctypes as C

    from . import _native as N
    from .costs import OracleSelfCollision

    if samples < 1000:
        raise ContractError("need at least 1000 samples")
    if not chain.pair_a.size:
        raise ContractError(f"chain {chain.name!r} has no self-collision pairs")
    rng = np.random.default_rng(seed)
    q = rng.uniform(chain.joint_limits[:, 0], chain.joint_limits[:, 1], size=(samples, chain.dof))
    y = OracleSelfCollision(chain).distance(q)
    split = int(samples * 0.9)
    x_train = np.ascontiguousarray(positional_encoding(q[:split]))
    y_train = np.ascontiguousarray(y[:split])
    x_hold = np.ascontiguousarray(positional_encoding(q[split:]))
    y_hold = np.ascontiguousarray(y[split:])
    net = MLP(2 * chain.dof, rng)
    order = np.empty((epochs, split), dtype=np.int64)
    for e in range(epochs):  # the reference draws one permutation per epoch, in this order
        order[e] = rng.permutation(split)
    lrs, cur = np.empty(epochs), lr
    for e in range(epochs):
        if e in (50, 75):
            cur *= 0.5
        lrs[e] = cur
    batches = (split + batch_size - 1) // batch_size
    t = np.arange(1, epochs * batches + 1)
    bc1 = np.array([1.0 - 0.9 ** int(k) for k in t])  # Python float power, as Adam.step
    bc2 = np.array([1.0 - 0.999 ** int(k) for k in t])
    W = [np.ascontiguousarray(w, dtype=np.float64).copy() for w in net.weights]
    b = [np.ascontiguousarray(v, dtype=np.float64).copy() for v in net.biases]
    desc = N.TrainDesc()
    desc.in_dim, desc.n_train, desc.n_hold = 2 * chain.dof, split, samples - split
    desc.epochs, desc.batch_size = epochs, batch_size
    desc.x_train, desc.y_train = N.dptr(x_train), N.dptr(y_train)
    desc.x_hold, desc.y_hold = N.dptr(x_hold), N.dptr(y_hold)
    desc.order = order.ctypes.data_as(C.POINTER(C.c_int64))
    desc.lr, desc.bias_corr1, desc.bias_corr2 = N.dptr(lrs), N.dptr(bc1), N.dptr(bc2)
    res = N.TrainResult()
    losses = np.empty(max(epochs * batches, 1))
    res.losses = N.dptr(losses)
    wp = (N._dp * 4)(*[N.dptr(w) for w in W])
    bp = (N._dp * 4)(*[N.dptr(v) for v in b])
    N.require_device()
    N.check(N.load_library().mppi_train_mlp(C.byref(desc), wp, bp, C.byref(res)))
    if res.diverged_epoch >= 0:
        raise TrainingError(f"loss diverged at epoch {res.diverged_epoch} (last finite {res.last_finite_loss:.6g})",
                            last_loss=float(res.last_finite_loss))
    net.weights, net.biases = W, b
    model = LearnedSelfCollision(net=net, dof=chain.dof, holdout_mae=float(res.holdout_mae),
                                 sign_agreement=float(res.sign_agreement))
    if return_losses:
        return model, losses[:epochs * batches], float(res.device_ms)
    return model
