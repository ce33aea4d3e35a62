"""Batches of independent controllers (BASELINE config 4).

The reference has one Controller per object (controller.py:93-96). Here B
independent controllers share one plan: one fused rollout over B*N particles
(grid over instance x particle), one tensor-core MLP launch over all B*N*H
rows, one statistics kernel with a block-record combine per instance. Every
instance has its own policy, state and goal; the Halton perturbation block is
shared (it is a constant of the controller configuration, controller.py:166)
and stays L2-resident.

Parity is per instance: instance b reproduces a reference Controller built
with the same kwargs and goal b (tests/test_gpu_batched.py).

Multi-GPU: ``shard_instances`` splits B over ranks; each rank owns an
independent BatchedController on its own device and there is no data-path
collective.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .costs import CostStack, CostWeights, GoalSpec
from .engine import Plan, PlanSpec
from .errors import ContractError
from .policy import ISOTROPIC, PER_JOINT, PolicyParams, UpdateConfig
from .rollout import make_dt_schedule
from .sampling import HALTON, PSEUDORANDOM, SmoothingSpec, smoothing_code


def shard_instances(total: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) instance range of `rank` (sizes differ by at most 1)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ContractError("bad rank / world size")
    base, rem = divmod(total, world_size)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


@dataclass
class BatchDiagnostics:
    status: np.ndarray  # (B,) mppi_status per instance (0 ok)
    fallback: list  # per instance: "", "reissue", "brake"
    best_cost: np.ndarray
    mean_cost: np.ndarray
    device_ms: float
    stage_ms: dict


class BatchedController:
    """B independent MPPI controllers stepped together on one device."""

    def __init__(self, chain, goals, *, horizon=30, particles=200, dt_base=0.05, dt_ramp="two_phase",
                 gamma=0.99, terminal_weight=1.0, generator=HALTON, smoothing: SmoothingSpec | None = None,
                 null_count=2, weights: CostWeights | None = None, world=None, self_collision=None,
                 beta=0.5, alpha_mu=0.9, alpha_sigma=0.5, sigma0_sq=1.0, sigma_sq_min=1e-4,
                 sigma_sq_max=0.0, policy_mode=PER_JOINT, iterations=1, seed=0, precision="fp32",
                 device=0):
        goals = list(goals)
        if not goals:
            raise ContractError("need at least one goal / instance")
        if particles <= null_count + 1:
            raise ContractError("need more particles than reserved sequences")
        if generator not in (HALTON, PSEUDORANDOM):
            raise ContractError(f"unknown generator {generator!r}")
        self.chain = chain
        self.B = len(goals)
        self.dof = chain.dof
        self.horizon = horizon
        self.particles = particles
        self.policy_mode = policy_mode
        self.smoothing = smoothing or SmoothingSpec()
        self.sched = make_dt_schedule(horizon, dt_base, dt_ramp)
        self.update_cfg = UpdateConfig(beta=beta, alpha_mu=alpha_mu, alpha_sigma=alpha_sigma, gamma=gamma,
                                       sigma_sq_min=sigma_sq_min,
                                       sigma_sq_max=sigma_sq_max if sigma_sq_max > 0.0 else sigma0_sq)
        self.sigma0_sq = sigma0_sq
        self.cost_stack = CostStack(chain=chain, weights=weights or CostWeights(), goal=goals[0], world=world,
                                    self_collision=self_collision)
        spec = PlanSpec(
            horizon=horizon, particles=particles, dts=self.sched.dts, null_count=null_count,
            instances=self.B, iterations=max(1, iterations),
            policy_mode=N.POLICY_ISOTROPIC if policy_mode == ISOTROPIC else N.POLICY_PER_JOINT,
            precision=N.FP64 if precision == "fp64" else N.FP32,
            generator=N.GEN_HALTON if generator == HALTON else N.GEN_PSEUDORANDOM,
            smoothing=smoothing_code(self.smoothing), spline_degree=self.smoothing.spline_degree,
            knots=self.smoothing.knot_count(horizon), device=device, particles_total=particles, seed=seed,
            comb=tuple(self.smoothing.comb_coeffs), gamma=gamma, terminal_weight=terminal_weight, beta=beta,
            alpha_mu=alpha_mu, alpha_sigma=alpha_sigma, sigma0_sq=sigma0_sq,
            sigma_sq_min=self.update_cfg.sigma_sq_min, sigma_sq_max=self.update_cfg.sigma_sq_max,
            default_tail=self.update_cfg.default_tail)
        world_arg = world if (world is not None and getattr(world, "obstacle_count", 0)) else None
        self.plan = Plan(chain, self.cost_stack.weights, spec, provider=self.cost_stack.self_collision,
                         world=world_arg)
        if generator == HALTON:
            self.plan.init_noise()
        self.set_goals(goals)
        self._prev = np.zeros((self.B, self.dof))
        self._armed = np.zeros(self.B, dtype=bool)

    def set_goals(self, goals, first: int = 0):
        goals = list(goals)
        R = np.stack([g.target_pose.rotation for g in goals])
        t = np.stack([g.target_pose.translation for g in goals])
        modes = [g.mode_code for g in goals]
        self.plan.set_goals(R, t, modes, first)

    def policy(self, instance: int) -> PolicyParams:
        m, v = self.plan.get_policy(instance)
        if self.policy_mode == ISOTROPIC:
            v = v[:, 0].copy()
        return PolicyParams(means=m, variances=v, mode=self.policy_mode, tail_variance=self.sigma0_sq)

    def control_step(self, theta, theta_dot):
        """theta, theta_dot (B, d) -> commands (B, d), BatchDiagnostics.

        Per-instance fallback ladder as controller.py:224-241 (reissue once, then brake)."""
        theta = np.asarray(theta, dtype=np.float64).reshape(self.B, self.dof)
        theta_dot = np.asarray(theta_dot, dtype=np.float64).reshape(self.B, self.dof)
        if not (np.isfinite(theta).all() and np.isfinite(theta_dot).all()):
            raise ContractError("joint state is not finite")
        cmds, infos = self.plan.step(theta, theta_dot)
        return self._apply_ladder(cmds, infos)

    def _apply_ladder(self, cmds, infos):
        """Per-instance statuses of the last plan step -> fallback ladder and diagnostics."""
        cols = self.plan.info_columns  # (B,) record view of infos
        status = cols["status"].astype(np.int32)
        fallback = [""] * self.B
        bad = np.flatnonzero(status != N.OK)
        if bad.size:
            for b in bad:
                exc = N.status_exception(int(status[b]))
                if not isinstance(exc, (ContractError, N.PolicyStateError)):
                    raise exc
                if not self._armed[b]:
                    self._armed[b] = True
                    cmds[b] = self._prev[b]
                    fallback[b] = "reissue"
                else:
                    cmds[b] = 0.0
                    fallback[b] = "brake"
        ok = status == N.OK
        self._armed[ok] = False
        self._prev[ok] = cmds[ok]
        i0 = infos[0]
        diag = BatchDiagnostics(
            status=status, fallback=fallback,
            best_cost=cols["best_cost"].copy(), mean_cost=cols["mean_cost"].copy(),
            device_ms=float(i0.device_ms),
            stage_ms={"sample": i0.sample_ms, "rollout": i0.rollout_ms, "mlp": i0.mlp_ms,
                      "update": i0.update_ms})
        return cmds, diag
