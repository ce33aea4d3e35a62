"""One controller, particles sharded over GPUs (BASELINE config 5).

Each rank owns particles [offset, offset + N/G) of a single controller (the
perturbation rows of the global Halton block, centred over all N rows; null
and mean rows live on rank 0) and the full, replicated policy. One iteration is

  rank-local: rollout + costs + MLP + weights relative to the LOCAL best cost
              -> record = [m_k, S0_k, count_k, sumfinite_k, status, bad,
                           S1_k (H*d), S2_k (H*d)]         (mppi_stats_dev)
  exchange:   every rank's record to every rank (426 doubles each for arm7
              H=30: 3.4 KB per rank): fused into the statistics kernel as
              NVLink P2P stores + a release flag (PeerExchange), or ONE NCCL
              all-gather between two kernels (RecordExchange)
  replicated: fixed-order combine, rescaling record k by exp(-(m_k - m)/beta),
              then the mean/covariance update, shift and command on every
              rank identically (mppi_finalize_dev)

All ranks therefore hold bit-identical policies without a broadcast, and the
result does not depend on the order NCCL delivers records in.
"""

from __future__ import annotations

import numpy as np

from .errors import ContractError


def particle_shard(total: int, world_size: int, rank: int) -> tuple[int, int]:
    """(offset, count) of rank's contiguous particle rows."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ContractError("bad rank / world size")
    base, rem = divmod(total, world_size)
    offset = rank * base + min(rank, rem)
    return offset, base + (1 if rank < rem else 0)


class RecordExchange:
    """All-gather of one fixed-length float64 record per rank (the only
    collective of the sharded update). Works with any torch.distributed
    backend: NCCL on device tensors in production, gloo on CPU in tests."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)

    def all_gather(self, record):
        import torch

        out = torch.empty(self.world * record.numel(), dtype=record.dtype, device=record.device)
        self.dist.all_gather_into_tensor(out, record.contiguous(), group=self.group)
        return out


class PeerExchange:
    """The exchange fused into the statistics kernel over NVLink peer memory
    (mppi_step_exchange): every rank's kernel pushes its record straight into
    slot [rank] of every rank's receive buffer and publishes it with a flag;
    no NCCL call, no separate finalize launch. This object only wires the
    buffers: it exports CUDA IPC handles of this rank's receive buffer and
    flags, gathers every rank's handles with one host-side collective (any
    torch.distributed backend) and hands the kernel a pointer table whose
    slot k addresses rank k's buffers (slot [rank] = the plan's own).

    `ops` defaults to the plan; tests pass a stand-in with the same four
    methods (peer_buffers, ipc_handle, ipc_open, set_peers).
    """

    def __init__(self, group=None, timeout_s: float | None = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.timeout_s = timeout_s  # bounded wait of the fused exchange (plan default 5 s)
        self.opened: list[int] = []
        self.tables = None

    def attach(self, ops):
        """Allocate, export, gather, open; returns (recv pointers, flag pointers) in rank order."""
        recv, flags = ops.peer_buffers(self.world)
        mine = (ops.ipc_handle(recv), ops.ipc_handle(flags))
        gathered = [None] * self.world
        self.dist.all_gather_object(gathered, mine, group=self.group)
        recv_ptrs, flag_ptrs = [], []
        for k, (hr, hf) in enumerate(gathered):
            if k == self.rank:
                recv_ptrs.append(recv)
                flag_ptrs.append(flags)
            else:
                pr, pf = ops.ipc_open(hr), ops.ipc_open(hf)
                self.opened += [pr, pf]
                recv_ptrs.append(pr)
                flag_ptrs.append(pf)
        ops.set_peers(self.rank, recv_ptrs, flag_ptrs)
        self.tables = (recv_ptrs, flag_ptrs)
        return self.tables

    def close(self, ops):
        for ptr in self.opened:
            ops.ipc_close(ptr)
        self.opened = []


class ShardedController:
    """Config-5 controller: the reference Controller's step, particle-sharded.

    Construct on every rank after ``torch.distributed.init_process_group``.
    Mirrors Controller's kwargs (configs.make_controller builds the single-GPU
    twin); ``control_step(state)`` returns the same command on every rank.
    """

    def __init__(self, chain, goal, *, particles: int, world_size: int, rank: int, device: int,
                 exchange: RecordExchange, **kw):
        import torch

        from . import _native as N
        from .costs import CostStack, CostWeights
        from .engine import Plan, PlanSpec
        from .policy import ISOTROPIC, PER_JOINT, UpdateConfig
        from .rollout import make_dt_schedule
        from .sampling import HALTON, SmoothingSpec, smoothing_code

        self.torch = torch
        self.exchange = exchange
        self.world = world_size
        offset, count = particle_shard(particles, world_size, rank)
        smoothing = kw.pop("smoothing", None) or SmoothingSpec()
        horizon = kw.pop("horizon", 30)
        sigma0_sq = kw.pop("sigma0_sq", 1.0)
        smax = kw.pop("sigma_sq_max", 0.0)
        policy_mode = kw.pop("policy_mode", PER_JOINT)
        self.cfg = UpdateConfig(beta=kw.pop("beta", 0.5), alpha_mu=kw.pop("alpha_mu", 0.9),
                                alpha_sigma=kw.pop("alpha_sigma", 0.5), gamma=kw.pop("gamma", 0.99),
                                sigma_sq_min=kw.pop("sigma_sq_min", 1e-4),
                                sigma_sq_max=smax if smax > 0.0 else sigma0_sq)
        sched = make_dt_schedule(horizon, kw.pop("dt_base", 0.05), kw.pop("dt_ramp", "two_phase"))
        weights = kw.pop("weights", None) or CostWeights()
        self.cost_stack = CostStack(chain=chain, weights=weights, goal=goal, world=kw.pop("world", None),
                                    self_collision=kw.pop("self_collision", None))
        spec = PlanSpec(horizon=horizon, particles=count, dts=sched.dts, null_count=kw.pop("null_count", 2),
                        iterations=max(1, kw.pop("iterations", 1)),
                        policy_mode=N.POLICY_ISOTROPIC if policy_mode == ISOTROPIC else N.POLICY_PER_JOINT,
                        precision=N.FP64 if kw.pop("precision", "fp32") == "fp64" else N.FP32,
                        generator=N.GEN_HALTON if kw.pop("generator", HALTON) == HALTON else N.GEN_PSEUDORANDOM,
                        smoothing=smoothing_code(smoothing), spline_degree=smoothing.spline_degree,
                        knots=smoothing.knot_count(horizon), device=device, particle_offset=offset,
                        particles_total=particles, seed=kw.pop("seed", 0), gamma=self.cfg.gamma,
                        terminal_weight=kw.pop("terminal_weight", 1.0), beta=self.cfg.beta,
                        alpha_mu=self.cfg.alpha_mu, alpha_sigma=self.cfg.alpha_sigma, sigma0_sq=sigma0_sq,
                        sigma_sq_min=self.cfg.sigma_sq_min, sigma_sq_max=self.cfg.sigma_sq_max)
        for k in ("workers", "command_mode", "control_period", "latency_budget", "filter_lambda"):
            kw.pop(k, None)
        if kw:
            raise ContractError(f"unknown ShardedController kwargs {sorted(kw)}")
        self.iterations = spec.iterations
        self.plan = Plan(chain, weights, spec, provider=self.cost_stack.self_collision)
        self.plan.init_noise()
        g = goal
        self.plan.set_goal(g.target_pose.rotation, g.target_pose.translation, g.mode_code, 0)
        self.dev = torch.device("cuda", device)
        self.record = torch.empty(self.plan.record_len(), dtype=torch.float64, device=self.dev)
        if isinstance(exchange, PeerExchange):
            torch.cuda.set_device(device)
            exchange.attach(self.plan)
            if exchange.timeout_s is not None:
                self.plan.set_exchange_timeout(exchange.timeout_s)

    def control_step(self, state):
        if isinstance(self.exchange, PeerExchange):  # exchange fused into the statistics kernel
            try:
                theta = np.asarray(state.theta, dtype=np.float64)
                theta_dot = np.asarray(state.theta_dot, dtype=np.float64)
                if not (np.isfinite(theta).all() and np.isfinite(theta_dot).all()):
                    raise ContractError("joint state is not finite")
            except Exception:
                # this rank will not run the step: release the ranks that would wait for it
                self.plan.exchange_abort()
                raise
            # a rank that does not arrive within the plan's exchange timeout, or
            # aborts, fails the step on every rank with DeviceError (mppi status 9)
            cmd, info = self.plan.step_exchange(theta, theta_dot)
            return cmd, info
        torch = self.torch
        stream = torch.cuda.current_stream(self.dev).cuda_stream
        cmd = info = None
        for it in range(self.iterations):
            th = state.theta if it == 0 else None
            thd = state.theta_dot if it == 0 else None
            self.plan.stats_dev(th, thd, self.record.data_ptr(), stream)
            gathered = self.exchange.all_gather(self.record)
            cmd, info = self.plan.finalize_dev(gathered.data_ptr(), self.world, stream)
        return np.asarray(cmd), info
