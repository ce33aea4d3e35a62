"""Python handle around one native plan (``mppi_plan`` in include/mppi_b200.h).

A plan owns every device buffer of one controller batch: the packed chain and
cost parameters, the fixed perturbation block, the per-instance policy, goal
and state, the learned-collision weights, the world, and the captured CUDA
graph of one control step. Controller, BatchedController, CostStack and
evaluate_rollouts all sit on top of this class.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ConfigError

_F64 = np.dtype(np.float64)


@dataclass
class PlanSpec:
    horizon: int
    particles: int
    dts: np.ndarray
    null_count: int = 2
    instances: int = 1
    iterations: int = 1
    policy_mode: int = N.POLICY_PER_JOINT
    precision: int = N.FP32
    generator: int = N.GEN_HALTON
    smoothing: int = N.SMOOTH_BSPLINE
    spline_degree: int = 3
    knots: int = 0
    device: int = 0
    particle_offset: int = 0
    particles_total: int = 0
    dump: int = 0
    seed: int = 0
    comb: tuple = (0.3, 0.4, 0.3)
    gamma: float = 0.99
    terminal_weight: float = 1.0
    beta: float = 0.5
    alpha_mu: float = 0.9
    alpha_sigma: float = 0.5
    sigma0_sq: float = 1.0
    sigma_sq_min: float = 1e-4
    sigma_sq_max: float = 1.0
    default_tail: float = 0.0


def chain_desc(chain):
    """Build a ChainDesc; returns (desc, keepalive arrays)."""
    keep = {
        "axes": N.f64(chain.axes), "orot": N.f64(chain.origin_rot), "otrans": N.f64(chain.origin_trans),
        "jtype": N.i64(chain.jtype), "lim": N.f64(chain.joint_limits),
        "vel": N.f64(chain.velocity_limits), "acc": N.f64(chain.accel_limits),
        "p0": N.f64(chain.cap_p0).reshape(-1, 3), "p1": N.f64(chain.cap_p1).reshape(-1, 3),
        "r": N.f64(chain.cap_r), "link": N.i64(chain.cap_link),
        "pa": N.i64(chain.pair_a), "pb": N.i64(chain.pair_b),
    }
    d = N.ChainDesc()
    d.dof = chain.dof
    d.task_dim = int(chain.task_dim)
    d.n_caps = int(keep["r"].shape[0])
    d.n_pairs = int(keep["pa"].shape[0])
    d.axes, d.origin_rot, d.origin_trans = N.dptr(keep["axes"]), N.dptr(keep["orot"]), N.dptr(keep["otrans"])
    d.jtype = N.lptr(keep["jtype"])
    d.joint_limits, d.velocity_limits, d.accel_limits = N.dptr(keep["lim"]), N.dptr(keep["vel"]), N.dptr(keep["acc"])
    d.cap_p0, d.cap_p1, d.cap_r = N.dptr(keep["p0"]), N.dptr(keep["p1"]), N.dptr(keep["r"])
    d.cap_link, d.pair_a, d.pair_b = N.lptr(keep["link"]), N.lptr(keep["pa"]), N.lptr(keep["pb"])
    return d, keep


def cost_desc(weights, provider_kind: int) -> N.CostDesc:
    c = N.CostDesc()
    for i in range(3):
        c.alpha_rot[i] = float(weights.alpha_rot[i])
        c.alpha_trans[i] = float(weights.alpha_trans[i])
    c.alpha_stop = float(weights.alpha_stop)
    c.alpha_joint = float(weights.alpha_joint)
    c.alpha_manip = float(weights.alpha_manip)
    c.alpha_coll = float(weights.alpha_coll)
    c.k_jl = float(weights.k_jl)
    c.k_m = float(weights.k_m)
    c.self_collision = int(provider_kind)
    return c


def provider_kind(provider) -> int:
    if provider is None:
        return N.SELFCOLL_NONE
    kind = getattr(provider, "kind", None)
    if kind == "oracle":
        return N.SELFCOLL_ORACLE
    if kind == "learned":
        return N.SELFCOLL_LEARNED
    raise ConfigError(f"unknown self-collision provider kind {kind!r}")


class Plan:
    """Owns one ``mppi_plan``. Not thread safe (like the reference Controller)."""

    def __init__(self, chain, weights, spec: PlanSpec, provider=None, world=None):
        N.require_device()
        self.lib = N.load_library()
        self.chain = chain
        self.spec = spec
        self.dof = chain.dof
        self.kind = provider_kind(provider)
        cd, self._keep_chain = chain_desc(chain)
        wd = cost_desc(weights, self.kind)
        self._dts = N.f64(spec.dts)
        pd = N.PlanDesc()
        for name in ("horizon", "particles", "null_count", "instances", "iterations", "policy_mode",
                     "precision", "generator", "smoothing", "spline_degree", "knots", "device",
                     "particle_offset", "particles_total", "dump"):
            setattr(pd, name, int(getattr(spec, name)))
        pd.seed = int(spec.seed) & ((1 << 64) - 1)
        for i in range(3):
            pd.comb[i] = float(spec.comb[i])
        for name in ("gamma", "terminal_weight", "beta", "alpha_mu", "alpha_sigma", "sigma0_sq",
                     "sigma_sq_min", "sigma_sq_max", "default_tail"):
            setattr(pd, name, float(getattr(spec, name)))
        pd.dts = N.dptr(self._dts)
        h = C.c_void_p()
        N.check(self.lib.mppi_plan_create(C.byref(cd), C.byref(wd), C.byref(pd), C.byref(h)))
        self.handle = h
        self.B = spec.instances
        self.H = spec.horizon
        self.N = spec.particles
        self._cmd = np.empty((self.B, self.dof))
        self._info = (N.StepInfo * self.B)()
        self._th = np.zeros((self.B, self.dof))
        self._thd = np.zeros((self.B, self.dof))
        self._p_th, self._p_thd, self._p_cmd = N.dptr(self._th), N.dptr(self._thd), N.dptr(self._cmd)
        self._step_fn = self.lib.mppi_step
        # address-level entry for the single-controller latency path: caller
        # arrays go straight to mppi_step (it copies them into pinned staging)
        proto = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
        self._step_raw = proto(C.cast(self.lib.mppi_step, C.c_void_p).value)
        self._a_cmd, self._a_info = self._cmd.ctypes.data, C.addressof(self._info)
        # staging rows of instance 0 and every address the latency path passes,
        # resolved once (an ndarray's .ctypes.data costs ~1-2 us per access,
        # more than copying 7 doubles into a staging row)
        self._th0, self._thd0 = self._th[0], self._thd[0]
        self._a_th, self._a_thd = self._th.ctypes.data, self._thd.ctypes.data
        self._h = self.handle.value
        self.profile_level = 0  # device stage times are only filled when profiling
        self._fn = C.cast(self.lib.mppi_step, C.c_void_p).value
        self._fast = N.fast_module() if self.B == 1 else None
        # the same memory as a numpy record array: batched callers read whole
        # columns (status, costs) without touching B ctypes structs
        self.info_columns = np.ctypeslib.as_array(self._info)
        if provider is not None and self.kind == N.SELFCOLL_LEARNED:
            self.set_mlp(provider)
        if world is not None:
            self.set_world(world)

    # ---------------------------------------------------------------- lifecycle
    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.mppi_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- setup
    def init_noise(self):
        N.check(self.lib.mppi_init_noise(self.handle, None))

    def set_noise(self, eps):
        eps = N.f64(eps, (self.N, self.H, self.dof))
        N.check(self.lib.mppi_set_noise(self.handle, N.dptr(eps)))

    def get_noise(self) -> np.ndarray:
        out = np.empty((self.N, self.H, self.dof))
        N.check(self.lib.mppi_get_noise(self.handle, N.dptr(out)))
        return out

    def set_goal(self, rotation, translation, mode: int, instance: int = -1):
        R = N.f64(rotation, (3, 3))
        t = N.f64(translation, (3,))
        N.check(self.lib.mppi_set_goal(self.handle, int(instance), N.dptr(R), N.dptr(t), int(mode)))

    def set_goals(self, rotations, translations, modes, first: int = 0):
        R = N.f64(rotations).reshape(-1, 9)
        t = N.f64(translations).reshape(-1, 3)
        m = np.ascontiguousarray(np.asarray(modes, dtype=np.int32).reshape(-1))
        N.check(self.lib.mppi_set_goals(self.handle, int(first), R.shape[0], N.dptr(R), N.dptr(t),
                                        m.ctypes.data_as(C.POINTER(C.c_int32))))

    def set_world(self, world):
        grid = getattr(world, "voxel_grid", None)
        sp = N.f64(world.spheres).reshape(-1, 4)
        if grid is not None:
            occ = np.ascontiguousarray(grid.occupancy, dtype=np.uint8)
            nx, ny, nz = occ.shape
            origin = N.f64(grid.origin, (3,))
            N.check(self.lib.mppi_set_voxel_world(
                self.handle, occ.ctypes.data_as(C.POINTER(C.c_uint8)), nx, ny, nz, N.dptr(origin),
                float(grid.voxel), N.dptr(sp), sp.shape[0]))
        else:
            bx = N.f64(world.boxes).reshape(-1, 6)
            N.check(self.lib.mppi_set_world(self.handle, N.dptr(sp), sp.shape[0], N.dptr(bx), bx.shape[0]))

    def set_mlp(self, provider):
        net = provider.net
        Ws = [N.f64(w) for w in net.weights]
        bs = [N.f64(b) for b in net.biases]
        if len(Ws) != 4 or Ws[0].shape[1] != 256 or Ws[1].shape != (256, 128) or Ws[2].shape != (128, 64) \
                or Ws[3].shape != (64, 1):
            raise ConfigError("surrogate must be the (2d)->256->128->64->1 net of surrogate.py:21")
        args = []
        for W, b in zip(Ws, bs):
            args += [N.dptr(W), N.dptr(b)]
        self._keep_mlp = (Ws, bs)
        N.check(self.lib.mppi_set_mlp(self.handle, Ws[0].shape[0], *args))

    def set_policy(self, means, variances, instance: int = 0):
        m = N.f64(means, (self.H, self.dof))
        v = N.f64(variances)
        if v.ndim == 1:  # isotropic storage is replicated per joint
            v = np.repeat(v[:, None], self.dof, axis=1)
        v = np.ascontiguousarray(v.reshape(self.H, self.dof))
        N.check(self.lib.mppi_set_policy(self.handle, int(instance), N.dptr(m), N.dptr(v)))

    def get_policy(self, instance: int = 0):
        m = np.empty((self.H, self.dof))
        v = np.empty((self.H, self.dof))
        N.check(self.lib.mppi_get_policy(self.handle, int(instance), N.dptr(m), N.dptr(v)))
        return m, v

    # ---------------------------------------------------------------- hot path
    def step(self, theta, theta_dot):
        """One control step for all instances. Returns (commands (B,d), infos).

        The host side of the hot path: inputs are copied into pre-pinned
        staging arrays whose ctypes pointers are built once, so a step costs
        one ctypes call (H2D, graph replay and the mapped D2H happen inside).
        """
        np.copyto(self._th, np.reshape(theta, self._th.shape))
        np.copyto(self._thd, np.reshape(theta_dot, self._thd.shape))
        rc = self._step_fn(self.handle, self._p_th, self._p_thd, self._p_cmd, self._info)
        if rc:
            N.check(rc)
        return self._cmd.copy(), self._info

    def step_single(self, theta, theta_dot):
        """step() for B = 1 with float64 (d,) inputs: no staging copies on the
        Python side. Returns (command (d,) view of the plan's output buffer,
        info of instance 0); the view is overwritten by the next step."""
        if self._fast is not None:  # caller float64 vectors straight to mppi_step (csrc/mppi_fast.c)
            rc = self._fast.step(self._fn, self._h, theta, theta_dot, self._a_cmd, self._a_info, self.dof)
            if rc is not NotImplemented:
                if rc:
                    N.check(rc)
                return self._cmd[0], self._info[0]
        if (type(theta) is np.ndarray and type(theta_dot) is np.ndarray and theta.shape == self._th0.shape
                and theta_dot.shape == self._th0.shape):
            np.copyto(self._th0, theta)  # any real dtype / layout: numpy converts while copying
            np.copyto(self._thd0, theta_dot)
            rc = self._step_raw(self._h, self._a_th, self._a_thd, self._a_cmd, self._a_info)
            if rc:
                N.check(rc)
            return self._cmd[0], self._info[0]
        cmds, infos = self.step(theta, theta_dot)
        return self._cmd[0], infos[0]

    def profile_stages(self, level: int = 2):
        """0: lean graph, no timing; 1: device_ms of the lean graph; 2: the
        instrumented graph with per-stage event times (see mppi_profile_stages)."""
        N.check(self.lib.mppi_profile_stages(self.handle, int(level)))
        self.profile_level = int(level)

    def evaluate(self, mode: int, inputs0, inputs1, dts, gamma, terminal_weight, theta0=None,
                 theta_dot0=None, want=("positions", "velocities", "accelerations", "step_costs",
                                        "terms", "totals")):
        in0 = N.f64(inputs0)
        n, H, d = in0.shape
        in1 = N.f64(inputs1) if inputs1 is not None else None
        out = N.EvalOut()
        res = {}
        shapes = {"positions": (n, H, d), "velocities": (n, H, d), "accelerations": (n, H, d),
                  "step_costs": (n, H), "terms": (6, n, H), "totals": (n,)}
        for k in want:
            res[k] = np.empty(shapes[k])
            setattr(out, k, N.dptr(res[k]))
        dts = N.f64(dts)
        th0 = N.f64(theta0) if theta0 is not None else None
        thd0 = N.f64(theta_dot0) if theta_dot0 is not None else None
        rc = self.lib.mppi_evaluate(self.handle, int(mode), n, H, N.dptr(dts), float(gamma),
                                    float(terminal_weight), N.dptr(th0), N.dptr(thd0), N.dptr(in0),
                                    N.dptr(in1), C.byref(out))
        N.check(rc)
        res["quarantined"] = int(out.quarantined)
        return res

    def get_step_inputs(self, instance: int = 0):
        """(theta, theta_dot, means, stddev) the last step's last iteration ran from."""
        th, thd = np.empty(self.dof), np.empty(self.dof)
        m, sd = np.empty((self.H, self.dof)), np.empty((self.H, self.dof))
        N.check(self.lib.mppi_get_step_inputs(self.handle, int(instance), N.dptr(th), N.dptr(thd), N.dptr(m),
                                              N.dptr(sd)))
        return th, thd, m, sd

    def replay_bundle(self) -> dict:
        """The last step's last-iteration RolloutBundle of a lean plan (dump=0),
        recomputed on the device from its inputs (mppi_replay_bundle): controls
        from the perturbation block and the policy view of that iteration, one
        evaluation pass (rollout, cost stack, MLP, discounted totals) and the
        particle weights. Equal to the step's own rollouts up to the plan
        precision's rounding."""
        return self._bundle(self.lib.mppi_replay_bundle)

    def _bundle(self, fn) -> dict:
        from .costs import TERM_NAMES

        n, H, d = self.N, self.H, self.dof
        res = {"positions": np.empty((n, H, d)), "velocities": np.empty((n, H, d)),
               "accelerations": np.empty((n, H, d)), "step_costs": np.empty((n, H)),
               "terms": np.empty((6, n, H)), "totals": np.empty(n), "weights": np.empty(n)}
        out = N.EvalOut()
        for k in ("positions", "velocities", "accelerations", "step_costs", "terms", "totals"):
            setattr(out, k, N.dptr(res[k]))
        N.check(fn(self.handle, C.byref(out), N.dptr(res["weights"])))
        return {"positions": res["positions"], "velocities": res["velocities"],
                "accelerations": res["accelerations"], "step_costs": res["step_costs"],
                "term_breakdown": {nm: res["terms"][i] for i, nm in enumerate(TERM_NAMES)},
                "total_per_particle": res["totals"], "weights": res["weights"]}

    def get_bundle(self) -> dict:
        """Instance 0's last-iteration bundle (plan created with dump=1)."""
        return self._bundle(self.lib.mppi_get_bundle)

    def episode(self, steps: int, dt: float, filter_lambda: float, theta0, theta_dot0, *,
                prev_command=None, fallback_armed: bool = False, script=None, noise=None) -> dict:
        """Closed-loop episode on the device (mppi_episode). ``script`` is
        (times (W,), positions (W,3), interpolation code, goal-mode code) or
        None for the plan's current goal; ``noise`` (steps, 2d) are the plant
        noise draws. Returns the log columns trimmed to the steps run, the
        final filter / fallback / plant state and the device time."""
        d, S = self.dof, int(steps)
        desc = N.EpisodeDesc()
        desc.steps = S
        desc.dt = float(dt)
        desc.filter_lambda = float(filter_lambda)
        keep = []
        if script is not None:
            times, positions, interp, mode = script
            times = N.f64(times)
            positions = N.f64(positions).reshape(-1, 3)
            keep += [times, positions]
            desc.goal_source = N.GOAL_SCRIPT
            desc.interpolation = int(interp)
            desc.script_mode = int(mode)
            desc.waypoints = times.shape[0]
            desc.times = N.dptr(times)
            desc.positions = N.dptr(positions)
        if noise is not None:
            noise = N.f64(noise).reshape(S, 2 * d)
            keep.append(noise)
            desc.noise = N.dptr(noise)
        st = N.EpisodeState()
        if prev_command is not None:
            for j in range(d):
                st.prev_command[j] = float(prev_command[j])
        st.fallback_armed = int(bool(fallback_armed))
        S1 = max(S, 1)
        cols = {"t": np.zeros(S1), "theta": np.zeros((S1, d)), "theta_dot": np.zeros((S1, d)),
                "command": np.zeros((S1, d)), "goal": np.zeros((S1, 3)), "goal_rot": np.zeros((S1, 9)),
                "ee": np.zeros((S1, 3)), "ee_rot": np.zeros((S1, 9)), "cost_total": np.zeros(S1),
                "cost_terms": np.zeros((6, S1))}
        icols = {k: np.zeros(S1, dtype=np.int32) for k in ("collision", "fallback", "status")}
        lg = N.EpisodeLogC()
        for k, v in cols.items():
            setattr(lg, k, N.dptr(v))
        for k, v in icols.items():
            setattr(lg, k, v.ctypes.data_as(C.POINTER(C.c_int32)))
        done = C.c_int32(0)
        ms = C.c_double(0.0)
        th0 = N.f64(theta0, (d,))
        thd0 = N.f64(theta_dot0, (d,))
        N.check(self.lib.mppi_episode(self.handle, C.byref(desc), N.dptr(th0), N.dptr(thd0), C.byref(st),
                                      C.byref(lg), C.byref(done), C.byref(ms)))
        n = int(done.value)
        out = {k: (v[:, :n] if k == "cost_terms" else v[:n]) for k, v in cols.items()}
        out.update({k: v[:n] for k, v in icols.items()})
        out["steps_done"] = n
        out["device_ms"] = float(ms.value)
        out["aborted"] = bool(st.aborted)
        out["fallback_armed"] = bool(st.fallback_armed)
        out["last_estimate"] = np.array(st.last_estimate[:2 * d])
        out["last_command"] = np.array(st.last_command[:d])
        out["prev_command"] = np.array(st.prev_command[:d])
        out["plant"] = np.array(st.plant[:2 * d])
        return out

    def time_stage(self, stage: int, reps: int = 50) -> float:
        """Mean device ms per launch of one stage (0 rollout, 1 MLP, 2 stats, 3 whole graph)."""
        ms = C.c_double(0.0)
        N.check(self.lib.mppi_time_stage(self.handle, int(stage), int(reps), C.byref(ms)))
        return float(ms.value)

    def mlp_forward(self, q) -> np.ndarray:
        q = N.f64(q).reshape(-1, self.dof)
        out = np.empty(q.shape[0])
        N.check(self.lib.mppi_mlp_forward(self.handle, N.dptr(q), q.shape[0], N.dptr(out)))
        return out

    # ---------------------------------------------------------------- sharded update
    def record_len(self) -> int:
        n = C.c_int32(0)
        N.check(self.lib.mppi_stats_record_len(self.handle, C.byref(n)))
        return int(n.value)

    def stats_dev(self, theta, theta_dot, record_ptr: int, stream_ptr: int = 0):
        th = N.f64(theta, (self.dof,)) if theta is not None else None
        thd = N.f64(theta_dot, (self.dof,)) if theta_dot is not None else None
        N.check(self.lib.mppi_stats_dev(self.handle, N.dptr(th), N.dptr(thd), C.c_void_p(record_ptr),
                                        C.c_void_p(stream_ptr or None)))

    # ---- exchange over peer memory (mppi_step_exchange)
    def peer_buffers(self, world: int) -> tuple[int, int]:
        """(receive buffer, flags) device pointers of this rank for `world` ranks."""
        r, f = C.c_void_p(), C.c_void_p()
        N.check(self.lib.mppi_peer_buffers(self.handle, int(world), C.byref(r), C.byref(f)))
        return int(r.value), int(f.value)

    def set_peers(self, rank: int, recv_ptrs, flag_ptrs):
        world = len(recv_ptrs)
        rv = (C.c_void_p * world)(*[C.c_void_p(int(x)) for x in recv_ptrs])
        fv = (C.c_void_p * world)(*[C.c_void_p(int(x)) for x in flag_ptrs])
        N.check(self.lib.mppi_set_peers(self.handle, world, int(rank), rv, fv))

    def set_exchange_timeout(self, seconds: float):
        N.check(self.lib.mppi_set_exchange_timeout(self.handle, float(seconds)))

    def exchange_abort(self):
        """Abandon this rank's next exchange step (publishes an abort to every rank)."""
        N.check(self.lib.mppi_exchange_abort(self.handle))

    def step_exchange(self, theta, theta_dot):
        cmd = np.empty(self.dof)
        info = N.StepInfo()
        N.check(self.lib.mppi_step_exchange(self.handle, N.dptr(N.f64(theta, (self.dof,))),
                                            N.dptr(N.f64(theta_dot, (self.dof,))), N.dptr(cmd), C.byref(info)))
        return cmd, info

    def ipc_handle(self, ptr: int) -> bytes:
        buf = C.create_string_buffer(64)
        N.check(self.lib.mppi_ipc_get_handle(C.c_void_p(int(ptr)), buf))
        return buf.raw

    def ipc_open(self, handle: bytes) -> int:
        out = C.c_void_p()
        N.check(self.lib.mppi_ipc_open_handle(bytes(handle), C.byref(out)))
        return int(out.value)

    def ipc_close(self, ptr: int):
        N.check(self.lib.mppi_ipc_close(C.c_void_p(int(ptr))))

    def finalize_dev(self, records_ptr: int, n_records: int, stream_ptr: int = 0):
        cmd = np.empty(self.dof)
        info = N.StepInfo()
        N.check(self.lib.mppi_finalize_dev(self.handle, C.c_void_p(records_ptr), int(n_records),
                                           N.dptr(cmd), C.byref(info), C.c_void_p(stream_ptr or None)))
        return cmd, info
