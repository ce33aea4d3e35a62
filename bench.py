"""Benchmark: MPC step latency of the B200 MPPI step (BASELINE config 2) and
particle-steps/s of the batched-controller config at 1/2/4/8 GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload auto|c1|c2|c3|c4|c5] [--precision fp32|fp64] [--dry-run]

``--workload auto`` (default): config 2 (BASELINE configs[1], the latency
headline) at N=1; config 4 (4096 controllers, instance-sharded, whole-job
particle-steps/s) at N>1. ``--gpus N`` without torchrun's environment
re-executes this script under ``torch.distributed.run`` with N ranks on
127.0.0.1; under torchrun, WORLD_SIZE must equal N. ``--dry-run`` checks that
plumbing without a GPU (gloo, no device work).

Config 2 (N=1): arm7 (the reference's Franka model) reach task, 500 particles
x H=30, full cost stack (pose, joint limits, braking envelope,
manipulability, learned self-collision MLP), Halton + B-spline sampling, FP32
fused rollout. A "step" is one Controller.control_step (shift + sample +
rollout/costs + MLP + weights/update + command).

* value: mean device time of the lean step graph's replay (two CUDA events on
  the plan stream around it), L2 flushed (256 MiB memset) before every step.
* e2e: mean wall time of Controller.control_step (the public API) with host
  buffers: H2D of the joint state, graph replay, mapped D2H of command + status.
* fp64: the same two numbers for the float64 plan.
* bundle: the device time of the step graph that also dumps the rollout
  bundle (keep_bundle=True) and the first-access cost of the lean graph's
  replayed StepDiagnostics.bundle.
* roofline / kernels / stage_ms: per-kernel device times from a second timed
  pass over the instrumented copy of the graph (event-record nodes between the
  stages); the dominant kernel is the one with the largest share of the step
  in the committed ncu launch list of this command (profiles/), falling back
  to the event times.
* cpu_baseline: the unmodified reference (oracle/_ref, numba backend) timed
  on this host (SURVEY §8(d) protocol: workers = all threads and workers = 1
  with single-threaded BLAS, config 4 from 8 instances x 512 "extrapolated",
  config 5 measured to N = 32768 and extrapolated linearly beyond).

Multi-GPU: configs 1-3 do not shard: each rank runs a replica
and the latency is the max over ranks. Config 4 splits the instances over the
ranks with no data-path collective; config 5 splits one controller's
particles with one record exchange per iteration.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MPC step latency (ms) @500×H30 Franka; particle-steps/sec at 1/2/4/8 GPUs"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


def _ncu_summary(tag: str):
    """The newest committed ncu summary profiles/r*_<tag>.json (list of launches)."""
    files = sorted((ROOT / "profiles").glob(f"r*_{tag}.json"))
    if not files:
        return None, None
    try:
        return json.loads(files[-1].read_text()), f"profiles/{files[-1].name}"
    except (OSError, ValueError):
        return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        # NVML polled from a thread every 5 ms (nvidia-smi's -lms floor is too coarse
        # for sub-second timed regions); nvidia-smi is the fallback
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}

            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def sample():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                act = ["Active" if r & b else "Not Active" for b in bits.values()]
                self.lines.append(f"{sm}, {mx}, {r}, " + ", ".join(act))

            def poll():
                while not self._stop.is_set():
                    sample()
                    time.sleep(0.005)

            self._sample = sample
            sample()  # one sample at the start of the timed region, however short it is
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self._stop.set()
        if getattr(self, "_sample", None) is not None:  # one sample at the end of the timed region
            try:
                self._sample()
            except Exception:
                pass
        if getattr(self, "t", None) is not None and self.proc is None:
            self.t.join(timeout=1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _spawn(args) -> int:
    """--gpus N without torchrun's environment: re-execute under
    torch.distributed.run with N local ranks on 127.0.0.1."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def _maybe_init_dist(ws, local):
    if ws <= 1:
        return None
    # the communicator lines (rank count, NVLink/NVLS transport) on the init, so
    # the rank check is observable in the log
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import torch
    import torch.distributed as dist

    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {local} needs GPU {local}, but only {torch.cuda.device_count()} "
                         "visible (one process per GPU)")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist


def _max_over_ranks(dist, x: float, local: int) -> float:
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- workloads
L2_NOTE = "GPU arm: 256 MiB memset (> 126 MB L2) before every timed step; CPU arm: no flush"


def workload_config(workload: str, args, ws: int) -> dict:
    """The `config` object of a workload: the SAME dict on both arms."""
    if workload in ("c1", "c2"):
        cfg = 1 if workload == "c1" else 2
        return {"workload": f"config{cfg}: arm7 reach, "
                            + ("full cost stack + learned self-collision MLP" if cfg == 2
                               else "goal pose + joint limits")
                            + f", {args.particles} particles x H30, K=1",
                "particles": args.particles, "horizon": 30, "iterations": 1,
                "parallelism": f"replicas x{ws}" if ws > 1 else "single", "l2": L2_NOTE}
    if workload == "c3":
        return {"workload": f"config3: moving-target tracking, 64^3 voxel world (8 boxes), {args.particles} x H30, "
                            "closed loop", "particles": args.particles, "horizon": 30,
                "parallelism": f"replicas x{ws}" if ws > 1 else "single", "l2": L2_NOTE}
    if workload == "c4":
        return {"workload": f"config4: {args.instances} arm7 controllers x {args.particles} particles x H30, "
                            "config-2 cost stack (learned MLP), instance-sharded",
                "instances": args.instances, "particles": args.particles, "horizon": 30,
                "parallelism": f"instance-sharded x{ws}", "l2": L2_NOTE}
    return {"workload": f"config5: one controller, {args.particles} particles x H30, config-2 costs, "
                        + (f"particle-sharded x{ws}, 1 record exchange/iteration" if ws > 1 else "single GPU"),
            "particles": args.particles, "horizon": 30, "l2": L2_NOTE}


# ---------------------------------------------------------------- reference arm (CPU)
def _reference_controller(particles=500, workers=None, config=2, world=None, goal=None):
    """The unmodified reference from oracle/_ref (bench-only): a Controller of
    BASELINE config 1/2/3 built from the same numbers as ours (configs.py)."""
    sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    from jointmpc.controller import Controller
    from jointmpc.costs import FULL_POSE, CostWeights, GoalSpec
    from jointmpc.kinematics import Pose, _rpy_matrix, load_chain
    from jointmpc.rollout import JointState
    from jointmpc.surrogate import LearnedSelfCollision

    from paper_2104_13542_b200 import configs

    kw = dict(configs.CONTROLLER_KW)
    kw["particles"] = particles
    kw["workers"] = workers or (os.cpu_count() or 1)
    if goal is None:
        goal = GoalSpec(target_pose=Pose(rotation=_rpy_matrix(*configs.REACH_GOAL_RPY),
                                         translation=configs.REACH_GOAL_POS.copy()), mode=FULL_POSE)
    surr = (LearnedSelfCollision.load(ROOT / "paper_2104_13542_b200" / "data" / "arm7_surrogate.npz")
            if config == 2 else None)
    c = Controller(load_chain("arm7.chain"), goal, weights=CostWeights(**configs.WEIGHTS[config]),
                   self_collision=surr, world=world, **kw)
    st = JointState(theta=configs.REACH_START.copy(), theta_dot=np.zeros(7), theta_ddot=np.zeros(7))
    return c, st


def _have_reference() -> bool:
    return (ROOT / "oracle" / "_ref" / "jointmpc" / "controller.py").exists()


def _port_controller(particles=500, config=2):
    """The oracle port (oracle/mppi_oracle.py) of the same step: the CPU
    baseline when the reference itself is not installed (bench-only)."""
    from oracle import mppi_oracle as O
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import ARM7_SURROGATE

    with np.load(ARM7_SURROGATE) as z:
        mlp = {k: z[k] for k in z.files if k.startswith(("W", "b"))}
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = particles
    return O.OracleController(load_chain("arm7.chain"), configs.make_weights(config), configs.reach_goal_rotation(),
                              configs.REACH_GOAL_POS, True, provider="learned" if config == 2 else None,
                              mlp_state=mlp, **kw)


def _cpu_stepper(particles=500, config=2, workers=None):
    """(step(), workers, kind) for one reference (or port) controller."""
    if _have_reference():
        c, st = _reference_controller(particles, workers, config)
        return (lambda: c.control_step(st)), c.workers, "reference"
    from paper_2104_13542_b200 import configs

    oc = _port_controller(particles, config)
    th = configs.REACH_START.copy()
    return (lambda: oc.step(th, np.zeros(7))), 1, "port"


def _time_steps(step, steps: int, warmup: int, budget_s: float | None = None):
    for _ in range(max(1, warmup)):
        step()
    lat = []
    t_end = time.perf_counter() + budget_s if budget_s else None
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        step()
        lat.append((time.perf_counter() - t0) * 1e3)
        if t_end and time.perf_counter() > t_end and len(lat) >= 3:
            break
    return lat


def _cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


def _cpu_probe(spec: dict) -> dict:
    """One measurement of the CPU protocol (run in a subprocess so the thread
    environment, e.g. single-threaded BLAS, applies from the first import)."""
    kind = spec["kind"]
    w = spec.get("workers")
    if _have_reference():
        sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    if kind == "latency":  # latency_probe (reference bench.py:91-109)
        step, workers, impl = _cpu_stepper(spec.get("particles", 500), spec.get("config", 2), w)
        lat = _time_steps(step, spec.get("steps", 10), spec.get("warmup", 1), spec.get("budget_s"))
        return {"median_ms": float(np.median(lat)), "mean_ms": float(np.mean(lat)), "steps": len(lat),
                "workers": workers, "kind": impl}
    if kind == "instances":  # config 4 sample: k independent controllers stepped in sequence
        from paper_2104_13542_b200 import configs

        k = spec["k"]
        lat = []
        impl = "reference"
        for i in range(k):
            if _have_reference():
                from jointmpc.costs import FULL_POSE, GoalSpec
                from jointmpc.kinematics import Pose

                goals, th0 = _c4_problem_host(i)
                g = GoalSpec(target_pose=Pose(rotation=goals[0], translation=goals[1]), mode=FULL_POSE)
                c, st = _reference_controller(500, w, 2, goal=g)
                st.theta = th0
                step = lambda: c.control_step(st)  # noqa: E731
            else:
                step, _, impl = _cpu_stepper(500, 2, w)
            lat += _time_steps(step, 1, 1)
        return {"per_instance_step_ms": float(np.mean(lat)), "instances_timed": k, "kind": impl}
    raise ValueError(kind)


def _c4_problem_host(i: int):
    """Config-4 instance i's goal (R, t) and start state, computed on the host
    with the reference's FK (no device needed in the CPU arm)."""
    from jointmpc.kinematics import fk_batch, load_chain

    from paper_2104_13542_b200 import configs

    chain = load_chain("arm7.chain")
    lo, hi = chain.joint_limits[:, 0], chain.joint_limits[:, 1]
    k = 0.1
    lo_s, hi_s = lo + k * (hi - lo), hi - k * (hi - lo)
    q = np.random.default_rng(i).uniform(lo_s, hi_s)
    th0 = np.random.default_rng(10000 + i).uniform(lo_s, hi_s)
    rot, trans = fk_batch(chain, q[None])
    return (rot[0, -1], trans[0, -1]), th0


def _probe_subprocess(spec: dict, single_thread: bool = False, timeout: float = 300.0) -> dict:
    env = dict(os.environ)
    env.pop("OMP_NUM_THREADS", None)  # torchrun's per-rank pin does not apply to the CPU arm
    if single_thread:
        for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
            env[k] = "1"
    r = subprocess.run([sys.executable, str(Path(__file__).resolve()), "--cpu-probe", json.dumps(spec)],
                       capture_output=True, text=True, env=env, timeout=timeout)
    for ln in r.stdout.splitlines()[::-1]:
        if ln.startswith("{"):
            return json.loads(ln)
    return {"error": (r.stderr or r.stdout)[-300:]}


def cpu_protocol(full: bool = True) -> dict:
    """SURVEY §8(d) CPU baseline protocol on this host: config 2 at workers =
    all threads and workers = 1 (single-threaded BLAS), config 4 from 8
    sequential instances x 512 ("extrapolated"), config 5 measured to N=32768
    and extrapolated linearly to 262144."""
    ncpu = os.cpu_count() or 1
    out = {"cpu_model": _cpu_model(), "host_threads": ncpu}
    out["c2_workers_all"] = _probe_subprocess({"kind": "latency", "config": 2, "steps": 20, "budget_s": 8.0})
    out["c2_workers_all_blas1"] = _probe_subprocess({"kind": "latency", "config": 2, "steps": 20, "budget_s": 8.0},
                                                    single_thread=True)
    out["c2_workers_1"] = _probe_subprocess({"kind": "latency", "config": 2, "workers": 1, "steps": 8,
                                             "budget_s": 6.0}, single_thread=True)
    if full:
        c4 = _probe_subprocess({"kind": "instances", "k": 8}, single_thread=True)
        c4["blas"] = "single-threaded (the reference's fastest setup at config 2)"
        if "per_instance_step_ms" in c4:  # 4096 instances stepped in sequence
            c4["extrapolated_step_s_4096"] = c4["per_instance_step_ms"] * 4096 / 1e3
            c4["extrapolated_particle_steps_per_s"] = 4096 * 500 * 30 / c4["extrapolated_step_s_4096"]
            c4["label"] = "extrapolated x512 from 8 sequential instances (workers = all threads, single-threaded BLAS)"
        out["c4"] = c4
        c5 = {}
        for n in (2048, 8192, 32768):
            r = _probe_subprocess({"kind": "latency", "config": 2, "particles": n, "steps": 2, "budget_s": 6.0},
                                  single_thread=True)
            if "median_ms" in r:
                c5[str(n)] = {"ms": r["median_ms"], "particle_steps_per_s": n * 30 / (r["median_ms"] * 1e-3)}
        if "32768" in c5:
            per = c5["32768"]["ms"] / 32768
            c5["extrapolated"] = {str(n): {"ms": per * n, "label": "linear from N=32768"}
                                  for n in (65536, 131072, 262144)}
        out["c5"] = c5
    return out


def run_reference(args, workload: str):
    """The reference's own CPU implementation on this host (rank 0 only), on
    our arm's workload, config, metric and unit."""
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    if ws > 1:
        # torchrun pins OMP_NUM_THREADS=1 in every rank; the CPU arm gets all
        # host threads, so rank 0 measures in a clean child process
        env = {k: v for k, v in os.environ.items()
               if k not in ("OMP_NUM_THREADS", "WORLD_SIZE", "RANK", "LOCAL_RANK", "LOCAL_WORLD_SIZE",
                            "GROUP_RANK", "ROLE_RANK", "ROLE_WORLD_SIZE", "GROUP_WORLD_SIZE")}
        env["MPPI_REF_REPORT_WS"] = str(ws)
        argv = [a for a in sys.argv[1:]]
        cmd = [sys.executable, str(Path(__file__).resolve()), *argv, "--gpus", "1", "--workload", workload]
        if "--weak" in cmd:
            cmd.remove("--weak")
            cmd += ["--instances", str(args.instances)]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True)
        line = next((ln for ln in r.stdout.splitlines()[::-1] if ln.startswith("{")), None)
        print(line if line else json.dumps({"impl": "reference", "unavailable": (r.stderr or "no output")[-200:]}))
        return 0
    ws = int(os.environ.get("MPPI_REF_REPORT_WS", ws))
    cores = os.cpu_count() or 1
    cfg = workload_config(workload, args, ws)
    extra = {}
    if workload in ("c1", "c2", "c3"):
        config = {"c1": 1, "c2": 2, "c3": 3}[workload]
        if workload == "c3" and _have_reference():
            c, st, set_goal = _reference_tracking(args.particles)
            i = [0]

            def step():
                set_goal(i[0] * 0.05)
                i[0] += 1
                c.control_step(st)

            workers, kind = c.workers, "reference"
            lat = _time_steps(step, min(args.steps, 5), 1)
            sample = f"{len(lat)} closed-loop tracking steps (8-box world, {args.particles} particles)"
        elif _have_reference():
            # the reference's best thread setup on this host: its rollout workers
            # and numpy's BLAS threads compete for the same cores, so all three
            # are measured (each in its own process, the thread environment set
            # before numpy loads) and the fastest is the reported arm
            spec = {"kind": "latency", "config": config, "particles": args.particles, "steps": args.steps,
                    "warmup": args.warmup, "budget_s": 60.0}
            runs = {"workers=all, default BLAS threads": _probe_subprocess(spec),
                    "workers=all, single-threaded BLAS": _probe_subprocess(spec, single_thread=True),
                    "workers=1, single-threaded BLAS": _probe_subprocess(dict(spec, workers=1), single_thread=True)}
            ok = {k: r for k, r in runs.items() if "mean_ms" in r}
            best = min(ok, key=lambda k: ok[k]["mean_ms"])
            r = ok[best]
            lat = [r["mean_ms"]]
            workers, kind = r["workers"], r["kind"]
            sample = (f"{r['steps']} control_steps of config {config} after {args.warmup} warm-up, the fastest of "
                      f"three thread setups ({best})")
            extra["thread_setups"] = {k: {"mean_ms": v.get("mean_ms"), "median_ms": v.get("median_ms")}
                                      for k, v in runs.items()}
            extra["median_ms"] = r["median_ms"]
        else:
            step, workers, kind = _cpu_stepper(args.particles, min(config, 2), None)
            lat = _time_steps(step, args.steps, args.warmup, budget_s=120.0)
            sample = f"{len(lat)} control_steps of config {config} after {args.warmup} warm-up"
        v, unit, hib = float(np.mean(lat)), "ms", False
        extra.setdefault("median_ms", float(np.median(lat)))
    elif workload == "c4":
        spec = {"kind": "instances", "k": max(2, min(8, args.steps))}
        if _have_reference():  # the faster of the two BLAS thread setups (see the config-2 arm)
            runs = [_probe_subprocess(spec), _probe_subprocess(spec, single_thread=True)]
            runs = [x for x in runs if "per_instance_step_ms" in x]
            r = min(runs, key=lambda x: x["per_instance_step_ms"]) if runs else _cpu_probe(spec)
        else:
            r = _cpu_probe(spec)
        per_ms = r["per_instance_step_ms"]
        step_s = per_ms * args.instances / 1e3
        v, unit, hib = args.instances * args.particles * 30 / step_s, "particle-steps/s", True
        kind, workers = r["kind"], cores
        sample = (f"{r['instances_timed']} sequential config-2 instances x {args.particles} particles, "
                  f"extrapolated x{args.instances // r['instances_timed']} to {args.instances} instances")
        extra["extrapolated"] = True
    else:
        n_meas = min(args.particles, 32768)
        if _have_reference():  # the faster of the two BLAS thread setups
            spec = {"kind": "latency", "config": 2, "particles": n_meas, "steps": min(args.steps, 3),
                    "warmup": 1, "budget_s": 60.0}
            runs = [_probe_subprocess(spec), _probe_subprocess(spec, single_thread=True)]
            runs = [x for x in runs if "median_ms" in x]
            best = min(runs, key=lambda x: x["median_ms"])
            lat, workers, kind = [best["median_ms"]] * best["steps"], best["workers"], best["kind"]
        else:
            step, workers, kind = _cpu_stepper(n_meas, 2, None)
            lat = _time_steps(step, min(args.steps, 3), 1, budget_s=60.0)
        ms = float(np.median(lat)) * args.particles / n_meas
        v, unit, hib = args.particles * 30 / (ms * 1e-3), "particle-steps/s", True
        sample = f"{len(lat)} control_steps at N={n_meas}" + (
            f", extrapolated linearly to N={args.particles}" if n_meas != args.particles else "")
    line = {
        "metric": METRIC, "value": v, "unit": unit, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": v if unit == "ms" else None, "higher_is_better": hib,
        "scaling": "weak" if workload != "c5" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg, "impl": "reference",
        "cpu_baseline": {"value": v, "unit": unit, "cores": workers if kind == "reference" else 1, "kind": kind,
                         "sample": sample + (", numba backend, workers=%d" % workers if kind == "reference"
                                             else ", oracle port (numpy float64; oracle/_ref not installed)")},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        **extra,
    }
    print(json.dumps(line))
    return 0


def _reference_tracking(particles: int):
    """Config 3 on the reference: the same script and box world (built with the
    reference's FK), goal from the script every step."""
    sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    from jointmpc.kinematics import fk_batch as rfk
    from jointmpc.simworld import TargetScript, WorldModel, target_at

    from paper_2104_13542_b200 import configs

    script, world = configs.tracking_problem(fk=rfk)
    rworld = WorldModel(spheres=np.zeros((0, 4)), boxes=world.boxes, bounds_min=np.full(3, -1.0),
                        bounds_max=np.full(3, 1.0))
    rs = TargetScript(times=script.times, positions=script.positions, interpolation="linear", mode="position_only")
    c, st = _reference_controller(particles, None, 3, world=rworld, goal=target_at(rs, 0.0))
    return c, st, (lambda t: c.set_goal(target_at(rs, t)))


# ---------------------------------------------------------------- our arm
def _flush_l2(buf):
    buf.zero_()


def run_ours(args):
    ws, rank, local = _dist_env()
    dist = _maybe_init_dist(ws, local)
    import torch

    torch.cuda.set_device(local)
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200 import _native as N

    N.require_device()
    peaks, peaks_kind = _peaks()
    particles = args.particles
    config = 1 if args.workload == "c1" else 2
    ctrl = configs.make_controller(config, particles=particles, device=local, precision=args.precision)
    plan = ctrl.plan
    st = configs.start_state()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    for _ in range(max(3, args.warmup)):
        ctrl.control_step(st)

    # ---- device-timed loop (value): the lean step graph between two CUDA
    # events on the plan stream, L2 flushed before each step
    theta = st.theta[None, :]
    thetad = st.theta_dot[None, :]
    plan.profile_stages(1)
    dev_ms = []
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        for _ in range(args.steps):
            _flush_l2(flush)
            torch.cuda.synchronize()
            _, infos = plan.step(theta, thetad)
            dev_ms.append(infos[0].device_ms)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    if dist is not None:
        dist.barrier()
    # ---- kernel attribution: the same steps through the instrumented graph
    # (event-record nodes between the stages), separately timed
    plan.profile_stages(2)
    for _ in range(3):
        plan.step(theta, thetad)
    stages = {"sample": [], "rollout": [], "mlp": [], "update": []}
    prof_ms = []
    for _ in range(args.steps):
        _flush_l2(flush)
        torch.cuda.synchronize()
        _, infos = plan.step(theta, thetad)
        inf = infos[0]
        prof_ms.append(inf.device_ms)
        stages["sample"].append(inf.sample_ms)
        stages["rollout"].append(inf.rollout_ms)
        stages["mlp"].append(inf.mlp_ms)
        stages["update"].append(inf.update_ms)
    plan.profile_stages(0)
    value_local = float(np.mean(dev_ms))
    value = _max_over_ranks(dist, value_local, local)

    # ---- end to end through the public API (Controller.control_step, host buffers), lean graph
    for _ in range(max(3, args.warmup)):  # untimed: back on the lean graph after the instrumented pass
        _flush_l2(flush)
        torch.cuda.synchronize()
        ctrl.control_step(st)
    e2e = []
    for _ in range(args.steps):
        _flush_l2(flush)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctrl.control_step(st)
        e2e.append((time.perf_counter() - t0) * 1e3)
    e2e_v = _max_over_ranks(dist, float(np.mean(e2e)), local)

    # ---- roofline of the dominant kernel (stage times from the timed replays)
    from paper_2104_13542_b200 import roofline as RL

    st_mean = {k: float(np.mean(v)) for k, v in stages.items()}
    rows = particles * 30
    ncu_sum, ncu_src = _ncu_summary("full_c2_metrics") if config == 2 else (None, None)
    share, share_src = RL.launch_shares(ROOT / "profiles", "bench_launches")
    roof = RL.step_roofline(st_mean, rows=rows, particles=particles, horizon=30, dof=7, config=config,
                            peaks=peaks, peaks_kind=peaks_kind, ncu_summary=ncu_sum, ncu_source=ncu_src,
                            ncu_share=share, ncu_share_source=share_src)
    kernels = RL.all_rooflines(st_mean, rows=rows, dof=7, config=config, peaks=peaks, peaks_kind=peaks_kind,
                               ncu_summary=ncu_sum, ncu_source=ncu_src)

    # ---- the float64 plan: the same lean-graph and end-to-end loops
    fp64 = None
    if args.precision == "fp32":
        c64 = configs.make_controller(config, particles=particles, device=local, precision="fp64")
        p64 = c64.plan
        for _ in range(3):
            c64.control_step(st)
        p64.profile_stages(1)
        d64 = []
        for _ in range(min(args.steps, 100)):
            _flush_l2(flush)
            torch.cuda.synchronize()
            _, inf64 = p64.step(theta, thetad)
            d64.append(inf64[0].device_ms)
        p64.profile_stages(0)
        e64 = []
        for _ in range(min(args.steps, 100)):
            _flush_l2(flush)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c64.control_step(st)
            e64.append((time.perf_counter() - t0) * 1e3)
        fp64 = {"value": _max_over_ranks(dist, float(np.mean(d64)), local), "unit": "ms",
                "e2e_ms": _max_over_ranks(dist, float(np.mean(e64)), local), "dtype": "f64",
                "note": "float64 plan (FP64 rollout/statistics; the MLP keeps its tensor-core split products)"}

    # ---- the rollout bundle: the dump graph (keep_bundle=True) and the lean
    # graph's replayed bundle on first access (StepDiagnostics.bundle)
    cdump = configs.make_controller(config, particles=particles, device=local, precision=args.precision,
                                    keep_bundle=True)
    for _ in range(3):
        cdump.control_step(st)
    cdump.plan.profile_stages(1)
    dd = []
    for _ in range(min(args.steps, 50)):
        _flush_l2(flush)
        torch.cuda.synchronize()
        _, infd = cdump.plan.step(theta, thetad)
        dd.append(infd[0].device_ms)
    rep = []
    for _ in range(5):
        _, diag = ctrl.control_step(st)
        t0 = time.perf_counter()
        diag.bundle.total_per_particle
        rep.append((time.perf_counter() - t0) * 1e3)
    bundle = {"keep_bundle_device_ms": float(np.mean(dd)),
              "lean_bundle_first_access_ms": float(np.median(rep)),
              "note": "diag.bundle is always set; the lean graph replays the step's last iteration on first access"}

    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": value, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": args.precision.replace("fp", "f"),
        "data": "synthetic (bundled arm7 chain, reach goal, Halton perturbations, trained surrogate)",
        "config": workload_config(args.workload, args, ws),
        "particle_steps_per_s": ws * particles * 30 / (value * 1e-3),
        "median_ms": float(np.median(dev_ms)), "p99_ms": float(np.percentile(dev_ms, 99)),
        "stage_ms": st_mean,
        "instrumented_step_ms": float(np.mean(prof_ms)),
        "e2e": {"value": e2e_v, "unit": "ms", "h2d_bytes_per_step": 2 * 7 * 8,
                "d2h_bytes_per_step": 7 * 8 + 80, "median_ms": float(np.median(e2e)),
                "api": "Controller.control_step"},
        "gpu_launches": args.steps * (3 if config == 2 else 2),
        "roofline": roof,
        "kernels": kernels,
        "clocks": clk.summary(),
        "timed_wall_s": t_wall,
        "fp64": fp64,
        "bundle": bundle,
    }
    if not args.no_scale_roofline:
        line["roofline_at_scale"] = _scale_roofline(args, local, peaks, peaks_kind)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = _cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def run_batched(args):
    """Config 4: B independent controllers, instances sharded over ranks, no
    data-path collective. value = whole-job particle-steps/s."""
    ws, rank, local = _dist_env()
    dist = _maybe_init_dist(ws, local)
    import torch

    torch.cuda.set_device(local)
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200 import _native as N
    from paper_2104_13542_b200 import roofline as RL
    from paper_2104_13542_b200.batched import BatchedController, shard_instances
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import load_arm7_surrogate

    N.require_device()
    peaks, peaks_kind = _peaks()
    B = args.instances
    a, b = shard_instances(B, ws, rank)
    goals, th0 = configs.batched_problem(b - a, first=a)
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = args.particles
    bc = BatchedController(load_chain("arm7.chain"), goals, weights=configs.make_weights(2),
                           self_collision=load_arm7_surrogate(), precision=args.precision, device=local, **kw)
    thd = np.zeros_like(th0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    # value: the lean step graph (the instance chunks' rollout and MLP
    # overlapped on two graph branches), device time between two events
    bc.plan.profile_stages(1)
    for _ in range(max(3, args.warmup)):
        bc.control_step(th0, thd)
    dev_ms, stages = [], {"sample": [], "rollout": [], "mlp": [], "update": []}
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            _flush_l2(flush)
            torch.cuda.synchronize()
            _, diag = bc.control_step(th0, thd)
            dev_ms.append(diag.device_ms)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    # stage attribution: the instrumented graph (stages in sequence, events between)
    bc.plan.profile_stages(2)
    for _ in range(2):
        bc.control_step(th0, thd)
    inst_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        _flush_l2(flush)
        torch.cuda.synchronize()
        _, diag = bc.control_step(th0, thd)
        inst_ms.append(diag.device_ms)
        for k in stages:
            stages[k].append(diag.stage_ms[k])
    step_ms = _max_over_ranks(dist, float(np.mean(dev_ms)), local)
    units = B * args.particles * 30
    value = units / (step_ms * 1e-3)
    e2e = []
    bc.plan.profile_stages(0)
    for _ in range(2):  # untimed: the level-0 graph is captured on its first replay
        bc.control_step(th0, thd)
    for _ in range(max(3, args.steps // 2)):
        _flush_l2(flush)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bc.control_step(th0, thd)
        e2e.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = _max_over_ranks(dist, float(np.mean(e2e)), local)
    st_mean = {k: float(np.mean(v)) for k, v in stages.items()}
    # the newest batch capture (scripts/profile_batched.py): 80 controllers (paired rollout), else 64
    ncu_sum, ncu_src = _ncu_summary("full_b80_metrics")
    ncu_rows = 80 * 500 * 30
    if ncu_sum is None:
        ncu_sum, ncu_src = _ncu_summary("full_b64_metrics")
        ncu_rows = 64 * 500 * 30
    roof = RL.step_roofline(st_mean, rows=(b - a) * args.particles * 30, particles=(b - a) * args.particles,
                            horizon=30, dof=7, config=2, peaks=peaks, peaks_kind=peaks_kind, ncu_summary=ncu_sum,
                            ncu_source=ncu_src, ncu_rows=ncu_rows)
    line = {
        "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak"
        if args.weak else "strong", "vs_baseline": None, "dtype": args.precision.replace("fp", "f"),
        "data": "synthetic (goal_i = FK(q_i), q_i, theta0_i from default_rng(i), default_rng(10000+i))",
        "config": workload_config("c4", args, ws), "instances_per_gpu": b - a,
        "stage_ms": st_mean, "instrumented_step_ms": float(np.mean(inst_ms)),
        "e2e": {"value": units / (e2e_ms * 1e-3), "unit": "particle-steps/s",
                "h2d_bytes_per_step": B * 14 * 8 // ws, "d2h_bytes_per_step": B * (7 * 8 + 80) // ws,
                "ms_per_step": e2e_ms, "api": "BatchedController.control_step"},
        "gpu_launches": args.steps * 3,
        "roofline": roof,
        "kernels": RL.all_rooflines(st_mean, rows=(b - a) * args.particles * 30, dof=7, config=2, peaks=peaks,
                                    peaks_kind=peaks_kind),
        "clocks": clk.summary(),
    }
    if dist is not None:  # every rank's own roofline and step time (instances differ per rank)
        mine = {"rank": rank, "instances": b - a, "step_ms": float(np.mean(dev_ms)), "stage_ms": st_mean,
                "roofline": roof, "clocks": line["clocks"]}
        allr = [None] * ws
        dist.all_gather_object(allr, mine)
        line["per_rank"] = allr
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def run_tracking(args):
    """Config 3: moving-target tracking with the 64^3 voxel world, closed loop
    (goal from the TargetScript at t = i*dt, plant = semi-implicit Euler)."""
    ws, rank, local = _dist_env()
    import torch

    torch.cuda.set_device(local)
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200 import _native as N
    from paper_2104_13542_b200 import roofline as RL
    from paper_2104_13542_b200.controller import Controller
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.simworld import target_at

    N.require_device()
    peaks, peaks_kind = _peaks()
    script, world = configs.tracking_problem()
    kw = dict(configs.CONTROLLER_KW)
    kw["particles"] = args.particles
    from paper_2104_13542_b200.controller import run_episode

    def make():
        return Controller(load_chain("arm7.chain"), target_at(script, 0.0), weights=configs.make_weights(3),
                          world=world, precision=args.precision, device=local, **kw)

    ctrl = make()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def loop(level, steps, record):
        """Host closed loop: goal from the script, plant = semi-implicit Euler."""
        ctrl.profile_stages(level)
        st = configs.start_state()
        out = []
        total = max(3, args.warmup) + steps
        for i in range(total):
            ctrl.set_goal(target_at(script, i * 0.05))
            _flush_l2(flush)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cmd, diag = ctrl.control_step(st)
            wall = (time.perf_counter() - t0) * 1e3
            if i >= total - steps:
                out.append(record(wall, ctrl.plan._info[0]))
            st.theta_dot = st.theta_dot + 0.05 * cmd
            st.theta = st.theta + 0.05 * st.theta_dot
        return out

    # the lean graph (value, e2e), then the instrumented graph (stage attribution)
    with ClockSampler(local) as clk:
        rec = loop(1, args.steps, lambda wall, inf: (wall, inf.device_ms))
    dev_ms = [d for _, d in rec]
    # end to end on the lean graph without device events (level 0), as the
    # config-2 line does: the events of level 1 are host calls inside control_step
    e2e = loop(0, args.steps, lambda wall, inf: wall)
    srec = loop(2, min(args.steps, 50), lambda wall, inf: (inf.sample_ms, inf.rollout_ms, inf.mlp_ms,
                                                          inf.update_ms))
    st_mean = {k: float(np.mean([r[j] for r in srec])) for j, k in enumerate(("sample", "rollout", "mlp",
                                                                                "update"))}
    value = float(np.mean(dev_ms))
    # the whole closed loop on the device (run_episode -> mppi_episode): one
    # graph replay per step, no host round trip, no L2 flush between steps
    ep_ctrl = make()
    pol0 = ep_ctrl.policy
    for _ in range(2):  # warm-up: graph capture, then the cached graph
        run_episode(ep_ctrl, configs.start_state(), script, args.steps)
    ep_ctrl.policy = pol0  # timed episode from the fresh controller state
    ep_ctrl._prev_command = np.zeros(7)
    ep_ctrl._fallback_armed = False
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lg = run_episode(ep_ctrl, configs.start_state(), script, args.steps)
    ep_wall = (time.perf_counter() - t0) * 1e3
    episode = {"api": "controller.run_episode (device loop)", "steps": int(lg.steps),
               "device_ms_per_step": float(np.mean(lg.latency_ms)),
               "e2e_ms_per_step": ep_wall / max(lg.steps, 1),
               "l2": "not flushed between steps (one device-resident loop)",
               "collisions": int(lg.collision.sum()),
               "final_goal_distance_m": float(np.linalg.norm(lg.ee[-1] - lg.goal[-1]))}
    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": value, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision.replace("fp", "f"), "data": "synthetic",
        "config": workload_config("c3", args, ws),
        "stage_ms": st_mean,
        "e2e": {"value": float(np.mean(e2e)), "unit": "ms", "h2d_bytes_per_step": 112 + 16 * 8,
                "d2h_bytes_per_step": 136, "api": "Controller.control_step + set_goal"},
        "gpu_launches": args.steps * 2,
        "roofline": RL.step_roofline(st_mean, rows=args.particles * 30, particles=args.particles, horizon=30,
                                     dof=7, config=1, peaks=peaks, peaks_kind=peaks_kind),
        "episode": episode, "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line))
    return 0


def run_sweep(args):
    """Config 5: one controller, N particles; 1 GPU = plain Controller, N GPUs =
    particle-sharded with one record all-gather per iteration."""
    ws, rank, local = _dist_env()
    dist = _maybe_init_dist(ws, local)
    import torch

    torch.cuda.set_device(local)
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200 import _native as N
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import load_arm7_surrogate

    N.require_device()
    Np = args.particles
    st = configs.start_state()
    if ws == 1:
        ctrl = configs.make_controller(2, particles=Np, precision=args.precision, device=local)
        step = lambda: ctrl.control_step(st)  # noqa: E731
    else:
        from paper_2104_13542_b200.sharded import PeerExchange, RecordExchange, ShardedController

        kw = dict(configs.CONTROLLER_KW)
        kw.pop("particles")
        # the record exchange fused into the statistics kernel over NVLink peer
        # memory; MPPI_EXCHANGE=nccl: one NCCL all-gather between two kernels
        nccl = os.environ.get("MPPI_EXCHANGE", "nccl") != "peer"
        ctrl = ShardedController(load_chain("arm7.chain"), configs.make_goal(2), particles=Np, world_size=ws,
                                 rank=rank, device=local, exchange=RecordExchange() if nccl else PeerExchange(),
                                 weights=configs.make_weights(2), self_collision=load_arm7_surrogate(),
                                 precision=args.precision, **kw)
        step = lambda: ctrl.control_step(st)  # noqa: E731
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    for _ in range(max(3, args.warmup)):
        step()
    times, walls = [], []
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            _flush_l2(flush)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s0.record()
            step()
            s1.record()
            torch.cuda.synchronize()
            walls.append((time.perf_counter() - t0) * 1e3)
            times.append(s0.elapsed_time(s1))
    ms = _max_over_ranks(dist, float(np.mean(times)), local)
    wall_ms = _max_over_ranks(dist, float(np.mean(walls)), local)
    line = {
        "metric": METRIC, "value": Np * 30 / (ms * 1e-3), "unit": "particle-steps/s", "n_gpus": ws,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.precision.replace("fp", "f"), "data": "synthetic",
        "config": workload_config("c5", args, ws),
        **({"exchange": "nccl all-gather" if nccl else "fused peer-memory push (NVLink P2P)"} if ws > 1 else {}),
        "e2e": {"value": Np * 30 / (wall_ms * 1e-3), "unit": "particle-steps/s", "h2d_bytes_per_step": 112,
                "d2h_bytes_per_step": 136, "wall_ms_per_step": wall_ms,
                "api": "Controller / ShardedController.control_step (host wall clock)"},
        "gpu_launches": args.steps * 3, "clocks": clk.summary(),
    }
    if ws == 1:  # per-kernel roofline from the instrumented graph (stage events)
        from paper_2104_13542_b200 import roofline as RL

        peaks, peaks_kind = _peaks()
        ctrl.profile_stages(2)
        stg = {"sample": [], "rollout": [], "mlp": [], "update": []}
        for _ in range(min(args.steps, 20)):
            _flush_l2(flush)
            torch.cuda.synchronize()
            ctrl.control_step(st)
            inf = ctrl.plan._info[0]
            for k in stg:
                stg[k].append(getattr(inf, f"{k}_ms"))
        ctrl.profile_stages(0)
        sm = {k: float(np.mean(v)) for k, v in stg.items()}
        line["stage_ms"] = sm
        line["roofline"] = RL.step_roofline(sm, rows=Np * 30, particles=Np, horizon=30, dof=7, config=2,
                                            peaks=peaks, peaks_kind=peaks_kind)
        line["kernels"] = RL.all_rooflines(sm, rows=Np * 30, dof=7, config=2, peaks=peaks, peaks_kind=peaks_kind)
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def _scale_roofline(args, local, peaks, peaks_kind, instances=256, steps=5):
    """The 500x30 step is latency-bound; the kernels' roofline
    fractions are measured on a config-4-shaped batch (instances x 500 x 30,
    same kernels, same cost stack) with CUDA-event stage times of the timed
    graph replays, L2 flushed before each step."""
    import torch

    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200 import roofline as RL
    from paper_2104_13542_b200.batched import BatchedController
    from paper_2104_13542_b200.kinematics import load_chain
    from paper_2104_13542_b200.surrogate import load_arm7_surrogate

    goals, th0 = configs.batched_problem(instances)
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    bc = BatchedController(load_chain("arm7.chain"), goals, weights=configs.make_weights(2),
                           self_collision=load_arm7_surrogate(), precision=args.precision, device=local, **kw)
    bc.plan.profile_stages(2)
    thd = np.zeros_like(th0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    for _ in range(3):
        bc.control_step(th0, thd)
    st = {"sample": [], "rollout": [], "mlp": [], "update": []}
    dev = []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        _, d = bc.control_step(th0, thd)
        dev.append(d.device_ms)
        for k in st:
            st[k].append(d.stage_ms[k])
    sm = {k: float(np.mean(v)) for k, v in st.items()}
    rows = instances * 500 * 30
    mlp_t = sm["mlp"] * 1e-3
    roll_t = sm["rollout"] * 1e-3
    fp32_peak = 2 * 128 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    mlp_ach = RL.MLP_TENSOR_FLOPS_PER_ROW * rows / mlp_t / 1e12
    roll_ach = RL.rollout_flops_per_unit(2) * rows / roll_t / 1e12
    return {
        "workload": f"{instances} controllers x 500 x 30 (config-4 shape), config-2 costs",
        "step_ms": float(np.mean(dev)), "stage_ms": sm,
        "mlp": {"bound": "tensor", "achieved": mlp_ach, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": mlp_ach / peaks["bf16_tflops"], "executed_frac": 3 * mlp_ach / peaks["bf16_tflops"],
                "peak_source": f"bf16_tflops ({peaks_kind}); executed = 3 split products per algorithmic MAC"},
        "rollout": {"bound": "fp32", "achieved": roll_ach, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": roll_ach / fp32_peak,
                    "peak_source": "2 x 128 FMA/clk x 148 SMs x sm_max_mhz"},
    }


def _cpu_baseline(args):
    """cpu_baseline of the config-2 line: the reference at workers = all host
    threads (headline) plus the rest of the §8(d) protocol."""
    prot = cpu_protocol(full=not args.quick_cpu)
    cands = [prot.get(k, {}) for k in ("c2_workers_all", "c2_workers_all_blas1", "c2_workers_1")]
    cands = [c for c in cands if "median_ms" in c]
    head = min(cands, key=lambda c: c["median_ms"]) if cands else {}
    kind = head.get("kind", "port")
    return {"value": head.get("median_ms"), "unit": "ms", "cores": head.get("workers", 1), "kind": kind,
            "sample": f"median of {head.get('steps')} reference control_steps (config 2, 500x30, numba, "
                      f"workers={head.get('workers')}; the fastest thread setup of protocol.c2_*) after 1 warm-up"
                      if kind == "reference" else
                      "oracle-port control steps (config 2, numpy float64; oracle/_ref not installed)",
            "protocol": prot}


def run_dry(args, workload: str) -> int:
    """--dry-run: the launch plumbing without a GPU (gloo ranks, a barrier and
    the max-over-ranks reduction; no device work, no timing claims)."""
    ws, rank, _ = _dist_env()
    dist = None
    if ws > 1:
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo")
        t = torch.tensor([float(rank)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        top = int(t.item())
        dist.barrier()
    else:
        top = 0
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": None, "n_gpus": ws, "dry_run": True,
                          "max_rank_seen": top, "workload": workload,
                          "config": workload_config(workload, args, ws)}))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "c1", "c2", "c3", "c4", "c5"],
                    help="auto: c2 at one GPU, c4 at more")
    ap.add_argument("--instances", type=int, default=4096, help="config 4: total controllers")
    ap.add_argument("--weak", action="store_true", help="config 4: --instances per GPU (weak scaling)")
    ap.add_argument("--particles", type=int, default=500)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick-cpu", action="store_true", help="cpu_baseline: config 2 only")
    ap.add_argument("--no-scale-roofline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launch plumbing only (gloo, no GPU)")
    ap.add_argument("--cpu-probe", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_probe:
        print(json.dumps(_cpu_probe(json.loads(args.cpu_probe))))
        return 0
    env_ws = os.environ.get("WORLD_SIZE")
    if env_ws is None and args.gpus > 1:
        return _spawn(args)
    if env_ws is not None and int(env_ws) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_ws}", file=sys.stderr)
        return 2
    workload = args.workload if args.workload != "auto" else ("c2" if args.gpus == 1 else "c4")
    if workload == "c4" and args.weak:
        args.instances *= args.gpus
    if args.dry_run:
        return run_dry(args, workload)
    if args.impl == "reference":
        return run_reference(args, workload)
    if workload == "c3":
        return run_tracking(args)
    if workload == "c5":
        return run_sweep(args)
    if workload == "c4":
        return run_batched(args)
    args.workload = workload
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
