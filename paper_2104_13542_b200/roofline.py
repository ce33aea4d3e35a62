"""Algorithmic work per particle-step and the roofline of each step kernel.

Counts follow SURVEY.md §8(d) for a generic 7-DOF revolute chain (FMA = 2
flops, no exploitation of arm7's zero entries — the kernels are generic over
chain data):

  sample affine 14 | integrate 28 | FK 7 x 178 = 1246 | pose (full) 120 |
  joint 49 | stop 28 | Jacobian 192 | manipulability 145 |
  capsule self-collision ~650 | total + discount 14 | update statistics 42
  learned MLP: 2*(14*256 + 256*128 + 128*64 + 64*1) = 89,216 tensor flops/row

Algorithmic bytes per particle-step of the fused step: eps read as float64
(H*d*8 / H = 56 B) by the rollout and again by the update, a 4 B step cost
write+read, the MLP's 64 B input row + 4 B output.
"""

from __future__ import annotations

FLOPS = {
    "sample": 14, "integrate": 28, "fk": 1246, "pose_full": 120, "pose_pos": 30, "joint": 49,
    "stop": 28, "jacobian": 192, "manip": 145, "selfcoll_oracle": 650, "total": 14, "update": 42,
}
MLP_TENSOR_FLOPS_PER_ROW = 2 * (14 * 256 + 256 * 128 + 128 * 64 + 64 * 1)  # 89,216


def rollout_flops_per_unit(config: int) -> int:
    f = FLOPS["sample"] + FLOPS["integrate"] + FLOPS["fk"] + FLOPS["pose_full"] + FLOPS["joint"] + FLOPS["total"]
    if config == 2:
        f += FLOPS["stop"] + FLOPS["jacobian"] + FLOPS["manip"]
    return f


def rollout_bytes_per_unit(dof: int = 7) -> int:
    return dof * 8 + 4 + 16 * 4  # eps row, step-cost write, posenc row (learned path)


def update_bytes_per_unit(dof: int = 7) -> int:
    return dof * 8 + 4 + 4  # eps row re-read, step cost + learned distance read


# kernel-name fragments of each stage in an ncu summary (scripts/ncu_summary.py)
NCU_KERNEL = {"rollout": "rollout_", "mlp": "mlp_tcgen05", "update": "stats_"}


def ncu_traffic(summary: list | None, stage: str):
    """DRAM bytes (read + write) per launch of the stage's kernel in a committed
    ``ncu --set full`` summary (one step's capture), or None."""
    for k in summary or []:
        if NCU_KERNEL[stage] in k.get("kernel", "") and k.get("dram_read_B") is not None:
            return float(k["dram_read_B"]) + float(k.get("dram_write_B") or 0.0)
    return None


def launch_shares(profiles_dir, tag: str):
    """Per-stage median device time (ns) of the step's kernels in the newest
    committed ncu launch list profiles/r*_<tag>.csv (`ncu --metrics
    gpu__time_duration.sum --clock-control none --csv`), or (None, None)."""
    import csv
    from pathlib import Path

    files = sorted(Path(profiles_dir).glob(f"r*_{tag}.csv"))
    if not files:
        return None, None
    # per stage, the most frequently launched kernel instantiation: the timed
    # loop's (the same command also launches the FP64 and bundle-dumping
    # variants a few times)
    times = {k: {} for k in NCU_KERNEL}
    try:
        with open(files[-1]) as fh:
            for r in csv.DictReader(ln for ln in fh if ln.startswith('"')):
                if r.get("Metric Name") != "gpu__time_duration.sum":
                    continue
                name = r.get("Kernel Name", "")
                for stage, frag in NCU_KERNEL.items():
                    if frag in name:
                        times[stage].setdefault(name, []).append(float(r["Metric Value"].replace(",", "")))
    except (OSError, ValueError, KeyError):
        return None, None
    med = {}
    for stage, by_name in times.items():
        if by_name:
            v = sorted(max(by_name.values(), key=len))
            med[stage] = v[len(v) // 2]
    return (med or None), f"profiles/{files[-1].name}"


def all_rooflines(stage_ms: dict, rows: int, dof: int, config: int, peaks: dict, peaks_kind: str,
                  ncu_summary: list | None = None, ncu_source: str | None = None) -> dict:
    """The roofline entry of every kernel of the step (not only the dominant one)."""
    out = {}
    for stage in ("rollout", "mlp", "update"):
        if stage == "mlp" and config != 2:
            continue
        e = _stage_roofline(stage, stage_ms, rows, dof, config, peaks, peaks_kind)
        tr = ncu_traffic(ncu_summary, stage)
        if tr is not None and e.get("kernel"):
            e["traffic"] = tr
            e["traffic_source"] = ncu_source
        e["stage_ms"] = stage_ms.get(stage)
        out[stage] = e
    return out


def step_roofline(stage_ms: dict, rows: int, particles: int, horizon: int, dof: int, config: int,
                  peaks: dict, peaks_kind: str, ncu_summary: list | None = None,
                  ncu_source: str | None = None, ncu_rows: int | None = None, ncu_share: dict | None = None,
                  ncu_share_source: str | None = None) -> dict:
    """Roofline entry for the dominant kernel of the step (stage_ms from the
    event-record nodes of the timed graph replays); `traffic` from the
    committed ncu summary of the same kernel when one is given. `ncu_rows`:
    the rows of the captured launch when it was a smaller batch than this
    step's — its bytes per row are then scaled to this launch and labelled so.
    The dominant kernel is the largest in the committed ncu launch list of the
    same command (`ncu_share`, per-stage ns) when given: the event times of
    adjacent stages can tie within their resolution."""
    stages = ("rollout", "mlp", "update") if config == 2 else ("rollout", "update")
    if ncu_share:
        stage = max(stages, key=lambda k: ncu_share.get(k, 0.0))
    else:
        stage = max(stages, key=lambda k: stage_ms.get(k, 0.0))
    out = _stage_roofline(stage, stage_ms, rows, dof, config, peaks, peaks_kind)
    if ncu_share:
        tot = sum(ncu_share.get(k, 0.0) for k in stages)
        out["dominant_by"] = f"{ncu_share_source}: median gpu__time_duration per launch"
        out["ncu_share"] = {k: ncu_share.get(k, 0.0) / tot for k in stages if tot > 0}
    else:
        out["dominant_by"] = "CUDA-event stage times of the instrumented graph"
    tr = ncu_traffic(ncu_summary, stage)
    if tr is not None and out.get("kernel"):
        src = f"{ncu_source}: dram__bytes_read.sum + dram__bytes_write.sum (ncu replay, cold L2)"
        if ncu_rows and ncu_rows != rows:
            src += f"; captured at {ncu_rows} rows ({tr / ncu_rows:.1f} B/row), scaled to this launch's {rows}"
            tr = tr / ncu_rows * rows
        out["traffic"] = tr
        out["traffic_source"] = src
    return out


def _stage_roofline(stage: str, stage_ms: dict, rows: int, dof: int, config: int, peaks: dict,
                    peaks_kind: str) -> dict:
    t = stage_ms[stage] * 1e-3
    if not t > 0.0:  # stage events disabled (MPPI_STAGE_EVENTS=0): no per-kernel time
        return {"kernel": None, "bound": None, "achieved": None, "peak": None, "unit": None, "frac": None,
                "traffic": None, "note": "stage events disabled"}
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    if stage == "mlp":
        achieved = MLP_TENSOR_FLOPS_PER_ROW * rows / t / 1e12
        peak = peaks["bf16_tflops"]
        return {"kernel": "mlp (learned self-collision, tcgen05)", "bound": "tensor", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                "peak_source": f"bf16_tflops ({peaks_kind})",
                "algorithmic": f"{MLP_TENSOR_FLOPS_PER_ROW} flop/row x {rows} rows"}
    if stage == "rollout":
        fl = rollout_flops_per_unit(config)
        achieved = fl * rows / t / 1e12
        peak = 2 * 128 * 148 * sm_mhz * 1e6 / 1e12  # FP32 FMA pipe at the measured max SM clock
        return {"kernel": "rollout (fused integrate+FK+costs)", "bound": "fp32", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                "peak_source": f"2 x 128 FMA/clk x 148 SMs x sm_max_mhz ({peaks_kind} clock)",
                "algorithmic": f"{fl} flop/particle-step x {rows}"}
    by = update_bytes_per_unit(dof) * rows
    achieved = by / t / 1e9
    peak = peaks["hbm_gbs"]
    return {"kernel": "stats/update (weights + mean/cov + shift)", "bound": "hbm", "achieved": achieved,
            "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
            "peak_source": f"hbm_gbs ({peaks_kind})",
            "algorithmic": f"{update_bytes_per_unit(dof)} B/particle-step x {rows}",
            "note": "operand bytes per particle-step, eps row counted per instance: a batch shares one eps "
                    "block served from L2, so DRAM carries ~8 B/particle-step and the batched kernel is "
                    "instruction-bound (profiles/r2c_full_c4_stats_multi_metrics.json: 75 % issue, 10.7 % DRAM)"}
