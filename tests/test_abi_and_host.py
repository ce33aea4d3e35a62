"""CPU-only checks: the C-ABI library loads and exports every symbol the header
declares; host-side validation mirrors the reference's exceptions; loaders read
the reference's file formats; compute entry points fail loudly without a GPU."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _header_functions():
    text = (ROOT / "include" / "mppi_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mppi_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2104_13542_b200 import _native as N

    lib = N.load_library()
    declared = _header_functions()
    assert len(declared) >= 30
    missing = [f for f in declared if not hasattr(lib, f)]
    assert not missing, missing
    # and the Python binding types every one of them
    assert set(declared) <= set(N.EXPORTED), sorted(set(declared) - set(N.EXPORTED))


def test_library_is_sm100a_build():
    from paper_2104_13542_b200 import _native as N

    info = N.load_library().mppi_build_info().decode()
    assert "sm_100a" in info


def test_no_gpu_means_loud_failure(monkeypatch):
    from paper_2104_13542_b200 import _native as N
    from paper_2104_13542_b200.errors import DeviceError

    if N.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(DeviceError):
        N.require_device()
    from paper_2104_13542_b200 import configs

    with pytest.raises(DeviceError):
        configs.make_controller(1, particles=16)


def test_missing_library_raises(tmp_path):
    from paper_2104_13542_b200 import _native as N
    from paper_2104_13542_b200.errors import DeviceError

    with pytest.raises(DeviceError):
        N.load_library(tmp_path / "nope.so")


def test_chain_loading_and_validation():
    import json

    from paper_2104_13542_b200.errors import ChainError
    from paper_2104_13542_b200.kinematics import FIXTURES, chain_from_dict, load_chain

    for f in FIXTURES.glob("*.chain"):
        assert load_chain(f).dof >= 1
    arm7 = load_chain("arm7.chain")
    assert arm7.dof == 7 and arm7.cap_r.shape == (5,) and arm7.pair_a.shape == (6,)
    data = json.loads((FIXTURES / "slider1.chain").read_text())
    data["joints"][0]["axis"] = [0.0, 0.0, 2.0]
    with pytest.raises(ChainError):
        chain_from_dict(data)
    data = json.loads((FIXTURES / "planar2.chain").read_text())
    data["self_collision_pairs"] = [[0, 9]]
    with pytest.raises(ChainError):
        chain_from_dict(data)
    with pytest.raises(ChainError):
        load_chain("/nonexistent/x.chain")


def test_fixture_matches_reference_numbers():
    """The re-emitted arm7 fixture carries the reference's exact numbers."""
    from paper_2104_13542_b200.kinematics import load_chain

    c = load_chain("arm7.chain")
    np.testing.assert_array_equal(c.accel_limits, [15.0, 7.5, 10.0, 12.5, 15.0, 20.0, 20.0])
    np.testing.assert_array_equal(c.origin_trans[3], [-0.0825, 0.0, 0.384])


def test_value_type_validation():
    from paper_2104_13542_b200.costs import CostWeights, GoalSpec, goal_at_position
    from paper_2104_13542_b200.errors import ContractError, PolicyStateError
    from paper_2104_13542_b200.kinematics import Pose
    from paper_2104_13542_b200.policy import PolicyParams, UpdateConfig, make_policy, shift
    from paper_2104_13542_b200.rollout import DtSchedule, JointState, make_dt_schedule
    from paper_2104_13542_b200.sampling import SmoothingSpec, default_knot_count

    with pytest.raises(ContractError):
        CostWeights(alpha_stop=-1.0)
    with pytest.raises(ContractError):
        CostWeights(k_jl=0.5)
    with pytest.raises(ContractError):
        GoalSpec(target_pose=Pose(rotation=2 * np.eye(3), translation=np.zeros(3)))
    with pytest.raises(ContractError):
        goal_at_position([0, 0, 0], mode="sideways")
    with pytest.raises(ContractError):
        UpdateConfig(beta=0.0)
    with pytest.raises(ContractError):
        UpdateConfig(sigma_sq_min=2.0, sigma_sq_max=1.0)
    with pytest.raises(PolicyStateError):
        PolicyParams(means=np.zeros((2, 1)), variances=np.zeros((2, 1)), mode="per_joint_diagonal",
                     tail_variance=1.0)
    with pytest.raises(ContractError):
        JointState(theta=[np.nan], theta_dot=[0.0], theta_ddot=[0.0])
    with pytest.raises(ContractError):
        DtSchedule(dts=np.array([0.1, 0.05]))
    with pytest.raises(ContractError):
        make_dt_schedule(10, 0.05, "geometric")
    s = make_dt_schedule(30, 0.05, "two_phase")
    assert s.dts[0] == 0.05 and s.dts[-1] == 0.1 and (s.dts == 0.05).sum() == 15
    assert default_knot_count(30) == 5 and default_knot_count(8) == 4
    assert SmoothingSpec().knot_count(30) == 5
    pol = make_policy(5, 2, 7.5)
    pol.means[:] = np.arange(10.0).reshape(5, 2)
    out = shift(pol, 0.25)
    np.testing.assert_array_equal(out.means[:-1], pol.means[1:])
    np.testing.assert_array_equal(out.means[-1], [0.25, 0.25])
    np.testing.assert_array_equal(out.variances[-1], [7.5, 7.5])


def test_voxel_box_decomposition_is_exact():
    from paper_2104_13542_b200.simworld import VoxelGrid

    rng = np.random.default_rng(0)
    occ = (rng.random((12, 10, 9)) < 0.3).astype(np.uint8)
    grid = VoxelGrid(occupancy=occ, origin=np.array([-1.0, -0.5, 0.0]), voxel=0.1)
    boxes = grid.boxes()
    rebuilt = np.zeros_like(occ)
    for b in boxes:
        lo = np.round((b[:3] - grid.origin) / grid.voxel).astype(int)
        hi = np.round((b[3:] - grid.origin) / grid.voxel).astype(int)
        assert (rebuilt[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] == 0).all()  # disjoint
        rebuilt[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = 1
    np.testing.assert_array_equal(rebuilt, occ)


def test_surrogate_weights_layout():
    from paper_2104_13542_b200.surrogate import load_arm7_surrogate

    s = load_arm7_surrogate()
    assert s.dof == 7 and s.kind == "learned"
    assert [w.shape for w in s.net.weights] == [(14, 256), (256, 128), (128, 64), (64, 1)]
    assert s.sign_agreement > 0.95 and s.holdout_mae < 0.02  # test_acceptance.py:267-279 thresholds


def test_roofline_counts():
    from paper_2104_13542_b200 import roofline as RL

    assert RL.MLP_TENSOR_FLOPS_PER_ROW == 89216
    assert 1400 < RL.rollout_flops_per_unit(1) < 1600
    assert 1700 < RL.rollout_flops_per_unit(2) < 2000


def test_reference_arm_bench_line():
    """`bench.py --impl reference` (the reference's own CPU control_step from
    oracle/_ref on the host cores) prints one JSON line with the contract's
    keys and the reference arm's e2e / cpu_baseline blocks."""
    import json
    import subprocess
    import sys

    root = Path(__file__).resolve().parents[1]
    if not (root / "oracle" / "_ref" / "jointmpc").exists():
        pytest.skip("reference not installed (oracle/build_ref.py)")
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"):
        assert k in line, k
    assert line["impl"] == "reference" and line["unit"] == "ms" and line["higher_is_better"] is False
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["value"] > 0.0


def test_roofline_dominant_kernel_from_launch_list(tmp_path):
    """bench.py's roofline picks the dominant kernel from the committed ncu
    launch list (the timed instantiation of each stage), not from the event
    times, which tie between adjacent stages."""
    from paper_2104_13542_b200 import roofline as RL

    rows = ['"ID","Kernel Name","Metric Name","Metric Unit","Metric Value"']
    times = [("void mppi::rollout_kernel<float, 7, 1, 1>(x)", [7600, 7700, 7500]),
             ("void mppi::rollout_kernel<double, 7, 1, 0>(x)", [10500]),  # the FP64 plan's, launched once
             ("void mppi::mlp_tcgen05_kernel<1>(x)", [8900, 8800, 9000]),
             ("void mppi::stats_cluster_kernel<float, 7, 1>(x)", [10000, 10100, 9900])]
    i = 0
    for name, ts in times:
        for t in ts:
            rows.append(f'"{i}","{name}","gpu__time_duration.sum","ns","{t}"')
            i += 1
    (tmp_path / "r9_bench_launches.csv").write_text("\n".join(rows) + "\n")
    share, src = RL.launch_shares(tmp_path, "bench_launches")
    assert src.endswith("r9_bench_launches.csv")
    assert share == {"rollout": 7600.0, "mlp": 8900.0, "update": 10000.0}
    peaks = {"hbm_gbs": 6000.0, "bf16_tflops": 1600.0, "sm_max_mhz": 1965.0}
    stage_ms = {"rollout": 0.0120, "mlp": 0.0123, "update": 0.0122}  # events: the MLP looks longest
    roof = RL.step_roofline(stage_ms, rows=15000, particles=500, horizon=30, dof=7, config=2, peaks=peaks,
                            peaks_kind="measured", ncu_share=share, ncu_share_source=src)
    assert roof["kernel"].startswith("stats") and roof["bound"] == "hbm"
    kern = RL.all_rooflines(stage_ms, rows=15000, dof=7, config=2, peaks=peaks, peaks_kind="measured")
    assert set(kern) == {"rollout", "mlp", "update"}


def test_fast_entry_declines_what_needs_a_conversion():
    """The CPython latency entry (csrc/mppi_fast.c) takes only C-contiguous
    float64 vectors of length d; anything else returns NotImplemented so the
    caller converts on the ctypes path. No device call is made here."""
    import numpy as np

    from paper_2104_13542_b200 import _native as N

    m = N.fast_module()
    if m is None:
        pytest.skip("fast entry not built")
    ok = np.zeros(7)
    assert m.step(1, 1, ok.astype(np.float32), ok, 0, 0, 7) is NotImplemented
    assert m.step(1, 1, ok, np.zeros(6), 0, 0, 7) is NotImplemented
    assert m.step(1, 1, np.zeros(14)[::2], ok, 0, 0, 7) is NotImplemented
    assert m.step(1, 1, [0.0] * 7, ok, 0, 0, 7) is NotImplemented
    with pytest.raises(ValueError):
        m.step(0, 1, ok, ok, 0, 0, 7)
