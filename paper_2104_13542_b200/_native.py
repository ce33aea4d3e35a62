"""ctypes binding of the C ABI in include/mppi_b200.h.

The library is built in-tree (``__graft_entry__.build`` or
``python -m paper_2104_13542_b200.build``) to
``paper_2104_13542_b200/_mppi_b200.so``. There is no CPU fallback: if the
library is missing, or no CUDA device is visible when a compute entry point is
called, this module raises instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import ConfigError, ContractError, DeviceError, PolicyStateError

LIB_PATH = Path(os.environ.get("MPPI_LIB") or Path(__file__).resolve().parent / "_mppi_b200.so")  # MPPI_LIB: A/B builds

# enum mppi_status
OK = 0
E_NONFINITE_CONTROL = 1
E_ALL_QUARANTINED = 2
E_WEIGHT_UNDERFLOW = 3
E_BAD_ARGUMENT = 4
E_CUDA = 5
E_NONPOSITIVE_VARIANCE = 6
E_CONFIG = 7
E_SKIPPED = 8  # the on-device episode aborted before this step
E_EXCHANGE = 9  # particle-sharded exchange aborted / timed out (DeviceError)

GOAL_POSITION_ONLY = 0
GOAL_FULL_POSE = 1
SELFCOLL_NONE, SELFCOLL_ORACLE, SELFCOLL_LEARNED = 0, 1, 2
GEN_HALTON, GEN_PSEUDORANDOM, GEN_EXTERNAL = 0, 1, 2
SMOOTH_BSPLINE, SMOOTH_COMB, SMOOTH_NONE = 0, 1, 2
POLICY_PER_JOINT, POLICY_ISOTROPIC = 0, 1
FP32, FP64 = 0, 1
GOAL_FIXED, GOAL_SCRIPT = 0, 1
INTERP_HOLD, INTERP_LINEAR = 0, 1
FALLBACK_NONE, FALLBACK_REISSUE, FALLBACK_BRAKE = 0, 1, 2

MAX_DOF = 8
MAX_HORIZON = 32
MAX_CAPSULES = 16
MAX_PAIRS = 64

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_int64)


class ChainDesc(C.Structure):
    _fields_ = [
        ("dof", C.c_int32), ("task_dim", C.c_int32), ("n_caps", C.c_int32), ("n_pairs", C.c_int32),
        ("axes", _dp), ("origin_rot", _dp), ("origin_trans", _dp), ("jtype", _lp),
        ("joint_limits", _dp), ("velocity_limits", _dp), ("accel_limits", _dp),
        ("cap_p0", _dp), ("cap_p1", _dp), ("cap_r", _dp), ("cap_link", _lp),
        ("pair_a", _lp), ("pair_b", _lp),
    ]


class CostDesc(C.Structure):
    _fields_ = [
        ("alpha_rot", C.c_double * 3), ("alpha_trans", C.c_double * 3),
        ("alpha_stop", C.c_double), ("alpha_joint", C.c_double), ("alpha_manip", C.c_double),
        ("alpha_coll", C.c_double), ("k_jl", C.c_double), ("k_m", C.c_double),
        ("self_collision", C.c_int32), ("_pad", C.c_int32),
    ]


class PlanDesc(C.Structure):
    _fields_ = [
        ("horizon", C.c_int32), ("particles", C.c_int32), ("null_count", C.c_int32),
        ("instances", C.c_int32), ("iterations", C.c_int32), ("policy_mode", C.c_int32),
        ("precision", C.c_int32), ("generator", C.c_int32), ("smoothing", C.c_int32),
        ("spline_degree", C.c_int32), ("knots", C.c_int32), ("device", C.c_int32),
        ("particle_offset", C.c_int32), ("particles_total", C.c_int32),
        ("dump", C.c_int32), ("_pad0", C.c_int32), ("seed", C.c_uint64), ("comb", C.c_double * 3),
        ("gamma", C.c_double), ("terminal_weight", C.c_double), ("beta", C.c_double),
        ("alpha_mu", C.c_double), ("alpha_sigma", C.c_double), ("sigma0_sq", C.c_double),
        ("sigma_sq_min", C.c_double), ("sigma_sq_max", C.c_double), ("default_tail", C.c_double),
        ("dts", _dp),
    ]


class StepInfo(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("bad_particle", C.c_int32), ("finite_count", C.c_int32),
        ("_pad", C.c_int32), ("best_cost", C.c_double), ("mean_cost", C.c_double),
        ("device_ms", C.c_double), ("sample_ms", C.c_double), ("rollout_ms", C.c_double),
        ("mlp_ms", C.c_double), ("update_ms", C.c_double),
    ]


class EvalOut(C.Structure):
    _fields_ = [
        ("positions", _dp), ("velocities", _dp), ("accelerations", _dp), ("step_costs", _dp),
        ("terms", _dp), ("totals", _dp), ("bad_particle", C.c_int32), ("quarantined", C.c_int32),
    ]


_ip = C.POINTER(C.c_int32)


class EpisodeDesc(C.Structure):
    _fields_ = [
        ("steps", C.c_int32), ("goal_source", C.c_int32), ("interpolation", C.c_int32),
        ("script_mode", C.c_int32), ("waypoints", C.c_int32), ("_pad", C.c_int32),
        ("dt", C.c_double), ("filter_lambda", C.c_double),
        ("times", _dp), ("positions", _dp), ("noise", _dp),
    ]


class EpisodeLogC(C.Structure):
    _fields_ = [(n, _dp) for n in ("t", "theta", "theta_dot", "command", "goal", "goal_rot", "ee",
                                   "ee_rot", "cost_total", "cost_terms")] + \
               [(n, _ip) for n in ("collision", "fallback", "status")]


class EpisodeState(C.Structure):
    _fields_ = [
        ("last_estimate", C.c_double * (2 * MAX_DOF)), ("last_command", C.c_double * MAX_DOF),
        ("prev_command", C.c_double * MAX_DOF), ("plant", C.c_double * (2 * MAX_DOF)),
        ("fallback_armed", C.c_int32), ("aborted", C.c_int32),
    ]


class TrainDesc(C.Structure):
    _fields_ = [
        ("in_dim", C.c_int32), ("n_train", C.c_int32), ("n_hold", C.c_int32), ("epochs", C.c_int32),
        ("batch_size", C.c_int32), ("_pad", C.c_int32),
        ("x_train", _dp), ("y_train", _dp), ("x_hold", _dp), ("y_hold", _dp),
        ("order", C.POINTER(C.c_int64)), ("lr", _dp), ("bias_corr1", _dp), ("bias_corr2", _dp),
    ]


class TrainResult(C.Structure):
    _fields_ = [
        ("steps", C.c_int64), ("diverged_epoch", C.c_int32), ("_pad", C.c_int32),
        ("last_finite_loss", C.c_double), ("holdout_mae", C.c_double), ("sign_agreement", C.c_double),
        ("device_ms", C.c_double), ("losses", _dp),
    ]


# name -> (restype, argtypes); every function returns int status unless noted
_vp = C.c_void_p
_SIGS = {
    "mppi_abi_version": (C.c_int32, []),
    "mppi_last_error": (C.c_char_p, []),
    "mppi_build_info": (C.c_char_p, []),
    "mppi_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "mppi_plan_create": (C.c_int, [C.POINTER(ChainDesc), C.POINTER(CostDesc), C.POINTER(PlanDesc),
                                   C.POINTER(_vp)]),
    "mppi_plan_destroy": (C.c_int, [_vp]),
    "mppi_init_noise": (C.c_int, [_vp, _dp]),
    "mppi_set_noise": (C.c_int, [_vp, _dp]),
    "mppi_get_noise": (C.c_int, [_vp, _dp]),
    "mppi_set_goal": (C.c_int, [_vp, C.c_int32, _dp, _dp, C.c_int32]),
    "mppi_set_goals": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp, _dp, C.POINTER(C.c_int32)]),
    "mppi_set_world": (C.c_int, [_vp, _dp, C.c_int32, _dp, C.c_int32]),
    "mppi_set_voxel_world": (C.c_int, [_vp, C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int32,
                                       _dp, C.c_double, _dp, C.c_int32]),
    "mppi_set_mlp": (C.c_int, [_vp, C.c_int32] + [_dp] * 8),
    "mppi_set_policy": (C.c_int, [_vp, C.c_int32, _dp, _dp]),
    "mppi_get_policy": (C.c_int, [_vp, C.c_int32, _dp, _dp]),
    "mppi_step": (C.c_int, [_vp, _dp, _dp, _dp, C.POINTER(StepInfo)]),
    "mppi_evaluate": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, _dp, C.c_double, C.c_double,
                                _dp, _dp, _dp, _dp, C.POINTER(EvalOut)]),
    "mppi_get_bundle": (C.c_int, [_vp, C.POINTER(EvalOut), _dp]),
    "mppi_get_step_inputs": (C.c_int, [_vp, C.c_int32, _dp, _dp, _dp, _dp]),
    "mppi_replay_bundle": (C.c_int, [_vp, C.POINTER(EvalOut), _dp]),
    "mppi_episode": (C.c_int, [_vp, C.POINTER(EpisodeDesc), _dp, _dp, C.POINTER(EpisodeState),
                               C.POINTER(EpisodeLogC), _ip, _dp]),
    "mppi_top_rollouts": (C.c_int, [_vp, C.c_int32, _ip, _dp, _dp]),
    "mppi_train_mlp": (C.c_int, [C.POINTER(TrainDesc), C.POINTER(_dp), C.POINTER(_dp), C.POINTER(TrainResult)]),
    "mppi_time_stage": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp]),
    "mppi_profile_stages": (C.c_int, [_vp, C.c_int32]),
    "mppi_stats_record_len":(C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "mppi_stats_dev": (C.c_int, [_vp, _dp, _dp, _vp, _vp]),
    "mppi_finalize_dev": (C.c_int, [_vp, _vp, C.c_int32, _dp, C.POINTER(StepInfo), _vp]),
    "mppi_peer_buffers": (C.c_int, [_vp, C.c_int32, C.POINTER(_vp), C.POINTER(_vp)]),
    "mppi_set_peers": (C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(_vp), C.POINTER(_vp)]),
    "mppi_step_exchange": (C.c_int, [_vp, _dp, _dp, _dp, C.POINTER(StepInfo)]),
    "mppi_set_exchange_timeout": (C.c_int, [_vp, C.c_double]),
    "mppi_exchange_abort": (C.c_int, [_vp]),
    "mppi_ipc_get_handle": (C.c_int, [_vp, C.c_char_p]),
    "mppi_ipc_open_handle": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "mppi_ipc_close": (C.c_int, [_vp]),
    "mppi_halton_points": (C.c_int, [C.c_int64, C.c_int32, _dp]),
    "mppi_gaussianize": (C.c_int, [_dp, C.c_int64, _dp]),
    "mppi_bspline_basis": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _dp]),
    "mppi_smooth_sequences": (C.c_int, [_dp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _dp, _dp,
                                        C.c_int32, _dp]),
    "mppi_build_controls": (C.c_int, [_dp, _dp, _dp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _dp]),
    "mppi_particle_weights": (C.c_int, [_dp, C.c_int64, C.c_double, _dp]),
    "mppi_update_policy": (C.c_int, [_dp, _dp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                     C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int32, _dp,
                                     _dp]),
    "mppi_mlp_forward": (C.c_int, [_vp, _dp, C.c_int64, _dp]),
    "mppi_fk_batch": (C.c_int, [_dp, C.c_int64, C.c_int32, _dp, _dp, _dp, _lp, _dp, _dp]),
    "mppi_jacobian_batch": (C.c_int, [_dp, C.c_int64, C.c_int32, _dp, _dp, _dp, _lp, _dp]),
    "mppi_manip_batch": (C.c_int, [_dp, C.c_int64, C.c_int32, C.c_int32, _dp]),
    "mppi_self_collision_batch": (C.c_int, [_dp, _dp, C.c_int64, C.c_int32, _dp, _dp, _dp, _lp,
                                            C.c_int32, _lp, _lp, C.c_int32, _dp]),
    "mppi_env_collision_batch": (C.c_int, [_dp, _dp, C.c_int64, C.c_int32, _dp, _dp, _dp, _lp,
                                           C.c_int32, _dp, C.c_int32, _dp, C.c_int32, _lp]),
    "mppi_integrate_batch": (C.c_int, [_dp, C.c_int64, C.c_int32, C.c_int32, _dp, _dp, _dp, _dp,
                                       _dp]),
    "mppi_pose_cost": (C.c_int, [_dp, _dp, C.c_int64, _dp, _dp, C.c_int32, _dp, _dp, _dp]),
    "mppi_stop_cost": (C.c_int, [_dp, C.c_int64, C.c_int32, C.c_int32, _dp, _dp]),
    "mppi_joint_limit_cost": (C.c_int, [_dp, C.c_int64, C.c_int32, _dp, _dp, _dp]),
    "mppi_manipulability_cost": (C.c_int, [_dp, C.c_int64, C.c_double, _dp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load (once) and type the native library. Raises DeviceError when absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise DeviceError(
            f"native library {p} is missing; build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (there is no CPU fallback)"
        )
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.mppi_abi_version() != 2:
        raise DeviceError("native library ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


_fast = False


def fast_module():
    """The CPython entry of the latency path (csrc/mppi_fast.c, built beside
    the library), or None when it is not built or MPPI_NO_FAST is set (A/B):
    callers then take the ctypes path to the same mppi_step."""
    global _fast
    if _fast is False:
        _fast = None
        if not os.environ.get("MPPI_NO_FAST"):
            try:
                from . import _mppi_fast as m  # noqa: PLC0415

                _fast = m
            except ImportError:
                _fast = None
    return _fast


def last_error() -> str:
    return load_library().mppi_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map an mppi_status to the reference exception classes (errors.py)."""
    if rc == OK:
        return
    msg = last_error() or what
    if rc in (E_NONFINITE_CONTROL, E_BAD_ARGUMENT):
        raise ContractError(msg)
    if rc in (E_ALL_QUARANTINED, E_WEIGHT_UNDERFLOW, E_NONPOSITIVE_VARIANCE):
        raise PolicyStateError(msg)
    if rc == E_CONFIG:
        raise ConfigError(msg)
    raise DeviceError(msg or f"mppi status {rc}")


def status_exception(code: int, bad_particle: int = -1) -> Exception:
    """Exception for a per-instance device status word (mppi_step_info.status)."""
    if code == E_NONFINITE_CONTROL:
        return ContractError("control batch contains non-finite entries"
                             + (f" (particle {bad_particle})" if bad_particle >= 0 else ""))
    if code == E_NONPOSITIVE_VARIANCE:
        return PolicyStateError("covariance entries must be positive")
    if code == E_ALL_QUARANTINED:
        return PolicyStateError("all particles quarantined; no finite costs")
    if code == E_WEIGHT_UNDERFLOW:
        return PolicyStateError("all particle weights underflowed to zero; increase beta")
    if code == E_EXCHANGE:
        return DeviceError("particle-sharded exchange aborted or timed out (policy kept shifted)")
    return DeviceError(f"device status {code}")


def device_count() -> int:
    n = C.c_int32(0)
    rc = load_library().mppi_device_count(C.byref(n))
    if rc != OK:
        return 0
    return int(n.value)


def require_device() -> None:
    if device_count() < 1:
        raise DeviceError("no CUDA device visible: the B200 path has no CPU fallback")


def f64(a, shape=None) -> np.ndarray:
    """C-contiguous float64 copy/view."""
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        out = out.reshape(shape)
    return out


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def lptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_lp)
