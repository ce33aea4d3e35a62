"""The reference's operator seam, executed on the B200.

jointmpc/kernels/__init__.py:50-66 exposes a six-function table
(fk_batch, jacobian_batch, manip_batch, self_collision_batch,
env_collision_batch, integrate_batch) plus BACKEND_NAME. This module has the
same names, signatures, dtypes (float64 in/out, int64 indices) and ownership
(fresh caller-owned outputs), backed by the float64 seam kernels of the
native library (csrc/mppi_aux_kernels.cuh). Because the signatures match, the
table can be installed into an unmodified reference process.

The fused hot path does NOT go through this seam: control_step and
evaluate_rollouts run the fused rollout kernel (the numpy seam
would materialise every link pose of every configuration).
"""

from __future__ import annotations

from contextlib import contextmanager

import numpy as np

from . import _native as N

BACKEND_NAME = "cuda-sm100a"


def _lib():
    return N.load_library()


def fk_batch(q, axes, origin_rot, origin_trans, jtype):
    """(M,d) -> rot (M,d,3,3), trans (M,d,3) (jit.py:89-111)."""
    q = N.f64(q)
    M, d = q.shape
    rot = np.empty((M, d, 3, 3))
    trans = np.empty((M, d, 3))
    N.check(_lib().mppi_fk_batch(N.dptr(q), M, d, N.dptr(N.f64(axes)), N.dptr(N.f64(origin_rot)),
                                 N.dptr(N.f64(origin_trans)), N.lptr(N.i64(jtype)), N.dptr(rot),
                                 N.dptr(trans)))
    return rot, trans


def jacobian_batch(q, rot, trans, axes, jtype):
    """Geometric Jacobian (M,6,d), linear rows first (jit.py:114-148)."""
    q = N.f64(q)
    M, d = q.shape
    J = np.empty((M, 6, d))
    N.check(_lib().mppi_jacobian_batch(N.dptr(q), M, d, N.dptr(N.f64(rot)), N.dptr(N.f64(trans)),
                                       N.dptr(N.f64(axes)), N.lptr(N.i64(jtype)), N.dptr(J)))
    return J


def manip_batch(J, task_dim):
    """sqrt(max(det(Jp Jp^T), 0)) or |det Jp| when square (jit.py:151-185)."""
    J = N.f64(J)
    M, _, d = J.shape
    out = np.empty(M)
    N.check(_lib().mppi_manip_batch(N.dptr(J), M, d, int(task_dim), N.dptr(out)))
    return out


def self_collision_batch(rot, trans, cap_p0, cap_p1, cap_r, cap_link, pair_a, pair_b):
    """max over pairs of r_i + r_j - segdist; NO_CONTACT without pairs (jit.py:241-260)."""
    rot = N.f64(rot)
    M, d = rot.shape[0], rot.shape[1]
    out = np.empty(M)
    cap_r = N.f64(cap_r)
    pa = N.i64(pair_a)
    N.check(_lib().mppi_self_collision_batch(
        N.dptr(rot), N.dptr(N.f64(trans)), M, d, N.dptr(N.f64(cap_p0).reshape(-1)),
        N.dptr(N.f64(cap_p1).reshape(-1)), N.dptr(cap_r), N.lptr(N.i64(cap_link)), cap_r.shape[0],
        N.lptr(pa), N.lptr(N.i64(pair_b)), pa.shape[0], N.dptr(out)))
    return out


def env_collision_batch(rot, trans, cap_p0, cap_p1, cap_r, cap_link, spheres, boxes):
    """First colliding obstacle index (spheres first), -1 when clear (jit.py:289-332)."""
    rot = N.f64(rot)
    M, d = rot.shape[0], rot.shape[1]
    hit = np.empty(M, dtype=np.int64)
    cap_r = N.f64(cap_r)
    sp = N.f64(spheres).reshape(-1, 4)
    bx = N.f64(boxes).reshape(-1, 6)
    N.check(_lib().mppi_env_collision_batch(
        N.dptr(rot), N.dptr(N.f64(trans)), M, d, N.dptr(N.f64(cap_p0).reshape(-1)),
        N.dptr(N.f64(cap_p1).reshape(-1)), N.dptr(cap_r), N.lptr(N.i64(cap_link)), cap_r.shape[0],
        N.dptr(sp), sp.shape[0], N.dptr(bx), bx.shape[0], N.lptr(hit)))
    return hit


def integrate_batch(u, dts, th0, thd0):
    """Semi-implicit Euler, sequential per (n, joint) (jit.py:335-349)."""
    u = N.f64(u)
    n, h, d = u.shape
    pos = np.empty_like(u)
    vel = np.empty_like(u)
    N.check(_lib().mppi_integrate_batch(N.dptr(u), n, h, d, N.dptr(N.f64(dts)), N.dptr(N.f64(th0)),
                                        N.dptr(N.f64(thd0)), N.dptr(pos), N.dptr(vel)))
    return pos, vel


_EXPORTED = ("fk_batch", "jacobian_batch", "manip_batch", "self_collision_batch",
             "env_collision_batch", "integrate_batch")


_BACKEND_NAMES = ("cuda", BACKEND_NAME)


def get_backend(name: str = "cuda"):
    """The kernel module for `name` (kernels/__init__.py:25-33). This build has
    exactly one backend, the sm_100a seam; the reference's "numpy"/"numba"
    names raise ValueError, as the reference does for unknown names — there is
    no CPU fallback to select."""
    import sys

    if name not in _BACKEND_NAMES:
        raise ValueError(f"unknown kernel backend {name!r} (this build has only {BACKEND_NAME!r})")
    return sys.modules[__name__]


def active_backend():
    """The kernel module in effect (kernels/__init__.py:44-46)."""
    import sys

    return sys.modules[__name__]


@contextmanager
def use_backend(name: str):
    """Temporarily rebind the six exported functions to the named backend
    (kernels/__init__.py:69-83). Consumers resolve ``kernels.fk_batch`` at call
    time, so rebinding the module attributes redirects them all. Not thread
    safe (the reference's contract): for tests and benchmarks, not the loop."""
    module = get_backend(name)
    g = globals()
    saved = {fn: g[fn] for fn in _EXPORTED}
    g.update({fn: getattr(module, fn) for fn in _EXPORTED})
    try:
        yield module
    finally:
        g.update(saved)


def install_into(module) -> dict:
    """Rebind a reference-style kernel table (e.g. ``jointmpc.kernels``) to this
    backend; returns the previous bindings so the caller can restore them."""
    saved = {fn: getattr(module, fn) for fn in _EXPORTED}
    for fn in _EXPORTED:
        setattr(module, fn, globals()[fn])
    return saved
