"""CPU ORACLE — test infrastructure only. NOT part of the product.

A float64 numpy restatement of the reference's per-step MPPI algorithm
(jointmpc, /root/reference/pkg/src/jointmpc/, cited below as <module>:<line>).
Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` leg may
import this module, and only as the checker / CPU timing arm — never as a
code path of the package. The package has no CPU fallback.

Parity status: PINNED. tests/test_oracle_golden.py checks every function here
against golden vectors produced by running the reference itself
(tests/golden/make_golden.py, committed with its output), including full
control steps at the BASELINE configs.

Chains, weights and goals are duck-typed: any object with the reference's
attribute names (KinematicChain, CostWeights, GoalSpec) works.
"""

from __future__ import annotations

import math

import numpy as np

# kernels/shared.py:8-21
REORTHO_EVERY = 8
POLAR_ITERS = 2
TERNARY_ITERS = 60
SEG_EPS = 1e-12
NO_CONTACT = -1.0e30

FIRST_PRIMES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71,
                73, 79, 83, 89, 97, 101, 103, 107, 109, 113, 127, 131, 137, 139, 149, 151, 157, 163,
                167, 173)  # sampling.py:28-36

# ============================================================== sampling
def van_der_corput(i: int, base: int) -> float:
    """Radical inverse with integer digit reversal, one rounded divide (sampling.py:89-97)."""
    digits_rev, scale = 0, 1
    while i:
        i, digit = divmod(i, base)
        digits_rev = digits_rev * base + digit
        scale *= base
    return digits_rev / scale


def halton(count: int, dims: int) -> np.ndarray:
    """(count, dims), row i column j = phi_{p_j}(i+1) (sampling.py:100-115)."""
    return np.array([[van_der_corput(i + 1, FIRST_PRIMES[j]) for j in range(dims)]
                     for i in range(count)], dtype=np.float64).reshape(count, dims)


_A = (-3.969683028665376e01, 2.209460984245205e02, -2.759285104469687e02, 1.383577518672690e02,
      -3.066479806614716e01, 2.506628277459239e00)
_B = (-5.447609879822406e01, 1.615858368580409e02, -1.556989798598866e02, 6.680131188771972e01,
      -1.328068155288572e01)
_C = (-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e00, -2.549732539343734e00,
      4.374664141464968e00, 2.938163982698783e00)
_D = (7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e00, 3.754408661907416e00)
_PLOW = 0.02425


def _horner(coeffs, x):
    acc = np.zeros_like(x) + coeffs[0]
    for c in coeffs[1:]:
        acc = acc * x + c
    return acc


def acklam(p) -> np.ndarray:
    """Acklam rational inverse normal CDF with its three branches (sampling.py:146-202)."""
    p = np.asarray(p, dtype=np.float64)
    if np.any((p < 0.0) | (p >= 1.0)):
        raise ValueError("unit samples must lie in [0, 1)")
    p = np.where(p == 0.0, np.nextafter(0.0, 1.0), p)
    out = np.empty_like(p)
    lo = p < _PLOW
    hi = p > 1.0 - _PLOW
    mid = ~(lo | hi)
    for mask, tail in ((lo, p), (hi, 1.0 - p)):
        q = np.sqrt(-2.0 * np.log(tail[mask]))
        val = _horner(_C, q) / (_horner(_D, q) * q + 1.0)
        out[mask] = val if tail is p else -val
    q = p[mid] - 0.5
    r = q * q
    out[mid] = _horner(_A, r) * q / (_horner(_B, r) * r + 1.0)
    return out


def knot_count(horizon: int, degree: int = 3, override: int = 0) -> int:
    """default_knot_count (sampling.py:84-86) with the SmoothingSpec override (:62-72)."""
    return override or max(degree + 1, math.ceil(horizon / 6))


def bspline_design(horizon: int, k: int, degree: int) -> np.ndarray:
    """Clamped uniform B-spline basis at linspace(0,1,H) via Cox-de Boor (sampling.py:205-237)."""
    knots = np.concatenate([np.zeros(degree + 1), np.linspace(0.0, 1.0, k - degree + 1)[1:-1],
                            np.ones(degree + 1)])
    B = np.zeros((horizon, k))
    for row, t in enumerate(np.linspace(0.0, 1.0, horizon)):
        span = k - 1 if t >= 1.0 else int(np.searchsorted(knots, t, side="right")) - 1
        N = [1.0] + [0.0] * degree
        left = [0.0] * (degree + 1)
        right = [0.0] * (degree + 1)
        for j in range(1, degree + 1):
            left[j] = t - knots[span + 1 - j]
            right[j] = knots[span + j] - t
            carry = 0.0
            for r in range(j):
                frac = N[r] / (right[r + 1] + left[j - r])
                N[r] = carry + right[r + 1] * frac
                carry = left[j - r] * frac
            N[j] = carry
        B[row, span - degree:span + 1] = N
    return B


def smooth(knot_values: np.ndarray, mode: str, horizon: int, degree: int = 3,
           comb=(0.3, 0.4, 0.3)) -> np.ndarray:
    """(N,K,d) knot values -> (N,H,d) (sampling.py:240-265)."""
    x = np.asarray(knot_values, dtype=np.float64)
    if mode == "none":
        return x
    if mode == "comb":
        out = comb[0] * x
        out[:, 1:] += comb[1] * x[:, :-1]
        out[:, 2:] += comb[2] * x[:, :-2]
        return out
    return np.einsum("hk,nkd->nhd", bspline_design(horizon, x.shape[1], degree), x)


def fixed_halton_block(particles: int, horizon: int, dof: int, mode: str = "bspline",
                       degree: int = 3, knots: int = 0, comb=(0.3, 0.4, 0.3)) -> np.ndarray:
    """The Controller's once-drawn, batch-centred Halton set (controller.py:166-176)."""
    k = knot_count(horizon, degree, knots) if mode == "bspline" else horizon
    unit = halton(particles * k, dof).reshape(particles, k, dof)
    eps = smooth(acklam(unit), mode, horizon, degree, comb)
    return eps - eps.mean(axis=0, keepdims=True)


def shape_controls(eps, means, variances, null_count: int) -> np.ndarray:
    """u = mu + sqrt(var) eps with reserved rows (sampling.py:268-290). No clamping."""
    var = np.asarray(variances, dtype=np.float64)
    sd = np.sqrt(var) if var.ndim == 2 else np.sqrt(var)[:, None] * np.ones((1, means.shape[1]))
    u = means[None] + sd[None] * eps
    u[:null_count] = 0.0
    u[null_count] = means
    return u


def dt_schedule(horizon: int, dt_base: float, ramp: str) -> np.ndarray:
    """rollout.py:67-81."""
    if ramp == "uniform":
        return np.full(horizon, dt_base)
    if ramp == "two_phase":
        first = (horizon + 1) // 2
        return np.r_[np.full(first, dt_base), np.full(horizon - first, 2.0 * dt_base)]
    return np.linspace(dt_base, 2.0 * dt_base, horizon)


# ============================================================== dynamics + kinematics
def euler(u, dts, th0, thd0):
    """Sequential semi-implicit Euler (jit.py:335-349), vectorised over particles/joints."""
    u = np.asarray(u, dtype=np.float64)
    pos = np.empty_like(u)
    vel = np.empty_like(u)
    v = np.broadcast_to(np.asarray(thd0, float), u[:, 0].shape).copy()
    p = np.broadcast_to(np.asarray(th0, float), u[:, 0].shape).copy()
    for h in range(u.shape[1]):
        v = v + dts[h] * u[:, h]
        p = p + dts[h] * v
        vel[:, h] = v
        pos[:, h] = p
    return pos, vel


def _rodrigues(axis, angle):
    x, y, z = axis
    K = np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])
    s = np.sin(angle)[:, None, None]
    c = (1.0 - np.cos(angle))[:, None, None]
    return np.eye(3) + s * K + c * (K @ K)


def _polar(R):
    for _ in range(POLAR_ITERS):
        R = 0.5 * (R + np.swapaxes(np.linalg.inv(R), -1, -2))
    return R


def link_poses(q, chain):
    """World pose of every link frame: T_k = T_{k-1} Motion_k(q_k) Origin_k (jit.py:89-111)."""
    q = np.asarray(q, dtype=np.float64)
    M, d = q.shape
    rot = np.empty((M, d, 3, 3))
    trans = np.empty((M, d, 3))
    R = np.broadcast_to(np.eye(3), (M, 3, 3)).copy()
    t = np.zeros((M, 3))
    for k in range(d):
        if chain.jtype[k] == 0:
            Rm = _rodrigues(chain.axes[k], q[:, k])
            step_R = Rm @ chain.origin_rot[k]
            step_t = Rm @ chain.origin_trans[k]
        else:
            step_R = np.broadcast_to(chain.origin_rot[k], (M, 3, 3))
            step_t = q[:, k, None] * chain.axes[k] + chain.origin_trans[k]
        t = t + np.einsum("mij,mj->mi", R, step_t)
        R = R @ step_R
        if (k + 1) % REORTHO_EVERY == 0:
            R = _polar(R)
        rot[:, k] = R
        trans[:, k] = t
    return rot, trans


def geometric_jacobian(rot, trans, chain):
    """(M,6,d): a_k x (p_ee - p_{k-1}) over a_k, prismatic a_k over 0 (jit.py:114-148)."""
    M, d = trans.shape[0], trans.shape[1]
    J = np.zeros((M, 6, d))
    ee = trans[:, -1]
    for k in range(d):
        a = np.broadcast_to(chain.axes[0], (M, 3)) if k == 0 else rot[:, k - 1] @ chain.axes[k]
        origin = np.zeros((M, 3)) if k == 0 else trans[:, k - 1]
        if chain.jtype[k] == 0:
            J[:, :3, k] = np.cross(a, ee - origin)
            J[:, 3:, k] = a
        else:
            J[:, :3, k] = a
    return J


def manipulability(J, task_dim: int) -> np.ndarray:
    """sqrt(max(det(Jp Jp^T),0)), |det Jp| when square (jit.py:151-185)."""
    Jp = J[:, :task_dim, :]
    if Jp.shape[2] == task_dim:
        return np.abs(np.linalg.det(Jp))
    return np.sqrt(np.maximum(np.linalg.det(Jp @ np.swapaxes(Jp, 1, 2)), 0.0))


def _capsules_world(rot, trans, chain):
    R = rot[:, chain.cap_link]
    t = trans[:, chain.cap_link]
    return (np.einsum("mcij,cj->mci", R, chain.cap_p0) + t,
            np.einsum("mcij,cj->mci", R, chain.cap_p1) + t)


def segment_distance(p0, p1, q0, q1):
    """Closest distance of segment pairs with the numba branch order (jit.py:188-226)."""
    d1, d2, r = p1 - p0, q1 - q0, p0 - q0
    a = (d1 * d1).sum(-1)
    e = (d2 * d2).sum(-1)
    f = (d2 * r).sum(-1)
    c = (d1 * r).sum(-1)
    b = (d1 * d2).sum(-1)
    s = np.zeros_like(a)
    t = np.zeros_like(a)
    clip = lambda x: np.minimum(np.maximum(x, 0.0), 1.0)  # noqa: E731
    with np.errstate(divide="ignore", invalid="ignore"):
        pa, pe = a <= SEG_EPS, e <= SEG_EPS
        only_a = pa & ~pe
        t = np.where(only_a, clip(f / e), t)
        only_e = pe & ~pa
        s = np.where(only_e, clip(-c / a), s)
        gen = ~pa & ~pe
        den = a * e - b * b
        sg = np.where(np.abs(den) > SEG_EPS, clip((b * f - c * e) / den), 0.0)
        tg = (b * sg + f) / e
        sg = np.where(tg < 0.0, clip(-c / a), np.where(tg > 1.0, clip((b - c) / a), sg))
        tg = clip(tg)
        s = np.where(gen, sg, s)
        t = np.where(gen, tg, t)
    gap = (p0 + s[..., None] * d1) - (q0 + t[..., None] * d2)
    return np.sqrt((gap * gap).sum(-1))


def capsule_self_collision(rot, trans, chain) -> np.ndarray:
    """max_pairs r_i + r_j - segdist, NO_CONTACT without pairs (jit.py:241-260)."""
    if len(chain.pair_a) == 0:
        return np.full(rot.shape[0], NO_CONTACT)
    P0, P1 = _capsules_world(rot, trans, chain)
    ia, ib = chain.pair_a, chain.pair_b
    dist = segment_distance(P0[:, ia], P1[:, ia], P0[:, ib], P1[:, ib])
    return ((chain.cap_r[ia] + chain.cap_r[ib])[None] - dist).max(axis=1)


def _box_gap(p, lo, hi):
    g = np.maximum(lo - p, 0.0) + np.maximum(p - hi, 0.0)
    return np.sqrt((g * g).sum(-1))


def segment_box_distance(p0, p1, lo, hi):
    """TERNARY_ITERS ternary-search steps on the convex gap (jit.py:263-286)."""
    a = np.zeros(p0.shape[:-1])
    b = np.ones(p0.shape[:-1])
    d = p1 - p0
    for _ in range(TERNARY_ITERS):
        m1 = a + (b - a) / 3.0
        m2 = b - (b - a) / 3.0
        go_left = _box_gap(p0 + m1[..., None] * d, lo, hi) <= _box_gap(p0 + m2[..., None] * d, lo, hi)
        b = np.where(go_left, m2, b)
        a = np.where(go_left, a, m1)
    mid = 0.5 * (a + b)
    return _box_gap(p0 + mid[..., None] * d, lo, hi)


def first_obstacle_hit(rot, trans, chain, spheres, boxes) -> np.ndarray:
    """First obstacle index (spheres, then boxes), -1 when clear; strict (jit.py:289-332)."""
    M = rot.shape[0]
    hit = np.full(M, -1, dtype=np.int64)
    if len(chain.cap_r) == 0 or (len(spheres) == 0 and len(boxes) == 0):
        return hit
    P0, P1 = _capsules_world(rot, trans, chain)
    d = P1 - P0
    dd = (d * d).sum(-1)
    for o, sph in enumerate(spheres):
        with np.errstate(divide="ignore", invalid="ignore"):
            t = np.where(dd <= SEG_EPS, 0.0,
                         np.minimum(np.maximum(((sph[:3] - P0) * d).sum(-1) / dd, 0.0), 1.0))
        close = P0 + t[..., None] * d - sph[:3]
        inside = (np.sqrt((close * close).sum(-1)) < chain.cap_r[None] + sph[3]).any(axis=1)
        hit = np.where((hit < 0) & inside, o, hit)
    for ob, box in enumerate(boxes):
        inside = (segment_box_distance(P0, P1, box[:3], box[3:]) < chain.cap_r[None]).any(axis=1)
        hit = np.where((hit < 0) & inside, len(spheres) + ob, hit)
    return hit


def obstacle_margin(rot, trans, chain, spheres, boxes) -> np.ndarray:
    """Signed clearance behind first_obstacle_hit's decision (jit.py:289-332):
    min over capsules and obstacles of (segment distance - contact radius);
    the reference reports a hit exactly when this is < 0 (strict). +inf with
    no capsules or no obstacles. Test infrastructure for the SURVEY §8(c)
    decision band: entries with |margin| < band may take either branch."""
    M = rot.shape[0]
    out = np.full(M, np.inf)
    if len(chain.cap_r) == 0 or (len(spheres) == 0 and len(boxes) == 0):
        return out
    P0, P1 = _capsules_world(rot, trans, chain)
    d = P1 - P0
    dd = (d * d).sum(-1)
    for sph in spheres:
        with np.errstate(divide="ignore", invalid="ignore"):
            t = np.where(dd <= SEG_EPS, 0.0,
                         np.minimum(np.maximum(((sph[:3] - P0) * d).sum(-1) / dd, 0.0), 1.0))
        close = P0 + t[..., None] * d - sph[:3]
        gap = np.sqrt((close * close).sum(-1)) - (chain.cap_r[None] + sph[3])
        out = np.minimum(out, gap.min(axis=1))
    for box in boxes:
        gap = segment_box_distance(P0, P1, box[:3], box[3:]) - chain.cap_r[None]
        out = np.minimum(out, gap.min(axis=1))
    return out


# ============================================================== costs
TERMS = ("pose", "stop", "joint", "manip", "selfcoll", "envcoll")


def pose_term(rot_ee, trans_ee, goal_R, goal_t, full_pose: bool, a_rot, a_trans):
    """costs.py:76-95: ||a_t * Rg^T (t - tg)|| (+ ||diag(a_r)(I - Rg^T R)||_F)."""
    err = np.einsum("ji,...j->...i", goal_R, trans_ee - goal_t)
    out = np.sqrt(((np.asarray(a_trans) * err) ** 2).sum(-1))
    if full_pose:
        res = np.asarray(a_rot)[:, None] * (np.eye(3) - np.einsum("ji,...jk->...ik", goal_R, rot_ee))
        out = out + np.sqrt((res * res).sum((-2, -1)))
    return out


def mlp_distance(q, state: dict) -> np.ndarray:
    """posenc + ReLU MLP, float64 (surrogate.py:24-52, 120-125)."""
    h = np.concatenate([np.sin(q), np.cos(q)], axis=-1)
    i = 0
    while f"W{i}" in state:
        h = h @ state[f"W{i}"] + state[f"b{i}"]
        if f"W{i + 1}" in state:
            h = np.maximum(h, 0.0)
        i += 1
    return h[..., 0]


def cost_terms(pos, vel, dts, chain, weights, goal_R, goal_t, full_pose: bool, provider=None,
               mlp_state=None, spheres=None, boxes=None, decisions=None):
    """CostStack.evaluate (costs.py:209-242): returns (step (n,H), terms dict).

    provider: None | "oracle" | "learned" (mlp_state holds W0..W3, b0..b3).
    decisions: optional dict, filled with the margins of the two discontinuous
    branches (SURVEY §8(c) decision bands): "manip" = m - k_m (the cost jumps
    where it crosses 0, costs.py:126-127) and "env" = obstacle_margin (hit iff
    < 0), both (n,H); +inf where the term is off.
    """
    n, H, d = pos.shape
    flat = pos.reshape(-1, d)
    rot, trans = link_poses(flat, chain)
    terms = {k: np.zeros((n, H)) for k in TERMS}
    terms["pose"] = pose_term(rot[:, -1], trans[:, -1], goal_R, goal_t, full_pose, weights.alpha_rot,
                              weights.alpha_trans).reshape(n, H)
    if weights.alpha_stop > 0.0:
        remaining = np.cumsum(np.asarray(dts)[::-1])[::-1]
        limit = remaining[:, None] * np.asarray(chain.accel_limits)[None]
        excess = np.maximum(np.abs(vel) - limit[None], 0.0)
        terms["stop"] = np.sqrt((excess * excess).sum(-1))
    if weights.alpha_joint > 0.0:
        span = chain.joint_limits[:, 1] - chain.joint_limits[:, 0]
        lo = chain.joint_limits[:, 0] + weights.k_jl * span
        hi = chain.joint_limits[:, 1] - weights.k_jl * span
        depth = np.maximum(lo - pos, 0.0) + np.maximum(pos - hi, 0.0)
        terms["joint"] = np.sqrt((depth * depth).sum(-1))
    if weights.alpha_manip > 0.0:
        m = manipulability(geometric_jacobian(rot, trans, chain), chain.task_dim).reshape(n, H)
        terms["manip"] = np.where(m < weights.k_m, 1.0 - m, 0.0)
        if decisions is not None:
            decisions["manip"] = m - weights.k_m
    if weights.alpha_coll > 0.0 and provider == "oracle":
        terms["selfcoll"] = np.maximum(capsule_self_collision(rot, trans, chain), 0.0).reshape(n, H)
    elif weights.alpha_coll > 0.0 and provider == "learned":
        terms["selfcoll"] = np.maximum(mlp_distance(pos, mlp_state), 0.0)
    n_obs = (0 if spheres is None else len(spheres)) + (0 if boxes is None else len(boxes))
    if weights.alpha_coll > 0.0 and n_obs:
        sp = np.zeros((0, 4)) if spheres is None else spheres
        bx = np.zeros((0, 6)) if boxes is None else boxes
        terms["envcoll"] = (first_obstacle_hit(rot, trans, chain, sp, bx) >= 0).astype(float).reshape(n, H)
        if decisions is not None:
            decisions["env"] = obstacle_margin(rot, trans, chain, sp, bx).reshape(n, H)
    if decisions is not None:
        for k in ("manip", "env"):
            decisions.setdefault(k, np.full((n, H), np.inf))
    step = (terms["pose"] + weights.alpha_stop * terms["stop"] + weights.alpha_joint * terms["joint"]
            + weights.alpha_manip * terms["manip"]
            + weights.alpha_coll * (terms["selfcoll"] + terms["envcoll"]))
    return step, terms


def discounted(step, gamma: float, terminal_weight: float) -> np.ndarray:
    """rollout.py:111-121."""
    H = step.shape[1]
    g = gamma ** np.arange(H)
    return step[:, :-1] @ g[:-1] + g[-1] * terminal_weight * step[:, -1]


def rollout_scores(th0, thd0, u, dts, chain, weights, goal_R, goal_t, full_pose, gamma, terminal_weight,
                   chunk=None, keep=None, **kw):
    """evaluate_rollouts (rollout.py:124-180) incl. quarantine of non-finite rows.

    chunk: evaluate `chunk` particles at a time (the reference's own per-slice
    evaluation, rollout.py:149-162, is what makes this exact: rows are
    independent) so N >= 65k fits in memory (SURVEY §8(c) "Scale limits").
    keep: names of the per-row outputs to keep (default all); with "decisions"
    the branch margins of cost_terms are returned as well.
    """
    if not np.isfinite(u).all():
        bad = int(np.flatnonzero(~np.isfinite(u).all(axis=(1, 2)))[0])
        raise ValueError(f"non-finite control in particle {bad}")
    keep = set(keep or ("positions", "velocities", "accelerations", "step_costs", "terms"))
    n = u.shape[0]
    chunk = n if not chunk else int(chunk)
    parts = []
    for a in range(0, n, chunk):
        uc = u[a:a + chunk]
        pos, vel = euler(uc, dts, th0, thd0)
        dec = {} if "decisions" in keep else None
        step, terms = cost_terms(pos, vel, dts, chain, weights, goal_R, goal_t, full_pose, decisions=dec, **kw)
        ok = np.isfinite(step).all(axis=1)
        step = np.where(ok[:, None], step, 0.0)
        totals = discounted(step, gamma, terminal_weight)
        totals[~ok] = np.inf
        rec = dict(positions=pos, velocities=vel, accelerations=uc, step_costs=step, terms=terms,
                   totals=totals, decisions=dec)
        parts.append({k: v for k, v in rec.items() if k in keep or k == "totals"})
    if len(parts) == 1:
        return parts[0]
    out = {}
    for k in parts[0]:
        if isinstance(parts[0][k], dict):
            out[k] = {t: np.concatenate([p[k][t] for p in parts]) for t in parts[0][k]}
        else:
            out[k] = np.concatenate([p[k] for p in parts])
    return out


# ============================================================== policy update
def weights_from_totals(totals, beta: float) -> np.ndarray:
    """exp(-(c - min_finite)/beta), +inf -> 0 (policy.py:103-121)."""
    ok = np.isfinite(totals)
    if not ok.any():
        raise RuntimeError("all particles quarantined; no finite costs")
    w = np.zeros_like(totals)
    w[ok] = np.exp(-(totals[ok] - totals[ok].min()) / beta)
    if w.sum() <= 0.0:
        raise RuntimeError("all particle weights underflowed to zero; increase beta")
    return w


def blend_policy(means, variances, u, w, alpha_mu, alpha_sigma, smin, smax, isotropic=False):
    """update_mean then update_covariance around the NEW mean (policy.py:124-155)."""
    W = w.sum()
    mu = (1.0 - alpha_mu) * means + alpha_mu * np.einsum("n,nhd->hd", w, u) / W
    dev = u - mu[None]
    emp = np.einsum("n,nhd->hd", w, dev * dev) / W
    if isotropic:
        emp = emp.mean(axis=1)
    var = np.clip((1.0 - alpha_sigma) * variances + alpha_sigma * emp, smin, smax)
    return mu, var


def shifted(means, variances, tail_mean: float, tail_var: float):
    """policy.py:158-167."""
    m = np.concatenate([means[1:], np.full((1,) + means.shape[1:], tail_mean)])
    v = np.concatenate([variances[1:], np.full((1,) + variances.shape[1:], tail_var)])
    return m, v


def shard_record(totals, dev, beta: float) -> np.ndarray:
    """Restatement of one rank's statistics record for the particle-sharded
    update: [m_k, S0_k, count_k, sumfinite_k, status, bad,
    S1_k (H*d), S2_k (H*d)] with weights relative to the LOCAL minimum and
    deviations dev = u - mu_old (n_local, H, d)."""
    ok = np.isfinite(totals)
    m = totals[ok].min() if ok.any() else np.inf
    w = np.zeros_like(totals)
    if ok.any():
        w[ok] = np.exp(-(totals[ok] - m) / beta)
    s1 = np.einsum("n,nhd->hd", w, dev).ravel()
    s2 = np.einsum("n,nhd->hd", w, dev * dev).ravel()
    head = [m, w.sum(), float(ok.sum()), float(totals[ok].sum()), 0.0, 2147483647.0]
    return np.concatenate([head, s1, s2])


def combine_and_update(records, means, variances, alpha_mu, alpha_sigma, smin, smax, beta,
                       isotropic=False):
    """Fixed-order combine of rank records + update_mean/update_covariance,
    algebraically equal to blend_policy over the concatenated particles."""
    records = np.asarray(records)
    HD = means.size
    ok = records[:, 2] > 0
    m = records[ok, 0].min()
    scale = np.where(ok, np.exp(-(records[:, 0] - m) / beta), 0.0)
    S0 = (scale * records[:, 1]).sum()
    S1 = (scale[:, None] * records[:, 6:6 + HD]).sum(0).reshape(means.shape)
    S2 = (scale[:, None] * records[:, 6 + HD:6 + 2 * HD]).sum(0).reshape(means.shape)
    mu = (1.0 - alpha_mu) * means + alpha_mu * (means + S1 / S0)
    delta = mu - means
    emp = S2 / S0 - 2.0 * delta * (S1 / S0) + delta * delta
    if isotropic:
        emp = emp.mean(axis=1)
    var = np.clip((1.0 - alpha_sigma) * variances + alpha_sigma * emp, smin, smax)
    return mu, var


class OracleController:
    """Controller.control_step (controller.py:198-260) restated: shift, K x
    (perturb, shape, rollout, weights, mean, covariance), command = means[0].

    ``eps_source`` is a callable returning the (N,H,d) perturbation block of
    each iteration (the fixed centred Halton set by default).
    """

    def __init__(self, chain, weights, goal_R, goal_t, full_pose, *, horizon=30, particles=200,
                 dt_base=0.05, dt_ramp="two_phase", gamma=0.99, terminal_weight=1.0, null_count=2,
                 beta=0.5, alpha_mu=0.9, alpha_sigma=0.5, sigma0_sq=1.0, sigma_sq_min=1e-4,
                 sigma_sq_max=0.0, isotropic=False, iterations=1, provider=None, mlp_state=None,
                 spheres=None, boxes=None, smoothing="bspline", degree=3, knots=0, eps_source=None,
                 chunk=None, keep=None):
        self.chain, self.weights = chain, weights
        self.goal_R, self.goal_t, self.full_pose = np.asarray(goal_R, float), np.asarray(goal_t, float), full_pose
        self.H, self.N, self.null = horizon, particles, null_count
        self.dts = dt_schedule(horizon, dt_base, dt_ramp)
        self.gamma, self.tw, self.beta = gamma, terminal_weight, beta
        self.alpha_mu, self.alpha_sigma = alpha_mu, alpha_sigma
        self.sigma0_sq = sigma0_sq
        self.smin = sigma_sq_min
        self.smax = sigma_sq_max if sigma_sq_max > 0.0 else sigma0_sq
        self.iso = isotropic
        self.iterations = max(1, iterations)
        self.kw = dict(provider=provider, mlp_state=mlp_state, spheres=spheres, boxes=boxes)
        d = chain.axes.shape[0]
        self.means = np.zeros((horizon, d))
        self.variances = np.full(horizon, sigma0_sq) if isotropic else np.full((horizon, d), sigma0_sq)
        if eps_source is None:
            block = fixed_halton_block(particles, horizon, d, smoothing, degree, knots)
            eps_source = lambda: block  # noqa: E731
        self.eps_source = eps_source
        self.chunk, self.keep = chunk, keep  # chunked evaluation for N >= 65k (rollout_scores)
        self.last = None

    def step(self, theta, theta_dot):
        self.means, self.variances = shifted(self.means, self.variances, 0.0, self.sigma0_sq)
        for _ in range(self.iterations):
            eps = self.eps_source()
            u = shape_controls(eps, self.means, self.variances, self.null)
            res = rollout_scores(theta, theta_dot, u, self.dts, self.chain, self.weights, self.goal_R,
                                 self.goal_t, self.full_pose, self.gamma, self.tw, chunk=self.chunk,
                                 keep=self.keep, **self.kw)
            res["controls"] = u
            w = weights_from_totals(res["totals"], self.beta)
            self.means, self.variances = blend_policy(self.means, self.variances, u, w, self.alpha_mu,
                                                      self.alpha_sigma, self.smin, self.smax, self.iso)
            res["weights"] = w
            res["eps"] = eps
        fin = res["totals"][np.isfinite(res["totals"])]
        res["best_cost"], res["mean_cost"] = float(fin.min()), float(fin.mean())
        res["command"] = self.means[0].copy()
        self.last = res
        return res["command"]
