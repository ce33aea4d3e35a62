"""World models for the collision term (jointmpc/simworld.py:30-105) plus the
voxel-grid world of BASELINE config 3.

WorldModel keeps the reference's packed primitives (spheres (ns,4), boxes
(nb,6); indices count spheres first). A VoxelGrid world is an occupancy grid
whose occupied set is exactly a union of voxel-aligned boxes: the GPU gets the
grid (clearance field for the broad phase) and the exact box decomposition for
the narrow phase, the CPU oracle gets the same boxes as ``WorldModel.boxes``,
so both evaluate the same occupied set (SURVEY §8(c) "Config 3 bridge").
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ConfigError, ContractError
from .kinematics import FIXTURES

_SLAB = 1.0e18  # z half-extent of extruded planar boxes (simworld.py:24)
HOLD = "hold"
LINEAR = "linear"


@dataclass(frozen=True)
class VoxelGrid:
    occupancy: np.ndarray  # (nx, ny, nz) uint8/bool
    origin: np.ndarray  # (3,) world position of voxel (0,0,0)'s min corner
    voxel: float

    def boxes(self) -> np.ndarray:
        """Exact box decomposition of the occupied set (same greedy order as the
        native mppi_set_voxel_world): z-runs, grown along y, then x."""
        occ = np.asarray(self.occupancy).astype(bool).copy()
        nx, ny, nz = occ.shape
        out = []
        for i in range(nx):
            for j in range(ny):
                for k in range(nz):
                    if not occ[i, j, k]:
                        continue
                    k1 = k
                    while k1 + 1 < nz and occ[i, j, k1 + 1]:
                        k1 += 1
                    j1 = j
                    while j1 + 1 < ny and occ[i, j1 + 1, k:k1 + 1].all():
                        j1 += 1
                    i1 = i
                    while i1 + 1 < nx and occ[i1 + 1, j:j1 + 1, k:k1 + 1].all():
                        i1 += 1
                    occ[i:i1 + 1, j:j1 + 1, k:k1 + 1] = False
                    o, v = self.origin, self.voxel
                    out.append([o[0] + i * v, o[1] + j * v, o[2] + k * v,
                                o[0] + (i1 + 1) * v, o[1] + (j1 + 1) * v, o[2] + (k1 + 1) * v])
        return np.asarray(out, dtype=np.float64).reshape(-1, 6)


@dataclass(frozen=True)
class WorldModel:
    spheres: np.ndarray
    boxes: np.ndarray
    bounds_min: np.ndarray
    bounds_max: np.ndarray
    name: str = "world"
    voxel_grid: VoxelGrid | None = None

    def __post_init__(self):
        if self.spheres.size and np.any(self.spheres[:, 3] <= 0.0):
            raise ConfigError("sphere radii must be positive")
        if self.boxes.size and np.any(self.boxes[:, 3:] <= self.boxes[:, :3]):
            raise ConfigError("box min must be strictly below max componentwise")

    @property
    def obstacle_count(self) -> int:
        return self.spheres.shape[0] + self.boxes.shape[0]


def empty_world() -> WorldModel:
    return WorldModel(spheres=np.zeros((0, 4)), boxes=np.zeros((0, 6)),
                      bounds_min=np.array([-1.0, -1.0, -1.0]), bounds_max=np.array([1.0, 1.0, 1.0]),
                      name="empty")


def world_from_dict(data: dict, name: str = "world") -> WorldModel:
    spheres, boxes = [], []
    for i, ob in enumerate(data.get("obstacles", [])):
        kind = ob.get("type")
        if kind == "disc":
            cx, cy = ob["center"]
            spheres.append([cx, cy, 0.0, ob["radius"]])
        elif kind == "sphere":
            spheres.append([*ob["center"], ob["radius"]])
        elif kind == "box":
            lo, hi = list(ob["min"]), list(ob["max"])
            if len(lo) == 2:
                lo, hi = [*lo, -_SLAB], [*hi, _SLAB]
            boxes.append(lo + hi)
        else:
            raise ConfigError(f"obstacle {i}: unknown type {kind!r}")
    bounds = data.get("bounds", {})
    lo = list(bounds.get("min", (-1.0, -1.0)))
    hi = list(bounds.get("max", (1.0, 1.0)))
    if len(lo) == 2:
        lo, hi = [*lo, -1.0], [*hi, 1.0]
    return WorldModel(spheres=np.asarray(spheres, dtype=np.float64).reshape(-1, 4),
                      boxes=np.asarray(boxes, dtype=np.float64).reshape(-1, 6),
                      bounds_min=np.asarray(lo, dtype=np.float64),
                      bounds_max=np.asarray(hi, dtype=np.float64), name=data.get("name", name))


def load_world(path) -> WorldModel:
    p = Path(path)
    if not p.exists():
        candidate = FIXTURES / p.name
        if not candidate.exists():
            raise ConfigError(f"world file not found: {path}")
        p = candidate
    with open(p) as fh:
        return world_from_dict(json.load(fh), name=p.stem)


def voxel_world(occupancy, origin, voxel: float, spheres=None, name: str = "voxel") -> WorldModel:
    grid = VoxelGrid(occupancy=np.asarray(occupancy, dtype=np.uint8), origin=np.asarray(origin, float),
                     voxel=float(voxel))
    boxes = grid.boxes()
    sp = np.zeros((0, 4)) if spheres is None else np.asarray(spheres, dtype=np.float64).reshape(-1, 4)
    o = grid.origin
    ext = np.array(grid.occupancy.shape) * grid.voxel
    return WorldModel(spheres=sp, boxes=boxes, bounds_min=o.copy(), bounds_max=o + ext, name=name,
                      voxel_grid=grid)


def seeded_box_grid(n_boxes: int = 8, dims: int = 64, lo: float = -1.0, hi: float = 1.0, seed: int = 0,
                    keep_clear=None, max_extent: int = 10) -> WorldModel:
    """Config 3 world: a dims^3 grid over [lo,hi]^3 built from n_boxes seeded
    voxel-aligned boxes. ``keep_clear(box) -> bool`` rejects boxes (e.g. ones
    overlapping the start pose's capsules)."""
    rng = np.random.default_rng(seed)
    voxel = (hi - lo) / dims
    occ = np.zeros((dims, dims, dims), dtype=np.uint8)
    placed = 0
    tries = 0
    while placed < n_boxes:
        tries += 1
        if tries > 10000:
            raise ConfigError("could not place the requested boxes")
        size = rng.integers(2, max_extent + 1, size=3)
        start = np.array([rng.integers(0, dims - s + 1) for s in size])
        box = np.concatenate([lo + start * voxel, lo + (start + size) * voxel])
        if keep_clear is not None and not keep_clear(box):
            continue
        occ[start[0]:start[0] + size[0], start[1]:start[1] + size[1], start[2]:start[2] + size[2]] = 1
        placed += 1
    return voxel_world(occ, origin=np.full(3, lo), voxel=voxel, name=f"grid{dims}_seed{seed}")


# ---------------------------------------------------------------- goal scripting (host, per step)
@dataclass(frozen=True)
class TargetScript:
    """Timed goal positions, hold or linear interpolation (simworld.py:130-149)."""

    times: np.ndarray
    positions: np.ndarray
    interpolation: str = HOLD
    source: str = "scripted"
    mode: str = "position_only"

    def __post_init__(self):
        object.__setattr__(self, "times", np.asarray(self.times, dtype=np.float64))
        object.__setattr__(self, "positions", np.atleast_2d(np.asarray(self.positions, dtype=np.float64)))
        if self.times.size == 0:
            raise ConfigError("target script needs at least one waypoint")
        if np.any(np.diff(self.times) <= 0.0):
            raise ConfigError("waypoint times must be strictly increasing")
        if self.interpolation not in (HOLD, LINEAR):
            raise ConfigError(f"unknown interpolation {self.interpolation!r}")


def target_position_at(script: TargetScript, t: float) -> np.ndarray:
    if t < 0.0:
        raise ContractError("time must be non-negative")
    times, pts = script.times, script.positions
    if t <= times[0]:
        return pts[0].copy()
    if t >= times[-1]:
        return pts[-1].copy()
    hi = int(np.searchsorted(times, t, side="right"))
    lo = hi - 1
    if script.interpolation == HOLD:
        return pts[lo].copy()
    frac = (t - times[lo]) / (times[hi] - times[lo])
    return (1.0 - frac) * pts[lo] + frac * pts[hi]


def target_at(script: TargetScript, t: float):
    from .costs import goal_at_position

    return goal_at_position(target_position_at(script, t), mode=script.mode)


def script_from_waypoints(waypoints, interpolation: str = HOLD, mode: str = "position_only") -> TargetScript:
    """TargetScript from (time, position) pairs or flat [time, x, y(, z)] rows (simworld.py:152-165)."""
    times, positions = [], []
    for w in waypoints:
        times.append(float(w[0]))
        positions.append(_pad3(w[1] if len(w) == 2 and np.ndim(w[1]) == 1 else w[1:]))
    return TargetScript(times=np.array(times), positions=np.array(positions),
                        interpolation=interpolation, mode=mode)


def _pad3(p) -> np.ndarray:
    """Planar positions get z = 0 (simworld.py:168-172)."""
    p = np.asarray(p, dtype=np.float64).ravel()
    return np.array([p[0], p[1], 0.0]) if p.size == 2 else p


# ---------------------------------------------------------------- plant (host form)
def sim_step(state, command, dt: float, noise_sigma: float = 0.0, rng=None):
    """One plant step (simworld.py:108-127): the rollouts' semi-implicit Euler
    plus optional Gaussian state noise drawn from ``rng`` (position first, then
    velocity). run_episode's device loop consumes the same draws."""
    from .rollout import JointState

    if dt <= 0.0:
        raise ContractError("dt must be positive")
    u = np.asarray(command, dtype=np.float64)
    vel = state.theta_dot + dt * u
    pos = state.theta + dt * vel
    if noise_sigma > 0.0:
        if rng is None:
            raise ContractError("state noise requires an rng")
        pos = pos + rng.normal(0.0, noise_sigma, size=pos.shape)
        vel = vel + rng.normal(0.0, noise_sigma, size=vel.shape)
    return JointState(theta=pos, theta_dot=vel, theta_ddot=u.copy(), stamp=state.stamp + dt)


def collision_query(world: WorldModel, chain, rot, trans):
    """(collided, first obstacle index) of one configuration's link poses
    through the operator seam's env_collision_batch (simworld.py:200-212)."""
    from . import kernels

    rot = np.asarray(rot, dtype=np.float64).reshape(1, chain.dof, 3, 3)
    trans = np.asarray(trans, dtype=np.float64).reshape(1, chain.dof, 3)
    hit = kernels.env_collision_batch(rot, trans, chain.cap_p0, chain.cap_p1, chain.cap_r, chain.cap_link,
                                      world.spheres, world.boxes)[0]
    return bool(hit >= 0), int(hit)
