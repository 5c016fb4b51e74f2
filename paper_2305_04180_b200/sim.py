"""Host-side environment description: maps, per-episode parameters, config.

Mirrors the reference's configuration surface so callers can switch without
edits (``sim/params.py``, ``sim/gridmap.py``, ``sim/reward.py:16-30``,
``sim/core.py:35``).  These are plain host objects; all stepping happens in
libsparrow.  Any object exposing the same attributes (e.g. the reference's
own ``GridMap`` / ``DiversityRanges`` / ``EnvConfig``) is accepted wherever
these types are.

Differences from the reference, both deliberate:
* the observation width is ``5 + n_beams`` for every beam count (the
  reference hard-codes ``STATE_DIM = 32``, ``sim/core.py:32``, which only
  fits 27 beams);
* no EDT is stored with a map: the GPU marcher derives its own skip table.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import IntEnum
from pathlib import Path

import numpy as np

ACTION_TABLE = ((0.36, 1.0), (18.0, 1.0), (18.0, 0.0), (18.0, -1.0), (0.36, -1.0))  # params.py:12-18
MAX_CONTROL_DELAY = 64  # params.py:20

REWARD_COLLISION = -10.0  # reward.py:23-24
REWARD_ARRIVAL = 75.0


class Event(IntEnum):  # reward.py:16-20
    NONE = 0
    COLLISION = 1
    ARRIVAL = 2
    TIMEOUT = 3


class MapError(ValueError):
    """Malformed or unusable map, mixed grid shapes, or no spawn pose found."""


class EpisodeTerminated(RuntimeError):
    """A finished lane was stepped without a reset (auto_reset=False)."""


@dataclass(frozen=True)
class SimParams:
    """One episode's physics draw (params.py:23-52)."""

    k: float = 0.6
    control_interval_s: float = 0.1
    control_delay_steps: int = 1
    v_linear_max_cm_s: float = 18.0
    v_angular_max_rad_s: float = 1.0
    lidar_noise_std_cm: float = 1.0

    def __post_init__(self):
        problems = []
        if not 0.0 < self.k < 1.0:
            problems.append(f"k must lie in (0, 1), got {self.k}")
        if self.control_interval_s <= 0:
            problems.append("control interval must be positive")
        if not 0 <= self.control_delay_steps <= MAX_CONTROL_DELAY:
            problems.append(f"control delay must be in [0, {MAX_CONTROL_DELAY}]")
        if self.v_linear_max_cm_s <= 0 or self.v_angular_max_rad_s <= 0:
            problems.append("velocity limits must be positive")
        if self.lidar_noise_std_cm < 0:
            problems.append("lidar noise std must be non-negative")
        if problems:
            raise ValueError("; ".join(problems))


_PARAM_FIELDS = ("k", "control_interval_s", "control_delay_steps", "v_linear_max_cm_s",
                 "v_angular_max_rad_s", "lidar_noise_std_cm")


@dataclass(frozen=True)
class DiversityRanges:
    """Per-episode resampling intervals, one per SimParams field (params.py:55-121).
    Sampling happens on the GPU, in the fixed order k, dt, delay, vmax_l,
    vmax_a, noise (uniform / uniform / integer-inclusive / uniform x3)."""

    k: tuple = (0.6, 0.6)
    control_interval_s: tuple = (0.1, 0.1)
    control_delay_steps: tuple = (1, 1)
    v_linear_max_cm_s: tuple = (18.0, 18.0)
    v_angular_max_rad_s: tuple = (1.0, 1.0)
    lidar_noise_std_cm: tuple = (1.0, 1.0)

    def __post_init__(self):
        for name in _PARAM_FIELDS:
            lo, hi = getattr(self, name)
            if lo > hi:
                raise ValueError(f"{name} interval is reversed: ({lo}, {hi})")
        SimParams(*(getattr(self, f)[0] for f in _PARAM_FIELDS))
        SimParams(*(getattr(self, f)[1] for f in _PARAM_FIELDS))

    @classmethod
    def around(cls, nominal: SimParams, fraction: float) -> "DiversityRanges":
        """+/- fraction bands; the delay band rounds outward (params.py:85-110)."""
        if fraction < 0:
            raise ValueError("diversity fraction must be non-negative")
        lo_f, hi_f = 1.0 - fraction, 1.0 + fraction
        d = nominal.control_delay_steps
        bands = {name: (getattr(nominal, name) * lo_f, getattr(nominal, name) * hi_f)
                 for name in _PARAM_FIELDS if name != "control_delay_steps"}
        bands["control_delay_steps"] = (max(0, math.floor(d * lo_f)),
                                        min(MAX_CONTROL_DELAY, math.ceil(d * hi_f)))
        return cls(**bands)

    def sample(self, rng) -> SimParams:
        """Host-side draw in the reference order (for API parity; the GPU
        performs the same draws in-kernel)."""
        return SimParams(
            k=float(rng.uniform(*self.k)),
            control_interval_s=float(rng.uniform(*self.control_interval_s)),
            control_delay_steps=int(rng.integers(self.control_delay_steps[0],
                                                 self.control_delay_steps[1] + 1)),
            v_linear_max_cm_s=float(rng.uniform(*self.v_linear_max_cm_s)),
            v_angular_max_rad_s=float(rng.uniform(*self.v_angular_max_rad_s)),
            lidar_noise_std_cm=float(rng.uniform(*self.lidar_noise_std_cm)),
        )


@dataclass(frozen=True)
class LidarConfig:
    """Beam fan centred on the heading (params.py:124-133)."""

    n_beams: int = 27
    fov_rad: float = math.radians(270.0)
    max_range_cm: float = 300.0

    def beam_offsets(self) -> np.ndarray:
        return np.linspace(-self.fov_rad / 2.0, self.fov_rad / 2.0, self.n_beams)

    @property
    def state_dim(self) -> int:
        return 5 + self.n_beams


@dataclass(frozen=True)
class EnvConfig:
    """Episode-independent settings (params.py:136-151)."""

    robot_radius_cm: float = 9.0
    timeout_steps: int = 1000
    max_planning_dist_cm: float = 0.0
    obstacle_penalty_range_cm: float = 30.0
    lidar: LidarConfig = field(default_factory=LidarConfig)
    action_table: tuple = ACTION_TABLE
    spawn_attempts: int = 256

    def planning_dist(self, grid_map) -> float:
        if self.max_planning_dist_cm > 0:
            return self.max_planning_dist_cm
        return math.hypot(grid_map.width_cm, grid_map.height_cm)


class GridMap:
    """Bordered occupancy grid with a goal disc and a spawn rectangle.

    Cell (ix, iy) covers [ix*c, (ix+1)*c) x [iy*c, (iy+1)*c); ``occupancy`` is
    indexed [iy, ix]; the text format lists rows top (high y) first with
    ``#`` obstacle, ``.`` free, ``G`` goal, ``S`` spawn and a
    ``width height cell`` header (gridmap.py:107-176).
    """

    def __init__(self, width_cm, height_cm, cell_size_cm, occupancy, goal_center,
                 goal_radius_cm, spawn_region):
        self.width_cm = int(width_cm)
        self.height_cm = int(height_cm)
        self.cell_size_cm = int(cell_size_cm)
        self.occupancy = np.asarray(occupancy, dtype=bool)
        self.goal_center = (float(goal_center[0]), float(goal_center[1]))
        self.goal_radius_cm = float(goal_radius_cm)
        self.spawn_region = tuple(float(v) for v in spawn_region)
        self._check()

    @property
    def n_cols(self) -> int:
        return self.width_cm // self.cell_size_cm

    @property
    def n_rows(self) -> int:
        return self.height_cm // self.cell_size_cm

    @property
    def diagonal_cm(self) -> float:
        return math.hypot(self.width_cm, self.height_cm)

    def cell_of(self, x_cm: float, y_cm: float) -> tuple:
        c = self.cell_size_cm
        return int(math.floor(x_cm / c)), int(math.floor(y_cm / c))

    def in_bounds(self, x_cm: float, y_cm: float) -> bool:
        return 0.0 <= x_cm < self.width_cm and 0.0 <= y_cm < self.height_cm

    def edt_cells(self) -> np.ndarray:
        """Euclidean distance (cell units, centre to centre) to the nearest
        occupied cell (gridmap.py:62-71). The device path does not use it: the
        marcher skips free space with its own per-cell free-box table. It is
        kept for API parity and computed once on first use."""
        if getattr(self, "_edt", None) is None:
            from scipy import ndimage
            self._edt = ndimage.distance_transform_edt(~self.occupancy).astype(np.float64)
        return self._edt

    def to_ascii(self, robot_xy=None) -> str:
        """Text-format body without the header; 'R' marks the robot's cell when
        a pose is given (gridmap.py:185-195)."""
        rows = self.to_text().splitlines()[1:]
        if robot_xy is not None:
            ix, iy = self.cell_of(*robot_xy)
            k = self.n_rows - 1 - iy
            if 0 <= k < len(rows) and 0 <= ix < self.n_cols:
                rows[k] = rows[k][:ix] + "R" + rows[k][ix + 1:]
        return "\n".join(rows)

    def _check(self) -> None:  # gridmap.py:75-103
        c = self.cell_size_cm
        if c <= 0:
            raise MapError("cell size must be a positive integer")
        if self.width_cm <= 0 or self.height_cm <= 0:
            raise MapError("map dimensions must be positive")
        if self.width_cm % c or self.height_cm % c:
            raise MapError("width and height must be exact multiples of the cell size")
        if self.occupancy.shape != (self.n_rows, self.n_cols):
            raise MapError(f"occupancy shape {self.occupancy.shape} does not match the "
                           f"declared {self.n_rows}x{self.n_cols} grid")
        occ = self.occupancy
        if not (occ[0].all() and occ[-1].all() and occ[:, 0].all() and occ[:, -1].all()):
            raise MapError("border cells must all be occupied")
        gx, gy = self.goal_center
        if not self.in_bounds(gx, gy):
            raise MapError("goal center lies outside map bounds")
        ix, iy = self.cell_of(gx, gy)
        if occ[iy, ix]:
            raise MapError("goal center lies on an occupied cell")
        if self.goal_radius_cm <= 0:
            raise MapError("goal radius must be positive")
        x0, y0, x1, y1 = self.spawn_region
        if not (0 <= x0 <= x1 <= self.width_cm and 0 <= y0 <= y1 <= self.height_cm):
            raise MapError("spawn region must be a rectangle inside map bounds")

    @classmethod
    def from_text(cls, text: str) -> "GridMap":
        lines = text.splitlines()
        if not lines:
            raise MapError("empty map text")
        head = lines[0].split()
        if len(head) != 3:
            raise MapError("header must be 'width height cell_size'")
        try:
            width, height, cell = (int(v) for v in head)
        except ValueError as exc:
            raise MapError(f"non-integer map header: {lines[0]!r}") from exc
        if cell <= 0 or width % cell or height % cell:
            raise MapError("dimensions must be positive multiples of the cell size")
        n_rows, n_cols = height // cell, width // cell
        rows = [ln for ln in lines[1:] if ln.strip()]
        if len(rows) != n_rows:
            raise MapError(f"expected {n_rows} grid rows, found {len(rows)}")
        if any(len(r) != n_cols for r in rows):
            bad = next(i for i, r in enumerate(rows) if len(r) != n_cols)
            raise MapError(f"row {bad + 1} has {len(rows[bad])} characters, expected {n_cols}")
        grid = np.array([list(r) for r in rows[::-1]], dtype="<U1").reshape(n_rows, n_cols)
        unknown = ~np.isin(grid, list("#.GS"))
        if unknown.any():
            r, _ = np.argwhere(unknown)[0]
            raise MapError(f"unknown map character {grid[unknown][0]!r} in row {n_rows - r}")
        occ = grid == "#"
        occ[0, :] = occ[-1, :] = occ[:, 0] = occ[:, -1] = True  # implicit walls
        goal = np.argwhere(grid == "G")  # (iy, ix)
        spawn = np.argwhere(grid == "S")
        if goal.size == 0:
            raise MapError("map has no goal ('G') cells")
        if spawn.size == 0:
            raise MapError("map has no spawn ('S') cells")
        centers = (goal[:, ::-1].astype(np.float64) + 0.5) * cell  # (x, y)
        # same cell ordering as a row-major scan of the text (gridmap.py:280-303)
        order = np.lexsort((goal[:, 1], -goal[:, 0]))
        centers = centers[order]
        goal_center = centers.mean(axis=0)
        radius = float(np.hypot(*(centers - goal_center).T).max() + cell / 2.0)
        sx, sy = spawn[:, 1], spawn[:, 0]
        region = (sx.min() * cell, sy.min() * cell, (sx.max() + 1) * cell, (sy.max() + 1) * cell)
        return cls(width, height, cell, occ, tuple(goal_center), radius, region)

    def to_text(self) -> str:
        c = self.cell_size_cm
        cx = (np.arange(self.n_cols) + 0.5) * c
        cy = (np.arange(self.n_rows) + 0.5) * c
        gx, gy = np.meshgrid(cx, cy)
        goal = np.hypot(gx - self.goal_center[0], gy - self.goal_center[1]) <= self.goal_radius_cm
        x0, y0, x1, y1 = self.spawn_region
        spawn = (gx >= x0) & (gx <= x1) & (gy >= y0) & (gy <= y1)
        grid = np.where(self.occupancy, "#", np.where(goal, "G", np.where(spawn, "S", ".")))
        body = "\n".join("".join(row) for row in grid[::-1])
        return f"{self.width_cm} {self.height_cm} {c}\n{body}\n"

    @classmethod
    def load(cls, path) -> "GridMap":
        return cls.from_text(Path(path).read_text())

    def save(self, path) -> None:
        Path(path).write_text(self.to_text())


def state_dim(config) -> int:
    return 5 + int(config.lidar.n_beams)
