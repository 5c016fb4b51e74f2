"""Procedural arenas, host side.

Drop-in for the reference's ``color_rl.mapgen`` (``mapgen.py:19-125``): a
bordered square arena with rectangular obstacle blocks, a spawn square in the
lower-left corner and a goal disc in the upper-right one. Map generation is
offline, one-time CPU work, so it stays on the host (numpy + scipy) and feeds
``GridMap``. The device tables are built from the GridMap at VecEnv creation
(per-cell free-box table + bitmap, ``sp_capi.cu build_cell_table``).

Determinism contract: the same ``numpy.random.Generator`` consumes the same
draws in the same order as the reference. Per block attempt that is
``uniform(w)``, ``uniform(h)``, ``integers(ix)``, ``integers(iy)``. So a seed
yields the reference's maps cell for cell. ``tests/test_host.py`` checks this
against ``tests/golden/maps16.npz``, which the reference generated with seed 0.
"""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np

from .sim import GridMap, MapError

__all__ = ["MapGenError", "generate_map", "generate_maps", "write_maps"]


class MapGenError(MapError):
    """No acceptable layout found for the requested parameters (mapgen.py:19-20)."""


def _bordered(n: int) -> np.ndarray:
    occ = np.zeros((n, n), dtype=bool)
    occ[0, :] = occ[-1, :] = occ[:, 0] = occ[:, -1] = True
    return occ


def _cell_centres(n: int, cell: int):
    c = (np.arange(n) + 0.5) * cell
    return np.meshgrid(c, c)  # (x, y) per cell, indexed [iy, ix]


def _scatter_blocks(rng, occ: np.ndarray, cell: int, target: int, size_range, gap: int) -> int:
    """Drop random rectangles until `target` new cells are covered or 10,000
    tries pass (mapgen.py:73-87). A rectangle that would sit within `gap`
    cells of an existing block without touching one is rejected. That way
    blocks either merge into clusters or leave a passable corridor. Returns the
    number of newly covered cells."""
    n = occ.shape[0]
    covered = 0
    for _ in range(10_000):
        if covered >= target:
            break
        w = int(rng.uniform(*size_range) / cell)
        h = int(rng.uniform(*size_range) / cell)
        ix = int(rng.integers(1, max(n - 1 - w, 2)))
        iy = int(rng.integers(1, max(n - 1 - h, 2)))
        rect = occ[iy:iy + h, ix:ix + w]
        halo = occ[max(iy - gap, 0):iy + h + gap, max(ix - gap, 0):ix + w + gap]
        overlap = int(rect.sum())
        if overlap == 0 and halo.any():
            continue
        rect[...] = True
        covered += w * h - overlap
    return covered


def _protected(n: int, cell: int, spawn_rect, goal_center, goal_radius: float,
               clear: float) -> np.ndarray:
    """Cells kept free: the spawn square and goal disc, grown by `clear`
    (mapgen.py:91-98)."""
    cx, cy = _cell_centres(n, cell)
    x0, y0, x1, y1 = spawn_rect
    near_spawn = (cx >= x0 - clear) & (cx <= x1 + clear) & (cy >= y0 - clear) & (cy <= y1 + clear)
    near_goal = np.sqrt((cx - goal_center[0]) ** 2 + (cy - goal_center[1]) ** 2) <= goal_radius + clear
    return near_spawn | near_goal


def _reachable(occ: np.ndarray, cell: int, spawn_rect, goal_center, goal_radius: float,
               robot_radius: float) -> bool:
    """Does one connected component of the robot's configuration space (cells
    whose centre has more than `robot_radius` of Euclidean clearance) meet both
    the spawn square and the goal disc? (mapgen.py:23-41)"""
    from scipy import ndimage
    free = ndimage.distance_transform_edt(~occ) * cell > robot_radius
    comp, count = ndimage.label(free)
    if count == 0:
        return False
    cx, cy = _cell_centres(occ.shape[0], cell)
    x0, y0, x1, y1 = spawn_rect
    at_spawn = free & (cx >= x0) & (cx <= x1) & (cy >= y0) & (cy <= y1)
    at_goal = free & (np.sqrt((cx - goal_center[0]) ** 2 + (cy - goal_center[1]) ** 2) <= goal_radius)
    a, b = np.unique(comp[at_spawn]), np.unique(comp[at_goal])
    return a.size > 0 and b.size > 0 and bool(np.intersect1d(a, b).size)


def generate_map(rng: np.random.Generator, size_cm: int = 366, cell_size_cm: int = 1,
                 density: float = 0.08, robot_radius_cm: float = 9.0,
                 goal_radius_cm: float = 20.0, spawn_size_cm: float = 70.0,
                 margin_cm: float = 10.0, block_range_cm=(20.0, 60.0),
                 min_gap_cm: float = 34.0, layout_attempts: int = 50) -> GridMap:
    """One random arena (mapgen.py:44-108). Raises MapGenError when no layout
    within `layout_attempts` both reaches 80 % of the requested density and
    connects spawn to goal for the robot's disc."""
    if not 0.0 <= density < 1.0:
        raise ValueError("density must lie in [0, 1)")
    cell = int(cell_size_cm)
    n = size_cm // cell
    if n < 8:
        raise ValueError("map too small for the requested cell size")
    spawn_rect = (margin_cm, margin_cm, margin_cm + spawn_size_cm, margin_cm + spawn_size_cm)
    corner = size_cm - margin_cm - goal_radius_cm - 10.0
    goal_center = (corner, corner)
    gap = max(int(math.ceil(min_gap_cm / cell)), 1)
    target = int(density * (n - 2) * (n - 2))
    keep = None
    for _ in range(layout_attempts):
        occ = _bordered(n)
        if _scatter_blocks(rng, occ, cell, target, block_range_cm, gap) < 0.8 * target:
            continue  # the gap rule could not realize the density: new layout
        if keep is None:
            keep = _protected(n, cell, spawn_rect, goal_center, goal_radius_cm,
                              robot_radius_cm + 3.0)
        occ &= ~keep
        occ |= _bordered(n)
        if _reachable(occ, cell, spawn_rect, goal_center, goal_radius_cm, robot_radius_cm):
            return GridMap(size_cm, size_cm, cell, occ, goal_center, goal_radius_cm, spawn_rect)
    raise MapGenError(f"no connected layout at density {density} after {layout_attempts} attempts")


def generate_maps(count: int, seed: int, size_cm: int = 366, cell_size_cm: int = 1,
                  density: float = 0.08, **kwargs) -> list:
    """`count` arenas from one Generator seeded with `seed` (mapgen.py:111-115)."""
    rng = np.random.default_rng(seed)
    return [generate_map(rng, size_cm=size_cm, cell_size_cm=cell_size_cm, density=density,
                         **kwargs) for _ in range(count)]


def write_maps(maps, out_dir, prefix: str = "map") -> list:
    """Save as ``<prefix>NN.txt`` (at least two digits) in the reference's text
    format (mapgen.py:118-125)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    width = max(2, len(str(max(len(maps) - 1, 1))))
    paths = []
    for i, m in enumerate(maps):
        p = out / f"{prefix}{i:0{width}d}.txt"
        m.save(p)
        paths.append(p)
    return paths
