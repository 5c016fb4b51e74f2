"""Shared test helpers: golden maps, configs, tolerance checks."""

from __future__ import annotations

import os

import numpy as np

from paper_2305_04180_b200.sim import DiversityRanges, EnvConfig, GridMap, LidarConfig, SimParams

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# Parity tolerance for floating outputs (north star: 1e-5 relative, fp32);
# absolute floor = fp32 resolution of each component's scale.
RTOL = 1e-5
ATOL_OBS = 2e-6     # obs are normalized to [-1, 1]
ATOL_REWARD = 1e-6


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def load_maps(n=16):
    z = golden("maps16.npz")
    ncols = int(z["n_cols"])
    out = []
    for i in range(n):
        occ = np.unpackbits(z["occ_packed"][i], axis=1)[:, :ncols].astype(bool)
        gx, gy, gr, x0, y0, x1, y1, w, h, c = z["meta"][i]
        out.append(GridMap(int(w), int(h), int(c), occ, (gx, gy), gr, (x0, y0, x1, y1)))
    return out


def config(n_beams=32, **kw):
    return EnvConfig(lidar=LidarConfig(n_beams=n_beams, **kw.pop("lidar_kw", {})), **kw)


def ranges(div=0.0):
    return DiversityRanges.around(SimParams(), div) if div > 0 else DiversityRanges()


def make_map(n_cells=20, cell=1, goal=None, goal_radius=2.0, spawn=None, blocks=()):
    """Bordered square map with rectangular blocks (cells [ix0, ix1) x [iy0, iy1))."""
    occ = np.zeros((n_cells, n_cells), dtype=bool)
    occ[0, :] = occ[-1, :] = occ[:, 0] = occ[:, -1] = True
    for ix0, iy0, ix1, iy1 in blocks:
        occ[iy0:iy1, ix0:ix1] = True
    size = n_cells * cell
    goal = goal or (0.7 * size, 0.7 * size)
    spawn = spawn or (0.3 * size, 0.3 * size, 0.45 * size, 0.45 * size)
    return GridMap(size, size, cell, occ, goal, goal_radius, spawn)


def assert_close(got, want, rtol=RTOL, atol=0.0, what=""):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    bad = np.abs(got - want) > atol + rtol * np.abs(want)
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(
            f"{what}: {int(bad.sum())}/{bad.size} outside rtol={rtol} atol={atol}; first "
            f"{[(tuple(i), float(got[tuple(i)]), float(want[tuple(i)])) for i in idx]}")
