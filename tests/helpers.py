"""Shared test helpers: golden maps, configs, tolerance checks."""

from __future__ import annotations

import os

import numpy as np

from paper_2305_04180_b200.sim import DiversityRanges, EnvConfig, GridMap, LidarConfig, SimParams

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# Parity tolerances.  The north star allows 1e-5 relative (fp32) for poses,
# velocities, LiDAR ranges and rewards; the kernels meet far tighter bars, and
# the tests hold them there so regressions show:
# * obs (float32, normalized to [-1, 1]): 2 float32 ulps at 1.0 -- the two
#   sides round fp64 values that agree to ~1e-13 (CUDA vs glibc libm ulps,
#   fp32 Box-Muller LiDAR noise ~1e-7 of sigma) to float32, so they may land
#   on adjacent floats, never further apart.  The oracle meets the same bar
#   against the reference (test_oracle_golden.OBS_ATOL);
# * rewards (float64): 1e-10 absolute + relative.  The reward arithmetic
#   itself agrees to ulps, but poses drift apart by up to ~1e-9 cm over an
#   episode: integrate_unicycle's x += (v/w)(sin h1 - sin h0) (kinematics.py:
#   52-55) multiplies a 1-ulp libm sin difference (CUDA vs glibc) by v/w,
#   up to 1.8e7 at |w| just above the 1e-6 straight-line cut.  Largest
#   reward difference observed at cfg3 scale: 1.2e-12;
# * poses: 1e-5 relative (the north star's own bar; observed ~1e-13).
RTOL = 1e-5
ATOL_OBS = 2.4e-7
RTOL_OBS = 2.4e-7
ATOL_REWARD = 1e-10
RTOL_REWARD = 1e-10


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


def assert_obs(got, want, what=""):
    assert_close(got, want, rtol=RTOL_OBS, atol=ATOL_OBS, what=what)


def assert_rewards(got, want, what=""):
    assert_close(got, want, rtol=RTOL_REWARD, atol=ATOL_REWARD, what=what)
