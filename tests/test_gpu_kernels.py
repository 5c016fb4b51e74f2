"""The per-op plugin seam (kernels.cast_rays / disc_collides on the GPU),
ported from the reference's tests/test_kernels.py, plus injection of the
CUDA backend into the UNMODIFIED reference simulator."""

import numpy as np
import pytest
from scipy import ndimage

from helpers import config, load_maps, make_map

pytestmark = pytest.mark.gpu


def edt_of(occ):
    return ndimage.distance_transform_edt(~occ).astype(np.float64)


def cast(occ, x, y, angles, max_range=100.0):
    from paper_2305_04180_b200 import kernels
    n = len(angles)
    return kernels.cast_rays(occ[None].astype(np.uint8), edt_of(occ)[None], np.zeros(n, np.int64),
                             np.full(n, x), np.full(n, y), np.cos(angles), np.sin(angles), 1.0,
                             max_range)


def bordered(n):
    occ = np.zeros((n, n), dtype=bool)
    occ[0, :] = occ[-1, :] = occ[:, 0] = occ[:, -1] = True
    return occ


def random_scene(rng, n_cells=60, n_blocks=8):  # tests/util.py:99-116
    occ = bordered(n_cells)
    for _ in range(n_blocks):
        w, h = rng.integers(2, max(3, n_cells // 5), 2)
        ix = int(rng.integers(1, n_cells - 1 - w))
        iy = int(rng.integers(1, n_cells - 1 - h))
        occ[iy:iy + h, ix:ix + w] = True

    def sample():
        while True:
            x, y = rng.uniform(1.0, n_cells - 1.0), rng.uniform(1.0, n_cells - 1.0)
            if not occ[int(np.floor(y)), int(np.floor(x))]:
                return x, y
    return occ, sample


def test_empty_map_reports_max_range():  # test_kernels.py:23-28
    out = cast(bordered(50), 25.3, 24.7, np.linspace(-np.pi, np.pi, 13), max_range=10.0)
    assert np.all(out == 10.0)


def test_perpendicular_wall_distance_is_exact():  # test_kernels.py:31-36
    occ = bordered(40)
    occ[:, 30] = True
    assert cast(occ, 10.0, 20.5, np.array([0.0]))[0] == pytest.approx(20.0, abs=1e-12)


def test_origin_inside_obstacle_and_outside_grid():  # test_kernels.py:39-44
    occ = bordered(10)
    occ[5, 5] = True
    assert cast(occ, 5.5, 5.5, np.zeros(1))[0] == 0.0
    assert cast(occ, -3.0, 5.0, np.zeros(1))[0] == 0.0


def test_axis_aligned_rays_do_not_hang():  # test_kernels.py:70-76
    out = cast(bordered(30), 15.5, 15.5, np.array([0.0, np.pi / 2, np.pi, -np.pi / 2]), 200.0)
    assert np.all(np.isfinite(out)) and np.all(out <= 15.5)


def test_bit_identical_to_oracle_on_random_scenes():  # test_kernels.py:79-110
    from oracle import oracle as O
    from paper_2305_04180_b200 import kernels
    rng = np.random.default_rng(5)
    for _ in range(10):
        occ, sample = random_scene(rng)
        x, y = sample()
        angles = rng.uniform(-np.pi, np.pi, 27)
        a = cast(occ, x, y, angles)
        occ8, edt = occ[None].astype(np.uint8), edt_of(occ)[None]
        b = O.cast_rays(occ8, edt, np.zeros(27, np.int64), np.full(27, x), np.full(27, y),
                        np.cos(angles), np.sin(angles), 1.0, 100.0)
        assert np.array_equal(a, b)
        single = np.concatenate([cast(occ, x, y, angles[i:i + 1]) for i in range(0, 27, 5)])
        assert np.array_equal(a[::5], single)
        px = np.array([sample()[0] for _ in range(16)])
        py = np.array([sample()[1] for _ in range(16)])
        r = rng.uniform(0.5, 4.0, 16)
        mi = np.zeros(16, np.int64)
        assert np.array_equal(kernels.disc_collides(occ8, mi, px, py, r, 1.0),
                              O.disc_collides(occ8, mi, px, py, r, 1.0))


def test_unbordered_grids_match_the_reference_jump_semantics():
    """Grids without an occupied border: the reference's EDT jump can land
    outside the grid and reports the landing distance; the seam reproduces it."""
    from oracle import oracle as O
    rng = np.random.default_rng(8)
    for _ in range(20):
        h, w = rng.integers(8, 50, 2)
        occ = rng.random((h, w)) < 0.05
        n = 300
        px, py = rng.uniform(-2, w + 2, n), rng.uniform(-2, h + 2, n)
        ang = rng.uniform(-np.pi, np.pi, n)
        occ8, edt = occ[None].astype(np.uint8), edt_of(occ)[None]
        from paper_2305_04180_b200 import kernels
        for mr in (5.0, 40.0, 500.0):
            a = kernels.cast_rays(occ8, edt, np.zeros(n, np.int64), px, py, np.cos(ang),
                                  np.sin(ang), 1.0, mr)
            b = O.cast_rays(occ8, edt, np.zeros(n, np.int64), px, py, np.cos(ang), np.sin(ang),
                            1.0, mr)
            assert np.array_equal(a, b)


def test_disc_collides_against_cell_oracle():  # test_kernels.py:113-124
    from paper_2305_04180_b200 import kernels
    rng = np.random.default_rng(21)
    occ, _ = random_scene(rng, n_cells=30, n_blocks=5)
    xs, ys, rs = rng.uniform(-2, 32, 200), rng.uniform(-2, 32, 200), rng.uniform(0.3, 5.0, 200)
    got = kernels.disc_collides(occ[None].astype(np.uint8), np.zeros(200, np.int64), xs, ys, rs,
                                1.0)
    for k in range(200):
        x, y, r = xs[k], ys[k], rs[k]
        want = x - r < 0 or y - r < 0 or x + r > 30 or y + r > 30
        if not want:
            iy, ix = np.nonzero(occ)
            nx = np.minimum(np.maximum(x, ix), ix + 1.0)
            ny = np.minimum(np.maximum(y, iy), iy + 1.0)
            want = bool(((x - nx) ** 2 + (y - ny) ** 2 <= r * r).any())
        assert bool(got[k]) == want


def test_cuda_backend_drives_the_unmodified_reference():
    """SURVEY 8(b) seam: sim._kernel = our module; the reference's own step
    then matches its stock Cython run bit for bit."""
    from oracle import oracle as O
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    O.import_reference(37)
    import color_rl.vecenv as vmod
    from color_rl.sim.gridmap import GridMap as RG
    from color_rl.sim.params import DiversityRanges, EnvConfig, LidarConfig, SimParams
    from oracle.philox_shim import random_actions, reference_rng_proxy
    from paper_2305_04180_b200 import kernels
    maps = [RG.from_text(m.to_text()) for m in load_maps(4)]
    cfg = EnvConfig(lidar=LidarConfig(n_beams=32))
    rg = DiversityRanges.around(SimParams(), 0.3)
    stock = vmod.VecEnv(maps, 32, rg, cfg)
    ours = vmod.VecEnv(maps, 32, rg, cfg)
    ours.sim._kernel = kernels
    with reference_rng_proxy(vmod):
        a0 = stock.reset_all(5)
        b0 = ours.reset_all(5)
    assert np.array_equal(a0, b0)
    for t in range(30):
        acts = random_actions(5, np.arange(32), t)
        x, y = stock.step_batch(acts), ours.step_batch(acts)
        assert np.array_equal(x.states, y.states) and np.array_equal(x.rewards, y.rewards)


def _slab_entry(occ, x, y, ang, max_range):
    """Exact geometry, independent of any DDA: the smallest entry parameter of
    the ray into an occupied cell rectangle (slab test over every occupied
    cell), capped at max_range; plus that crossing's chord length."""
    dx, dy = np.cos(ang), np.sin(ang)
    iy, ix = np.nonzero(occ)
    with np.errstate(divide="ignore", invalid="ignore"):
        tx0, tx1 = (ix - x) / dx, (ix + 1 - x) / dx
        ty0, ty1 = (iy - y) / dy, (iy + 1 - y) / dy
    if dx == 0.0:
        inside = (ix <= x) & (x < ix + 1)
        tx0 = np.where(inside, -np.inf, np.inf)
        tx1 = np.where(inside, np.inf, -np.inf)
    if dy == 0.0:
        inside = (iy <= y) & (y < iy + 1)
        ty0 = np.where(inside, -np.inf, np.inf)
        ty1 = np.where(inside, np.inf, -np.inf)
    t_in = np.maximum(np.minimum(tx0, tx1), np.minimum(ty0, ty1))
    t_out = np.minimum(np.maximum(tx0, tx1), np.maximum(ty0, ty1))
    ok = (t_out >= np.maximum(t_in, 0.0))
    if not ok.any():
        return max_range, 0.0
    k = np.argmin(np.where(ok, np.maximum(t_in, 0.0), np.inf))
    t = max(t_in[k], 0.0)
    return (min(t, max_range), t_out[k] - t) if t < max_range else (max_range, 0.0)


def test_matches_exact_slab_geometry():  # test_kernels.py:47-67 (exact oracle instead of a fine march)
    """Every range equals the exact first entry into an occupied cell, except
    tangential grazes (chord ~0) where the DDA's face order decides."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        occ, sample = random_scene(rng)
        x, y = sample()
        angles = rng.uniform(-np.pi, np.pi) + np.linspace(-2.3, 2.3, 27)
        got = cast(occ, x, y, angles, max_range=45.0)
        for a, g in zip(angles, got):
            t, chord = _slab_entry(occ, x, y, a, 45.0)
            if abs(g - t) > 1e-9:
                assert chord < 1e-9 and g > t, (x, y, a, g, t, chord)


def test_batched_equals_per_ray():  # test_kernels.py:102-110
    rng = np.random.default_rng(9)
    occ, sample = random_scene(rng)
    x, y = sample()
    angles = rng.uniform(-np.pi, np.pi, 27)
    batched = cast(occ, x, y, angles)
    single = np.concatenate([cast(occ, x, y, angles[i:i + 1]) for i in range(27)])
    assert np.array_equal(batched, single)
