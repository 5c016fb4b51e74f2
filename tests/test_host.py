"""Host-side logic of the drop-in (no GPU): map text format, parameter
ranges, beam offsets, sharding.  Mirrors the reference's test_gridmap.py /
params checks and is cross-checked against the reference where built."""

import math

import numpy as np
import pytest

from helpers import load_maps, make_map
from oracle import oracle as O
from paper_2305_04180_b200 import dist
from paper_2305_04180_b200.sim import (
    DiversityRanges,
    EnvConfig,
    GridMap,
    LidarConfig,
    MapError,
    SimParams,
)

MAP_TEXT = """\
8 8 1
########
#....GG#
#....GG#
#......#
#......#
#SS....#
#SS....#
########
"""


def test_from_text_goal_and_spawn():
    m = GridMap.from_text(MAP_TEXT)
    assert (m.width_cm, m.height_cm, m.cell_size_cm) == (8, 8, 1)
    assert m.goal_center == (6.0, 6.0)
    assert m.goal_radius_cm == pytest.approx(math.hypot(0.5, 0.5) + 0.5)
    assert m.spawn_region == (1.0, 1.0, 3.0, 3.0)
    assert m.occupancy[0].all() and not m.occupancy[3, 3]


def test_text_round_trip_and_row_order():
    m = GridMap.from_text(MAP_TEXT)
    m2 = GridMap.from_text(m.to_text())
    assert np.array_equal(m.occupancy, m2.occupancy)
    assert m2.goal_center == m.goal_center and m2.spawn_region == m.spawn_region
    t = GridMap.from_text("4 4 1\n####\n#.G#\n#S.#\n####\n")
    assert t.spawn_region == (1.0, 1.0, 2.0, 2.0) and t.goal_center == (2.5, 2.5)
    c = GridMap.from_text("20 20 5\n####\n#.G#\n#S.#\n####\n")
    assert c.goal_center == (12.5, 12.5) and c.spawn_region == (5.0, 5.0, 10.0, 10.0)


@pytest.mark.parametrize("bad", [
    "not a header\n", "8 8 3\n", MAP_TEXT.replace("G", "."), MAP_TEXT.replace("S", "."),
    MAP_TEXT.replace(".", "?", 1), "\n".join(MAP_TEXT.splitlines()[:-1]) + "\n"])
def test_rejects_malformed_text(bad):
    with pytest.raises(MapError):
        GridMap.from_text(bad)


def test_constructor_invariants():
    occ = np.zeros((10, 10), dtype=bool)
    occ[0, :] = occ[-1, :] = occ[:, 0] = occ[:, -1] = True
    with pytest.raises(MapError):
        GridMap(10, 10, 3, occ, (5, 5), 1.0, (1, 1, 3, 3))
    bad = occ.copy()
    bad[0, 4] = False
    with pytest.raises(MapError):
        GridMap(10, 10, 1, bad, (5, 5), 1.0, (1, 1, 3, 3))
    with pytest.raises(MapError):
        GridMap(10, 10, 1, occ, (15, 5), 1.0, (1, 1, 3, 3))
    with pytest.raises(MapError):
        GridMap(10, 10, 1, occ, (0.5, 0.5), 1.0, (1, 1, 3, 3))
    with pytest.raises(MapError):
        GridMap(10, 10, 1, occ, (5, 5), 1.0, (1, 1, 30, 3))


@pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")
def test_gridmap_and_params_equal_reference():
    O.import_reference()
    from color_rl.sim.gridmap import GridMap as RG
    from color_rl.sim.params import DiversityRanges as RD, LidarConfig as RL, SimParams as RS
    for m in load_maps(16):
        t = m.to_text()
        a, b = RG.from_text(t), GridMap.from_text(t)
        assert a.to_text() == b.to_text()
        assert (a.goal_center, a.goal_radius_cm, a.spawn_region) == \
               (b.goal_center, b.goal_radius_cm, b.spawn_region)
    for frac in (0.0, 0.1, 0.3, 0.5):
        for d in (0, 1, 3, 40):
            nom = SimParams(control_delay_steps=d)
            rnom = RS(control_delay_steps=d)
            assert DiversityRanges.around(nom, frac).__dict__ == RD.around(rnom, frac).__dict__
    for n in (1, 27, 32, 128, 256):
        assert np.array_equal(LidarConfig(n_beams=n).beam_offsets(), RL(n_beams=n).beam_offsets())


def test_params_validation():
    with pytest.raises(ValueError):
        SimParams(k=1.0)
    with pytest.raises(ValueError):
        SimParams(control_delay_steps=65)
    with pytest.raises(ValueError):
        DiversityRanges(k=(0.7, 0.6))
    with pytest.raises(ValueError):
        DiversityRanges.around(SimParams(), -0.1)
    r = DiversityRanges.around(SimParams(), 0.3)
    assert r.control_delay_steps == (0, 2)


def test_config_planning_distance():
    m = make_map(40)
    assert EnvConfig().planning_dist(m) == pytest.approx(math.hypot(40, 40))
    assert EnvConfig(max_planning_dist_cm=100.0).planning_dist(m) == 100.0
    assert LidarConfig(n_beams=32).state_dim == 37


def test_shard_partitions_global_ids():
    for total, world in ((65536 * 8, 8), (1000, 3), (5, 8)):
        parts = [dist.shard(total, r, world) for r in range(world)]
        ids = [i for off, n in parts for i in range(off, off + n)]
        assert ids == list(range(total))
    with pytest.raises(ValueError):
        dist.shard(10, 3, 3)


def test_eval_report_matches_reference_formatting():
    """EvalReport/MapEval/summarize_rates host logic (evaluate.py:22-133):
    same dicts and rendered table as the reference for the same counts."""
    from oracle import oracle as O
    from paper_2305_04180_b200 import evaluate as E
    rows = [("a", 10, 7, 2, 1, 3.25, 41.5), ("bb", 4, 0, 4, 0, -10.0, 12.0)]
    got = E.EvalReport(seed=3, results=[E.MapEval(*r) for r in rows])
    assert got.episodes == 14 and got.arrival_rate == 0.5
    assert got.to_dict()["maps"][1]["arrival_rate"] == 0.0
    assert E.summarize_rates([]) == {"per_seed": [], "mean": 0.0, "std": 0.0}
    if not O.reference_available():
        return
    O.import_reference()
    from color_rl import evaluate as R
    want = R.EvalReport(seed=3, results=[R.MapEval(*r) for r in rows])
    assert got.to_dict() == want.to_dict()
    assert got.render() == want.render()
    assert E.summarize_rates([got, got]) == R.summarize_rates([want, want])


def test_mapgen_reproduces_golden_maps():
    """mapgen restatement: seed 0 regenerates the reference-made golden maps
    cell for cell (tests/golden/maps16.npz came from the reference's
    generate_maps(16, seed=0))."""
    import hashlib
    from helpers import golden
    from paper_2305_04180_b200.mapgen import generate_maps
    from paper_2305_04180_b200.sim import GridMap as G
    want = load_maps(4)  # stored after the reference's text round trip
    sha = golden("maps16.npz")["sha256"]  # of the reference's original map text
    got = generate_maps(4, seed=0)
    for g, w, h in zip(got, want, sha):
        assert np.array_equal(g.occupancy, w.occupancy)
        assert hashlib.sha256(g.to_text().encode()).hexdigest() == str(h)
        rt = G.from_text(g.to_text())
        assert rt.goal_center == w.goal_center and rt.goal_radius_cm == w.goal_radius_cm
        assert rt.spawn_region == w.spawn_region


def test_mapgen_matches_reference_small(tmp_path):
    """Small arenas, other seeds and densities: same maps as the reference's
    generate_maps; write_maps names and round-trips; errors as the reference."""
    from oracle import oracle as O
    from paper_2305_04180_b200.mapgen import MapGenError, generate_map, generate_maps, write_maps
    from paper_2305_04180_b200.sim import GridMap as G
    maps = generate_maps(3, seed=5, size_cm=120)
    paths = write_maps(maps, tmp_path)
    assert [p.name for p in paths] == ["map00.txt", "map01.txt", "map02.txt"]
    for p, m in zip(paths, maps):
        assert np.array_equal(G.load(p).occupancy, m.occupancy)
    with pytest.raises(ValueError):
        generate_map(np.random.default_rng(0), density=1.0)
    with pytest.raises(ValueError):
        generate_map(np.random.default_rng(0), size_cm=6)
    with pytest.raises(MapGenError):
        generate_map(np.random.default_rng(0), size_cm=120, robot_radius_cm=60.0, layout_attempts=2)
    if not O.reference_available():
        return
    O.import_reference()
    from color_rl import mapgen as R
    for seed, size, dens in ((5, 120, 0.08), (7, 200, 0.15), (11, 366, 0.05)):
        a = generate_maps(2, seed=seed, size_cm=size, density=dens)
        b = R.generate_maps(2, seed=seed, size_cm=size, density=dens)
        for x, y in zip(a, b):
            assert x.to_text() == y.to_text()
    m = G.from_text(maps[0].to_text())
    ref_m = R.GridMap.from_text(maps[0].to_text())
    assert np.array_equal(m.edt_cells(), ref_m.edt_cells())
    assert m.to_ascii((30.0, 30.0)) == ref_m.to_ascii((30.0, 30.0))
    assert m.to_ascii() == ref_m.to_ascii()


@pytest.mark.parametrize("max_range", [150.0, 300.0, 500.0])
def test_ray_cell_count_equals_pure_dda(max_range):
    """raycells.dda_cells (the bench's ray-cells/s accounting: Manhattan
    distance origin cell -> stopping cell, + 1) equals the oracle's
    cell-by-cell pure DDA count (_cy.pyx:89-105 without the EDT jump)."""
    import torch
    from paper_2305_04180_b200.raycells import dda_cells
    maps = load_maps(16)
    occ = np.stack([m.occupancy for m in maps]).astype(np.uint8)
    edt = np.stack([O.edt_cells(m.occupancy) for m in maps])
    rng = np.random.default_rng(int(max_range))
    n, R = 400, 32
    qm = rng.integers(0, 16, n)
    qx, qy = rng.uniform(12, 354, n), rng.uniform(12, 354, n)
    qh = rng.uniform(-np.pi, np.pi, n)
    off = LidarConfig(n_beams=R).beam_offsets()
    ang = qh[:, None] + off[None, :]
    args = (np.repeat(qm, R), np.repeat(qx, R), np.repeat(qy, R), np.cos(ang).ravel(),
            np.sin(ang).ravel(), 1.0, max_range)
    _, hit = O.cast_rays(occ, edt, *args, return_cells=True)
    want = O.count_dda_cells(occ, *args).reshape(n, R)
    hit = hit.reshape(n, R)
    got = dda_cells(qx, qy, qh, off, hit, 366, 1.0, max_range)
    assert (got == want).mean() > 0.9999 and np.abs(got - want).max() <= 1
    got_t = dda_cells(torch.from_numpy(qx), torch.from_numpy(qy), torch.from_numpy(qh), off,
                      torch.from_numpy(hit), 366, 1.0, max_range)
    assert np.array_equal(got_t.numpy(), got)
