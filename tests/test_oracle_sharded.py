"""CPU: the sharded oracle (the checker of the BASELINE-size GPU parity runs)
is the single-process oracle, and its recorded hit cells are cast_rays'."""

import numpy as np

from helpers import config, load_maps, ranges
from oracle.oracle import OracleVecEnv, ShardedOracle, cast_rays, edt_cells
from oracle.philox_shim import random_actions


def test_sharded_oracle_equals_single_process():
    maps = load_maps(4)
    n, seed = 203, 11
    one = OracleVecEnv(maps, n, ranges(0.3), config(32, timeout_steps=9))
    many = ShardedOracle(maps, n, ranges(0.3), config(32, timeout_steps=9), shards=5)
    try:
        assert np.array_equal(one.reset_all(seed), many.reset_all(seed))
        for t in range(14):
            a = random_actions(seed, np.arange(n), t)
            x, y = one.step_batch(a), many.step_batch(a)
            for f in range(6):
                assert np.array_equal(x[f], y[f]), (t, f)
            cx, cy = one.cells(), many.cells()
            for k in cx:
                assert np.array_equal(cx[k], cy[k]), (t, k)
        for k, v in one.pose().items():
            assert np.array_equal(v, many.pose()[k]), k
    finally:
        many.close()


def test_recorded_cells_are_cast_rays_cells():
    """The states-row hit cells equal cast_rays' at the current poses (no
    auto-reset happened for lanes that are still running)."""
    maps = load_maps(2)
    n, seed, R = 32, 3, 32
    cfg = config(R)
    env = OracleVecEnv(maps, n, ranges(0.0), cfg)
    env.reset_all(seed)
    for t in range(5):
        env.step_batch(random_actions(seed, np.arange(n), t))
    p = env.pose()
    occ = np.stack([m.occupancy for m in maps]).astype(np.uint8)
    edt = np.stack([edt_cells(m.occupancy) for m in maps])
    ang = p["heading"][:, None] + cfg.lidar.beam_offsets()[None, :]
    midx = np.repeat(np.arange(n) % 2, R)
    _, cells = cast_rays(occ, edt, midx, np.repeat(p["x"], R), np.repeat(p["y"], R),
                         np.cos(ang).ravel(), np.sin(ang).ravel(), 1.0,
                         cfg.lidar.max_range_cm, return_cells=True)
    assert np.array_equal(env.cells()["state"].ravel(), cells)
