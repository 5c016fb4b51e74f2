"""GPU parity: the fused CUDA step vs the reference (golden fixtures recorded
from the unmodified reference) and vs the C oracle, on identical seeds.

Bar (BASELINE north star): events/dones/truncated, RNG draw counts and
episode counters bit-exact; poses, obs (incl. LiDAR ranges) and rewards
within 1e-5 relative (+ fp32-resolution absolute floor, see helpers.py).
"""

import numpy as np
import pytest

from helpers import assert_close, assert_obs, assert_rewards, config, golden, load_maps, make_map, ranges
from oracle.philox_shim import random_actions

pytestmark = pytest.mark.gpu


def _vec(maps, n, rg, cfg, **kw):
    from paper_2305_04180_b200 import VecEnv
    return VecEnv(maps, n, rg, cfg, **kw)


def _replay_golden(name, maps, rg, n):
    z = golden(name)
    seed = int(z["seed"])
    env = _vec(maps, n, rg, config(32))
    s0 = env.reset_all(seed).cpu().numpy()
    assert_obs(s0, z["reset_states"], what="reset states")
    steps = z["rewards"].shape[0]
    obs_steps = list(z["obs_steps"])
    k = 0
    for t in range(steps):
        b = env.step_batch(random_actions(seed, np.arange(n), t))
        ev = b.events.cpu().numpy()
        assert np.array_equal(ev, z["events"][t]), f"events differ at step {t}"
        assert np.array_equal(b.dones.cpu().numpy(), z["dones"][t]), t
        assert np.array_equal(b.truncated.cpu().numpy(), z["truncated"][t]), t
        assert_rewards(b.rewards.cpu().numpy(), z["rewards"][t], what=f"rewards step {t}")
        if k < len(obs_steps) and obs_steps[k] == t:
            assert_obs(b.store_states.cpu().numpy(), z["store_states"][k], what=f"store_states step {t}")
            assert_obs(b.states.cpu().numpy(), z["states"][k], what=f"states step {t}")
            k += 1
    sim = env.sim
    assert_close(sim.x, z["final_x"], what="x")
    assert_close(sim.y, z["final_y"], what="y")
    assert np.array_equal(sim.rng_ctr.astype(np.uint64), z["rng_ctr"]), "draw counts differ"
    snap = env.snapshot_stats()
    assert [c.episodes for c in snap.per_copy] == z["episodes"].tolist()
    assert [c.arrivals for c in snap.per_copy] == z["arrivals"].tolist()
    assert_close([c.return_sum for c in snap.per_copy], z["return_sum"], atol=1e-9,
                 what="return_sum")
    assert_close(snap.recent_returns, z["recent_returns"], atol=1e-9, what="recent returns")


def test_cfg1_golden_1000_steps():
    """cfg1: 16 envs, default map, 32 beams, 1000 random-action steps."""
    _replay_golden("traj_cfg1.npz", load_maps(1), ranges(0.0), 16)


def test_cfg2_golden_slice():
    """cfg2 slice: 256 envs over 16 maps with +/-30 % diversity, 100 steps."""
    _replay_golden("traj_cfg2.npz", load_maps(16), ranges(0.3), 256)


@pytest.mark.parametrize("n,steps,div", [(4096, 60, 0.3), (1000, 40, 0.0)])
def test_vs_oracle(n, steps, div):
    from oracle.oracle import OracleVecEnv
    maps = load_maps(16)
    cfg = config(32)
    seed = 4242
    gpu = _vec(maps, n, ranges(div), cfg)
    cpu = OracleVecEnv(maps, n, ranges(div), cfg)
    assert_obs(gpu.reset_all(seed).cpu().numpy(), cpu.reset_all(seed), what="reset")
    for t in range(steps):
        a = random_actions(seed, np.arange(n), t)
        g = gpu.step_batch(a)
        c = cpu.step_batch(a)
        assert np.array_equal(g.events.cpu().numpy(), c.events), f"events step {t}"
        assert np.array_equal(g.dones.cpu().numpy(), c.dones)
        assert_rewards(g.rewards.cpu().numpy(), c.rewards, what=f"reward {t}")
        assert_obs(g.store_states.cpu().numpy(), c.store_states, what=f"store {t}")
        assert_obs(g.states.cpu().numpy(), c.states, what=f"states {t}")
    p = cpu.pose()
    assert_close(gpu.sim.x, p["x"], what="x")
    assert_close(gpu.sim.heading, p["heading"], atol=1e-12, what="heading")
    assert np.array_equal(gpu.sim.rng_ctr.astype(np.uint64), p["rng_ctr"])


@pytest.mark.parametrize("max_range", [150.0, 300.0, 500.0])
def test_op_level_cast_rays_bit_identical(max_range):
    """The plugin seam (kernels.cast_rays) reproduces the Cython backend
    bit for bit (golden recorded from _cy.pyx)."""
    from paper_2305_04180_b200 import kernels
    from oracle.oracle import edt_cells
    maps = load_maps(16)
    z = golden("rays16.npz")
    occ = np.stack([m.occupancy for m in maps]).astype(np.uint8)
    edt = np.stack([edt_cells(m.occupancy) for m in maps])
    ang = z["qh"][:, None] + config(32).lidar.beam_offsets()[None, :]
    px, py = np.repeat(z["qx"], 32), np.repeat(z["qy"], 32)
    got = kernels.cast_rays(occ, edt, np.repeat(z["qmap"], 32), px, py, np.cos(ang).ravel(),
                            np.sin(ang).ravel(), 1.0, max_range)
    assert np.array_equal(got, z[f"out_{int(max_range)}"])
    disc = kernels.disc_collides(occ, z["qmap"], z["qx"], z["qy"], np.full(len(z["qx"]), 9.0),
                                 1.0)
    assert np.array_equal(disc, z["disc"])


@pytest.mark.parametrize("n_beams", [32, 128, 256])
@pytest.mark.parametrize("max_range", [150.0, 300.0, 500.0])
def test_fast_marcher_hit_cells(n_beams, max_range):
    """cfg4: the fused step's SMEM marcher stops in the reference's cell
    (bit-exact hit cell) with the reference's range (1e-5 relative)."""
    from oracle import oracle as O
    maps = load_maps(16)
    cfg = config(n_beams, lidar_kw={"max_range_cm": max_range})
    env = _vec(maps, 16, ranges(0.0), cfg)
    rng = np.random.default_rng(n_beams + int(max_range))
    qx, qy, qh, qm = [], [], [], []
    for m, gm in enumerate(maps):
        free = np.argwhere(~gm.occupancy)
        for iy, ix in free[rng.integers(0, len(free), 24)]:
            qx.append(ix + rng.random()); qy.append(iy + rng.random())
            qh.append(rng.uniform(-np.pi, np.pi)); qm.append(m)
    qx, qy, qh, qm = map(np.array, (qx, qy, qh, qm))
    got, cells = env.scan(qx, qy, qh, qm, return_cells=True)
    got, cells = got.cpu().numpy(), cells.cpu().numpy()
    occ = np.stack([m.occupancy for m in maps]).astype(np.uint8)
    edt = np.stack([O.edt_cells(m.occupancy) for m in maps])
    ang = qh[:, None] + cfg.lidar.beam_offsets()[None, :]
    want, wcells = O.cast_rays(occ, edt, np.repeat(qm, n_beams), np.repeat(qx, n_beams),
                               np.repeat(qy, n_beams), np.cos(ang).ravel(), np.sin(ang).ravel(),
                               1.0, max_range, return_cells=True)
    want = want.reshape(-1, n_beams)
    wcells = wcells.reshape(-1, n_beams)
    # hit cell: the reference reports the stopping occupied cell; both sides -1 otherwise
    mism = cells != wcells
    assert mism.sum() == 0, f"{mism.sum()} hit cells differ of {mism.size}"
    assert_close(got, want, rtol=1e-9, atol=1e-9, what="ranges")


def test_unbordered_maps_are_rejected():
    """A map whose border is not fully occupied (GridMap validates this,
    gridmap.py:90-95; here the border is cleared after construction, as a raw
    map could arrive) raises MapError: the marcher has no grid-exit tests.
    The op-level seam (sp_cast_rays) takes any grid, test_gpu_kernels.py."""
    import copy
    from paper_2305_04180_b200.sim import MapError
    maps = [copy.deepcopy(m) for m in load_maps(2)]
    maps[1].occupancy[0, 5] = False
    with pytest.raises(MapError):
        _vec(maps, 4, ranges(0.0), config(32))


def _vs_oracle_run(maps, n, div, steps, seed, n_beams=32):
    from oracle.oracle import OracleVecEnv
    cfg = config(n_beams)
    gpu = _vec(maps, n, ranges(div), cfg)
    cpu = OracleVecEnv(maps, n, ranges(div), cfg)
    assert_obs(gpu.reset_all(seed).cpu().numpy(), cpu.reset_all(seed), what="reset")
    for t in range(steps):
        a = random_actions(seed, np.arange(n), t)
        g = gpu.step_batch(a)
        c = cpu.step_batch(a)
        assert np.array_equal(g.events.cpu().numpy(), c.events), f"events step {t}"
        assert_rewards(g.rewards.cpu().numpy(), c.rewards, what=f"reward {t}")
        assert_obs(g.states.cpu().numpy(), c.states, what=f"states {t}")
        assert_obs(g.store_states.cpu().numpy(), c.store_states, what=f"store {t}")
    return gpu


def test_maps_too_large_for_shared_memory():
    """1100 x 1100-cell maps: the block table (302 KB) does not fit in shared
    memory, so the kernel reads the tables through L1/L2 (kSmem = false)."""
    from paper_2305_04180_b200.mapgen import generate_maps
    maps = generate_maps(2, seed=3, size_cm=1100, density=0.05)
    _vs_oracle_run(maps, 96, 0.3, 12, seed=77)  # 302 KB table > 227 KB: the HBM path


def test_more_maps_than_ctas():
    """200 small maps > 148 CTAs: CTAs span several maps and rebind their
    shared-memory tables between chunks."""
    rng = np.random.default_rng(5)
    maps = []
    for _ in range(200):  # blocks in the upper band, clear of the spawn square (18..27)
        xs, ys = rng.integers(4, 34, 3), rng.integers(38, 52, 3)  # goal disc at (42, 42)
        maps.append(make_map(60, blocks=[(int(x), int(y), int(x) + 4, int(y) + 3)
                                         for x, y in zip(xs, ys)]))
    _vs_oracle_run(maps, 600, 0.3, 15, seed=91)


def test_vs_oracle_256_beams():
    """R = 256 (D = 261): the widest cfg4 scan, 64 noise blocks per scan and
    the smallest chunk capacity, stepped against the C oracle."""
    _vs_oracle_run(load_maps(4), 300, 0.3, 10, seed=13, n_beams=256)
