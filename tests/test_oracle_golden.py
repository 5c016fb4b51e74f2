"""Pin the CPU oracle to the reference: golden vectors recorded from the
unmodified reference (tests/golden/make_golden.py) and Philox known-answer
tests.  Runs without a GPU."""

import numpy as np
import pytest

from helpers import config, golden, load_maps, ranges
from oracle import oracle as O
from oracle.philox_shim import PhiloxStream, blocks, philox4x32_10, random_actions

# Oracle vs reference: identical op order in IEEE double; only numpy's SIMD
# atan2 differs from glibc in the last ulp (reward, obs[2]).
OBS_ATOL = 2.4e-7   # 2 float32 ulps at |x| <= 1
REW_ATOL = 1e-12


def test_philox_known_answers():
    """Random123 philox4x32-10 KAT vectors."""
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in kat:
        got = philox4x32_10(np.array([ctr], dtype=np.uint32), *key)[0]
        assert tuple(int(v) for v in got) == want


def test_numpy_stream_matches_c_oracle():
    import ctypes
    lib = O.load_lib()
    for kind, lo, hi in ((0, -3.0, 7.5), (1, 0, 1_000_003), (1, 5, 6)):
        out = np.empty(64)
        lib.or_stream_draw(ctypes.c_uint64(12345), 9, 0, ctypes.c_uint64(77), kind,
                           ctypes.c_double(lo), ctypes.c_double(hi), 64,
                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        s = PhiloxStream(12345, 9, 0, 77)
        ref = s.uniform(lo, hi, 64) if kind == 0 else s.integers(int(lo), int(hi), 64)
        assert np.array_equal(out, np.asarray(ref, dtype=np.float64))
    z = PhiloxStream(1, 2).normal(0.0, 1.0, 40000)
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1.0) < 0.02


def test_integer_draws_are_unbiased_mulhi():
    b = blocks(5, 0, 2, np.arange(200000, dtype=np.uint64))
    from oracle.philox_shim import mulhi_range
    idx = mulhi_range(b, 1000)
    assert idx.min() >= 0 and idx.max() < 1000
    counts = np.bincount(idx, minlength=1000)
    from scipy import stats
    assert stats.chisquare(counts).pvalue > 0.001


def _replay(name, maps, rg, n):
    z = golden(name)
    seed = int(z["seed"])
    env = O.OracleVecEnv(maps, n, rg, config(32))
    s0 = env.reset_all(seed)
    np.testing.assert_allclose(s0, z["reset_states"], rtol=0, atol=OBS_ATOL)
    k = 0
    for t in range(z["rewards"].shape[0]):
        b = env.step_batch(random_actions(seed, np.arange(n), t))
        assert np.array_equal(b.events, z["events"][t]), t
        assert np.array_equal(b.dones, z["dones"][t])
        assert np.array_equal(b.truncated, z["truncated"][t])
        np.testing.assert_allclose(b.rewards, z["rewards"][t], rtol=0, atol=REW_ATOL)
        if k < len(z["obs_steps"]) and z["obs_steps"][k] == t:
            np.testing.assert_allclose(b.store_states, z["store_states"][k], rtol=0, atol=OBS_ATOL)
            np.testing.assert_allclose(b.states, z["states"][k], rtol=0, atol=OBS_ATOL)
            k += 1
    p = env.pose()
    assert np.array_equal(p["x"], z["final_x"]) and np.array_equal(p["y"], z["final_y"])
    assert np.array_equal(p["heading"], z["final_heading"])
    assert np.array_equal(p["rng_ctr"], z["rng_ctr"])
    st = env.stats()
    assert np.array_equal(st["episodes"], z["episodes"])
    assert np.array_equal(st["arrivals"], z["arrivals"])
    np.testing.assert_allclose(st["return_sum"], z["return_sum"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(st["recent_returns"], z["recent_returns"], rtol=0, atol=1e-9)


def test_oracle_cfg1_golden():
    _replay("traj_cfg1.npz", load_maps(1), ranges(0.0), 16)


def test_oracle_cfg2_golden():
    _replay("traj_cfg2.npz", load_maps(16), ranges(0.3), 256)


@pytest.mark.parametrize("max_range", [150.0, 300.0, 500.0])
def test_oracle_cast_rays_golden(max_range):
    maps = load_maps(16)
    z = golden("rays16.npz")
    occ = np.stack([m.occupancy for m in maps]).astype(np.uint8)
    edt = np.stack([O.edt_cells(m.occupancy) for m in maps])
    ang = z["qh"][:, None] + config(32).lidar.beam_offsets()[None, :]
    got = O.cast_rays(occ, edt, np.repeat(z["qmap"], 32), np.repeat(z["qx"], 32),
                      np.repeat(z["qy"], 32), np.cos(ang).ravel(), np.sin(ang).ravel(), 1.0,
                      max_range)
    assert np.array_equal(got, z[f"out_{int(max_range)}"])
    disc = O.disc_collides(occ, z["qmap"], z["qx"], z["qy"], np.full(len(z["qx"]), 9.0), 1.0)
    assert np.array_equal(disc, z["disc"])


def test_replay_oracle_golden():
    z = golden("replay.npz")
    buf = O.ReplayOracle(1000, 4)
    for start in range(0, 1500, 100):
        base = np.arange(start, start + 100, dtype=np.float32)
        buf.append_batch(np.tile(base[:, None], (1, 4)), base.astype(np.int64) % 5, base * 0.5,
                         np.tile(base[:, None], (1, 4)) + 0.25, base.astype(np.int64) % 7 == 0)
    g = PhiloxStream(int(z["seed"]), int(z["stream"]), tag=2)
    for i in range(4):
        (s, a, r, s2, d), _ = buf.sample(256, g)
        assert np.array_equal(s, z["states"][i]) and np.array_equal(a, z["actions"][i])
        assert np.array_equal(r, z["rewards"][i]) and np.array_equal(d, z["dones"][i])


def test_golden_maps_are_mapgen_defaults():
    z = golden("maps16.npz")
    assert z["sha256"][0].startswith("2b362396f4c5")  # map00
    maps = load_maps(16)
    assert all(m.occupancy.shape == (366, 366) for m in maps)
    occ = np.mean([m.occupancy.mean() for m in maps])
    assert 0.08 < occ < 0.12
