"""Pin the CPU oracle against the live, unmodified reference (oracle/_ref,
built by oracle/build_ref.sh from /root/reference) on fresh inputs.  Skipped
where the reference build is absent."""

import numpy as np
import pytest

from helpers import load_maps, make_map
from oracle import oracle as O
from oracle.philox_shim import PhiloxStream, random_actions, reference_rng_proxy

pytestmark = pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")


def _ref_env(maps_np, n, div, n_beams, timeout=1000, auto_reset=True):
    O.import_reference(5 + n_beams)
    from color_rl.sim.gridmap import GridMap as RG
    from color_rl.sim.params import DiversityRanges, EnvConfig, LidarConfig, SimParams
    from color_rl.vecenv import VecEnv
    maps = [RG.from_text(m.to_text()) for m in maps_np]
    rg = DiversityRanges.around(SimParams(), div) if div else DiversityRanges()
    cfg = EnvConfig(lidar=LidarConfig(n_beams=n_beams), timeout_steps=timeout)
    return VecEnv(maps, n, rg, cfg, auto_reset=auto_reset), maps, rg, cfg


@pytest.mark.parametrize("n,n_maps,div,n_beams,steps,timeout", [
    (8, 1, 0.0, 27, 150, 1000),     # reference defaults (STATE_DIM 32, unpatched)
    (64, 16, 0.3, 32, 80, 1000),    # cfg2-like
    (24, 4, 0.5, 128, 40, 30),      # many beams, short timeouts (truncation path)
])
def test_oracle_matches_reference(n, n_maps, div, n_beams, steps, timeout):
    ref, maps, rg, cfg = _ref_env(load_maps(n_maps), n, div, n_beams, timeout)
    import color_rl.vecenv as vmod
    seed = 99 + n
    with reference_rng_proxy(vmod):
        s_ref = ref.reset_all(seed)
    orc = O.OracleVecEnv(maps, n, rg, cfg)
    assert np.array_equal(orc.reset_all(seed), s_ref)
    for t in range(steps):
        a = random_actions(seed, np.arange(n), t)
        b, c = ref.step_batch(a), orc.step_batch(a)
        assert np.array_equal(b.events, c.events)
        assert np.array_equal(b.truncated, c.truncated)
        np.testing.assert_allclose(c.rewards, b.rewards, rtol=0, atol=1e-12)
        np.testing.assert_allclose(c.states, b.states, rtol=0, atol=2.4e-7)
        np.testing.assert_allclose(c.store_states, b.store_states, rtol=0, atol=2.4e-7)
    p = orc.pose()
    assert np.array_equal(p["x"], ref.sim.x) and np.array_equal(p["heading"], ref.sim.heading)


def test_episode_terminated_without_auto_reset():
    ref, maps, rg, cfg = _ref_env([make_map(40)], 2, 0.0, 27, timeout=2, auto_reset=False)
    orc = O.OracleVecEnv(maps, 2, rg, cfg, auto_reset=False)
    import color_rl.vecenv as vmod
    from color_rl.sim.core import EpisodeTerminated
    with reference_rng_proxy(vmod):
        ref.reset_all(6)
    orc.reset_all(6)
    for _ in range(2):
        ref.step_batch([2, 2])
        orc.step_batch([2, 2])
    with pytest.raises(EpisodeTerminated):
        ref.step_batch([2, 2])
    with pytest.raises(O.OracleVecEnv.EpisodeTerminated):
        orc.step_batch([2, 2])


def test_cast_rays_edge_cases_match_reference():
    """Unbordered grids, origins outside/in obstacles, axis-aligned and
    diagonal rays: the oracle's cast_rays equals the Cython backend exactly."""
    O.import_reference()
    from color_rl import kernels
    cy = kernels.get_backend("cy")
    rng = np.random.default_rng(3)
    for trial in range(30):
        h, w = rng.integers(8, 60, 2)
        occ = rng.random((h, w)) < rng.uniform(0.0, 0.3)
        if trial % 3 == 0:  # bordered
            occ[0, :] = occ[-1, :] = occ[:, 0] = occ[:, -1] = True
        occ8 = occ[None].astype(np.uint8)
        edt = O.edt_cells(occ)[None]
        n = 200
        px = rng.uniform(-2, w + 2, n)
        py = rng.uniform(-2, h + 2, n)
        px[:20] = np.floor(px[:20]) + 0.5
        ang = rng.uniform(-np.pi, np.pi, n)
        ang[:40] = rng.integers(0, 8, 40) * (np.pi / 4)
        dx, dy = np.cos(ang), np.sin(ang)
        mi = np.zeros(n, dtype=np.int64)
        for mr in (5.0, 40.0, 500.0):
            a = cy.cast_rays(occ8, edt, mi, px, py, dx, dy, 1.0, mr)
            b = O.cast_rays(occ8, edt, mi, px, py, dx, dy, 1.0, mr)
            assert np.array_equal(a, b), (trial, mr)
        r = rng.uniform(0.2, 6.0, n)
        assert np.array_equal(cy.disc_collides(occ8, mi, px, py, r, 1.0),
                              O.disc_collides(occ8, mi, px, py, r, 1.0))


def test_replay_sampling_matches_reference():
    O.import_reference()
    from color_rl.replay import ReplayBuffer
    ref = ReplayBuffer(capacity=300, state_dim=5)
    orc = O.ReplayOracle(300, 5)
    rng = np.random.default_rng(0)
    for _ in range(7):
        n = int(rng.integers(1, 120))
        s = rng.random((n, 5), dtype=np.float32)
        args = (s, rng.integers(0, 5, n), rng.random(n), s + 1, rng.random(n) < 0.2)
        ref.append_batch(*args)
        orc.append_batch(*args)
        g1, g2 = PhiloxStream(11, 4, tag=2), PhiloxStream(11, 4, tag=2)
        tb = ref.sample(64, g1)
        (s_, a_, r_, s2_, d_), _ = orc.sample(64, g2)
        assert np.array_equal(tb.states, s_) and np.array_equal(tb.actions, a_)
        assert np.array_equal(tb.rewards, r_) and np.array_equal(tb.dones, d_)
