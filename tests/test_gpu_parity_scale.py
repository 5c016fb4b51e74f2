"""GPU parity at the BASELINE sizes the headline is quoted on.

cfg3 (BASELINE.json configs[2]): 65,536 envs per GPU, 16 maps, +/-30 %
diversity, 32 beams -- the workload of bench.py's `value`.  The fused step is
stepped against the C oracle (``oracle/``, itself pinned to the unmodified
reference) on the same seeds and actions for >= 30 steps with auto-reset, and
every step is compared:

* bit-exact: events, dones, truncated, and the LiDAR HIT CELL of every ray of
  both scans an env can take in a step (the post-step scan behind
  store_states and the scan behind states -- a fresh-spawn scan after an
  auto-reset), read from the kernel's recording outputs against the oracle's
  DDA (``_cy.pyx:89-105``);
* rewards within 1e-10, obs within 2 float32 ulps (tests/helpers.py);
* at the end: poses (1e-5 relative), RNG draw counters, per-copy episode and
  arrival counters (exact), return sums.

The oracle runs sharded over the host cores by env id (oracle.ShardedOracle:
lanes are independent and keyed by global env id), so these sizes take
seconds per step.  Sizes: cfg3 itself; 262,144 envs (several chunks per CTA,
so CTAs walk multi-chunk ranges); one shard of an 8-GPU run
(env_id_offset = 7 * 65,536); and a reset-heavy cfg3 (timeout 6 steps: every
CTA's spare scan slots overflow into the second pass).
"""

import numpy as np
import pytest

from helpers import assert_close, assert_obs, assert_rewards, config, load_maps, ranges
from oracle.philox_shim import random_actions

pytestmark = pytest.mark.gpu

CFG3 = 65_536


def _run(n, steps, seed, div=0.3, offset=0, timeout=None, check_every=1, n_beams=32):
    from oracle.oracle import ShardedOracle
    from paper_2305_04180_b200 import VecEnv
    maps = load_maps(16)
    kw = {} if timeout is None else {"timeout_steps": timeout}
    cfg = config(n_beams, **kw)
    gpu = VecEnv(maps, n, ranges(div), cfg, env_id_offset=offset)
    gpu.record()
    cpu = ShardedOracle(maps, n, ranges(div), cfg, env_id_offset=offset)
    ids = offset + np.arange(n)
    try:
        assert_obs(gpu.reset_all(seed).cpu().numpy(), cpu.reset_all(seed), what="reset_all")
        rec = gpu.recorded()
        oc = cpu.cells()
        assert np.array_equal(rec["hit_state"].cpu().numpy(), oc["state"]), "reset hit cells"
        ends = 0
        for t in range(steps):
            a = random_actions(seed, ids, t)
            g = gpu.step_batch(a)
            c = cpu.step_batch(a)
            ev = g.events.cpu().numpy()
            assert np.array_equal(ev, c.events), f"events differ at step {t}"
            assert np.array_equal(g.dones.cpu().numpy(), c.dones), f"dones step {t}"
            assert np.array_equal(g.truncated.cpu().numpy(), c.truncated), f"truncated step {t}"
            ends += int((ev != 0).sum())
            if t % check_every and t != steps - 1:
                continue
            assert_rewards(g.rewards.cpu().numpy(), c.rewards, what=f"rewards step {t}")
            assert_obs(g.store_states.cpu().numpy(), c.store_states, what=f"store_states {t}")
            assert_obs(g.states.cpu().numpy(), c.states, what=f"states {t}")
            oc = cpu.cells()
            hs, hx = rec["hit_store"].cpu().numpy(), rec["hit_state"].cpu().numpy()
            bad = hs != oc["store"]
            assert not bad.any(), f"step {t}: {int(bad.sum())} post-step hit cells differ"
            bad = hx != oc["state"]
            assert not bad.any(), f"step {t}: {int(bad.sum())} states-row hit cells differ"
            assert_close(rec["scan_state"].cpu().numpy(), oc["last_scan"], rtol=1e-9, atol=1e-5,
                         what=f"last_scan {t}")
        p = cpu.pose()
        sim = gpu.sim
        assert_close(sim.x, p["x"], what="x")
        assert_close(sim.y, p["y"], what="y")
        assert_close(sim.heading, p["heading"], atol=1e-12, what="heading")
        assert np.array_equal(sim.step_count, p["step_count"]), "step counts"
        assert np.array_equal(sim.rng_ctr.astype(np.uint64), p["rng_ctr"]), "draw counters"
        st = cpu.stats()
        mine = gpu._per_copy_arrays()
        for f in ("episodes", "arrivals", "first_event", "first_steps"):
            assert np.array_equal(mine[f], st[f].astype(mine[f].dtype)), f
        assert_close(mine["return_sum"], st["return_sum"], rtol=1e-12, atol=1e-9,
                     what="return_sum")
        return ends
    finally:
        cpu.close()


def test_cfg3_headline_parity():
    """The headline workload itself: 65,536 envs, 30 steps, every step checked."""
    ends = _run(CFG3, 30, seed=20230504)
    assert ends > 1000  # auto-resets happen at this size (~0.9 % of env-steps)


def test_262144_envs_multi_chunk_ctas():
    """4 x cfg3 on one GPU: ~1,770 envs per CTA, so every CTA walks several
    chunks of its range and rebinds per chunk (bench.py's env sweep top)."""
    _run(4 * CFG3, 30, seed=7, check_every=3)


def test_eighth_shard_of_an_8_gpu_run():
    """Rank 7 of 8 at cfg3: global env ids [7*65,536, 8*65,536) -- lanes are
    bit-identical to those of one big run (RNG and map keyed by global id)."""
    _run(CFG3, 30, seed=99, offset=7 * CFG3)


def test_cfg3_reset_heavy():
    """Timeout 6 steps: after step 6 every env resets, far more resets per
    chunk than spare scan slots -> the overflow pass runs in every CTA."""
    _run(CFG3, 14, seed=5, timeout=6)


@pytest.mark.parametrize("timeout", [None, 6])
def test_inline_resets_match(monkeypatch, timeout):
    """The inline auto-reset path (the env lane resets after its own header;
    used when a chunk leaves no spare idle warp for the reset warp), forced
    with SPARROW_LATE_RESETS=0, against the oracle at cfg3 and reset-heavy."""
    monkeypatch.setenv("SPARROW_LATE_RESETS", "0")
    _run(CFG3, 12, seed=31, timeout=timeout, check_every=3)
