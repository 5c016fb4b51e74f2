"""Behavioural tests of the CUDA env, ported from the reference's
tests/test_env.py and tests/test_vecenv.py (same scenarios and bars), run
through the drop-in API (RobotEnv / VecEnv)."""

import numpy as np
import pytest

from helpers import config, load_maps, make_map, ranges
from oracle.philox_shim import random_actions
from paper_2305_04180_b200.sim import (
    DiversityRanges,
    EnvConfig,
    EpisodeTerminated,
    Event,
    LidarConfig,
    MapError,
    SimParams,
)

pytestmark = pytest.mark.gpu

NOMINAL = SimParams(k=0.6, control_interval_s=0.1, control_delay_steps=0, v_linear_max_cm_s=18.0,
                    v_angular_max_rad_s=1.0, lidar_noise_std_cm=0.0)


def fixed_ranges(**over):
    p = {f: getattr(NOMINAL, f) for f in ("k", "control_interval_s", "control_delay_steps",
                                          "v_linear_max_cm_s", "v_angular_max_rad_s",
                                          "lidar_noise_std_cm")}
    p.update(over)
    return DiversityRanges(**{k: (v, v) for k, v in p.items()})


def make_env(n_cells=40, cfg=None, blocks=(), **over):
    from paper_2305_04180_b200.env import RobotEnv
    return RobotEnv(make_map(n_cells, blocks=blocks), fixed_ranges(**over), cfg or EnvConfig())


def place(env, x, y, heading=0.0):
    v = env.vec
    v.place("x", x); v.place("y", y); v.place("heading", heading)
    v.place("start_x", x); v.place("start_y", y)
    v.place("start_cos", np.cos(heading)); v.place("start_sin", np.sin(heading))


# -- test_env.py ---------------------------------------------------------------

def test_straight_action_advances_18cm_per_sim_second():  # test_env.py:45-54
    env = make_env(60, k=0.000001, control_interval_s=1.0)
    env.reset(0)
    place(env, 20.0, 20.0, 0.0)
    out = env.step(2)
    st = env.state
    assert st.x_cm == pytest.approx(38.0, abs=1e-3)
    assert st.y_cm == pytest.approx(20.0, abs=1e-9)
    assert st.heading_rad == pytest.approx(0.0)
    assert out.event is Event.NONE and not out.done


def test_action_table_targets():  # test_env.py:57-71
    for a, w in ((0, 1.0), (4, -1.0)):
        env = make_env(60, k=0.000001)
        env.reset(1)
        place(env, 20.0, 20.0, 0.0)
        env.step(a)
        st = env.state
        assert st.v_linear_cm_s == pytest.approx(0.36, rel=1e-5)
        assert st.v_angular_rad_s == pytest.approx(w, rel=1e-5)


@pytest.mark.parametrize("delay", [0, 1, 3, 17, 40, 64])
def test_control_delay_fidelity(delay):  # test_env.py:74-86 (+ delays past one history word)
    env = make_env(60, k=0.000001, control_delay_steps=delay)
    env.reset(2)
    place(env, 20.0, 20.0, 0.0)
    speeds = []
    for t in range(delay + 2):
        env.step(2 if t % 2 == 0 else 1)
        speeds.append(env.state.v_linear_cm_s)
    for t in range(delay):
        assert speeds[t] == pytest.approx(0.0, abs=1e-9)
    assert speeds[delay] == pytest.approx(18.0, rel=1e-4)


def test_arrival_event_and_reward():  # test_env.py:89-97
    env = make_env(40)
    env.reset(3)
    gx, gy = env.grid_map.goal_center
    place(env, gx - 1.0, gy, 0.0)
    out = env.step(2)
    assert out.event is Event.ARRIVAL and out.done and not out.truncated
    assert out.reward == 75.0


def test_collision_event_and_reward():  # test_env.py:100-107
    env = make_env(40, blocks=((20, 18, 22, 24),))
    env.reset(4)
    place(env, 15.0, 20.5, 0.0)
    out = env.step(2)
    assert out.event is Event.COLLISION and out.done and not out.truncated
    assert out.reward == -10.0


def test_timeout_truncates_without_done():  # test_env.py:110-121
    env = make_env(60, cfg=EnvConfig(timeout_steps=5), k=0.000001)
    env.reset(5)
    place(env, 20.0, 20.0, np.pi / 2)
    outs = [env.step(0) for _ in range(5)]
    assert [o.event for o in outs[:-1]] == [Event.NONE] * 4
    assert outs[-1].event is Event.TIMEOUT and outs[-1].truncated and not outs[-1].done
    assert -1.1 <= outs[-1].reward <= 1.1


def test_stepping_after_terminal_raises():  # test_env.py:124-134
    env = make_env(60, cfg=EnvConfig(timeout_steps=2))
    env.reset(6)
    env.step(0)
    env.step(0)
    with pytest.raises(EpisodeTerminated):
        env.step(0)
    env.reset(7)
    assert env.step(0).event in (Event.NONE, Event.COLLISION)
    env2 = make_env(60, cfg=EnvConfig(timeout_steps=2))
    env2.reset(6)
    env2.step(0)
    env2.step(0)
    env2.reset()  # continue the stream (SimBatch.reset_lane)
    assert not env2.episode_over and env2.steps_taken == 0


def test_event_exclusivity_random_rollouts():  # test_env.py:137-148
    env = make_env(50, blocks=((34, 10, 40, 30),))
    rng = np.random.default_rng(8)
    for _ in range(10):
        env.reset(int(rng.integers(1 << 31)))
        for _ in range(200):
            out = env.step(int(rng.integers(5)))
            assert out.done == (out.event in (Event.COLLISION, Event.ARRIVAL))
            assert out.truncated == (out.event is Event.TIMEOUT)
            if out.done or out.truncated:
                break


def test_determinism_same_seed_bit_identical():  # test_env.py:151-169
    actions = np.random.default_rng(1).integers(0, 5, 60)

    def rollout():
        env = make_env(40, lidar_noise_std_cm=1.0)
        states = [env.reset(123)]
        rewards = []
        for a in actions:
            out = env.step(int(a))
            states.append(out.state)
            rewards.append(out.reward)
            if out.done or out.truncated:
                env.reset(456)
        return np.stack(states), np.array(rewards)

    s1, r1 = rollout()
    s2, r2 = rollout()
    assert np.array_equal(s1, s2) and np.array_equal(r1, r2)


def test_encode_dx_endpoint_is_one():  # test_env.py:192-200 (via a step with k~0, v=0)
    cfg = EnvConfig(max_planning_dist_cm=100.0)
    env = make_env(200, cfg=cfg, k=0.000001)
    env.reset(10)
    gx, gy = env.grid_map.goal_center
    place(env, gx - 100.0, gy, 0.0)
    out = env.step(0)  # 0.36 cm/s x 0.1 s forward: dx = (100 - 0.036...) / 100
    assert out.state[0] == pytest.approx(1.0, abs=1e-3)
    assert out.state[1] == pytest.approx(0.0, abs=1e-3)


def test_state_bounds_within_planning_distance():  # test_env.py:226-236
    env = make_env(40, lidar_noise_std_cm=1.0)
    rng = np.random.default_rng(13)
    for _ in range(15):
        s = env.reset(int(rng.integers(1 << 31)))
        assert (np.abs(s) <= 1.0).all()
        for _ in range(40):
            out = env.step(int(rng.integers(5)))
            assert (np.abs(out.state) <= 1.0 + 1e-6).all()
            if out.done or out.truncated:
                break


def test_reset_zero_width_ranges_yield_nominals():  # test_env.py:242-245
    env = make_env(40)
    env.reset(14)
    assert env.params == NOMINAL


def test_reset_resampling_stays_inside_intervals():  # test_env.py:248-268 (vectorized)
    from paper_2305_04180_b200 import VecEnv
    rg = DiversityRanges.around(SimParams(), 0.3)
    env = VecEnv([make_map(40)], 10_000, rg)
    env.reset_all(15)
    sim = env.sim
    seen = {"k": sim.param_k, "control_interval_s": sim.param_dt,
            "control_delay_steps": sim.param_delay, "v_linear_max_cm_s": sim.param_vmax[:, 0],
            "v_angular_max_rad_s": sim.param_vmax[:, 1], "lidar_noise_std_cm": sim.param_noise}
    for f, arr in seen.items():
        lo, hi = getattr(rg, f)
        assert arr.min() >= lo and arr.max() <= hi
        if hi > lo:
            assert arr.max() - arr.min() > 0.5 * (hi - lo)


def test_reset_spawns_inside_region_collision_free():  # test_env.py:271-279
    from paper_2305_04180_b200 import VecEnv
    from paper_2305_04180_b200.env import check_collision
    m = make_map(40)
    env = VecEnv([m], 200, fixed_ranges())
    env.reset_all(16)
    x0, y0, x1, y1 = m.spawn_region
    xs, ys = env.sim.x, env.sim.y
    assert ((xs >= x0) & (xs <= x1) & (ys >= y0) & (ys <= y1)).all()
    assert not any(check_collision(m, (x, y), radius_cm=9.0) for x, y in zip(xs[:20], ys[:20]))


def test_no_spawn_pose_raises_map_error():
    from paper_2305_04180_b200 import VecEnv
    m = make_map(40, blocks=((10, 10, 20, 20),), spawn=(11.0, 11.0, 18.0, 18.0))
    env = VecEnv([m], 4, fixed_ranges(), EnvConfig(spawn_attempts=5))
    with pytest.raises(MapError):
        env.reset_all(1)


def test_lidar_scan_and_collision_helpers():  # test_env.py:301-329
    from paper_2305_04180_b200.env import RobotState, check_collision, lidar_scan
    m = make_map(30)
    pose = RobotState(15.0, 15.0, 0.3, 0, 0, 9.0)
    scan = lidar_scan(m, pose, LidarConfig(max_range_cm=10.0))
    assert scan.shape == (27,) and np.array_equal(scan, np.full(27, 10.0))
    m2 = make_map(100, blocks=((50, 50, 52, 52),))
    assert not check_collision(m2, (25.0, 25.0), radius_cm=9.0)
    assert check_collision(m2, (50.5, 50.5), radius_cm=1.0)
    assert check_collision(m2, (41.0, 51.0), radius_cm=9.0)
    assert check_collision(m2, (5.0, 5.0), radius_cm=9.0)


def test_axis_parallel_beam_from_a_cell_boundary():
    """A beam exactly along +x (heading 0, centre beam offset 0.0) from a
    row boundary (integer y, cell 1 cm) never crosses a y face: its range is
    the x-face entry alone (the wall face at x = 30), from any origin."""
    from paper_2305_04180_b200 import VecEnv
    lc = LidarConfig(n_beams=27, max_range_cm=100.0)
    j = int(np.flatnonzero(lc.beam_offsets() == 0.0)[0])
    m = make_map(40, blocks=((30, 0, 32, 40),))
    env = VecEnv([m], 1, fixed_ranges(), EnvConfig(lidar=lc))
    xs, ys = [10.0, 10.0, 10.5, 12.0, 10.25], [20.0, 20.5, 20.0, 7.0, 33.0]
    got = env.scan(xs, ys, np.zeros(5)).cpu().numpy()
    assert np.array_equal(got[:, j], 30.0 - np.asarray(xs))


# -- test_vecenv.py --------------------------------------------------------------

def _rg(frac=0.3):
    return DiversityRanges.around(SimParams(), frac)


def test_reset_shapes_and_determinism():  # test_vecenv.py:15-24
    from paper_2305_04180_b200 import VecEnv
    maps = [make_map(40), make_map(40, blocks=((30, 8, 34, 20),))]
    s1 = VecEnv(maps, 16, _rg()).reset_all(7).cpu().numpy()
    assert s1.shape == (16, 32) and s1.dtype == np.float32
    assert np.array_equal(s1, VecEnv(maps, 16, _rg()).reset_all(7).cpu().numpy())
    assert not np.array_equal(s1, VecEnv(maps, 16, _rg()).reset_all(8).cpu().numpy())


def test_lanes_are_independent_of_batch_and_shard():  # test_vecenv.py:42-67 (+ sharding)
    """Lane i of an N-lane run equals a 1-lane run with env_id_offset=i, and a
    run split into shards equals the whole run -- the multi-GPU invariant."""
    from paper_2305_04180_b200 import VecEnv
    maps = load_maps(4)
    n, cfg, seed = 24, config(32, timeout_steps=25), 11
    full = VecEnv(maps, n, _rg(), cfg)
    fs = [full.reset_all(seed).cpu().numpy()]
    shards = [VecEnv(maps, 10, _rg(), cfg, env_id_offset=0),
              VecEnv(maps, 14, _rg(), cfg, env_id_offset=10)]
    ss = [np.concatenate([sh.reset_all(seed).cpu().numpy() for sh in shards])]
    solo = VecEnv(maps, 1, _rg(), cfg, env_id_offset=7)
    so = [solo.reset_all(seed).cpu().numpy()]
    for t in range(60):
        a = random_actions(seed, np.arange(n), t)
        fs.append(full.step_batch(a).store_states.cpu().numpy())
        ss.append(np.concatenate([shards[0].step_batch(a[:10]).store_states.cpu().numpy(),
                                  shards[1].step_batch(a[10:]).store_states.cpu().numpy()]))
        so.append(solo.step_batch(a[7:8]).store_states.cpu().numpy())
    fs, ss, so = np.stack(fs), np.stack(ss), np.stack(so)
    assert np.array_equal(fs, ss)
    assert np.array_equal(fs[:, 7:8], so)


def test_sharded_recent_returns_merge_into_the_single_run_deque():  # vecenv.py:79, 109
    """Shards' keyed recent returns (step, global env id) merge into exactly
    the deque(maxlen=256) of one VecEnv stepping every id (dist.py)."""
    from paper_2305_04180_b200 import VecEnv
    from paper_2305_04180_b200.dist import merge_recent_returns, pooled_stats
    maps = load_maps(4)
    n, cfg, seed = 300, config(32, timeout_steps=9), 13
    full = VecEnv(maps, n, _rg(), cfg)
    full.reset_all(seed)
    shards = [VecEnv(maps, 120, _rg(), cfg, env_id_offset=0),
              VecEnv(maps, 180, _rg(), cfg, env_id_offset=120)]
    for sh in shards:
        sh.reset_all(seed)
    for t in range(40):
        a = random_actions(seed, np.arange(n), t)
        full.step_batch(a)
        shards[0].step_batch(a[:120])
        shards[1].step_batch(a[120:])
    want = full.recent_returns()
    assert len(want) == 256
    keys, vals = full.recent_returns_keyed()
    assert vals.tolist() == want and np.all(np.diff(keys.astype(np.float64)) > 0)
    got = merge_recent_returns([sh.recent_returns_keyed() for sh in shards])
    assert got == want
    assert pooled_stats(full)["recent_returns"] == want  # world size 1: no collective


def test_auto_reset_reports_fresh_state_and_stores_terminal():  # test_vecenv.py:70-82
    from paper_2305_04180_b200 import VecEnv
    env = VecEnv([make_map(40)], 3, _rg(0.0), EnvConfig(timeout_steps=4))
    env.reset_all(5)
    last = None
    for _ in range(4):
        last = env.step_batch([2, 2, 2])
    ended = (last.dones | last.truncated).cpu().numpy()
    assert ended.any()
    st, ss = last.states.cpu().numpy(), last.store_states.cpu().numpy()
    for i in np.flatnonzero(ended):
        assert not np.array_equal(st[i], ss[i])
    assert env.snapshot_stats().episodes == int(ended.sum())


def test_auto_reset_off_requires_manual_reset():  # test_vecenv.py:85-92
    from paper_2305_04180_b200 import VecEnv
    env = VecEnv([make_map(40)], 2, _rg(0.0), EnvConfig(timeout_steps=2), auto_reset=False)
    env.reset_all(6)
    env.step_batch([2, 2])
    env.step_batch([2, 2])
    with pytest.raises(EpisodeTerminated):
        env.step_batch([2, 2])
    env.reset_lanes([1, 1])
    env.step_batch([2, 2])


def test_shape_contract_and_episode_conservation():  # test_vecenv.py:95-115
    from paper_2305_04180_b200 import VecEnv
    env = VecEnv([make_map(40)], 5, _rg(0.0), EnvConfig(timeout_steps=3))
    env.reset_all(7)
    total = 0
    for t in range(30):
        b = env.step_batch(np.random.default_rng(t).integers(0, 5, 5))
        assert b.states.shape == (5, 32) and b.store_states.shape == (5, 32)
        assert b.rewards.shape == (5,) and b.rewards.dtype.is_floating_point
        assert b.dones.shape == (5,)
        total += int((b.dones | b.truncated).sum())
    assert env.snapshot_stats().episodes == total


def test_per_copy_maps_encode_their_own_geometry():  # test_vecenv.py:118-124
    from paper_2305_04180_b200 import VecEnv
    env = VecEnv([make_map(40), make_map(40, goal=(12.0, 30.0))], 4, _rg(0.0))
    env.reset_all(9)
    assert np.array_equal(env.map_index, [0, 1, 0, 1])
    assert env.sim.goal_x[1] == 12.0 and env.sim.goal_x[0] == 28.0


def test_stats_snapshot_and_reset():  # test_vecenv.py:127-152
    from paper_2305_04180_b200 import VecEnv
    env = VecEnv([make_map(40)], 2, _rg(0.0), EnvConfig(timeout_steps=3))
    env.reset_all(10)
    assert env.snapshot_stats().arrival_rate is None
    for _ in range(6):
        env.step_batch([2, 2])
    snap = env.snapshot_stats(reset=True)
    assert snap.episodes == 4
    assert snap.arrivals == sum(c.arrivals for c in snap.per_copy)
    assert len(snap.recent_returns) == 4
    assert env.snapshot_stats().episodes == 0
    outs = env.first_episode_outcomes()
    assert all(o is not None and o[2] == 3 for o in outs) and env.all_first_episodes_done


def test_bad_inputs_rejected():  # test_vecenv.py:155-164
    from paper_2305_04180_b200 import VecEnv
    env = VecEnv([make_map(40)], 3, _rg(0.0))
    env.reset_all(12)
    with pytest.raises(ValueError):
        env.step_batch([1, 2])
    with pytest.raises(ValueError):
        env.step_batch([1, 2, 5])
    import torch
    with pytest.raises(ValueError):
        env.step_batch(torch.tensor([0, -1, 2], device="cuda"))
    with pytest.raises(MapError):
        VecEnv([make_map(40), make_map(50)], 2, _rg())
    with pytest.raises(ValueError):
        VecEnv([make_map(40)], 0)


def test_device_action_errors_surface_lazily():
    from paper_2305_04180_b200 import VecEnv
    import torch
    env = VecEnv([make_map(40)], 3, _rg(0.0), check_actions=False)
    env.reset_all(12)
    env.step_batch(torch.tensor([0, 9, 2], device="cuda"))
    with pytest.raises(ValueError):
        env.check()


def test_many_resets_in_one_step_use_the_overflow_pass():
    """All lanes time out together (timeout 3): more resets than extra scan
    slots -- the overflow pass must produce the same rows as the oracle."""
    from paper_2305_04180_b200 import VecEnv
    from oracle.oracle import OracleVecEnv
    from helpers import assert_close, assert_obs
    maps = [make_map(40)]
    cfg = config(32, timeout_steps=3)
    n = 3000
    gpu = VecEnv(maps, n, fixed_ranges(lidar_noise_std_cm=1.0), cfg)
    cpu = OracleVecEnv(maps, n, fixed_ranges(lidar_noise_std_cm=1.0), cfg)
    gpu.reset_all(3)
    cpu.reset_all(3)
    for t in range(7):
        a = np.zeros(n, dtype=np.int64)  # slow turns: everyone survives to the timeout
        g, c = gpu.step_batch(a), cpu.step_batch(a)
        assert np.array_equal(g.events.cpu().numpy(), c.events)
        assert_obs(g.states.cpu().numpy(), c.states, what=f"states {t}")
        assert_obs(g.store_states.cpu().numpy(), c.store_states, what="store")


def test_mass_timeouts_across_all_ctas():
    """4096 lanes on 16 maps (every CTA busy) all time out on the same steps:
    every chunk takes the reset path at once (reset slots, step-count history
    of reset scans) and the rows still match the oracle."""
    from paper_2305_04180_b200 import VecEnv
    from oracle.oracle import OracleVecEnv
    from helpers import assert_close, assert_obs
    import torch
    maps = load_maps(16)
    cfg = config(32, timeout_steps=4)
    n = 4096
    gpu = VecEnv(maps, n, ranges(0.3), cfg)
    cpu = OracleVecEnv(maps, n, ranges(0.3), cfg)
    gpu.reset_all(5)
    cpu.reset_all(5)
    for t in range(13):
        a = np.zeros(n, dtype=np.int64)  # slow turns: lanes survive to the timeout
        g, c = gpu.step_batch(a), cpu.step_batch(a)
        torch.cuda.synchronize()
        assert np.array_equal(g.events.cpu().numpy(), c.events), t
        assert_obs(g.states.cpu().numpy(), c.states, what=f"states {t}")
        assert_obs(g.store_states.cpu().numpy(), c.store_states, what="store")
    gpu.check()


def test_step_host_matches_device_step():
    """VecEnv.step_host (numpy in, numpy StepBatch out through page-locked
    buffers) gives the same StepBatch as the device path."""
    from paper_2305_04180_b200 import VecEnv
    maps = load_maps(4)
    n = 1000
    a_env = VecEnv(maps, n, ranges(0.3), config(32))
    b_env = VecEnv(maps, n, ranges(0.3), config(32))
    a_env.reset_all(3)
    b_env.reset_all(3)
    for t in range(60):
        acts = random_actions(3, np.arange(n), t)
        x = a_env.step_batch(acts)
        y = b_env.step_host(acts)
        assert isinstance(y.states, np.ndarray) and y.states.dtype == np.float32
        for f in ("states", "store_states", "rewards", "dones", "truncated", "events"):
            assert np.array_equal(getattr(x, f).cpu().numpy(), getattr(y, f)), (t, f)
    with pytest.raises(ValueError):
        b_env.step_host(np.full(n, 7))


@pytest.mark.parametrize("n", [257, 20_000])
def test_step_host_bad_action_steps_nothing(n):
    """core.py:169-170: one action out of range raises ValueError before any
    lane steps -- sp_env_step_host checks on the host while the actions'
    copy is in flight (one part and the row-part path): the next valid step
    equals a twin env's that never saw the bad call."""
    from paper_2305_04180_b200 import VecEnv
    maps = load_maps(16)
    a_env = VecEnv(maps, n, ranges(0.3), config(32))
    b_env = VecEnv(maps, n, ranges(0.3), config(32))
    a_env.reset_all(11)
    b_env.reset_all(11)
    acts = np.ascontiguousarray(random_actions(11, np.arange(n), 0), np.int64)
    bad = acts.copy()
    bad[n // 2] = 5
    with pytest.raises(ValueError, match="out of range"):
        b_env.step_host(bad)
    x, y = a_env.step_host(acts), b_env.step_host(acts)
    for f in ("states", "store_states", "rewards", "dones", "truncated", "events"):
        assert np.array_equal(getattr(x, f), getattr(y, f)), f
    b_env.check()  # no sticky device error


@pytest.mark.parametrize("n,parts", [(65_536, None), (4_096, "3"), (3_000, "8")])
def test_step_host_row_parts_match_device_step(monkeypatch, n, parts):
    """sp_env_step_host in row parts (a launch per part, each part's rows read
    back while the next part steps; 2 parts (1:3) by default from 16,384 envs,
    SPARROW_HOST_PARTS otherwise) gives the device step's StepBatch, and the
    two handles' episode statistics agree."""
    from paper_2305_04180_b200 import VecEnv
    if parts:
        monkeypatch.setenv("SPARROW_HOST_PARTS", parts)
    maps = load_maps(16)
    a_env = VecEnv(maps, n, ranges(0.3), config(32, timeout_steps=9))
    b_env = VecEnv(maps, n, ranges(0.3), config(32, timeout_steps=9))
    a_env.reset_all(5)
    b_env.reset_all(5)
    for t in range(12):
        acts = random_actions(5, np.arange(n), t)
        x = a_env.step_batch(acts)
        y = b_env.step_host(acts)
        for f in ("states", "store_states", "rewards", "dones", "truncated", "events"):
            assert np.array_equal(getattr(x, f).cpu().numpy(), getattr(y, f)), (t, f)
    sa, sb = a_env.snapshot_stats(), b_env.snapshot_stats()
    assert (sa.episodes, sa.arrivals) == (sb.episodes, sb.arrivals)
    assert list(sa.recent_returns) == list(sb.recent_returns)


def test_reset_clears_terminal_flag_and_velocity():  # test_env.py:282-296
    env = make_env(40, cfg=EnvConfig(timeout_steps=3))
    env.reset(17)
    for _ in range(3):
        out = env.step(2)
        if out.done or out.truncated:
            break
    assert env.episode_over
    env.reset(18)
    assert not env.episode_over
    st = env.state
    assert st.v_linear_cm_s == 0.0 and st.v_angular_rad_s == 0.0
    assert env.steps_taken == 0


def test_lidar_scan_noise_is_clamped_and_seeded():  # test_env.py:310-319
    from paper_2305_04180_b200.env import RobotState, lidar_scan
    m = make_map(30)
    pose = RobotState(15.0, 15.0, 0.0, 0, 0, 9.0)
    cfg = LidarConfig(max_range_cm=50.0)
    a = lidar_scan(m, pose, cfg, noise_std=5.0, rng=np.random.default_rng(1))
    b = lidar_scan(m, pose, cfg, noise_std=5.0, rng=np.random.default_rng(1))
    assert np.array_equal(a, b)
    assert (a >= 0).all() and (a <= 50.0).all()
    assert not np.array_equal(a, lidar_scan(m, pose, cfg, noise_std=0.0))


def test_pooled_rate_matches_raw_counters():  # test_vecenv.py:141-152
    from paper_2305_04180_b200 import VecEnv
    env = VecEnv([make_map(40)], 3, _rg(0.0), EnvConfig(timeout_steps=2))
    env.reset_all(11)
    for _ in range(8):
        env.step_batch([0, 1, 2])
    snap = env.snapshot_stats()
    eps = sum(c.episodes for c in snap.per_copy)
    arr = sum(c.arrivals for c in snap.per_copy)
    assert snap.episodes == eps == 3 * 4
    assert (snap.arrival_rate or 0.0) == pytest.approx(arr / eps if eps else 0.0)


def test_mixed_grid_shapes_rejected():  # test_vecenv.py:162-164
    from paper_2305_04180_b200 import VecEnv
    with pytest.raises(MapError):
        VecEnv([make_map(40), make_map(50)], 2, [_rg(), _rg()])
    with pytest.raises(ValueError):
        VecEnv([make_map(40)], 2, [_rg()])  # one DiversityRanges per lane


def test_n1_matches_single_env():  # test_vecenv.py:27-39
    """A 1-copy VecEnv and the single-robot RobotEnv on the same map and seed
    reset and step identically (the RobotEnv is lane 0 of the same kernel)."""
    from paper_2305_04180_b200 import VecEnv
    from paper_2305_04180_b200.env import RobotEnv
    m = make_map(40)
    vec = VecEnv([m], 1, _rg())
    sv = vec.reset_all(3).cpu().numpy()
    env = RobotEnv(m, _rg())
    ss = env.reset(3)
    assert np.array_equal(sv[0], ss)
    for a in (2, 0, 4, 2, 1):
        b = vec.step_batch([a])
        out = env.step(a)
        assert np.array_equal(b.store_states[0].cpu().numpy(), out.state)
        assert float(b.rewards[0]) == out.reward


def test_render_ascii_marks_robot():  # env.py:109-110
    env = make_env(40)
    env.reset(5)
    place(env, 12.5, 20.5, 0.0)
    txt = env.render_ascii()
    rows = txt.splitlines()
    assert len(rows) == 40 and sum(r.count("R") for r in rows) == 1
    assert rows[40 - 1 - 20][12] == "R"


def test_c_abi_host_step_with_pageable_buffers():
    """sp_env_step_host straight from numpy (pageable) memory: the documented
    block layout, the same results as the device step."""
    import ctypes
    from paper_2305_04180_b200 import VecEnv, _lib
    maps = load_maps(2)
    n = 257
    a_env = VecEnv(maps, n, ranges(0.3), config(32))
    b_env = VecEnv(maps, n, ranges(0.3), config(32))
    a_env.reset_all(9)
    b_env.reset_all(9)
    D = b_env.state_dim
    nbytes = int(b_env._lib.sp_env_host_out_bytes(b_env._h))
    assert nbytes == n * (8 + 8 * D + 3)
    block = np.zeros(nbytes, np.uint8)
    for t in range(25):
        acts = np.ascontiguousarray(random_actions(9, np.arange(n), t), np.int64)
        x = a_env.step_batch(acts)
        _lib.check(b_env._lib.sp_env_step_host(b_env._h, acts.ctypes.data, block.ctypes.data,
                                               b_env._stream()), "step_host")
        off = 0
        rew = block[off:off + 8 * n].view(np.float64); off += 8 * n
        st = block[off:off + 4 * n * D].view(np.float32).reshape(n, D); off += 4 * n * D
        ss = block[off:off + 4 * n * D].view(np.float32).reshape(n, D); off += 4 * n * D
        dn, tr, ev = block[off:off + n], block[off + n:off + 2 * n], block[off + 2 * n:].view(np.int8)
        assert np.array_equal(x.rewards.cpu().numpy(), rew)
        assert np.array_equal(x.states.cpu().numpy(), st)
        assert np.array_equal(x.store_states.cpu().numpy(), ss)
        assert np.array_equal(x.dones.cpu().numpy(), dn.astype(bool))
        assert np.array_equal(x.truncated.cpu().numpy(), tr.astype(bool))
        assert np.array_equal(x.events.cpu().numpy(), ev)
    del ctypes


# -- drop-in surface: SimBatch views the reference's own tests read ----------

@pytest.mark.parametrize("delay", [0, 2, 17])
def test_pending_actions_queue(delay):  # sim/env.py:39, 94; core.py:156, 176-182
    """RobotState.pending_actions / sim._pending mirror the reference deque:
    d (0, 0) fillers after a reset, then each issued target in order."""
    env = make_env(60, k=0.5, control_delay_steps=delay)
    env.reset(4)
    place(env, 20.0, 20.0, 0.0)
    assert env.state.pending_actions == ((0.0, 0.0),) * delay
    table = [tuple(p) for p in EnvConfig().action_table]
    issued = []
    for t in range(delay + 3):
        a = (1, 3, 2, 0, 4)[t % 5]
        env.step(a)
        issued.append(table[a])
        want = ([(0.0, 0.0)] * delay + issued)[-delay:] if delay else []
        assert env.state.pending_actions == tuple(want), t
        assert list(env.vec.sim._pending[0]) == want


def test_last_scan_and_params_views():  # core.py:97, 104; sim/env.py:80-99
    """sim.last_scan is the noisy clipped range behind the states rows: exact
    f64 while recording, and equal (to float32 rounding) to the obs columns."""
    from oracle.oracle import OracleVecEnv
    from paper_2305_04180_b200 import VecEnv
    maps = load_maps(4)
    n, seed = 96, 21
    g = VecEnv(maps, n, ranges(0.3), config(32))
    c = OracleVecEnv(maps, n, ranges(0.3), config(32))
    s_plain = g.reset_all(seed)
    approx = g.sim.last_scan  # not recording: from the float32 obs columns
    c.reset_all(seed)
    want = c.cells()["last_scan"]
    assert_close = __import__("helpers").assert_close
    assert_close(approx, want, rtol=1.2e-7, atol=1e-9, what="last_scan (obs-derived)")
    g.record()
    for t in range(6):
        a = random_actions(seed, np.arange(n), t)
        g.step_batch(a)
        c.step_batch(a)
        assert_close(g.sim.last_scan, c.cells()["last_scan"], rtol=1e-9, atol=1e-5,
                     what=f"last_scan step {t}")
    ps = g.sim.params
    assert len(ps) == n and all(isinstance(p, SimParams) for p in ps)
    assert [p.control_delay_steps for p in ps] == list(g.sim.param_delay)
    assert np.allclose([p.k for p in ps], g.sim.param_k)
    del s_plain


def test_overlapping_state_buffers_rejected():
    """states and store_states must be distinct rows (each scan parks its
    noise in its own row): overlapping buffers raise ValueError."""
    import torch
    from paper_2305_04180_b200 import VecEnv
    from paper_2305_04180_b200.vecenv import StepBatch
    env = VecEnv(load_maps(1), 8, ranges(0.0), config(32))
    env.reset_all(1)
    D = env.state_dim
    rows = torch.empty((8, D), dtype=torch.float32, device=env.device)
    out = StepBatch(rows, torch.empty(8, dtype=torch.float64, device=env.device),
                    torch.empty(8, dtype=torch.bool, device=env.device),
                    torch.empty(8, dtype=torch.bool, device=env.device), rows,
                    torch.empty(8, dtype=torch.int8, device=env.device))
    with pytest.raises(ValueError):
        env.step_batch(np.zeros(8, np.int64), out=out)


def test_recent_returns_keep_time_order_across_reset_all():  # vecenv.py:79, 84-92, 109
    """reset_all does not clear the recent-returns deque in the reference; the
    returns of episodes after a second reset_all are the newest entries."""
    from oracle.oracle import OracleVecEnv
    from paper_2305_04180_b200 import VecEnv
    maps = load_maps(2)
    n = 64
    cfg = config(32, timeout_steps=4)
    g = VecEnv(maps, n, ranges(0.3), cfg)
    c = OracleVecEnv(maps, n, ranges(0.3), cfg)
    for seed, steps in ((1, 9), (2, 9)):
        g.reset_all(seed)
        c.reset_all(seed)
        for t in range(steps):
            a = random_actions(seed, np.arange(n), t)
            g.step_batch(a)
            c.step_batch(a)
    got = g.snapshot_stats().recent_returns
    want = c.stats()["recent_returns"]
    assert len(got) == len(want) == 256
    # the same multiset per step; order within a step follows env id on both sides
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)
