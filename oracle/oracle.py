"""CPU ORACLE wrapper -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg may import this module.  It is the checker, never the thing measured or
shipped: the product package (``paper_2305_04180_b200``) never imports it.

Contents
* ``load_lib``       -- ctypes handle to ``oracle/_build/liboracle.so`` (the C
  restatement in ``sparrow_oracle.c``; built by ``make -C oracle``).
* ``cast_rays`` / ``disc_collides`` -- restate ``kernels/_cy.pyx:19-158`` with
  the signature of ``kernels/__init__.py:62-86``.
* ``OracleVecEnv``   -- restates ``VecEnv`` (``vecenv.py:61-145``) over
  ``SimBatch`` (``sim/core.py:47-261``) driven by the Philox contract
  (``oracle/philox_shim.py``).
* ``ReplayOracle``   -- numpy restatement of ``ReplayBuffer``
  (``replay.py:31-87``).

Parity is pinned against the real reference by
``tests/test_oracle_vs_reference.py`` and ``tests/golden/``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import NamedTuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref")

_lib = None

c_dp = ctypes.POINTER(ctypes.c_double)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_i8p = ctypes.POINTER(ctypes.c_int8)
c_fp = ctypes.POINTER(ctypes.c_float)
c_u64p = ctypes.POINTER(ctypes.c_uint64)


def build(quiet: bool = True) -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)
    return LIB_PATH


def load_lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    lib = ctypes.CDLL(LIB_PATH)
    lib.or_env_create.restype = ctypes.c_void_p
    lib.or_env_create.argtypes = [
        ctypes.c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
        ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_dp, ctypes.c_int64, ctypes.c_int64,
        ctypes.c_int64, ctypes.c_double, c_u8p, c_dp, c_dp, c_dp, c_dp, c_dp, c_dp,
        ctypes.c_int64, c_i64p, c_dp, c_dp, ctypes.c_int64]
    lib.or_env_destroy.argtypes = [ctypes.c_void_p]
    lib.or_env_reset_all.argtypes = [ctypes.c_void_p, ctypes.c_uint64, c_fp]
    lib.or_env_step.argtypes = [ctypes.c_void_p, c_i64p, c_fp, c_fp, c_dp, c_u8p, c_u8p, c_i8p]
    lib.or_env_get_pose.argtypes = [ctypes.c_void_p, c_dp, c_dp, c_dp, c_dp, c_dp, c_i64p, c_u64p]
    lib.or_env_get_stats.argtypes = [ctypes.c_void_p, c_i64p, c_i64p, c_dp, c_i8p, c_dp, c_i64p,
                                     c_dp, c_i64p]
    lib.or_env_reset_stats.argtypes = [ctypes.c_void_p]
    lib.or_env_err_lane.argtypes = [ctypes.c_void_p]
    lib.or_env_get_cells.argtypes = [ctypes.c_void_p, c_i64p, c_i64p, c_dp]
    lib.or_cast_rays.argtypes = [c_u8p, c_dp, ctypes.c_int64, ctypes.c_int64, c_i64p, c_dp, c_dp,
                                 c_dp, c_dp, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                 c_dp, c_i64p]
    lib.or_count_dda_cells.argtypes = [c_u8p, ctypes.c_int64, ctypes.c_int64, c_i64p, c_dp, c_dp,
                                       c_dp, c_dp, ctypes.c_int64, ctypes.c_double,
                                       ctypes.c_double, c_i64p]
    lib.or_disc_collides.argtypes = [c_u8p, ctypes.c_int64, ctypes.c_int64, c_i64p, c_dp, c_dp,
                                     c_dp, ctypes.c_int64, ctypes.c_double, c_u8p]
    lib.or_stream_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_int, c_dp]
    _lib = lib
    return lib


def _p(a, t):
    return a.ctypes.data_as(t)


# -- kernels -------------------------------------------------------------------

def cast_rays(occ, edt, map_idx, px, py, dirx, diry, cell, max_range, return_cells=False):
    """Restates kernels.cast_rays (``kernels/__init__.py:62-76``, ``_cy.pyx:19-106``)."""
    lib = load_lib()
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    edt = np.ascontiguousarray(edt, dtype=np.float64)
    m, h, w = occ.shape
    midx = np.ascontiguousarray(map_idx, dtype=np.int64)
    px, py, dx, dy = (np.ascontiguousarray(a, dtype=np.float64) for a in (px, py, dirx, diry))
    n = px.shape[0]
    out = np.empty(n, dtype=np.float64)
    cells = np.empty(n, dtype=np.int64)
    lib.or_cast_rays(_p(occ, c_u8p), _p(edt, c_dp), h, w, _p(midx, c_i64p), _p(px, c_dp),
                     _p(py, c_dp), _p(dx, c_dp), _p(dy, c_dp), n, float(cell), float(max_range),
                     _p(out, c_dp), _p(cells, c_i64p))
    return (out, cells) if return_cells else out


def count_dda_cells(occ, map_idx, px, py, dirx, diry, cell, max_range):
    """Cells entered by the pure DDA (``_cy.pyx:89-105`` without the EDT jump):
    the algorithmic unit of the ray-cells/s metric."""
    lib = load_lib()
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    m, h, w = occ.shape
    midx = np.ascontiguousarray(map_idx, dtype=np.int64)
    px, py, dx, dy = (np.ascontiguousarray(a, dtype=np.float64) for a in (px, py, dirx, diry))
    out = np.empty(px.shape[0], dtype=np.int64)
    lib.or_count_dda_cells(_p(occ, c_u8p), h, w, _p(midx, c_i64p), _p(px, c_dp), _p(py, c_dp),
                           _p(dx, c_dp), _p(dy, c_dp), px.shape[0], float(cell),
                           float(max_range), _p(out, c_i64p))
    return out


def disc_collides(occ, map_idx, px, py, radius, cell):
    """Restates kernels.disc_collides (``kernels/__init__.py:79-86``, ``_cy.pyx:109-158``)."""
    lib = load_lib()
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    m, h, w = occ.shape
    midx = np.ascontiguousarray(map_idx, dtype=np.int64)
    px, py, r = (np.ascontiguousarray(a, dtype=np.float64) for a in (px, py, radius))
    out = np.empty(px.shape[0], dtype=np.uint8)
    lib.or_disc_collides(_p(occ, c_u8p), h, w, _p(midx, c_i64p), _p(px, c_dp), _p(py, c_dp),
                         _p(r, c_dp), px.shape[0], float(cell), _p(out, c_u8p))
    return out


def edt_cells(occupancy) -> np.ndarray:
    """``gridmap.py:62-71``: scipy EDT of the free space, cell units, float64."""
    from scipy import ndimage
    return ndimage.distance_transform_edt(~np.asarray(occupancy, dtype=bool)).astype(np.float64)


# -- env -------------------------------------------------------------------------

class OracleStep(NamedTuple):
    states: np.ndarray
    rewards: np.ndarray
    dones: np.ndarray
    truncated: np.ndarray
    store_states: np.ndarray
    events: np.ndarray


def _ranges_row(r) -> list:
    return [r.k[0], r.k[1], r.control_interval_s[0], r.control_interval_s[1],
            r.control_delay_steps[0], r.control_delay_steps[1],
            r.v_linear_max_cm_s[0], r.v_linear_max_cm_s[1],
            r.v_angular_max_rad_s[0], r.v_angular_max_rad_s[1],
            r.lidar_noise_std_cm[0], r.lidar_noise_std_cm[1]]


class OracleVecEnv:
    """C-oracle VecEnv.  ``maps``/``ranges``/``config`` are duck-typed like the
    reference's GridMap / DiversityRanges / EnvConfig (``sim/params.py``)."""

    class EpisodeTerminated(RuntimeError):
        pass

    def __init__(self, maps, n_copies, ranges, config, map_index=None, auto_reset=True,
                 env_id_offset=0):
        lib = load_lib()
        self._lib = lib
        self.n = int(n_copies)
        lid = config.lidar
        self.n_beams = int(lid.n_beams)
        self.D = 5 + self.n_beams
        if map_index is None:
            map_index = [(env_id_offset + i) % len(maps) for i in range(self.n)]
        self.map_index = np.ascontiguousarray(map_index, dtype=np.int64)
        if not isinstance(ranges, (list, tuple)):
            ranges = [ranges] * self.n
        self._ranges = np.ascontiguousarray([_ranges_row(r) for r in ranges], dtype=np.float64)
        first = maps[0]
        h, w = first.occupancy.shape
        self._occ = np.ascontiguousarray(np.stack([m.occupancy for m in maps]).astype(np.uint8))
        self._edt = np.ascontiguousarray(np.stack([edt_cells(m.occupancy) for m in maps]))
        self._gx = np.array([m.goal_center[0] for m in maps], dtype=np.float64)
        self._gy = np.array([m.goal_center[1] for m in maps], dtype=np.float64)
        self._gr = np.array([m.goal_radius_cm for m in maps], dtype=np.float64)
        pd = float(config.max_planning_dist_cm)
        self._pd = np.array([pd if pd > 0 else math.hypot(m.width_cm, m.height_cm)
                             for m in maps], dtype=np.float64)
        self._spawn = np.ascontiguousarray([list(m.spawn_region) for m in maps], dtype=np.float64)
        self._offsets = np.ascontiguousarray(
            np.linspace(-lid.fov_rad / 2.0, lid.fov_rad / 2.0, self.n_beams), dtype=np.float64)
        table = np.ascontiguousarray(np.asarray(config.action_table, dtype=np.float64).ravel())
        self._table = table
        self.n_actions = len(config.action_table)
        self.cell = float(first.cell_size_cm)
        self._h = lib.or_env_create(
            self.n_beams, float(lid.max_range_cm), float(config.robot_radius_cm),
            float(config.obstacle_penalty_range_cm), int(config.timeout_steps),
            int(config.spawn_attempts), int(bool(auto_reset)), self.n_actions,
            _p(table, c_dp), len(maps), h, w, self.cell, _p(self._occ, c_u8p),
            _p(self._edt, c_dp), _p(self._gx, c_dp), _p(self._gy, c_dp), _p(self._gr, c_dp),
            _p(self._pd, c_dp), _p(self._spawn, c_dp), self.n, _p(self.map_index, c_i64p),
            _p(self._ranges, c_dp), _p(self._offsets, c_dp), int(env_id_offset))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.or_env_destroy(h)
            self._h = None

    def _check(self, rc):
        if rc == 0:
            return
        if rc == 2:
            raise ValueError("action index out of range")
        if rc == 3:
            raise OracleVecEnv.EpisodeTerminated("lane finished its episode")
        if rc == 4:
            raise ValueError("no collision-free spawn pose (MapError)")
        raise RuntimeError(f"oracle error {rc}")

    def reset_all(self, seed: int) -> np.ndarray:
        out = np.empty((self.n, self.D), dtype=np.float32)
        self._check(self._lib.or_env_reset_all(self._h, seed, _p(out, c_fp)))
        return out

    def step_batch(self, actions) -> OracleStep:
        a = np.ascontiguousarray(actions, dtype=np.int64)
        if a.shape != (self.n,):
            raise ValueError("bad action shape")
        states = np.empty((self.n, self.D), dtype=np.float32)
        store = np.empty((self.n, self.D), dtype=np.float32)
        rew = np.empty(self.n, dtype=np.float64)
        dones = np.empty(self.n, dtype=np.uint8)
        trunc = np.empty(self.n, dtype=np.uint8)
        ev = np.empty(self.n, dtype=np.int8)
        self._check(self._lib.or_env_step(self._h, _p(a, c_i64p), _p(states, c_fp),
                                          _p(store, c_fp), _p(rew, c_dp), _p(dones, c_u8p),
                                          _p(trunc, c_u8p), _p(ev, c_i8p)))
        return OracleStep(states, rew, dones.astype(bool), trunc.astype(bool), store, ev)

    def pose(self) -> dict:
        n = self.n
        out = {k: np.empty(n) for k in ("x", "y", "heading", "v_linear", "v_angular")}
        sc = np.empty(n, dtype=np.int64)
        ctr = np.empty(n, dtype=np.uint64)
        self._lib.or_env_get_pose(self._h, *(_p(out[k], c_dp) for k in
                                             ("x", "y", "heading", "v_linear", "v_angular")),
                                  _p(sc, c_i64p), _p(ctr, c_u64p))
        out["step_count"] = sc
        out["rng_ctr"] = ctr
        return out

    def stats(self) -> dict:
        n = self.n
        eps = np.empty(n, dtype=np.int64)
        arr = np.empty(n, dtype=np.int64)
        rs = np.empty(n)
        fe = np.empty(n, dtype=np.int8)
        fr = np.empty(n)
        fs = np.empty(n, dtype=np.int64)
        rec = np.empty(256)
        cnt = np.zeros(1, dtype=np.int64)
        self._lib.or_env_get_stats(self._h, _p(eps, c_i64p), _p(arr, c_i64p), _p(rs, c_dp),
                                   _p(fe, c_i8p), _p(fr, c_dp), _p(fs, c_i64p), _p(rec, c_dp),
                                   _p(cnt, c_i64p))
        c = int(cnt[0])
        if c <= 256:
            recent = rec[:c].copy()
        else:
            recent = np.roll(rec, -(c % 256))
        return dict(episodes=eps, arrivals=arr, return_sum=rs, first_event=fe,
                    first_return=fr, first_steps=fs, recent_returns=recent)

    def reset_stats(self):
        self._lib.or_env_reset_stats(self._h)

    def cells(self) -> dict:
        """Hit cells (iy*W+ix, -1 none) of the last step's post-step scans
        (``store``) and of the scans behind the current states rows
        (``state``), plus ``last_scan`` (cm, ``core.py:97``); (N, R) each."""
        k = (self.n, self.n_beams)
        store = np.empty(k, dtype=np.int64)
        last = np.empty(k, dtype=np.int64)
        ls = np.empty(k, dtype=np.float64)
        self._lib.or_env_get_cells(self._h, _p(store, c_i64p), _p(last, c_i64p), _p(ls, c_dp))
        return {"store": store, "state": last, "last_scan": ls}


class ShardedOracle:
    """``OracleVecEnv`` over ``shards`` contiguous env-id ranges stepped on
    host threads (the C calls release the GIL).  Lanes are independent and
    keyed by global env id, so this is exactly the
    single-process oracle, at host-core speed for BASELINE-size parity runs."""

    def __init__(self, maps, n_copies, ranges, config, env_id_offset=0, shards=None):
        from concurrent.futures import ThreadPoolExecutor
        n = int(n_copies)
        shards = max(1, min(int(shards or os.cpu_count() or 1), n))
        cuts = [n * k // shards for k in range(shards + 1)]
        self.cuts = cuts
        self.n = n
        self.parts = [OracleVecEnv(maps, cuts[k + 1] - cuts[k], ranges, config,
                                   env_id_offset=env_id_offset + cuts[k])
                      for k in range(shards)]
        self._pool = ThreadPoolExecutor(shards)

    def _map(self, fn):
        return list(self._pool.map(fn, range(len(self.parts))))

    def reset_all(self, seed):
        return np.concatenate(self._map(lambda k: self.parts[k].reset_all(seed)))

    def step_batch(self, actions) -> OracleStep:
        a = np.ascontiguousarray(actions, dtype=np.int64)
        outs = self._map(lambda k: self.parts[k].step_batch(a[self.cuts[k]:self.cuts[k + 1]]))
        return OracleStep(*(np.concatenate([o[f] for o in outs]) for f in range(6)))

    def pose(self) -> dict:
        ps = self._map(lambda k: self.parts[k].pose())
        return {f: np.concatenate([p[f] for p in ps]) for f in ps[0]}

    def cells(self) -> dict:
        cs = self._map(lambda k: self.parts[k].cells())
        return {f: np.concatenate([c[f] for c in cs]) for f in cs[0]}

    def stats(self) -> dict:
        """Per-copy counters (the recent-returns deque is per shard: not merged)."""
        ss = self._map(lambda k: self.parts[k].stats())
        return {f: np.concatenate([s[f] for s in ss])
                for f in ("episodes", "arrivals", "return_sum", "first_event", "first_return",
                          "first_steps")}

    def close(self):
        self._pool.shutdown()


# -- replay ----------------------------------------------------------------------

class ReplayOracle:
    """Restates ``ReplayBuffer`` (``replay.py:31-87``): FIFO ring, uniform
    with-replacement sampling through a Philox ``integers`` stream."""

    def __init__(self, capacity: int, state_dim: int):
        self.capacity = capacity
        self.s = np.zeros((capacity, state_dim), np.float32)
        self.a = np.zeros(capacity, np.int64)
        self.r = np.zeros(capacity, np.float32)
        self.s2 = np.zeros((capacity, state_dim), np.float32)
        self.d = np.zeros(capacity, bool)
        self.cursor = 0
        self.size = 0

    def __len__(self):
        return self.size

    def append_batch(self, s, a, r, s2, d):
        n = len(s)
        if n > self.capacity:
            raise ValueError("batch exceeds capacity")
        idx = (self.cursor + np.arange(n)) % self.capacity  # replay.py:60
        self.s[idx] = np.asarray(s, np.float32)
        self.a[idx] = np.asarray(a, np.int64)
        self.r[idx] = np.asarray(r, np.float32)
        self.s2[idx] = np.asarray(s2, np.float32)
        self.d[idx] = np.asarray(d, bool)
        self.cursor = (self.cursor + n) % self.capacity
        self.size = min(self.size + n, self.capacity)

    def sample_indices(self, batch_size: int, rng) -> np.ndarray:
        if self.size < batch_size:
            raise RuntimeError("BufferNotReady")
        return rng.integers(0, self.size, batch_size)  # replay.py:76

    def sample(self, batch_size: int, rng):
        idx = self.sample_indices(batch_size, rng)
        return (self.s[idx].copy(), self.a[idx].copy(), self.r[idx].copy(),
                self.s2[idx].copy(), self.d[idx].copy()), idx


# -- the real reference (oracle/_ref) ----------------------------------------------

def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_PATH, "color_rl"))


def import_reference(state_dim: int | None = None):
    """Import the built, unmodified reference from oracle/_ref.  For R != 27 the
    hard-coded ``STATE_DIM = 32`` (``sim/core.py:32``, re-imported at
    ``vecenv.py:18``) is patched to 5 + R, as SURVEY 8(c) prescribes."""
    import sys
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import color_rl  # noqa: F401
    import color_rl.sim.core as core
    import color_rl.vecenv as vecenv
    if state_dim is not None:
        core.STATE_DIM = state_dim
        vecenv.STATE_DIM = state_dim
    return color_rl
