"""Drop-in ``VecEnv``: N lockstep Sparrow copies stepped by one CUDA launch.

API of the reference ``color_rl.vecenv.VecEnv`` (``vecenv.py:61-145``):
``reset_all(seed)``, ``step_batch(actions) -> StepBatch``,
``snapshot_stats(reset)``, ``first_episode_outcomes()``,
``all_first_episodes_done``, ``n_copies``, ``map_index``, ``sim``.

Returned arrays are CUDA tensors (the paper's conversion-free data flow,
``PAPER.md:237``) with the reference's dtypes: states/store_states float32
``(N, 5+R)``, rewards float64, dones/truncated bool, events int8.  Each call
returns fresh tensors.

Randomness: lane i draws from the Philox stream (seed, env_id_offset + i)
 instead of ``SeedSequence(seed).spawn(N)``; a
shard of a larger run (``env_id_offset``) therefore reproduces exactly the
lanes of a single-GPU run.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import NamedTuple, Sequence

import numpy as np

from paper_2305_04180_b200 import _lib
from paper_2305_04180_b200.sim import (
    DiversityRanges,
    EnvConfig,
    Event,
    EpisodeTerminated,
    MapError,
)


class StepBatch(NamedTuple):  # vecenv.py:24-30
    states: "torch.Tensor"        # (N, D) float32, post-reset rows for finished copies
    rewards: "torch.Tensor"       # (N,) float64
    dones: "torch.Tensor"         # (N,) bool; collision/arrival only
    truncated: "torch.Tensor"     # (N,) bool; timeouts
    store_states: "torch.Tensor"  # (N, D) float32; true s' rows
    events: "torch.Tensor"        # (N,) int8 Event codes


class HostStep(NamedTuple):
    """Page-locked buffers of ``VecEnv.step_host``."""
    actions: "torch.Tensor"    # (N,) int64
    out: StepBatch             # views into h_flat, StepBatch dtypes
    h_flat: "torch.Tensor"     # the sp_env_step_host output block


@dataclass
class CopyStats:  # vecenv.py:33-41
    episodes: int = 0
    arrivals: int = 0
    return_sum: float = 0.0

    @property
    def arrival_rate(self):
        return self.arrivals / self.episodes if self.episodes else None


@dataclass
class StatsSnapshot:  # vecenv.py:44-58
    per_copy: list
    episodes: int
    arrivals: int
    return_sum: float
    recent_returns: list = field(default_factory=list)

    @property
    def arrival_rate(self):
        return self.arrivals / self.episodes if self.episodes else None

    @property
    def mean_return(self):
        return self.return_sum / self.episodes if self.episodes else None


def _map_desc(m, config) -> tuple:
    occ = np.ascontiguousarray(np.asarray(m.occupancy, dtype=bool).astype(np.uint8))
    desc = _lib.SpMapDesc()
    desc.n_rows, desc.n_cols = occ.shape
    desc.cell_cm = float(m.cell_size_cm)
    desc.occupancy = occ.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    desc.goal_x, desc.goal_y = (float(v) for v in m.goal_center)
    desc.goal_radius = float(m.goal_radius_cm)
    for i, v in enumerate(m.spawn_region):
        desc.spawn[i] = float(v)
    pd = float(getattr(config, "max_planning_dist_cm", 0.0))
    desc.planning_dist = pd if pd > 0 else math.hypot(m.width_cm, m.height_cm)
    return desc, occ


def _ranges_struct(r) -> "_lib.SpRanges":
    s = _lib.SpRanges()
    s.k[:] = [float(v) for v in r.k]
    s.dt[:] = [float(v) for v in r.control_interval_s]
    s.delay[:] = [int(v) for v in r.control_delay_steps]
    s.vmax_linear[:] = [float(v) for v in r.v_linear_max_cm_s]
    s.vmax_angular[:] = [float(v) for v in r.v_angular_max_rad_s]
    s.noise_std[:] = [float(v) for v in r.lidar_noise_std_cm]
    return s


class SimView:
    """Read-only view of the device SoA with the reference SimBatch attribute
    names (``sim/core.py:81-108``).  Each attribute read copies to host."""

    _FIELDS = {"x": 0, "y": 1, "heading": 2, "start_x": 5, "start_y": 6, "param_k": 7,
               "param_dt": 8, "param_noise": 12, "rng_ctr": 15, "start_cos": 17,
               "start_sin": 18}

    def __init__(self, env: "VecEnv"):
        self._env = env
        maps = env._maps
        mi = env.map_index
        self.goal_x = np.array([maps[i].goal_center[0] for i in mi])
        self.goal_y = np.array([maps[i].goal_center[1] for i in mi])
        self.goal_radius = np.array([maps[i].goal_radius_cm for i in mi])
        self.planning_dist = np.array([env._plan_dist[i] for i in mi])
        self.map_index = mi
        self.n_lanes = env.n_copies
        self.n_beams = env.n_beams
        self.cell = float(maps[0].cell_size_cm)

    def _read(self, field_id: int) -> np.ndarray:
        return self._env._read_state(field_id)

    def __getattr__(self, name):
        fid = SimView._FIELDS.get(name)
        if fid is None:
            raise AttributeError(name)
        return self._read(fid)

    @property
    def v(self) -> np.ndarray:
        return np.stack([self._read(3), self._read(4)], axis=1)

    @property
    def param_vmax(self) -> np.ndarray:
        return np.stack([self._read(10), self._read(11)], axis=1)

    @property
    def param_delay(self) -> np.ndarray:
        return self._read(9).astype(np.int64)

    @property
    def step_count(self) -> np.ndarray:
        return self._read(13).astype(np.int64)

    @property
    def needs_reset(self) -> np.ndarray:
        return self._read(14).astype(bool)

    @property
    def episode_return(self) -> np.ndarray:
        return self._read(16)

    @property
    def last_scan(self) -> np.ndarray:
        """(N, R) noisy clipped ranges (cm) behind the last returned states rows
        (``core.py:97, 159-161, 206``).  Exact float64 while recording is on
        (``VecEnv.record``); otherwise recovered from those rows' float32
        LiDAR columns (relative error <= 6e-8)."""
        return self._env._last_scan()

    @property
    def params(self) -> list:
        """Per-lane ``SimParams`` of the current episodes (``core.py:104, 126``)."""
        from paper_2305_04180_b200.sim import SimParams
        k, dt, d = self._read(7), self._read(8), self._read(9)
        vl, va, sg = self._read(10), self._read(11), self._read(12)
        return [SimParams(k=float(k[i]), control_interval_s=float(dt[i]),
                          control_delay_steps=int(d[i]), v_linear_max_cm_s=float(vl[i]),
                          v_angular_max_rad_s=float(va[i]), lidar_noise_std_cm=float(sg[i]))
                for i in range(self.n_lanes)]

    @property
    def _pending(self) -> list:
        """Per-lane delay queues of (v_linear, v_angular) targets, oldest first
        (``core.py:106, 156, 176-182``), decoded from the device FIFO."""
        from collections import deque
        return [deque(q) for q in self._env.pending_actions()]


class VecEnv:
    def __init__(self, maps: Sequence, n_copies: int,
                 ranges: DiversityRanges | Sequence[DiversityRanges] | None = None,
                 config: EnvConfig | None = None, map_index: Sequence[int] | None = None,
                 auto_reset: bool = True, kernel_backend=None, *, device=None,
                 env_id_offset: int = 0, check_actions: bool = True):
        if kernel_backend not in (None, "cuda", "auto", "active"):
            raise ValueError(f"kernel backend {kernel_backend!r}: this build has only 'cuda'")
        if n_copies < 1:
            raise ValueError("need at least one copy")  # vecenv.py:66-67
        import torch
        self._torch = torch
        self.device = _lib.require_cuda(device)
        lib = _lib.load()
        self._lib = lib
        self.n_copies = int(n_copies)
        self.auto_reset = bool(auto_reset)
        self.check_actions = bool(check_actions)
        self.config = config or EnvConfig()
        self._maps = list(maps)
        if not self._maps:
            raise ValueError("need at least one map")
        first = self._maps[0]
        for m in self._maps:
            if (np.asarray(m.occupancy).shape != np.asarray(first.occupancy).shape
                    or m.cell_size_cm != first.cell_size_cm):
                raise MapError("all maps in one batch must share grid shape and cell size")
        if map_index is None:
            map_index = [(env_id_offset + i) % len(self._maps) for i in range(self.n_copies)]
        self.map_index = np.asarray(map_index, dtype=np.int64)
        if self.map_index.shape != (self.n_copies,):
            raise ValueError("need one map index per copy")
        if self.map_index.min() < 0 or self.map_index.max() >= len(self._maps):
            raise ValueError("map_index out of range")
        if isinstance(ranges, (list, tuple)):
            rl = list(ranges)
            if len(rl) != self.n_copies:
                raise ValueError("need one DiversityRanges per lane")
        else:
            rl = [ranges or DiversityRanges()]
        lid = self.config.lidar
        self.n_beams = int(lid.n_beams)
        self.state_dim = 5 + self.n_beams
        table = [tuple(p) for p in self.config.action_table]
        self.n_actions = len(table)

        cfg = _lib.SpConfig()
        cfg.n_beams = self.n_beams
        cfg.max_range_cm = float(lid.max_range_cm)
        cfg.robot_radius_cm = float(self.config.robot_radius_cm)
        cfg.timeout_steps = int(self.config.timeout_steps)
        cfg.proximity_cm = float(self.config.obstacle_penalty_range_cm)
        cfg.n_actions = self.n_actions
        for i, (v, w) in enumerate(table):
            cfg.action_table[2 * i] = float(v)
            cfg.action_table[2 * i + 1] = float(w)
        cfg.spawn_attempts = int(self.config.spawn_attempts)
        cfg.auto_reset = 1 if self.auto_reset else 0
        self._offsets = np.ascontiguousarray(lid.beam_offsets(), dtype=np.float64)
        cfg.beam_offsets = self._offsets.ctypes.data_as(_lib.c_dp)

        descs = (_lib.SpMapDesc * len(self._maps))()
        keep = []
        self._plan_dist = []
        for i, m in enumerate(self._maps):
            desc, occ = _map_desc(m, self.config)
            descs[i] = desc
            keep.append(occ)
            self._plan_dist.append(desc.planning_dist)
        rarr = (_lib.SpRanges * len(rl))(*[_ranges_struct(r) for r in rl])
        midx = np.ascontiguousarray(self.map_index, dtype=np.int32)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            rc = lib.sp_env_create(ctypes.byref(cfg), descs, len(self._maps), self.n_copies,
                                   midx.ctypes.data_as(_lib.c_i32p), rarr, len(rl),
                                   int(env_id_offset), self.device.index, ctypes.byref(handle))
        _lib.check(rc, "sp_env_create")
        self._h = handle
        self.env_id_offset = int(env_id_offset)
        self._sim = None
        self._seeded = False
        self._last_states = None  # the states rows last returned (SimView.last_scan)
        self._rec = None          # recording buffers (record())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._lib.sp_env_destroy(h)
            except Exception:  # noqa: BLE001 (interpreter shutdown)
                pass
            self._h = None

    # -- helpers --------------------------------------------------------------
    def _stream(self) -> int:
        return self._torch.cuda.current_stream(self.device).cuda_stream

    def _read_state(self, field_id: int) -> np.ndarray:
        out = np.empty(self.n_copies, dtype=np.float64)
        _lib.check(self._lib.sp_env_read_state(self._h, field_id, out.ctypes.data_as(_lib.c_dp),
                                               self._stream()), "read_state")
        return out

    def _actions_to_device(self, actions):
        torch = self._torch
        if isinstance(actions, torch.Tensor):
            if actions.shape != (self.n_copies,):
                raise ValueError(f"expected {self.n_copies} actions, got shape {tuple(actions.shape)}")
            a = actions.to(device=self.device, dtype=torch.int64)
            if self.check_actions and a.device.type == "cuda":
                lo, hi = torch.aminmax(a)
                if int(lo) < 0 or int(hi) >= self.n_actions:
                    raise ValueError("action index out of range")
            return a.contiguous()
        a = np.asarray(actions, dtype=np.int64)
        if a.shape != (self.n_copies,):
            raise ValueError(f"expected {self.n_copies} actions, got shape {a.shape}")
        if a.min() < 0 or a.max() >= self.n_actions:  # core.py:169-170
            raise ValueError("action index out of range")
        return torch.from_numpy(a).to(self.device, non_blocking=False)

    def check(self) -> None:
        """Raise any error a device-side step flagged (invalid device action,
        missing spawn pose); synchronizes the current stream."""
        err_env = ctypes.c_int64(0)
        _lib.check(self._lib.sp_env_check(self._h, self._stream(), ctypes.byref(err_env)),
                   "step")

    # -- lifecycle ----------------------------------------------------------------
    def reset_all(self, seed: int):
        torch = self._torch
        states = torch.empty((self.n_copies, self.state_dim), dtype=torch.float32,
                             device=self.device)
        _lib.check(self._lib.sp_env_reset_all(self._h, int(seed) & 0xFFFFFFFFFFFFFFFF,
                                              states.data_ptr(), self._stream()), "reset_all")
        self._seeded = True
        self.check()  # MapError if a lane found no spawn pose (core.py:144-147)
        self._last_states = states
        return states

    def step_batch(self, actions, out: StepBatch | None = None) -> StepBatch:
        if not self._seeded:
            raise EpisodeTerminated("reset_all(seed) must be called before stepping")
        torch = self._torch
        a = self._actions_to_device(actions)
        if not self.auto_reset:
            flag = ctypes.c_int32(0)
            _lib.check(self._lib.sp_env_any_needs_reset(self._h, self._stream(),
                                                        ctypes.byref(flag)), "step")
            if flag.value:
                raise EpisodeTerminated("some lanes finished their episode; reset before stepping")
        if out is None:
            n, d = self.n_copies, self.state_dim
            dev = self.device
            out = StepBatch(
                torch.empty((n, d), dtype=torch.float32, device=dev),
                torch.empty(n, dtype=torch.float64, device=dev),
                torch.empty(n, dtype=torch.bool, device=dev),
                torch.empty(n, dtype=torch.bool, device=dev),
                torch.empty((n, d), dtype=torch.float32, device=dev),
                torch.empty(n, dtype=torch.int8, device=dev))
        self._launch_step(a, out)
        self._last_states = out.states
        return out

    def _launch_step(self, a, out: StepBatch) -> None:
        """sp_env_step through the torch extension (tensor checks in C++,
        ATen's current stream), or ctypes when it is not built."""
        rb = out.states.numel() * out.states.element_size()
        s0, s1 = out.states.data_ptr(), out.store_states.data_ptr()
        if s0 < s1 + rb and s1 < s0 + rb:  # the C-ABI's own check, before the op's alias rules
            raise ValueError("states and store_states must not overlap")
        ops = _lib.torch_ops()
        if ops is not None:
            try:
                ops.env_step(self._h.value, a, out.states, out.store_states, out.rewards,
                             out.dones, out.truncated, out.events)
            except RuntimeError as exc:  # the C-ABI status, mapped like ctypes calls
                _lib.check(_lib.status_of(exc), "step")
                raise
            return
        _lib.check(self._lib.sp_env_step(self._h, a.data_ptr(), out.states.data_ptr(),
                                         out.store_states.data_ptr(), out.rewards.data_ptr(),
                                         out.dones.data_ptr(), out.truncated.data_ptr(),
                                         out.events.data_ptr(), self._stream()), "step")

    def new_batch(self) -> StepBatch:
        """Device output tensors for ``step_batch(actions, out=...)``."""
        torch = self._torch
        n, d, dev = self.n_copies, self.state_dim, self.device
        return StepBatch(torch.empty((n, d), dtype=torch.float32, device=dev),
                         torch.empty(n, dtype=torch.float64, device=dev),
                         torch.empty(n, dtype=torch.bool, device=dev),
                         torch.empty(n, dtype=torch.bool, device=dev),
                         torch.empty((n, d), dtype=torch.float32, device=dev),
                         torch.empty(n, dtype=torch.int8, device=dev))

    def host_buffers(self) -> "HostStep":
        """Page-locked host buffers for ``step_host``. The outputs are views into
        one flat block in ``sp_env_step_host``'s layout (include/sparrow.h)."""
        torch = self._torch
        n, d = self.n_copies, self.state_dim
        total = int(self._lib.sp_env_host_out_bytes(self._h))
        h_flat = torch.empty(total, dtype=torch.uint8).pin_memory()
        fields = ((n, torch.float64, 8), ((n, d), torch.float32, 4), ((n, d), torch.float32, 4),
                  (n, torch.bool, 1), (n, torch.bool, 1), (n, torch.int8, 1))
        views, off = [], 0
        for sh, dt, sz in fields:
            nb = int(np.prod(sh)) * sz
            views.append(h_flat[off:off + nb].view(dt).view(sh))
            off += nb
        assert off == total
        r, st, ss, dn, tr, ev = views
        return HostStep(torch.empty(n, dtype=torch.int64).pin_memory(),
                        StepBatch(st, r, dn, tr, ss, ev), h_flat)

    def step_host(self, actions, bufs: "HostStep | None" = None) -> StepBatch:
        """The reference's numpy ``step_batch`` (vecenv.py:94-116): host actions
        in, a StepBatch of numpy arrays out, through ``sp_env_step_host``: one
        H2D copy, the fused step and one D2H copy of a flat page-locked block
        in a single C call that returns after the stream synchronized. The
        arrays are views of ``bufs`` (default: buffers owned by this env), so the
        next call overwrites them. ``actions`` may already be ``bufs.actions``."""
        if not self._seeded:
            raise EpisodeTerminated("reset_all(seed) must be called before stepping")
        torch = self._torch
        if bufs is None:
            if getattr(self, "_host_bufs", None) is None:
                self._host_bufs = self.host_buffers()
            bufs = self._host_bufs
        if not (isinstance(actions, torch.Tensor) and actions.data_ptr() == bufs.actions.data_ptr()):
            a = np.asarray(actions.cpu() if isinstance(actions, torch.Tensor) else actions)
            if a.shape != (self.n_copies,):
                raise ValueError(f"expected {self.n_copies} actions, got shape {a.shape}")
            np.copyto(bufs.actions.numpy(), a, casting="same_kind")
        # sp_env_step_host checks the actions on the host before it launches
        # (SP_EACTION -> ValueError, nothing stepped: core.py:169-170); the
        # no-auto-reset path checks them here too, because the reference
        # raises for bad actions before it raises for lanes awaiting a reset
        if self.check_actions and not self.auto_reset:
            av = bufs.actions.numpy()
            if av.min() < 0 or av.max() >= self.n_actions:  # core.py:169-170
                raise ValueError("action index out of range")
        if not self.auto_reset:
            flag = ctypes.c_int32(0)
            _lib.check(self._lib.sp_env_any_needs_reset(self._h, self._stream(),
                                                        ctypes.byref(flag)), "step")
            if flag.value:
                raise EpisodeTerminated("some lanes finished their episode; reset before stepping")
        _lib.check(self._lib.sp_env_step_host(self._h, bufs.actions.data_ptr(),
                                              bufs.h_flat.data_ptr(), self._stream()), "step")
        return StepBatch(*(t.numpy() for t in bufs.out))

    def step_device(self, actions_ptr: int, out: StepBatch) -> None:
        """Raw launch on pre-validated device actions (benchmarks, CUDA graphs)."""
        _lib.check(self._lib.sp_env_step(self._h, actions_ptr, out.states.data_ptr(),
                                         out.store_states.data_ptr(), out.rewards.data_ptr(),
                                         out.dones.data_ptr(), out.truncated.data_ptr(),
                                         out.events.data_ptr(), self._stream()), "step")

    def reset_lanes(self, mask):
        """SimBatch.reset_lane (core.py:114-161) for every lane with mask[i]
        set, continuing each lane's stream (the manual reset a caller needs
        with auto_reset=False).  Returns the fresh (N, D) state rows (rows of
        unmasked lanes are left unspecified)."""
        torch = self._torch
        m = torch.as_tensor(np.asarray(mask, dtype=np.uint8) if not isinstance(mask, torch.Tensor)
                            else mask.to(torch.uint8)).to(self.device).reshape(-1).contiguous()
        if m.numel() != self.n_copies:
            raise ValueError("need one mask entry per copy")
        states = torch.empty((self.n_copies, self.state_dim), dtype=torch.float32,
                             device=self.device)
        _lib.check(self._lib.sp_env_reset_lanes(self._h, m.data_ptr(), states.data_ptr(),
                                                self._stream()), "reset_lanes")
        self.check()
        if self._last_states is not None and self._last_states.shape == states.shape:
            keep = self._last_states.clone()
            keep[m.bool()] = states[m.bool()]
            self._last_states = keep
        else:
            self._last_states = states
        return states

    def place(self, field: str, values) -> None:
        """Overwrite a pose field for every lane (test hook; the reference tests
        poke SimBatch arrays the same way, test_env.py:37-42)."""
        ids = {"x": 0, "y": 1, "heading": 2, "v_linear": 3, "v_angular": 4, "start_x": 5,
               "start_y": 6, "start_cos": 17, "start_sin": 18}
        v = np.ascontiguousarray(np.broadcast_to(np.asarray(values, dtype=np.float64),
                                                 (self.n_copies,)))
        _lib.check(self._lib.sp_env_write_state(self._h, ids[field], v.ctypes.data_as(_lib.c_dp),
                                                self._stream()), "place")

    # -- recording (parity / inspection) -------------------------------------
    def record(self, on: bool = True) -> None:
        """Make every following launch also record, per row and beam, the
        occupied cell each LiDAR ray stopped in (post-step scan and the scan
        behind the states rows) and the noisy float64 ranges behind the states
        rows (``sp_env_set_recording``).  Off by default: it costs a kernel
        variant with a few extra stores per ray."""
        torch = self._torch
        if on:
            n, R = self.n_copies, self.n_beams
            dev = self.device
            self._rec = {"hit_store": torch.full((n, R), -2, dtype=torch.int32, device=dev),
                         "hit_state": torch.full((n, R), -2, dtype=torch.int32, device=dev),
                         "scan_state": torch.zeros((n, R), dtype=torch.float64, device=dev)}
            ptrs = [self._rec[k].data_ptr() for k in ("hit_store", "hit_state", "scan_state")]
        else:
            self._rec = None
            ptrs = [None, None, None]
        _lib.check(self._lib.sp_env_set_recording(self._h, *ptrs), "record")

    def recorded(self) -> dict:
        """The recording buffers (device tensors, overwritten by the next launch):
        ``hit_store`` / ``hit_state`` int32 (N, R) cells iy*W+ix or -1,
        ``scan_state`` float64 (N, R) cm."""
        if self._rec is None:
            raise RuntimeError("recording is off: call record() before stepping")
        return self._rec

    def _last_scan(self) -> np.ndarray:
        if self._rec is not None:
            return self._rec["scan_state"].cpu().numpy()
        if self._last_states is None:
            return np.full((self.n_copies, self.n_beams), float(self.config.lidar.max_range_cm))
        cols = self._last_states[:, 5:].double().cpu().numpy()
        return cols * float(self.config.lidar.max_range_cm)

    def pending_actions(self) -> list:
        """Per-lane tuples of pending (v_linear, v_angular) targets, oldest
        first: the delay queue ``SimBatch._pending`` (``core.py:156, 176-182``)."""
        n = self.n_copies
        words = np.empty((n, 4), dtype=np.uint64)
        _lib.check(self._lib.sp_env_read_fifo(self._h, words.ctypes.data, self._stream()),
                   "read_fifo")
        delay = self._read_state(9).astype(np.int64)
        table = [tuple(float(v) for v in p) for p in self.config.action_table]
        out = []
        for i in range(n):
            q = []
            for k in range(int(delay[i]) - 1, -1, -1):  # nibble k = issued k steps ago
                code = int((int(words[i, k >> 4]) >> (4 * (k & 15))) & 15)
                q.append((0.0, 0.0) if code == 15 else table[code])
            out.append(tuple(q))
        return out

    # -- reporting -------------------------------------------------------------
    def _per_copy_arrays(self) -> dict:
        n = self.n_copies
        eps = np.empty(n, np.int64)
        arr = np.empty(n, np.int64)
        rs = np.empty(n, np.float64)
        fe = np.empty(n, np.int8)
        fr = np.empty(n, np.float64)
        fs = np.empty(n, np.int64)
        _lib.check(self._lib.sp_env_stats_read(
            self._h, eps.ctypes.data_as(_lib.c_i64p), arr.ctypes.data_as(_lib.c_i64p),
            rs.ctypes.data_as(_lib.c_dp), fe.ctypes.data_as(_lib.c_i8p),
            fr.ctypes.data_as(_lib.c_dp), fs.ctypes.data_as(_lib.c_i64p), self._stream()),
            "stats")
        return dict(episodes=eps, arrivals=arr, return_sum=rs, first_event=fe,
                    first_return=fr, first_steps=fs)

    def recent_returns(self) -> list:
        buf = np.empty(256, np.float64)
        n = ctypes.c_int32(0)
        _lib.check(self._lib.sp_env_recent_returns(self._h, buf.ctypes.data_as(_lib.c_dp),
                                                   ctypes.byref(n), self._stream()), "stats")
        return buf[: n.value].tolist()

    def recent_returns_keyed(self):
        """(keys, returns) of the last <= 256 episode returns, keys =
        (step << 32) | global env id in append order (dist.merge_recent_returns)."""
        buf = np.empty(256, np.float64)
        keys = np.empty(256, np.uint64)
        n = ctypes.c_int32(0)
        _lib.check(self._lib.sp_env_recent_returns_keyed(
            self._h, buf.ctypes.data_as(_lib.c_dp), keys.ctypes.data, ctypes.byref(n),
            self._stream()), "stats")
        return keys[: n.value].copy(), buf[: n.value].copy()

    def snapshot_stats(self, reset: bool = False) -> StatsSnapshot:  # vecenv.py:120-132
        self.check()
        st = self._per_copy_arrays()
        per_copy = [CopyStats(int(e), int(a), float(r))
                    for e, a, r in zip(st["episodes"], st["arrivals"], st["return_sum"])]
        snap = StatsSnapshot(per_copy=per_copy, episodes=int(st["episodes"].sum()),
                             arrivals=int(st["arrivals"].sum()),
                             return_sum=sum(c.return_sum for c in per_copy),
                             recent_returns=self.recent_returns())
        if reset:
            _lib.check(self._lib.sp_env_stats_reset(self._h, 1, self._stream()), "stats")
        return snap

    def stats_totals(self):
        """Device tensor [episodes, arrivals, return_sum] (float64) -- the
        payload of the multi-GPU all-reduce (see paper_2305_04180_b200.dist)."""
        out = self._torch.empty(3, dtype=self._torch.float64, device=self.device)
        _lib.check(self._lib.sp_env_stats_totals(self._h, out.data_ptr(), self._stream()),
                   "stats")
        return out

    def first_episode_outcomes(self) -> list:  # vecenv.py:134-137
        st = self._per_copy_arrays()
        return [None if e < 0 else (Event(int(e)), float(r), int(s))
                for e, r, s in zip(st["first_event"], st["first_return"], st["first_steps"])]

    @property
    def all_first_episodes_done(self) -> bool:
        return self.first_pending() == 0

    def first_pending(self) -> int:
        """Copies whose first episode since reset_all is still running: a
        device count and one 8-byte read (``sp_env_first_pending``)."""
        c = ctypes.c_int64(0)
        _lib.check(self._lib.sp_env_first_pending(self._h, ctypes.byref(c), self._stream()),
                   "first_pending")
        return int(c.value)

    @property
    def sim(self) -> SimView:
        if self._sim is None:
            self._sim = SimView(self)
        return self._sim

    def launch_info(self) -> dict:
        smem = ctypes.c_int64(0)
        thr = ctypes.c_int32(0)
        ctas = ctypes.c_int32(0)
        self._lib.sp_env_map_info(self._h, None, ctypes.byref(smem), ctypes.byref(thr),
                                  ctypes.byref(ctas))
        return {"smem_bytes": smem.value, "threads_per_cta": thr.value, "ctas": ctas.value}

    def partition(self) -> dict:
        """The step kernel's CTA slot cuts and the SM cycles each CTA took in
        the last step (diagnostics; synchronizes the device)."""
        g = self.launch_info()["ctas"]
        cuts = np.zeros(g + 1, np.int64)
        cyc = np.zeros(g, np.uint32)
        _lib.check(self._lib.sp_env_launch_info(self._h, cuts.ctypes.data_as(_lib.c_i64p),
                                                cyc.ctypes.data), "launch_info")
        return {"cuts": cuts, "cta_cycles": cyc}

    def scan_raw(self, qoff: np.ndarray, x, y, heading, ranges, hit_cell=None) -> None:
        """Raw launch: device float64 x/y/heading already grouped by map
        (``qoff`` host int64 offsets, n_maps + 1), outputs preallocated."""
        qoff = np.ascontiguousarray(qoff, dtype=np.int64)
        _lib.check(self._lib.sp_env_scan(
            self._h, int(x.numel()), qoff.ctypes.data_as(_lib.c_i64p), x.data_ptr(),
            y.data_ptr(), heading.data_ptr(), ranges.data_ptr(),
            hit_cell.data_ptr() if hit_cell is not None else None, self._stream()), "scan")

    def scan(self, x, y, heading, map_of_query=None, return_cells: bool = False):
        """LiDAR ranges (no noise) from the fused step's marcher at caller poses:
        (n, R) float64 [, (n, R) int32 hit cell iy*W+ix or -1]."""
        torch = self._torch
        x = torch.as_tensor(x, dtype=torch.float64, device=self.device).reshape(-1)
        y = torch.as_tensor(y, dtype=torch.float64, device=self.device).reshape(-1)
        h = torch.as_tensor(heading, dtype=torch.float64, device=self.device).reshape(-1)
        n = x.numel()
        if map_of_query is None:
            mq = torch.zeros(n, dtype=torch.int64)
        else:
            mq = torch.as_tensor(np.asarray(map_of_query), dtype=torch.int64).reshape(-1)
        order = torch.argsort(mq, stable=True)
        counts = torch.bincount(mq, minlength=len(self._maps)).numpy()
        qoff = np.zeros(len(self._maps) + 1, dtype=np.int64)
        qoff[1:] = np.cumsum(counts)
        od = order.to(self.device)
        xs, ys, hs = x[od].contiguous(), y[od].contiguous(), h[od].contiguous()
        R = self.n_beams
        rng = torch.empty((n, R), dtype=torch.float64, device=self.device)
        cells = torch.empty((n, R), dtype=torch.int32, device=self.device)
        _lib.check(self._lib.sp_env_scan(self._h, n, qoff.ctypes.data_as(_lib.c_i64p),
                                         xs.data_ptr(), ys.data_ptr(), hs.data_ptr(),
                                         rng.data_ptr(), cells.data_ptr(), self._stream()),
                   "scan")
        out_r = torch.empty_like(rng)
        out_c = torch.empty_like(cells)
        out_r[od] = rng
        out_c[od] = cells
        return (out_r, out_c) if return_cells else out_r
