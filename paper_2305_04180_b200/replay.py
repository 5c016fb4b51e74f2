"""Drop-in ``ReplayBuffer``: a GPU-resident FIFO transition ring.

API of the reference ``color_rl.replay`` (``replay.py:19-87``):
``ReplayBuffer(capacity, state_dim)``, ``append_batch`` (alias ``add``,
the paper's ``Sharer.buffer.add``), ``sample(batch_size, rng)``, ``len()``,
``snapshot()``, ``BufferNotReady``, ``TransitionBatch``.

Columns live in HBM (s, s2: float32 (C, D); a: int64; r: float32; done:
bool) -- 309 B/row at D=37, 309 MB at the paper's 1M capacity.  Appends are
one ring-write launch; samples are one Philox-index + gather launch.

``rng`` is a counter-based stream handle (``PhiloxGenerator``): sample i of a
call draws block ``ctr + i`` of (seed, stream_id, tag 2) and maps it to
``mulhi64(w, size)``; the handle's counter
advances by ``batch_size``.  Any object with ``seed``/``lane``/``ctr``
attributes (the oracle's PhiloxStream) is accepted the same way, and a numpy
``Generator`` is accepted by deriving a seed from it.

Concurrency (replay.py:43,59,71): one appender and one sampler thread.  A
host lock makes each call atomic, and CUDA events order the device work:
a sample waits for the last append, an append waits for the last sample,
so rows are never torn and never come from unwritten slots, even when the
actor and learner run on different streams.
"""

from __future__ import annotations

import ctypes
import threading
from typing import NamedTuple

import numpy as np

from paper_2305_04180_b200 import _lib


class BufferNotReady(RuntimeError):
    """Sampling was requested before enough transitions were stored."""


class TransitionBatch(NamedTuple):  # replay.py:23-28
    states: "torch.Tensor"       # (B, D) float32
    actions: "torch.Tensor"      # (B,) int64
    rewards: "torch.Tensor"      # (B,) float32
    next_states: "torch.Tensor"  # (B, D) float32
    dones: "torch.Tensor"        # (B,) bool


class PhiloxGenerator:
    """Counter-based sampling stream (seed, stream_id); ``ctr`` counts blocks."""

    def __init__(self, seed: int, stream_id: int = 0, ctr: int = 0):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.lane = int(stream_id) & 0xFFFFFFFF
        self.ctr = int(ctr)

    def __repr__(self):
        return f"PhiloxGenerator(seed={self.seed}, stream_id={self.lane}, ctr={self.ctr})"


def _stream_of(rng) -> tuple:
    if hasattr(rng, "seed") and hasattr(rng, "lane") and hasattr(rng, "ctr"):
        return rng
    if isinstance(rng, (int, np.integer)):
        return PhiloxGenerator(int(rng))
    if hasattr(rng, "integers"):  # numpy Generator: derive a stream once, keep it on the object
        g = getattr(rng, "_sparrow_stream", None)
        if g is None:
            g = PhiloxGenerator(int(rng.integers(0, 2**63)))
            try:
                rng._sparrow_stream = g
            except AttributeError:
                pass
        return g
    raise TypeError(f"unsupported rng {type(rng).__name__}")


def _check_out(out: TransitionBatch, b: int, dim: int, dev, torch) -> None:
    want = (((b, dim), torch.float32), ((b,), torch.int64), ((b,), torch.float32),
            ((b, dim), torch.float32), ((b,), torch.bool))
    for t, (shape, dtype) in zip(out, want):
        if (tuple(t.shape) != shape or t.dtype != dtype or t.device != dev
                or not t.is_contiguous()):
            raise ValueError(f"out batch tensor {tuple(t.shape)} {t.dtype} on {t.device}: "
                             f"need contiguous {shape} {dtype} on {dev}")


class ReplayBuffer:
    def __init__(self, capacity: int = 1_000_000, state_dim: int = 32, device=None):
        if capacity < 1:
            raise ValueError("capacity must be positive")
        import torch
        self._torch = torch
        self.device = _lib.require_cuda(device)
        self._lib = _lib.load()
        self.capacity = int(capacity)
        self.state_dim = int(state_dim)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._lib.sp_rb_create(self.capacity, self.state_dim, self.device.index,
                                              ctypes.byref(h)), "ReplayBuffer")
        self._h = h
        self._lock = threading.Lock()
        self._last_append = None
        self._last_sample = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._lib.sp_rb_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None

    def __len__(self) -> int:
        size = ctypes.c_int64(0)
        self._lib.sp_rb_size(self._h, ctypes.byref(size), None)
        return size.value

    # -- helpers --------------------------------------------------------------
    def _dev(self, x, dtype):
        torch = self._torch
        if isinstance(x, torch.Tensor):
            return x.to(device=self.device, dtype=dtype).contiguous()
        return torch.as_tensor(np.asarray(x), dtype=dtype).to(self.device).contiguous()

    def _order_after(self, event):
        torch = self._torch
        if event is not None:
            torch.cuda.current_stream(self.device).wait_event(event)

    def _record(self):
        ev = self._torch.cuda.Event()
        ev.record(self._torch.cuda.current_stream(self.device))
        return ev

    # -- API ---------------------------------------------------------------------
    def append_batch(self, states, actions, rewards, next_states, dones) -> None:
        torch = self._torch
        s = self._dev(states, torch.float32)
        n = s.shape[0]
        if n > self.capacity:  # replay.py:51-52
            raise ValueError(f"batch of {n} exceeds capacity {self.capacity}")
        a = self._dev(actions, torch.int64).reshape(-1)
        if isinstance(rewards, torch.Tensor) and rewards.dtype == torch.float64:
            r, r64 = rewards.to(self.device).contiguous().reshape(-1), 1
        else:
            r, r64 = self._dev(rewards, torch.float32).reshape(-1), 0
        s2 = self._dev(next_states, torch.float32)
        d = self._dev(dones, torch.bool).reshape(-1)
        if not (len(a) == len(r) == len(s2) == len(d) == n):
            raise ValueError("transition fields have mismatched lengths")
        if n and (s.shape[1] != self.state_dim or s2.shape[1] != self.state_dim):
            raise ValueError(f"state rows must have {self.state_dim} columns")
        with self._lock:
            self._order_after(self._last_sample)
            ops = _lib.torch_ops()
            if ops is not None:
                try:
                    ops.rb_append(self._h.value, s, a, r, s2, d)
                except RuntimeError as exc:
                    _lib.check(_lib.status_of(exc), "append_batch")
                    raise
            else:
                _lib.check(self._lib.sp_rb_append(self._h, s.data_ptr(), a.data_ptr(),
                                                  r.data_ptr(), r64, s2.data_ptr(), d.data_ptr(),
                                                  n, _lib.stream_ptr(self.device)),
                           "append_batch")
            self._last_append = self._record()

    add = append_batch  # the paper's Sharer.buffer.add

    def sample(self, batch_size: int, rng, return_indices: bool = False,
               out: TransitionBatch | None = None):
        """Uniform with replacement over the filled slots. Returns fresh tensors,
        or fills ``out`` (contiguous device tensors of the batch shape, e.g. a
        CUDA-graphed learner's static batch) in place."""
        torch = self._torch
        g = _stream_of(rng)
        b, dim, dev = int(batch_size), self.state_dim, self.device
        if out is not None:
            ok = getattr(self, "_out_ok", None)
            if ok is None or ok[0] is not out or ok[1] != b:  # validate each new (out, B) once
                _check_out(out, b, dim, dev, torch)
                self._out_ok = (out, b)
        else:
            out = TransitionBatch(torch.empty((b, dim), dtype=torch.float32, device=dev),
                                  torch.empty(b, dtype=torch.int64, device=dev),
                                  torch.empty(b, dtype=torch.float32, device=dev),
                                  torch.empty((b, dim), dtype=torch.float32, device=dev),
                                  torch.empty(b, dtype=torch.bool, device=dev))
        idx = torch.empty(b, dtype=torch.int64, device=dev)
        with self._lock:
            self._order_after(self._last_append)
            rc = self._lib.sp_rb_sample(self._h, b, g.seed, g.lane, g.ctr, out.states.data_ptr(),
                                        out.actions.data_ptr(), out.rewards.data_ptr(),
                                        out.next_states.data_ptr(), out.dones.data_ptr(),
                                        idx.data_ptr(), _lib.stream_ptr(dev))
            _lib.check(rc, "sample")
            g.ctr += b
            self._last_sample = self._record()
        return (out, idx) if return_indices else out

    def sample_dev(self, batch_size: int, rng, d_ctr, out: TransitionBatch) -> None:
        """Enqueue ``sp_rb_sample_dev``: the draws of ``sample(batch_size, rng)``
        with the first Philox block read from the device counter ``d_ctr``
        (uint64 scalar tensor, advanced by batch_size on the device) and the
        fill level read on the device, so the launch can sit inside a CUDA
        graph. The caller gates on ``len(self) >= batch_size`` and orders the
        stream after appends (``DdqnLearner.update_from``)."""
        g = _stream_of(rng)
        b = int(batch_size)
        ok = getattr(self, "_out_ok", None)
        if ok is None or ok[0] is not out or ok[1] != b:
            _check_out(out, b, self.state_dim, self.device, self._torch)
            self._out_ok = (out, b)
        _lib.check(self._lib.sp_rb_sample_dev(self._h, b, g.seed, g.lane, d_ctr.data_ptr(),
                                              out.states.data_ptr(), out.actions.data_ptr(),
                                              out.rewards.data_ptr(), out.next_states.data_ptr(),
                                              out.dones.data_ptr(), None, _lib.stream_ptr(self.device)),
                   "sample_dev")

    def snapshot(self) -> TransitionBatch:
        """All stored transitions in storage order (replay.py:81-87)."""
        torch = self._torch
        with self._lock:
            n = len(self)
            dim, dev = self.state_dim, self.device
            out = TransitionBatch(torch.empty((n, dim), dtype=torch.float32, device=dev),
                                  torch.empty(n, dtype=torch.int64, device=dev),
                                  torch.empty(n, dtype=torch.float32, device=dev),
                                  torch.empty((n, dim), dtype=torch.float32, device=dev),
                                  torch.empty(n, dtype=torch.bool, device=dev))
            self._order_after(self._last_append)
            if n:
                _lib.check(self._lib.sp_rb_gather(self._h, out.states.data_ptr(),
                                                  out.actions.data_ptr(), out.rewards.data_ptr(),
                                                  out.next_states.data_ptr(),
                                                  out.dones.data_ptr(),
                                                  _lib.stream_ptr(dev)), "snapshot")
            self._last_sample = self._record()
        return out
