"""Actor-Sharer-Learner on the GPU (BASELINE cfg5).

Restates the reference's learner side in torch on the same device as the
environment, so the whole ASL loop runs without host round-trips:

* ``QNet``: the [5+R, 256, 128, 5] ReLU MLP of ``net.py``.
  - He-uniform fan-in init from a numpy Generator, so a given rng yields the
    reference's exact initial weights (``net.py:52-60``).
  - Explicit backprop of the mean Huber(delta=1) loss on the chosen-action
    outputs (``net.py:88-115``).
  - Bias-corrected Adam in the reference's operation order
    (``net.py:141-161``).
  - The ``COLORNET`` checkpoint format (``net.py:178-228``), byte-compatible.
* ``compute_targets`` / ``DdqnLearner``: double-DQN (``ddqn.py:38-77``).
* ``VemSchedule`` / ``select_actions``: per-copy epsilon-greedy
  (``asl/vem.py``).  Draws come from a device-side Philox stream
  (``sp_philox_fill``) with the reference's call order: ``random(n)``, then
  ``integers(0, A, n)``.
* ``TfmConfig`` / ``TfmState``: time-feedback pacing (``asl/tfm.py``).
* ``Sharer``, ``actor_loop``, ``learner_loop``, ``start_session``,
  ``Session``: the two-thread ASL session (``asl/sharer.py``,
  ``asl/loops.py``).  Each thread runs on its own CUDA stream; the GPU
  replay ring orders appends and samples with CUDA events.

Matmuls are plain cuBLAS through torch (library GEMM). TF32 is disabled, so
the fp32 numerics follow the numpy reference to ~1e-6.
"""

from __future__ import annotations

import contextlib
import ctypes
import gc
import io
import math
import struct
import threading
import time
import zlib
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from paper_2305_04180_b200 import _lib
from paper_2305_04180_b200.replay import BufferNotReady, PhiloxGenerator, ReplayBuffer

CHECKPOINT_MAGIC = b"COLORNET"  # net.py:19-20
CHECKPOINT_FORMAT_VERSION = 1
HIDDEN = (256, 128)


class CheckpointError(ValueError):
    """Malformed, truncated, or shape-incompatible checkpoint data."""


class TrainingDiverged(RuntimeError):
    """A non-finite loss appeared during optimization (ddqn.py:68-71)."""


@contextlib.contextmanager
def no_gc():
    """Cyclic garbage collection off for a CUDA graph capture: a collected
    handle of an earlier env or buffer would cudaFree mid-capture, which
    invalidates the capture (torch.cuda.graph collects once before it begins)."""
    was = gc.isenabled()
    gc.disable()
    try:
        yield
    finally:
        if was:
            gc.enable()


def _torch():
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    return torch


# -- Q-network (net.py) -----------------------------------------------------------

class QNet:
    """Weights (fan_in, fan_out) and biases as float32 CUDA tensors + version."""

    def __init__(self, weights, biases, version: int = 0):
        self.weights = list(weights)
        self.biases = list(biases)
        self.version = int(version)

    @property
    def sizes(self) -> tuple:
        return (int(self.weights[0].shape[0]),) + tuple(int(w.shape[1]) for w in self.weights)

    @classmethod
    def init(cls, rng: np.random.Generator, sizes, device=None) -> "QNet":
        """He-style uniform fan-in init, zero biases (net.py:52-60)."""
        torch = _torch()
        dev = _lib.require_cuda(device)
        ws, bs = [], []
        for fan_in, fan_out in zip(sizes[:-1], sizes[1:]):
            bound = np.sqrt(6.0 / fan_in)
            w = rng.uniform(-bound, bound, (fan_in, fan_out)).astype(np.float32)
            ws.append(torch.from_numpy(w).to(dev))
            bs.append(torch.zeros(fan_out, dtype=torch.float32, device=dev))
        return cls(ws, bs)

    @classmethod
    def from_numpy(cls, weights, biases, version=0, device=None) -> "QNet":
        torch = _torch()
        dev = _lib.require_cuda(device)
        return cls([torch.as_tensor(np.asarray(w, np.float32)).to(dev) for w in weights],
                   [torch.as_tensor(np.asarray(b, np.float32)).to(dev) for b in biases], version)

    def copy(self) -> "QNet":
        return QNet([w.clone() for w in self.weights], [b.clone() for b in self.biases],
                    self.version)

    def copy_from(self, other: "QNet") -> None:
        for a, b in zip(self.weights, other.weights):
            a.copy_(b)
        for a, b in zip(self.biases, other.biases):
            a.copy_(b)
        self.version = other.version

    def forward_cached(self, states):
        """Forward pass keeping pre-activations for backprop (net.py:63-74)."""
        torch = _torch()
        h = states.to(torch.float32)
        acts, pre = [h], []
        last = len(self.weights) - 1
        for li, (w, b) in enumerate(zip(self.weights, self.biases)):
            z = torch.addmm(b, h, w)
            pre.append(z)
            h = z if li == last else torch.relu(z)
            acts.append(h)
        return acts, pre

    def forward(self, states):
        """Batched Q-values (B, n_actions) (net.py:77-80)."""
        return self.forward_cached(states)[0][-1]

    # -- checkpoints (net.py:178-228) ----------------------------------------
    # The COLORNET byte layout is the reference's (little-endian): magic,
    # u32 format version, u32 layer count, u32 sizes, then per layer the f32
    # weights (fan_in, fan_out) and f32 biases, then the u64 version.  Here the
    # whole parameter payload crosses PCIe once each way: the device tensors
    # are concatenated on the GPU and read back in one copy; loading validates
    # the header and the exact payload length first, then uploads one buffer
    # and splits it into per-layer views.
    def to_bytes(self) -> bytes:
        torch = _torch()
        sizes = self.sizes
        head = CHECKPOINT_MAGIC + np.array([CHECKPOINT_FORMAT_VERSION, len(sizes), *sizes],
                                           dtype="<u4").tobytes()
        flat = torch.cat([t.reshape(-1) for pair in zip(self.weights, self.biases) for t in pair])
        return (head + flat.cpu().numpy().astype("<f4", copy=False).tobytes()
                + np.array([self.version], dtype="<u8").tobytes())

    @classmethod
    def from_bytes(cls, data: bytes, expect_sizes=None, device=None) -> "QNet":
        torch = _torch()
        view = memoryview(data)
        pos = 0

        def take(n, what):
            nonlocal pos
            if pos + n > len(view):
                raise CheckpointError(f"truncated checkpoint while reading {what}")
            out = view[pos:pos + n]
            pos += n
            return out

        if bytes(take(len(CHECKPOINT_MAGIC), "magic")) != CHECKPOINT_MAGIC:
            raise CheckpointError("bad magic bytes; not a COLORNET checkpoint")
        fmt, n_sizes = (int(v) for v in np.frombuffer(take(8, "header"), dtype="<u4"))
        if fmt != CHECKPOINT_FORMAT_VERSION:
            raise CheckpointError(f"unsupported checkpoint format version {fmt}")
        if not 2 <= n_sizes <= 64:
            raise CheckpointError(f"implausible layer count {n_sizes}")
        sizes = tuple(int(v) for v in np.frombuffer(take(4 * n_sizes, "layer sizes"), dtype="<u4"))
        if expect_sizes is not None and sizes != tuple(expect_sizes):
            raise CheckpointError(f"layer sizes {sizes} do not match {tuple(expect_sizes)}")
        shapes = [(a, b) for a, b in zip(sizes[:-1], sizes[1:])]
        n_floats = sum(a * b + b for a, b in shapes)
        payload = np.frombuffer(take(4 * n_floats, "weights and biases"), dtype="<f4")
        (version,) = (int(v) for v in np.frombuffer(take(8, "version"), dtype="<u8"))
        if pos != len(view):
            raise CheckpointError("trailing bytes after checkpoint payload")
        dev = _lib.require_cuda(device)
        flat = torch.from_numpy(payload.astype(np.float32)).to(dev)  # one upload
        ws, bs, off = [], [], 0
        for a, b in shapes:
            ws.append(flat[off:off + a * b].view(a, b).clone())
            off += a * b
            bs.append(flat[off:off + b].clone())
            off += b
        return cls(ws, bs, version)


def huber_residual_grad(residual):
    """d mean-Huber(delta=1) / d residual, before the 1/B (net.py:83-105)."""
    return residual.clamp(-1.0, 1.0)


def backward(net: QNet, states, actions, targets):
    """Gradients of the mean Huber loss on q[i, a_i] (net.py:88-115).
    Returns (grad_w, grad_b, loss tensor, mean |td| tensor)."""
    torch = _torch()
    acts, pre = net.forward_cached(states)
    q = acts[-1]
    batch = q.shape[0]
    rows = torch.arange(batch, device=q.device)
    residual = q[rows, actions] - targets.to(q.dtype)
    a = residual.abs()
    loss = torch.where(a <= 1.0, 0.5 * residual * residual, a - 0.5).mean()
    mean_abs_td = a.mean()
    dq = torch.zeros_like(q)
    dq[rows, actions] = huber_residual_grad(residual) / batch
    gw = [None] * len(net.weights)
    gb = [None] * len(net.biases)
    delta = dq
    for li in range(len(net.weights) - 1, -1, -1):
        gw[li] = acts[li].t() @ delta
        gb[li] = delta.sum(dim=0)
        if li > 0:
            delta = (delta @ net.weights[li].t()) * (pre[li - 1] > 0)
    return gw, gb, loss, mean_abs_td


@dataclass
class AdamState:  # net.py:118-139
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    step: int = 0
    m_weights: list = field(default_factory=list)
    v_weights: list = field(default_factory=list)
    m_biases: list = field(default_factory=list)
    v_biases: list = field(default_factory=list)

    @classmethod
    def for_params(cls, net: QNet, lr: float = 1e-4) -> "AdamState":
        torch = _torch()
        z = torch.zeros_like
        return cls(lr=lr, m_weights=[z(w) for w in net.weights], v_weights=[z(w) for w in net.weights],
                   m_biases=[z(b) for b in net.biases], v_biases=[z(b) for b in net.biases])


def _adam_launch(net: QNet, gw, gb, st: AdamState, step_dev=None, step_host: int = 0,
                 gate=None) -> None:
    """One ``sp_adam_step`` launch over every weight and bias tensor
    (net.py:141-161 ``_adam_update`` per tensor, fused)."""
    torch = _torch()
    ps = list(net.weights) + list(net.biases)
    gs = [g.contiguous() for g in list(gw) + list(gb)]
    ms = list(st.m_weights) + list(st.m_biases)
    vs = list(st.v_weights) + list(st.v_biases)
    for t in ps + ms + vs:
        if not t.is_contiguous() or t.dtype != torch.float32:
            raise ValueError("adam: parameters and moments must be contiguous float32")
    n = len(ps)
    arr = ctypes.c_void_p * n
    numels = (ctypes.c_int64 * n)(*[t.numel() for t in ps])
    lib = _lib.load()
    dev = ps[0].device
    _lib.check(lib.sp_adam_step(
        n, arr(*[t.data_ptr() for t in ps]), arr(*[t.data_ptr() for t in gs]),
        arr(*[t.data_ptr() for t in ms]), arr(*[t.data_ptr() for t in vs]), numels,
        None if step_dev is None else step_dev.data_ptr(), int(step_host),
        None if gate is None else gate.data_ptr(), float(st.lr), float(st.beta1),
        float(st.beta2), float(st.eps), _lib.stream_ptr(dev)), "adam_step")


def adam_step(net: QNet, gw, gb, st: AdamState) -> QNet:  # net.py:151-161
    st.step += 1
    _adam_launch(net, gw, gb, st, step_host=st.step)
    net.version += 1
    return net


# -- DDQN (ddqn.py) ---------------------------------------------------------------------

@dataclass(frozen=True)
class DdqnConfig:
    gamma: float = 0.98
    target_sync_period: int = 200
    batch_size: int = 256
    lr: float = 1e-4

    def __post_init__(self):
        if not 0.0 <= self.gamma < 1.0:
            raise ValueError(f"gamma must lie in [0, 1), got {self.gamma}")
        if self.target_sync_period < 1 or self.batch_size < 1:
            raise ValueError("target_sync_period and batch_size must be positive")


class UpdateStats(NamedTuple):
    loss: float
    mean_abs_td: float
    version: int
    target_synced: bool


def compute_targets(batch, online: QNet, target: QNet, gamma: float):
    """y = r + gamma (1 - done) Q_target(s', argmax_a Q_online(s', a)) (ddqn.py:38-51);
    argmax ties break toward the lowest index."""
    torch = _torch()
    best = torch.argmax(online.forward(batch.next_states), dim=1)
    q_target = target.forward(batch.next_states)
    bootstrap = q_target[torch.arange(best.shape[0], device=best.device), best]
    not_done = (~batch.dones.bool()).to(q_target.dtype)
    return batch.rewards.to(q_target.dtype) + gamma * not_done * bootstrap


class _GraphedUpdate:
    """One DDQN update captured as a CUDA graph: the targets, the backward and
    Adam (about 90 small kernels, launch-bound when eager) replay as one
    ``cudaGraphLaunch``.

    The batch lives in static tensors that the replay sampler fills in place
    (``ReplayBuffer.sample(out=...)``). The Adam step count is a device scalar,
    so the bias corrections need no host constants. The fused Adam kernel
    (``sp_adam_step``) is gated on ``isfinite(loss)``: a diverged update
    leaves the parameters and moments untouched, exactly as the reference
    raises before stepping (``ddqn.py:66-71``). The graph holds the tensor addresses of ``online``, ``target`` and
    the moments, so those tensors are only ever updated in place."""

    def __init__(self, learner: "DdqnLearner", batch_size: int, state_dim: int):
        from paper_2305_04180_b200.replay import TransitionBatch
        torch = _torch()
        self.learner = learner
        on = learner.online
        dev = on.weights[0].device
        b, d = int(batch_size), int(state_dim)
        self.batch_size, self.state_dim = b, d
        self.batch = TransitionBatch(torch.zeros((b, d), dtype=torch.float32, device=dev),
                                     torch.zeros(b, dtype=torch.int64, device=dev),
                                     torch.zeros(b, dtype=torch.float32, device=dev),
                                     torch.zeros((b, d), dtype=torch.float32, device=dev),
                                     torch.zeros(b, dtype=torch.bool, device=dev))
        self.t = torch.full((), float(learner.adam.step), dtype=torch.float64, device=dev)
        self.loss = torch.zeros((), dtype=torch.float32, device=dev)
        self.mad = torch.zeros((), dtype=torch.float32, device=dev)
        ad = learner.adam
        state = on.weights + on.biases + ad.m_weights + ad.v_weights + ad.m_biases + ad.v_biases
        saved = [x.clone() for x in state]
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm-up: cuBLAS handles/workspaces, allocator
            for _ in range(2):
                self._body()
        torch.cuda.current_stream(dev).wait_stream(side)
        for x, y in zip(state, saved):
            x.copy_(y)
        self.t.fill_(float(ad.step))
        self.graph = torch.cuda.CUDAGraph()
        # thread_local: the actor thread keeps syncing its own stream meanwhile
        with no_gc(), torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
            self._body()

    def _body(self) -> None:
        torch = _torch()
        lr = self.learner
        on, ad = lr.online, lr.adam
        bt = self.batch
        targets = compute_targets(bt, on, lr.target, lr.config.gamma)
        gw, gb, loss, mad = backward(on, bt.states, bt.actions, targets)
        self.loss.copy_(loss)
        self.mad.copy_(mad)
        # gated on isfinite(loss); advances the device step count itself
        _adam_launch(on, gw, gb, ad, step_dev=self.t, gate=self.loss)

    def run(self, batch) -> None:
        if batch is not self.batch:
            for dst, src in zip(self.batch, batch):
                dst.copy_(src.reshape(dst.shape), non_blocking=True)
        self.graph.replay()


class _FusedUpdate:
    """One DDQN update as ``sp_ddqn_update``: two hand-written kernels plus a
    one-thread step tick (csrc/sp_learn.cu), instead of ~100 small torch ones.
    - ``ddqn_rows_kernel``: one CTA per 2-row tile, weights TMA-staged per layer.
      It computes the targets, the cached forward, the Huber gradient and the
      layer deltas.
    - ``ddqn_grad_adam_kernel``: the weight gradients as 16x16 tiles over the
      batch (fixed row order), with the finite-gated Adam step in the epilogue.
    Optionally the three launches replay as one CUDA graph. Same static-batch
    and device-step contract as ``_GraphedUpdate``."""

    def __init__(self, learner: "DdqnLearner", batch_size: int, state_dim: int, graph: bool,
                 sampler=None):
        from paper_2305_04180_b200.replay import TransitionBatch
        torch = _torch()
        self.learner = learner
        on, tg, ad = learner.online, learner.target, learner.adam
        if len(on.weights) != 3:
            raise ValueError("the fused learner kernel supports the 3-layer Q-net only")
        dev = on.weights[0].device
        b, d = int(batch_size), int(state_dim)
        self.batch_size, self.state_dim = b, d
        self.batch = TransitionBatch(torch.zeros((b, d), dtype=torch.float32, device=dev),
                                     torch.zeros(b, dtype=torch.int64, device=dev),
                                     torch.zeros(b, dtype=torch.float32, device=dev),
                                     torch.zeros((b, d), dtype=torch.float32, device=dev),
                                     torch.zeros(b, dtype=torch.bool, device=dev))
        self.t = torch.full((), float(ad.step), dtype=torch.float64, device=dev)
        self.stats = torch.zeros(2, dtype=torch.float32, device=dev)
        self._lib = _lib.load()
        sizes = (ctypes.c_int32 * 4)(*on.sizes)
        n = int(self._lib.sp_ddqn_scratch_floats(sizes, b))
        if n < 0:
            raise ValueError(f"Q-net {on.sizes} with batch {b} exceeds the fused learner kernels' "
                             "shared memory; use graph=True without fused")
        self.scratch = torch.empty(n, dtype=torch.float32, device=dev)
        for t in on.weights + on.biases + tg.weights + tg.biases:
            if not t.is_contiguous() or t.dtype != torch.float32:
                raise ValueError("Q-net tensors must be contiguous float32")

        def mlp(net):
            m = _lib.SpMlp()
            for i, v in enumerate(net.sizes):
                m.sizes[i] = v
            for i in range(3):
                m.W[i] = net.weights[i].data_ptr()
                m.b[i] = net.biases[i].data_ptr()
            return m
        self._on, self._tg = mlp(on), mlp(tg)
        arr = ctypes.c_void_p * 6
        self._m = arr(*[t.data_ptr() for t in ad.m_weights + ad.m_biases])
        self._v = arr(*[t.data_ptr() for t in ad.v_weights + ad.v_biases])
        # optional replay source sampled inside the graph (update_from):
        # (buffer, rng) with rng's Philox counter mirrored on the device
        self.sampler = sampler
        self.d_ctr = None
        if sampler is not None:
            self.d_ctr = torch.full((), int(sampler[1].ctr), dtype=torch.int64, device=dev)
        self.graph = None
        if graph:
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            state = on.weights + on.biases + ad.m_weights + ad.v_weights + ad.m_biases + ad.v_biases
            saved = [x.clone() for x in state]
            with torch.cuda.stream(side):
                self._launch()  # warm-up (attribute setup) before capture
            torch.cuda.current_stream(dev).wait_stream(side)
            for x, y in zip(state, saved):
                x.copy_(y)
            self.t.fill_(float(ad.step))
            if self.d_ctr is not None:
                self.d_ctr.fill_(int(sampler[1].ctr))
            self.graph = torch.cuda.CUDAGraph()
            with no_gc(), torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
                self._launch()

    @property
    def loss(self):
        return self.stats[0]

    @property
    def mad(self):
        return self.stats[1]

    def _launch(self) -> None:
        lr, ad, bt = self.learner, self.learner.adam, self.batch
        dev = lr.online.weights[0].device
        if self.sampler is not None:  # the batch comes straight from the replay ring
            self.sampler[0].sample_dev(self.batch_size, self.sampler[1], self.d_ctr, bt)
        _lib.check(self._lib.sp_ddqn_update(
            ctypes.byref(self._on), ctypes.byref(self._tg), bt.states.data_ptr(),
            bt.actions.data_ptr(), bt.rewards.data_ptr(), bt.next_states.data_ptr(),
            bt.dones.data_ptr(), self.batch_size, float(lr.config.gamma), self._m, self._v,
            self.t.data_ptr(), float(ad.lr), float(ad.beta1), float(ad.beta2), float(ad.eps),
            self.scratch.data_ptr(), self.scratch.numel(), self.stats.data_ptr(),
            _lib.stream_ptr(dev)), "ddqn_update")

    def run(self, batch) -> None:
        if batch is not self.batch:
            for dst, src in zip(self.batch, batch):
                dst.copy_(src.reshape(dst.shape), non_blocking=True)
        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch()


class DdqnLearner:
    """Online/target pair and one update per batch (ddqn.py:54-77).

    Update paths, same numerics contract (fp32, tests at 1e-4 vs the reference):
    - eager torch (default);
    - ``graph=True``: the torch update replayed as one CUDA graph (``_GraphedUpdate``);
    - ``fused=True``: the hand-written ``sp_ddqn_update`` kernels (``_FusedUpdate``),
      optionally graph-replayed too.
    ``graph_batch(B, D)`` returns the static batch a sampler should fill to
    skip the copy-in (None on the eager path)."""

    def __init__(self, params: QNet, config: DdqnConfig | None = None, check_finite: bool = True,
                 graph: bool = False, fused: bool = False):
        self.config = config or DdqnConfig()
        self.online = params
        self.target = params.copy()
        self.adam = AdamState.for_params(params, lr=self.config.lr)
        self.update_count = 0
        self.check_finite = check_finite
        self.graph = bool(graph)
        self.fused = bool(fused)
        self._graphed = None

    def graph_batch(self, batch_size: int, state_dim: int):
        if not (self.graph or self.fused):
            return None
        g = self._graphed
        if (g is None or g.batch_size != batch_size or g.state_dim != state_dim
                or getattr(g, "sampler", None)):
            g = self._graphed = (_FusedUpdate(self, batch_size, state_dim, self.graph)
                                 if self.fused else _GraphedUpdate(self, batch_size, state_dim))
        return g.batch

    def _update_graphed(self, batch) -> UpdateStats:
        b, d = int(batch.states.shape[0]), int(batch.states.shape[1])
        g = self._graphed
        if g is None or g.batch_size != b or g.state_dim != d or getattr(g, "sampler", None):
            g = self._graphed = (_FusedUpdate(self, b, d, self.graph) if self.fused
                                 else _GraphedUpdate(self, b, d))
        g.run(batch)
        return self._finish_update(g)

    def _finish_update(self, g) -> UpdateStats:
        if self.check_finite:
            if isinstance(g, _FusedUpdate):
                loss_v, mad_v = g.stats.tolist()  # one read-back of {loss, mean |td|}
            else:
                loss_v, mad_v = float(g.loss), float(g.mad)
            if not math.isfinite(loss_v):
                raise TrainingDiverged(f"non-finite loss {loss_v!r} at update "
                                       f"{self.update_count + 1} (parameter version "
                                       f"{self.online.version})")
        else:
            loss_v = mad_v = float("nan")
        self.adam.step += 1
        self.online.version += 1
        self.update_count += 1
        synced = self.update_count % self.config.target_sync_period == 0
        if synced:
            self.target.copy_from(self.online)
        return UpdateStats(loss_v, mad_v, self.online.version, synced)

    def update_from(self, buffer, rng, batch_size: int | None = None) -> UpdateStats:
        """Sample a batch from ``buffer`` with ``rng`` and update: the
        learner's step (loops.py:83-88). With ``fused=True, graph=True`` the
        sample (``sp_rb_sample_dev``) and the update replay as one CUDA graph.
        The Philox counter advances on the device and is mirrored in
        ``rng.ctr``, so the draws equal ``buffer.sample(B, rng)``. Raises
        BufferNotReady like ``ReplayBuffer.sample``."""
        b = int(batch_size or self.config.batch_size)
        d = int(buffer.state_dim)
        if not (self.fused and self.graph) or not hasattr(rng, "ctr"):
            return self.update(buffer.sample(b, rng, out=self.graph_batch(b, d)))
        g = self._graphed
        if (g is None or g.batch_size != b or g.state_dim != d or g.sampler is None
                or g.sampler[0] is not buffer or g.sampler[1] is not rng):
            g = self._graphed = _FusedUpdate(self, b, d, True, sampler=(buffer, rng))
            g.ctr_mirror = int(rng.ctr)
        with buffer._lock:
            if len(buffer) < b:
                from paper_2305_04180_b200.replay import BufferNotReady
                raise BufferNotReady(f"buffer holds {len(buffer)} transitions, need {b}")
            if int(rng.ctr) != g.ctr_mirror:  # rng also drew elsewhere: resync the device copy
                g.d_ctr.fill_(int(rng.ctr))
            buffer._order_after(buffer._last_append)
            g.graph.replay()
            rng.ctr += b
            g.ctr_mirror = int(rng.ctr)
            buffer._last_sample = buffer._record()
        return self._finish_update(g)

    def update(self, batch) -> UpdateStats:
        if self.graph or self.fused:
            return self._update_graphed(batch)
        targets = compute_targets(batch, self.online, self.target, self.config.gamma)
        gw, gb, loss, mad = backward(self.online, batch.states, batch.actions, targets)
        loss_v = float(loss) if self.check_finite else float("nan")
        if self.check_finite and not math.isfinite(loss_v):
            raise TrainingDiverged(f"non-finite loss {loss_v!r} at update {self.update_count + 1} "
                                   f"(parameter version {self.online.version})")
        adam_step(self.online, gw, gb, self.adam)
        self.update_count += 1
        synced = self.update_count % self.config.target_sync_period == 0
        if synced:
            self.target.copy_from(self.online)
        return UpdateStats(loss_v, float(mad) if self.check_finite else float("nan"),
                           self.online.version, synced)


# -- VEM (asl/vem.py) ------------------------------------------------------------------

@dataclass(frozen=True)
class VemSchedule:
    n_envs: int
    or_init: int = 16
    or_final: int = 3
    decay_steps: int = 500_000
    e_min: float = 0.01
    e_max: float = 0.8

    def __post_init__(self):
        if not 1 <= self.or_final <= self.or_init <= self.n_envs:
            raise ValueError(f"need 1 <= or_final <= or_init <= n_envs, got "
                             f"{self.or_final}, {self.or_init}, {self.n_envs}")
        if not 0.0 <= self.e_min <= self.e_max <= 1.0:
            raise ValueError("need 0 <= e_min <= e_max <= 1")
        if self.decay_steps < 1:
            raise ValueError("decay_steps must be positive")

    def exploring_interval(self, t_step: int) -> int:  # vem.py:38-40
        frac = min(t_step / self.decay_steps, 1.0)
        return int(math.floor(self.or_init + (self.or_final - self.or_init) * frac + 0.5))

    def epsilons(self, t_step: int) -> np.ndarray:  # vem.py:42-54, vectorized
        size = self.exploring_interval(t_step)
        first = self.n_envs - size
        i = np.arange(self.n_envs)
        ramp = self.e_min + (self.e_max - self.e_min) * (i - first) / max(size - 1, 1)
        eps = np.where(i < first, self.e_min, ramp)
        eps[-1] = self.e_max if size >= 1 else eps[-1]
        return eps.astype(np.float64)

    def epsilon(self, i: int, t_step: int) -> float:
        if not 0 <= i < self.n_envs:
            raise ValueError(f"copy index {i} out of range [0, {self.n_envs})")
        return float(self.epsilons(t_step)[i])


def philox_fill(n: int, stream, kind: int, lo: float, hi: float, device=None):
    """Device draws from a PhiloxGenerator-like stream (seed, lane, ctr, tag);
    advances its counter by n blocks.  kind 0: uniform f64, kind 1: integers."""
    torch = _torch()
    dev = _lib.require_cuda(device)
    out = torch.empty(n, dtype=torch.float64 if kind == 0 else torch.int64, device=dev)
    tag = int(getattr(stream, "tag", 3))
    _lib.check(_lib.load().sp_philox_fill(n, stream.seed, stream.lane, tag, stream.ctr, kind,
                                          float(lo), float(hi), out.data_ptr(),
                                          _lib.stream_ptr(dev)), "philox_fill")
    stream.ctr += n
    return out


def select_actions(q, epsilons, rng):
    """Row-wise epsilon-greedy on device (vem.py:57-66): random action with
    probability eps (draws: random(n), then integers(0, A, n)), else argmax
    (ties to the lowest index)."""
    torch = _torch()
    n, n_actions = q.shape
    eps = torch.as_tensor(epsilons, dtype=torch.float64, device=q.device)
    explore = philox_fill(n, rng, 0, 0.0, 1.0, q.device) < eps
    randoms = philox_fill(n, rng, 1, 0, n_actions, q.device)
    greedy = torch.argmax(q, dim=1)
    return torch.where(explore, randoms, greedy)


def select_actions_fused(params: QNet, states, vem: VemSchedule, t_step: int, rng,
                         env0: int = 0, out=None, q_out=None):
    """The actor's ``net.forward`` -> ``vem.epsilons(t_step)`` -> ``select_actions``
    (loops.py:57-59) as one kernel launch (``sp_actor_select``): the epsilons
    are computed on the device from the scalar ``t_step``, so nothing crosses
    the host per step.  Same draws as ``select_actions`` (random(n), then
    integers(0, A, n) from ``rng``; its counter advances by 2n).  ``env0``: VEM
    copy index of row 0 (a shard's env id offset)."""
    torch = _torch()
    n = int(states.shape[0])
    dev = states.device
    if out is None:
        out = torch.empty(n, dtype=torch.int64, device=dev)
    m = _lib.SpMlp()
    m.sizes[:] = list(params.sizes)
    for i in range(3):
        m.W[i] = params.weights[i].data_ptr()
        m.b[i] = params.biases[i].data_ptr()
    v = _lib.SpVem(vem.n_envs, vem.or_init, vem.or_final, vem.decay_steps, vem.e_min, vem.e_max)
    st = states if states.dtype == torch.float32 and states.is_contiguous() else \
        states.to(torch.float32).contiguous()
    tag = int(getattr(rng, "tag", 3))
    _lib.check(_lib.load().sp_actor_select(
        ctypes.byref(m), st.data_ptr(), n, int(env0), ctypes.byref(v), int(t_step), rng.seed,
        rng.lane, tag, rng.ctr, out.data_ptr(), q_out.data_ptr() if q_out is not None else None,
        _lib.stream_ptr(dev)), "actor_select")
    rng.ctr += 2 * n
    return out


# -- TFM (asl/tfm.py) -------------------------------------------------------------------

@dataclass(frozen=True)
class TfmConfig:
    """Time-feedback pacing targets (asl/tfm.py:15-29): n_envs interactions
    per actor period, batch_size samples per learner update, and the target
    transitions-per-sample ratio tps; rho = n_envs * tps / batch_size is the
    learner updates one actor period should take."""
    n_envs: int
    tps: float
    batch_size: int
    warmup_samples: int = 10
    max_sleep_s: float = 1.0

    def __post_init__(self):
        if self.n_envs < 1 or self.batch_size < 1 or self.tps <= 0:
            raise ValueError("n_envs, batch_size must be >= 1 and tps > 0")

    @property
    def rho(self) -> float:
        return self.n_envs * self.tps / self.batch_size


class TfmState:
    """Time-feedback modulation (asl/tfm.py:32-77, paper Alg. 1).

    Keeps exponential moving averages (weight ``ema_factor`` on the newest
    sample, the first sample taken as is) of the actor's interaction period
    and the learner's update period.  Here the periods are device times: the
    actor loop feeds the CUDA-event time between its iteration-end events
    (``record_interaction_events``), so the pacing sees the GPU's work, not
    the host's enqueue time.  With xi = rho * T_update - T_interaction, the
    faster side sleeps: the actor for xi when xi > 0, the learner for
    -xi / rho otherwise, each capped at max_sleep_s, and neither before both
    averages hold warmup_samples samples."""

    def __init__(self, ema_factor: float = 0.1):
        self.ema_factor = float(ema_factor)
        self.v_period_s = None  # actor interaction period (s), EMA
        self.b_period_s = None  # learner update period (s), EMA
        self.v_count = 0
        self.b_count = 0

    def _fold(self, avg, x):
        return x if avg is None else (1.0 - self.ema_factor) * avg + self.ema_factor * x

    def record_interaction(self, seconds: float) -> None:
        self.v_period_s = self._fold(self.v_period_s, seconds)
        self.v_count += 1

    def record_optimization(self, seconds: float) -> None:
        self.b_period_s = self._fold(self.b_period_s, seconds)
        self.b_count += 1

    def record_interaction_events(self, start, end) -> None:
        """An interaction period measured on the device (two CUDA events)."""
        self.record_interaction(start.elapsed_time(end) / 1e3)

    def ready(self, cfg: TfmConfig) -> bool:
        return min(self.v_count, self.b_count) >= cfg.warmup_samples

    def compute_xi(self, cfg: TfmConfig) -> float:
        if self.v_period_s is None or self.b_period_s is None:
            raise ValueError("both loop periods must be recorded before computing xi")
        return cfg.rho * self.b_period_s - self.v_period_s

    def actor_sleep(self, cfg: TfmConfig) -> float:
        if not self.ready(cfg):
            return 0.0
        xi = self.compute_xi(cfg)
        return min(xi, cfg.max_sleep_s) if xi > 0 else 0.0

    def learner_sleep(self, cfg: TfmConfig) -> float:
        if not self.ready(cfg):
            return 0.0
        xi = self.compute_xi(cfg)
        return min(-xi / cfg.rho, cfg.max_sleep_s) if xi <= 0 else 0.0


# -- Sharer + loops (asl/sharer.py, asl/loops.py) ------------------------------------------

class PublishedModel:
    """A published parameter snapshot (sharer.py:18-24): version, a private
    copy of the parameters, and the crc32 of their ``COLORNET`` bytes.

    The checksum is taken from that private copy the first time it is read,
    not in the learner's publish call. Nothing writes the copy after
    publication, so the value is the same, and the learner does not pay a
    device-to-host read and a CRC every ``upload_period`` updates. Unpacks
    like the reference's NamedTuple."""

    __slots__ = ("version", "params", "_crc", "ready")

    def __init__(self, version: int, params: QNet, checksum: int | None = None, ready=None):
        self.version = int(version)
        self.params = params
        self._crc = checksum
        self.ready = ready  # CUDA event: the copy kernels have written params

    def wait(self, stream=None) -> None:
        """Order `stream` (default: the current one) after the copy that made
        this snapshot; the reader must call it before touching params."""
        if self.ready is not None:
            (stream or _torch().cuda.current_stream()).wait_event(self.ready)

    @property
    def checksum(self) -> int:
        if self._crc is None:
            if self.ready is not None:
                self.ready.synchronize()
            self._crc = _checksum(self.params)
        return self._crc

    def __iter__(self):
        return iter((self.version, self.params, self.checksum))


def _checksum(params: QNet) -> int:
    return zlib.crc32(params.to_bytes())


def verify_snapshot(snapshot: PublishedModel) -> bool:
    return _checksum(snapshot.params) == snapshot.checksum


class Sharer:
    """Replay ring + counters + versioned parameter exchange (sharer.py:34-86)."""

    def __init__(self, buffer: ReplayBuffer, tfm: TfmState | None = None):
        self.buffer = buffer
        self.tfm = tfm or TfmState()
        self.t_step = 0
        self.b_step = 0
        self.publish_count = 0
        self.stop = threading.Event()
        self._published: PublishedModel | None = None
        self._error: BaseException | None = None

    def publish_params(self, params: QNet) -> PublishedModel:
        torch = _torch()
        snap_params = params.copy()  # clone kernels on the publisher's stream
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(snap_params.weights[0].device))
        # readers order their stream after `ready` (PublishedModel.wait) before
        # touching the copy: the reference copies on the host, so it has no
        # window in which a half-written snapshot is visible
        snap = PublishedModel(params.version, snap_params, ready=ready)  # crc32 on first read
        self._published = snap  # atomic reference swap
        self.publish_count += 1
        return snap

    def fetch_params(self, newer_than: int) -> PublishedModel | None:
        snap = self._published
        return snap if snap is not None and snap.version > newer_than else None

    @property
    def published_version(self):
        snap = self._published
        return snap.version if snap is not None else None

    def measured_tps(self, batch_size: int):
        return None if self.t_step == 0 else batch_size * self.b_step / self.t_step

    def record_error(self, exc: BaseException) -> None:
        if self._error is None:
            self._error = exc
        self.stop.set()

    def raise_if_failed(self) -> None:
        if self._error is not None:
            raise self._error

    @property
    def failed(self) -> bool:
        return self._error is not None


_IDLE_POLL_S = 0.002


def actor_loop(sharer: Sharer, vec_env, initial_states, params: QNet, vem: VemSchedule,
               tfm_cfg: TfmConfig, max_steps: int, rng, env0: int = 0) -> None:
    """loops.py:43-71 on device with no host round trip per iteration: one
    ``sp_actor_select`` launch (forward, VEM epsilons from the scalar t_step,
    epsilon-greedy), the fused env step, the ring append.  Outputs alternate
    between two StepBatch buffers (stream order keeps iteration k's append
    reading its rows while step k + 1 writes the other set).  The host runs at
    most two iterations ahead of the GPU, and the TFM interaction period is
    the CUDA-event time between iteration ends, recorded once completed."""
    from collections import deque
    torch = _torch()
    dev = vec_env.device
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        states = initial_states
        params = params.copy()
        version = params.version
        n = vec_env.n_copies
        outs = [vec_env.new_batch(), vec_env.new_batch()]
        acts = [torch.empty(n, dtype=torch.int64, device=dev) for _ in range(2)]
        ends = deque()  # iteration-end events not yet folded into the TFM
        k = 0
        try:
            while sharer.t_step < max_steps and not sharer.stop.is_set():
                if len(ends) >= 3:  # bounded run-ahead: wait for iteration k - 2
                    ends[-3].synchronize()
                while len(ends) >= 2 and ends[1].query():
                    sharer.tfm.record_interaction_events(ends[0], ends[1])
                    ends.popleft()
                snap = sharer.fetch_params(version)
                if snap is not None:
                    snap.wait(stream)
                    params, version = snap.params, snap.version
                a = select_actions_fused(params, states, vem, sharer.t_step, rng, env0,
                                         out=acts[k & 1])
                batch = outs[k & 1]
                vec_env.step_device(a.data_ptr(), batch)  # actions valid by construction
                sharer.buffer.append_batch(states, a, batch.rewards, batch.store_states,
                                           batch.dones)
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(stream)
                ends.append(ev)
                states = batch.states
                sharer.t_step += n
                k += 1
                nap = sharer.tfm.actor_sleep(tfm_cfg)
                if nap > 0:
                    time.sleep(nap)
            stream.synchronize()
        finally:
            sharer.stop.set()


def learner_loop(sharer: Sharer, algo: DdqnLearner, tfm_cfg: TfmConfig, learn_start: int,
                 upload_period: int, rng) -> None:
    """loops.py:74-99 on device."""
    torch = _torch()
    dev = algo.online.weights[0].device
    batch_size = tfm_cfg.batch_size
    with torch.cuda.stream(torch.cuda.Stream(dev)):
        while not sharer.stop.is_set():
            if len(sharer.buffer) <= learn_start:
                time.sleep(_IDLE_POLL_S)
                continue
            started = time.perf_counter()
            try:
                algo.update_from(sharer.buffer, rng, batch_size)  # sample + update
            except BufferNotReady:
                time.sleep(_IDLE_POLL_S)
                continue
            sharer.b_step += 1
            published = sharer.b_step % upload_period == 0
            if published:
                sharer.publish_params(algo.online)
            if published or not algo.check_finite:  # else the loss read already synchronized
                torch.cuda.current_stream(dev).synchronize()
            sharer.tfm.record_optimization(time.perf_counter() - started)
            nap = sharer.tfm.learner_sleep(tfm_cfg)
            if nap > 0:
                time.sleep(nap)


@dataclass
class Session:
    sharer: Sharer
    actor: threading.Thread
    learner: threading.Thread
    max_steps: int

    @property
    def running(self) -> bool:
        return self.actor.is_alive() or self.learner.is_alive()

    def wait(self, timeout: float | None = None) -> None:
        self.actor.join(timeout)
        self.learner.join(timeout)
        self.sharer.raise_if_failed()

    def abort(self) -> None:
        self.sharer.stop.set()


def _guarded(fn, sharer: Sharer, *args) -> None:
    try:
        fn(sharer, *args)
    except BaseException as exc:  # noqa: BLE001 (re-raised by Session.wait)
        sharer.record_error(exc)


def start_session(sharer: Sharer, vec_env, initial_states, params: QNet, vem: VemSchedule,
                  tfm_cfg: TfmConfig, max_steps: int, algo: DdqnLearner, learn_start: int,
                  upload_period: int, seed: int) -> Session:
    """Publish the initial model and start the actor and learner threads
    (loops.py:130-149); their streams are (seed, 0xAC) / (seed, 0x1E)."""
    sharer.publish_params(params)
    algo.graph_batch(tfm_cfg.batch_size, sharer.buffer.state_dim)  # capture before threads run
    actor_rng = PhiloxGenerator(seed, 0xAC)
    actor_rng.tag = 3
    learner_rng = PhiloxGenerator(seed, 0x1E)
    actor = threading.Thread(target=_guarded, name="color-actor", daemon=True,
                             args=(actor_loop, sharer, vec_env, initial_states, params, vem,
                                   tfm_cfg, max_steps, actor_rng))
    learner = threading.Thread(target=_guarded, name="color-learner", daemon=True,
                               args=(learner_loop, sharer, algo, tfm_cfg, learn_start,
                                     upload_period, learner_rng))
    actor.start()
    learner.start()
    return Session(sharer, actor, learner, max_steps)
