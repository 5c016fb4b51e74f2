"""Counter-based RNG shim -- TEST INFRASTRUCTURE ONLY (the oracle side).

The reference draws from numpy PCG64 streams spawned per lane
(``vecenv.py:86-89``: ``SeedSequence(seed).spawn(N)`` -> ``default_rng``).
No GPU can reproduce those streams, so every parity run replaces them, on
BOTH sides, with the Philox4x32-10 stream contract in DESIGN.md ("RNG
contract"):

* key = (seed & 0xffffffff, seed >> 32); counter = (block_lo, block_hi,
  lane, tag); ``tag`` 0 = env lane stream, 1 = benchmark random actions,
  2 = replay sampling.
* ``uniform(lo, hi)``  = lo + (hi - lo) * u53, u53 = (x1:x0 >> 11) * 2**-53
  (numpy ``Generator.uniform`` arithmetic, ``params.py:114-120``,
  ``core.py:136-138``); one block per value.
* ``integers(lo, hi)`` = lo + mulhi64(x1:x0, hi - lo); one block per value
  (``params.py:116-117``, ``replay.py:76``).
* ``normal(loc, scale, n)`` = loc + scale * z, z from Box-Muller on
  (x0, x1) and (x2, x3) -- four normals per block (``core.py:240``).

``PhiloxStream`` duck-types the four ``numpy.random.Generator`` methods the
reference calls (``uniform``, ``integers``, ``normal``, ``random``), so it can
be injected into the UNMODIFIED reference: ``reference_rng_proxy`` swaps
``color_rl.vecenv.np`` for a proxy whose ``random.SeedSequence(seed).spawn``
and ``random.default_rng`` hand out PhiloxStreams keyed by (seed, lane).
Normal draws call the compiled oracle (glibc log/cos/sin) so the oracle and
the shim-driven reference agree bit for bit.
"""

from __future__ import annotations

import ctypes

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint32(0x9E3779B9)
W1 = np.uint32(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)

TAG_ENV = 0
TAG_ACTIONS = 1
TAG_REPLAY = 2


def philox4x32_10(ctr: np.ndarray, key0: int, key1: int) -> np.ndarray:
    """Vectorized Philox4x32-10. ctr: (n, 4) uint32 -> (n, 4) uint32."""
    c = np.asarray(ctr, dtype=np.uint32).reshape(-1, 4).astype(np.uint64)
    c0, c1, c2, c3 = c[:, 0], c[:, 1], c[:, 2], c[:, 3]
    k0 = np.uint64(key0 & 0xFFFFFFFF)
    k1 = np.uint64(key1 & 0xFFFFFFFF)
    for _ in range(10):
        p0 = c0 * M0
        p1 = c2 * M1
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ k0
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ k1
        c1 = p1 & MASK32
        c3 = p0 & MASK32
        c0 = n0 & MASK32
        c2 = n2 & MASK32
        k0 = (k0 + np.uint64(W0)) & MASK32
        k1 = (k1 + np.uint64(W1)) & MASK32
    return np.stack([c0, c1, c2, c3], axis=1).astype(np.uint32)


def blocks(seed: int, lane, tag: int, ctr) -> np.ndarray:
    """Philox blocks for (lane, ctr) pairs (broadcast), shape (n, 4) uint32."""
    lane = np.asarray(lane, dtype=np.uint64)
    ctr = np.asarray(ctr, dtype=np.uint64)
    lane, ctr = np.broadcast_arrays(lane, ctr)
    c = np.stack([ctr & MASK32, ctr >> np.uint64(32), lane & MASK32,
                  np.full(ctr.shape, tag, dtype=np.uint64)], axis=-1)
    return philox4x32_10(c.reshape(-1, 4), seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)


def word64(b: np.ndarray) -> np.ndarray:
    return (b[:, 1].astype(np.uint64) << np.uint64(32)) | b[:, 0].astype(np.uint64)


def u53(b: np.ndarray) -> np.ndarray:
    return (word64(b) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def mulhi_range(b: np.ndarray, span: int) -> np.ndarray:
    """floor(word64 * span / 2**64) exactly, for 0 < span < 2**63."""
    w = word64(b)
    lo = w & MASK32
    hi = w >> np.uint64(32)
    s_lo = np.uint64(span & 0xFFFFFFFF)
    s_hi = np.uint64(span >> 32)
    # 128-bit product via 32-bit limbs
    ll = lo * s_lo
    lh = lo * s_hi
    hl = hi * s_lo
    hh = hi * s_hi
    mid = (ll >> np.uint64(32)) + (lh & MASK32) + (hl & MASK32)
    top = hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))
    return top.astype(np.int64)


_ORACLE_LIB = None


def _oracle_lib():
    global _ORACLE_LIB
    if _ORACLE_LIB is None:
        from oracle.oracle import load_lib
        _ORACLE_LIB = load_lib()
    return _ORACLE_LIB


class PhiloxStream:
    """Duck-typed numpy Generator over one Philox stream (seed, lane, tag)."""

    def __init__(self, seed: int, lane: int, tag: int = TAG_ENV, ctr: int = 0):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.lane = int(lane) & 0xFFFFFFFF
        self.tag = int(tag)
        self.ctr = int(ctr)

    def _take(self, n: int) -> np.ndarray:
        b = blocks(self.seed, self.lane, self.tag,
                   np.arange(self.ctr, self.ctr + n, dtype=np.uint64))
        self.ctr += n
        return b

    def uniform(self, low=0.0, high=1.0, size=None):
        n = 1 if size is None else int(np.prod(size))
        u = u53(self._take(n))
        out = low + (high - low) * u
        return float(out[0]) if size is None else out.reshape(size)

    def integers(self, low, high=None, size=None, dtype=np.int64, endpoint=False):
        if high is None:
            low, high = 0, low
        low, high = int(low), int(high) + (1 if endpoint else 0)
        if high <= low:
            raise ValueError("high <= low")
        n = 1 if size is None else int(np.prod(size))
        out = low + mulhi_range(self._take(n), high - low)
        return int(out[0]) if size is None else out.astype(dtype).reshape(size)

    def random(self, size=None):
        return self.uniform(0.0, 1.0, size)

    def standard_normal_raw(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        lib = _oracle_lib()
        lib.or_stream_draw(ctypes.c_uint64(self.seed), ctypes.c_uint32(self.lane),
                           ctypes.c_uint32(self.tag), ctypes.c_uint64(self.ctr), 2,
                           ctypes.c_double(0.0), ctypes.c_double(0.0), n,
                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        self.ctr += (n + 3) // 4
        return out

    def normal(self, loc=0.0, scale=1.0, size=None):
        n = 1 if size is None else int(np.prod(size))
        z = self.standard_normal_raw(n)
        out = loc + scale * z
        return float(out[0]) if size is None else out.reshape(size)


def random_actions(seed: int, env_ids, step: int, n_actions: int = 5) -> np.ndarray:
    """Benchmark/test action stream: env e at step t draws integers(0, A) from
    block t of (seed, e, TAG_ACTIONS)."""
    env_ids = np.asarray(env_ids, dtype=np.uint64)
    b = blocks(seed, env_ids, TAG_ACTIONS, np.full(env_ids.shape, step, dtype=np.uint64))
    return mulhi_range(b, n_actions)


# -- driving the UNMODIFIED reference ------------------------------------------

class _SeedToken:
    def __init__(self, seed: int, lane: int):
        self.seed, self.lane = seed, lane


class _SeedSequenceShim:
    def __init__(self, seed, lane_offset: int = 0):
        self._seed = int(seed)
        self._offset = lane_offset

    def spawn(self, n):
        return [_SeedToken(self._seed, self._offset + i) for i in range(n)]


class _RandomShim:
    def __init__(self, lane_offset: int):
        self._offset = lane_offset

    def SeedSequence(self, seed=None, *a, **k):  # noqa: N802 (numpy name)
        return _SeedSequenceShim(seed, self._offset)

    def default_rng(self, seed=None):
        if isinstance(seed, _SeedToken):
            return PhiloxStream(seed.seed, seed.lane, TAG_ENV)
        return np.random.default_rng(seed)

    def __getattr__(self, name):
        return getattr(np.random, name)


class _NumpyProxy:
    def __init__(self, lane_offset: int):
        self.random = _RandomShim(lane_offset)

    def __getattr__(self, name):
        return getattr(np, name)


class reference_rng_proxy:
    """Context manager: while active, the reference's ``VecEnv.reset_all(seed)``
    (vecenv.py:84-92) hands lane i the PhiloxStream (seed, lane_offset + i)."""

    def __init__(self, vecenv_module, lane_offset: int = 0):
        self._mod = vecenv_module
        self._offset = lane_offset
        self._saved = None

    def __enter__(self):
        self._saved = self._mod.np
        self._mod.np = _NumpyProxy(self._offset)
        return self

    def __exit__(self, *exc):
        self._mod.np = self._saved
        return False
