"""The GPU replay ring vs the reference's replay tests (tests/test_replay.py)
and bit-exact sampled rows against golden vectors and the numpy oracle."""

import threading

import numpy as np
import pytest

from helpers import golden
from oracle.oracle import ReplayOracle
from oracle.philox_shim import PhiloxStream

pytestmark = pytest.mark.gpu


def batch_of(n, offset=0, dim=4):
    base = np.arange(n, dtype=np.float32) + offset
    s = np.tile(base[:, None], (1, dim))
    return s, base.astype(np.int64) % 5, base * 0.5, s + 0.25, (base.astype(np.int64) % 7) == 0


def rb(cap, dim=4):
    from paper_2305_04180_b200 import ReplayBuffer
    return ReplayBuffer(capacity=cap, state_dim=dim)


def test_sizes_grow_then_saturate():  # test_replay.py:20-27
    buf = rb(50)
    assert len(buf) == 0
    buf.append_batch(*batch_of(16))
    assert len(buf) == 16
    for i in range(5):
        buf.append_batch(*batch_of(16, offset=16 * (i + 1)))
    assert len(buf) == 50


def test_rows_stored_bit_exact():  # test_replay.py:30-39
    buf = rb(32)
    s, a, r, s2, d = batch_of(10)
    buf.append_batch(s, a, r, s2, d)
    snap = buf.snapshot()
    assert np.array_equal(snap.states.cpu().numpy(), s)
    assert np.array_equal(snap.actions.cpu().numpy(), a)
    assert np.array_equal(snap.rewards.cpu().numpy(), r)
    assert np.array_equal(snap.next_states.cpu().numpy(), s2)
    assert np.array_equal(snap.dones.cpu().numpy(), d)


def test_fifo_overwrite_keeps_most_recent():  # test_replay.py:42-52
    cap = 40
    buf = rb(cap)
    for start in range(0, 2 * cap, 8):
        buf.append_batch(*batch_of(8, offset=start))
    present = sorted(buf.snapshot().states[:, 0].cpu().numpy().tolist())
    assert len(buf) == cap and present == list(np.arange(cap, 2 * cap, dtype=np.float32))


def test_wrapping_batches_and_f64_rewards_from_device():
    import torch
    buf = rb(10, dim=3)
    orc = ReplayOracle(10, 3)
    for start in (0, 7, 14, 23):
        s, a, r, s2, d = batch_of(7, offset=start, dim=3)
        buf.append_batch(torch.from_numpy(s).cuda(), torch.from_numpy(a).cuda(),
                         torch.from_numpy(r.astype(np.float64)).cuda(),
                         torch.from_numpy(s2).cuda(), torch.from_numpy(d).cuda())
        orc.append_batch(s, a, r, s2, d)
    snap = buf.snapshot()
    assert np.array_equal(snap.states.cpu().numpy(), orc.s[: orc.size])
    assert np.array_equal(snap.rewards.cpu().numpy(), orc.r[: orc.size])


def test_oversized_batch_and_not_ready():  # test_replay.py:55-78
    from paper_2305_04180_b200 import BufferNotReady, PhiloxGenerator
    buf = rb(8)
    with pytest.raises(ValueError):
        buf.append_batch(*batch_of(9))
    buf = rb(16)
    buf.append_batch(*batch_of(3))
    with pytest.raises(BufferNotReady):
        buf.sample(4, PhiloxGenerator(0))
    buf = rb(16)
    buf.append_batch(*batch_of(1))
    g = PhiloxGenerator(0)
    for _ in range(6):
        got = buf.sample(1, g)
        assert got.actions.cpu().numpy().tolist() == [0]
    with pytest.raises(BufferNotReady):
        buf.sample(2, g)


def test_sample_never_reads_unwritten_slots():  # test_replay.py:81-87
    from paper_2305_04180_b200 import PhiloxGenerator
    buf = rb(1000)
    buf.append_batch(*batch_of(37))
    g = PhiloxGenerator(1)
    for _ in range(50):
        assert (buf.sample(16, g).states[:, 0] < 37).all()


def test_sampling_uniformity_chi_square():  # test_replay.py:90-102
    from scipy import stats
    from paper_2305_04180_b200 import PhiloxGenerator
    buf = rb(1000)
    for start in range(0, 1000, 100):
        buf.append_batch(*batch_of(100, offset=start))
    g = PhiloxGenerator(2)
    counts = np.zeros(1000)
    for _ in range(100):
        ids = buf.sample(1000, g).states[:, 0].cpu().numpy().astype(int)
        np.add.at(counts, ids, 1)
    assert stats.chisquare(counts).pvalue > 0.01


def test_transitions_are_copies():  # test_replay.py:105-110
    from paper_2305_04180_b200 import PhiloxGenerator
    buf = rb(8)
    buf.append_batch(*batch_of(4))
    got = buf.sample(2, PhiloxGenerator(3))
    got.states[:] = -1
    assert (buf.snapshot().states >= 0).all()


def test_sampled_indices_and_rows_match_reference_golden():
    z = golden("replay.npz")
    buf = rb(1000)
    for start in range(0, 1500, 100):
        buf.append_batch(*batch_of(100, offset=start))
    g = PhiloxStream(int(z["seed"]), int(z["stream"]), tag=2)
    for i in range(4):
        got = buf.sample(256, g)
        assert np.array_equal(got.states.cpu().numpy(), z["states"][i])
        assert np.array_equal(got.actions.cpu().numpy(), z["actions"][i])
        assert np.array_equal(got.rewards.cpu().numpy(), z["rewards"][i])
        assert np.array_equal(got.dones.cpu().numpy(), z["dones"][i])


def test_large_ring_indices_match_oracle():
    """cfg5 shape: 1M capacity, D=37, 4096-row appends, batch 256."""
    import torch
    cap, dim = 1_000_000, 37
    buf = rb(cap, dim)
    orc = ReplayOracle(cap, dim)
    rng = np.random.default_rng(0)
    for k in range(5):
        n = 4096
        s = rng.random((n, dim), dtype=np.float32)
        a = rng.integers(0, 5, n)
        r = rng.random(n)
        d = rng.random(n) < 0.05
        buf.append_batch(torch.from_numpy(s).cuda(), torch.from_numpy(a).cuda(),
                         torch.from_numpy(r).cuda(), torch.from_numpy(s + 1).cuda(),
                         torch.from_numpy(d).cuda())
        orc.append_batch(s, a, r, s + 1, d)
    g1, g2 = PhiloxStream(9, 1, tag=2), PhiloxStream(9, 1, tag=2)
    for _ in range(8):
        got, idx = buf.sample(256, g1, return_indices=True)
        (s_, a_, r_, s2_, d_), widx = orc.sample(256, g2)
        assert np.array_equal(idx.cpu().numpy(), widx)
        assert np.array_equal(got.states.cpu().numpy(), s_)
        assert np.array_equal(got.next_states.cpu().numpy(), s2_)
        assert np.array_equal(got.rewards.cpu().numpy(), r_)


def test_concurrent_append_sample_rows_never_torn():  # test_replay.py:113-158
    """One appender and one sampler thread on separate CUDA streams."""
    import torch
    from paper_2305_04180_b200 import BufferNotReady, PhiloxGenerator
    dim = 6
    buf = rb(256, dim)
    stop = threading.Event()
    errors = []

    def producer():
        with torch.cuda.stream(torch.cuda.Stream()):
            i = 0
            while not stop.is_set():
                base = np.arange(i, i + 16, dtype=np.float32)
                s = np.tile(base[:, None], (1, dim))
                buf.append_batch(s, base.astype(np.int64) % 5, base * 0.5, s + 0.25,
                                 (base.astype(np.int64) % 2) == 0)
                i += 16

    def consumer():
        g = PhiloxGenerator(4)
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                for _ in range(600):
                    try:
                        got = buf.sample(32, g)
                    except BufferNotReady:
                        continue
                    s = got.states.cpu().numpy()
                    ids = s[:, 0]
                    assert (s == ids[:, None]).all(), "torn state row"
                    assert np.array_equal(got.actions.cpu().numpy(), ids.astype(np.int64) % 5)
                    assert np.array_equal(got.rewards.cpu().numpy(), (ids * 0.5).astype(np.float32))
                    assert (got.next_states.cpu().numpy() == ids[:, None] + 0.25).all()
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    p, c = threading.Thread(target=producer), threading.Thread(target=consumer)
    p.start()
    c.start()
    c.join()
    stop.set()
    p.join()
    assert not errors, errors[0]


def test_capacity_one_ring_and_empty_append():
    """Edge sizes: a one-slot ring keeps only the newest row; an empty batch
    is a no-op."""
    from paper_2305_04180_b200 import PhiloxGenerator
    buf = rb(1)
    buf.append_batch(*batch_of(0))
    assert len(buf) == 0
    for k in range(3):
        buf.append_batch(*batch_of(1, offset=10 * k))
        assert len(buf) == 1
        got = buf.sample(1, PhiloxGenerator(k))  # B <= size, as replay.py:73-75 gates
        assert got.states.cpu().numpy()[:, 0].tolist() == [10.0 * k]


@pytest.mark.parametrize("dim", [37, 4, 1, 5])
def test_append_any_cursor_alignment_matches_oracle(dim):
    """The vectorized append (16-byte ring stores, float4 or scalar source
    reads by alignment, <= 2 segments per column) stores every column
    bit-exact for batch sizes that leave the cursor at every residue mod 4,
    across wraps, from device and host inputs."""
    import torch
    rng = np.random.default_rng(dim)
    cap = 1000 + dim
    buf = rb(cap, dim=dim)
    orc = ReplayOracle(cap, dim)
    for k, n in enumerate((1, 3, 2, 5, 7, 64, 333, 999, 17, cap, 6, 1000)):
        s = rng.standard_normal((n, dim)).astype(np.float32)
        s2 = rng.standard_normal((n, dim)).astype(np.float32)
        a = rng.integers(0, 5, n)
        r = rng.standard_normal(n)
        d = rng.random(n) < 0.3
        if k % 2:
            buf.append_batch(*(torch.from_numpy(np.ascontiguousarray(x)).cuda()
                               for x in (s, a, r, s2, d)))
        else:
            buf.append_batch(s, a, r.astype(np.float32), s2, d)
        orc.append_batch(s, a, r.astype(np.float32), s2, d)
        snap = buf.snapshot()
        m = orc.size
        assert np.array_equal(snap.states.cpu().numpy(), orc.s[:m]), (k, n)
        assert np.array_equal(snap.next_states.cpu().numpy(), orc.s2[:m]), (k, n)
        assert np.array_equal(snap.actions.cpu().numpy(), orc.a[:m]), (k, n)
        assert np.array_equal(snap.rewards.cpu().numpy(), orc.r[:m]), (k, n)
        assert np.array_equal(snap.dones.cpu().numpy(), orc.d[:m]), (k, n)
