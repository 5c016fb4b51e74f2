"""ASL learner side on the GPU vs the reference's
numpy implementation (oracle/_ref): Q-net init/forward/backward/Adam, DDQN
targets and updates, VEM epsilons and epsilon-greedy draws, TFM pacing,
COLORNET checkpoints; plus a cfg5-shaped session on the CUDA env + replay."""

import numpy as np
import pytest

from helpers import config, load_maps, ranges
from oracle import oracle as O
from oracle.philox_shim import PhiloxStream

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")]

SIZES = (37, 256, 128, 5)


def ref():
    O.import_reference(37)
    import color_rl
    return color_rl


def _batch(rng, n, dim=37, torch_dev=None):
    s = rng.standard_normal((n, dim)).astype(np.float32)
    a = rng.integers(0, 5, n)
    r = rng.standard_normal(n).astype(np.float32)
    s2 = rng.standard_normal((n, dim)).astype(np.float32)
    d = rng.random(n) < 0.1
    return s, a, r, s2, d


def _tb(arrs):
    import torch
    from paper_2305_04180_b200 import TransitionBatch
    s, a, r, s2, d = arrs
    return TransitionBatch(*(torch.from_numpy(np.ascontiguousarray(x)).cuda()
                             for x in (s, a, r, s2, d)))


def test_init_and_forward_match_reference():
    ref()
    from color_rl import net
    from paper_2305_04180_b200.asl import QNet
    p_ref = net.init_params(np.random.default_rng(7), SIZES)
    p = QNet.init(np.random.default_rng(7), SIZES)
    for w, wr in zip(p.weights, p_ref.weights):
        assert np.array_equal(w.cpu().numpy(), wr)
    x = np.random.default_rng(1).standard_normal((512, 37)).astype(np.float32)
    import torch
    np.testing.assert_allclose(p.forward(torch.from_numpy(x).cuda()).cpu().numpy(),
                               net.forward(p_ref, x), rtol=1e-5, atol=1e-5)


LEARNER_MODES = {"eager": {}, "graph": {"graph": True}, "fused": {"fused": True},
                 "fused_graph": {"fused": True, "graph": True}}


def _load_state(gl, rl):
    """Copy the reference learner's weights and Adam moments into ours, in place
    (the fused/graphed paths hold these tensors' addresses)."""
    import torch
    pairs = list(zip(gl.online.weights + gl.online.biases, rl.online.weights + rl.online.biases))
    pairs += zip(gl.target.weights + gl.target.biases, rl.target.weights + rl.target.biases)
    ga, ra = gl.adam, rl.adam
    pairs += zip(ga.m_weights + ga.m_biases + ga.v_weights + ga.v_biases,
                 ra.m_weights + ra.m_biases + ra.v_weights + ra.v_biases)
    for t, a in pairs:
        t.copy_(torch.from_numpy(np.ascontiguousarray(a)))


@pytest.mark.parametrize("mode", list(LEARNER_MODES))
def test_ddqn_updates_match_reference(mode):
    """12 updates against the reference learner (ddqn.py:54-77).

    eager/graph (torch, cuBLAS) run chained. The fused kernels restart every
    update from the reference's state. The reason: Adam's first steps are ~lr*sign(g).
    A legitimate fp32 difference can flip the sign of a near-zero gradient
    element (e.g. a ReLU mask on a pre-activation within rounding noise of 0).
    Chaining then amplifies that into a 2*lr weight difference. On such an
    element the fused kernel was the one agreeing with an fp64 recomputation.
    Per update, targets, loss, |td| and the gradient moments (m = (1-b1) g
    accumulated) must match."""
    ref()
    from color_rl import net
    from color_rl.ddqn import DdqnConfig as RC, DdqnLearner as RL
    from color_rl.replay import TransitionBatch as RTB
    from paper_2305_04180_b200.asl import DdqnConfig, DdqnLearner, QNet, compute_targets
    from color_rl.ddqn import compute_targets as ref_targets
    chained = not LEARNER_MODES[mode].get("fused")
    rl = RL(net.init_params(np.random.default_rng(3), SIZES), RC(target_sync_period=5))
    gl = DdqnLearner(QNet.init(np.random.default_rng(3), SIZES), DdqnConfig(target_sync_period=5),
                     **LEARNER_MODES[mode])
    rng = np.random.default_rng(11)
    for k in range(12):
        arrs = _batch(rng, 256)
        tb = _tb(arrs)
        if not chained:
            _load_state(gl, rl)
        y_ref = ref_targets(RTB(*arrs), rl.online, rl.target, 0.98)
        y = compute_targets(tb, gl.online, gl.target, 0.98).cpu().numpy()
        np.testing.assert_allclose(y, y_ref, rtol=1e-4, atol=1e-5)
        sr = rl.update(RTB(*arrs))
        sg = gl.update(tb)
        assert sg.version == sr.version and sg.target_synced == sr.target_synced
        np.testing.assert_allclose(sg.loss, sr.loss, rtol=1e-4)
        np.testing.assert_allclose(sg.mean_abs_td, sr.mean_abs_td, rtol=1e-4)
        if not chained:
            # >= 99 % of every gradient tensor within 1e-4: a ReLU-mask flip on
            # one near-zero pre-activation legitimately moves one column
            for mg, mr in zip(gl.adam.m_weights + gl.adam.m_biases,
                              rl.adam.m_weights + rl.adam.m_biases):
                a = mg.cpu().numpy()
                bad = np.abs(a - mr) > 1e-4 * np.abs(mr) + 1e-5 * float(np.abs(mr).max())
                assert bad.mean() <= 0.01, (k, int(bad.sum()), bad.size)
    if chained:
        for w, wr in zip(gl.online.weights, rl.online.weights):
            np.testing.assert_allclose(w.cpu().numpy(), wr, rtol=1e-4, atol=1e-6)
        for w, wr in zip(gl.target.weights, rl.target.weights):
            np.testing.assert_allclose(w.cpu().numpy(), wr, rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("mode", ["fused", "fused_graph"])
def test_fused_updates_chained_against_reference(mode):
    """The fused learner run chained for 20 updates (no restarts) against the
    reference learner on the same batches.  Adam's early steps are about
    lr * sign(g), so an element whose gradient is within fp32 rounding of 0
    may step the other way; every weight must therefore be within 1e-4
    relative or 2 lr per update of the reference, and at least 99.9 % of the
    elements of every tensor within 1e-4 relative (+1e-6 absolute).  Losses
    and |td| agree to 1e-4 at every update."""
    ref()
    from color_rl import net
    from color_rl.ddqn import DdqnConfig as RC, DdqnLearner as RL
    from color_rl.replay import TransitionBatch as RTB
    from paper_2305_04180_b200.asl import DdqnConfig, DdqnLearner, QNet
    lr, n_up = 1e-4, 20
    rl = RL(net.init_params(np.random.default_rng(5), SIZES), RC(target_sync_period=7))
    gl = DdqnLearner(QNet.init(np.random.default_rng(5), SIZES), DdqnConfig(target_sync_period=7),
                     **LEARNER_MODES[mode])
    rng = np.random.default_rng(17)
    for k in range(n_up):
        arrs = _batch(rng, 256)
        sr = rl.update(RTB(*arrs))
        sg = gl.update(_tb(arrs))
        assert sg.version == sr.version and sg.target_synced == sr.target_synced
        np.testing.assert_allclose(sg.loss, sr.loss, rtol=1e-4)
        np.testing.assert_allclose(sg.mean_abs_td, sr.mean_abs_td, rtol=1e-4)
    for mine, theirs in ((gl.online.weights + gl.online.biases, rl.online.weights + rl.online.biases),
                         (gl.target.weights + gl.target.biases, rl.target.weights + rl.target.biases)):
        for w, wr in zip(mine, theirs):
            a = w.cpu().numpy()
            dev = np.abs(a - wr)
            assert (dev <= 1e-4 * np.abs(wr) + 2 * lr * n_up).all(), float(dev.max())
            assert (dev > 1e-4 * np.abs(wr) + 1e-6).mean() <= 1e-3, int((dev > 1e-4 * np.abs(wr) + 1e-6).sum())


def test_fused_adam_bit_exact_vs_reference():
    """sp_adam_step over all six tensors == net.py:151-161 adam_step (numpy
    fp32, weak Python-float scalars) bit for bit, over several steps."""
    ref()
    from color_rl import net
    from paper_2305_04180_b200.asl import AdamState, QNet, adam_step
    import torch
    p_ref = net.init_params(np.random.default_rng(12), SIZES)
    st_ref = net.AdamState.for_params(p_ref, lr=3e-4)
    p = QNet.from_numpy(p_ref.weights, p_ref.biases)
    st = AdamState.for_params(p, lr=3e-4)
    rng = np.random.default_rng(13)
    for _ in range(7):
        gw = [rng.standard_normal(w.shape).astype(np.float32) * 1e-2 for w in p_ref.weights]
        gb = [rng.standard_normal(b.shape).astype(np.float32) * 1e-2 for b in p_ref.biases]
        net.adam_step(p_ref, net.Gradients(gw, gb), st_ref)
        adam_step(p, [torch.from_numpy(g).cuda() for g in gw],
                  [torch.from_numpy(g).cuda() for g in gb], st)
    assert p.version == p_ref.version == 7
    for a, b in zip(p.weights + p.biases + st.m_weights + st.v_weights,
                    p_ref.weights + p_ref.biases + st_ref.m_weights + st_ref.v_weights):
        assert np.array_equal(a.cpu().numpy(), b)


@pytest.mark.parametrize("mode", ["graph", "fused", "fused_graph"])
def test_graphed_update_nonfinite_aborts_and_keeps_params(mode):
    """ddqn.py:66-71 / test_ddqn.py:113-119: a non-finite loss raises
    TrainingDiverged; the gated graph leaves parameters, moments and the
    Adam step count untouched, and the next finite update proceeds."""
    from paper_2305_04180_b200.asl import DdqnLearner, QNet, TrainingDiverged
    import torch
    gl = DdqnLearner(QNet.init(np.random.default_rng(4), SIZES), **LEARNER_MODES[mode])
    rng = np.random.default_rng(5)
    gl.update(_tb(_batch(rng, 64)))
    before = [w.clone() for w in gl.online.weights + gl.adam.m_weights]
    bad = _batch(rng, 64)
    bad[0][3, 7] = np.inf
    with pytest.raises(TrainingDiverged):
        gl.update(_tb(bad))
    for x, y in zip(gl.online.weights + gl.adam.m_weights, before):
        assert torch.equal(x, y)
    assert gl.adam.step == 1 and gl.online.version == 1
    eager = DdqnLearner(QNet.init(np.random.default_rng(4), SIZES))
    rng = np.random.default_rng(5)
    eager.update(_tb(_batch(rng, 64)))
    _batch(rng, 64)
    nxt = _batch(rng, 64)
    s1, s2 = gl.update(_tb(nxt)), eager.update(_tb(nxt))
    assert s1.version == s2.version == 2
    np.testing.assert_allclose(s1.loss, s2.loss, rtol=1e-4)
    for w, we in zip(gl.online.weights, eager.online.weights):
        np.testing.assert_allclose(w.cpu().numpy(), we.cpu().numpy(), rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("mode", ["graph", "fused"])
def test_graphed_update_samples_into_static_batch(mode):
    """ReplayBuffer.sample(out=learner.graph_batch(...)) fills the graph's
    static batch in place; the update equals the eager one on the same rows."""
    from paper_2305_04180_b200 import PhiloxGenerator, ReplayBuffer
    from paper_2305_04180_b200.asl import DdqnLearner, QNet
    import torch
    buf = ReplayBuffer(4096, 37)
    s, a, r, s2, d = _tb(_batch(np.random.default_rng(6), 3000))
    buf.append_batch(s, a, r, s2, d)
    gl = DdqnLearner(QNet.init(np.random.default_rng(8), SIZES), **LEARNER_MODES[mode])
    el = DdqnLearner(QNet.init(np.random.default_rng(8), SIZES))
    for k in range(6):
        out = gl.graph_batch(256, 37)
        got = buf.sample(256, PhiloxGenerator(9, 0, ctr=256 * k), out=out)
        assert got is out
        want = buf.sample(256, PhiloxGenerator(9, 0, ctr=256 * k))
        for x, y in zip(out, want):
            assert torch.equal(x, y)
        sg, se = gl.update(out), el.update(want)
        np.testing.assert_allclose(sg.loss, se.loss, rtol=1e-4)
    with pytest.raises(ValueError):
        buf.sample(128, PhiloxGenerator(9), out=gl.graph_batch(256, 37))


@pytest.mark.parametrize("batch", [256, 64, 13])
def test_fused_gradient_matches_torch(batch):
    """One update from identical weights: the first Adam moment m = (1-b1) g
    of every tensor equals the torch backward's to fp32 summation-order noise
    (the direct gradient check of sp_ddqn_update), and so does the loss."""
    import torch
    from paper_2305_04180_b200.asl import DdqnLearner, QNet
    rng = np.random.default_rng(21)
    arrs = _batch(rng, batch)
    eager = DdqnLearner(QNet.init(np.random.default_rng(22), SIZES))
    fused = DdqnLearner(QNet.init(np.random.default_rng(22), SIZES), fused=True)
    se, sf = eager.update(_tb(arrs)), fused.update(_tb(arrs))
    np.testing.assert_allclose(sf.loss, se.loss, rtol=1e-5)
    np.testing.assert_allclose(sf.mean_abs_td, se.mean_abs_td, rtol=1e-5)
    for me, mf in zip(eager.adam.m_weights + eager.adam.m_biases,
                      fused.adam.m_weights + fused.adam.m_biases):
        a, b = me.cpu().numpy(), mf.cpu().numpy()
        scale = np.abs(a).max()
        np.testing.assert_allclose(b, a, rtol=1e-4, atol=1e-5 * scale)
    for ve, vf in zip(eager.adam.v_weights, fused.adam.v_weights):
        np.testing.assert_allclose(vf.cpu().numpy(), ve.cpu().numpy(), rtol=1e-3,
                                   atol=1e-8 * float(ve.max()))
    del torch


def test_vem_epsilons_and_selection_match_reference():
    ref()
    from color_rl.asl.vem import VemSchedule as RV, select_actions as ref_select
    from paper_2305_04180_b200.asl import VemSchedule, select_actions
    import torch
    for n, t in ((16, 0), (16, 250_000), (4096, 10), (4096, 999_999), (3, 5)):
        kw = dict(or_init=min(16, n), or_final=min(3, n))
        assert np.array_equal(VemSchedule(n, **kw).epsilons(t), RV(n, **kw).epsilons(t))
    q = np.random.default_rng(2).standard_normal((4096, 5)).astype(np.float32)
    q[:8] = 0.0  # ties -> lowest index
    eps = RV(4096).epsilons(100)
    want = ref_select(q, eps, PhiloxStream(5, 0xAC, tag=3))
    g = PhiloxStream(5, 0xAC, tag=3)
    got = select_actions(torch.from_numpy(q).cuda(), eps, g).cpu().numpy()
    assert np.array_equal(got, want)
    assert g.ctr == 2 * 4096


def test_tfm_matches_reference():
    ref()
    from color_rl.asl import tfm as rt
    from paper_2305_04180_b200 import asl
    cfg, rcfg = asl.TfmConfig(4096, 256, 256, warmup_samples=3), rt.TfmConfig(4096, 256, 256, warmup_samples=3)
    a, b = asl.TfmState(), rt.TfmState()
    rng = np.random.default_rng(0)
    for _ in range(20):
        v, w = rng.uniform(1e-3, 5e-3), rng.uniform(1e-4, 1e-3)
        a.record_interaction(v); b.record_interaction(v)
        a.record_optimization(w); b.record_optimization(w)
        assert a.actor_sleep(cfg) == b.actor_sleep(rcfg)
        assert a.learner_sleep(cfg) == b.learner_sleep(rcfg)
    assert cfg.rho == rcfg.rho == 4096


def test_checkpoint_bytes_compatible():
    ref()
    from color_rl import net
    from paper_2305_04180_b200.asl import CheckpointError, QNet
    p_ref = net.init_params(np.random.default_rng(9), SIZES)
    p_ref.version = 42
    p = QNet.from_numpy(p_ref.weights, p_ref.biases, 42)
    assert p.to_bytes() == net.to_bytes(p_ref)
    back = QNet.from_bytes(net.to_bytes(p_ref), expect_sizes=SIZES)
    assert back.version == 42 and back.to_bytes() == p.to_bytes()
    with pytest.raises(CheckpointError):
        QNet.from_bytes(b"NOTCOLOR" + p.to_bytes()[8:])
    with pytest.raises(CheckpointError):
        QNet.from_bytes(p.to_bytes()[:-3])


def test_asl_session_cfg5_shape():
    """cfg5 shape: 4096 CUDA envs -> 1M GPU replay -> batch-256 DDQN with TFM
    pacing; runs a few seconds, both loops make progress, no failures."""
    import time
    from paper_2305_04180_b200 import ReplayBuffer, VecEnv
    from paper_2305_04180_b200.asl import (DdqnConfig, DdqnLearner, QNet, Sharer, TfmConfig,
                                           VemSchedule, start_session)
    n = 4096
    env = VecEnv(load_maps(16), n, ranges(0.3), config(32), check_actions=False)
    states = env.reset_all(0)
    algo = DdqnLearner(QNet.init(np.random.default_rng(0), SIZES), DdqnConfig(), fused=True,
                       graph=True)
    sharer = Sharer(ReplayBuffer(1_000_000, 37))
    tfm = TfmConfig(n, 256.0, 256)
    session = start_session(sharer, env, states, algo.online, VemSchedule(n), tfm,
                            max_steps=n * 400, algo=algo, learn_start=20_000, upload_period=50,
                            seed=0)
    t0 = time.time()
    while session.running and time.time() - t0 < 6.0:
        time.sleep(0.1)
    session.abort()
    session.wait(timeout=30)
    assert sharer.t_step > 20_000
    assert sharer.b_step > 10
    assert len(sharer.buffer) == min(sharer.t_step, 1_000_000)
    assert sharer.publish_count >= 1 + sharer.b_step // 50
    snap = env.snapshot_stats()
    assert snap.episodes > 0


def test_published_snapshot_checksum():
    """sharer.py:18-31: the snapshot's crc32 is that of its COLORNET bytes and
    verify_snapshot holds; the snapshot is a private copy."""
    import zlib
    from paper_2305_04180_b200 import ReplayBuffer
    from paper_2305_04180_b200.asl import QNet, Sharer, verify_snapshot
    p = QNet.init(np.random.default_rng(31), SIZES)
    sh = Sharer(ReplayBuffer(16, 37))
    snap = sh.publish_params(p)
    version, params, crc = snap
    assert crc == zlib.crc32(p.to_bytes()) and verify_snapshot(snap)
    p.weights[0].add_(1.0)  # the learner keeps training: the snapshot is unaffected
    assert snap.checksum == crc and verify_snapshot(snap)
    assert sh.fetch_params(version - 1) is snap and sh.fetch_params(version) is None


def test_update_from_samples_inside_the_graph():
    """DdqnLearner.update_from with fused+graph: sp_rb_sample_dev inside the
    CUDA graph draws the same rows as ReplayBuffer.sample with the same
    PhiloxGenerator (the device counter is mirrored in rng.ctr), so weights
    match a fused learner fed by host-side sampling bit for bit; draws made
    with the rng elsewhere are picked up."""
    import torch
    from paper_2305_04180_b200 import BufferNotReady, PhiloxGenerator, ReplayBuffer
    from paper_2305_04180_b200.asl import DdqnLearner, QNet
    buf = ReplayBuffer(5000, 37)
    with pytest.raises(BufferNotReady):
        DdqnLearner(QNet.init(np.random.default_rng(8), SIZES), fused=True, graph=True).update_from(
            buf, PhiloxGenerator(1), 64)
    s, a, r, s2, d = _tb(_batch(np.random.default_rng(6), 3000))
    buf.append_batch(s, a, r, s2, d)
    gl = DdqnLearner(QNet.init(np.random.default_rng(8), SIZES), fused=True, graph=True)
    hl = DdqnLearner(QNet.init(np.random.default_rng(8), SIZES), fused=True)
    g_rng, h_rng = PhiloxGenerator(9, 3), PhiloxGenerator(9, 3)
    for k in range(8):
        if k == 4:  # both streams draw outside update_from: the device counter resyncs
            buf.sample(32, g_rng)
            buf.sample(32, h_rng)
        if k == 6:  # more rows arrive between updates (device fill level follows)
            s, a, r, s2, d = _tb(_batch(np.random.default_rng(60 + k), 1000))
            buf.append_batch(s, a, r, s2, d)
        sg = gl.update_from(buf, g_rng, 256)
        sh = hl.update(buf.sample(256, h_rng))
        assert g_rng.ctr == h_rng.ctr
        assert sg.loss == sh.loss and sg.version == sh.version
    for w, wh in zip(gl.online.weights + gl.online.biases, hl.online.weights + hl.online.biases):
        assert torch.equal(w, wh)


@pytest.mark.parametrize("n,t_step,env0,n_envs", [(4096, 100, 0, 4096), (4096, 499_999, 0, 4096),
                                                   (1000, 10**7, 3000, 4096), (37, 0, 0, 37)])
def test_fused_actor_matches_reference(n, t_step, env0, n_envs):
    """sp_actor_select (one launch: forward, device VEM epsilons, epsilon-greedy)
    against the unmodified reference: net.forward (Q within 1e-5), VEM
    epsilons of copies env0.. at t_step, select_actions on the same Philox
    draws -- actions identical wherever the reference's top two Q-values are
    not within fp32 summation-order noise (1e-5) of each other."""
    ref()
    import torch
    from color_rl import net
    from color_rl.asl.vem import VemSchedule as RV, select_actions as ref_select
    from paper_2305_04180_b200.asl import QNet, VemSchedule, select_actions_fused
    p_ref = net.init_params(np.random.default_rng(3), SIZES)
    p = QNet.init(np.random.default_rng(3), SIZES)
    x = np.random.default_rng(n + t_step).standard_normal((n, 37)).astype(np.float32)
    kw = dict(or_init=min(16, n_envs), or_final=min(3, n_envs), decay_steps=500_000)
    q_ref = net.forward(p_ref, x)
    eps = RV(n_envs, **kw).epsilons(t_step)[env0:env0 + n]
    want = ref_select(q_ref, eps, PhiloxStream(9, 0xAC, tag=3))
    g = PhiloxStream(9, 0xAC, tag=3)
    q = torch.empty((n, 5), dtype=torch.float32, device="cuda")
    got = select_actions_fused(p, torch.from_numpy(x).cuda(), VemSchedule(n_envs, **kw), t_step, g,
                               env0=env0, q_out=q).cpu().numpy()
    assert g.ctr == 2 * n
    np.testing.assert_allclose(q.cpu().numpy(), q_ref, rtol=1e-5, atol=1e-5)
    top2 = np.sort(q_ref, axis=1)[:, -2:]
    clear = (top2[:, 1] - top2[:, 0]) > 1e-5
    assert clear.mean() > 0.99
    assert np.array_equal(got[clear], want[clear])


def test_fused_actor_equals_torch_path_and_explores():
    """The fused kernel against this package's own torch path (QNet.forward +
    select_actions with host epsilons): same draws, same actions away from
    near-ties; at e_min = e_max = 1 every action is the random draw."""
    import torch
    from paper_2305_04180_b200.asl import QNet, VemSchedule, select_actions, select_actions_fused
    from paper_2305_04180_b200.replay import PhiloxGenerator
    p = QNet.init(np.random.default_rng(5), SIZES)
    n = 65536
    x = torch.randn((n, 37), generator=torch.Generator().manual_seed(0)).cuda()
    vem = VemSchedule(n)
    q = p.forward(x)
    g1, g2 = PhiloxGenerator(4, 0xAC), PhiloxGenerator(4, 0xAC)
    g1.tag = g2.tag = 3
    want = select_actions(q, vem.epsilons(1234), g1).cpu().numpy()
    got = select_actions_fused(p, x, vem, 1234, g2).cpu().numpy()
    assert g1.ctr == g2.ctr
    qs = torch.sort(q, dim=1).values
    clear = ((qs[:, -1] - qs[:, -2]) > 1e-5).cpu().numpy()
    assert np.array_equal(got[clear], want[clear])
    allr = VemSchedule(n, e_min=1.0, e_max=1.0)
    g3, g4 = PhiloxGenerator(4, 0xAC), PhiloxGenerator(4, 0xAC)
    g3.tag = g4.tag = 3
    got = select_actions_fused(p, x, allr, 0, g3).cpu().numpy()
    from paper_2305_04180_b200.asl import philox_fill
    philox_fill(n, g4, 0, 0.0, 1.0)
    rnd = philox_fill(n, g4, 1, 0, 5).cpu().numpy()
    assert np.array_equal(got, rnd)
