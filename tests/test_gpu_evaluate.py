"""Greedy evaluation on the GPU against the reference's
``evaluate_params`` (pkg/tests/test_evaluate.py cases, then report parity vs
the unmodified reference driven through the Philox shim)."""

import numpy as np
import pytest

from helpers import config, load_maps, make_map, ranges
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _params(seed, sizes=(32, 256, 128, 5)):
    from paper_2305_04180_b200.asl import QNet
    return QNet.init(np.random.default_rng(seed), sizes)


def test_degenerate_map_spawn_on_goal_scores_one():  # test_evaluate.py:8-18
    from paper_2305_04180_b200.evaluate import evaluate_params
    from paper_2305_04180_b200.sim import EnvConfig, SimParams
    m = make_map(60, goal=(25.0, 25.0), goal_radius=12.0, spawn=(22.0, 22.0, 28.0, 28.0))
    rep = evaluate_params(_params(0), [m], ["degenerate"], episodes_per_map=8, seed=1,
                          config=EnvConfig(), nominal=SimParams())
    assert rep.arrival_rate == 1.0
    assert rep.results[0].episodes == 8
    assert rep.results[0].mean_steps <= 3


def test_report_deterministic_for_seed():  # test_evaluate.py:21-29
    from paper_2305_04180_b200.evaluate import evaluate_params
    from paper_2305_04180_b200.sim import EnvConfig
    m = make_map(60)
    cfg = EnvConfig(timeout_steps=120)
    p = _params(1)
    a = evaluate_params(p, [m], ["m"], 6, seed=5, config=cfg)
    b = evaluate_params(p, [m], ["m"], 6, seed=5, config=cfg)
    assert a.to_dict() == b.to_dict()
    c = evaluate_params(p, [m], ["m"], 6, seed=6, config=cfg)
    assert a.to_dict() != c.to_dict() or a.arrival_rate == c.arrival_rate


def test_counts_partition_episodes():  # test_evaluate.py:32-38
    from paper_2305_04180_b200.evaluate import evaluate_params
    from paper_2305_04180_b200.sim import EnvConfig
    m = make_map(60, blocks=((38, 8, 44, 34),))
    rep = evaluate_params(_params(2), [m], ["m"], 10, seed=3, config=EnvConfig(timeout_steps=80))
    r = rep.results[0]
    assert r.arrivals + r.collisions + r.timeouts == r.episodes == 10


def test_randomization_flag_changes_rollouts():  # test_evaluate.py:41-48
    from paper_2305_04180_b200.evaluate import evaluate_params
    from paper_2305_04180_b200.sim import EnvConfig
    m = make_map(60)
    cfg = EnvConfig(timeout_steps=60)
    p = _params(3)
    plain = evaluate_params(p, [m], ["m"], 6, seed=7, config=cfg)
    rand = evaluate_params(p, [m], ["m"], 6, seed=7, config=cfg, randomize_fraction=0.3)
    assert plain.to_dict() != rand.to_dict()


def test_summarize_rates():  # test_evaluate.py:51-57
    from paper_2305_04180_b200.evaluate import evaluate_params, summarize_rates
    m = make_map(60, goal=(25.0, 25.0), goal_radius=12.0, spawn=(22.0, 22.0, 28.0, 28.0))
    p = _params(4)
    reports = [evaluate_params(p, [m], ["m"], 4, seed=s) for s in (0, 1)]
    s = summarize_rates(reports)
    assert s["mean"] == 1.0 and s["std"] == 0.0 and s["per_seed"] == [1.0, 1.0]


def _compare_reports(got, want):
    g, w = got.to_dict(), want.to_dict()
    assert g["seed"] == w["seed"] and g["episodes"] == w["episodes"]
    for a, b in zip(g["maps"], w["maps"]):
        for k in ("name", "episodes", "arrivals", "collisions", "timeouts", "mean_steps"):
            assert a[k] == b[k], (k, a, b)
        np.testing.assert_allclose(a["mean_return"], b["mean_return"], rtol=1e-5, atol=1e-6)


@pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("div,n_beams,eps,timeout", [
    (0.0, 27, 24, 200),     # reference defaults (STATE_DIM 32)
    (0.3, 32, 32, 150),     # cfg2-like diversity
])
def test_reports_match_reference(div, n_beams, eps, timeout):
    """Per-map layout: the reference's evaluate_params (numpy forward, stock
    Cython env, Philox-shimmed RNG) and ours give the same report."""
    O.import_reference(5 + n_beams)
    import color_rl.vecenv as vmod
    from color_rl import net
    from color_rl.evaluate import evaluate_params as ref_eval
    from color_rl.sim.gridmap import GridMap as RG
    from color_rl.sim.params import EnvConfig as REC, LidarConfig as RLC, SimParams as RSP
    from oracle.philox_shim import reference_rng_proxy
    from paper_2305_04180_b200.evaluate import evaluate_params
    from paper_2305_04180_b200.sim import SimParams
    maps = load_maps(3)
    names = [f"map{i}" for i in range(len(maps))]
    p_ref = net.init_params(np.random.default_rng(11), (5 + n_beams, 256, 128, 5))
    with reference_rng_proxy(vmod):
        want = ref_eval(p_ref, [RG.from_text(m.to_text()) for m in maps], names, eps, seed=13,
                        config=REC(lidar=RLC(n_beams=n_beams), timeout_steps=timeout),
                        nominal=RSP(), randomize_fraction=div)
    got = evaluate_params(p_ref, maps, names, eps, seed=13,
                          config=config(n_beams, timeout_steps=timeout), nominal=SimParams(),
                          randomize_fraction=div)
    _compare_reports(got, want)


def test_fused_layout_matches_oracle_rollout():
    """fused=True: one launch for all maps; the same greedy rollout on the C
    oracle (numpy forward) gives identical per-map outcomes."""
    from paper_2305_04180_b200.evaluate import _map_seed, evaluate_params
    maps = load_maps(4)
    names = [f"m{i}" for i in range(4)]
    cfg = config(32, timeout_steps=120)
    p = _params(5, (37, 256, 128, 5))
    got = evaluate_params(p, maps, names, 16, seed=21, config=cfg, randomize_fraction=0.3,
                          fused=True)
    n = 4 * 16
    orc = O.OracleVecEnv(maps, n, ranges(0.3), cfg, map_index=np.repeat(np.arange(4), 16))
    w = [x.cpu().numpy() for x in p.weights]
    b = [x.cpu().numpy() for x in p.biases]

    def fwd(s):
        h = s.astype(np.float32)
        for i, (wi, bi) in enumerate(zip(w, b)):
            h = h @ wi + bi
            if i < len(w) - 1:
                h = np.maximum(h, 0)
        return h

    s = orc.reset_all(_map_seed(21, 0))
    for _ in range(cfg.timeout_steps + 1):
        s = orc.step_batch(np.argmax(fwd(s), axis=1)).states
    st = orc.stats()
    fe, fr, fs = st["first_event"], st["first_return"], st["first_steps"]
    assert (fe >= 0).all()
    for mi, r in enumerate(got.results):
        sl = slice(mi * 16, (mi + 1) * 16)
        assert r.arrivals == int((fe[sl] == 2).sum())
        assert r.collisions == int((fe[sl] == 1).sum())
        assert r.timeouts == int((fe[sl] == 3).sum())
        assert r.mean_steps == float(np.mean(fs[sl]))
        np.testing.assert_allclose(r.mean_return, np.mean(fr[sl]), rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("fused", [False, True])
def test_graphed_rollout_equals_stepwise(fused):
    """The CUDA-graph rollout (fused actor kernel with exploration off + env
    step, check_every steps per replay) gives the step-by-step cuBLAS/argmax
    rollout's report."""
    from paper_2305_04180_b200.evaluate import evaluate_params
    from paper_2305_04180_b200.sim import EnvConfig, LidarConfig
    maps = load_maps(4)
    cfg = EnvConfig(lidar=LidarConfig(n_beams=32), timeout_steps=200)
    p = _params(3, (37, 256, 128, 5))
    kw = dict(config=cfg, fused=fused, check_every=5)
    a = evaluate_params(p, maps, [f"m{i}" for i in range(4)], 64, seed=2, graph=True, **kw)
    b = evaluate_params(p, maps, [f"m{i}" for i in range(4)], 64, seed=2, graph=False, **kw)
    assert a.to_dict() == b.to_dict()
