"""cfg5: the full ASL loop -- 4096 envs feeding a 1M-transition replay ring,
batch-256 DDQN learner with TFM pacing (BASELINE.json configs[4]).

    python tools/bench_asl.py [--seconds 20] [--impl ours|reference]

Reports interaction throughput (env-steps/s = t_step / wall), learner
updates/s (b_step / wall), measured TPS (B * b_step / t_step), and the
learner's mean update time; the reference runs its own threads
(color_rl.asl.loops.start_session, numpy DDQN, Cython env) on the host.
TFM pacing makes this learner-bound by construction (rho = N*TPS/B = 4096).
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

N, TPS, B, CAP, LEARN_START, UPLOAD = 4096, 256.0, 256, 1_000_000, 30_000, 50


def run_ours(seconds, eager=False, learner="fused"):
    import torch
    from helpers import config, load_maps, ranges
    from paper_2305_04180_b200 import ReplayBuffer, VecEnv
    from paper_2305_04180_b200.asl import (DdqnConfig, DdqnLearner, QNet, Sharer, TfmConfig,
                                           VemSchedule, start_session)
    env = VecEnv(load_maps(16), N, ranges(0.3), config(32), check_actions=False)
    states = env.reset_all(0)
    algo = DdqnLearner(QNet.init(np.random.default_rng(0), (37, 256, 128, 5)), DdqnConfig(),
                       graph=not eager, fused=learner == "fused")
    sharer = Sharer(ReplayBuffer(CAP, 37))
    tfm = TfmConfig(N, TPS, B)
    t0 = time.perf_counter()
    s = start_session(sharer, env, states, algo.online, VemSchedule(N), tfm, N * 10**6, algo,
                      LEARN_START, UPLOAD, 0)
    while time.perf_counter() - t0 < seconds and not sharer.failed:
        time.sleep(0.05)
    s.abort()
    s.wait(timeout=60)
    wall = time.perf_counter() - t0
    torch.cuda.synchronize()
    return sharer, wall


def run_actor(iters=300, fused=True):
    """The actor's iteration alone (no learner): forward + VEM + selection,
    env step, ring append, 4096 envs -- sp_actor_select (fused) against the
    torch path (addmm forward, host VEM epsilons, philox draws, argmax)."""
    import torch
    from helpers import config, load_maps, ranges
    from paper_2305_04180_b200 import ReplayBuffer, VecEnv
    from paper_2305_04180_b200.asl import QNet, VemSchedule, select_actions, select_actions_fused
    from paper_2305_04180_b200.replay import PhiloxGenerator
    env = VecEnv(load_maps(16), N, ranges(0.3), config(32), check_actions=False)
    states = env.reset_all(0)
    p = QNet.init(np.random.default_rng(0), (37, 256, 128, 5))
    rb = ReplayBuffer(CAP, 37)
    vem = VemSchedule(N)
    g = PhiloxGenerator(0, 0xAC)
    g.tag = 3
    outs = [env.new_batch(), env.new_batch()]
    acts = [torch.empty(N, dtype=torch.int64, device=env.device) for _ in range(2)]
    t_step = 0

    def it(k):
        nonlocal states, t_step
        if fused:
            a = select_actions_fused(p, states, vem, t_step, g, out=acts[k & 1])
        else:
            a = select_actions(p.forward(states), vem.epsilons(t_step), g)
        b = outs[k & 1]
        env.step_device(a.data_ptr(), b)
        rb.append_batch(states, a, b.rewards, b.store_states, b.dones)
        states = b.states
        t_step += N
    for k in range(20):
        it(k)
    torch.cuda.synchronize()
    s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    s_.record()
    for k in range(iters):
        it(k)
    e_.record()
    e_.synchronize()
    wall = time.perf_counter() - w0
    dev_s = s_.elapsed_time(e_) / 1e3
    return {"mode": "actor only (no learner), " + ("sp_actor_select" if fused else "torch path"),
            "iters": iters, "us_per_iter_device": dev_s / iters * 1e6,
            "us_per_iter_wall": wall / iters * 1e6, "env_steps_per_s": N * iters / wall}


def run_reference(seconds):
    from oracle import oracle as O
    O.import_reference(37)
    from color_rl import net
    from color_rl.asl.loops import start_session
    from color_rl.asl.sharer import Sharer
    from color_rl.asl.tfm import TfmConfig
    from color_rl.asl.vem import VemSchedule
    from color_rl.ddqn import DdqnLearner
    from color_rl.replay import ReplayBuffer
    from color_rl.sim.gridmap import GridMap as RG
    from color_rl.sim.params import DiversityRanges, EnvConfig, LidarConfig, SimParams
    from color_rl.vecenv import VecEnv
    from helpers import load_maps
    maps = [RG.from_text(m.to_text()) for m in load_maps(16)]
    env = VecEnv(maps, N, DiversityRanges.around(SimParams(), 0.3),
                 EnvConfig(lidar=LidarConfig(n_beams=32)))
    states = env.reset_all(0)
    params = net.init_params(np.random.default_rng(0), (37, 256, 128, 5))
    algo = DdqnLearner(params)
    sharer = Sharer(ReplayBuffer(CAP, 37))
    tfm = TfmConfig(N, TPS, B)
    t0 = time.perf_counter()
    s = start_session(sharer, env, states, algo.online, VemSchedule(N), tfm, N * 10**6, algo,
                      LEARN_START, UPLOAD, 0)
    while time.perf_counter() - t0 < seconds and not sharer.failed:
        time.sleep(0.05)
    s.abort()
    s.wait(timeout=120)
    return sharer, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=20.0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--eager", action="store_true", help="learner updates without CUDA graph")
    ap.add_argument("--learner", default="fused", choices=["fused", "torch"],
                    help="fused sp_ddqn_update kernels or the torch update")
    ap.add_argument("--actor-only", action="store_true",
                    help="time the actor iteration alone, fused kernel vs the torch path")
    a = ap.parse_args()
    if a.actor_only:
        for fused in (True, False):
            print(json.dumps(run_actor(fused=fused)))
        return
    if a.impl == "ours":
        sharer, wall = run_ours(a.seconds, a.eager, a.learner)
    else:
        sharer, wall = run_reference(a.seconds)
    tfm = sharer.tfm
    print(json.dumps({
        "workload": "cfg5: 4096 envs (16 maps, diversity 0.3, 32 beams) -> 1M replay -> "
                    "batch-256 DDQN [37,256,128,5], TPS 256 (rho 4096), learn_start 30000",
        "impl": a.impl, "graph": a.impl == "ours" and not a.eager,
        "learner": a.learner if a.impl == "ours" else "reference numpy", "wall_s": wall, "t_step": sharer.t_step, "b_step": sharer.b_step,
        "env_steps_per_s": sharer.t_step / wall, "updates_per_s": sharer.b_step / wall,
        "measured_tps": sharer.measured_tps(B),
        "actor_period_ms": None if tfm.v_period_s is None else tfm.v_period_s * 1e3,
        "learner_period_ms": None if tfm.b_period_s is None else tfm.b_period_s * 1e3,
        "buffer_size": len(sharer.buffer), "failed": sharer.failed}))


if __name__ == "__main__":
    main()
