"""Greedy evaluation throughput: evaluate_params over
16 maps, per-map (reference layout) and fused (one launch per step for all
maps), against the reference's evaluate_params on the host.

    python tools/bench_eval.py [--episodes 4096] [--ref-episodes 32]

Scored episodes/s = maps * episodes_per_map / wall; also env-steps/s (every
copy steps until the last first-episode ends).
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))

N_MAPS, BEAMS, TIMEOUT = 16, 32, 1000


def _policy_np():
    # a trained-looking policy is not available offline; random init, fixed seed
    return np.random.default_rng(0)


def run_ours(episodes, fused):
    import torch
    from helpers import config, load_maps
    from paper_2305_04180_b200.asl import QNet
    from paper_2305_04180_b200.evaluate import evaluate_params
    maps = load_maps(N_MAPS)
    names = [f"map{i}" for i in range(N_MAPS)]
    cfg = config(BEAMS, timeout_steps=TIMEOUT)
    p = QNet.init(_policy_np(), (5 + BEAMS, 256, 128, 5))
    evaluate_params(p, maps[:2], names[:2], 64, seed=0, config=cfg, fused=fused)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = evaluate_params(p, maps, names, episodes, seed=1, config=cfg, fused=fused)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"impl": "ours", "fused": fused, "episodes": rep.episodes, "wall_s": wall,
           "episodes_per_s": rep.episodes / wall, "arrival_rate": rep.arrival_rate,
           "mean_steps": float(np.mean([r.mean_steps for r in rep.results]))}
    # share of the wall time spent in the step kernel (torch profiler / CUPTI)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        evaluate_params(p, maps, names, episodes, seed=1, config=cfg, fused=fused)
        torch.cuda.synchronize()
        wall_p = time.perf_counter() - t0
    step_us = sum(e.device_time_total for e in prof.key_averages()
                  if "env_step_kernel" in e.key)
    actor_us = sum(e.device_time_total for e in prof.key_averages() if "actor_kernel" in e.key)
    out["step_kernel_share_of_wall"] = step_us / 1e6 / wall_p
    out["actor_kernel_share_of_wall"] = actor_us / 1e6 / wall_p
    out["profiled_wall_s"] = wall_p
    return out


def run_reference(episodes):
    from helpers import load_maps
    from oracle import oracle as O
    O.import_reference(5 + BEAMS)
    from color_rl import net
    from color_rl.evaluate import evaluate_params
    from color_rl.sim.gridmap import GridMap as RG
    from color_rl.sim.params import EnvConfig, LidarConfig
    maps = [RG.from_text(m.to_text()) for m in load_maps(N_MAPS)]
    names = [f"map{i}" for i in range(N_MAPS)]
    cfg = EnvConfig(lidar=LidarConfig(n_beams=BEAMS), timeout_steps=TIMEOUT)
    p = net.init_params(_policy_np(), (5 + BEAMS, 256, 128, 5))
    t0 = time.perf_counter()
    rep = evaluate_params(p, maps, names, episodes, seed=1, config=cfg)
    wall = time.perf_counter() - t0
    return {"impl": "reference", "episodes": rep.episodes, "wall_s": wall,
            "episodes_per_s": rep.episodes / wall, "arrival_rate": rep.arrival_rate,
            "threads": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--episodes", type=int, default=4096)
    ap.add_argument("--ref-episodes", type=int, default=32)
    a = ap.parse_args()
    for fused in (False, True):
        print(json.dumps(run_ours(a.episodes, fused)), flush=True)
    if a.ref_episodes > 0:
        print(json.dumps(run_reference(a.ref_episodes)), flush=True)


if __name__ == "__main__":
    main()
