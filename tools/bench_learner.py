"""DDQN learner update rate (batch 256, [37,256,128,5]): eager torch vs
CUDA-graphed, each sampling from a 1M GPU replay ring. Also times the
reference's numpy update on the host cores.

    python tools/bench_learner.py [--updates 2000]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))

B, D, CAP = 256, 37, 1_000_000


def run_ours(updates, graph, fused=False, in_graph_sample=False):
    import torch
    from paper_2305_04180_b200 import PhiloxGenerator, ReplayBuffer
    from paper_2305_04180_b200.asl import DdqnLearner, QNet
    dev = torch.device("cuda:0")
    buf = ReplayBuffer(CAP, D)
    g = torch.Generator(device=dev).manual_seed(0)
    n = 200_000
    buf.append_batch(torch.randn((n, D), device=dev, generator=g),
                     torch.randint(0, 5, (n,), device=dev, generator=g),
                     torch.randn(n, device=dev, generator=g),
                     torch.randn((n, D), device=dev, generator=g),
                     torch.rand(n, device=dev, generator=g) < 0.05)
    algo = DdqnLearner(QNet.init(np.random.default_rng(0), (D, 256, 128, 5)), graph=graph,
                       fused=fused)
    rng = PhiloxGenerator(1)

    def one():
        if in_graph_sample:  # learner_loop's path: sample + update in one graph replay
            algo.update_from(buf, rng, B)
        else:
            batch = buf.sample(B, rng, out=algo.graph_batch(B, D))
            algo.update(batch)  # reads the loss: one sync per update, as the learner loop does

    for _ in range(20):
        one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(updates):
        one()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return {"impl": "ours", "graph": graph, "fused": fused, "sample_in_graph": in_graph_sample,
            "updates": updates,
            "updates_per_s": updates / dt,
            "ms_per_update": dt / updates * 1e3}


def run_reference(updates):
    from oracle import oracle as O
    O.import_reference(D)
    from color_rl import net
    from color_rl.ddqn import DdqnLearner
    from color_rl.replay import TransitionBatch
    rng = np.random.default_rng(0)
    algo = DdqnLearner(net.init_params(rng, (D, 256, 128, 5)))
    batches = [TransitionBatch(rng.standard_normal((B, D)).astype(np.float32),
                               rng.integers(0, 5, B), rng.standard_normal(B).astype(np.float32),
                               rng.standard_normal((B, D)).astype(np.float32),
                               rng.random(B) < 0.05) for _ in range(16)]
    for k in range(5):
        algo.update(batches[k % 16])
    t0 = time.perf_counter()
    for k in range(updates):
        algo.update(batches[k % 16])
    dt = time.perf_counter() - t0
    return {"impl": "reference", "updates": updates, "updates_per_s": updates / dt,
            "ms_per_update": dt / updates * 1e3, "threads": os.cpu_count()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--updates", type=int, default=2000)
    ap.add_argument("--reference-updates", type=int, default=300)
    a = ap.parse_args()
    for graph, fused, ig in ((False, False, False), (True, False, False), (False, True, False),
                             (True, True, False), (True, True, True)):
        print(json.dumps(run_ours(a.updates, graph, fused, ig)), flush=True)
    print(json.dumps(run_reference(a.reference_updates)), flush=True)


if __name__ == "__main__":
    main()
