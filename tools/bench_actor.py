"""sp_actor_select alone (host-side tool): device time per launch of the fused
actor (forward of the [5+R, 256, 128, 5] MLP, VEM epsilons, epsilon-greedy) at
n rows, CUDA events around K launches after warm-up, L2 not flushed (the
weights are re-staged from L2 by every CTA anyway).  Prints one JSON line per n.

    python tools/bench_actor.py [n ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(ns):
    import numpy as np
    import torch
    from paper_2305_04180_b200.asl import QNet, VemSchedule, select_actions_fused
    from paper_2305_04180_b200.replay import PhiloxGenerator
    dev = torch.device("cuda", 0)
    sizes = (37, 256, 128, 5)
    p = QNet.init(np.random.default_rng(5), sizes)
    flop_row = 2 * sum(a * b for a, b in zip(sizes[:-1], sizes[1:]))
    for n in ns:
        x = torch.randn((n, 37), generator=torch.Generator().manual_seed(0)).to(dev)
        vem = VemSchedule(n)
        g = PhiloxGenerator(4, 0xAC)
        g.tag = 3
        out = torch.empty(n, dtype=torch.int64, device=dev)
        for _ in range(5):
            select_actions_fused(p, x, vem, 1234, g, out=out)
        K = 50
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(K):
            select_actions_fused(p, x, vem, 1234, g, out=out)
        e.record()
        e.synchronize()
        us = s.elapsed_time(e) * 1e3 / K
        print(json.dumps({"n": n, "us_per_launch": us, "rows_per_s": n / us * 1e6,
                          "tflops": flop_row * n / us / 1e6}))


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [4096, 65536])
