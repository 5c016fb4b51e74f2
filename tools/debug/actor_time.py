"""Device time of one sp_actor_select launch at several row counts (debug)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np, torch
from paper_2305_04180_b200.asl import QNet, VemSchedule, select_actions_fused
from paper_2305_04180_b200 import PhiloxGenerator
dev = torch.device("cuda", 0)
net = QNet.init(np.random.default_rng(0), (37, 256, 128, 5), device=dev)
for n in (4096, 16384, 65536):
    x = torch.randn(n, 37, device=dev)
    vem = VemSchedule(n_envs=n)
    rng = PhiloxGenerator(1, 3)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    for _ in range(3):
        select_actions_fused(net, x, vem, 0, rng, out=out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        select_actions_fused(net, x, vem, 0, rng, out=out)
    e.record(); e.synchronize()
    us = s.elapsed_time(e) / 20 * 1e3
    flops = 2 * n * (37 * 256 + 256 * 128 + 128 * 5)
    print(f"rows {n}: {us:.1f} us per launch, {flops / us / 1e6:.2f} TFLOP/s fp32")
