"""Fused learner updates only (for ncu launch timing of sample + ddqn kernels)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np
import torch
from paper_2305_04180_b200 import PhiloxGenerator, ReplayBuffer
from paper_2305_04180_b200.asl import DdqnLearner, QNet
dev = torch.device("cuda:0")
buf = ReplayBuffer(1_000_000, 37)
g = torch.Generator(device=dev).manual_seed(0)
n = 1_000_000
for c in range(0, n, 200_000):
    m = 200_000
    buf.append_batch(torch.randn((m, 37), device=dev, generator=g), torch.randint(0, 5, (m,), device=dev, generator=g),
                     torch.randn(m, device=dev, generator=g), torch.randn((m, 37), device=dev, generator=g),
                     torch.rand(m, device=dev, generator=g) < 0.05)
algo = DdqnLearner(QNet.init(np.random.default_rng(0), (37, 256, 128, 5)), fused=True)
rng = PhiloxGenerator(1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    algo.update(buf.sample(256, rng, out=algo.graph_batch(256, 37)))
torch.cuda.synchronize()
print("ok")
