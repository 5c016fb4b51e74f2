"""Per-update weight drift of the fused / graphed learner vs eager torch (debug)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import numpy as np
import torch
from paper_2305_04180_b200.asl import DdqnConfig, DdqnLearner, QNet
from paper_2305_04180_b200 import TransitionBatch
SIZES = (37, 256, 128, 5)
def batch(rng, n):
    return (rng.standard_normal((n, 37)).astype(np.float32), rng.integers(0, 5, n),
            rng.standard_normal(n).astype(np.float32), rng.standard_normal((n, 37)).astype(np.float32),
            rng.random(n) < 0.1)
def tb(a):
    return TransitionBatch(*(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in a))
for mode in ({"graph": True}, {"fused": True}):
    e = DdqnLearner(QNet.init(np.random.default_rng(3), SIZES), DdqnConfig(target_sync_period=5))
    f = DdqnLearner(QNet.init(np.random.default_rng(3), SIZES), DdqnConfig(target_sync_period=5), **mode)
    rng = np.random.default_rng(11)
    for k in range(12):
        arrs = batch(rng, 256)
        se, sf = e.update(tb(arrs)), f.update(tb(arrs))
        dw = [float((a - b).abs().max()) for a, b in zip(e.online.weights, f.online.weights)]
        nflip = [int(((a - b).abs() > 1e-5).sum()) for a, b in zip(e.online.weights, f.online.weights)]
        print(mode, k, "loss", se.loss, sf.loss, "max|dW|", ["%.2e" % x for x in dw], "n>1e-5", nflip)
