"""Which W1 gradient elements flip between the eager and fused learner (debug)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np
import torch
from paper_2305_04180_b200.asl import DdqnConfig, DdqnLearner, QNet, backward, compute_targets
from paper_2305_04180_b200 import TransitionBatch
SIZES = (37, 256, 128, 5)
rng = np.random.default_rng(11)
arrs = (rng.standard_normal((256, 37)).astype(np.float32), rng.integers(0, 5, 256),
        rng.standard_normal(256).astype(np.float32), rng.standard_normal((256, 37)).astype(np.float32),
        rng.random(256) < 0.1)
tb = TransitionBatch(*(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in arrs))
e = DdqnLearner(QNet.init(np.random.default_rng(3), SIZES), DdqnConfig(target_sync_period=5))
f = DdqnLearner(QNet.init(np.random.default_rng(3), SIZES), DdqnConfig(target_sync_period=5), fused=True)
y = compute_targets(tb, e.online, e.target, 0.98)
gw, gb, loss, mad = backward(e.online, tb.states, tb.actions, y)
# float64 reference gradient
w64 = [w.double() for w in e.online.weights]; b64 = [b.double() for b in e.online.biases]
x = tb.states.double(); acts=[x]; pre=[]
h = x
for i,(w,b) in enumerate(zip(w64,b64)):
    z = h @ w + b; pre.append(z); h = z if i == 2 else torch.relu(z); acts.append(h)
q = acts[-1]; rows = torch.arange(256, device=q.device)
res = q[rows, tb.actions] - y.double()
dq = torch.zeros_like(q); dq[rows, tb.actions] = res.clamp(-1, 1) / 256
d = dq; g64 = [None]*3
for li in (2,1,0):
    g64[li] = acts[li].t() @ d
    if li > 0: d = (d @ w64[li].t()) * (pre[li-1] > 0)
e.update(tb); f.update(tb)
diff = (e.online.weights[0] - f.online.weights[0]).abs()
idx = torch.nonzero(diff > 1e-5)
print("n flipped", len(idx))
mf = f.adam.m_weights[0] / 0.1  # m = (1-b1) g at step 1
for k, j in idx.tolist()[:10]:
    print(k, j, "eager g %.3e" % gw[0][k, j].item(), "fused g %.3e" % mf[k, j].item(), "f64 g %.3e" % g64[0][k, j].item(),
          "col max %.3e" % gw[0][:, j].abs().max().item())
