"""Per-CTA step durations over many steps: systematic (per-CTA mean) vs random
(per-step) spread (debug; sp_env_launch_info)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import numpy as np, torch
from helpers import config, load_maps, ranges
from paper_2305_04180_b200 import VecEnv
from paper_2305_04180_b200.vecenv import StepBatch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
env = VecEnv(load_maps(16), n, ranges(0.3), config(32), check_actions=False)
env.reset_all(0)
dev, D = env.device, env.state_dim
out = StepBatch(torch.empty((n, D), device=dev), torch.empty(n, dtype=torch.float64, device=dev),
                torch.empty(n, dtype=torch.bool, device=dev), torch.empty(n, dtype=torch.bool, device=dev),
                torch.empty((n, D), device=dev), torch.empty(n, dtype=torch.int8, device=dev))
acts = torch.randint(0, 5, (n,), device=dev)
T = []
for k in range(int(os.environ.get("STEPS", "40"))):
    env.step_device(acts.data_ptr(), out)
    p = env.partition()
    if k >= 5:
        T.append(p["cta_cycles"].astype(np.float64) / 1965.0)
T = np.array(T)  # steps x CTAs, us
sz = np.diff(p["cuts"])
mean = T.mean(0)
print(f"envs/CTA {sz.min()}..{sz.max()}")
print(f"per-step max CTA: mean {T.max(1).mean():.1f} us; median CTA {np.median(T):.1f} us")
print(f"per-CTA mean over steps: min {mean.min():.1f} med {np.median(mean):.1f} max {mean.max():.1f} us")
print(f"per-CTA std over steps: median {np.median(T.std(0)):.2f} max {T.std(0).max():.2f} us")
print(f"corr(envs, mean time) {np.corrcoef(sz, mean)[0, 1]:.2f}")
dev_ = T - mean
print(f"random part: p50 {np.percentile(dev_, 50):.1f} p99 {np.percentile(dev_, 99):.1f} max {dev_.max():.1f} us")
worst = np.argsort(-mean)[:8]
print("slowest CTAs (id, envs, mean us, std):", [(int(i), int(sz[i]), round(mean[i], 1), round(T[:, i].std(), 1)) for i in worst])
