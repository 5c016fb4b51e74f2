import os, sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from helpers import config, load_maps, ranges
from paper_2305_04180_b200 import VecEnv
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
mode = sys.argv[2] if len(sys.argv) > 2 else "random"
env = VecEnv(load_maps(16), n, ranges(0.3), config(32), check_actions=False)
s = env.reset_all(0)
torch.cuda.synchronize()
g = torch.Generator(device="cuda"); g.manual_seed(0)
side = os.environ.get("SIDE_STREAM") == "1"
ctx = torch.cuda.stream(torch.cuda.Stream()) if side else torch.cuda.stream(torch.cuda.current_stream())
ctx.__enter__()
for t in range(3000):
    if mode == "const":
        a = torch.full((n,), 2, dtype=torch.int64, device="cuda")
    else:
        a = torch.randint(0, 5, (n,), device="cuda", generator=g)
    b = env.step_batch(a)
    if t % 50 == 0:
        try:
            torch.cuda.synchronize()
        except Exception as e:
            print("fail at step", t, e); sys.exit(1)
print("ok", env.snapshot_stats().episodes)
