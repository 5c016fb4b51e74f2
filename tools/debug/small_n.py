"""Step time at small N: back-to-back vs after an L2 flush (debug)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import numpy as np, torch
from helpers import config, load_maps, ranges
from paper_2305_04180_b200 import VecEnv, _lib
from paper_2305_04180_b200.vecenv import StepBatch
for n in (1024, 4096, 16384):
    env = VecEnv(load_maps(16), n, ranges(0.3), config(32), check_actions=False)
    env.reset_all(0)
    dev = env.device; D = env.state_dim
    out = StepBatch(torch.empty((n, D), device=dev), torch.empty(n, dtype=torch.float64, device=dev),
                    torch.empty(n, dtype=torch.bool, device=dev), torch.empty(n, dtype=torch.bool, device=dev),
                    torch.empty((n, D), device=dev), torch.empty(n, dtype=torch.int8, device=dev))
    acts = torch.randint(0, 5, (n,), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    for mode in ("b2b", "flush", "smallflush"):
        ts = []
        for k in range(30):
            if mode == "flush": flush.fill_(k & 255)
            if mode == "smallflush": flush[: 8 << 20].fill_(k & 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); env.step_device(acts.data_ptr(), out); b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = [x.elapsed_time(y) for x, y in ts[5:]]
        print(n, mode, "median %.4f ms" % np.median(ms), "min %.4f" % min(ms))
