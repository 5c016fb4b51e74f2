import cProfile, pstats, io, os, sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo/tools')
import numpy as np, torch
import bench_eval as be
from helpers import config, load_maps
from paper_2305_04180_b200.asl import QNet
from paper_2305_04180_b200.evaluate import evaluate_params
maps = load_maps(16); names = [f"map{i}" for i in range(16)]
cfg = config(32, timeout_steps=1000)
p = QNet.init(np.random.default_rng(0), (37, 256, 128, 5))
evaluate_params(p, maps[:2], names[:2], 64, seed=0, config=cfg, fused=True)
torch.cuda.synchronize()
pr = cProfile.Profile(); t0 = time.perf_counter(); pr.enable()
evaluate_params(p, maps, names, 4096, seed=1, config=cfg, fused=True)
torch.cuda.synchronize(); pr.disable(); print("wall", time.perf_counter() - t0)
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25); print(s.getvalue()[:6000])
