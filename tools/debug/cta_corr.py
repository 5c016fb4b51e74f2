"""Per-CTA cycles of consecutive cfg3 steps (debug): how stationary is the
CTA imbalance?  SPARROW_REBALANCE=0 python tools/debug/cta_corr.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np, torch
import bench
from paper_2305_04180_b200 import VecEnv, _lib
from paper_2305_04180_b200.sim import DiversityRanges, SimParams
dev = torch.device("cuda", 0)
n = bench.N_PER_GPU
env = VecEnv(bench.load_maps(), n, DiversityRanges.around(SimParams(), bench.DIVERSITY), bench.env_config(),
             device=dev, check_actions=False)
lib = _lib.load()
env.reset_all(bench.SEED)
out = env.new_batch()
acts = torch.empty(n, dtype=torch.int64, device=dev)
stream = torch.cuda.current_stream(dev)
G = 148
cyc = np.zeros((40, G), np.uint32)
cuts = np.zeros((40, G + 1), np.int64)
for t in range(40):
    _lib.check(lib.sp_random_actions(n, bench.SEED, 0, t, 5, acts.data_ptr(), stream.cuda_stream))
    env.step_device(acts.data_ptr(), out)
    _lib.check(lib.sp_env_launch_info(env._h, cuts[t].ctypes.data_as(_lib.c_i64p),
                                      cyc[t].ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
c = cyc[10:].astype(np.float64)
print("max/mean per step:", np.round(c.max(1) / c.mean(1), 3)[:10])
print("corr(step t, t+1) of per-CTA cycles: %.3f" % np.corrcoef(c[:-1].ravel() - c[:-1].mean(1).repeat(G), c[1:].ravel() - c[1:].mean(1).repeat(G))[0, 1])
m = c.mean(0)
print("stationary part: std of per-CTA mean %.0f vs per-step std %.0f" % (m.std(), c.std(1).mean()))
print("argmax CTA per step:", c.argmax(1)[:20])
print("cut changes (first vs last):", np.abs(cuts[-1] - cuts[0]).max())
# map 4's CTAs (cuts and cycles over time)
pm = np.zeros(G, np.int64)
for b in range(G):
    pm[b] = np.searchsorted(np.arange(17) * (n // 16), cuts[0][b], side="right") - 1
k = np.flatnonzero(pm == 4)
for t in (0, 8, 16, 24, 32, 39):
    print("t=%2d cuts" % t, (cuts[t][k[0]:k[-1] + 2] - cuts[t][k[0]]).tolist(), "cyc/1000", (cyc[t][k] // 1000).tolist())
