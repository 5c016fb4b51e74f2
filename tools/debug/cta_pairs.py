"""Per-CTA cycles of 40 cfg3 steps with the current launch plan (debug):
what would sharing rays inside CTA pairs of the same map buy?  Saves
gpurun_out/cta_cycles.npz and prints max-over-CTAs vs max-over-pair-means."""
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
T = 40
cyc = np.zeros((T, G), np.uint32)
cuts = np.zeros((T, G + 1), np.int64)
for t in range(T):
    _lib.check(lib.sp_random_actions(n, bench.SEED, 0, t, 5, acts.data_ptr(), stream.cuda_stream))
    env.step_device(acts.data_ptr(), out)
    _lib.check(lib.sp_env_launch_info(env._h, cuts[t].ctypes.data_as(_lib.c_i64p),
                                      cyc[t].ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/cta_cycles.npz", cyc=cyc, cuts=cuts)
c = cyc[10:].astype(np.float64)
print("max/mean per step:", np.round(c.max(1) / c.mean(1), 3)[:10])
print("mean max/mean %.3f" % (c.max(1) / c.mean(1)).mean())
