"""Timeline of sp_env_step_host's row parts at cfg3 (debug; needs a library
built with -DSP_HOST_TIMING, selected by SPARROW_LIB_PATH): prints, per call,
event times in us from the call's start (stderr) and the call's wall time."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np, torch
import bench
from paper_2305_04180_b200 import VecEnv
from paper_2305_04180_b200.sim import DiversityRanges, SimParams
dev = torch.device("cuda", 0)
n = bench.N_PER_GPU
env = VecEnv(bench.load_maps(), n, DiversityRanges.around(SimParams(), bench.DIVERSITY), bench.env_config(),
             device=dev, check_actions=False)
env.reset_all(bench.SEED)
hb = env.host_buffers()
rng = np.random.default_rng(0)
for t in range(12):
    hb.actions.copy_(torch.from_numpy(rng.integers(0, 5, n)))
    t0 = time.perf_counter()
    env.step_host(hb.actions, hb)
    print("call %d wall %.1f us" % (t, (time.perf_counter() - t0) * 1e6), file=sys.stderr, flush=True)
