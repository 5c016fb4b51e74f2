"""ASL session reproduction with knobs (debug): LEARN_START, DURATION."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import numpy as np, torch
from helpers import config, load_maps, ranges
from paper_2305_04180_b200 import ReplayBuffer, VecEnv
from paper_2305_04180_b200.asl import (DdqnConfig, DdqnLearner, QNet, Sharer, TfmConfig,
                                       VemSchedule, start_session)
SIZES = (37, 256, 128, 5)
n = 4096
env = VecEnv(load_maps(16), n, ranges(0.3), config(32), check_actions=False)
states = env.reset_all(0)
algo = DdqnLearner(QNet.init(np.random.default_rng(0), SIZES), DdqnConfig(), fused=True, graph=True)
sharer = Sharer(ReplayBuffer(1_000_000, 37))
tfm = TfmConfig(n, 256.0, 256)
session = start_session(sharer, env, states, algo.online, VemSchedule(n), tfm, max_steps=n * 400,
                        algo=algo, learn_start=int(os.environ.get("LEARN_START", "20000")),
                        upload_period=50, seed=0)
t0 = time.time()
while session.running and time.time() - t0 < float(os.environ.get("DURATION", "6")):
    time.sleep(0.1)
session.abort()
session.wait(timeout=30)
print("t_step", sharer.t_step, "b_step", sharer.b_step)
torch.cuda.synchronize()
print("ok")
