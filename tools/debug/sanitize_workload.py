"""Workload for tools/gpu_sanitize.sh: a few steps of the fused step kernel
at 4,096 and 65,536 envs (random actions), a reset-heavy config (timeout 3
steps: every CTA's extra scan slots overflow), recording on, and the replay
kernels (append with wrap, sample, gather)."""
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import config, load_maps, ranges  # noqa: E402
from oracle.philox_shim import random_actions  # noqa: E402
from paper_2305_04180_b200 import ReplayBuffer, VecEnv  # noqa: E402


def run_env(n, steps, timeout=None, record=False):
    kw = {} if timeout is None else {"timeout_steps": timeout}
    env = VecEnv(load_maps(16), n, ranges(0.3), config(32, **kw))
    if record:
        env.record()
    env.reset_all(3)
    for t in range(steps):
        env.step_batch(random_actions(3, np.arange(n), t))
    env.check()
    torch.cuda.synchronize()
    print(f"env n={n} steps={steps} timeout={timeout} ok", flush=True)


def run_replay():
    rb = ReplayBuffer(10_000, 37)
    rng = np.random.default_rng(0)
    for n in (4096, 3001, 5000, 17):
        s = rng.standard_normal((n, 37)).astype(np.float32)
        rb.append_batch(s, rng.integers(0, 5, n), rng.standard_normal(n), s + 1, rng.random(n) < .1)
    rb.sample(256, 7)
    rb.snapshot()
    torch.cuda.synchronize()
    print("replay ok", flush=True)


if __name__ == "__main__":
    run_env(4096, 3)
    run_env(65536, 2)
    run_env(4096, 7, timeout=3, record=True)
    run_replay()
