"""The product's N>1 path on the GPU: two processes (gloo), each stepping its
shard of the global env ids through the CUDA VecEnv, then the pooled
statistics (paper_2305_04180_b200.dist.pooled_stats: the one all-reduce of
episode counters and the all-gather of keyed recent returns).  Compared with
one process stepping every id on the same GPU: per-lane obs, rewards and
events bit-identical, counters exact, the merged recent-returns deque the
single run's deque (vecenv.py:79, 109, 120-132).

Both ranks share the one GPU of this pool; their kernels never wait on each
other (the collective runs on host tensors over gloo), so this is the real
code path, not a stand-in for an NVLink exchange.
"""

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_TOTAL, STEPS, SEED = 3000, 25, 17


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg():
    from helpers import config
    return config(32, timeout_steps=7)  # many episodes end: the deque wraps


def _run(rank, world, port, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from helpers import load_maps, ranges
    from oracle.philox_shim import random_actions
    from paper_2305_04180_b200 import VecEnv
    from paper_2305_04180_b200.dist import pooled_stats, shard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    offset, n = shard(N_TOTAL, rank, world)
    env = VecEnv(load_maps(16), n, ranges(0.3), _cfg(), env_id_offset=offset, device="cuda:0")
    obs, rew, ev = [env.reset_all(SEED).cpu().numpy()], [], []
    for t in range(STEPS):
        b = env.step_batch(random_actions(SEED, np.arange(offset, offset + n), t))
        obs.append(b.store_states.cpu().numpy())
        rew.append(b.rewards.cpu().numpy())
        ev.append(b.events.cpu().numpy())
    pooled = pooled_stats(env)
    np.savez(os.path.join(out, f"rank{rank}.npz"), obs=np.stack(obs), rew=np.stack(rew),
             ev=np.stack(ev), offset=offset, recent=np.asarray(pooled["recent_returns"]),
             tot=np.array([pooled["episodes"], pooled["arrivals"], pooled["return_sum"]]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_cuda_shards_match_one_process(tmp_path):
    import torch.multiprocessing as mp
    from helpers import load_maps, ranges
    from oracle.philox_shim import random_actions
    from paper_2305_04180_b200 import VecEnv

    port = _free_port()
    mp.start_processes(_run, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    env = VecEnv(load_maps(16), N_TOTAL, ranges(0.3), _cfg())
    obs, rew, ev = [env.reset_all(SEED).cpu().numpy()], [], []
    for t in range(STEPS):
        b = env.step_batch(random_actions(SEED, np.arange(N_TOTAL), t))
        obs.append(b.store_states.cpu().numpy())
        rew.append(b.rewards.cpu().numpy())
        ev.append(b.events.cpu().numpy())
    obs, rew, ev = np.stack(obs), np.stack(rew), np.stack(ev)
    snap = env.snapshot_stats()
    for r in range(2):
        z = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        o = int(z["offset"])
        n = z["obs"].shape[1]
        assert np.array_equal(z["obs"], obs[:, o:o + n]), r
        assert np.array_equal(z["rew"], rew[:, o:o + n]), r
        assert np.array_equal(z["ev"], ev[:, o:o + n]), r
        tot = z["tot"]
        assert int(tot[0]) == snap.episodes and int(tot[1]) == snap.arrivals
        assert abs(tot[2] - snap.return_sum) <= 1e-9 * max(1.0, abs(snap.return_sum))
        assert len(snap.recent_returns) == 256
        assert np.array_equal(z["recent"], np.asarray(snap.recent_returns)), r
