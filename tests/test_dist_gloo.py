"""Multi-process (world size 2, gloo, CPU) coverage of the N>1 path.

Each rank steps its shard of the global env ids and the only collective is
the all-reduce of episode counters (paper_2305_04180_b200.dist).  The env
arithmetic here is the C oracle (the CPU stand-in for the device step; the
GPU step is pinned to it by tests/test_gpu_parity.py), so the test checks the
sharding contract itself: lanes keyed by GLOBAL env id reproduce the
single-process run bit for bit, and the all-reduced totals equal the
single-process totals.
"""

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank, world, port, n_total, steps, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from helpers import config, load_maps, ranges
    from oracle.oracle import OracleVecEnv
    from oracle.philox_shim import random_actions
    from paper_2305_04180_b200.dist import all_reduce_totals, shard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    offset, n = shard(n_total, rank, world)
    env = OracleVecEnv(load_maps(16), n, ranges(0.3), config(32), env_id_offset=offset)
    seed = 31
    obs = [env.reset_all(seed)]
    for t in range(steps):
        b = env.step_batch(random_actions(seed, np.arange(offset, offset + n), t))
        obs.append(b.store_states)
    st = env.stats()
    totals = torch.tensor([st["episodes"].sum(), st["arrivals"].sum(), st["return_sum"].sum()],
                          dtype=torch.float64)
    all_reduce_totals(totals)
    np.savez(os.path.join(out, f"rank{rank}.npz"), obs=np.stack(obs), totals=totals.numpy(),
             offset=offset)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process(tmp_path):
    import torch.multiprocessing as mp
    from helpers import config, load_maps, ranges
    from oracle.oracle import OracleVecEnv
    from oracle.philox_shim import random_actions

    n_total, steps, world = 96, 40, 2
    mp.spawn(_run, args=(world, _free_port(), n_total, steps, str(tmp_path)), nprocs=world,
             join=True)
    full = OracleVecEnv(load_maps(16), n_total, ranges(0.3), config(32))
    seed = 31
    obs = [full.reset_all(seed)]
    for t in range(steps):
        obs.append(full.step_batch(random_actions(seed, np.arange(n_total), t)).store_states)
    obs = np.stack(obs)
    st = full.stats()
    want = np.array([st["episodes"].sum(), st["arrivals"].sum(), st["return_sum"].sum()])
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        off = int(z["offset"])
        n = z["obs"].shape[1]
        assert np.array_equal(z["obs"], obs[:, off:off + n]), f"rank {r} lanes differ"
        np.testing.assert_allclose(z["totals"], want, rtol=1e-12)
    assert want[0] > 0
