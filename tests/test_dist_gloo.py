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


def _gather_run(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2305_04180_b200.dist import gather_recent_returns
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r's lanes are global ids r*1000 + i; uneven counts per rank
    n = 200 + 70 * rank
    steps = np.arange(n) // 7
    ids = rank * 1000 + np.arange(n) % 7
    keys = (steps.astype(np.uint64) << np.uint64(32)) | ids.astype(np.uint64)
    vals = rank * 1e3 + np.arange(n, dtype=np.float64)
    merged = gather_recent_returns(keys[-256:], vals[-256:])
    np.save(os.path.join(out, f"gather{rank}.npy"), np.array(merged))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_recent_returns_gather(tmp_path):
    """dist.gather_recent_returns (world size 2, gloo): every rank gets the
    merged (step, global env id)-ordered last 256 returns of all ranks."""
    import torch.multiprocessing as mp
    from paper_2305_04180_b200.dist import merge_recent_returns
    port = _free_port()
    mp.start_processes(_gather_run, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    shards = []
    for rank in range(2):
        n = 200 + 70 * rank
        steps = np.arange(n) // 7
        ids = rank * 1000 + np.arange(n) % 7
        keys = (steps.astype(np.uint64) << np.uint64(32)) | ids.astype(np.uint64)
        vals = rank * 1e3 + np.arange(n, dtype=np.float64)
        shards.append((keys[-256:], vals[-256:]))
    want = merge_recent_returns(shards)
    assert len(want) == 256
    for rank in range(2):
        assert np.load(tmp_path / f"gather{rank}.npy").tolist() == want
