"""Multi-GPU: env-index sharding + the one collective (episode statistics).

Env copies are independent (``test_vecenv.py:42-67`` pins lane i of a vector
run to a width-1 run of lane i), so N GPUs each own a contiguous slice of the
global env ids: rank g steps ids [g*n, (g+1)*n).  Every per-lane quantity is
keyed by the GLOBAL id (Philox stream, default map ``id % M``), so a lane's
trajectory does not depend on the GPU count.  There is no collective on the
step path; the only exchange is a sum of the episode counters
(``vecenv.py:120-132`` pooling) at the metrics cadence -- one all-reduce of
three float64 values over NCCL (NVLink/NVSwitch) or gloo (CPU tests) -- plus,
for the report, one all-gather of each rank's last 256 episode returns keyed
by (step, global env id), which merge into exactly the deque a single process
stepping all ids would hold (``vecenv.py:79, 109``).
"""

from __future__ import annotations


def shard(n_total: int, rank: int, world: int) -> tuple:
    """(env_id_offset, n_local) of `rank` when n_total ids split contiguously."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(n_total), world)
    offset = rank * base + min(rank, extra)
    return offset, base + (1 if rank < extra else 0)


def all_reduce_totals(totals, group=None):
    """Sum a per-rank [episodes, arrivals, return_sum] float64 tensor in place."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(totals, op=dist.ReduceOp.SUM, group=group)
    return totals


def merge_recent_returns(shards, keep: int = 256) -> list:
    """Merge per-shard (keys, returns) -- keys (step << 32) | global env id --
    into the reference's deque(maxlen=256) order: by step, then env id."""
    import numpy as np
    keys = np.concatenate([np.asarray(k, dtype=np.uint64) for k, _ in shards] or [np.empty(0, np.uint64)])
    vals = np.concatenate([np.asarray(v, dtype=np.float64) for _, v in shards] or [np.empty(0)])
    order = np.argsort(keys, kind="stable")
    return vals[order][-keep:].tolist() if keep else []


def gather_recent_returns(keys, vals, group=None, device=None) -> list:
    """All-gather every rank's keyed recent returns (<= 256 each, padded)
    and merge them (merge_recent_returns)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return merge_recent_returns([(keys, vals)])
    n = len(keys)
    kt = torch.zeros(256, dtype=torch.int64, device=device)
    kt[:n] = torch.from_numpy(np.asarray(keys, np.uint64).view(np.int64))
    vt = torch.zeros(256, dtype=torch.float64, device=device)
    vt[:n] = torch.from_numpy(np.asarray(vals, np.float64))
    nt = torch.tensor([n], dtype=torch.int64, device=device)
    world = dist.get_world_size(group)
    ks = [torch.empty_like(kt) for _ in range(world)]
    vs = [torch.empty_like(vt) for _ in range(world)]
    ns = [torch.empty_like(nt) for _ in range(world)]
    dist.all_gather(ns, nt, group=group)
    dist.all_gather(ks, kt, group=group)
    dist.all_gather(vs, vt, group=group)
    shards = []
    for k, v, c in zip(ks, vs, ns):
        c = int(c.item())
        shards.append((k[:c].cpu().numpy().view(np.uint64), v[:c].cpu().numpy()))
    return merge_recent_returns(shards)


def pooled_stats(env, group=None) -> dict:
    """Whole-job episode statistics of a sharded VecEnv: one all-reduce of the
    counters and one all-gather of the keyed recent returns."""
    import torch.distributed as dist
    t = env.stats_totals()
    gloo = dist.is_available() and dist.is_initialized() and dist.get_backend(group) == "gloo"
    if gloo:
        t = t.cpu()
    all_reduce_totals(t, group)
    episodes, arrivals, return_sum = (float(v) for v in t.tolist())
    keys, vals = env.recent_returns_keyed()
    recent = gather_recent_returns(keys, vals, group, device=None if gloo else t.device)
    return {"episodes": int(round(episodes)), "arrivals": int(round(arrivals)),
            "return_sum": return_sum,
            "arrival_rate": arrivals / episodes if episodes else None,
            "mean_return": return_sum / episodes if episodes else None,
            "recent_returns": recent}
