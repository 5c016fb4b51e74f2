"""Multi-GPU: env-index sharding + the one collective (episode statistics).

Env copies are independent (``test_vecenv.py:42-67`` pins lane i of a vector
run to a width-1 run of lane i), so N GPUs each own a contiguous slice of the
global env ids: rank g steps ids [g*n, (g+1)*n).  Every per-lane quantity is
keyed by the GLOBAL id (Philox stream, default map ``id % M``), so a lane's
trajectory does not depend on the GPU count.  There is no collective on the
step path; the only exchange is a sum of the episode counters
(``vecenv.py:120-132`` pooling) at the metrics cadence -- one all-reduce of
three float64 values over NCCL (NVLink/NVSwitch) or gloo (CPU tests).
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


def pooled_stats(env, group=None) -> dict:
    """Whole-job episode statistics of a sharded VecEnv (one all-reduce)."""
    import torch.distributed as dist
    t = env.stats_totals()
    if dist.is_available() and dist.is_initialized() and dist.get_backend(group) == "gloo":
        t = t.cpu()
    all_reduce_totals(t, group)
    episodes, arrivals, return_sum = (float(v) for v in t.tolist())
    return {"episodes": int(round(episodes)), "arrivals": int(round(arrivals)),
            "return_sum": return_sum,
            "arrival_rate": arrivals / episodes if episodes else None,
            "mean_return": return_sum / episodes if episodes else None}
