"""Benchmark: Sparrow env-steps/s on B200 (BASELINE.json metric, cfg3 workload).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[2]): 65,536 envs per GPU over the 16
``color mapgen`` maps (tests/golden/maps16.npz), +/-30 % diversity, 32 LiDAR
beams (max 300 cm), Philox random actions (bench.py:97-105 in the reference
draws random actions the same way on the host).  A "step" = one
``VecEnv.step_batch`` over all envs incl. fused auto-reset; weak scaling
(fixed envs per GPU), env ids sharded contiguously across ranks.

* value   -- device time: K steps with actions already in HBM; each step timed
             with CUDA events on the launching stream; L2 flushed between
             timed steps outside the events (256 MiB write, then a 256 MiB
             read so the flush's dirty lines drain outside too); max over ranks.
* e2e     -- same metric through the public API with HOST buffers: per step
             pinned actions H2D, step, D2H of every StepBatch field; timed
             with CUDA events around copies + step.
* roofline -- dominant kernel env_step_kernel: algorithmic HBM bytes per
             env-step x N / mean launch time vs the
             measured copy bandwidth in MEASURED_PEAKS.json.
* cpu_baseline -- the reference itself (oracle/_ref, Cython backend) on this
             host's cores, P processes x a bounded sample of the workload.

``--impl reference`` times only the reference CPU implementation (rank 0;
other ranks exit 0) and prints the same JSON line with impl=reference.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PER_GPU = 65_536
CFG2_ENVS = 4096  # BASELINE configs[1], reported beside the headline
N_BEAMS = 32
N_MAPS = 16
DIVERSITY = 0.3
SEED = 20230504
METRIC = "Sparrow env-steps/sec"
UNIT = "env-steps/s"
# algorithmic HBM bytes per env-step at R=32 (D=37)
BYTES_PER_ENV_STEP = 161 + 376


def env_config():
    from paper_2305_04180_b200.sim import EnvConfig, LidarConfig
    return EnvConfig(lidar=LidarConfig(n_beams=N_BEAMS))


def load_maps():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import load_maps as lm
    return lm(N_MAPS)


def ncu_metrics():
    """Per-launch metrics of env_step_kernel from the committed ncu capture
    (DRAM traffic, issue-slot utilization): profiles/ncu_step_traffic.json."""
    p = os.path.join(ROOT, "profiles", "ncu_step_traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, interval_ms: int = 10):
        self.index = index
        self.interval_ms = interval_ms
        self.proc = None
        self.lines = []
        self._first = threading.Event()

    def __enter__(self):
        """Start sampling and block until nvidia-smi produced its first sample,
        so the timed region that follows is covered."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            self._first.wait(timeout=10.0)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())
            self._first.set()

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------- reference --

def _ref_worker(args):
    """One host process: the UNMODIFIED reference VecEnv (Cython kernels)."""
    n_local, seconds, seed, mode = args
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    sys.path.insert(0, ROOT)
    if mode == "reference":
        import color_rl.sim.core as core
        import color_rl.vecenv as vmod
        core.STATE_DIM = vmod.STATE_DIM = 5 + N_BEAMS
        from color_rl.sim.gridmap import GridMap as RG
        from color_rl.sim.params import DiversityRanges, EnvConfig, LidarConfig, SimParams
        from color_rl.vecenv import VecEnv as RV
        maps = [RG.from_text(m.to_text()) for m in load_maps()]
        env = RV(maps, n_local, DiversityRanges.around(SimParams(), DIVERSITY),
                 EnvConfig(lidar=LidarConfig(n_beams=N_BEAMS)))
        env.reset_all(seed)
        rng = np.random.default_rng(seed)
        step = lambda: env.step_batch(rng.integers(0, 5, n_local))  # noqa: E731 (bench.py:100)
    else:
        from oracle.oracle import OracleVecEnv
        from paper_2305_04180_b200.sim import DiversityRanges, SimParams
        env = OracleVecEnv(load_maps(), n_local, DiversityRanges.around(SimParams(), DIVERSITY),
                           env_config())
        env.reset_all(seed)
        rng = np.random.default_rng(seed)
        step = lambda: env.step_batch(rng.integers(0, 5, n_local))  # noqa: E731
    for _ in range(2):
        step()
    steps = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        step()
        steps += 1
    wall = time.perf_counter() - t0
    return n_local * steps, wall


def cpu_reference(seconds=4.0, n_local=2048, procs=None):
    """env-steps/s of the reference on all host cores (P independent processes)."""
    import multiprocessing as mp
    mode = "reference" if os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "color_rl")) else "port"
    if mode == "port":
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    procs = procs or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        res = pool.map(_ref_worker, [(n_local, seconds, SEED + i, mode) for i in range(procs)])
    total = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {"value": total / wall, "unit": UNIT, "cores": procs, "kind": mode,
            "sample": f"{procs} processes x {n_local} envs (cfg3 maps/diversity/beams), "
                      f"~{seconds:.0f} s of stepping each after reset+2 warm-up steps"}


# ----------------------------------------------------------------------- ours --

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2305_04180_b200 import VecEnv, _lib
    from paper_2305_04180_b200.sim import DiversityRanges, SimParams
    from paper_2305_04180_b200.vecenv import StepBatch

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n = args.envs
    offset = rank * n
    env = VecEnv(load_maps(), n, DiversityRanges.around(SimParams(), DIVERSITY), env_config(),
                 device=dev, env_id_offset=offset, check_actions=False)
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev)
    env.reset_all(SEED)
    D = env.state_dim
    K, W = args.steps, args.warmup
    total_steps = W + K
    acts = torch.empty((total_steps, n), dtype=torch.int64, device=dev)
    for t in range(total_steps):
        _lib.check(lib.sp_random_actions(n, SEED, offset, t, 5, acts[t].data_ptr(),
                                         stream.cuda_stream))
    out = StepBatch(torch.empty((n, D), dtype=torch.float32, device=dev),
                    torch.empty(n, dtype=torch.float64, device=dev),
                    torch.empty(n, dtype=torch.bool, device=dev),
                    torch.empty(n, dtype=torch.bool, device=dev),
                    torch.empty((n, D), dtype=torch.float32, device=dev),
                    torch.empty(n, dtype=torch.int8, device=dev))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    clean = torch.zeros(64 << 20, dtype=torch.float32, device=dev)  # 256 MiB, read-only

    def flush_l2(k):
        """Evict L2 outside the timed events: write 256 MiB (> 126 MB L2), then
        read another 256 MiB so the write's dirty lines drain to DRAM here and
        not inside the next timed step (which then starts from a clean, cold L2)."""
        flush.fill_(k & 0xFF)
        clean.sum()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    # the clock sampler runs from the warm-up (GPU already loaded) to the end
    # of the timed region
    with ClockSampler(local_rank) as clocks:
        for t in range(W):
            env.step_device(acts[t].data_ptr(), out)
        env.check()
        torch.cuda.synchronize(dev)
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize(dev)
        wall0 = time.perf_counter()
        for k in range(K):
            flush_l2(k)  # evict L2 (outside the timed events)
            starts[k].record(stream)
            env.step_device(acts[W + k].data_ptr(), out)
            stops[k].record(stream)
        torch.cuda.synchronize(dev)
        if dist.is_initialized():
            dist.barrier()
    wall = time.perf_counter() - wall0
    env.check()
    per_step = [s.elapsed_time(e) for s, e in zip(starts, stops)]  # ms
    t_dev = sum(per_step) / 1e3
    t_max = torch.tensor([t_dev], dtype=torch.float64, device=dev)
    if dist.is_initialized():
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_dev_max = float(t_max.item())
    value = world * n * K / t_dev_max

    # cfg2 (BASELINE configs[1]: 4096 envs on one GPU) on the same protocol,
    # reported beside the headline (which is cfg3, the per-GPU scaling config)
    cfg2 = None
    if world == 1 and n > CFG2_ENVS:
        n2 = CFG2_ENVS
        env2 = VecEnv(load_maps(), n2, DiversityRanges.around(SimParams(), DIVERSITY), env_config(),
                      device=dev, check_actions=False)
        env2.reset_all(SEED)
        out2 = StepBatch(torch.empty((n2, D), dtype=torch.float32, device=dev),
                         torch.empty(n2, dtype=torch.float64, device=dev),
                         torch.empty(n2, dtype=torch.bool, device=dev),
                         torch.empty(n2, dtype=torch.bool, device=dev),
                         torch.empty((n2, D), dtype=torch.float32, device=dev),
                         torch.empty(n2, dtype=torch.int8, device=dev))
        for t in range(W):  # lanes 0..4095 of the same Philox actions (keyed by env id)
            env2.step_device(acts[t].data_ptr(), out2)
        s2 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        e2 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        for k in range(K):
            flush_l2(k)
            s2[k].record(stream)
            env2.step_device(acts[W + k].data_ptr(), out2)
            e2[k].record(stream)
        torch.cuda.synchronize(dev)
        env2.check()
        ms2 = [x.elapsed_time(y) for x, y in zip(s2, e2)]
        cfg2 = {"workload": "cfg2: Sparrow 4096 envs, 16 maps, diversity 0.3, 32 LiDAR beams @300 cm, "
                            "random actions, fused auto-reset (same protocol as the headline)",
                "value": n2 * K / (sum(ms2) / 1e3), "unit": UNIT, "ms_per_step": sum(ms2) / K,
                "per_step_ms": {"min": min(ms2), "median": statistics.median(ms2), "max": max(ms2)}}
        del env2

    # one pooled-statistics all-reduce (the only collective; metrics cadence)
    from paper_2305_04180_b200.dist import pooled_stats
    t0 = time.perf_counter()
    pooled = pooled_stats(env)
    pooled["recent_returns"] = len(pooled["recent_returns"])  # the count, not the list
    t_allreduce_ms = (time.perf_counter() - t0) * 1e3

    # ---- e2e through the public API with host buffers -----------------------
    Ke = max(3, min(K, args.e2e_steps))
    h_act = [torch.from_numpy(acts[W + k % K].cpu().numpy()).pin_memory() for k in range(Ke)]
    hb = env.host_buffers()
    env.step_host(h_act[0], hb)  # warm-up: the first call allocates the device staging block
    e_starts = [torch.cuda.Event(enable_timing=True) for _ in range(Ke)]
    e_stops = [torch.cuda.Event(enable_timing=True) for _ in range(Ke)]
    for k in range(Ke):
        flush_l2(k)
        hb.actions.copy_(h_act[k])  # the step's inputs, already in pinned host memory
        e_starts[k].record(stream)
        res = env.step_host(hb.actions, hb)  # H2D actions, step, D2H of every field, sync
        e_stops[k].record(stream)
        e_stops[k].synchronize()
        _ = float(res.rewards[0])  # the step's result read on the host
    e2e_ms = [s.elapsed_time(e) for s, e in zip(e_starts, e_stops)]
    e2e_t = sum(e2e_ms) / 1e3
    et = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
    if dist.is_initialized():
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = world * n * Ke / float(et.item())
    h2d = n * 8
    d2h = sum(t.numel() * t.element_size() for t in out)

    result = None
    if rank == 0:
        peak, peak_kind = measured_peaks()
        mean_launch = t_dev / K
        achieved = BYTES_PER_ENV_STEP * n / mean_launch / 1e9
        info = env.launch_info()
        nm = ncu_metrics() if n == N_PER_GPU else {}
        traffic, traffic_src = nm.get("traffic_bytes_per_launch"), nm.get("source")
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": t_dev_max / K * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: 16 mapgen maps (seed 0, 366 cm, density 0.08), Philox random "
                    "actions, random-init env state",
            "config": {"workload": "cfg3: Sparrow 65,536 envs/GPU, 16 maps, diversity 0.3, "
                                   "32 LiDAR beams @300 cm, random actions, fused auto-reset",
                       "envs_per_gpu": n, "global_envs": n * world, "n_beams": N_BEAMS,
                       "n_maps": N_MAPS, "diversity": DIVERSITY, "parallelism": f"env-shard x{world}",
                       "l2": "flushed between timed steps, outside the events: 256 MiB write, then a 256 MiB read so the write-back of the dirty flush lines also happens outside",
                       "launch": info},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": Ke,
                    "per_step_ms": {"min": min(e2e_ms), "median": statistics.median(e2e_ms),
                                    "max": max(e2e_ms)},
                    "path": "VecEnv.step_host: pinned host actions in, every StepBatch field out as numpy"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "bytes per launch (dram read+write)",
                         "traffic_source": traffic_src,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                         "algorithmic_bytes_per_env_step": BYTES_PER_ENV_STEP,
                         "kernel": "env_step_kernel", "mean_launch_ms": mean_launch * 1e3,
                         "note": "issue/latency-bound (fp64 LiDAR march); see DESIGN.md 4"},
            "compute_roofline": {"bound": "issue", "unit": "% of issue slots (4/clk/SM)",
                                 "achieved": nm.get("issue_active_pct"),
                                 "simt_threads_per_inst": nm.get("simt_threads_per_inst"),
                                 "source": nm.get("source")},
            "clocks": clocks.summary(),
            "gpu_launches": K,
            "per_step_ms": {"min": min(per_step), "median": statistics.median(per_step),
                            "max": max(per_step)},
            "wall_s_timed_region": wall,
            "pooled_stats": pooled, "stats_allreduce_ms": t_allreduce_ms,
            "configs": {"cfg2": cfg2},
        }
    return result


def _json_out():
    """Keep stdout for the one JSON line: anything else written to fd 1 (NCCL's
    version banner, library chatter) goes to stderr."""
    sys.stdout.flush()
    fd = os.dup(1)
    os.dup2(2, 1)

    def emit(obj):
        os.write(fd, (json.dumps(obj) + "\n").encode())
    return emit


def main():
    emit = _json_out()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=N_PER_GPU)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=4.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        base = cpu_reference(seconds=args.cpu_seconds)
        line = {"metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
                "data": "synthetic (same maps/diversity/beams as ours)",
                "config": {"workload": "cfg3 sample on host cores (reference color_rl VecEnv, "
                                       "Cython kernels)", "parallelism": "host processes"},
                "cpu_baseline": base,
                "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        emit(line)
        return

    # under torchrun (any world size) the NCCL plumbing is always exercised
    launched = "MASTER_ADDR" in os.environ and "RANK" in os.environ
    if launched:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    result = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            result["cpu_baseline"] = cpu_reference(seconds=args.cpu_seconds)
        emit(result)
    if launched:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
