"""Benchmark: Sparrow env-steps/s on B200 (BASELINE.json metric, cfg3 workload),
plus the metric's second clause (LiDAR ray-cells/s vs roofline, cfg4) and the
replay path (cfg5 ring).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[2]): 65,536 envs per GPU over the 16
``color mapgen`` maps (tests/golden/maps16.npz), +/-30 % diversity, 32 LiDAR
beams (max 300 cm), Philox random actions (bench.py:97-105 in the reference
draws random actions the same way on the host).  A "step" = one
``VecEnv.step_batch`` over all envs incl. fused auto-reset; weak scaling
(fixed envs per GPU), env ids sharded contiguously across ranks.

* value    -- device time: K steps with actions already in HBM; each step
              timed with CUDA events on the launching stream; L2 flushed
              between timed steps outside the events (256 MiB write, then a
              256 MiB read so the flush's dirty lines drain outside too); max
              over ranks.
* e2e      -- same metric through the public API with HOST buffers: per step
              pinned actions H2D, step, D2H of every StepBatch field; timed
              with CUDA events around copies + step.  The process and its
              pinned buffers are bound to the GPU's NUMA node first.
* roofline -- the binding resource of env_step_kernel: shared
              memory, one 32-bit word per pure-DDA ray-cell.  Ray-cells per
              launch are counted in this run (a recorded step after the timed
              region: per-ray hit cells -> raycells.dda_cells), peak =
              SMs x 128 B/clk x the SM clock sampled during the timed region.
              roofline_hbm keeps the algorithmic-bytes view.
* lidar    -- cfg4: the marcher alone (env_scan_kernel) at R in {32,128,256} x
              max range in {150,300,500} cm: rays/s, ray-cells/s, frac.
* replay   -- cfg5 ring (1M x D=37): append GB/s and frac of HBM (4,096-row
              appends, and 65,536-row appends = one cfg3 step of
              transitions), sample latency at B=256.
* cpu_baseline -- the reference itself (oracle/_ref, Cython backend) on this
              host's cores, P processes x N/P envs of the same workload.

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
MAX_MHZ = 1965.0  # B200 max SM clock (fallback when nvidia-smi is unavailable)


def env_config():
    from paper_2305_04180_b200.sim import EnvConfig, LidarConfig
    return EnvConfig(lidar=LidarConfig(n_beams=N_BEAMS))


def load_maps():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import load_maps as lm
    return lm(N_MAPS)


def ncu_metrics():
    """Per-launch metrics of env_step_kernel from the committed ncu capture
    (DRAM traffic, issue-slot utilization): profiles/ncu_step_traffic.json,
    used only when its source hash is this build's (else reported stale)."""
    from paper_2305_04180_b200.build import source_hash
    p = os.path.join(ROOT, "profiles", "ncu_step_traffic.json")
    if not os.path.exists(p):
        return {"stale": "no capture"}
    with open(p) as f:
        d = json.load(f)
    cur = source_hash()
    if d.get("source_hash") != cur:
        return {"stale": f"capture of sources {d.get('source_hash')} != this build {cur}"}
    return d


def smem_issued(nm: dict, n_sm: int, mhz: float) -> dict:
    """Shared-memory wavefronts per launch (all phases, bank conflicts included)
    over the capture's kernel duration, against one wavefront per clock per SM
    at this run's sampled SM clock."""
    wf, dur = nm.get("smem_wavefronts"), nm.get("duration_us")
    if not (wf and dur and mhz):
        return {"source": nm.get("stale") or "no capture"}
    rate = wf / (dur * 1e-6)
    peak = n_sm * mhz * 1e6
    return {"wavefronts_per_launch": wf, "bank_conflicts_per_launch": nm.get("smem_bank_conflicts"),
            "wavefronts_per_s": rate, "peak_wavefronts_per_s": peak, "frac": rate / peak,
            "source": nm.get("source")}


def numa_bind(local_rank: int) -> dict:
    """Bind this process to the CPUs of the GPU's NUMA node (pinned host
    buffers allocated afterwards are first-touched there), so the e2e copies
    do not cross the socket interconnect.  Returns what was done."""
    import torch
    try:
        p = torch.cuda.get_device_properties(local_rank)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            node = int(f.read().strip())
        if node < 0:
            return {"node": None, "pci": bus, "note": "no NUMA affinity reported"}
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        prev = os.sched_getaffinity(0)
        os.sched_setaffinity(0, cpus)
        return {"node": node, "pci": bus, "cpus": spec, "_prev": prev}
    except (OSError, ValueError, AttributeError) as e:
        return {"node": None, "note": f"not bound: {e}"}


def smem_peak_gbs(n_sm: int, mhz: float) -> float:
    """Shared-memory bandwidth: 32 banks x 4 B per clock per SM."""
    return n_sm * 128.0 * mhz * 1e6 / 1e9


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


def cpu_reference(seconds=4.0, n_total=N_PER_GPU, procs=None):
    """env-steps/s of the reference on all host cores: P independent processes,
    each stepping N/P envs of the workload."""
    import multiprocessing as mp
    mode = "reference" if os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "color_rl")) else "port"
    if mode == "port":
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    procs = procs or len(os.sched_getaffinity(0)) or 1
    n_local = max(1, n_total // procs)
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        res = pool.map(_ref_worker, [(n_local, seconds, SEED + i, mode) for i in range(procs)])
    total = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {"value": total / wall, "unit": UNIT, "cores": procs, "kind": mode,
            "sample": f"{procs} processes x {n_local} envs (cfg3 maps/diversity/beams), "
                      f"~{seconds:.0f} s of stepping each after reset+2 warm-up steps"}


# ----------------------------------------------------------------------- ours --

def _poses(maps, n, seed=0, clearance=10.0):
    """n LiDAR origins spread evenly over the maps, uniform over each map's
    cells with > `clearance` cells of free space (cfg4 scan workload)."""
    from scipy import ndimage
    rng = np.random.default_rng(seed)
    per = n // len(maps)
    qx, qy, qh, qm = [], [], [], []
    for m, gm in enumerate(maps):
        free = np.argwhere(ndimage.distance_transform_edt(~gm.occupancy) > clearance)
        pick = free[rng.integers(0, len(free), per)]
        qy.append(pick[:, 0] + rng.random(per))
        qx.append(pick[:, 1] + rng.random(per))
        qh.append(rng.uniform(-np.pi, np.pi, per))
        qm.append(np.full(per, m))
    return tuple(map(np.concatenate, (qx, qy, qh, qm)))


def lidar_sweep(dev, flush_l2, n_sm, mhz, reps=7, n_poses=65_536):
    """cfg4: the marcher alone (env_scan_kernel, VecEnv.scan_raw) on n_poses
    origins over the 16 maps, R x max range; device time (median of reps,
    L2 flushed before each), ray-cells counted from the returned hit cells."""
    import torch
    from paper_2305_04180_b200 import VecEnv
    from paper_2305_04180_b200.raycells import dda_cells
    from paper_2305_04180_b200.sim import DiversityRanges, EnvConfig, LidarConfig
    maps = load_maps()
    qx, qy, qh, qm = _poses(maps, n_poses)
    n = len(qx)
    qoff = np.zeros(len(maps) + 1, dtype=np.int64)
    qoff[1:] = np.cumsum(np.bincount(qm, minlength=len(maps)))
    xd, yd, hd = (torch.from_numpy(v).to(dev) for v in (qx, qy, qh))  # grouped by map
    stream = torch.cuda.current_stream(dev)
    rows = []
    for R in (32, 128, 256):
        for mr in (150.0, 300.0, 500.0):
            cfg = EnvConfig(lidar=LidarConfig(n_beams=R, max_range_cm=mr))
            env = VecEnv(maps, 16, DiversityRanges(), cfg, device=dev)
            out = torch.empty((n, R), dtype=torch.float64, device=dev)
            cells = torch.empty((n, R), dtype=torch.int32, device=dev)
            for _ in range(2):
                env.scan_raw(qoff, xd, yd, hd, out, cells)
            ms = []
            for k in range(reps):
                flush_l2(k)
                s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s_.record(stream)
                env.scan_raw(qoff, xd, yd, hd, out, cells)
                e_.record(stream)
                e_.synchronize()
                ms.append(s_.elapsed_time(e_))
            t = statistics.median(ms) / 1e3
            mean_cells = float(dda_cells(xd, yd, hd, cfg.lidar.beam_offsets(), cells,
                                         maps[0].occupancy.shape[1], 1.0, mr).double().mean())
            rc = n * R * mean_cells / t
            peak = smem_peak_gbs(n_sm, mhz) / 4 * 1e9  # words (= ray-cells) per second
            rows.append({"beams": R, "max_range_cm": mr, "ms": t * 1e3, "rays_per_s": n * R / t,
                         "mean_dda_cells_per_ray": mean_cells, "ray_cells_per_s": rc,
                         "frac": rc / peak})
            del env
    return {"workload": f"cfg4: {n} origins over the 16 maps (uniform over cells with >10 "
                        "cells clearance), noise-free scans, env_scan_kernel",
            "peak_ray_cells_per_s": smem_peak_gbs(n_sm, mhz) / 4 * 1e9,
            "peak_basis": f"{n_sm} SMs x 32 words/clk x {mhz:.0f} MHz (one SMEM word per "
                          "pure-DDA cell, SURVEY 8(d))",
            "sweep": rows}


def replay_bench(dev, flush_l2, peak_gbs, reps=7):
    """cfg5 ring (1M rows, D = 37): device time of sp_rb_append for 4,096 and
    65,536-row batches (the ring wraps during the run) and of sp_rb_sample
    at B = 256.  Append moves 2 x 309 B per row (read the batch, write the
    ring), the same read+write accounting as the measured copy peak."""
    import torch
    from paper_2305_04180_b200 import _lib
    from paper_2305_04180_b200.replay import ReplayBuffer
    C, D = 1_000_000, 5 + N_BEAMS
    rb = ReplayBuffer(C, D, device=dev)
    lib = rb._lib
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    row_bytes = 4 * D * 2 + 8 + 4 + 1
    res = {"workload": f"cfg5: ring of {C} transitions, D = {D} ({row_bytes} B/row: s, s2 "
                       "f32, a i64, r f32, done u8)", "row_bytes": row_bytes, "append": []}
    for n in (4096, 65_536):
        g = torch.Generator(device=dev)
        g.manual_seed(n)
        s = torch.rand((n, D), device=dev, generator=g)
        s2 = torch.rand((n, D), device=dev, generator=g)
        a = torch.randint(0, 5, (n,), device=dev, generator=g)
        r = torch.rand(n, device=dev, generator=g)
        d = torch.rand(n, device=dev, generator=g) < 0.01

        def append():
            _lib.check(lib.sp_rb_append(rb._h, s.data_ptr(), a.data_ptr(), r.data_ptr(), 0,
                                        s2.data_ptr(), d.data_ptr(), n, sp), "append")
        for _ in range(3):
            append()
        ms = []
        for k in range(max(reps, (C // n) // 4)):
            flush_l2(k)
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record(stream)
            append()
            e_.record(stream)
            e_.synchronize()
            ms.append(s_.elapsed_time(e_))
        t = statistics.median(ms) / 1e3
        gbs = 2 * row_bytes * n / t / 1e9
        row = {"rows_per_call": n, "us": t * 1e6, "rows_per_s": n / t,
               "achieved_gbs": gbs, "peak_gbs": peak_gbs, "frac": gbs / peak_gbs,
               "timing": "one call between CUDA events (includes the launch latency)"}
        if n >= 65_536:  # streaming: a full ring pass of back-to-back calls
            calls = C // n
            flush_l2(99)
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record(stream)
            for _ in range(calls):
                append()
            e_.record(stream)
            e_.synchronize()
            ts = s_.elapsed_time(e_) / 1e3
            sg = 2 * row_bytes * n * calls / ts / 1e9
            row["stream"] = {"calls": calls, "rows": n * calls, "us_per_call": ts / calls * 1e6,
                             "achieved_gbs": sg, "frac": sg / peak_gbs,
                             "timing": "calls back to back between one pair of events "
                                       "(a whole 1M-row ring pass; > L2)"}
        res["append"].append(row)
    B = 256
    out = [torch.empty((B, D), device=dev), torch.empty(B, dtype=torch.int64, device=dev),
           torch.empty(B, device=dev), torch.empty((B, D), device=dev),
           torch.empty(B, dtype=torch.bool, device=dev)]
    idx = torch.empty(B, dtype=torch.int64, device=dev)
    ms = []
    for k in range(reps + 3):
        flush_l2(k)
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record(stream)
        _lib.check(lib.sp_rb_sample(rb._h, B, SEED, 3, k * B, *(t.data_ptr() for t in out),
                                    idx.data_ptr(), sp), "sample")
        e_.record(stream)
        e_.synchronize()
        ms.append(s_.elapsed_time(e_))
    ms = ms[3:]
    res["sample"] = {"batch": B, "us_median": statistics.median(ms) * 1e3,
                     "us_min": min(ms) * 1e3, "ring_rows": len(rb),
                     "note": "latency-bound (one launch); L2 flushed before each"}
    del rb
    return res


def d2h_probe(dev, nbytes, reps=5):
    """Effective pinned D2H bandwidth of this box (GB/s): the e2e step's
    transfer in isolation."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    stream = torch.cuda.current_stream(dev)
    ms = []
    for _ in range(reps):
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record(stream)
        dst.copy_(src, non_blocking=True)
        e_.record(stream)
        e_.synchronize()
        ms.append(s_.elapsed_time(e_))
    return nbytes / (statistics.median(ms) / 1e3) / 1e9


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2305_04180_b200 import VecEnv, _lib
    from paper_2305_04180_b200.raycells import dda_cells
    from paper_2305_04180_b200.sim import DiversityRanges, SimParams
    from paper_2305_04180_b200.vecenv import StepBatch

    numa = numa_bind(local_rank)
    prev_affinity = numa.pop("_prev", None)
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
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
    acts = torch.empty((total_steps + 1, n), dtype=torch.int64, device=dev)
    for t in range(total_steps + 1):
        _lib.check(lib.sp_random_actions(n, SEED, offset, t, 5, acts[t].data_ptr(),
                                         stream.cuda_stream))

    def batch(m):
        return StepBatch(torch.empty((m, D), dtype=torch.float32, device=dev),
                         torch.empty(m, dtype=torch.float64, device=dev),
                         torch.empty(m, dtype=torch.bool, device=dev),
                         torch.empty(m, dtype=torch.bool, device=dev),
                         torch.empty((m, D), dtype=torch.float32, device=dev),
                         torch.empty(m, dtype=torch.int8, device=dev))
    out = batch(n)
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
        for t in range(W - 1):
            env.step_device(acts[t].data_ptr(), out)
        env.check()
        torch.cuda.synchronize(dev)
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize(dev)
        # the last warm-up step runs the timed loop's pattern (L2 flush, step)
        # right before it, so the first timed step does not start from an
        # idle GPU after the host synchronisation (it took ~2x the others)
        flush_l2(W - 1)
        env.step_device(acts[W - 1].data_ptr(), out)
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
    if os.environ.get("BENCH_PER_STEP"):  # debug: every timed step's ms
        print(json.dumps([round(x, 4) for x in per_step]), file=sys.stderr)
    t_dev = sum(per_step) / 1e3
    t_max = torch.tensor([t_dev], dtype=torch.float64, device=dev)
    if dist.is_initialized():
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_dev_max = float(t_max.item())
    value = world * n * K / t_dev_max
    clk = clocks.summary()
    mhz = float(clk.get("sm_mhz") or MAX_MHZ)

    # ray-cells of a step, counted in this run: one more (untimed) step with
    # the kernel's recording on -> per-ray hit cells of the scans behind the
    # states rows -> pure-DDA cells per ray (raycells.dda_cells).  That is N
    # scans per step; the ~0.9 % extra fresh-spawn scans of resetting envs are
    # not credited, so the count is a lower bound.
    env.record()
    env.step_device(acts[total_steps].data_ptr(), out)
    rec = env.recorded()
    sim = env.sim
    xs, ys, hs = (torch.from_numpy(v).to(dev) for v in (sim.x, sim.y, sim.heading))
    cells_per_ray = float(dda_cells(xs, ys, hs, env._offsets, rec["hit_state"],
                                    env._maps[0].occupancy.shape[1],
                                    float(env._maps[0].cell_size_cm),
                                    float(env.config.lidar.max_range_cm)).double().mean())
    env.record(False)
    ray_cells_per_launch = n * N_BEAMS * cells_per_ray

    # cfg2 (BASELINE configs[1]: 4096 envs on one GPU) on the same protocol,
    # reported beside the headline (which is cfg3, the per-GPU scaling config)
    cfg2 = None
    if world == 1 and n > CFG2_ENVS:
        n2 = CFG2_ENVS
        env2 = VecEnv(load_maps(), n2, DiversityRanges.around(SimParams(), DIVERSITY), env_config(),
                      device=dev, check_actions=False)
        env2.reset_all(SEED)
        out2 = batch(n2)
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
    d2h_gbs = d2h_probe(dev, d2h)

    result = None
    if rank == 0:
        peak, peak_kind = measured_peaks()
        mean_launch = t_dev / K
        achieved = BYTES_PER_ENV_STEP * n / mean_launch / 1e9
        info = env.launch_info()
        nm = ncu_metrics() if n == N_PER_GPU else {"stale": "capture is of the 65,536-env step"}
        smem_ach = 4.0 * ray_cells_per_launch / mean_launch / 1e9
        smem_peak = smem_peak_gbs(n_sm, mhz)
        lidar = None if args.no_lidar else lidar_sweep(dev, flush_l2, n_sm, mhz)
        replay = None if args.no_replay else replay_bench(dev, flush_l2, peak)
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
                    "ms_per_step_mean": e2e_t / Ke * 1e3,
                    "per_step_ms": {"min": min(e2e_ms), "median": statistics.median(e2e_ms),
                                    "max": max(e2e_ms)},
                    "d2h_probe_gbs": d2h_gbs,
                    "pcie_share": (d2h / d2h_gbs / 1e9) / (e2e_t / Ke),
                    "numa": numa,
                    "path": "VecEnv.step_host: pinned host actions in (range-checked on the host "
                            "before any launch, as the reference's step_all), every StepBatch "
                            "field out as numpy"},
            "roofline": {"bound": "smem", "achieved": smem_ach, "peak": smem_peak, "unit": "GB/s",
                         "frac": smem_ach / smem_peak,
                         "traffic": nm.get("traffic_bytes_per_launch"),
                         "traffic_unit": "DRAM bytes per launch (read+write), ncu --set full",
                         "traffic_source": nm.get("source") or nm.get("stale"),
                         "ray_cells_per_s": ray_cells_per_launch / mean_launch,
                         "ray_cells_per_launch": ray_cells_per_launch,
                         "dda_cells_per_ray": cells_per_ray,
                         "peak_ray_cells_per_s": smem_peak / 4 * 1e9,
                         "peak_basis": f"{n_sm} SMs x 128 B/clk x {mhz:.0f} MHz (median SM clock "
                                       "sampled in the timed region); one 4 B SMEM word per "
                                       "pure-DDA ray-cell (SURVEY 8(d))",
                         "achieved_basis": "ray-cells per launch (N scans x R rays x pure-DDA "
                                           "cells per ray, counted from a recorded step in this "
                                           "run; reset scans not credited) x 4 B / mean launch",
                         "kernel": "env_step_kernel", "mean_launch_ms": mean_launch * 1e3,
                         # SURVEY 8(d)'s alternative: the SMEM wavefronts the kernel
                         # actually issues (the free-box march looks up far fewer
                         # cells than a pure DDA enters), from the ncu capture
                         "smem_issued": smem_issued(nm, n_sm, mhz)},
            "roofline_hbm": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak,
                             "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                             "algorithmic_bytes_per_env_step": BYTES_PER_ENV_STEP},
            "compute_roofline": {"bound": "issue", "unit": "% of issue slots (4/clk/SM)",
                                 "achieved": nm.get("issue_active_pct"),
                                 "simt_threads_per_inst": nm.get("simt_threads_per_inst"),
                                 "source": nm.get("source") or nm.get("stale")},
            "clocks": clk,
            "gpu_launches": K,
            "per_step_ms": {"min": min(per_step), "median": statistics.median(per_step),
                            "max": max(per_step), "mean": t_dev / K * 1e3},
            "wall_s_timed_region": wall,
            "pooled_stats": pooled, "stats_allreduce_ms": t_allreduce_ms,
            "configs": {"cfg2": cfg2},
            "lidar": lidar,
            "replay": replay,
        }
    if prev_affinity:
        os.sched_setaffinity(0, prev_affinity)  # the CPU baseline uses every host core
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
    ap.add_argument("--no-lidar", action="store_true", help="skip the cfg4 marcher sweep")
    ap.add_argument("--no-replay", action="store_true", help="skip the cfg5 replay section")
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
                "steps": args.steps, "warmup": args.warmup,
                # one cfg3 step (65,536 envs) at the measured rate
                "ms_per_step": N_PER_GPU / base["value"] * 1e3,
                "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
                "data": "synthetic (same maps/diversity/beams as ours)",
                "config": {"workload": "cfg3: Sparrow 65,536 envs/GPU, 16 maps, diversity 0.3, "
                                       "32 LiDAR beams @300 cm, random actions, fused auto-reset "
                                       "(sampled on the host cores: reference color_rl VecEnv, "
                                       "Cython kernels)",
                           "envs_per_gpu": N_PER_GPU, "n_beams": N_BEAMS, "n_maps": N_MAPS,
                           "diversity": DIVERSITY, "parallelism": "host processes"},
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
