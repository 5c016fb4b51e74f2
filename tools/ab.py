"""A/B of libsparrow.so variants on one box, interleaved (host-side tool).

    python tools/ab.py TAG lib1.so lib2.so[@GSHIFT=5,REFILL_MIN=24] ... [--reps 3] [--steps 60]

Each measurement runs in its own process (SPARROW_LIB_PATH=lib): the cfg3
step (65,536 envs, 16 maps, R = 32; L2 flushed between device-timed steps,
bench.py's protocol) and the cfg4 R = 32 scan of the marcher alone.  Prints
and appends to gpurun_out/ab_TAG.txt: mean / median step ms and scan ms.
"""

import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(steps):
    import numpy as np
    import torch
    import bench
    from paper_2305_04180_b200 import VecEnv, _lib
    from paper_2305_04180_b200.sim import DiversityRanges, SimParams
    from paper_2305_04180_b200.vecenv import StepBatch
    dev = torch.device("cuda", 0)
    n = bench.N_PER_GPU
    env = VecEnv(bench.load_maps(), n, DiversityRanges.around(SimParams(), bench.DIVERSITY),
                 bench.env_config(), device=dev, check_actions=False)
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev)
    env.reset_all(bench.SEED)
    D = env.state_dim
    W = 5
    acts = torch.empty((W + steps, n), dtype=torch.int64, device=dev)
    for t in range(W + steps):
        _lib.check(lib.sp_random_actions(n, bench.SEED, 0, t, 5, acts[t].data_ptr(),
                                         stream.cuda_stream))
    out = StepBatch(torch.empty((n, D), device=dev), torch.empty(n, dtype=torch.float64, device=dev),
                    torch.empty(n, dtype=torch.bool, device=dev),
                    torch.empty(n, dtype=torch.bool, device=dev), torch.empty((n, D), device=dev),
                    torch.empty(n, dtype=torch.int8, device=dev))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    clean = torch.zeros(64 << 20, dtype=torch.float32, device=dev)

    def flush_l2(k):
        flush.fill_(k & 0xFF)
        clean.sum()
    for t in range(W):
        env.step_device(acts[t].data_ptr(), out)
    graph = None
    if os.environ.get("AB_GRAPH") == "1":  # the step as a CUDA-graph replay (actions buffer fixed)
        act_buf = acts[W].clone()
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            env.step_device(act_buf.data_ptr(), out)
        stream.wait_stream(side)
    ms = []
    for k in range(steps):
        flush_l2(k)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if graph is not None:
            act_buf.copy_(acts[W + k])
        s.record(stream)
        if graph is not None:
            graph.replay()
        else:
            env.step_device(acts[W + k].data_ptr(), out)
        e.record(stream)
        e.synchronize()
        ms.append(s.elapsed_time(e))
    env.check()
    sw = bench.lidar_sweep.__globals__  # reuse the sweep's pose generator
    maps = bench.load_maps()
    qx, qy, qh, qm = sw["_poses"](maps, 65536)
    from paper_2305_04180_b200.sim import EnvConfig, LidarConfig
    senv = VecEnv(maps, 16, DiversityRanges(), EnvConfig(lidar=LidarConfig(n_beams=32)), device=dev)
    qoff = np.zeros(17, dtype=np.int64)
    qoff[1:] = np.cumsum(np.bincount(qm, minlength=16))
    xd, yd, hd = (torch.from_numpy(v).to(dev) for v in (qx, qy, qh))
    r = torch.empty((len(qx), 32), dtype=torch.float64, device=dev)
    for _ in range(2):
        senv.scan_raw(qoff, xd, yd, hd, r)
    sms = []
    for k in range(9):
        flush_l2(k)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        senv.scan_raw(qoff, xd, yd, hd, r)
        e.record(stream)
        e.synchronize()
        sms.append(s.elapsed_time(e))
    print(json.dumps({"mean": sum(ms) / len(ms), "median": statistics.median(ms),
                      "scan32": statistics.median(sms)}))


def main():
    if sys.argv[1] == "--one":
        one(int(sys.argv[2]))
        return
    tag, rest = sys.argv[1], sys.argv[2:]
    reps, steps = 3, 60
    libs = []
    it = iter(rest)
    for a in it:
        if a == "--reps":
            reps = int(next(it))
        elif a == "--steps":
            steps = int(next(it))
        else:
            libs.append(a)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    res = {lib: [] for lib in libs}
    for rep in range(reps):
        for lib in libs:
            path, _, extra = lib.partition("@")  # lib.so@GSHIFT=5,REFILL_MIN=24
            env = dict(os.environ, SPARROW_LIB_PATH=os.path.abspath(path))
            for kv in filter(None, extra.split(",")):
                k, _, v = kv.partition("=")
                env["SPARROW_" + k] = v
            p = subprocess.run([sys.executable, os.path.abspath(__file__), "--one", str(steps)],
                               env=env, capture_output=True, text=True, cwd=ROOT, timeout=600)
            line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-400:]
            try:
                d = json.loads(line)
            except ValueError:
                d = {"error": line}
            res[lib].append(d)
            msg = f"{rep} {os.path.basename(lib)} {json.dumps(d)}"
            print(msg, flush=True)
            with open(os.path.join(ROOT, "gpurun_out", f"ab_{tag}.txt"), "a") as f:
                f.write(msg + "\n")
    for lib, v in res.items():
        ok = [d for d in v if "mean" in d]
        if ok:
            print(f"{os.path.basename(lib)}: step mean {statistics.median([d['mean'] for d in ok]):.4f}"
                  f" median {statistics.median([d['median'] for d in ok]):.4f}"
                  f" scan32 {statistics.median([d['scan32'] for d in ok]):.4f}")


if __name__ == "__main__":
    main()
