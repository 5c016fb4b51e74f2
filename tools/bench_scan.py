"""LiDAR marcher throughput on its own (cfg4): rays/s and pure-DDA ray-cells/s.

    python tools/bench_scan.py [--poses 65536] [--beams 32] [--max-range 300] [--reps 10]

Poses: uniform over each map's collision-free cells (disc of the robot radius),
spread evenly over the 16 mapgen maps.  Device time of the scan kernel via
CUDA events; L2 is flushed between repetitions.  The ray-cell count (cells the
reference's pure DDA enters) is measured on a subsample with the
C oracle (test infrastructure, counting only).
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--poses", type=int, default=65536)
    ap.add_argument("--beams", type=int, default=32)
    ap.add_argument("--max-range", type=float, default=300.0)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    from helpers import config, load_maps, ranges
    from paper_2305_04180_b200 import VecEnv
    from oracle import oracle as O

    maps = load_maps(16)
    cfg = config(args.beams, lidar_kw={"max_range_cm": args.max_range})
    env = VecEnv(maps, 16, ranges(0.0), cfg)
    rng = np.random.default_rng(0)
    per = args.poses // len(maps)
    qx, qy, qh, qm = [], [], [], []
    from scipy import ndimage
    for m, gm in enumerate(maps):
        clear = ndimage.distance_transform_edt(~gm.occupancy) > 10
        free = np.argwhere(clear)
        pick = free[rng.integers(0, len(free), per)]
        qy.append(pick[:, 0] + rng.random(per)); qx.append(pick[:, 1] + rng.random(per))
        qh.append(rng.uniform(-np.pi, np.pi, per)); qm.append(np.full(per, m))
    qx, qy, qh, qm = map(np.concatenate, (qx, qy, qh, qm))
    n = len(qx)
    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    qoff = np.zeros(len(maps) + 1, dtype=np.int64)
    qoff[1:] = np.cumsum(np.bincount(qm, minlength=len(maps)))
    xd, yd, hd = (torch.from_numpy(v).to(dev) for v in (qx, qy, qh))  # already grouped by map
    out = torch.empty((n, args.beams), dtype=torch.float64, device=dev)
    for _ in range(3):
        env.scan_raw(qoff, xd, yd, hd, out)
    torch.cuda.synchronize()
    times = []
    for k in range(args.reps):
        flush.fill_(k)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        env.scan_raw(qoff, xd, yd, hd, out)
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e) / 1e3)
    t = float(np.median(times))
    rays = n * args.beams
    # pure-DDA cells per ray on a subsample (counting only)
    sub = rng.choice(n, min(n, 2048), replace=False)
    ang = qh[sub, None] + cfg.lidar.beam_offsets()[None, :]
    occ = np.stack([m.occupancy for m in maps]).astype(np.uint8)
    cells = O.count_dda_cells(occ, np.repeat(qm[sub], args.beams), np.repeat(qx[sub], args.beams),
                              np.repeat(qy[sub], args.beams), np.cos(ang).ravel(),
                              np.sin(ang).ravel(), 1.0, args.max_range)
    out = {"poses": n, "beams": args.beams, "max_range": args.max_range,
           "refill_min": os.environ.get("SPARROW_REFILL_MIN", "32 (default)"),
           "ms": t * 1e3, "rays_per_s": rays / t, "mean_dda_cells_per_ray": float(cells.mean()),
           "ray_cells_per_s": rays * float(cells.mean()) / t, "launch": env.launch_info()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
