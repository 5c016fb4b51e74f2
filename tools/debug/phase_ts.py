"""Per-CTA phase durations of env_step_kernel from the SP_TIMING variant (debug).
SPARROW_LIB_PATH=variants/lib_timing.so python tools/debug/phase_ts.py"""
import sys, os, ctypes
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import numpy as np, torch
from helpers import config, load_maps, ranges
from paper_2305_04180_b200 import VecEnv, _lib
from paper_2305_04180_b200.vecenv import StepBatch
lib = ctypes.CDLL(_lib.LIB_PATH)
names = ["prologue", "bind_map", "phaseA", "order+noise", "rays", "phaseC", "rows"]
for n in (int(os.environ.get("N", "65536")),):
    env = VecEnv(load_maps(16), n, ranges(0.3), config(32), check_actions=False)
    env.reset_all(0)
    dev = env.device; D = env.state_dim
    out = StepBatch(torch.empty((n, D), device=dev), torch.empty(n, dtype=torch.float64, device=dev),
                    torch.empty(n, dtype=torch.bool, device=dev), torch.empty(n, dtype=torch.bool, device=dev),
                    torch.empty((n, D), device=dev), torch.empty(n, dtype=torch.int8, device=dev))
    acts = torch.randint(0, 5, (n,), device=dev)
    if os.environ.get("ACTIONS") == "turn":  # no collisions: phase A without resets
        acts = torch.zeros(n, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    clean = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
    for k in range(int(os.environ.get("STEPS", "10"))):
        if os.environ.get("FLUSH", "1") == "1":  # bench.py's protocol: cold L2 per step
            flush.fill_(k & 0xFF)
            clean.sum()
        if os.environ.get("ACTIONS") == "fresh":  # new random actions every step (bench.py)
            acts = torch.randint(0, 5, (n,), device=dev)
        env.step_device(acts.data_ptr(), out)
    torch.cuda.synchronize()
    ts = np.zeros((148, 160), np.uint64)
    lib.sp_debug_read_ts(ts.ctypes.data_as(ctypes.c_void_p), 148)
    ts = ts.astype(np.int64)
    if os.environ.get("SAVE"):  # raw stamps for offline analysis
        np.save(os.environ["SAVE"], ts)

    g0, g1 = ts[:, 36].copy(), ts[:, 37].copy()
    print("   globaltimer: CTA starts span %.2f us, ends span %.2f us, kernel span %.2f us; "
          "CTA durations median %.1f max %.1f us"
          % ((g0.max() - g0.min()) / 1e3, (g1.max() - g1.min()) / 1e3, (g1.max() - g0.min()) / 1e3,
             np.median(g1 - g0) / 1e3, (g1 - g0).max() / 1e3))
    es = ts[:, 38:44].copy()
    rel = (es - ts[:, 2:3]) * (1000.0 / 1.965) / 1e6  # us from stamp 2 (phase A start)
    print("   env 0 in step_env (us after phase A start, median): action loaded %.2f, physics done %.2f, "
          "map ready %.2f, disc %.2f, reward %.2f, header %.2f"
          % tuple(np.median(rel, axis=0)))
    cyc = 1000.0 / 1.965 / 1e3  # cycles -> ns
    t0_ = ts[:, :1]
    def wq(a, b):  # per-warp stamps [a, b) in ns from the CTA start
        return (ts[:, a:b] - t0_) * cyc
    pa, oe, rs, re_ = wq(12, 36), wq(48, 72), wq(72, 96), wq(96, 120)
    print("   per-CTA (ns from CTA start, median over CTAs): last warp ends phase A %.0f; "
          "first / last warp leaves ordering %.0f / %.0f; first / last warp enters rays %.0f / %.0f; "
          "first / last warp leaves rays %.0f / %.0f"
          % (np.median(pa.max(1)), np.median(oe.min(1)), np.median(oe.max(1)), np.median(rs.min(1)),
             np.median(rs.max(1)), np.median(re_.min(1)), np.median(re_.max(1))))
    ln = np.zeros((5, 148, 768), np.uint64)
    lib.sp_debug_read_lane(ln.ctypes.data_as(ctypes.c_void_p), 148)
    ln = ln.astype(np.int64)
    if os.environ.get("LANES"):
        np.save(os.environ["LANES"], ln)
    rows = []  # per env warp: the last lane past each step_env point (ns from the CTA start;
    # a build with -DSP_TIMING_LANES, else all zero)
    for b in range(148):
        nb_ = int(ts[b, 8])
        for w in range((nb_ + 31) // 32):
            sl = slice(w * 32, min(nb_, (w + 1) * 32))
            rows.append([((ln[p, b, sl] - ts[b, 0]) * cyc).max() for p in range(4)])
    rows = np.array(rows)
    if ln.any():
        print("   env warps, last lane past loads / physics / disc / events (ns, median): %s; p90: %s"
              % (np.median(rows, 0).round().tolist(), np.percentile(rows, 90, 0).round().tolist()))
    wa = ts[:, 12:36].copy()  # per-warp phase-A arrivals (cycles), relative to the CTA start
    wa = (wa - ts[:, :1]) * (1000.0 / 1.965) / 1e6  # -> us
    ts = ts[:, :12]
    print("   per-warp end of phase A (us from CTA start), median over CTAs by warp:",
          " ".join("%.1f" % v for v in np.median(wa, axis=0)))
    print("   slowest warp per CTA: ids", np.bincount(wa.argmax(1), minlength=24).tolist())
    nenv, mapi = ts[:, 8].copy(), ts[:, 9].copy()
    ts = (ts - ts[:, :1]) * (1000.0 / 1.965)  # cycles -> ns at 1.965 GHz (per-SM clocks)
    ts[:, 0] = 0
    t0 = ts[:, 0].min()
    d = np.diff(ts, axis=1) / 1e3
    print(f"n={n}: longest CTA {ts[:, 7].max() / 1e3:.1f} us (clock64, ns)")
    d = np.diff(ts[:, :8], axis=1) / 1e3
    for i, nm in enumerate(names):
        print(f"   {nm:12s} median {np.median(d[:, i]):6.0f} ns  max {d[:, i].max():6.0f} ns")
    order = (ts[:, 11] - ts[:, 3]) / 1e3
    print("   of order+noise: ordering %.2f us median (max %.2f)" % (np.median(order), order.max()))
    if os.environ.get("SYNC2"):
        b1 = (ts[:, 10] - ts[:, 3]) / 1e3
        print("   sync2: first barrier after A %.2f us median (max %.2f)" % (np.median(b1), b1.max()))
    rays = d[:, 4]
    drain = (ts[:, 10] - ts[:, 4]) / 1e3  # queue drained, relative to the ray phase start
    print("   ray queue drained %.1f us into the ray phase (median); tail after it: median %.1f us, max %.1f us"
          % (np.median(drain), np.median(rays - drain), (rays - drain).max()))
    print("   CTA envs: min %d max %d; CTAs spanning 2 maps: n/a; rays max/mean %.1f/%.1f us" % (nenv.min(), nenv.max(), rays.max(), rays.mean()))
    tot = ts[:, 7] / 1e3
    print("   per-map (ns): map  ctas  envs/cta  rays mean/min/max   CTA total mean/min/max")
    for m in sorted(set(mapi.tolist())):
        k = mapi == m
        print(f"   {m:4d} {k.sum():5d} {nenv[k].mean():9.1f} {rays[k].mean():8.0f} {rays[k].min():8.0f} {rays[k].max():8.0f}"
              f"   {tot[k].mean():8.0f} {tot[k].min():8.0f} {tot[k].max():8.0f}")
