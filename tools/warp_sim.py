"""Issue-slot model of one CTA's LiDAR ray phase (host-side design tool).

Per-ray march-step counts come from the free-box march rule (march_sim.py,
per-cell table) on realistic poses: the C oracle env stepped with random
actions (so robots sit where the bench's robots sit).  The model then plays
the kernel's schedule: 24 warps on 4 schedulers, 2 ray slots per lane, a
shared ray queue, refill when >= refill_min of a warp's 64 slots are idle,
`group` march steps per slot between refill checks.  A warp iteration costs
its issue slots (march steps of both slots for every lane -- finished rays
step as fixed points -- plus SIMT-wide setup / finish code when any lane
needs it) and cannot finish faster than its dependent step chains.

    python tools/warp_sim.py [--envs 443] [--steps 30]

Used to rank dispatch orders / refill policies before spending GPU time; the
absolute cycle counts are a model, not a measurement.
"""

import argparse
import heapq
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))

C_STEP = 47      # warp instructions per march step per slot
C_LOOP = 20      # votes, branch per iteration
C_REFILL = 30    # atomics, shuffles of a refill
C_SETUP = 60     # ray_setup + noise prefetch (SIMT-wide if any lane sets up)
C_FIN = 45       # retirement (noise, division, stores, atomics)
LAT_STEP = 130   # cycles of one march step's dependent chain


def step_counts(n_envs, steps, seed=3, beams=32, max_range=300.0):
    from helpers import config, load_maps, ranges
    from march_sim import cell_box, march
    from oracle.oracle import OracleVecEnv
    from oracle.philox_shim import random_actions
    maps = load_maps(16)
    env = OracleVecEnv(maps, n_envs * 16, ranges(0.3), config(beams))
    env.reset_all(seed)
    for t in range(steps):
        env.step_batch(random_actions(seed, np.arange(n_envs * 16), t))
    p = env.pose()
    out = []
    off = np.linspace(-np.radians(135), np.radians(135), beams)
    for m in range(16):  # one CTA's worth of envs on each map
        sel = np.arange(m, n_envs * 16, 16)[:n_envs]
        occ = np.asarray(maps[m].occupancy, bool)
        ang = (p["heading"][sel][:, None] + off[None, :]).ravel()
        st = march(occ, np.repeat(p["x"][sel], beams), np.repeat(p["y"][sel], beams),
                   np.cos(ang), np.sin(ang), max_range, cell_box(occ))
        out.append(st.reshape(len(sel), beams))
    return out


def simulate(order, steps, refill_min=32, group=4, warps=24, scheds=4):
    """order: ray ids in dispatch order; steps[id]: march steps (incl. the
    finishing one).  Returns the cycle at which the last warp finishes."""
    q = list(order)
    head = 0
    sched_free = [0] * scheds
    # per warp: remaining steps of each of its 64 slots (0 = idle)
    rem = [np.zeros(64, np.int64) for _ in range(warps)]
    busy = [np.zeros(64, bool) for _ in range(warps)]
    ev = [(0, w) for w in range(warps)]
    heapq.heapify(ev)
    end = 0
    drained = False
    while ev:
        t, w = heapq.heappop(ev)
        s = w % scheds
        r, b = rem[w], busy[w]
        idle = (r <= 0)
        cost = C_LOOP
        n_idle = int(idle.sum())
        if n_idle >= refill_min or head >= len(q):
            fin_slots = idle & b
            if fin_slots[:32].any():
                cost += C_FIN
            if fin_slots[32:].any():
                cost += C_FIN
            b[fin_slots] = False
            if head >= len(q):
                if not b.any():
                    end = max(end, t)
                    continue
            else:
                cost += C_REFILL
                free = np.flatnonzero(idle)
                take = min(len(free), len(q) - head)
                for k in range(take):
                    r[free[k]] = steps[q[head + k]]
                    b[free[k]] = True
                head += take
                if take and (free[:take] < 32).any():
                    cost += C_SETUP
                if take and (free[:take] >= 32).any():
                    cost += C_SETUP
        cost += group * 2 * C_STEP
        r -= group
        start = max(t, sched_free[s])
        sched_free[s] = start + cost
        nxt = max(start + cost, t + group * LAT_STEP)
        heapq.heappush(ev, (nxt, w))
        end = max(end, nxt)
    del drained
    return end


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=443)
    ap.add_argument("--steps", type=int, default=30)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    per_map = step_counts(a.envs, a.steps)
    res = {}
    for st in per_map:
        n, R = st.shape
        flat = st.ravel() + 1  # + the finishing step
        env_max = st.max(axis=1)
        noisy = lambda v: v * rng.lognormal(0, 0.25, v.shape)  # noqa: E731 (prediction error)
        env_pred = noisy(env_max.astype(float))
        ray_pred = noisy(flat.astype(float))
        grp_pred = noisy(st.reshape(n, R // 8, 8).max(axis=2).astype(float))
        ids = np.arange(n * R).reshape(n, R)
        orders = {
            "env LPT (shipped)": ids[np.argsort(-env_pred, kind="stable")].ravel(),
            "no order": ids.ravel(),
            "ray LPT exact": np.argsort(-flat, kind="stable"),
            "ray LPT predicted": np.argsort(-ray_pred, kind="stable"),
            "8-beam group LPT": ids.reshape(n, R // 8, 8)[
                np.unravel_index(np.argsort(-grp_pred, axis=None, kind="stable"),
                                 grp_pred.shape)].ravel(),
        }
        for name, order in orders.items():
            for rm in (16, 32, 48):
                for g in (2, 4, 8):
                    res.setdefault((name, rm, g), []).append(simulate(order, flat, rm, g))
        ideal = (flat.sum() * C_STEP) / 4 / 2  # perfectly packed, 4 schedulers
        res.setdefault(("ideal issue", 0, 0), []).append(ideal)
    base = np.mean(res[("env LPT (shipped)", 32, 4)])
    for k, v in sorted(res.items(), key=lambda kv: np.mean(kv[1])):
        print(f"{k[0]:20s} refill_min {k[1]:2d} group {k[2]}: {np.mean(v):9.0f} cycles "
              f"({np.mean(v) / base:5.2f}x shipped)")


if __name__ == "__main__":
    main()
