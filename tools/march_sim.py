"""Step-count model of the LiDAR marcher (host-side design tool, not a test).

Replays the kernel's march rule (sp_env.cu ray_step) in numpy over many rays
from random collision-free poses on the golden maps and reports march steps
per ray, for the current 2x2-block chessboard table and for alternative
free-space tables:

  block    2x2 blocks: 0x80|mask if any cell occupied, else radius r of the
           free (2r+1)^2-block box around the block   (the shipped table)
  quad     per-quadrant forward boxes: for travel direction (sx, sy) the
           largest free square of blocks whose back corner is the ray's block
  cell     1x1-cell chessboard radius (box centred on the ray's cell)

    python tools/march_sim.py [--rays 200000]
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))


LEVELS16 = np.array([0, 1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 48, 64, 96])


def quantize(q, levels):
    """Largest level <= q (a smaller forward square is still free)."""
    return levels[np.searchsorted(levels, q, side="right") - 1]


def chessboard(blocked):
    """L-inf distance (in grid units) from every cell to the nearest blocked
    cell, with outside-the-grid counting as blocked."""
    H, W = blocked.shape
    INF = 1 << 20
    yy, xx = np.mgrid[0:H, 0:W]
    border = np.minimum(np.minimum(xx + 1, yy + 1), np.minimum(W - xx, H - yy))
    d = np.where(blocked, 0, border).astype(np.int64)
    d = np.minimum(d, INF)
    for y in range(H):
        for x in range(W):
            v = d[y, x]
            if x > 0: v = min(v, d[y, x - 1] + 1)
            if y > 0:
                v = min(v, d[y - 1, x] + 1)
                if x > 0: v = min(v, d[y - 1, x - 1] + 1)
                if x + 1 < W: v = min(v, d[y - 1, x + 1] + 1)
            d[y, x] = v
    for y in range(H - 1, -1, -1):
        for x in range(W - 1, -1, -1):
            v = d[y, x]
            if x + 1 < W: v = min(v, d[y, x + 1] + 1)
            if y + 1 < H:
                v = min(v, d[y + 1, x] + 1)
                if x + 1 < W: v = min(v, d[y + 1, x + 1] + 1)
                if x > 0: v = min(v, d[y + 1, x - 1] + 1)
            d[y, x] = v
    return d


def forward_square(blocked, sx, sy):
    """Side q of the largest all-free square of cells whose back corner (w.r.t.
    travel direction sx, sy) is the cell: q[y,x] = 1 + min(q[y+sy,x], q[y,x+sx],
    q[y+sy,x+sx]) for free cells, 0 for blocked; outside = blocked."""
    H, W = blocked.shape
    q = np.zeros((H + 2, W + 2), np.int64)
    ys = range(H - 1, -1, -1) if sy > 0 else range(H)
    xs = list(range(W - 1, -1, -1) if sx > 0 else range(W))
    for y in ys:
        for x in xs:
            if blocked[y, x]:
                continue
            q[y + 1, x + 1] = 1 + min(q[y + 1 + sy, x + 1], q[y + 1, x + 1 + sx],
                                      q[y + 1 + sy, x + 1 + sx])
    return q[1:-1, 1:-1]


def sample_rays(occ, n, rng, beams=32, clearance=9):
    H, W = occ.shape
    d = chessboard(occ)
    free = np.argwhere(d > clearance)
    pick = free[rng.integers(0, len(free), n // beams)]
    x0 = pick[:, 1] + rng.random(len(pick))
    y0 = pick[:, 0] + rng.random(len(pick))
    h = rng.uniform(-np.pi, np.pi, len(pick))
    off = np.linspace(-np.radians(135), np.radians(135), beams)
    ang = (h[:, None] + off[None, :]).ravel()
    return np.repeat(x0, beams), np.repeat(y0, beams), np.cos(ang), np.sin(ang)


def march(occ, x0, y0, dx, dy, max_range, box):
    """box(ix, iy, sx, sy) -> (cellwise mask, ex, ey): per-step forward edge
    cells on each axis. Returns steps per ray."""
    n = len(x0)
    ix = np.floor(x0).astype(np.int64)
    iy = np.floor(y0).astype(np.int64)
    sx = np.where(dx >= 0, 1, -1)
    sy = np.where(dy >= 0, 1, -1)
    fx = (sx + 1) // 2
    fy = (sy + 1) // 2
    with np.errstate(divide="ignore"):
        idx = np.where(dx == 0, np.inf, 1.0 / dx)
        idy = np.where(dy == 0, np.inf, 1.0 / dy)
    live = np.ones(n, bool)
    steps = np.zeros(n, np.int64)
    while live.any():
        k = np.flatnonzero(live)
        occupied = occ[iy[k], ix[k]]
        steps[k] += 1
        ex, ey = box(ix[k], iy[k], sx[k], sy[k])
        tx = (ex + fx[k] - x0[k]) * idx[k]
        ty = (ey + fy[k] - y0[k]) * idy[k]
        xs = tx <= ty
        t = np.where(xs, tx, ty)
        c = np.floor(np.where(xs, y0[k] + tx * dy[k], x0[k] + ty * dx[k])).astype(np.int64)
        cy = np.where(sy[k] > 0, np.minimum(np.maximum(c, iy[k]), ey), np.maximum(np.minimum(c, iy[k]), ey))
        cx = np.where(sx[k] > 0, np.minimum(np.maximum(c, ix[k]), ex), np.maximum(np.minimum(c, ix[k]), ex))
        nx = np.where(xs, ex + sx[k], cx)
        ny = np.where(xs, cy, ey + sy[k])
        fin = occupied | (t > max_range)
        live[k[fin]] = False
        go = k[~fin]
        ix[go] = nx[~fin]
        iy[go] = ny[~fin]
    return steps


def block_box(occ):
    H, W = occ.shape
    Hb, Wb = (H + 1) // 2, (W + 1) // 2
    pad = np.ones((2 * Hb, 2 * Wb), bool)
    pad[:H, :W] = occ
    blk_occ = pad.reshape(Hb, 2, Wb, 2).any(axis=(1, 3))
    r = np.clip(chessboard(blk_occ) - 1, 0, 127)

    def box(ix, iy, sx, sy):
        bo = blk_occ[iy >> 1, ix >> 1]
        rr = r[iy >> 1, ix >> 1]
        ex = np.where(bo, ix, (ix & ~1) + (sx + 1) // 2 + sx * 2 * rr)
        ey = np.where(bo, iy, (iy & ~1) + (sy + 1) // 2 + sy * 2 * rr)
        return ex, ey
    return box


def hybrid_box(occ, levels=LEVELS16):
    """centred block radius r (exact, 1 byte) + per-quadrant forward extent
    quantized down to `levels` (4 bits each): forward extent max(r, e_q)."""
    H, W = occ.shape
    Hb, Wb = (H + 1) // 2, (W + 1) // 2
    pad = np.ones((2 * Hb, 2 * Wb), bool)
    pad[:H, :W] = occ
    blk_occ = pad.reshape(Hb, 2, Wb, 2).any(axis=(1, 3))
    r = np.clip(chessboard(blk_occ) - 1, 0, 127)
    e = {(a, b): quantize(np.maximum(forward_square(blk_occ, a, b) - 1, 0), levels)
         for a in (-1, 1) for b in (-1, 1)}

    def box(ix, iy, sx, sy):
        ex = ix.copy()
        ey = iy.copy()
        for (a, b), ee in e.items():
            m = (sx == a) & (sy == b)
            if not m.any():
                continue
            bo = blk_occ[iy[m] >> 1, ix[m] >> 1]
            ext = np.maximum(r[iy[m] >> 1, ix[m] >> 1], ee[iy[m] >> 1, ix[m] >> 1])
            ex[m] = np.where(bo, ix[m], (ix[m] & ~1) + (a + 1) // 2 + a * 2 * ext)
            ey[m] = np.where(bo, iy[m], (iy[m] & ~1) + (b + 1) // 2 + b * 2 * ext)
        return ex, ey
    return box


def cell_box(occ, cap=255):
    r = np.clip(chessboard(occ) - 1, 0, cap)

    def box(ix, iy, sx, sy):
        rr = r[iy, ix]
        return ix + sx * rr, iy + sy * rr
    return box


def quad_box(occ, cap=127, levels=None):
    H, W = occ.shape
    Hb, Wb = (H + 1) // 2, (W + 1) // 2
    pad = np.ones((2 * Hb, 2 * Wb), bool)
    pad[:H, :W] = occ
    blk_occ = pad.reshape(Hb, 2, Wb, 2).any(axis=(1, 3))
    q = {(a, b): np.clip(forward_square(blk_occ, a, b), 0, cap) for a in (-1, 1) for b in (-1, 1)}
    if levels is not None:
        q = {k: quantize(v, levels) for k, v in q.items()}

    def box(ix, iy, sx, sy):
        ex = ix.copy()
        ey = iy.copy()
        for (a, b), qq in q.items():
            m = (sx == a) & (sy == b)
            if not m.any():
                continue
            s = qq[iy[m] >> 1, ix[m] >> 1]  # free forward square side in blocks (0: occupied)
            bo = s == 0
            # from the ray's block, s blocks forward (incl. its own) are free
            ex[m] = np.where(bo, ix[m], (ix[m] & ~1) + (a + 1) // 2 + a * 2 * (s - 1))
            ey[m] = np.where(bo, iy[m], (iy[m] & ~1) + (b + 1) // 2 + b * 2 * (s - 1))
        return ex, ey
    return box


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rays", type=int, default=64000)
    ap.add_argument("--maps", type=int, default=4)
    a = ap.parse_args()
    from helpers import load_maps
    rng = np.random.default_rng(0)
    tot = {}
    for m in load_maps(a.maps):
        occ = np.asarray(m.occupancy, bool)
        rays = sample_rays(occ, a.rays, rng)
        for name, mk in (("block", block_box), ("quad", quad_box), ("quad16", lambda o: quad_box(o, 16)),
                         ("quadlog", lambda o: quad_box(o, 127, LEVELS16)),
                         ("hybrid", hybrid_box),
                         ("cell", cell_box), ("cell14", lambda o: cell_box(o, 14)),
                         ("cell6", lambda o: cell_box(o, 6))):
            st = march(occ, *rays, 300.0, mk(occ))
            tot.setdefault(name, []).append(st)
    for name, v in tot.items():
        s = np.concatenate(v)
        print(f"{name:6s} mean steps/ray {s.mean():6.2f}  p50 {np.median(s):4.0f}  p90 "
              f"{np.percentile(s, 90):4.0f}  max {s.max()}")


if __name__ == "__main__":
    main()
