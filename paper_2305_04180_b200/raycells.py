"""Pure-DDA ray-cell accounting: the algorithmic unit of BASELINE.json's
"LiDAR ray-cells/sec" metric.

One ray-cell is one grid cell the reference's pure DDA (``_cy.pyx:89-105``
without the EDT jump) enters, from the origin cell through the cell the ray
stops in, or up to the last cell entered at t <= max_range.  A 4-connected
DDA walk changes one cell coordinate by one per step and moves monotonically
on both axes, so a ray that starts in cell (ix0, iy0) and stops in
(ix1, iy1) enters exactly |ix1 - ix0| + |iy1 - iy0| + 1 cells.  The stopping
cell is the hit cell the marcher reports (kernel recording / ``VecEnv.scan``),
or, for a ray that reaches max_range, the cell holding the point at
t = max_range.  The count is therefore exact per ray (up to rays passing
exactly through a cell corner at max_range) and costs one elementwise pass
on the device instead of a second march; ``tests/test_host.py`` pins it to
the oracle's cell-by-cell DDA count.
"""

from __future__ import annotations


def dda_cells(x, y, heading, beam_offsets, hit_cells, n_cols: int, cell: float,
              max_range: float):
    """Cells entered per ray.  x, y, heading: (N,) float64 origins (cm, rad);
    beam_offsets: (R,); hit_cells: (N, R) int (iy * W + ix of the occupied
    stopping cell, or -1 when the ray reached max_range).  torch tensors (any
    device) or numpy arrays; returns (N, R) int64 of the same kind."""
    try:
        import torch
        is_t = isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_t = False
    if is_t:
        lib = torch
        off = torch.as_tensor(beam_offsets, dtype=torch.float64, device=x.device)
        hit = hit_cells.to(torch.int64)
        floor = torch.floor
    else:
        import numpy as lib  # noqa: N813
        off = lib.asarray(beam_offsets, dtype=lib.float64)
        hit = lib.asarray(hit_cells).astype(lib.int64)
        floor = lib.floor
    ang = heading[:, None] + off[None, :]
    ix0 = floor(x / cell)[:, None]
    iy0 = floor(y / cell)[:, None]
    ex = floor((x[:, None] + max_range * lib.cos(ang)) / cell)
    ey = floor((y[:, None] + max_range * lib.sin(ang)) / cell)
    hx = lib.where(hit >= 0, hit % n_cols, ex)
    hy = lib.where(hit >= 0, hit // n_cols, ey)
    cells = abs(hx - ix0) + abs(hy - iy0) + 1
    return cells.to(torch.int64) if is_t else cells.astype(lib.int64)
