"""CUDA kernel backend for the reference's per-op plugin seam.

The reference selects a kernel module per SimBatch (``sim/core.py:60``;
modules ``kernels/_cy.pyx`` / ``kernels/_py.py``, dispatcher
``kernels/__init__.py:20-86``) and calls exactly two functions on it.  This
module has the same surface -- ``BACKEND_NAME``, ``cast_rays`` and
``disc_collides`` with host numpy in/out -- and runs both on the GPU
(``sp_cast_rays`` / ``sp_disc_collides``), so ``sim._kernel = kernels``
drives the UNMODIFIED reference simulator with device ray casting.

``cast_rays`` runs the reference algorithm itself (DDA + EDT jump,
``_cy.pyx:19-106``) in IEEE fp64 without contraction: its output is
bit-identical to the Cython backend.  Occupancy/EDT stacks are uploaded once
per array object (the reference builds them once, ``core.py:68-71``, and
never mutates them); call ``invalidate()`` after mutating one in place.
"""

from __future__ import annotations

import numpy as np

from paper_2305_04180_b200 import _lib

BACKEND_NAME = "cuda"

_cache: dict = {}


def invalidate() -> None:
    _cache.clear()


def _upload(arr: np.ndarray, device):
    import torch
    key = id(arr)
    hit = _cache.get(key)
    if hit is not None and hit[0] is arr:
        return hit[1]
    t = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
    _cache[key] = (arr, t)
    return t


def _dev_f64(a, device):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)


def cast_rays(occ, edt, map_idx, px, py, dirx, diry, cell, max_range, backend=None):
    """First-hit distance per ray, capped at max_range; 0 for origins inside an
    obstacle or outside the grid (kernels/__init__.py:62-76)."""
    import torch
    dev = _lib.require_cuda()
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    edt = np.ascontiguousarray(edt, dtype=np.float64)
    if occ.ndim != 3 or edt.shape != occ.shape:
        raise ValueError("occ and edt must be (M, H, W) stacks of the same shape")
    n = int(np.asarray(px).shape[0])
    out = torch.empty(n, dtype=torch.float64, device=dev)
    if n:
        o = _upload(occ, dev)
        e = _upload(edt, dev)
        mi = torch.from_numpy(np.ascontiguousarray(map_idx, dtype=np.int64)).to(dev)
        bufs = [_dev_f64(v, dev) for v in (px, py, dirx, diry)]
        _lib.check(_lib.load().sp_cast_rays(
            o.data_ptr(), e.data_ptr(), occ.shape[0], occ.shape[1], occ.shape[2], mi.data_ptr(),
            *(b.data_ptr() for b in bufs), n, float(cell), float(max_range), out.data_ptr(),
            _lib.stream_ptr(dev)), "cast_rays")
    return out.cpu().numpy()


def disc_collides(occ, map_idx, px, py, radius, cell, backend=None):
    """Whether each disc overlaps an occupied cell or leaves the grid
    (kernels/__init__.py:79-86)."""
    import torch
    dev = _lib.require_cuda()
    occ = np.ascontiguousarray(occ, dtype=np.uint8)
    if occ.ndim != 3:
        raise ValueError("occ must be an (M, H, W) stack")
    n = int(np.asarray(px).shape[0])
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    if n:
        o = _upload(occ, dev)
        mi = torch.from_numpy(np.ascontiguousarray(map_idx, dtype=np.int64)).to(dev)
        bufs = [_dev_f64(v, dev) for v in (px, py, radius)]
        _lib.check(_lib.load().sp_disc_collides(
            o.data_ptr(), occ.shape[0], occ.shape[1], occ.shape[2], mi.data_ptr(),
            *(b.data_ptr() for b in bufs), n, float(cell), out.data_ptr(),
            _lib.stream_ptr(dev)), "disc_collides")
    return out.cpu().numpy()
