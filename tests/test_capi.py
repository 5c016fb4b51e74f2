"""The drop-in boundary: libsparrow.so loads without a GPU and exports every
entry point include/sparrow.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

from paper_2305_04180_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "sparrow.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|const char\*)\s+(sp_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("sp_env_create", "sp_env_reset_all", "sp_env_step", "sp_cast_rays",
                 "sp_disc_collides", "sp_rb_create", "sp_rb_append", "sp_rb_sample"):
        assert must in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_symbols()) == bound


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the C structs have the C compiler's sizes and offsets."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        import pytest
        pytest.skip("gcc not available")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sparrow.h"', "int main(){"]
    expect = []
    for cls in (_lib.SpConfig, _lib.SpMapDesc, _lib.SpRanges, _lib.SpMlp):
        name = cls.__name__
        lines.append(f'printf("%zu\\n", sizeof({name}));')
        expect.append(ctypes.sizeof(cls))
        for fname, _ in cls._fields_:
            lines.append(f'printf("%zu\\n", offsetof({name}, {fname}));')
            expect.append(getattr(cls, fname).offset)
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert got == expect


def test_error_codes_and_version_without_gpu():
    lib = _lib.load()
    assert lib.sp_version() == 1
    # invalid arguments are rejected before touching CUDA
    h = ctypes.c_void_p()
    assert lib.sp_env_create(None, None, 0, 0, None, None, 0, 0, 0, ctypes.byref(h)) == _lib.SP_EINVAL
    assert "null" in _lib.last_error()
    assert lib.sp_rb_create(0, 4, 0, ctypes.byref(h)) == _lib.SP_EINVAL
    assert "capacity" in _lib.last_error()


def test_env_create_validates_before_touching_the_device():
    """sp_env_create rejects bad configs / maps with status codes and messages
    before any CUDA call (so this runs without a GPU): vecenv.py:66-67,
    core.py:56-66 errors."""
    import numpy as np
    lib = _lib.load()
    offs = np.linspace(-1.0, 1.0, 4)

    def cfg(**kw):
        c = _lib.SpConfig()
        c.n_beams, c.max_range_cm, c.robot_radius_cm, c.timeout_steps = 4, 300.0, 9.0, 1000
        c.proximity_cm, c.n_actions, c.spawn_attempts, c.auto_reset = 30.0, 5, 256, 1
        c.beam_offsets = offs.ctypes.data_as(_lib.c_dp)
        for k, v in kw.items():
            setattr(c, k, v)
        return c

    occ = np.ones((20, 20), np.uint8)

    def desc(rows=20, cols=20, cell=1.0):
        d = _lib.SpMapDesc()
        d.n_rows, d.n_cols, d.cell_cm = rows, cols, cell
        d.occupancy = occ.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
        return d

    rg = (_lib.SpRanges * 1)()
    rg[0].delay[0], rg[0].delay[1] = 0, 0
    h = ctypes.c_void_p()

    def create(c, maps, n_envs=4, ranges=rg, n_ranges=1, midx=None):
        arr = (_lib.SpMapDesc * len(maps))(*maps)
        mp = None if midx is None else np.ascontiguousarray(midx, np.int32).ctypes.data_as(_lib.c_i32p)
        return lib.sp_env_create(ctypes.byref(c), arr, len(maps), n_envs, mp, ranges, n_ranges,
                                 0, 0, ctypes.byref(h))

    cases = [
        (lambda: create(cfg(n_beams=0), [desc()]), _lib.SP_EINVAL, b"n_beams"),
        (lambda: create(cfg(max_range_cm=0.0), [desc()]), _lib.SP_EINVAL, b"max range"),
        (lambda: create(cfg(n_actions=16), [desc()]), _lib.SP_EINVAL, b"action table"),
        (lambda: create(cfg(), [desc()], n_envs=0), _lib.SP_EINVAL, b"at least one copy"),
        (lambda: create(cfg(), [desc(), desc(rows=30)]), _lib.SP_EMAP, b"grid shape"),
        (lambda: create(cfg(), [desc(cell=0.0)]), _lib.SP_EINVAL, b"cell size"),
        (lambda: create(cfg(), [desc()], midx=[0, 1, 0, 0]), _lib.SP_EINVAL, b"map_index"),
        (lambda: create(cfg(), [desc()], n_ranges=2), _lib.SP_EINVAL, b"DiversityRanges"),
    ]
    for call, want, msg in cases:
        rc = call()
        assert rc == want, (rc, want, msg)
        assert msg in lib.sp_last_error(), lib.sp_last_error()
    bad = (_lib.SpRanges * 1)()
    bad[0].delay[0], bad[0].delay[1] = 0, 65
    assert create(cfg(), [desc()], ranges=bad) == _lib.SP_EINVAL
    assert b"delay" in lib.sp_last_error()
    # GridMap's border invariant (gridmap.py:90-95), which the marcher relies on
    holed = np.ones((20, 20), np.uint8)
    holed[0, 7] = 0
    d = desc()
    d.occupancy = holed.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    assert create(cfg(), [d]) == _lib.SP_EMAP
    assert b"border" in lib.sp_last_error()


def test_torch_extension_registers_the_hot_ops():
    """The PyTorch C++ extension (csrc/sp_torch.cpp) loads, binds the very
    libsparrow.so the package loaded (dlsym) and registers torch.ops.sparrow
    env_step / rb_append with the reference's argument shapes; with a CPU
    tensor it raises (there is no CPU path) instead of computing."""
    import torch
    from paper_2305_04180_b200 import _lib
    ops = _lib.torch_ops()
    assert ops is not None, "build the extension: python -m paper_2305_04180_b200.build"
    assert "torch C++ extension" in _lib.binding()
    for name in ("env_step", "rb_append", "bind"):
        assert hasattr(ops, name)
    with pytest.raises(RuntimeError, match="CUDA"):
        ops.env_step(0, torch.zeros(4, dtype=torch.int64), torch.zeros((4, 37)),
                     torch.zeros((4, 37)), torch.zeros(4, dtype=torch.float64),
                     torch.zeros(4, dtype=torch.bool), torch.zeros(4, dtype=torch.bool),
                     torch.zeros(4, dtype=torch.int8))
