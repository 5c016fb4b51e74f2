"""The drop-in boundary: libsparrow.so loads without a GPU and exports every
entry point include/sparrow.h declares (no compute calls here)."""

import ctypes
import os
import re

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
