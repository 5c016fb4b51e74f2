"""Build libsparrow.so for sm_100a (run: ``python -m paper_2305_04180_b200.build``).

One nvcc invocation over csrc/sp_capi.cu (which includes the kernel TUs),
``-gencode arch=compute_100a,code=sm_100a -lineinfo``; output in-tree at
``paper_2305_04180_b200/_lib/libsparrow.so`` so it travels with the repo
snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libsparrow.so")
SOURCES = ["sp_capi.cu", "sp_env.cu", "sp_ops.cu", "sp_learn.cu", "sp_actor.cu", "sp_env.cuh",
           "sp_common.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, s) for s in SOURCES]
    deps.append(os.path.join(HERE, "..", "include", "sparrow.h"))
    return all(os.path.getmtime(p) <= t for p in deps if os.path.exists(p))


def source_hash() -> str:
    """sha256 over the CUDA/C sources the library is built from (csrc/ and
    include/sparrow.h): stamps measurements copied from a profiler capture
    (profiles/ncu_step_traffic.json) so a stale one is detected."""
    import hashlib
    h = hashlib.sha256()
    for name in SOURCES:
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(name.encode() + b"\0" + f.read())
    with open(os.path.join(HERE, "..", "include", "sparrow.h"), "rb") as f:
        h.update(f.read())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """Compile libsparrow.so; `defines` (e.g. ["SP_CTAS_PER_SM=1"]) build
    experimental variants to another `out` path."""
    if not force and out == OUT and not defines and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = out + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *(f"-D{x}" for x in defines), "-o", tmp,
           os.path.join(CSRC, "sp_capi.cu")]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr.strip():
        print(res.stderr, file=sys.stderr)
    os.replace(tmp, out)
    return out


TORCH_EXT = os.path.join(HERE, "_lib", "sparrow_torch.so")


def build_torch_ext(force: bool = False, verbose: bool = False) -> str:
    """The PyTorch C++ extension (csrc/sp_torch.cpp: torch.ops.sparrow.*) over
    the C-ABI, compiled in-tree next to libsparrow.so.  It resolves the C-ABI
    with dlsym from the library the package loaded, so it does not link it."""
    src = os.path.join(CSRC, "sp_torch.cpp")
    hdr = os.path.join(HERE, "..", "include", "sparrow.h")
    if (not force and os.path.exists(TORCH_EXT)
            and os.path.getmtime(TORCH_EXT) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return TORCH_EXT
    import glob
    from torch.utils.cpp_extension import load
    bdir = os.path.join(HERE, "_lib", "torch_build")
    os.makedirs(bdir, exist_ok=True)
    load(name="sparrow_torch", sources=[src], build_directory=bdir, with_cuda=True,
         is_python_module=False, extra_cflags=["-O2"], extra_ldflags=["-ldl"], verbose=verbose)
    built = glob.glob(os.path.join(bdir, "sparrow_torch*.so"))
    if not built:
        raise RuntimeError("torch extension build produced no library")
    shutil.copy2(built[0], TORCH_EXT + ".tmp")
    os.replace(TORCH_EXT + ".tmp", TORCH_EXT)
    return TORCH_EXT


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--force"]
    if args:  # python -m paper_2305_04180_b200.build OUT.so DEF=1 ...
        print(build(force=True, verbose=True, out=os.path.abspath(args[0]), defines=args[1:]))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
