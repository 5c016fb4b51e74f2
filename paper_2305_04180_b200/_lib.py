"""ctypes binding of the C-ABI in ``include/sparrow.h`` (``_lib/libsparrow.so``).

The product has exactly one compute path: this CUDA library.  There is no
CPU fallback -- if the shared object is missing or no CUDA device is visible
the import of a compute entry point raises immediately.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPARROW_LIB_PATH") or os.path.join(HERE, "_lib", "libsparrow.so")

SP_OK, SP_EINVAL, SP_EACTION, SP_EEPISODE, SP_EMAP, SP_ENOTREADY, SP_ECUDA, SP_ENOMEM = range(8)
SP_MAX_ACTIONS = 15
SP_MAX_DELAY = 64

c_dp = ctypes.POINTER(ctypes.c_double)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i8p = ctypes.POINTER(ctypes.c_int8)
c_vp = ctypes.c_void_p


class SpConfig(ctypes.Structure):
    _fields_ = [
        ("n_beams", ctypes.c_int32),
        ("max_range_cm", ctypes.c_double),
        ("robot_radius_cm", ctypes.c_double),
        ("timeout_steps", ctypes.c_int32),
        ("proximity_cm", ctypes.c_double),
        ("n_actions", ctypes.c_int32),
        ("action_table", ctypes.c_double * (2 * SP_MAX_ACTIONS)),
        ("spawn_attempts", ctypes.c_int32),
        ("auto_reset", ctypes.c_int32),
        ("beam_offsets", c_dp),
    ]


class SpMapDesc(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int32),
        ("n_cols", ctypes.c_int32),
        ("cell_cm", ctypes.c_double),
        ("occupancy", ctypes.POINTER(ctypes.c_uint8)),
        ("goal_x", ctypes.c_double),
        ("goal_y", ctypes.c_double),
        ("goal_radius", ctypes.c_double),
        ("spawn", ctypes.c_double * 4),
        ("planning_dist", ctypes.c_double),
    ]


class SpRanges(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_double * 2),
        ("dt", ctypes.c_double * 2),
        ("delay", ctypes.c_int32 * 2),
        ("vmax_linear", ctypes.c_double * 2),
        ("vmax_angular", ctypes.c_double * 2),
        ("noise_std", ctypes.c_double * 2),
    ]


# (name, restype, argtypes) -- every symbol include/sparrow.h declares
SIGNATURES = [
    ("sp_last_error", ctypes.c_char_p, []),
    ("sp_version", ctypes.c_int, []),
    ("sp_device_info", ctypes.c_int, [ctypes.c_int, c_i32p, c_i32p, c_i32p, c_i32p]),
    ("sp_env_create", ctypes.c_int,
     [ctypes.POINTER(SpConfig), ctypes.POINTER(SpMapDesc), ctypes.c_int32, ctypes.c_int64,
      c_i32p, ctypes.POINTER(SpRanges), ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
      ctypes.POINTER(c_vp)]),
    ("sp_env_destroy", ctypes.c_int, [c_vp]),
    ("sp_env_reset_all", ctypes.c_int, [c_vp, ctypes.c_uint64, c_vp, c_vp]),
    ("sp_env_step", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    ("sp_env_host_out_bytes", ctypes.c_int64, [c_vp]),
    ("sp_env_step_host", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    ("sp_env_set_recording", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    ("sp_env_read_fifo", ctypes.c_int, [c_vp, c_vp, c_vp]),
    ("sp_env_first_pending", ctypes.c_int, [c_vp, c_vp, c_vp]),
    ("sp_env_check", ctypes.c_int, [c_vp, c_vp, c_i64p]),
    ("sp_env_any_needs_reset", ctypes.c_int, [c_vp, c_vp, c_i32p]),
    ("sp_env_stats_read", ctypes.c_int, [c_vp, c_i64p, c_i64p, c_dp, c_i8p, c_dp, c_i64p, c_vp]),
    ("sp_env_recent_returns", ctypes.c_int, [c_vp, c_dp, c_i32p, c_vp]),
    ("sp_env_recent_returns_keyed", ctypes.c_int, [c_vp, c_dp, c_vp, c_i32p, c_vp]),
    ("sp_env_stats_reset", ctypes.c_int, [c_vp, ctypes.c_int, c_vp]),
    ("sp_env_stats_totals", ctypes.c_int, [c_vp, c_vp, c_vp]),
    ("sp_env_read_state", ctypes.c_int, [c_vp, ctypes.c_int, c_dp, c_vp]),
    ("sp_env_write_state", ctypes.c_int, [c_vp, ctypes.c_int, c_dp, c_vp]),
    ("sp_env_reset_lanes", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    ("sp_env_map_info", ctypes.c_int, [c_vp, c_i64p, c_i64p, c_i32p, c_i32p]),
    ("sp_env_launch_info", ctypes.c_int, [c_vp, c_i64p, c_vp]),
    ("sp_env_scan", ctypes.c_int, [c_vp, ctypes.c_int64, c_i64p, c_vp, c_vp, c_vp, c_vp, c_vp,
                                   c_vp]),
    ("sp_cast_rays", ctypes.c_int,
     [c_vp, c_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, c_vp, c_vp, c_vp, c_vp, c_vp,
      ctypes.c_int64, ctypes.c_double, ctypes.c_double, c_vp, c_vp]),
    ("sp_disc_collides", ctypes.c_int,
     [c_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, c_vp, c_vp, c_vp, c_vp,
      ctypes.c_int64, ctypes.c_double, c_vp, c_vp]),
    ("sp_rb_create", ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int,
                                    ctypes.POINTER(c_vp)]),
    ("sp_rb_destroy", ctypes.c_int, [c_vp]),
    ("sp_rb_append", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp,
                                    ctypes.c_int64, c_vp]),
    ("sp_rb_sample", ctypes.c_int, [c_vp, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                                    ctypes.c_uint64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    ("sp_rb_sample_dev", ctypes.c_int, [c_vp, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                                        c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    ("sp_rb_size", ctypes.c_int, [c_vp, c_i64p, c_i64p]),
    ("sp_rb_gather", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    ("sp_philox_fill", ctypes.c_int, [ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                                      ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_double, c_vp, c_vp]),
    ("sp_random_actions", ctypes.c_int, [ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int32, c_vp, c_vp]),
    ("sp_adam_step", ctypes.c_int, [ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_i64p, c_vp,
                                    ctypes.c_int64, c_vp, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, c_vp]),
    ("sp_ddqn_scratch_floats", ctypes.c_int64, [c_i32p, ctypes.c_int64]),
    ("sp_actor_select", ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, ctypes.c_int64, c_vp,
                                       ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                                       ctypes.c_uint32, ctypes.c_uint64, c_vp, c_vp, c_vp]),
    ("sp_ddqn_update", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int64,
                                      ctypes.c_float, c_vp, c_vp, c_vp, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double, c_vp,
                                      ctypes.c_int64, c_vp, c_vp]),
]

_lib = None


class SpMlp(ctypes.Structure):
    _fields_ = [
        ("sizes", ctypes.c_int32 * 4),
        ("W", ctypes.c_void_p * 3),
        ("b", ctypes.c_void_p * 3),
    ]


class SpVem(ctypes.Structure):
    _fields_ = [
        ("n_envs", ctypes.c_int64), ("or_init", ctypes.c_int64), ("or_final", ctypes.c_int64),
        ("decay_steps", ctypes.c_int64), ("e_min", ctypes.c_double), ("e_max", ctypes.c_double),
    ]


class SparrowError(RuntimeError):
    """A failure reported by libsparrow (CUDA error, bad handle, ...)."""


def load() -> ctypes.CDLL:
    """Load libsparrow.so; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2305_04180_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    variant = "SPARROW_LIB_PATH" in os.environ  # A/B builds may predate newer entry points
    for name, res, args in SIGNATURES:
        if variant and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


TORCH_EXT = os.path.join(HERE, "_lib", "sparrow_torch.so")
_ops = None


def torch_ops():
    """torch.ops.sparrow: the PyTorch C++ extension (csrc/sp_torch.cpp) bound to
    the loaded libsparrow.so -- the binding of the hot calls (env step, ring
    append).  It checks tensors in C++ and takes the current CUDA stream from
    ATen.  None when the extension was not built (then ctypes drives the same
    C-ABI entry points)."""
    global _ops
    if _ops is None:
        load()
        import torch
        if not os.path.exists(TORCH_EXT):
            _ops = False
        else:
            torch.ops.load_library(TORCH_EXT)
            torch.ops.sparrow.bind(os.path.abspath(LIB_PATH))
            _ops = torch.ops.sparrow
    return _ops or None


def status_of(exc: BaseException) -> int:
    """The SpStatus a torch.ops.sparrow call failed with (in its message); a
    failed tensor check in the extension is a ValueError like the ctypes
    path's argument checks."""
    import re
    m = re.search(r"\(status (\d+)\)", str(exc))
    return int(m.group(1)) if m else SP_EINVAL


def binding() -> str:
    return "torch C++ extension (torch.ops.sparrow)" if torch_ops() else "ctypes"


def last_error() -> str:
    return load().sp_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map an SpStatus to the reference's exception classes."""
    if rc == SP_OK:
        return
    from paper_2305_04180_b200.sim import EpisodeTerminated, MapError
    from paper_2305_04180_b200.replay import BufferNotReady
    msg = last_error() or what
    if rc in (SP_EINVAL, SP_EACTION):
        raise ValueError(msg)
    if rc == SP_EEPISODE:
        raise EpisodeTerminated(msg)
    if rc == SP_EMAP:
        raise MapError(msg)
    if rc == SP_ENOTREADY:
        raise BufferNotReady(msg)
    if rc == SP_ENOMEM:
        raise MemoryError(msg)
    raise SparrowError(f"{what}: {msg}" if what else msg)


def require_cuda(device=None):
    """The device every compute call runs on; raises when CUDA is absent."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2305_04180_b200 needs a CUDA device (no CPU fallback)")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def stream_ptr(device) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream
