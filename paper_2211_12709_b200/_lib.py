"""ctypes binding of libdfno.so (the C ABI declared in include/dfno.h).

The library is loaded from the package's ``lib/`` directory (built in-tree
by ``build.py``).  There is no fallback: if the library or a CUDA device is
missing, every hot-path call raises ``ExtensionMissingError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

from .errors import (
    DimensionMismatchError,
    DistFnoError,
    DTypeMismatchError,
    ExtensionMissingError,
    InfeasiblePartitionError,
    KernelError,
    ShapeMismatchError,
)

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libdfno.so"
MAX_RANKS = 64

F32, F64 = 0, 1
ACT_RELU, ACT_GELU, ACT_IDENTITY = 0, 1, 2
SRC_ACT, SRC_GRAD, SRC_RAW = 0, 1, 2

_STATUS_EXC = {
    -1: DimensionMismatchError,
    -2: DTypeMismatchError,
    -3: InfeasiblePartitionError,
    -4: ShapeMismatchError,
    -5: DistFnoError,
    -6: KernelError,
    -7: KernelError,
}

# Every symbol include/dfno.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "dfno_abi_version", "dfno_status_string", "dfno_build_info", "dfno_geom_validate", "dfno_sizes",
    "dfno_mix_fwd", "dfno_mix_bwd_partials", "dfno_mix_bwd", "dfno_reduce_partials",
    "dfno_dft_yzt_fwd", "dfno_dft_yzt_inv", "dfno_xspec_fwd", "dfno_xspec_bwd",
    "dfno_xspec_workspace", "dfno_xspec_fwd_ws", "dfno_xspec_bwd_ws",
    "dfno_xdft", "dfno_xmix_fwd", "dfno_xmix_bwd", "dfno_xidft",
    "dfno_mse_partials", "dfno_mse_grad", "dfno_adam", "dfno_adam_out",
)


class Geom(ctypes.Structure):
    """Mirror of ``dfno_geom`` (include/dfno.h)."""

    _fields_ = [(n, ctypes.c_int32) for n in (
        "batch", "c_in", "c", "c_out", "nx", "ny", "nz", "nt", "mx", "my", "mz", "mt",
        "rx", "ry", "rz", "rt", "nranks", "rank", "dtype", "act")] + [
        ("x_starts", ctypes.c_int32 * (MAX_RANKS + 1)),
        ("ky_starts", ctypes.c_int32 * (MAX_RANKS + 1)),
    ]


_lib = None


def load(path: Path = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the library.  Raises ExtensionMissingError."""
    global _lib
    if _lib is not None:
        return _lib
    if not path.exists():
        raise ExtensionMissingError(
            f"{path} is missing; build it with `python -m paper_2211_12709_b200.build` (no CPU fallback)"
        )
    lib = ctypes.CDLL(str(path))
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    gp = ctypes.POINTER(Geom)
    sig = {
        "dfno_abi_version": ([], i32),
        "dfno_status_string": ([i32], ctypes.c_char_p),
        "dfno_build_info": ([], ctypes.c_char_p),
        "dfno_geom_validate": ([gp], i32),
        "dfno_sizes": ([gp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
        "dfno_mix_fwd": ([gp, i64, i32, i32, vp, i32, vp, vp, vp, vp], i32),
        "dfno_mix_bwd_partials": ([gp, i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i32)], i32),
        "dfno_mix_bwd": ([gp, i64, i32, i32, vp, vp, vp, i32, vp, vp, vp, vp], i32),
        "dfno_reduce_partials": ([gp, i32, i64, vp, vp, vp], i32),
        "dfno_dft_yzt_fwd": ([gp, vp, vp, i32, dbl, vp, vp], i32),
        "dfno_dft_yzt_inv": ([gp, vp, dbl, vp, vp], i32),
        "dfno_xspec_fwd": ([gp, vp, vp, vp, vp, vp], i32),
        "dfno_xspec_bwd": ([gp, vp, vp, vp, vp, vp, vp], i32),
        "dfno_xspec_workspace": ([gp, ctypes.POINTER(i64)], i32),
        "dfno_xspec_fwd_ws": ([gp, vp, vp, vp, vp, vp, vp], i32),
        "dfno_xspec_bwd_ws": ([gp, vp, vp, vp, vp, vp, vp, vp], i32),
        "dfno_xdft": ([gp, vp, dbl, vp, vp], i32),
        "dfno_xmix_fwd": ([gp, vp, vp, vp, vp], i32),
        "dfno_xmix_bwd": ([gp, vp, vp, vp, vp, vp, vp], i32),
        "dfno_xidft": ([gp, vp, dbl, vp, vp], i32),
        "dfno_mse_partials": ([i64, ctypes.POINTER(i32)], i32),
        "dfno_mse_grad": ([gp, i64, vp, vp, dbl, vp, vp, vp, vp], i32),
        "dfno_adam": ([gp, i64, vp, vp, vp, vp, dbl, dbl, dbl, dbl, i32, vp], i32),
        "dfno_adam_out": ([gp, i64, vp, vp, vp, vp, vp, dbl, dbl, dbl, dbl, i32, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status != 0:
        lib = load()
        msg = lib.dfno_status_string(status).decode()
        raise _STATUS_EXC.get(status, DistFnoError)(f"{what}: {msg} (status {status})")


def require_device(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise ExtensionMissingError(f"{what} must live on a CUDA device (no CPU fallback)")


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def stream_handle() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_geom(*, batch, c_in, c, c_out, grid, modes, retained, nranks, rank, dtype, act, x_starts, ky_starts) -> Geom:
    g = Geom()
    g.batch, g.c_in, g.c, g.c_out = batch, c_in, c, c_out
    g.nx, g.ny, g.nz, g.nt = grid
    g.mx, g.my, g.mz, g.mt = modes
    g.rx, g.ry, g.rz, g.rt = retained
    g.nranks, g.rank, g.dtype, g.act = nranks, rank, dtype, act
    for i, v in enumerate(x_starts):
        g.x_starts[i] = v
    for i, v in enumerate(ky_starts):
        g.ky_starts[i] = v
    return g


def available() -> bool:
    """True when libdfno.so loads and a CUDA device is present."""
    try:
        load()
    except (ExtensionMissingError, OSError):
        return False
    return torch.cuda.is_available() and os.environ.get("DFNO_FORCE_UNAVAILABLE") != "1"
