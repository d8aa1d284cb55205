"""Run each libdfno kernel at the C2 benchmark geometry (64^3 x 32, c = 20,
m = 8) a few times -- a short, single-GPU command for ncu captures:

    ncu --set full -k regex:k_yzt_fwd_tc -c 1 python tools/kernel_driver.py yzt_fwd
"""

import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_12709_b200 import _lib  # noqa: E402
from paper_2211_12709_b200.partition import block_starts  # noqa: E402


def main(which: str, reps: int = 3, grid=(64, 64, 64, 32), c=20):
    lib = _lib.load()
    ret = tuple(min(16, n) for n in grid)
    g = _lib.make_geom(batch=1, c_in=c, c=c, c_out=c, grid=grid, modes=(8, 8, 8, 8), retained=ret, nranks=1,
                       rank=0, dtype=_lib.F32, act=_lib.ACT_GELU, x_starts=block_starts(grid[0], 1),
                       ky_starts=block_starts(ret[1], 1))
    gp = ctypes.byref(g)
    st = _lib.stream_handle()
    a = torch.randn((1, c) + grid, device="cuda")
    p = torch.randn((1, c) + grid, device="cuda")
    xk = torch.randn((1, c, grid[0], 16, 16, 16), dtype=torch.complex64, device="cuda")
    w = torch.randn((c, c, 16, 16, 16, 16), dtype=torch.complex64, device="cuda")
    spec = torch.empty((1, c, 16, 16, 16, 16), dtype=torch.complex64, device="cuda")
    out = torch.empty_like(xk)
    npts = grid[0] * grid[1] * grid[2] * grid[3]
    for _ in range(reps):
        if which in ("yzt_fwd", "all"):
            _lib.check(lib.dfno_dft_yzt_fwd(gp, _lib.ptr(a), None, _lib.SRC_ACT, 1.0, _lib.ptr(xk), st), "fwd")
        if which in ("yzt_fwd_grad", "all"):
            _lib.check(lib.dfno_dft_yzt_fwd(gp, _lib.ptr(a), _lib.ptr(p), _lib.SRC_GRAD, 1.0, _lib.ptr(xk), st), "g")
        if which in ("yzt_inv", "all"):
            _lib.check(lib.dfno_dft_yzt_inv(gp, _lib.ptr(xk), 1.0, _lib.ptr(a), st), "inv")
        if which in ("xspec", "all"):
            _lib.check(lib.dfno_xspec_fwd(gp, _lib.ptr(xk), _lib.ptr(w), _lib.ptr(spec), _lib.ptr(out), st), "x")
            _lib.check(lib.dfno_xspec_bwd(gp, _lib.ptr(xk), _lib.ptr(spec), _lib.ptr(w), _lib.ptr(spec),
                                          _lib.ptr(out), st), "xb")
        if which in ("mix", "all"):
            _lib.check(lib.dfno_mix_fwd(gp, npts, c, c, _lib.ptr(a), 1, _lib.ptr(w), _lib.ptr(p), None, st), "m")
            n = ctypes.c_int64()
            k = ctypes.c_int()
            lib.dfno_mix_bwd_partials(gp, npts, c, c, ctypes.byref(n), ctypes.byref(k))
            parts = torch.empty(n.value, device="cuda")
            b = torch.empty_like(a)
            _lib.check(lib.dfno_mix_bwd(gp, npts, c, c, _lib.ptr(a), _lib.ptr(p), _lib.ptr(a), 1, _lib.ptr(w),
                                        _lib.ptr(b), _lib.ptr(parts), st), "mb")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
