"""Time one libdfno kernel at the C2 geometry with CUDA events (median of N).
Usage: python tools/time_kernel.py yzt_fwd|yzt_fwd_grad|yzt_inv|xspec_fwd|xspec_bwd|xdft|xmix_fwd|xmix_bwd|xidft|mix_fwd|mix_bwd [reps]"""
import ctypes
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_12709_b200 import _lib  # noqa: E402
from paper_2211_12709_b200.partition import block_starts  # noqa: E402


def main(which, reps=20, grid=(64, 64, 64, 32), c=20):
    lib = _lib.load()
    ret = tuple(min(16, n) for n in grid)
    P = int(os.environ.get("TK_P", "1"))  # rank 0 of a P-way decomposition (buffers sized for P = 1)
    g = _lib.make_geom(batch=1, c_in=c, c=c, c_out=c, grid=grid, modes=(8, 8, 8, 8), retained=ret, nranks=P,
                       rank=0, dtype=_lib.F32,
                       act=_lib.ACT_IDENTITY if os.environ.get("TK_ACT") == "id" else _lib.ACT_GELU, x_starts=block_starts(grid[0], P),
                       ky_starts=block_starts(ret[1], P))
    gp = ctypes.byref(g)
    st = _lib.stream_handle()
    a = torch.randn((1, c) + grid, device="cuda")
    p = torch.randn((1, c) + grid, device="cuda")
    b = torch.empty_like(a)
    s3 = torch.randn((1, c) + grid, device="cuda")  # distinct third activation (no aliasing in mix_bwd)
    xk = torch.randn((1, c, grid[0], 16, 16, 16), dtype=torch.complex64, device="cuda")
    w = torch.randn((c, c, 16, 16, 16, 16), dtype=torch.complex64, device="cuda")
    spec = torch.randn((1, c, 16, 16, 16, 16), dtype=torch.complex64, device="cuda")
    spec2 = torch.empty_like(spec)
    spec3 = torch.randn_like(spec)
    out = torch.empty_like(xk)
    gw = torch.empty_like(w)
    npts = grid[0] * grid[1] * grid[2] * grid[3]
    n = ctypes.c_int64()
    k = ctypes.c_int()
    lib.dfno_mix_bwd_partials(gp, npts, c, c, ctypes.byref(n), ctypes.byref(k))
    parts = torch.empty(n.value, device="cuda")
    ws = ctypes.c_int64()
    lib.dfno_xspec_workspace(gp, ctypes.byref(ws))
    work = torch.empty(ws.value, dtype=torch.uint8, device="cuda")
    fns = {
        "xspec_fwd_ws": lambda: lib.dfno_xspec_fwd_ws(gp, _lib.ptr(xk), _lib.ptr(w), _lib.ptr(spec), _lib.ptr(out),
                                                      _lib.ptr(work), st),
        "xspec_bwd_ws": lambda: lib.dfno_xspec_bwd_ws(gp, _lib.ptr(xk), _lib.ptr(spec), _lib.ptr(w), _lib.ptr(gw),
                                                      _lib.ptr(out), _lib.ptr(work), st),
        "yzt_fwd": lambda: lib.dfno_dft_yzt_fwd(gp, _lib.ptr(a), None, _lib.SRC_ACT, 1.0, _lib.ptr(xk), st),
        "yzt_fwd_grad": lambda: lib.dfno_dft_yzt_fwd(gp, _lib.ptr(a), _lib.ptr(p), _lib.SRC_GRAD, 1.0, _lib.ptr(xk), st),
        "yzt_inv": lambda: lib.dfno_dft_yzt_inv(gp, _lib.ptr(xk), 1.0, _lib.ptr(b), st),
        "xspec_fwd": lambda: lib.dfno_xspec_fwd(gp, _lib.ptr(xk), _lib.ptr(w), _lib.ptr(spec), _lib.ptr(out), st),
        "xspec_bwd": lambda: lib.dfno_xspec_bwd(gp, _lib.ptr(xk), _lib.ptr(spec), _lib.ptr(w), _lib.ptr(gw),
                                                _lib.ptr(out), st),
        "xdft": lambda: lib.dfno_xdft(gp, _lib.ptr(xk), ctypes.c_double(1.0), _lib.ptr(spec), st),
        "xmix_fwd": lambda: lib.dfno_xmix_fwd(gp, _lib.ptr(spec), _lib.ptr(w), _lib.ptr(spec2), st),
        "xmix_bwd": lambda: lib.dfno_xmix_bwd(gp, _lib.ptr(spec), _lib.ptr(spec3), _lib.ptr(w), _lib.ptr(gw),
                                              _lib.ptr(spec2), st),
        "xidft": lambda: lib.dfno_xidft(gp, _lib.ptr(spec), ctypes.c_double(1.0), _lib.ptr(out), st),
        "mix_fwd": lambda: lib.dfno_mix_fwd(gp, npts, c, c, _lib.ptr(a), 1, _lib.ptr(w), _lib.ptr(p), None, st),
        "mix_fwd_post": lambda: lib.dfno_mix_fwd(gp, npts, c, c, _lib.ptr(a), 0, _lib.ptr(w), _lib.ptr(p), _lib.ptr(b),
                                                 st),
        "mix_fwd_enc": lambda: lib.dfno_mix_fwd(gp, npts, c, c, _lib.ptr(a), 0, _lib.ptr(w), _lib.ptr(p), None, st),
        "mix_fwd_dec": lambda: lib.dfno_mix_fwd(gp, npts, c, c, _lib.ptr(a), 1, _lib.ptr(w), _lib.ptr(p), _lib.ptr(b),
                                                st),
        "mix_bwd_raw": lambda: lib.dfno_mix_bwd(gp, npts, c, c, _lib.ptr(a), _lib.ptr(p), _lib.ptr(s3), 0, _lib.ptr(w),
                                                _lib.ptr(b), _lib.ptr(parts), st),
        "mix_bwd": lambda: lib.dfno_mix_bwd(gp, npts, c, c, _lib.ptr(a), _lib.ptr(p), _lib.ptr(s3), 1, _lib.ptr(w),
                                            _lib.ptr(b), _lib.ptr(parts), st),
    }
    f = fns[which]
    for _ in range(3):
        _lib.check(f(), which)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(f(), which)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{which}: median {statistics.median(ts) * 1e3:.1f} us  min {min(ts) * 1e3:.1f} us")


if __name__ == "__main__":
    # TK_GRID=x,y,z,t selects another slab geometry (e.g. 33,118,64,86: one C4 P = 8 rank)
    grid = tuple(int(v) for v in os.environ["TK_GRID"].split(",")) if os.environ.get("TK_GRID") else (64, 64, 64, 32)
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20, grid=grid)
