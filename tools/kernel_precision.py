"""Per-kernel fp32 error against the same C-ABI entry in fp64 (SIMT) on the
same inputs, at a chosen geometry (default C2: 64^3 x 32, m = 8):

    python tools/kernel_precision.py [--grid 64,64,64,32] [--c 4]

Metric max|a-b| / max(max|a|, max|b|) (d/bench.py:83-85)."""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_12709_b200 import _lib  # noqa: E402
from paper_2211_12709_b200.partition import block_starts  # noqa: E402


def rel(a, b):
    dt = torch.complex128 if a.is_complex() else torch.float64
    a, b = a.to(dt), b.to(dt)
    return ((a - b).abs().max() / torch.maximum(a.abs().max(), b.abs().max())).item()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="64,64,64,32")
    ap.add_argument("--c", type=int, default=4)
    args = ap.parse_args()
    grid = tuple(int(v) for v in args.grid.split(","))
    c = args.c
    ret = tuple(min(16, n) for n in grid)
    lib = _lib.load()

    def geom(dt):
        return _lib.make_geom(batch=1, c_in=c, c=c, c_out=c, grid=grid, modes=(8, 8, 8, 8), retained=ret, nranks=1,
                              rank=0, dtype=dt, act=_lib.ACT_GELU, x_starts=block_starts(grid[0], 1),
                              ky_starts=block_starts(ret[1], 1))

    g32, g64 = geom(_lib.F32), geom(_lib.F64)
    st = _lib.stream_handle()
    torch.manual_seed(0)
    a = torch.randn((1, c) + grid, device="cuda", dtype=torch.float64)
    pre = torch.randn((1, c) + grid, device="cuda", dtype=torch.float64)
    xk_shape = (1, c, grid[0], ret[1], ret[2], ret[3])
    out = {}

    def both(fn, ins, out_shape, out_dtype):
        res = []
        for g, rdt in ((g32, torch.float32), (g64, torch.float64)):
            args_ = [t.to(rdt if not t.is_complex() else (torch.complex64 if rdt == torch.float32 else
                                                            torch.complex128)) for t in ins]
            odt = out_dtype(rdt)
            o = torch.zeros(out_shape, dtype=odt, device="cuda")
            fn(ctypes.byref(g), args_, o)
            res.append(o)
        torch.cuda.synchronize()
        return rel(res[0], res[1])

    cplx = lambda r: torch.complex64 if r == torch.float32 else torch.complex128  # noqa: E731
    real = lambda r: r  # noqa: E731
    for mode, name in ((_lib.SRC_RAW, "yzt_fwd.raw"), (_lib.SRC_ACT, "yzt_fwd.act"), (_lib.SRC_GRAD, "yzt_fwd.grad")):
        out[name] = both(lambda g, t, o: _lib.check(lib.dfno_dft_yzt_fwd(g, _lib.ptr(t[0]), _lib.ptr(t[1]), mode, 1.0,
                                                                       _lib.ptr(o), st), name),
                         [a, pre], xk_shape, cplx)
    xk = torch.randn(xk_shape, device="cuda", dtype=torch.complex128)
    n = grid[1] * grid[2] * grid[3]
    out["yzt_inv"] = both(lambda g, t, o: _lib.check(lib.dfno_dft_yzt_inv(g, _lib.ptr(t[0]), 1.0 / n, _lib.ptr(o),
                                                                        st), "inv"),
                          [xk], (1, c) + grid, real)
    w = torch.randn((c, c), device="cuda", dtype=torch.float64) / c ** 0.5
    npts = grid[0] * n
    out["mix_fwd.act"] = both(lambda g, t, o: _lib.check(lib.dfno_mix_fwd(g, npts, c, c, _lib.ptr(t[0]), 1,
                                                                         _lib.ptr(t[1]), _lib.ptr(o), None, st), "mf"),
                              [a, w], (1, c) + grid, real)
    ws32, ws64 = ctypes.c_int64(), ctypes.c_int64()
    lib.dfno_xspec_workspace(ctypes.byref(g32), ctypes.byref(ws32))
    lib.dfno_xspec_workspace(ctypes.byref(g64), ctypes.byref(ws64))
    work = torch.empty(max(ws32.value, ws64.value, 1), dtype=torch.uint8, device="cuda")
    kx = torch.randn((1, c, grid[0], ret[1], ret[2], ret[3]), device="cuda", dtype=torch.complex128)
    wsp = torch.randn((c, c, ret[0], ret[1], ret[2], ret[3]), device="cuda", dtype=torch.complex128) / c
    spec_shape = (1, c, ret[0], ret[1], ret[2], ret[3])

    def xs(g, t, o):
        spec = torch.empty(spec_shape, dtype=o.dtype, device="cuda")
        _lib.check(lib.dfno_xspec_fwd_ws(g, _lib.ptr(t[0]), _lib.ptr(t[1]), _lib.ptr(spec), _lib.ptr(o),
                                         _lib.ptr(work), st), "xs")

    out["xspec_fwd"] = both(xs, [kx, wsp], xk_shape, cplx)
    print(json.dumps({k: f"{v:.3e}" for k, v in out.items()}))


if __name__ == "__main__":
    main()
