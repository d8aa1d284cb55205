"""cuFFT comparison (north star item 1; SURVEY.md section 8d "cuFFT
comparator"): the reference's algorithm restated with torch.fft (cuFFT) on the
same B200, against the libdfno truncated-DFT path, at C2 (64^3 x 32, c = 20,
m = 8, 4 blocks, batch 1, fp32 / complex64).

  stage  yzt forward   ours: dfno_dft_yzt_fwd (act fused)      torch: gelu -> fftn(y,z,t) -> gather retained
  stage  yzt inverse   ours: dfno_dft_yzt_inv                  torch: zero-pad -> ifftn(y,z,t) -> real
  model  fwd + bwd     ours: fno_forward + fno_backward        torch: the reference's serial network
         (g = y)                                              (d/oracle.py:25-62) with torch.fft + autograd

Prints one JSON line; python tools/cufft_compare.py > profiles/<tag>_cufft_compare.json
"""

import ctypes
import json
import math
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2211_12709_b200 as P  # noqa: E402
from paper_2211_12709_b200 import _lib  # noqa: E402
from paper_2211_12709_b200.partition import block_starts  # noqa: E402

GRID, C, MODES, BLOCKS = (64, 64, 64, 32), 20, (8, 8, 8, 8), 4


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def keep(n, m, dev):
    idx = list(range(n)) if 2 * m >= n else list(range(m)) + list(range(n - m, n))
    return torch.tensor(idx, device=dev)


def gelu(h):
    return 0.5 * h * (1.0 + torch.erf(h * (1.0 / math.sqrt(2.0))))


def main():
    dev = torch.device("cuda")
    lib = _lib.load()
    ret = tuple(min(2 * m, n) for n, m in zip(GRID, MODES))
    g = _lib.make_geom(batch=1, c_in=C, c=C, c_out=C, grid=GRID, modes=MODES, retained=ret, nranks=1, rank=0,
                       dtype=_lib.F32, act=_lib.ACT_GELU, x_starts=block_starts(GRID[0], 1),
                       ky_starts=block_starts(ret[1], 1))
    gp, st = ctypes.byref(g), _lib.stream_handle()
    a = torch.randn((1, C) + GRID, device=dev)
    xk = torch.empty((1, C, GRID[0]) + ret[1:], dtype=torch.complex64, device=dev)
    out = torch.empty_like(a)
    ky, kz, kt = (keep(n, m, dev) for n, m in zip(GRID[1:], MODES[1:]))
    res = {"config": "C2 64^3 x 32, c = 20, m = 8, batch 1, fp32 / complex64", "unit": "ms (median, CUDA events)"}

    # ---- stage: yzt forward ------------------------------------------------
    res["yzt_fwd_ours_ms"] = timed(lambda: lib.dfno_dft_yzt_fwd(gp, _lib.ptr(a), None, _lib.SRC_ACT, 1.0,
                                                                   _lib.ptr(xk), st))

    def torch_fwd():
        s = torch.fft.fftn(gelu(a).to(torch.complex64), dim=(3, 4, 5))
        return s.index_select(3, ky).index_select(4, kz).index_select(5, kt)

    res["yzt_fwd_cufft_ms"] = timed(torch_fwd)
    ref = torch_fwd()
    lib.dfno_dft_yzt_fwd(gp, _lib.ptr(a), None, _lib.SRC_ACT, 1.0, _lib.ptr(xk), st)
    torch.cuda.synchronize()
    res["yzt_fwd_max_rel_diff"] = float((xk - ref).abs().max() / ref.abs().max())

    # ---- stage: yzt inverse ------------------------------------------------
    res["yzt_inv_ours_ms"] = timed(lambda: lib.dfno_dft_yzt_inv(gp, _lib.ptr(xk), 1.0 / (64 * 64 * 32), _lib.ptr(out),
                                                                   st))

    def torch_inv():
        pad = torch.zeros((1, C) + GRID, dtype=torch.complex64, device=dev)
        pad[:, :, :, ky[:, None, None], kz[None, :, None], kt[None, None, :]] = xk
        return torch.fft.ifftn(pad, dim=(3, 4, 5)).real

    res["yzt_inv_cufft_ms"] = timed(torch_inv)
    r2 = torch_inv()
    lib.dfno_dft_yzt_inv(gp, _lib.ptr(xk), 1.0 / (64 * 64 * 32), _lib.ptr(out), st)
    torch.cuda.synchronize()
    res["yzt_inv_max_rel_diff"] = float((out - r2).abs().max() / r2.abs().max())

    # ---- model: fwd + bwd --------------------------------------------------
    cfg = P.FnoConfig(*GRID, C, C, C, P.ModeSpec.of_xyzt(*MODES), BLOCKS, "gelu", "real32", 1)
    params = P.init_params(cfg, 42, device=dev)
    comm = P.run_ranks(1, lambda c: c)[0]
    x = P.DenseTensor(P.DATA_LABELS, torch.randn((1, C) + GRID, device=dev))

    def ours():
        cache = P.ForwardCache()
        y = P.fno_forward(comm, x, params, cfg, cache)
        P.fno_backward(comm, y, params, cfg, cache)

    res["model_ours_ms"] = timed(ours, reps=5, warm=2)
    we = params.we.data.clone().requires_grad_(True)
    wd = params.wd.data.clone().requires_grad_(True)
    ws = [w.data.clone().requires_grad_(True) for w in params.blocks]
    kx = keep(64, 8, dev)

    def torch_model():
        h = gelu(torch.einsum("bixyzt,io->boxyzt", x.data, we))
        for w in ws:
            s = torch.fft.fftn(h.to(torch.complex64), dim=(2, 3, 4, 5))
            s = s.index_select(2, kx).index_select(3, ky).index_select(4, kz).index_select(5, kt)
            s = torch.einsum("bi...,io...->bo...", s, w)
            pad = torch.zeros((1, C) + GRID, dtype=torch.complex64, device=dev)
            pad = pad.index_put((torch.arange(1, device=dev)[:, None, None, None, None, None],
                                 torch.arange(C, device=dev)[None, :, None, None, None, None],
                                 kx[None, None, :, None, None, None], ky[None, None, None, :, None, None],
                                 kz[None, None, None, None, :, None], kt[None, None, None, None, None, :]), s)
            h = gelu(torch.fft.ifftn(pad, dim=(2, 3, 4, 5)).real)
        y = gelu(torch.einsum("bixyzt,io->boxyzt", h, wd))
        (0.5 * (y * y).sum()).backward()

    res["model_cufft_autograd_ms"] = timed(torch_model, reps=5, warm=2)
    res["model_ours_samples_per_s"] = 1e3 / res["model_ours_ms"]
    res["model_cufft_samples_per_s"] = 1e3 / res["model_cufft_autograd_ms"]
    res["speedup_model"] = res["model_cufft_autograd_ms"] / res["model_ours_ms"]
    res["speedup_yzt_fwd"] = res["yzt_fwd_cufft_ms"] / res["yzt_fwd_ours_ms"]
    res["speedup_yzt_inv"] = res["yzt_inv_cufft_ms"] / res["yzt_inv_ours_ms"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
