"""Per-role mbarrier wait fractions of the yzt forward kernel (diagnostics
build: python tools/build_variant.py prof -DDFNO_WAIT_PROF, swapped in by
tools/wait_prof.sh).  Prints, per warp index, the share of its lifetime spent
waiting, averaged over CTAs; the bottleneck role waits least.
usage: [TK_GRID=x,y,z,t] python tools/wait_prof.py yzt_fwd|yzt_fwd_grad"""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_2211_12709_b200 import _lib  # noqa: E402
import time_kernel  # noqa: E402

ROLES = {0: "conv", 8: "T-epi", 16: "Z-epi", 20: "TMA", 21: "issT0", 22: "issT1", 23: "issZ", 24: "issY", 25: "twid"}
ROLES_INV = {0: "front", 4: "T-epi", 8: "O-epi", 16: "issY", 17: "issT", 18: "issZ", 20: "loader", 21: "twid"}


def main(which):
    grid = tuple(int(v) for v in os.environ["TK_GRID"].split(",")) if os.environ.get("TK_GRID") else (64, 64, 64, 32)
    time_kernel.main(which, 3, grid=grid)  # warm-up + timing print
    lib = _lib.load()
    buf = np.zeros((160, 32, 2), dtype=np.uint64)
    inv = which.startswith("yzt_inv")
    f = lib.dfno_debug_wait_prof_inv if inv else lib.dfno_debug_wait_prof_fwd
    roles = ROLES_INV if inv else ROLES
    f(buf.ctypes.data_as(ctypes.c_void_p))  # clear
    time_kernel.main(which, 1, grid=grid)
    f(buf.ctypes.data_as(ctypes.c_void_p))
    wait, life = buf[:, :, 0].astype(float), buf[:, :, 1].astype(float)
    act = life.sum(0) > 0
    print(f"{which} grid {grid}: per-warp wait share of lifetime (mean over CTAs); lifetime {life[:148].mean(0).max():.0f} cyc")
    for w in range(32):
        if not act[w]:
            continue
        role = max(k for k in roles if k <= w)
        share = wait[:, w].sum() / max(life[:, w].sum(), 1)
        print(f"  warp {w:2d} {roles[role]:6s} wait {100 * share:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
