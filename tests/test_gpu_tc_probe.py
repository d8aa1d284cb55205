"""Hardware probe of the tcgen05 building blocks (tests/probes/probe_tc.cu):
kind::tf32 MMA with SWIZZLE_NONE K-major descriptors at the padded LBO/SBO
strides the DFT kernels use, B negation, K-step descriptor advance,
accumulate flag, and the tcgen05.ld 32x32b read-back."""

import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "tests" / "probes" / "libprobe.so"


@pytest.fixture(scope="module")
def probe():
    src = ROOT / "tests" / "probes" / "probe_tc.cu"
    if not SO.exists() or SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler",
                        "-fPIC", "-shared", f"-I{ROOT / 'paper_2211_12709_b200' / 'csrc'}", f"-I{ROOT / 'include'}",
                        str(src), "-o", str(SO)], check=True)
    lib = ctypes.CDLL(str(SO))
    lib.probe_run.restype = ctypes.c_int
    return lib


def trunc_tf32(x):
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)


def run(lib, M, N, K, lbo_a, sbo_a, lbo_b, sbo_b, neg=0, twice=0, seed=0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    a, b = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda")
    d = torch.zeros((M, N), device="cuda")
    rc = lib.probe_run(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(d.data_ptr()),
                       M, N, K, lbo_a, sbo_a, lbo_b, sbo_b, neg, twice)
    assert rc == 0
    want = (trunc_tf32(A) @ trunc_tf32(B).T) * (-1 if neg else 1) * (2 if twice else 1)
    got = d.cpu().numpy().astype(np.float64)
    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
    exact = (A.astype(np.float64) @ B.astype(np.float64).T) * (-1 if neg else 1) * (2 if twice else 1)
    err_exact = np.max(np.abs(got - exact)) / np.max(np.abs(exact))
    return err, err_exact


@pytest.mark.parametrize("case", [
    dict(M=128, N=32, K=32, lbo_a=144, sbo_a=1152, lbo_b=128, sbo_b=1024),
    dict(M=128, N=16, K=16, lbo_a=160, sbo_a=608, lbo_b=128, sbo_b=512),
    dict(M=128, N=16, K=8, lbo_a=192, sbo_a=320, lbo_b=128, sbo_b=256),
    dict(M=128, N=16, K=64, lbo_a=128, sbo_a=2048, lbo_b=144, sbo_b=2304, neg=1),
    dict(M=128, N=32, K=32, lbo_a=144, sbo_a=1152, lbo_b=128, sbo_b=1024, twice=1),
])
def test_tf32_mma_layouts(probe, case):
    err, err_exact = run(probe, **case)
    print(case, "err vs truncated-tf32 product", err, "vs fp32 product", err_exact)
    assert err < 1e-5
