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


@pytest.mark.parametrize("M,N,K,lbo,sbo", [(128, 32, 32, 512, 2048), (128, 32, 32, 4096, 512), (128, 64, 8, 512, 2048)])
def test_tf32_mma_mn_major_a(probe, M, N, K, lbo, sbo):
    """MN-major tf32 A operand in the SWIZZLE_128B_BASE32B canonical form
    (4 K rows x 128 B atoms, 32-byte chunks XOR k % 4; LBO = MN-atom stride,
    SBO = 4-row K-group stride) -- the only MN-major tf32 layout the tensor
    core accepts (tools/probe_mn.py: no-swizzle / plain 128B give zeros)."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    a, b = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda")
    d = torch.zeros((M, N), device="cuda")
    probe.probe_run_mn.restype = ctypes.c_int
    rc = probe.probe_run_mn(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(d.data_ptr()),
                            M, N, K, lbo, sbo, 128, (K // 4) * 128, 3)
    assert rc == 0
    want = trunc_tf32(A) @ trunc_tf32(B).T
    assert np.max(np.abs(d.cpu().numpy() - want)) / np.max(np.abs(want)) < 1e-5


def _perf_lib():
    src = ROOT / "tests" / "probes" / "probe_tc_perf.cu"
    so = ROOT / "tests" / "probes" / "libprobe_perf.so"
    if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler",
                        "-fPIC", "-shared", f"-I{ROOT / 'paper_2211_12709_b200' / 'csrc'}", f"-I{ROOT / 'include'}",
                        str(src), "-o", str(so)], check=True)
    lib = ctypes.CDLL(str(so))
    lib.probe_perf_run.restype = ctypes.c_int
    return lib


@pytest.fixture(scope="module")
def perf():
    return _perf_lib()


def _perf(lib, mode, N, K, R, A=None, B=None):
    cyc = torch.zeros(2, dtype=torch.int64, device="cuda")
    d = torch.zeros((128, N), device="cuda")
    vp = ctypes.c_void_p
    rc = lib.probe_perf_run(mode, vp(A.data_ptr() if A is not None else 0), vp(B.data_ptr() if B is not None else 0),
                            vp(d.data_ptr()), N, K, R, vp(cyc.data_ptr()))
    assert rc == 0
    c = cyc.cpu()
    _perf.ns = int(c[1])
    return int(c[0]), d


def test_tf32_mma_a_from_tmem(perf):
    """tcgen05.mma kind::tf32 with A in TMEM (lane = row, column = k) matches
    the truncated-TF32 product."""
    rng = np.random.default_rng(3)
    for N, K in ((32, 32), (64, 16), (16, 64)):
        A = rng.standard_normal((128, K)).astype(np.float32)
        B = rng.standard_normal((N, K)).astype(np.float32)
        _, d = _perf(perf, 2, N, K, 1, torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda"))
        want = trunc_tf32(A) @ trunc_tf32(B).T
        err = np.max(np.abs(d.cpu().numpy() - want)) / np.max(np.abs(want))
        assert err < 1e-5, (N, K, err)


def report_tcgen05_throughput(perf):
    """Cycle counts behind the DFT kernels' tiling choices (printed; -s)."""
    R = 256
    a = torch.randn(4096, 4096, device="cuda")
    for _ in range(50):  # ramp the SM clock
        a = a @ a
        a /= a.norm()
    torch.cuda.synchronize()
    for N in (16, 32, 64, 128, 256):
        ss, _ = _perf(perf, 0, N, 32, R)
        ts, _ = _perf(perf, 1, N, 32, R)
        print(f"M=128 K=8 N={N:3d}: SS {ss / (4 * R):6.1f} cyc/MMA   TS {ts / (4 * R):6.1f} cyc/MMA "
              f"({_perf.ns / (4 * R):.1f} ns/MMA, clock {ts / _perf.ns:.2f} GHz)")
    for N in (16, 32, 64):
        for Pn in (2, 4, 8):
            if Pn * N > 256:
                continue
            ss, _ = _perf(perf, 10 + Pn, N, 32, R)
            ts, _ = _perf(perf, 20 + Pn, N, 32, R)
            print(f"N={N:3d} x {Pn} independent accumulators: SS {ss / (4 * R):6.1f} cyc/MMA   TS {ts / (4 * R):6.1f}")
    ld, _ = _perf(perf, 3, 32, 32, R)
    st, _ = _perf(perf, 4, 32, 32, R)
    print(f"tcgen05.ld 32x32b.x32 (4 warps, 16 KB): {ld / R:.1f} cyc  -> {16384 * R / ld:.0f} B/cyc")
    print(f"tcgen05.st 32x32b.x32 (4 warps, 16 KB): {st / R:.1f} cyc  -> {16384 * R / st:.0f} B/cyc")


def report_tcgen05_issue_rate(perf):
    """Back-to-back MMA rate with precomputed descriptors (printed; -s)."""
    a = torch.randn(4096, 4096, device="cuda")
    for _ in range(50):
        a = a @ a
        a /= a.norm()
    torch.cuda.synchronize()
    cyc = torch.zeros(2, dtype=torch.int64, device="cuda")
    R = 64
    for kind, ts, name in ((1, 0, "bf16 SS"), (0, 0, "tf32 SS"), (0, 1, "tf32 TS")):
        for N in (16, 32, 64, 128, 256):
            for Pn in (1, 4):
                if Pn * N > 384:
                    continue
                out = []
                for variant in (0, 1):
                    assert perf.probe_rate_run(kind, ts, N, Pn, R, ctypes.c_void_p(cyc.data_ptr()), variant) == 0
                    out.append(int(cyc[0]) / (8 * R))
                print(f"{name} M=128 N={N:3d} P={Pn}: spinning lanes {out[0]:7.1f}  parked lanes {out[1]:7.1f} cyc/MMA")


def report_tcgen05_lean_issue(perf):
    a = torch.randn(4096, 4096, device="cuda")
    for _ in range(50):
        a = a @ a
        a /= a.norm()
    torch.cuda.synchronize()
    cyc = torch.zeros(2, dtype=torch.int64, device="cuda")
    names = ["SS N16 P1", "SS N16 P4", "SS N32 P1", "SS N32 P4", "SS N64 P1", "SS N64 P4", "SS N128 P1",
             "TS N16 P4", "TS N32 P4", "TS N64 P4", "SS N16 2 issuing warps (cyc per warp-MMA)",
             "SS N16 4 issuing warps", "TS N32 2 issuing warps", "TS N32 4 issuing warps"]
    for i, n in enumerate(names):
        assert perf.probe_lean_run(i, 64, ctypes.c_void_p(cyc.data_ptr())) == 0
        print(f"lean tf32 M=128 {n}: {int(cyc[0]) / (8 * 64):6.1f} cyc/MMA")


def report_tcgen05_issue_under_contention(perf):
    a = torch.randn(4096, 4096, device="cuda")
    for _ in range(50):
        a = a @ a
        a /= a.norm()
    torch.cuda.synchronize()
    cyc = torch.zeros(2, dtype=torch.int64, device="cuda")
    R = 64
    for bg, name in ((0, "idle"), (1, "FFMA"), (2, "tcgen05.ld"), (3, "tcgen05.st")):
        for warps in (2, 8, 24):
            assert perf.probe_contention_run(R, bg, warps, ctypes.c_void_p(cyc.data_ptr())) == 0
            print(f"TS N=32 MMA issue, {warps - 1:2d} background warps ({name:10s}): {int(cyc[0]) / (8 * R):6.1f} cyc/MMA")


# The microbenchmarks behind the kernels' tiling choices are reports, not
# tests (they only print cycle counts):  python tests/test_gpu_tc_probe.py
if __name__ == "__main__":
    lib = _perf_lib()
    for fn in (report_tcgen05_throughput, report_tcgen05_issue_rate, report_tcgen05_lean_issue,
               report_tcgen05_issue_under_contention):
        fn(lib)
