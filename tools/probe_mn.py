"""Which (LBO, SBO) roles does an MN-major SWIZZLE_NONE tf32 A operand use?
Runs tests/probes/probe_tc.cu:probe_run_mn with the layout element (r, k) at
(r/4)*SBO + (k/8)*LBO + (k%8)*16 + (r%4)*4 and reports the error."""
import ctypes, subprocess, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "tests" / "probes" / "libprobe.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler", "-fPIC",
                "-shared", f"-I{ROOT / 'paper_2211_12709_b200' / 'csrc'}", f"-I{ROOT / 'include'}",
                str(ROOT / "tests" / "probes" / "probe_tc.cu"), "-o", str(SO)], check=True)
lib = ctypes.CDLL(str(SO))
def trunc(x):
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)
# control: the K-major probe on the same harness
rng = np.random.default_rng(0)
A = rng.standard_normal((128, 32)).astype(np.float32); B = rng.standard_normal((32, 32)).astype(np.float32)
a, b = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda"); d = torch.zeros((128, 32), device="cuda")
lib.probe_run(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(d.data_ptr()), 128, 32, 32,
              144, 1152, 128, 1024, 0, 0)
print("K-major control err", np.max(np.abs(d.cpu().numpy() - trunc(A) @ trunc(B).T)) / np.max(np.abs(trunc(A) @ trunc(B).T)))
for (M, N, K, lbo, sbo, sw) in [(128, 32, 32, 4096, 128, 0), (128, 32, 8, 128, 4096, 0), (128, 32, 32, 1024, 4096, 1),
                                (128, 32, 32, 4096, 1024, 1), (128, 32, 8, 1024, 4096, 1), (128, 32, 32, 1024, 4096, 2), (128, 32, 32, 512, 2048, 3), (128, 32, 32, 4096, 512, 3), (128, 32, 8, 512, 2048, 3)]:
    rng = np.random.default_rng(0)
    A = rng.standard_normal((M, K)).astype(np.float32); B = rng.standard_normal((N, K)).astype(np.float32)
    a, b = torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda")
    d = torch.zeros((M, N), device="cuda")
    rc = lib.probe_run_mn(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(d.data_ptr()),
                          M, N, K, lbo, sbo, 128, (K // 4) * 128, sw)
    want = trunc(A) @ trunc(B).T
    got = d.cpu().numpy().astype(np.float64)
    print(f"M{M} N{N} K{K} sw {sw} lbo {lbo} sbo {sbo}: rc {rc} err {np.max(np.abs(got - want)) / np.max(np.abs(want)):.3e} "
          f"zeros {np.mean(got == 0):.2f}")
