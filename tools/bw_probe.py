"""Write-only / read-only / copy HBM bandwidth on this GPU (torch kernels,
CUDA events, best of 20) for the roofline of write- or read-dominated kernels."""
import torch

n = 671088640 // 4
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
a.normal_()


def best(fn, bytes_):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    t = min(ts) * 1e-3
    return round(bytes_ / t / 1e9, 1), round(t * 1e6, 1)


print("write (fill_) GB/s, us:", best(lambda: b.fill_(1.0), n * 4))
print("read (sum) GB/s, us:", best(lambda: a.sum(), n * 4))
print("copy GB/s, us:", best(lambda: b.copy_(a), 2 * n * 4))
