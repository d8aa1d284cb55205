"""Pinned host -> HBM bandwidth for one 671 MB input, as one copy or split over
several copy streams (the e2e leg of bench.py is bound by this copy)."""
import torch

n = 1 * 20 * 64 * 64 * 64 * 32
host = torch.empty(n, dtype=torch.float32, pin_memory=True)
host.fill_(1.0)
dev = torch.empty(n, dtype=torch.float32, device="cuda")
for parts in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k, s in enumerate(streams):
            s.wait_event(e0)
            lo, hi = n * k // parts, n * (k + 1) // parts
            with torch.cuda.stream(s):
                dev[lo:hi].copy_(host[lo:hi], non_blocking=True)
        for s in streams:
            e1.wait_stream(s) if False else torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{parts} stream(s): {ms:.2f} ms  {4 * n / ms / 1e6:.1f} GB/s")
