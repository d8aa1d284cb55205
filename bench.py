"""Benchmark: domain-decomposed 4-D FNO forward+backward on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 runs the BASELINE.json headline workload C2: 3-D Navier-Stokes FNO,
64x64x64 grid x 32 time steps, width 20 (in = hidden = out), 4 spectral
blocks, 8 modes per dim, batch 1, fp32 / complex64, GELU -- forward +
backward (upstream gradient g = y, loss 0.5||y||^2, as the reference's
``drive_scale``, d/bench.py:381-390).  Under torchrun with N > 1 ranks it
runs the C5 weak-scaling sweep: each GPU keeps a 64x64x64x32 x-slab of a
(64N)x64x64x32 global grid, ranks exchange the truncated spectra over NCCL
all-to-all (2 per block per direction).

``value`` is whole-job throughput in 64^3x32-cell sample equivalents per
second (= samples/s of the C2 problem at N = 1; N x (1 / step time) under
weak scaling), timed on device with CUDA events, max over ranks, inputs
resident in HBM (each activation is 671 MB, > the 126 MB L2, so no flush is
needed).  ``e2e`` is the same metric through the public API with the input
in pinned host memory: H2D copy + forward + loss read-back + backward.
``--impl reference`` times the reference's CPU algorithm (oracle port) on the
host cores; see oracle/cpu_baseline.py.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GRID1 = (64, 64, 64, 32)
CHANNELS = 20
MODES = (8, 8, 8, 8)
BLOCKS = 4
SEED = 42
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-train", action="store_true")
    p.add_argument("--sample-ranks", type=int, default=16, help="CPU sample: 1/R of the job per process")
    p.add_argument("--config", choices=["auto", "C3", "C4rank", "C5rank"], default="auto",
                   help="auto: C2 at N = 1, C5 weak scaling under torchrun; C3: 128^3x32 on one GPU; C4rank: the "
                        "CO2 grid 262x118x64x86 as 8 thread-ranks on one GPU (every launch has a P = 8 rank's "
                        "geometry); C5rank: the P = 8 weak-scaling problem as 8 thread-ranks on one GPU")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(world):
    grid = (GRID1[0] * world,) + GRID1[1:]
    name = ("C2 3-D Navier-Stokes FNO 64x64x64x32, width 20, 4 blocks, modes 8, batch 1, fwd+bwd"
            if world == 1 else
            f"C5 weak scaling: global {grid[0]}x64x64x32 (64x64x64x32 per GPU), width 20, 4 blocks, modes 8, "
            "batch 1, fwd+bwd, x-slab / ky-pencil decomposition, NCCL all-to-all")
    return grid, name


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


# ---------------------------------------------------------------------------
# algorithmic bytes, per launch, per rank
# ---------------------------------------------------------------------------


def alg_bytes(cfg, xl, kyl, nranks, groups=1):
    """Compulsory HBM bytes per launch of each timed tag;
    with G channel groups (pipelined repartitions, N > 1) the yzt and x-DFT
    launches each cover 1/G of the channels."""
    b, c, cin, cout = 1, cfg.hidden_channels, cfg.in_channels, cfg.out_channels
    ny, nz, nt = cfg.ny, cfg.nz, cfg.nt
    rx, ry, rz, rt = cfg.retained
    n_loc = xl * ny * nz * nt
    A = 4 * b * c * n_loc
    Ain, Aout = 4 * b * cin * n_loc, 4 * b * cout * n_loc
    T_xk = 8 * b * c * xl * ry * rz * rt
    T_kx = 8 * b * c * cfg.nx * kyl * rz * rt
    S = 8 * b * c * rx * kyl * rz * rt
    W = 8 * c * c * rx * kyl * rz * rt
    G = groups
    return {
        "mix_fwd.enc": Ain + A,
        "mix_fwd.dec": A + 2 * Aout,
        "yzt_fwd.fwd": (A + T_xk) / G,
        "yzt_fwd.bwd": (2 * A + T_xk) / G,
        "yzt_fwd.bwd_raw": (A + T_xk) / G,  # last block: act' fused into the decoder's mix_bwd
        "xspec_fwd": T_kx + W + S + T_kx,
        "xspec_bwd": T_kx + S + W + W + T_kx,
        "xdft.fwd": (T_kx + S) / G, "xidft.fwd": (S + T_kx) / G, "xmix_fwd": 2 * S + W,
        "xdft.bwd": (T_kx + S) / G, "xidft.bwd": (S + T_kx) / G, "xmix_bwd": 3 * S + 2 * W,
        "yzt_inv.fwd": (T_xk + A) / G,
        "yzt_inv.bwd": (T_xk + A) / G,
        "mix_bwd.dec": 2 * Aout + A + A,
        "mix_bwd.enc": 2 * A + Ain + Ain,
        "reduce.dec": 0,
        "reduce.enc": 0,
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def _reader(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line))

    def start(self):
        """Start nvidia-smi (20 ms period) and return once it is producing
        samples, so the timed region that follows is covered."""
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        threading.Thread(target=self._reader, daemon=True).start()
        deadline = time.monotonic() + 10.0
        while not self.lines and time.monotonic() < deadline:
            time.sleep(0.01)

    def mark(self):
        """Call right before the timed region starts."""
        self.t0 = time.monotonic()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.t1 = time.monotonic()
        time.sleep(0.05)  # the sample in flight at the end of the region
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        t0 = self.t0 if self.t0 is not None else 0.0
        window = [ln for t, ln in self.lines if t0 - 0.025 <= t <= self.t1 + 0.025]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in window:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "period_ms": 20}


class KernelTimer:
    """CUDA-event pairs around every libdfno launch (current stream)."""

    def __init__(self):
        import threading

        import torch

        self.torch = torch
        self.events = {}
        self.launches = 0
        self.enabled = True
        self.lock = threading.Lock()  # thread-ranks share the stream: keep each event pair tight

    def __call__(self, name, fn):
        if not self.enabled:
            fn()
            return
        t = self.torch.cuda
        s, e = t.Event(enable_timing=True), t.Event(enable_timing=True)
        with self.lock:
            s.record()
            fn()
            e.record()
            self.events.setdefault(name, []).append((s, e))
            self.launches += 1

    def summary(self):
        out = {}
        for name, evs in self.events.items():
            ms = [s.elapsed_time(e) for s, e in evs]
            out[name] = (len(ms), sum(ms))
        return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2211_12709_b200 as P
    from paper_2211_12709_b200 import fno as F

    world, rank, local = dist_env()
    # DFNO_BENCH_SHARE_GPU=1 with DFNO_BENCH_BACKEND=gloo runs every rank on cuda:0 -- a one-GPU
    # check of the multi-process path (process groups, uneven all-to-all splits); not a timing mode
    share = os.environ.get("DFNO_BENCH_SHARE_GPU") == "1"
    backend = os.environ.get("DFNO_BENCH_BACKEND", "nccl")
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        comm = P.Communicator.from_process_group(device=dev)
    else:
        comm = P.run_ranks(1, lambda c: c)[0]
    grid, wname = workload(world)
    cfg = P.FnoConfig(*grid, CHANNELS, CHANNELS, CHANNELS, P.ModeSpec.of_xyzt(*MODES), BLOCKS, "gelu", "real32",
                      world)
    xl = cfg.x_partition().extent_of(rank)
    kyl = cfg.ky_partition().extent_of(rank)
    # weights: the reference's init (numpy PCG64 stream, d/fno.py:155-180), this rank's ky shard
    params = P.shard_params(P.init_params(cfg, SEED, device=dev), cfg, rank)
    torch.manual_seed(SEED + rank)
    x = P.DenseTensor(P.DATA_LABELS, torch.randn((1, CHANNELS, xl) + grid[1:], device=dev))

    def step(xin):
        cache = P.ForwardCache()
        y = P.fno_forward(comm, xin, params, cfg, cache)
        gx, grads = P.fno_backward(comm, y, params, cfg, cache)
        return y, gx, grads

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(x)
    barrier()
    # single rank: the step is one CUDA graph (P.FwdBwdGraph -- the same
    # kernels and buffers, captured after an eager warm-up); the eager loop
    # below times the same step launch by launch for the kernel table
    graph = P.FwdBwdGraph(comm, x, params, cfg) if world == 1 else None
    ms_graph = ms_fwd = None
    if graph is not None:
        for _ in range(max(1, args.warmup)):
            graph.replay()
        barrier()
        clocks_g = ClockSampler(local)
        clocks_g.start()
        clocks_g.mark()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(args.steps):
            graph.replay()
        g1.record()
        barrier()
        clock_info_g = clocks_g.stop()
        ms_graph = g0.elapsed_time(g1) / args.steps
        # forward alone (the reference scale driver's efficiency column, d/cli.py:171-178)
        fgraph = P.FwdBwdGraph(comm, x, params, cfg, backward=False)
        for _ in range(max(1, args.warmup)):
            fgraph.replay()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            fgraph.replay()
        f1.record()
        barrier()
        ms_fwd = f0.elapsed_time(f1) / args.steps
        del fgraph
    else:
        # several ranks: eager steps (NCCL exchanges on the comm stream), timed
        # without per-launch events; the instrumented pass below gives the table
        clocks_g = ClockSampler(local)
        clocks_g.start()
        barrier()
        clocks_g.mark()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(args.steps):
            step(x)
        g1.record()
        barrier()
        clock_info_g = clocks_g.stop()
        ms_graph = g0.elapsed_time(g1) / args.steps
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            P.fno_forward(comm, x, params, cfg)
        f1.record()
        barrier()
        ms_fwd = f0.elapsed_time(f1) / args.steps
        if world > 1:
            tt = torch.tensor([ms_fwd], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms_fwd = float(tt.item())

    timer = KernelTimer()
    F.set_kernel_timer(timer)
    # all-to-all (x <-> ky repartition) time and off-rank bytes, N > 1
    a2a = {"events": [], "bytes": 0}
    if world > 1:
        orig_exchange = comm.exchange

        def timed_exchange(send, recv, send_counts, recv_counts, label="", record=True):
            # events on the current stream: the comm stream of the pipelined exchanges
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            n = orig_exchange(send, recv, send_counts, recv_counts, label, record)
            e.record()
            a2a["events"].append((s, e))
            a2a["bytes"] += sum(n for p, n in enumerate(send_counts) if p != rank) * send.element_size()
            return n

        comm.exchange = timed_exchange
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    clocks.mark()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        step(x)
    t1.record()
    barrier()
    clock_info = clocks.stop()
    F.set_kernel_timer(None)
    a2a_info = None
    if world > 1:
        comm.exchange = orig_exchange
        a2a_ms = sum(s_.elapsed_time(e_) for s_, e_ in a2a["events"]) / args.steps
        a2a_bytes = a2a["bytes"] / args.steps
        a2a_info = {"exchanges_per_step": len(a2a["events"]) / args.steps, "ms_per_step": round(a2a_ms, 4),
                    "off_rank_bytes_per_step": int(a2a_bytes),
                    "GBps_per_direction": round(a2a_bytes / (a2a_ms * 1e-3) / 1e9, 1) if a2a_ms > 0 else None,
                    "nvlink_peak_GBps_per_direction": 900.0, "rank": rank}
    ms = t0.elapsed_time(t1) / args.steps
    ms_eager = ms
    if ms_graph is not None:
        ms, clock_info = ms_graph, clock_info_g
    ms_max = ms
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_max = float(tt.item())
    launches_per_step = timer.launches / args.steps
    ksum = timer.summary()

    # ---- training step: forward, global MSE, backward, Adam,
    #      replication check -- the reference's train_step (d/training.py:96-133)
    train = None
    if not args.no_train:
        from paper_2211_12709_b200 import training as T

        tgt = P.DenseTensor(P.DATA_LABELS, torch.zeros((1, CHANNELS, xl) + grid[1:], device=dev))
        st = T.AdamState()
        tp = params
        for _ in range(2):
            tp, _ = T.train_step(comm, x, tgt, tp, st, 1e-4, cfg)
        barrier()
        ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nt = max(2, min(args.steps, 5))
        ta.record()
        for _ in range(nt):
            tp, tloss = T.train_step(comm, x, tgt, tp, st, 1e-4, cfg)
        tb.record()
        barrier()
        tms = ta.elapsed_time(tb) / nt
        if world > 1:
            tt = torch.tensor([tms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tms = float(tt.item())
        train = {"metric": "train_step samples/s (fwd + MSE + bwd + Adam + replication check)",
                 "value": round(world * 1e3 / tms, 3), "unit": "samples/s", "ms_per_step": round(tms, 4),
                 "steps": nt, "loss": tloss}
        del tp, st

    # ---- e2e through the public API with host-resident input
    e2e = None
    if not args.no_e2e:
        host = torch.empty((1, CHANNELS, xl) + grid[1:], dtype=torch.float32, pin_memory=True)
        host.copy_(x.data.cpu())
        xh = P.DenseTensor(P.DATA_LABELS, host)
        # public API step loop: pinned host input staged to HBM on a copy
        # stream (P.InputStager), step k+1's H2D overlapping step k's compute;
        # every step's H2D and its loss read-back are inside the timed region
        stager = P.InputStager(host.shape, torch.float32, dev)

        def e2e_loop(n):
            loss = None
            stager.put(xh)
            for k in range(n):
                xin = stager.get()
                if k + 1 < n:
                    stager.put(xh)
                cache = P.ForwardCache()
                y = P.fno_forward(comm, xin, params, cfg, cache)
                loss = 0.5 * float(torch.linalg.vector_norm(y.data, dtype=torch.float64).item()) ** 2  # D2H
                P.fno_backward(comm, y, params, cfg, cache)
            return loss

        e2e_loop(2)
        barrier()
        h2d0 = stager.h2d_bytes
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record()
        loss = e2e_loop(args.steps)
        stager.synchronize()
        e1.record()
        barrier()
        wall = (time.perf_counter() - w0) / args.steps * 1e3
        ems = e0.elapsed_time(e1) / args.steps
        if world > 1:
            tt = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": round(world * 1e3 / ems, 3), "unit": "samples/s", "h2d_bytes_per_step": (stager.h2d_bytes - h2d0) // args.steps,
               "d2h_bytes_per_step": 8, "ms_per_step": round(ems, 4), "wall_ms_per_step": round(wall, 4),
               "loss": loss, "h2d_path": "pinned host -> HBM on a copy stream, step k+1 staged during step k "
                                         "(P.InputStager); loss = 0.5||y||^2 read back every step"}

    # ---- roofline of the dominant kernel
    hbm, hbm_kind = peaks()
    traffic_tbl, traffic_src = {}, None
    tf = sorted((ROOT / "profiles").glob("*_traffic.json"))
    if tf:
        tj = json.loads(tf[-1].read_text())
        traffic_tbl, traffic_src = tj.get("bytes_per_launch", {}), f"{tf[-1].name}: {tj.get('source', '')}"
    ab = alg_bytes(cfg, xl, kyl, world, max(1, len(F._plan(cfg, comm, 1).groups)))
    dom = max(ksum.items(), key=lambda kv: kv[1][1])
    dname, (dn, dms) = dom
    davg = dms / dn
    achieved = ab[dname] / (davg * 1e-3) / 1e9
    step_bytes = sum(ab[k] * n / args.steps for k, (n, _) in ksum.items())
    kernels = {k: {"launches_per_step": n / args.steps, "avg_ms": round(t / n, 5),
                   "share": round(t / sum(v[1] for v in ksum.values()), 4),
                   "alg_GBps": round(ab[k] / (t / n * 1e-3) / 1e9, 1) if ab[k] else None}
               for k, (n, t) in sorted(ksum.items(), key=lambda kv: -kv[1][1])}
    result = {
        "metric": "FNO fwd+bwd samples/s (64^3x32-cell sample equivalents, whole job)",
        "value": round(world * 1e3 / ms_max, 3),
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max, 4),
        "fwd_only": ({"value": round(world * 1e3 / ms_fwd, 3), "unit": "samples/s", "ms_per_step": round(ms_fwd, 4)}
                     if ms_fwd else None),
        "step_mode": ("one CUDA graph per step (P.FwdBwdGraph); eager launch-by-launch step "
                      f"{ms_eager:.4f} ms, which also gives the kernel table") if graph is not None else (
                      f"eager steps without per-launch events; the instrumented pass ({ms_eager:.4f} ms) gives "
                      "the kernel table"),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic: x ~ N(0,1) per rank, weights = reference init_params(seed 42) ky shard, g = y",
        "config": {"workload": wname, "grid": list(grid), "channels": CHANNELS, "modes": list(MODES),
                   "blocks": BLOCKS, "batch": 1, "parallelism": f"dd{world} (x-slab / ky-pencil)",
                   "l2": "inputs larger than L2 (671 MB activations > 126 MB L2); no flush"},
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1), "peak": hbm,
                     "peak_kind": f"{hbm_kind} (MEASURED_PEAKS.json hbm_gbs)" if hbm_kind == "measured" else
                     "fallback (B200_PROFILING.md)",
                     "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "alg_bytes_per_launch": ab[dname], "avg_launch_ms": round(davg, 5),
                     "traffic": traffic_tbl.get(dname), "traffic_source": traffic_src},
        "step_roofline": {"alg_bytes_per_step_per_gpu": int(step_bytes),
                          "achieved_GBps": round(step_bytes / (ms_max * 1e-3) / 1e9, 1),
                          "frac": round(step_bytes / (ms_max * 1e-3) / 1e9 / hbm, 4)},
        "kernels": kernels,
        "gpu_launches": int(round(timer.launches)),
        "gpu_launches_per_step": launches_per_step,
        "all_to_all": a2a_info,
        "clocks": clock_info,
        "e2e": e2e,
        "train_step": train,
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cfg.grid, args.sample_ranks * world, steps=1)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


SINGLE_GPU_CONFIGS = {
    # name: (grid, thread-ranks, workload)
    "C3": ((128, 128, 128, 32), 1, "C3 3-D Navier-Stokes FNO 128x128x128x32, width 20, 4 blocks, modes 8, batch 1, "
                                   "fwd+bwd, one B200"),
    "C4rank": ((262, 118, 64, 86), 8, "C4 CO2 FNO 262x118x64x86 (1.98 M cells x 86 steps), width 20, 4 blocks, "
                                      "modes 8, batch 1, fwd+bwd, as 8 thread-ranks on one B200 (x slabs 33x6 + "
                                      "32x2, ky pencils of 2)"),
    "C5rank": ((512, 64, 64, 32), 8, "C5 weak scaling at P = 8: global 512x64x64x32 (one 64x64x64x32 slab per "
                                     "rank), width 20, 4 blocks, modes 8, batch 1, fwd+bwd, as 8 thread-ranks on one "
                                     "B200 (ky pencils of 2, x-DFT over 512)"),
}


def run_single_gpu_config(args):
    """C3 / C4rank: the north-star grids on one GPU.  C4rank runs the P = 8
    decomposition as thread-ranks sharing the GPU (ThreadWorld), so every
    kernel launch has exactly one P = 8 rank's geometry; ``value`` is samples/s
    of the whole C4 problem on one GPU and each kernel's roofline is per launch."""
    import threading

    import torch

    import paper_2211_12709_b200 as P
    from paper_2211_12709_b200 import fno as F

    grid, ranks, wname = SINGLE_GPU_CONFIGS[args.config]
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    cfg = P.FnoConfig(*grid, CHANNELS, CHANNELS, CHANNELS, P.ModeSpec.of_xyzt(*MODES), BLOCKS, "gelu", "real32",
                      ranks)
    full = P.init_params(cfg, SEED, device=dev)
    torch.manual_seed(SEED)
    xpart = cfg.x_partition()
    timer = KernelTimer()
    clocks = ClockSampler(0)
    times = {}
    lock = threading.Lock()

    def body(comm):
        r = comm.rank
        params = P.shard_params(full, cfg, r)
        x = P.DenseTensor(P.DATA_LABELS, torch.randn((1, CHANNELS, xpart.extent_of(r)) + grid[1:], device=dev))

        def step():
            cache = P.ForwardCache()
            y = P.fno_forward(comm, x, params, cfg, cache)
            P.fno_backward(comm, y, params, cfg, cache)

        for _ in range(args.warmup):
            step()
        comm.barrier()
        if r == 0:
            torch.cuda.synchronize()
            F.set_kernel_timer(timer)
            clocks.start()
            clocks.mark()
            times["t0"] = torch.cuda.Event(enable_timing=True)
            times["t0"].record()
        comm.barrier()
        for _ in range(args.steps):
            step()
        comm.barrier()
        if r == 0:
            times["t1"] = torch.cuda.Event(enable_timing=True)
            times["t1"].record()
            torch.cuda.synchronize()
            F.set_kernel_timer(None)
        comm.barrier()
        with lock:
            times.setdefault("xl", {})[r] = (xpart.extent_of(r), cfg.ky_partition().extent_of(r))

    P.run_ranks(ranks, body)
    clock_info = clocks.stop()
    ms = times["t0"].elapsed_time(times["t1"]) / args.steps
    ksum = timer.summary()
    hbm, hbm_kind = peaks()
    # per-launch algorithmic bytes: launches alternate over ranks; use the
    # busiest rank's geometry (x_r = 33 / ky_r = 2 at C4, every rank at C3)
    xl = max(v[0] for v in times["xl"].values())
    kyl = max(v[1] for v in times["xl"].values())
    G = min(F.PIPELINE_GROUPS_THREADED, CHANNELS) if ranks > 1 else 1  # channel groups (thread ranks)
    ab = alg_bytes(cfg, xl, kyl, ranks, G)
    # mean per-launch bytes over ranks (uneven x slabs)
    ab_mean = {k: sum(alg_bytes(cfg, v[0], v[1], ranks, G)[k] for v in times["xl"].values()) / ranks for k in ab}
    kernels = {k: {"launches_per_step": n / args.steps, "avg_ms": round(t / n, 5),
                   "share": round(t / sum(v[1] for v in ksum.values()), 4),
                   "alg_GBps": round(ab_mean[k] / (t / n * 1e-3) / 1e9, 1) if ab_mean[k] else None,
                   "roofline_frac": round(ab_mean[k] / (t / n * 1e-3) / 1e9 / hbm, 4) if ab_mean[k] else None}
               for k, (n, t) in sorted(ksum.items(), key=lambda kv: -kv[1][1])}
    dname, (dn, dms) = max(ksum.items(), key=lambda kv: kv[1][1])
    achieved = ab_mean[dname] / (dms / dn * 1e-3) / 1e9
    step_bytes = sum(ab_mean[k] * n / args.steps for k, (n, _) in ksum.items())
    result = {
        "metric": f"FNO fwd+bwd samples/s ({args.config} problem, whole job on one GPU)",
        "value": round(1e3 / ms, 4), "unit": "samples/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "none", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic: x ~ N(0,1), weights = reference init_params(seed 42), g = y",
        "config": {"workload": wname, "grid": list(grid), "channels": CHANNELS, "modes": list(MODES),
                   "blocks": BLOCKS, "batch": 1, "thread_ranks": ranks,
                   "l2": "activations larger than L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1), "peak": hbm,
                     "peak_kind": hbm_kind, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "alg_bytes_per_launch": int(ab_mean[dname]), "avg_launch_ms": round(dms / dn, 5),
                     "traffic": None},
        "step_roofline": {"alg_bytes_per_step": int(step_bytes),
                          "achieved_GBps": round(step_bytes / (ms * 1e-3) / 1e9, 1),
                          "frac": round(step_bytes / (ms * 1e-3) / 1e9 / hbm, 4)},
        "kernels": kernels, "gpu_launches": int(timer.launches), "clocks": clock_info,
    }
    print(json.dumps(result), flush=True)


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


CALIBRATION = ("the real reference (distfno scale --transport proc, P = 8, C1) is 1.69x slower than this port on "
               "the same cores (profiles/r02_reference_calibration_32x32x32x16_P8.json), so this value overstates "
               "the reference's throughput")


def cpu_baseline(grid, ranks, steps):
    from oracle import cpu_baseline as cb

    cores = min(os.cpu_count() or 1, ranks)
    per_rank, job = cb.measure(grid, CHANNELS, MODES, BLOCKS, ranks, cores, steps=steps)
    t = statistics.median(job)
    units = grid[0] / GRID1[0]
    return {"value": round(units / t, 6), "unit": "samples/s", "cores": cores, "kind": "port",
            "sample": (f"one rank's fwd+bwd of a {ranks}-way x decomposition of the {grid} grid (reference's staged "
                       f"numpy pipeline, oracle/cpu_baseline.py), {cores} processes in parallel, 1 thread each; "
                       f"rank time {statistics.median(per_rank):.2f} s, job time = rank time x {ranks}/{cores}"),
            "job_seconds_per_sample": round(t / units, 3), "cpu_model": cpu_model(), "calibration": CALIBRATION}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import cpu_baseline as cb

    grid, wname = workload(world)
    ranks = args.sample_ranks * world
    cores = min(os.cpu_count() or 1, ranks)
    if args.warmup:
        cb.measure(grid, CHANNELS, MODES, BLOCKS, ranks, cores, steps=args.warmup)
    per_rank, job = cb.measure(grid, CHANNELS, MODES, BLOCKS, ranks, cores, steps=args.steps)
    t = statistics.median(job)
    value = world / t
    out = {
        "impl": "reference",
        "metric": "FNO fwd+bwd samples/s (64^3x32-cell sample equivalents, whole job)",
        "value": round(value, 6), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wname, "grid": list(grid), "channels": CHANNELS, "modes": list(MODES),
                   "blocks": BLOCKS, "batch": 1, "parallelism": f"cpu {cores} processes"},
        "cpu_baseline": {"value": round(value, 6), "unit": "samples/s", "cores": cores, "kind": "port",
                         "sample": f"per step: one rank's fwd+bwd of a {ranks}-way decomposition x {ranks}/{cores}",
                         "cpu_model": cpu_model(), "calibration": CALIBRATION},
        "e2e": {"value": round(value, 6), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.config != "auto":
        run_single_gpu_config(a)
    else:
        run_ours(a)
