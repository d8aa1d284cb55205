"""Assemble the judged evidence under profiles/ from a tools/gpu_profile_round.sh
run (gpurun_out/): bench lines, the ncu launch list of the bench, per-kernel
ncu --set full summaries, and the per-launch DRAM traffic table bench.py reads
for roofline.traffic.  Usage: python tools/make_profiles.py <tag>"""
import collections
import csv
import gzip
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G = ROOT / "gpurun_out"
P = ROOT / "profiles"

# ncu capture name -> bench.py kernel tag(s) it measures
CAPTURES = {
    "yzt_fwd_act": ["yzt_fwd.fwd"], "yzt_fwd_grad": ["yzt_fwd.bwd"], "yzt_inv": ["yzt_inv.fwd", "yzt_inv.bwd"],
    "mix_bwd": ["mix_bwd.dec", "mix_bwd.enc"], "mix_fwd": ["mix_fwd.enc"], "xmix": [], "xmix_bwd": [], "xdft": [],
    "xidft": [],
    # round-2 capture names (tools/gpu_r02_evidence.sh)
    "fwd_c2": ["yzt_fwd.fwd"], "inv_c2": ["yzt_inv.fwd", "yzt_inv.bwd"], "mixbwd_c2": ["mix_bwd.dec", "mix_bwd.enc"],
    "xdft_c2": [], "xidft_c2": [],
}


def raw_rows(path):
    rows = list(csv.reader(io.TextIOWrapper(gzip.open(path), "utf-8")))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def num(d, k):
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main(tag):
    P.mkdir(exist_ok=True)
    for f, out in (("bench.json", f"{tag}_bench.json"), ("bench_ref.json", f"{tag}_bench_reference.json"),
                   ("pytest_gpu.log", f"{tag}_pytest_gpu.log")):
        if (G / f).exists():
            shutil.copy(G / f, P / out)
    # launch list
    lc = G / "launches.csv"
    if lc.exists():
        rows = [r for r in csv.reader(open(lc)) if len(r) > 10]
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        d = collections.defaultdict(list)
        for r in rows[1:]:
            d[r[ki][:100]].append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in d.values())
        with open(P / f"{tag}_launches.txt", "w") as fh:
            fh.write("ncu --metrics gpu__time_duration.sum --clock-control none -c 400  python bench.py --steps 2 "
                     "--warmup 1 --no-cpu-baseline --no-e2e  (every launch of the command: 3 fwd+bwd steps plus the train-step measurement; cold, serialised)\n")
            fh.write(f"{'n':>4} {'avg_us':>9} {'total_ms':>9} {'share':>6} kernel\n")
            for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
                fh.write(f"{len(v):4d} {sum(v) / len(v) / 1e3:9.1f} {sum(v) / 1e6:9.3f} {sum(v) / tot:6.3f} {k}\n")
    # per-kernel full captures
    traffic = {}
    lines = [f"ncu --set full --clock-control none (one launch each, C2 geometry 64^3 x 32, c = 20, m = 8; "
             "tools/ncu_one.sh via tools/time_kernel.py)\n"]
    for name, tags in CAPTURES.items():
        raw = G / "ncu" / f"{name}.raw.csv.gz"
        if not raw.exists():
            continue
        rows = list(csv.reader(io.TextIOWrapper(gzip.open(raw), "utf-8")))
        hdr, units = rows[0], rows[1]
        u = dict(zip(hdr, units))
        for r in rows[2:3]:
            d = dict(zip(hdr, r))
            rd = num(d, "dram__bytes_read.sum") * unit_scale(u.get("dram__bytes_read.sum", "byte"))
            wr = num(d, "dram__bytes_write.sum") * unit_scale(u.get("dram__bytes_write.sum", "byte"))
            dur = num(d, "gpu__time_duration.sum") * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(
                u.get("gpu__time_duration.sum", "ns"), 1e-9)
            st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), num(d, k)) for k in hdr
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
            tot = sum(v for _, v in st if v == v) or 1
            st.sort(key=lambda kv: -kv[1])
            lines.append(
                f"== {name}: {d.get('Kernel Name', '?')[:110]}\n"
                f"   duration {dur * 1e6:.1f} us | DRAM read {rd / 1e6:.1f} MB write {wr / 1e6:.1f} MB -> "
                f"{(rd + wr) / dur / 1e9:.0f} GB/s | dram% {num(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}"
                f" | issue active {num(d, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}% | regs "
                f"{num(d, 'launch__registers_per_thread'):.0f} | tensor pipe active "
                f"{num(d, 'TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed'):.1f}%"
                f" | TMEM active {num(d, 'sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%\n"
                "   stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in st[:6]) + "\n")
            for t in tags:
                traffic[t] = int(rd + wr)
    (P / f"{tag}_ncu_kernels.txt").write_text("".join(lines))
    if traffic:
        (P / f"{tag}_traffic.json").write_text(json.dumps(
            {"source": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch (C2)",
             "bytes_per_launch": traffic}, indent=1))
    print("\n".join(sorted(p.name for p in P.iterdir())))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
