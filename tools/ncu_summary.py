"""Summarise an ncu --set full report: per kernel duration, DRAM bytes and
throughput, issue activity, tensor-pipe use, stall reasons and the hottest
SASS lines.  Usage: python tools/ncu_summary.py report.ncu-rep [top_lines]"""

import csv
import io
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


SCALE = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1.0, "byte": 1.0,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw_metrics(rep):
    """Rows of the raw page with durations in ns and byte counts in bytes (the
    second CSV row holds each metric's unit, which ncu picks per value)."""
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for k, u, v in zip(hdr, units, r):
            if u in SCALE:
                try:
                    v = str(float(v.replace(",", "")) * SCALE[u])
                except ValueError:
                    pass
            d[k] = v
        out.append(d)
    return out


def f(d, k):
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


def main(rep, top=12):
    for d in raw_metrics(rep):
        name = d.get("Kernel Name", "?")[:90]
        dur = f(d, "gpu__time_duration.sum")
        rd, wr = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
        print(f"== {name}")
        print(f"   duration {dur/1e3:.1f} us | dram read {rd/1e6:.1f} MB write {wr/1e6:.1f} MB "
              f"-> {(rd + wr) / dur:.0f} GB/s | dram% {f(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}")
        print(f"   issue active {f(d, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}% | "
              f"warps active {f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}% | "
              f"regs {f(d, 'launch__registers_per_thread'):.0f} | "
              f"tensor(tcgen05) {f(d, 'sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active'):.1f}% "
              f"| tmem-pipe {f(d, 'sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active'):.1f}%")
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), f(d, k)) for k in d
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        tot = sum(v for _, v in st if v == v) or 1
        st.sort(key=lambda kv: -kv[1])
        print("   stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
