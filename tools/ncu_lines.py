"""Map an `ncu --page source --csv` (SASS view) dump back to CUDA source
lines using the line table of the local build (nvdisasm -g on the cubin
extracted from lib/libdfno.so).  Prints per-source-line executed
warp-instructions and stall samples for one kernel.
Usage: python tools/ncu_lines.py source.csv[.gz] mangled_kernel_name [top]"""
import collections
import gzip
import io
import os
import re
import subprocess
import sys
import tempfile
import csv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2211_12709_b200", "lib", "libdfno.so")


def line_table(mangled):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, capture_output=True)
    for f in os.listdir(d):
        out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, f)], capture_output=True, text=True).stdout
        start = out.find(f".text.{mangled}:")
        if start < 0:
            continue
        end = out.find("//---------------------", start)
        body = out[start:end if end > 0 else None]
        table, cur = {}, None
        for ln in body.splitlines():
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and cur:
                table[int(m.group(1), 16)] = cur
        return table
    raise SystemExit(f"{mangled} not found in {LIB}")


def main(path, mangled, top=30):
    table = line_table(mangled)
    op = gzip.open if path.endswith(".gz") else open
    text = io.TextIOWrapper(op(path, "rb"), "utf-8").read()
    rows, cur = None, None
    demangled_hint = mangled
    sections = []
    for row in csv.reader(io.StringIO(text)):
        if row and row[0] == "Kernel Name":
            cur = [row[1]]
            sections.append(cur)
        elif cur is not None:
            cur.append(row)
    # pick the section whose SASS length matches the line table best
    best = None
    for sec in sections:
        n = len(sec) - 2
        if best is None or abs(n - len(table)) < abs(len(best) - 2 - len(table)):
            best = sec
    hdr = best[1]
    ia, ie, st = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(best[2][ia], 16)
    inst, stall = collections.Counter(), collections.Counter()
    for r in best[2:]:
        try:
            off = int(r[ia], 16) - base
        except ValueError:
            continue
        key = table.get(off, "?")
        inst[key] += int(r[ie] or 0)
        stall[key] += int(r[st] or 0)
    tot_i, tot_s = sum(inst.values()) or 1, sum(stall.values()) or 1
    print(f"== {best[0][:100]}  ({tot_i:,} warp-inst, {tot_s:,} stall samples)")
    print("   by stall samples:")
    for k, v in stall.most_common(top):
        print(f"   {k:28s} stall {100 * v / tot_s:5.1f}%   inst {100 * inst[k] / tot_i:5.1f}%")
    print("   by instructions:")
    for k, v in inst.most_common(top // 2):
        print(f"   {k:28s} inst {100 * v / tot_i:5.1f}%   stall {100 * stall[k] / tot_s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
