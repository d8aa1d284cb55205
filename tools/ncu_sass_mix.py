"""Instruction mix of one kernel from an `ncu --page source --csv` dump
(SASS view): executed warp-instructions per opcode and the top stall lines.
Usage: python tools/ncu_sass_mix.py source.csv[.gz] kernel_substring [top]"""
import collections
import csv
import gzip
import io
import sys


def sections(path):
    op = gzip.open if path.endswith(".gz") else open
    text = io.TextIOWrapper(op(path, "rb"), "utf-8").read()
    cur, rows = None, []
    for row in csv.reader(io.StringIO(text)):
        if row and row[0] == "Kernel Name":
            if cur:
                yield cur, rows
            cur, rows = row[1], []
        elif cur is not None:
            rows.append(row)
    if cur:
        yield cur, rows


def main(path, sub, top=25):
    for name, rows in sections(path):
        if sub not in name:
            continue
        hdr = rows[0]
        ie = hdr.index("Instructions Executed")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        src = hdr.index("Source")
        ops = collections.Counter()
        stalls = []
        total = 0
        for r in rows[1:]:
            try:
                n = int(r[ie])
            except (ValueError, IndexError):
                continue
            opc = r[src].strip().split()
            if not opc:
                continue
            o = opc[0] if not opc[0].startswith("@") else opc[1]
            ops[o.split(".")[0]] += n
            total += n
            stalls.append((int(r[st] or 0), r[src].strip()[:90]))
        print(f"== {name[:100]}\n   total warp-instructions {total:,}")
        for o, n in ops.most_common(top):
            print(f"   {o:12s} {n:14,d} {100 * n / total:5.1f}%")
        stalls.sort(reverse=True)
        print("   top stall lines:")
        for s, l in stalls[:12]:
            print(f"   {s:7d}  {l}")
        break


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
