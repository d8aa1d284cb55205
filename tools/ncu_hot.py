"""Hottest SASS lines (warp-stall samples) of an ncu --page source --csv dump
(gzip or plain).  Usage: python tools/ncu_hot.py file.source.csv[.gz] [top] [context]"""
import csv
import gzip
import io
import sys


def main(path, top=25, ctx=0):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(io.TextIOWrapper(op(path, "rb"), "utf-8")))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    col = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[col] or 0) for r in data) or 1.0
    order = sorted(range(len(data)), key=lambda i: -float(data[i][col] or 0))[:top]
    for i in sorted(order) if ctx else order:
        lo, hi = max(0, i - ctx), min(len(data), i + ctx + 1)
        for j in range(lo, hi):
            r = data[j]
            mark = ">" if j == i else " "
            print(f"{mark}{100 * float(r[col] or 0) / tot:5.1f}%  {r[1].strip()[:100]}")
        if ctx:
            print("   ...")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
