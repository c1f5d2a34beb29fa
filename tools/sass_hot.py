"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv` dump
(SASS view), with +-N instructions of context.   python tools/sass_hot.py src.csv [top] [ctx]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr)]
si, ni, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
tot = sum(int(r[si] or 0) for r in body)
print("total samples", tot, "instructions", len(body))
order = sorted(range(len(body)), key=lambda i: -int(body[i][si] or 0))[:top]
for i in sorted(order) if ctx else order:
    for j in range(max(0, i - ctx), min(len(body), i + ctx + 1)):
        r = body[j]
        mark = ">>" if j == i else "  "
        print(f"{mark}{j:5d} {int(r[si] or 0):6d} {100*int(r[si] or 0)/tot:5.1f}% ex={r[ei]:>8s} {r[ni].strip()[:90]}")
    if ctx:
        print("--")
