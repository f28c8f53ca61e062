"""Stall-reason totals and the hottest SASS lines from `ncu --page source --csv --print-source sass`.

    python tools/sass_stalls.py src.csv [top_n]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
isrc, iall, iex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot = Counter()
lines = []
for r in rows[2:]:
    if len(r) <= max(cols):
        continue
    for i in cols:
        tot[hdr[i]] += int(r[i] or 0)
    lines.append((int(r[iall] or 0), r[0], r[isrc].strip()[:90], r[iex]))
s = sum(tot.values())
print("stall reasons (share of samples):")
for k, v in tot.most_common(14):
    print(f"  {k:26s} {100 * v / s:5.1f}%")
print(f"hottest {top} SASS lines (samples, address, instr, executed):")
for n, a, src, ex in sorted(lines, reverse=True)[:top]:
    print(f"  {n:7d} {a:>6s} {src:90s} {ex}")
