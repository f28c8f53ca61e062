"""Dynamic SASS opcode histogram from `ncu --page source --csv --print-source sass` output.

    python tools/sass_hist.py src.csv [elements]   -> executed warp-instructions per opcode (per element)
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
elems = float(sys.argv[2]) if len(sys.argv) > 2 else None
hdr = rows[1]
ia, isrc, iex, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index(
    "Warp Stall Sampling (All Samples)")
ops, stall = Counter(), Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iex or not r[iex].isdigit():
        continue
    s = r[isrc].strip()
    tok = s.split()
    if not tok:
        continue
    op = tok[1] if tok[0].startswith("@") else tok[0]
    op = op.split(".")[0]
    n = int(r[iex])
    ops[op] += n
    stall[op] += int(r[ist] or 0)
    tot += n
print(f"total warp-instr {tot}" + (f"  = {32 * tot / elems:.2f} thread-instr/elem" if elems else ""))
st = sum(stall.values())
for op, n in ops.most_common(30):
    print(f"{op:10s} {n:12d} {100 * n / tot:5.1f}%" + (f" {32 * n / elems:6.2f}/elem" if elems else "")
          + f"  stall-samples {100 * stall[op] / max(st, 1):5.1f}%")
