#!/usr/bin/env python3
"""Per-opcode executed-instruction histogram from `ncu --page source --csv --print-source sass`."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(d["Instructions Executed"] or 0) for d in data)
print("total warp inst", tot)
c = Counter()
for d in data:
    s = d["Source"].strip().split()
    if not s:
        continue
    op = s[1] if s[0].startswith("@") and len(s) > 1 else s[0]
    c[op.split(".")[0]] += int(d["Instructions Executed"] or 0)
for op, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{op:10s} {n:12d} {n / tot * 100:5.1f}%")
if len(sys.argv) > 3:
    thr = int(sys.argv[3])
    for i, d in enumerate(data):
        n = int(d["Instructions Executed"] or 0)
        if n >= thr:
            print(i, n, d["Source"].strip()[:90])
