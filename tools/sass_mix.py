#!/usr/bin/env python3
"""Per-opcode executed-instruction mix (per output voxel) from an ncu --set full report.
usage: tools/sass_mix.py report.ncu-rep [voxels]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
vox = float(sys.argv[2]) if len(sys.argv) > 2 else 256 ** 3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ie, src, samp = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
by, smp, tot, tots, lines = collections.Counter(), collections.Counter(), 0, 0, []
for r in rows[2:]:
    try:
        n, s = int(r[ie]), int(r[samp])
    except (ValueError, IndexError):
        continue
    toks = r[src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    by[op] += n; smp[op] += s; tot += n; tots += s
    lines.append((s, n, r[src].strip()))
print(f"total {tot} warp-inst = {tot * 32 / vox:.1f} thread-inst per voxel")
for op, n in by.most_common(30):
    print(f"  {op:10s} {n * 32 / vox:7.1f}/vox   stall-samples {100 * smp[op] / max(tots, 1):5.1f}%")
print("top stall lines:")
for s, n, t in sorted(lines, reverse=True)[:15]:
    print(f"  {s:6d} {n:10d}  {t[:90]}")
