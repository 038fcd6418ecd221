#!/usr/bin/env python3
"""Per-kernel SASS listing with executed counts from an exported source page
(tools/ncu_export.sh): opcode mix per output voxel and the hottest regions.
usage: tools/src_csv.py X_src.csv.gz [voxels] [kernel-substring] [--dump]"""
import collections, csv, gzip, io, sys
path = sys.argv[1]
vox = float(sys.argv[2]) if len(sys.argv) > 2 else 256 ** 3
want = sys.argv[3] if len(sys.argv) > 3 else ""
dump = "--dump" in sys.argv
txt = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
rows = list(csv.reader(io.StringIO(txt)))
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kernels.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and r:
        cur["rows"].append(r)
for k in kernels:
    if want not in k["name"]:
        continue
    h = k["hdr"]
    ie, src, ss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    wfs = h.index("L1 Wavefronts Shared")
    by, tot, wf = collections.Counter(), 0, 0
    lines = []
    for r in k["rows"]:
        try:
            n = int(r[ie]); s = int(r[ss]); w = int(r[wfs] or 0)
        except (ValueError, IndexError):
            continue
        t = r[src].split()
        op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0] if t else "?"
        by[op] += n; tot += n; wf += w
        lines.append((n, s, w, r[src].strip()))
    print(f"== {k['name'][:110]}\n   {tot * 32 / vox:.1f} thread-inst/voxel, shared wavefronts {wf / vox:.3f}/voxel")
    print("   " + "  ".join(f"{op} {n * 32 / vox:.1f}" for op, n in by.most_common(24)))
    if dump:
        for i, (n, s, w, t) in enumerate(lines):
            print(f"{i:5d} {n:10d} {s:6d} {w:9d}  {t[:100]}")
