#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys


def load(fn):
    rows = list(csv.reader(open(fn)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((d["Kernel Name"], float(d["Metric Value"])))
    return out


if __name__ == "__main__":
    for fn in sys.argv[1:]:
        out = load(fn)
        tot = sum(t for _, t in out)
        print(f"{fn}: {len(out)} launches, {tot / 1e3:.1f} us total")
        for k, t in out:
            print(f"{t / 1e3:9.1f} us {100 * t / tot:5.1f}%  {k[:110]}")
