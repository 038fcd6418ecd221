#!/usr/bin/env python3
"""Halo vs point routing for the slab decomposition, MEASURED on the real
departure maps (SURVEY.md §8e collective 2; PAPER.md:545 routes off-rank
departure points).

For the bench state (synth rotation, v = v_true / 2, n_t = 4, cubic) at n^3 the
forward and backward RK2 maps are computed on one GPU (fp32 TMA engine), then
for every rank count P the bytes one SL gather moves per rank are counted:

* halo (dist.py, what ships): W = ceil(max |d0|) + 2 ghost planes on each side
  of the slab, fp32: 2 W n1 n2 4 B per gather per rank;
* routing: a point whose stencil base plane floor(i + d0) lies on another
  rank is sent to that rank once per map (12 B of coordinates) and its value
  comes back on every gather (4 B); points whose base is local still need the
  cubic stencil's 1 + 2 ghost planes (3 n1 n2 4 B per gather).  The maximum
  over ranks of the points a rank serves is reported.

    python tools/routing_bytes.py [n]      (default 1024; ~60 GB of HBM)
Writes profiles/r02_halo_vs_routing_<n>.json.
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_17493_b200 as F
from paper_2401_17493_b200.transport import departure_disp

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
grid = F.Grid((n, n, n), n_t=4, dtype=np.float32)
# rotation velocity (synth.py:46-63) at v_true / 2, built in fp32 plane chunks
ax = ((n // 2) - (torch.arange(n, dtype=torch.float64, device="cuda") + 1.0)) * (2 * math.pi / n)
v = torch.zeros((3, n, n, n), dtype=torch.float32, device="cuda")
mod = (1.0 + 0.3 * torch.cos(ax)).view(1, 1, n)
for i0 in range(0, n, 64):
    x0 = ax[i0:i0 + 64].view(-1, 1, 1)
    v[0, i0:i0 + 64] = (-0.35 * torch.cos(x0) * torch.sin(ax.view(1, n, 1)) * mod).float()
    v[1, i0:i0 + 64] = (0.35 * torch.sin(x0) * torch.cos(ax.view(1, n, 1)) * mod).float()
res = {"n": n, "state": "synth rotation, v = v_true / 2 (the bench state), n_t = 4, cubic", "maps": {}}
for name, sign in (("forward", 1.0), ("backward", -1.0)):
    disp = departure_disp(F.VectorField._wrap(grid, sign * v if sign < 0 else v), grid.h_t, "cubic")
    d0 = disp[0]
    del disp
    maxd = float(d0.abs().max())
    W = int(math.ceil(maxd)) + 2
    plane = n * n * 4
    rows = []
    for P in (2, 4, 8):
        if n % P:
            continue
        m = n // P
        served = torch.zeros(P, dtype=torch.int64, device="cuda")  # points other ranks route to rank q
        for i0 in range(0, n, 32):
            i = torch.arange(i0, i0 + 32, device="cuda").view(-1, 1, 1)
            base = (i + torch.floor(d0[i0:i0 + 32]).to(torch.int64)) % n
            own = i // m
            dst = base // m
            off = dst != own
            served += torch.bincount(dst[off].view(-1), minlength=P)
        routed = int(served.max())
        rows.append({"ranks": P, "halo_planes": W, "halo_bytes_per_gather_per_rank": 2 * W * plane,
                     "routed_points_max_rank": routed, "routed_fraction_of_slab": routed / (m * n * n),
                     "routing_bytes_per_gather_per_rank": routed * 4 + 3 * plane,
                     "routing_bytes_per_map_per_rank": routed * 12,
                     "halo_over_routing": 2 * W * plane / (routed * 4 + 3 * plane),
                     "slab_planes": m, "halo_fits_slab": W <= m})
    res["maps"][name] = {"max_abs_disp0": maxd, "rows": rows}
    del d0
    torch.cuda.empty_cache()
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   f"r02_halo_vs_routing_{n}.json")
with open(out, "w") as fh:
    json.dump(res, fh, indent=1)
for name, mres in res["maps"].items():
    for r in mres["rows"]:
        print(f"{name:8s} P={r['ranks']}: halo W={r['halo_planes']} {r['halo_bytes_per_gather_per_rank'] / 1e6:.1f} MB"
              f" | routing {r['routed_points_max_rank'] / 1e6:.2f} M points ({100 * r['routed_fraction_of_slab']:.1f}%"
              f" of the slab) {r['routing_bytes_per_gather_per_rank'] / 1e6:.1f} MB per gather"
              f" + {r['routing_bytes_per_map_per_rank'] / 1e6:.1f} MB per map | halo/routing "
              f"{r['halo_over_routing']:.2f}")
