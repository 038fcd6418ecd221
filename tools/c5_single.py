#!/usr/bin/env python3
"""C5's workflow (alpha continuation to alpha* = 1.773437e-3, PAPER.md:846;
cascade continuation.py:225-293) on ONE B200 at the largest grid that fits
(default 512^3; C5 proper is 1024^3 over 8 GPUs): synthetic rotation case,
reg preconditioner (or --precond 2level, the reference default), mixed
precision.  Prints one JSON line with per-stage counts and wall times.

    python tools/c5_single.py [--n 512] [--precond reg]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_17493_b200 as F
from paper_2401_17493_b200.continuation import cascade_alphas, continuation_solve

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--precond", default="reg")
ap.add_argument("--alpha", type=float, default=1.773437e-3)
a = ap.parse_args()

t0 = time.perf_counter()
m0, m1, _ = F.synth_case("rotation", a.n, seed=1, d=3)
torch.cuda.synchronize()
t_synth = time.perf_counter() - t0
reg = F.RegConfig(alpha=a.alpha, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
walls = []
for _ in range(2):  # the first run creates the cuFFT plans
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, total, stages = continuation_solve(m0, m1, a.alpha, reg=reg, precond=F.PrecondKind(a.precond),
                                          transport_dtype=np.float32)
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
print(json.dumps({
    "workload": f"C5 workflow on one GPU: alpha continuation to {a.alpha:g} at {a.n}^3 (synth rotation, "
                f"H1 near-incompressible beta=1e-4, cubic, fd8, precond {a.precond}, mixed precision)",
    "alphas": cascade_alphas(a.alpha), "seconds": walls[-1], "first_call_seconds": walls[0],
    "synth_seconds": t_synth, "status": total.status, "iterations": total.iterations, "matvecs": total.matvecs,
    "pde_solves": total.pde_solves, "mismatch": total.mismatch,
    "detgrad": [total.detgrad_min, total.detgrad_mean, total.detgrad_max],
    "stages": [{"iterations": s.iterations, "matvecs": s.matvecs, "status": s.status, "runtime": s.runtime,
                "mismatch": s.mismatch} for s in stages],
    "device_mem_used_gb_at_end": (lambda fr_tot: (fr_tot[1] - fr_tot[0]) / 1e9)(torch.cuda.mem_get_info()),
}))
