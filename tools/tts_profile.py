#!/usr/bin/env python3
"""Time-to-solution breakdown of register() at n^3 (per KktState method, synced)."""
import argparse
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_17493_b200 as F
from paper_2401_17493_b200 import kkt

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--precond", default="reg")
ap.add_argument("--incomp", default="near-incompressible")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()

acc = collections.defaultdict(float)
cnt = collections.Counter()
mx = collections.defaultdict(float)


def wrap(name):
    f = getattr(kkt.KktState, name)

    def g(self, *args, **kw):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(self, *args, **kw)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        acc[name] += dt
        cnt[name] += 1
        mx[name] = max(mx[name], dt)
        return r
    setattr(kkt.KktState, name, g)


for nm in ["__init__", "refresh", "gradient", "hessian_matvec", "apply_precond", "objective", "objective_at",
           "mismatch", "divergence_energy", "detgrad_stats"]:
    wrap(nm)

m0, m1, v = F.synth_case("rotation", a.n, seed=1, d=3)
reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode(a.incomp, 1e-4))
for rep in range(a.reps):
    acc.clear()
    cnt.clear()
    mx.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vs, r = F.register(m0, m1, reg=reg, precond=F.PrecondKind(a.precond), transport_dtype=np.float32)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"run {rep}: wall {wall:.3f}s it={r.iterations} mv={r.matvecs} status={r.status}")
    for k in sorted(acc, key=lambda k: -acc[k]):
        print(f"   {k:18s} {cnt[k]:4d} calls {acc[k]*1e3:9.1f} ms  (max {mx[k]*1e3:.2f} ms)")
