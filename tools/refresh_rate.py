#!/usr/bin/env python3
"""KktState.refresh (RK2 departure maps, state / adjoint solves, FD8) and
objective_at (one Armijo trial) at n^3, mixed precision, CUDA events; plus a
256^3 registration wall.  usage: python tools/refresh_rate.py [n] [method]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_17493_b200 as F

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
meth = sys.argv[2] if len(sys.argv) > 2 else "cubic"
m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
v = F.VectorField._wrap(m0.grid, 0.5 * vtrue.data)
st = F.KktState(m0, m1, reg, method=meth, v_init=v, transport_dtype=np.float32)
trial = F.VectorField._wrap(m0.grid, 0.4 * vtrue.data)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for what, fn in (("refresh", lambda: st.refresh(v)), ("objective_at", lambda: st.objective_at(trial))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{what} {n}^3 {meth}: {best * 1e3:.0f} us", flush=True)
del st
if n == 256:
    walls = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rep = F.register(m0, m1, reg=reg, precond=F.PrecondKind("reg"), method=meth,
                            scheme="fd8", transport_dtype=np.float32)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    print(f"register 256^3 {meth}: {min(walls[1:]):.4f} s ({rep.iterations} it, {rep.matvecs} mv)", flush=True)
