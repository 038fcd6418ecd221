#!/usr/bin/env python3
"""Small workload over every device path for compute-sanitizer
(memcheck / racecheck / synccheck): the KKT context at 64^3 (TMA engine, tile
plans, TMA epilogue, PDL) in mixed and f64 modes, every preconditioner, the
B-spline and fp16 interpolation modes, sample_nd and a short registration.

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_17493_b200 as F

n = int(os.environ.get("SAN_N", "64"))
m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
grid = m0.grid
reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
vt = F.VectorField._wrap(grid, 0.1 * torch.randn((3, n, n, n), dtype=torch.float64, device="cuda"))
for tdt, method, prec in ((np.float32, "cubic", "fp32"), (np.float32, "bspline", "fp32"),
                          (np.float32, "cubic", "fp16"), (None, "cubic", "fp32"), (np.float32, "linear", "fp32")):
    st = F.KktState(m0, m1, reg, method=method, v_init=F.VectorField._wrap(grid, 0.5 * vtrue.data),
                    transport_dtype=tdt, interp_precision=prec)
    st.gradient()
    for _ in range(3):  # third call: graph replay on small grids
        st.hessian_matvec(vt)
    if prec == "fp32" and method == "cubic":
        for k in ("reg", "h0", "2level"):
            st.apply_precond(vt, F.PrecondKind(k), 0.5)
        st.objective_at(F.VectorField._wrap(grid, 0.4 * vtrue.data))
        st.detgrad_stats()
    print(f"{method} {prec} {'mixed' if tdt else 'f64'} ok", flush=True)
    del st
q = torch.rand((3, 17, 19, 23), dtype=torch.float64, device="cuda") * 40 - 10
f = torch.rand((17, 19, 23), dtype=torch.float64, device="cuda")
for meth in ("nearest", "linear", "cubic", "bspline"):
    F.sample_nd(f, q, meth)
_, rep = F.register(m0, m1, reg=reg, precond=F.PrecondKind("reg"), transport_dtype=np.float32)
torch.cuda.synchronize()
print("sanitize workload done:", rep.status, rep.iterations, flush=True)
