#!/usr/bin/env python3
"""Profiling driver: one 256^3 Hessian matvec (the bench step) between
cudaProfilerStart/Stop, for `ncu --profile-from-start off`.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python tools/profile_step.py [--n 256] [--what matvec|refresh|gather]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2401_17493_b200 as F
from paper_2401_17493_b200 import _lib as L

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--what", default="matvec", choices=["matvec", "refresh", "gather", "gradient", "precond", "objective_at", "detgrad"])
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--precision", default="mixed")
ap.add_argument("--interp", default="fp32", choices=["fp32", "fp16"])
ap.add_argument("--method", default="cubic", choices=["cubic", "linear", "bspline"])
a = ap.parse_args()

n = a.n
dtype = np.float32 if a.precision == "f32" else np.float64
tdt = np.float32 if a.precision in ("mixed", "f32") else None
m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3, dtype=dtype)
grid = m0.grid
reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
v = F.VectorField._wrap(grid, 0.5 * vtrue.data)
st = F.KktState(m0, m1, reg, method=a.method, v_init=v, transport_dtype=tdt, interp_precision=a.interp)
gen = torch.Generator(device="cuda").manual_seed(0)
vt = F.VectorField._wrap(grid, 0.1 * torch.randn((3, n, n, n), generator=gen, dtype=grid.torch_dtype, device="cuda"))
out = torch.empty_like(vt.data)
disp = st.trajectory.disp.to(torch.float32).contiguous()
f = torch.randn((n, n, n), generator=gen, dtype=torch.float32, device="cuda")
g = torch.empty_like(f)
ins = (ctypes.c_void_p * 1)(f.data_ptr())
outs = (ctypes.c_void_p * 1)(g.data_ptr())
plan = torch.empty((L.lib().frg_tile_plan_count(L.n3((n, n, n))), 4), dtype=torch.int32, device="cuda")
L.check(L.lib().frg_tile_plan(L.n3((n, n, n)), 3, 2, ctypes.c_void_p(disp.data_ptr()), L.ptr(plan), L.stream()),
        "tile_plan")


def step():
    if a.what == "matvec":
        st.hessian_matvec(vt, out=out)
    elif a.what == "gradient":
        st.gradient()
    elif a.what == "refresh":
        st.refresh(v)
    elif a.what == "precond":
        st.apply_precond(vt, F.PrecondKind("reg"), 0.5, out=out)
    elif a.what == "objective_at":
        st.objective_at(F.VectorField._wrap(grid, 0.4 * vtrue.data))  # a smooth Armijo trial
    elif a.what == "detgrad":
        st.detgrad_stats()
    else:
        L.check(L.lib().frg_gather_planned(L.n3((n, n, n)), 3, 2, ctypes.c_void_p(disp.data_ptr()), L.ptr(plan), 1,
                                           ins, outs, L.stream()), "gather")


for _ in range(2):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.reps):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
