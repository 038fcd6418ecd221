#!/usr/bin/env python3
"""Event-timed 256^3 planned cubic gather and GN matvec for the library named
by FRG_LIB (compare build variants).  Debug/profiling helper (not a test)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2401_17493_b200 as F
from paper_2401_17493_b200 import _lib as L

n = int(os.environ.get("N", "256"))
m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
import numpy as np
st = F.KktState(m0, m1, reg, v_init=F.VectorField._wrap(m0.grid, 0.5 * vtrue.data), transport_dtype=np.float32)
gen = torch.Generator(device="cuda").manual_seed(0)
vt = F.VectorField._wrap(m0.grid, 0.1 * torch.randn((3, n, n, n), generator=gen, dtype=torch.float64, device="cuda"))
out = torch.empty_like(vt.data)
disp = st.trajectory.disp.to(torch.float32).contiguous()
f = torch.randn((n, n, n), generator=gen, dtype=torch.float32, device="cuda")
g = torch.empty_like(f)
ins = (ctypes.c_void_p * 1)(f.data_ptr())
outs = (ctypes.c_void_p * 1)(g.data_ptr())
nn = L.n3((n, n, n))
plan = torch.empty((L.lib().frg_tile_plan_count(nn), 4), dtype=torch.int32, device="cuda")
L.check(L.lib().frg_tile_plan(nn, 3, 2, ctypes.c_void_p(disp.data_ptr()), L.ptr(plan), L.stream()), "tile_plan")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = 0.0
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        t += a.elapsed_time(b)
    return 1e3 * t / reps


gat = timeit(lambda: L.check(L.lib().frg_gather_planned(nn, 3, 2, ctypes.c_void_p(disp.data_ptr()), L.ptr(plan), 1,
                                                        ins, outs, L.stream()), "gather"), 30)
mv = timeit(lambda: st.hessian_matvec(vt, out=out), 20)
vv = F.VectorField._wrap(m0.grid, 0.5 * vtrue.data)
rf = timeit(lambda: st.refresh(vv), 10)
dg = timeit(lambda: st.detgrad_stats(), 5)  # 12 three-field gathers + pointwise updates


def refresh_first_matvec():
    st.refresh(vv)
    st.hessian_matvec(vt, out=out)  # + the lazy grad m_j(y) gather (12 fields)


rm = timeit(refresh_first_matvec, 10) - rf - mv
print(f"{os.environ.get('FRG_LIB', 'default')}: gather {gat:.1f} us  matvec {mv:.1f} us  refresh {rf:.1f} us  "
      f"detgrad {dg:.1f} us  grads_y {rm:.1f} us")
