#!/usr/bin/env python3
"""Slab path at P = 1 (gloo, one process) vs the single-GPU context: matvec/s
at n^3 — the overhead of the slab machinery (ghost-plane buffers, 2D+1D FFT,
transposes) without any communication."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as tdist

import paper_2401_17493_b200 as F
from paper_2401_17493_b200 import dist as D

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
tdist.init_process_group("gloo", rank=0, world_size=1)
m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
reg = F.RegConfig(alpha=1e-2)
v = 0.5 * vtrue.data
vt = 0.1 * torch.randn((3, n, n, n), dtype=torch.float64, device="cuda")


def rate(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return reps / (e0.elapsed_time(e1) / 1e3)


st = F.KktState(m0, m1, reg, v_init=F.VectorField._wrap(m0.grid, v), transport_dtype=np.float32)
out = torch.empty_like(vt)
r1 = rate(lambda: st.hessian_matvec(F.VectorField._wrap(m0.grid, vt), out=out))
del st
ds = D.DistKktState(m0.values.float(), m1.values.float(), reg, D.SlabComm(), (n, n, n), v_init=v)
r2 = rate(lambda: ds.hessian_matvec(vt, out=out))
print(f"n={n}: single-GPU context {r1:.1f} matvec/s, slab path P=1 {r2:.1f} matvec/s")
if os.environ.get("PROFILE"):  # one slab matvec between cudaProfilerStart/Stop (ncu --profile-from-start off)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ds.hessian_matvec(vt, out=out)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
tdist.destroy_process_group()
