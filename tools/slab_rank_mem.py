#!/usr/bin/env python3
"""Device memory of ONE rank of a slab-decomposed problem, emulated at P = 1
on that rank's slab shape: e.g. C5 (1024^3 over 8 GPUs) = a (128, 1024, 1024)
slab whose axis-0 displacement is scaled so the ghost-plane halo has the width
the real 1024^3 rotation needs (~37 cells per step -> 39 planes).  Runs the
refresh, gradient, a GN matvec and the reg preconditioner, then reports the
peak device memory (torch allocator peak + the library's own buffers via
cudaMemGetInfo).

    python tools/slab_rank_mem.py [--n0 128] [--n 1024] [--disp0 37]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as tdist

import paper_2401_17493_b200 as F
from paper_2401_17493_b200 import dist as D

ap = argparse.ArgumentParser()
ap.add_argument("--n0", type=int, default=128)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--disp0", type=float, default=37.0, help="max axis-0 displacement per SL step, cells")
a = ap.parse_args()

os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29541")
tdist.init_process_group("gloo", rank=0, world_size=1)
comm = D.SlabComm()
shape = (a.n0, a.n, a.n)
free0, total = torch.cuda.mem_get_info()
gen = torch.Generator(device="cuda").manual_seed(0)
x = [torch.linspace(0, 2 * np.pi, s + 1, device="cuda", dtype=torch.float64)[:-1] for s in shape]
X0, X1, X2 = torch.meshgrid(*x, indexing="ij")
m0 = (torch.sin(X0) * torch.cos(X1) * torch.sin(2 * X2) + 1.0).float()
m1 = (torch.sin(X0 + 0.2) * torch.cos(X1 - 0.1) * torch.sin(2 * X2) + 1.0).float()
n_t = 4
h0 = 2 * np.pi / a.n0
amp0 = a.disp0 * h0 * n_t  # physical units: disp0 = (1/n_t) * v0 / h0
v = torch.stack([amp0 * torch.cos(X1), 0.5 * torch.sin(X0) * torch.cos(X2), 0.5 * torch.cos(X0)]).double()
del X0, X1, X2
reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
st = D.DistKktState(m0, m1, reg, comm, shape, v_init=v)
g = st.gradient()
vt = 0.1 * torch.randn(v.shape, generator=gen, dtype=torch.float64, device="cuda")
h = st.hessian_matvec(vt)
z = st.apply_precond(vt, F.PrecondKind("reg"), 0.5)
torch.cuda.synchronize()
free1, _ = torch.cuda.mem_get_info()
print(json.dumps({"slab": list(shape), "halo_planes": [st.Wf, st.Wb], "torch_peak_gb": torch.cuda.max_memory_allocated() / 1e9,
                  "device_used_gb": (total - free1) / 1e9, "device_used_before_gb": (total - free0) / 1e9,
                  "device_total_gb": total / 1e9}))
