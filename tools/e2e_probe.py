#!/usr/bin/env python3
"""Pipelined host-buffer matvec (KktState.hessian_matvec on pinned host
tensors) timed for several step counts.  Debug helper."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_17493_b200 as F

n = 256
m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
st = F.KktState(m0, m1, reg, v_init=F.VectorField._wrap(m0.grid, 0.5 * vtrue.data), transport_dtype=np.float32)
vt = 0.1 * torch.randn((3, n, n, n), dtype=torch.float64, device="cuda")
host_in = vt.cpu().pin_memory()
host_out = torch.empty_like(host_in).pin_memory()
stream = torch.cuda.current_stream()
for K in [int(x) for x in sys.argv[1:]] or [5, 10, 20, 30]:
    for _ in range(3):
        st.hessian_matvec(host_in, out=host_out)
    st.wait_host_io()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(K):
        st.hessian_matvec(host_in, out=host_out)
    st.wait_host_io()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"K={K}: {ms / K:.2f} ms/step  {1e3 * K / ms:.1f} matvec/s")
