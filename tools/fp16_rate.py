#!/usr/bin/env python3
"""GN matvec rate at n^3 with fp32 vs fp16 interpolation (mixed precision)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_17493_b200 as F

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
reg = F.RegConfig(alpha=1e-2)
vt = F.VectorField._wrap(m0.grid, 0.1 * torch.randn((3, n, n, n), dtype=torch.float64, device="cuda"))
for prec in ("fp32", "fp16"):
    st = F.KktState(m0, m1, reg, v_init=F.VectorField._wrap(m0.grid, 0.5 * vtrue.data), transport_dtype=np.float32,
                    interp_precision=prec)
    out = torch.empty_like(vt.data)
    for _ in range(3):
        st.hessian_matvec(vt, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        st.hessian_matvec(vt, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"{prec}: {20 / (e0.elapsed_time(e1) / 1e3):.1f} matvec/s")
    del st
