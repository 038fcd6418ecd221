#!/usr/bin/env python3
"""GN matvec rate of the small-grid configs (C1 64^3 H1 cubic, C2 128^3 H2
linear; mixed precision, near-incompressible), as bench.py's other_configs
measures them: 20 back-to-back calls after 3 warm-ups, CUDA events.
Also checks the result against the eager (non-graph) path of a second
context.  usage: python tools/small_rate.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_17493_b200 as F

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
gen = torch.Generator(device="cuda").manual_seed(0)
for tag, n, order, meth in (("C1", 64, 1, "cubic"), ("C2", 128, 2, "linear")):
    m0, m1, vv = F.synth_case("rotation", n, seed=1, d=3)
    rg = F.RegConfig(alpha=1e-2, operator=F.RegOperatorSpec(order, True),
                     incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
    st = F.KktState(m0, m1, rg, method=meth, v_init=F.VectorField._wrap(m0.grid, 0.5 * vv.data),
                    transport_dtype=np.float32)
    vt = F.VectorField._wrap(m0.grid, 0.1 * torch.randn((3, n, n, n), generator=gen, dtype=torch.float64,
                                                        device="cuda"))
    out = torch.empty_like(vt.data)
    first = st.hessian_matvec(vt).data.clone()  # eager (first call)
    for _ in range(3):
        st.hessian_matvec(vt, out=out)
    torch.cuda.synchronize()
    rel = float((out - first).norm() / first.norm())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best, host = 0.0, 1e9
    for _ in range(3):
        e0.record()
        t0 = time.perf_counter()
        for _ in range(reps):
            st.hessian_matvec(vt, out=out)
        host = min(host, (time.perf_counter() - t0) / reps)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, reps / (e0.elapsed_time(e1) / 1e3))
    # one call alone: device time of a single matvec with an idle queue
    one = 1e9
    for _ in range(20):
        torch.cuda.synchronize()
        e0.record()
        st.hessian_matvec(vt, out=out)
        e1.record()
        torch.cuda.synchronize()
        one = min(one, e0.elapsed_time(e1) * 1e3)
    print(f"{tag} {n}^3: {best:.0f} matvec/s ({1e6 / best:.1f} us/call back-to-back), host enqueue "
          f"{host * 1e6:.1f} us/call, single call {one:.1f} us; graph vs eager rel-L2 {rel:.2e}", flush=True)
    del st
