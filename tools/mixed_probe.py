#!/usr/bin/env python3
"""mixed (fp32 transport) vs f64 gradient / matvec rel-L2 over sizes and
regularisation variants.  Debug helper."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_17493_b200 as F

for n in [int(x) for x in sys.argv[1:]] or [64, 128, 256]:
    m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
    v = F.VectorField._wrap(m0.grid, 0.5 * vtrue.data)
    for name, reg in [("H1s+near", F.RegConfig(alpha=1e-2, operator=F.RegOperatorSpec(1, True),
                                               incomp=F.IncompressibilityMode("near-incompressible", 1e-4))),
                      ("H1s", F.RegConfig(alpha=1e-2, operator=F.RegOperatorSpec(1, True))),
                      ("H1+near", F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4)))]:
        res = []
        for _ in (0,):
            a = F.KktState(m0, m1, reg, v_init=v, transport_dtype=np.float32)
            ga = a.gradient().data.clone()
            e = F.KktState(m0, m1, reg, v_init=v)
            ge = e.gradient().data
            r = float((ga - ge).norm() / ge.norm())
            res.append(r)
            d = (ga - ge)[0]
            idx = torch.argmax(d.abs())
            res.append(float(d.abs().max() / ge.abs().max()))
            del a, e
        print(n, name, os.environ.get("FRG_FAST_SPECTRAL", "1"), "rel %.2e maxrel %.2e" % tuple(res),
              "gnorm", float(ge.norm()), "gmax", float(ge.abs().max()), flush=True)
