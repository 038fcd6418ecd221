#!/usr/bin/env python3
"""Quick check of the fp32 SL gather engine (frg_gather) against a float64
torch restatement of the periodic cubic / linear gather, at sizes where the
TMA path is active.  Debug/profiling helper (not a test)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2401_17493_b200 import _lib as L


def ref_gather(f, disp, method):
    n0, n1, n2 = f.shape
    dev = f.device
    f = f.double()
    i, j, k = torch.meshgrid(torch.arange(n0, device=dev), torch.arange(n1, device=dev), torch.arange(n2, device=dev),
                             indexing="ij")
    q = [i + disp[0].double(), j + disp[1].double(), k + disp[2].double()]
    fl = [torch.floor(x) for x in q]
    t = [x - y for x, y in zip(q, fl)]
    b = [y.long() for y in fl]
    if method == 2:
        def w(t):
            return [-t * (t - 1) * (t - 2) / 6, (t + 1) * (t - 1) * (t - 2) / 2, -(t + 1) * t * (t - 2) / 2,
                    (t + 1) * t * (t - 1) / 6]
        offs = [-1, 0, 1, 2]
    else:
        def w(t):
            return [1 - t, t]
        offs = [0, 1]
    W = [w(x) for x in t]
    out = torch.zeros_like(q[0])
    for a, oa in enumerate(offs):
        for bb, ob in enumerate(offs):
            for c, oc in enumerate(offs):
                val = f[(b[0] + oa) % n0, (b[1] + ob) % n1, (b[2] + oc) % n2]
                out += W[0][a] * W[1][bb] * W[2][c] * val
    return out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    amp = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
    g = torch.Generator(device="cuda").manual_seed(0)
    f = torch.randn((n, n, n), generator=g, device="cuda", dtype=torch.float32)
    x = torch.linspace(0, 6.283185307179586, n + 1, device="cuda")[:n]
    X0, X1, X2 = torch.meshgrid(x, x, x, indexing="ij")
    disp = torch.stack([amp * torch.sin(X1) * torch.cos(X2), amp * torch.cos(X0), amp * 0.5 * torch.sin(X0 + X2)])
    disp = disp.float().contiguous()
    for method in (1, 2):
        out = torch.empty_like(f)
        ins = (ctypes.c_void_p * 1)(f.data_ptr())
        outs = (ctypes.c_void_p * 1)(out.data_ptr())
        L.check(L.lib().frg_gather(L.n3((n, n, n)), 3, L.F32, method, ctypes.c_void_p(disp.data_ptr()), 1, ins, outs,
                                   L.stream()), "gather")
        torch.cuda.synchronize()
        r = ref_gather(f, disp, method)
        err = ((out.double() - r).norm() / r.norm()).item()
        print(f"n={n} method={method} rel L2 err {err:.3e} max {((out.double() - r).abs().max()).item():.3e}")


if __name__ == "__main__":
    main()
