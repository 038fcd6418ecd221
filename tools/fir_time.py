#!/usr/bin/env python3
"""Event-timed B-spline prefilter at 256^3 fp32 (sample_nd "bspline" of one
point: the prefilter dominates) for the library named by FRG_LIB, FIR vs the
spectral round trip (FRG_BSPLINE_SPECTRAL=1).  Profiling helper (not a test)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2401_17493_b200._kernels import sample_nd

n = int(os.environ.get("N", "256"))
u = torch.randn((n, n, n), dtype=torch.float32, device="cuda")
q = [torch.full((1,), 3.5, dtype=torch.float64, device="cuda")] * 3


def t(reps=20):
    for _ in range(3):
        sample_nd(u, q, "bspline")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        sample_nd(u, q, "bspline")
    b.record()
    torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / reps


fir = t()
os.environ["FRG_BSPLINE_SPECTRAL"] = "1"
spec = t()
print(f"{os.environ.get('FRG_LIB', 'default')}: prefilter {n}^3 fp32: FIR {fir:.1f} us, spectral {spec:.1f} us")
