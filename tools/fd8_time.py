#!/usr/bin/env python3
"""Event-timed FD8 gradient of 5 fp32 slices at 256^3 (the refresh's call) for
the library named by FRG_LIB.  Debug helper (not a test)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2401_17493_b200 import _lib as L

n = 256
u = torch.randn((5, n, n, n), generator=torch.Generator(device="cuda").manual_seed(0), dtype=torch.float32, device="cuda")
out = torch.empty((5, 3, n, n, n), dtype=torch.float32, device="cuda")
nn = L.n3((n, n, n))


def run():
    L.check(L.lib().frg_fd8_gradient(nn, 3, L.F32, 5, L.ptr(u), L.ptr(out), L.stream()), "fd8")


for _ in range(3):
    run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    run()
b.record()
torch.cuda.synchronize()
print(os.environ.get("FRG_LIB", "default"), "fd8 5 slices: %.1f us" % (a.elapsed_time(b) / 20 * 1e3),
      "checksum %.6e" % float(out.double().abs().sum()))

v = torch.randn((3, n, n, n), generator=torch.Generator(device="cuda").manual_seed(1), dtype=torch.float32, device="cuda")
dv = torch.empty((n, n, n), dtype=torch.float32, device="cuda")


def rund():
    L.check(L.lib().frg_fd8_divergence(nn, 3, L.F32, L.ptr(v), L.ptr(dv), L.stream()), "fd8 div")


for _ in range(3):
    rund()
torch.cuda.synchronize()
a.record()
for _ in range(20):
    rund()
b.record()
torch.cuda.synchronize()
print(os.environ.get("FRG_LIB", "default"), "fd8 divergence: %.1f us" % (a.elapsed_time(b) / 20 * 1e3),
      "checksum %.6e" % float(dv.double().abs().sum()))
