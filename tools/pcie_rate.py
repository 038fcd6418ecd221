#!/usr/bin/env python3
"""Pinned host<->device copy rates for the e2e matvec's 402 MB buffers:
H2D alone, D2H alone, both at once on two streams.  Debug helper."""
import torch

n = 3 * 256 ** 3
h_in = torch.randn(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


B = n * 8 / 1e9
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.2f} ms per 402 MB step  ({B / ms * 1e3:.1f} GB/s per direction)")
