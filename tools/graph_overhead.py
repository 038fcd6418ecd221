#!/usr/bin/env python3
"""Per-node cost of a CUDA-graph replay on this GPU: a graph of K dependent
tiny kernels (one 256-thread block adding to a 1 KB buffer) replayed
back-to-back, CUDA events.  The floor a K-kernel small-grid matvec graph
pays before any work."""
import torch

x = torch.zeros(256, device="cuda")
s = torch.cuda.Stream()
for k in (1, 21, 64):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        x.add_(1.0)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(k):
                x.add_(1.0)
    torch.cuda.synchronize()
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 200
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(f"graph of {k:3d} dependent tiny kernels: {us:7.1f} us per replay, {us / k:5.2f} us per node")
