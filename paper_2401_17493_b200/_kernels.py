"""Point sampling at fractional indices — the narrow drop-in boundary.

Mirrors ``flowreg._kernels.sample_nd`` (/root/reference/pkg/src/flowreg/
_kernels.py:222-251): same arguments, periodic floor-mod wrap, nearest /
multilinear / cubic-Lagrange (nodes at offsets -1..2), same output dtype rule
(input dtype for floats, int32 kept for nearest, f64 for non-float
linear/cubic) and ValueError on an unknown method.  The work runs in the
sm_100a kernel behind ``frg_sample``; numpy inputs are copied to HBM and the
result copied back, torch CUDA inputs stay on the device.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as L

__all__ = ["USING_CUDA", "sample_nd"]

USING_CUDA = True


def sample_nd(values, qs, method: str):
    if method not in L.METHODS:
        raise ValueError(f"unknown interpolation method {method!r}")
    L.require_cuda()
    host = not isinstance(values, torch.Tensor)
    v = torch.from_numpy(np.ascontiguousarray(values)) if host else values
    if v.dtype not in (torch.float32, torch.float64, torch.int32):
        v = v.to(torch.float64)
    v = v.cuda().contiguous()
    d = v.dim()
    if d not in (2, 3) or len(qs) != d:
        raise ValueError("values must be 2D or 3D with one query array per axis")
    q = [torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)) if not isinstance(x, torch.Tensor) else x
         for x in qs]
    q = [x.to("cuda", torch.float64).contiguous().reshape(-1) for x in q]
    npts = q[0].numel()
    if method == "nearest" or v.dtype != torch.int32:
        odt = v.dtype
    else:
        odt = torch.float64
    out = torch.empty(npts, dtype=odt, device="cuda")
    q0 = L.ptr(q[0]) if d == 3 else None
    q1, q2 = (q[1], q[2]) if d == 3 else (q[0], q[1])
    L.check(L.lib().frg_sample(L.ptr(v), L.dtype_code(v.dtype), L.n3(v.shape), q0, L.ptr(q1), L.ptr(q2), npts,
                               L.METHODS[method], L.ptr(out), L.stream()), "sample_nd")
    return out.cpu().numpy() if host else out
