"""CPU oracle for the GNK hot path — TEST INFRASTRUCTURE, NOT THE PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this module, and only as
the checker / CPU baseline.  The product (``paper_2401_17493_b200``) never
imports it and has no CPU fallback.

This is an arrays-only restatement of the reference ``flowreg`` package
(/root/reference/pkg/src/flowreg) for the hot path of SURVEY.md §8(a).  Every
function cites the reference file:line it restates.  The inner gathers run in
``oracle/csrc/gather_ref.c`` (OpenMP, f64 weights/accumulation, no FMA
contraction) like the reference's numba kernels; FFTs use scipy's pocketfft
(complex fftn/ifftn, as numpy.fft in the reference) with all host threads.

Pinning: ``tests/test_oracle_golden.py`` checks every function below against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``), so parity of the CUDA path against this
oracle is parity against the reference.

Conventions (fields.py:1-10, 105-114): periodic box [-pi, pi)^d, C-order,
node j holds x = (n/2 - (j+1)) h, so coordinates decrease with the index and
the fractional index of a physical point is q = n/2 - 1 - x/h.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np
import scipy.fft as _sfft

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_gather.so")
_WORKERS = os.cpu_count() or 1
_lib = None


def build_oracle_lib(force: bool = False) -> str:
    """Compile the C gather restatement (gcc, OpenMP, -ffp-contract=off)."""
    src = os.path.join(_HERE, "csrc", "gather_ref.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
        subprocess.check_call(
            ["gcc", "-O3", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
             "-fno-fast-math", src, "-o", _LIB_PATH, "-lm"]
        )
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build_oracle_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        for name in ("oracle_gather_f64", "oracle_gather_f32"):
            fn = getattr(lib, name)
            fn.argtypes = [P, I, I, I, P, P, P, I, ctypes.c_int, P]
            fn.restype = None
        lib.oracle_gather_i32.argtypes = [P, I, I, I, P, P, P, I, P]
        lib.oracle_gather_i32.restype = None
        _lib = lib
    return _lib


# ---------------------------------------------------------------------------
# grid helpers (fields.py:54-133)
# ---------------------------------------------------------------------------

TWO_PI = 2.0 * math.pi


def spacing(n):
    return tuple(TWO_PI / ni for ni in n)


def cell_volume(n):
    return float(np.prod(spacing(n)))


def axis_nodes(n_i, dtype=np.float64):
    """fields.py:105-114 — x_j = (n/2 - (j+1)) h."""
    h = TWO_PI / n_i
    j = np.arange(n_i, dtype=dtype)
    return ((n_i // 2) - (j + 1.0)) * np.asarray(h, dtype=dtype)


def mesh(n, dtype=np.float64):
    axes = np.meshgrid(*[axis_nodes(ni, dtype) for ni in n], indexing="ij")
    return np.stack(axes).astype(dtype)


def l2_inner(a, b, n):
    """fields.py:320-335 — sum(a*b) * prod(h) (pairwise sum in the dtype)."""
    return float(np.sum(a * b)) * cell_volume(n)


def norm_l2(a, n):
    return math.sqrt(max(l2_inner(a, a, n), 0.0))


def norm_inf(a):
    return float(np.max(np.abs(a)))


def trapezoid(slices):
    """fields.py:347-379 — weights (h/2, h, ..., h, h/2) with h = 1/(m-1)."""
    m = len(slices)
    if m < 2:
        raise ValueError("time integral needs at least 2 slices")
    ht = 1.0 / (m - 1)
    acc = 0.5 * ht * (slices[0] + slices[-1])
    for s in slices[1:-1]:
        acc = acc + ht * s
    return acc


# ---------------------------------------------------------------------------
# gathers (_kernels.py:222-251, interp.py:22-62)
# ---------------------------------------------------------------------------

METHOD_CODES = {"nearest": 0, "linear": 1, "cubic": 2}


def check_method(method):
    """interp.py:14-19."""
    if method == "cubic-lagrange":
        method = "cubic"
    if method not in METHOD_CODES:
        raise ValueError(f"unknown interpolation method {method!r}")
    return method


def frac_index(n, pts):
    """interp.py:22-34 — q = (n/2 - 1) - x/h in f64, no wrap."""
    h = spacing(n)
    return [np.ascontiguousarray(((n[i] / 2.0 - 1.0) - pts[i] / h[i]).ravel(), dtype=np.float64)
            for i in range(len(n))]


def sample(values, qs, method):
    """_kernels.sample_nd restated; C kernel (f64 accumulate)."""
    method = check_method(method)
    lib = _load()
    values = np.ascontiguousarray(values)
    d = values.ndim
    shp = values.shape if d == 3 else (1,) + values.shape
    qs = [np.ascontiguousarray(q, dtype=np.float64) for q in qs]
    q0 = qs[0].ctypes.data if d == 3 else None
    q1, q2 = (qs[1], qs[2]) if d == 3 else (qs[0], qs[1])
    npts = q1.shape[0]
    if method == "nearest" and values.dtype == np.int32:
        out = np.empty(npts, dtype=np.int32)
        lib.oracle_gather_i32(values.ctypes.data, *shp, q0, q1.ctypes.data, q2.ctypes.data, npts,
                              out.ctypes.data)
        return out
    if values.dtype not in (np.float32, np.float64):
        values = values.astype(np.float64)
    out = np.empty(npts, dtype=values.dtype)
    fn = lib.oracle_gather_f64 if values.dtype == np.float64 else lib.oracle_gather_f32
    fn(values.ctypes.data, *shp, q0, q1.ctypes.data, q2.ctypes.data, npts, METHOD_CODES[method],
       out.ctypes.data)
    return out


def sample_numpy(values, qs, method):
    """Pure-numpy twin of :func:`sample` (checks the C restatement itself)."""
    method = check_method(method)
    d = values.ndim
    n = values.shape
    if method == "nearest":
        idx = tuple(np.floor(qs[i] + 0.5).astype(np.int64) % n[i] for i in range(d))
        return values[idx]
    vals = values.astype(np.float64) if values.dtype.kind == "f" else values.astype(np.float64)
    fl = [np.floor(qs[i]) for i in range(d)]
    t = [qs[i] - fl[i] for i in range(d)]
    base = [fl[i].astype(np.int64) for i in range(d)]
    if method == "linear":
        out = np.zeros(qs[0].shape)
        for corner in range(1 << d):
            w = 1.0
            idx = []
            for i in range(d):
                bit = (corner >> (d - 1 - i)) & 1
                w = w * (t[i] if bit else 1.0 - t[i])
                idx.append((base[i] + bit) % n[i])
            out = out + w * vals[tuple(idx)]
    else:
        def lag(tt):
            return (-tt * (tt - 1.0) * (tt - 2.0) / 6.0, (tt + 1.0) * (tt - 1.0) * (tt - 2.0) / 2.0,
                    -(tt + 1.0) * tt * (tt - 2.0) / 2.0, (tt + 1.0) * tt * (tt - 1.0) / 6.0)
        w = [lag(t[i]) for i in range(d)]
        out = np.zeros(qs[0].shape)
        for taps in np.ndindex(*(4,) * d):
            ww = 1.0
            idx = []
            for i, a in enumerate(taps):
                ww = ww * w[i][a]
                idx.append((base[i] + a - 1) % n[i])
            out = out + ww * vals[tuple(idx)]
    return out.astype(values.dtype if values.dtype.kind == "f" else np.float64)


# ---------------------------------------------------------------------------
# cubic B-spline (north-star extension; NOT in the reference package, which
# lists it out of scope at SPEC.md:302 — parity unpinned, checked by
# properties: nodal exactness, polynomial/sine approximation order, and the
# CUDA path against this restatement).  Gather structure of _kernels.py:191-219
# with the uniform cubic B-spline weights; periodic interpolation condition
# (c_{j-1} + 4 c_j + c_{j+1}) / 6 = u_j solved spectrally per axis.
# ---------------------------------------------------------------------------
def bspline_prefilter(values):
    """Coefficients c with sum_a beta3 taps = values at every node (periodic)."""
    v = np.asarray(values, dtype=np.float64)
    sym = np.ones(v.shape)
    for axis, n in enumerate(v.shape):
        m = np.fft.fftfreq(n, 1.0 / n)
        shape = [1] * v.ndim
        shape[axis] = n
        sym = sym * ((4.0 + 2.0 * np.cos(2.0 * np.pi * m / n)) / 6.0).reshape(shape)
    return np.real(np.fft.ifftn(np.fft.fftn(v) / sym))


def bspline_weights(t):
    """beta3 at offsets -1, 0, 1, 2 for t in [0, 1)."""
    return ((1.0 - t) ** 3 / 6.0, (3.0 * t ** 3 - 6.0 * t ** 2 + 4.0) / 6.0,
            (-3.0 * t ** 3 + 3.0 * t ** 2 + 3.0 * t + 1.0) / 6.0, t ** 3 / 6.0)


def sample_bspline(values, qs):
    """Cubic B-spline interpolant of ``values`` at fractional indices qs (f64)."""
    c = bspline_prefilter(values)
    d, n = c.ndim, c.shape
    fl = [np.floor(qs[i]) for i in range(d)]
    w = [bspline_weights(qs[i] - fl[i]) for i in range(d)]
    base = [fl[i].astype(np.int64) for i in range(d)]
    out = np.zeros(np.asarray(qs[0]).shape)
    for taps in np.ndindex(*(4,) * d):
        ww = 1.0
        idx = []
        for i, a in enumerate(taps):
            ww = ww * w[i][a]
            idx.append((base[i] + a - 1) % n[i])
        out = out + ww * c[tuple(idx)]
    return out


def interp_field(u, pts, method):
    """interp.interpolate / interpolate_vector (interp.py:42-62)."""
    n = u.shape[-len(pts):]
    qs = frac_index(n, pts)
    if u.ndim == len(n):
        return sample(u, qs, method).reshape(n)
    return np.stack([sample(u[i], qs, method).reshape(n) for i in range(u.shape[0])])


# ---------------------------------------------------------------------------
# differential operators (diffops.py)
# ---------------------------------------------------------------------------

FD8 = ((1, -672.0), (2, 168.0), (3, -32.0), (4, 3.0))  # (distance, weight) diffops.py:77


def fd8_axis(u, axis, h):
    """diffops.py:80-95 — du/dx with the +h neighbour at index j-1.

    u(x - s h) sits at index j+s; u(x + s h) at j-s (np.roll by -s / +s).
    Accumulated s = 4, 3, 2, 1 like the reference loop, then / (840 h).
    """
    acc = np.zeros_like(u)
    for s, w in reversed(FD8):
        acc += w * np.roll(u, -s, axis=axis)
        acc -= w * np.roll(u, s, axis=axis)
    return acc / (840.0 * h)


def fd8_grad(u):
    n = u.shape
    if min(n) < 9:
        raise ValueError("8th-order stencil needs n_i >= 9")
    h = spacing(n)
    return np.stack([fd8_axis(u, i, h[i]) for i in range(u.ndim)])


def _fft(x):
    return _sfft.fftn(x, workers=_WORKERS)


def _ifft_real(x):
    return _sfft.ifftn(x, workers=_WORKERS).real


def int_freqs(n):
    """diffops.py:44-53 — integer DFT frequencies, broadcastable."""
    return np.meshgrid(*[np.fft.fftfreq(ni, d=1.0 / ni) for ni in n], indexing="ij", sparse=True)


def deriv_mult(n, axis):
    """diffops.py:56-64 — -i m per bin, Nyquist zeroed."""
    m = np.fft.fftfreq(n[axis], d=1.0 / n[axis])
    mult = -1j * m
    mult[n[axis] // 2] = 0.0
    shape = [1] * len(n)
    shape[axis] = n[axis]
    return mult.reshape(shape)


def spectral_grad(u):
    """diffops.py:67-73."""
    uh = _fft(u)
    return np.stack([_ifft_real(deriv_mult(u.shape, i) * uh) for i in range(u.ndim)]).astype(u.dtype)


def gradient(u, scheme="fd8"):
    if scheme == "fd8":
        return fd8_grad(u)
    if scheme == "spectral":
        return spectral_grad(u)
    raise ValueError(f"unknown derivative scheme {scheme!r}")


def divergence(v, scheme="spectral"):
    """diffops.py:117-129."""
    n = v.shape[1:]
    acc = np.zeros(n, dtype=v.dtype)
    if scheme == "spectral":
        for i in range(len(n)):
            acc += _ifft_real(deriv_mult(n, i) * _fft(v[i]))
    elif scheme == "fd8":
        h = spacing(n)
        for i in range(len(n)):
            acc += fd8_axis(v[i], i, h[i])
    else:
        raise ValueError(f"unknown derivative scheme {scheme!r}")
    return acc


def jacobian(v, scheme="fd8"):
    """diffops.py:132-139 — J[i, j] = d v_i / d x_j."""
    return np.stack([gradient(v[i], scheme) for i in range(v.shape[0])])


def laplacian(u):
    """diffops.py:142-147."""
    ksq = sum(f * f for f in int_freqs(u.shape))
    return _ifft_real(-ksq * _fft(u))


def reg_symbol(n, order=1, seminorm=True):
    """diffops.py:167-173."""
    ksq = np.broadcast_to(sum(f * f for f in int_freqs(n)), n)
    return ksq ** order if seminorm else (1.0 + ksq) ** order


def apply_symbol(v, sym):
    """diffops.py:176-181 — per component ifftn(sym * fftn(v_i)).real."""
    return np.stack([_ifft_real(sym * _fft(v[i])) for i in range(v.shape[0])]).astype(v.dtype)


def _kernel_completed(n, order, seminorm):
    sym = reg_symbol(n, order, seminorm).copy()
    sym[sym == 0.0] = 1.0
    return sym


def reg_apply(v, alpha, order=1, seminorm=True):
    """diffops.py:184-187."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    return apply_symbol(v, alpha * reg_symbol(v.shape[1:], order, seminorm))


def reg_inverse(v, alpha, order=1, seminorm=True):
    """diffops.py:190-196 — zero symbols replaced by 1."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    return apply_symbol(v, 1.0 / (alpha * _kernel_completed(v.shape[1:], order, seminorm)))


def reg_inv_sqrt(v, alpha, order=1, seminorm=True):
    """diffops.py:199-205."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    return apply_symbol(v, 1.0 / np.sqrt(alpha * _kernel_completed(v.shape[1:], order, seminorm)))


def incomp_multiplier(ksq, mode, beta, alpha):
    """diffops.py:222-242."""
    ksq = np.asarray(ksq, dtype=np.float64)
    if mode == "incompressible":
        return np.ones_like(ksq)
    if mode == "near-incompressible":
        inner = beta * (1.0 / ksq + 1.0)
        return 1.0 / (alpha / inner + 1.0)
    raise ValueError("no projection for mode 'none'")


def project(b, mode, beta, alpha):
    """diffops.py:245-280 — b^ - M(k) k (k.b^)/|k|^2, Nyquist-zeroed k."""
    if mode == "none":
        return b.copy()
    n = b.shape[1:]
    ks = []
    for i, f in enumerate(int_freqs(n)):
        e = np.broadcast_to(f, n).copy()
        e[np.abs(e) == n[i] // 2] = 0.0
        ks.append(e)
    ksq = sum(k * k for k in ks)
    safe = np.where(ksq == 0.0, 1.0, ksq)
    mult = np.where(ksq == 0.0, 0.0, incomp_multiplier(safe, mode, beta, alpha))
    bh = [_fft(b[i]) for i in range(len(n))]
    fac = mult * sum(k * c for k, c in zip(ks, bh)) / safe
    return np.stack([_ifft_real(bh[i] - ks[i] * fac) for i in range(len(n))]).astype(b.dtype)


def low_pass_mask(n):
    """diffops.py:283-289 — keep |k_i| < n_i/4 on every axis."""
    mask = np.ones(n, dtype=bool)
    for i, f in enumerate(int_freqs(n)):
        mask &= np.broadcast_to(np.abs(f) < n[i] / 4, n)
    return mask


def band_filter(u, keep_low=True):
    """diffops.py:292-301, 353-366."""
    mask = low_pass_mask(u.shape)
    if not keep_low:
        mask = ~mask
    return _ifft_real(_fft(u) * mask).astype(u.dtype)


def _coarse_bins(n_fine):
    """diffops.py:304-309."""
    nc = n_fine // 2
    kept = np.concatenate([np.arange(0, nc // 2), np.arange(n_fine - nc // 2 + 1, n_fine)])
    coarse = np.concatenate([np.arange(0, nc // 2), np.arange(nc - nc // 2 + 1, nc)])
    return kept, coarse


def restrict(u):
    """diffops.py:312-326."""
    n = u.shape
    for ni in n:
        if ni % 4:
            raise ValueError("coarsening requires n_i divisible by 4")
    nc = tuple(ni // 2 for ni in n)
    uh = _fft(u)
    ch = np.zeros(nc, dtype=complex)
    src = np.ix_(*[_coarse_bins(ni)[0] for ni in n])
    dst = np.ix_(*[_coarse_bins(ni)[1] for ni in n])
    ch[dst] = uh[src]
    return _ifft_real(ch * (np.prod(nc) / np.prod(n))).astype(u.dtype)


def prolong(u, n_fine):
    """diffops.py:329-340."""
    uh = _fft(u)
    fh = np.zeros(n_fine, dtype=complex)
    src = np.ix_(*[_coarse_bins(ni)[1] for ni in n_fine])
    dst = np.ix_(*[_coarse_bins(ni)[0] for ni in n_fine])
    fh[dst] = uh[src]
    return _ifft_real(fh * (np.prod(n_fine) / np.prod(u.shape))).astype(u.dtype)


# ---------------------------------------------------------------------------
# semi-Lagrangian transport (transport.py)
# ---------------------------------------------------------------------------


def departure(v, h_t, method="cubic"):
    """transport.py:37-45 — y = x - h_t/2 (v(x) + v(x - h_t v(x)))."""
    n = v.shape[1:]
    x = mesh(n, v.dtype)
    yt = x - h_t * v
    v_at = interp_field(v, yt, method)
    return (x - 0.5 * h_t * (v + v_at)).astype(v.dtype)


class Sampler:
    """transport.py:65-80 — fractional indices of one map, reused per gather."""

    def __init__(self, points, method):
        self.n = points.shape[1:]
        self.method = check_method(method)
        self.qs = frac_index(self.n, points)

    def __call__(self, arr):
        if arr.ndim == len(self.n):
            return sample(arr, self.qs, self.method).reshape(self.n)
        lead = arr.shape[: arr.ndim - len(self.n)]
        out = np.empty_like(arr)
        for idx in np.ndindex(*lead):
            out[idx] = sample(arr[idx], self.qs, self.method).reshape(self.n)
        return out


def solve_state(m0, y, n_t, method="cubic"):
    """transport.py:83-98 — m_{j+1} = m_j(y)."""
    smp = Sampler(y, method)
    out = np.empty((n_t + 1, *m0.shape), dtype=m0.dtype)
    out[0] = m0
    for j in range(n_t):
        out[j + 1] = smp(out[j])
    return out


def solve_adjoint(final, yb, divv, n_t, method="cubic"):
    """transport.py:105-135 — backward continuity eq., Heun with '+'."""
    smp = Sampler(yb, method)
    ht = 1.0 / n_t
    dy = smp(divv)
    out = np.empty((n_t + 1, *final.shape), dtype=final.dtype)
    out[n_t] = final
    for j in range(n_t, 0, -1):
        uy = smp(out[j])
        f0 = uy * dy
        up = uy + ht * f0
        f1 = up * divv
        out[j - 1] = uy + 0.5 * ht * (f0 + f1)
    return out


def solve_inc_state(grads, y, vt, n_t, method="cubic"):
    """transport.py:147-176 — d_t m~ = -grad m . v~, m~(0) = 0."""
    smp = Sampler(y, method)
    ht = 1.0 / n_t
    vty = smp(vt)
    shape = vt.shape[1:]
    out = np.empty((n_t + 1, *shape), dtype=vt.dtype)
    out[0] = 0.0
    for j in range(n_t):
        gy = smp(grads[j])
        f0 = -np.sum(gy * vty, axis=0)
        f1 = -np.sum(grads[j + 1] * vt, axis=0)
        out[j + 1] = smp(out[j]) + 0.5 * ht * (f0 + f1)
    return out


def deformation_tensor(v, n_t, method="cubic", scheme="fd8"):
    """transport.py:197-221 — d_t F = (grad v) F, F(0) = I."""
    y = departure(v, 1.0 / n_t, method)
    smp = Sampler(y, method)
    J = jacobian(v, scheme)
    Jy = smp(J)
    ht = 1.0 / n_t
    d = v.shape[0]
    F = np.zeros((d, d, *v.shape[1:]), dtype=v.dtype)
    for i in range(d):
        F[i, i] = 1.0
    for _ in range(n_t):
        Fy = smp(F)
        f0 = np.einsum("ik...,kj...->ij...", Jy, Fy)
        Fp = Fy + ht * f0
        f1 = np.einsum("ik...,kj...->ij...", J, Fp)
        F = Fy + 0.5 * ht * (f0 + f1)
    return F


def determinant(F):
    """fields.py:302-312."""
    if F.shape[0] == 2:
        return F[0, 0] * F[1, 1] - F[0, 1] * F[1, 0]
    return (F[0, 0] * (F[1, 1] * F[2, 2] - F[1, 2] * F[2, 1])
            - F[0, 1] * (F[1, 0] * F[2, 2] - F[1, 2] * F[2, 0])
            + F[0, 2] * (F[1, 0] * F[2, 1] - F[1, 1] * F[2, 0]))


def compose_map(v, n_t, method="cubic"):
    """transport.py:224-247 — per-step displacement composed n_t times."""
    n = v.shape[1:]
    x = mesh(n, v.dtype)
    disp = departure(v, 1.0 / n_t, method) - x
    pts = x + disp
    for _ in range(n_t - 1):
        qs = frac_index(n, pts)
        step = np.stack([sample(disp[i], qs, method).reshape(n) for i in range(len(n))])
        pts = pts + step
    return pts


# ---------------------------------------------------------------------------
# distance measures (distance.py:43-91)
# ---------------------------------------------------------------------------


class ZeroNormError(ValueError):
    pass


def _ncc_moments(md, mr, n):
    a = l2_inner(mr, md, n)
    b = l2_inner(md, md, n)
    c = l2_inner(mr, mr, n)
    if b <= 0.0 or c <= 0.0:
        raise ZeroNormError("normalized cross correlation needs nonzero images")
    return a, b, c


def dist_value(md, mr, kind="ssd"):
    n = md.shape
    if kind == "ssd":
        r = md - mr
        return 0.5 * l2_inner(r, r, n)
    a, b, c = _ncc_moments(md, mr, n)
    return 1.0 - (a * a) / (b * c)


def adjoint_final(md, mr, kind="ssd"):
    if kind == "ssd":
        return -(md - mr)
    a, b, c = _ncc_moments(md, mr, md.shape)
    return -2.0 * (a / (b * c)) * ((a / b) * md - mr)


def incremental_final(mt, md, mr, kind="ssd"):
    if kind == "ssd":
        return -mt
    n = md.shape
    a, b, c = _ncc_moments(md, mr, n)
    mm = l2_inner(md, mt, n)
    rm = l2_inner(mr, mt, n)
    q1 = 2.0 * a * mm / b ** 2 - rm / b
    q2 = 4.0 * a * a * mm / b ** 3 - 2.0 * a * rm / b ** 2
    q3 = a * a / b ** 2
    return (2.0 / c) * (-q1 * mr + q2 * md - q3 * mt)


# ---------------------------------------------------------------------------
# reduced KKT system (kkt.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Reg:
    """kkt.py:56-68 (+ diffops.RegOperatorSpec / IncompressibilityMode)."""

    alpha: float = 1e-2
    order: int = 1
    seminorm: bool = True
    incomp: str = "near-incompressible"
    beta: float = 1e-4


def inner_pcg(op, rhs, pre, tol_rel, max_it, n):
    """kkt.py:99-133 — returns (x, iterations, breakdown)."""
    x = np.zeros_like(rhs)
    r = rhs.copy()
    rn = norm_l2(rhs, n)
    if rn == 0.0:
        return x, 0, False
    z = pre(r)
    s = z.copy()
    rz = l2_inner(r, z, n)
    it = 0
    while it < max_it:
        q = op(s)
        sq = l2_inner(s, q, n)
        if not np.isfinite(sq) or sq <= 0.0:
            return x, it, True
        k = rz / sq
        x = x + k * s
        r = r - k * q
        it += 1
        if norm_l2(r, n) <= tol_rel * rn:
            break
        z = pre(r)
        rz2 = l2_inner(r, z, n)
        if not np.isfinite(rz2) or rz2 <= 0.0:
            return x, it, True
        mu = rz2 / rz
        rz = rz2
        s = z + mu * s
    return x, it, False


class Kkt:
    """kkt.py:136-341 restated on plain arrays."""

    def __init__(self, m0, m1, reg: Reg, n_t=4, distance="ssd", method="cubic", scheme="fd8",
                 v_init=None):
        if m0.shape != m1.shape:
            raise ValueError("images live on different grids")
        self.n = m0.shape
        self.d = m0.ndim
        self.n_t = n_t
        self.m0, self.m1 = m0, m1
        self.reg = reg
        self.distance, self.method, self.scheme = distance, check_method(method), scheme
        self.matvecs = self.pde_solves = self.precond_fallbacks = 0
        self.initial_mismatch = dist_value(m0, m1, distance)
        self.refresh(v_init if v_init is not None else np.zeros((self.d, *self.n), m0.dtype))

    def refresh(self, v):
        """kkt.py:166-187."""
        ht = 1.0 / self.n_t
        self.v = v
        self.y = departure(v, ht, self.method)
        self.yb = departure(-v, ht, self.method)
        self.divv = divergence(v, self.scheme)
        self.mseries = solve_state(self.m0, self.y, self.n_t, self.method)
        self.grads = [gradient(self.mseries[j], self.scheme) for j in range(self.n_t + 1)]
        lam1 = adjoint_final(self.mseries[-1], self.m1, self.distance)
        self.lamseries = solve_adjoint(lam1, self.yb, self.divv, self.n_t, self.method)
        self.pde_solves += 2
        self._gm = None
        self._coarse = None

    def _reg_energy(self, v):
        r = self.reg
        return 0.5 * l2_inner(reg_apply(v, r.alpha, r.order, r.seminorm), v, self.n)

    def objective(self):
        return dist_value(self.mseries[-1], self.m1, self.distance) + self._reg_energy(self.v)

    def objective_at(self, v):
        """kkt.py:201-205 — one state solve with a fresh trajectory."""
        ms = solve_state(self.m0, departure(v, 1.0 / self.n_t, self.method), self.n_t, self.method)
        self.pde_solves += 1
        return dist_value(ms[-1], self.m1, self.distance) + self._reg_energy(v)

    def mismatch(self):
        if self.initial_mismatch == 0.0:
            return 0.0
        return dist_value(self.mseries[-1], self.m1, self.distance) / self.initial_mismatch

    def divergence_energy(self):
        """kkt.py:207-218."""
        if self.reg.incomp != "near-incompressible":
            return 0.0
        w = self.divv
        gw = spectral_grad(w)
        return 0.5 * self.reg.beta * (l2_inner(w, w, self.n) + l2_inner(gw, gw, self.n))

    def _project(self, b):
        r = self.reg
        if r.incomp == "none":
            return b
        return project(b, r.incomp, r.beta, r.alpha)

    def body_force(self, series):
        """kkt.py:225-231."""
        return trapezoid([series[j] * self.grads[j] for j in range(series.shape[0])])

    def gradient(self):
        r = self.reg
        return reg_apply(self.v, r.alpha, r.order, r.seminorm) + self._project(self.body_force(self.lamseries))

    def hessian_matvec(self, vt):
        """kkt.py:237-260."""
        mt = solve_inc_state(self.grads, self.y, vt, self.n_t, self.method)
        fin = incremental_final(mt[-1], self.mseries[-1], self.m1, self.distance)
        lt = solve_adjoint(fin, self.yb, self.divv, self.n_t, self.method)
        self.matvecs += 1
        self.pde_solves += 2
        r = self.reg
        return reg_apply(vt, r.alpha, r.order, r.seminorm) + self._project(self.body_force(lt))

    # -- preconditioners (kkt.py:269-341) --
    def _inv(self, x):
        r = self.reg
        return reg_inverse(x, r.alpha, r.order, r.seminorm)

    def _inv_sqrt(self, x):
        r = self.reg
        return reg_inv_sqrt(x, r.alpha, r.order, r.seminorm)

    def _apply_h0(self, s):
        if self._gm is None:
            self._gm = gradient(self.mseries[-1], self.scheme)
        r = self.reg
        sym = self.reg.alpha * _kernel_completed(self.n, r.order, r.seminorm)
        out = apply_symbol(s, sym)
        return out + np.sum(self._gm * s, axis=0) * self._gm

    def _apply_coarse(self, w):
        if self._coarse is None:
            cm = restrict(self.mseries[-1])
            self._coarse = gradient(cm, self.scheme)
        gc = self._coarse
        sw = self._inv_sqrt(w)
        return w + self._inv_sqrt(np.sum(gc * sw, axis=0) * gc)

    def apply_precond(self, r, kind="reg", outer_tol=1e-6, inner_tol_factor=0.1, inner_max=50):
        if kind == "reg":
            return self._inv(r)
        tol = inner_tol_factor * outer_tol
        if kind == "h0":
            sol, _, broke = inner_pcg(self._apply_h0, r, self._inv, tol, inner_max, self.n)
            if broke:
                self.precond_fallbacks += 1
                return self._inv(r)
            return sol
        u = self._inv_sqrt(r)
        nc = tuple(ni // 2 for ni in self.n)
        ul = np.stack([restrict(band_filter(u[i], True)) for i in range(self.d)])
        sol, _, broke = inner_pcg(self._apply_coarse, ul, lambda x: x.copy(), tol, inner_max, nc)
        if broke:
            self.precond_fallbacks += 1
            return self._inv(r)
        sf = np.stack([band_filter(prolong(sol[i], self.n), True) for i in range(self.d)])
        s = sf + np.stack([band_filter(u[i], False) for i in range(self.d)])
        return self._inv_sqrt(s)


# ---------------------------------------------------------------------------
# optimizer (optimizer.py:81-281)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Opt:
    eps_opt: float = 5e-2
    grad_abs_tol: float = 1e-6
    max_outer: int = 50
    forcing: str = "superlinear"
    armijo_c1: float = 1e-4
    armijo_factor: float = 0.5
    armijo_max_trials: int = 20
    pcg_max_iterations: int = 500


def forcing_tolerance(g, mode="superlinear"):
    if g < 0:
        raise ValueError("gradient norm must be nonnegative")
    return min(0.5, math.sqrt(g)) if mode == "superlinear" else min(0.5, g)


def pcg_newton_step(st: Kkt, g, precond, eta, cfg: Opt):
    """optimizer.py:92-140."""
    n = st.n
    vt = np.zeros_like(g)
    info = {"flag": "converged", "residual_2": 0.0, "residual_inf": 0.0}
    gn = norm_l2(g, n)
    if gn == 0.0:
        return vt, 0, info
    target = eta * gn
    r = -g
    z = st.apply_precond(r, precond, eta)
    s = z.copy()
    rz = l2_inner(r, z, n)
    it = 0
    while it < cfg.pcg_max_iterations:
        hs = st.hessian_matvec(s)
        curv = l2_inner(s, hs, n)
        if not np.isfinite(curv) or curv <= 0.0:
            info["flag"] = "negative_curvature"
            break
        k = rz / curv
        vt = vt + k * s
        r = r - k * hs
        it += 1
        if norm_l2(r, n) < target:
            break
        z = st.apply_precond(r, precond, eta)
        rz2 = l2_inner(z, r, n)
        mu = rz2 / rz
        rz = rz2
        s = z + mu * s
    else:
        info["flag"] = "max_iterations"
    info["residual_2"] = norm_l2(r, n)
    info["residual_inf"] = norm_inf(r)
    return vt, it, info


def armijo(st: Kkt, vt, g, cfg: Opt):
    """optimizer.py:143-166 — returns (gamma or None, trials, J)."""
    slope = l2_inner(g, vt, st.n)
    if slope >= 0.0:
        raise ValueError("not a descent direction")
    j0 = st.objective()
    gamma = 1.0
    for trial in range(1, cfg.armijo_max_trials + 1):
        jt = st.objective_at(st.v + gamma * vt)
        if jt <= j0 + cfg.armijo_c1 * gamma * slope:
            return gamma, trial, jt
        gamma *= cfg.armijo_factor
    return None, cfg.armijo_max_trials, j0


def register(m0, m1, reg: Reg, opt: Opt = Opt(), n_t=4, distance="ssd", precond="2level",
             method="cubic", scheme="fd8", v0=None, compute_detgrad=True):
    """optimizer.py:174-281 — returns (v, report dict)."""
    st = Kkt(m0, m1, reg, n_t, distance, method, scheme, v0)
    g = st.gradient()
    gn = norm_inf(g)
    g0 = gn
    obj = st.objective()
    trace = [dict(iteration=0, objective=obj, mismatch=st.mismatch(), gnorm_inf=gn, step=0.0,
                  pcg_iterations=0, eta=0.0)]
    status, reason, it, ls = "max_iterations", "", 0, 0
    if gn <= opt.grad_abs_tol:
        status, reason = "converged", "absolute_gradient"
    else:
        while it < opt.max_outer:
            eta = forcing_tolerance(gn, opt.forcing)
            vt, pit, info = pcg_newton_step(st, g, precond, eta, opt)
            try:
                gamma, trials, _ = armijo(st, vt, g, opt)
            except ValueError:
                status, reason = "line_search_failed", "no_descent_direction"
                break
            ls += trials
            if gamma is None:
                status, reason = "line_search_failed", "armijo_exhausted"
                break
            st.refresh(st.v + gamma * vt)
            g = st.gradient()
            gn = norm_inf(g)
            new = st.objective()
            if new > obj + 1e-10 * max(1.0, abs(obj)):
                raise RuntimeError("objective increased across an accepted step")
            obj = new
            it += 1
            trace.append(dict(iteration=it, objective=obj, mismatch=st.mismatch(), gnorm_inf=gn,
                              step=gamma, pcg_iterations=pit, eta=eta))
            if gn <= opt.eps_opt * g0:
                status, reason = "converged", "relative_gradient"
                break
            if gn <= opt.grad_abs_tol:
                status, reason = "converged", "absolute_gradient"
                break
    rep = dict(iterations=it, matvecs=st.matvecs, pde_solves=st.pde_solves, line_search_evals=ls,
               precond_fallbacks=st.precond_fallbacks, mismatch=st.mismatch(),
               gradient=0.0 if g0 == 0.0 else gn / g0, status=status, exit_reason=reason,
               divergence_energy=st.divergence_energy(), trace=trace)
    if compute_detgrad:
        det = determinant(deformation_tensor(st.v, n_t, method, scheme))
        rep.update(detgrad_min=float(det.min()), detgrad_mean=float(det.mean()),
                   detgrad_max=float(det.max()))
    return st.v, rep


# ---------------------------------------------------------------------------
# synthetic inputs (synth.py:28-118) — input generation for parity tests
# ---------------------------------------------------------------------------


def _bump(n, rng, bumps=6, dtype=np.float64):
    xs = np.meshgrid(*[axis_nodes(ni) for ni in n], indexing="ij", sparse=True)
    vals = np.zeros(n)
    for _ in range(bumps):
        c = rng.uniform(-np.pi, np.pi, size=len(n))
        kappa = rng.uniform(1.0, 2.5)
        amp = rng.uniform(0.4, 1.0)
        b = np.ones(n)
        for ci, x in zip(c, xs):
            b = b * np.exp(kappa * (np.cos(x - ci) - 1.0))
        vals += amp * b
    vals -= vals.min()
    pk = vals.max()
    if pk > 0:
        vals /= pk
    return vals.astype(dtype)


def _vortex(n, amp, phases=(0.0, 0.0), dtype=np.float64):
    xs = [np.broadcast_to(c, n) for c in np.meshgrid(*[axis_nodes(ni) for ni in n], indexing="ij",
                                                        sparse=True)]
    p0, p1 = phases
    v = np.zeros((len(n), *n), dtype=dtype)
    v[0] = -amp * np.cos(xs[0] - p0) * np.sin(xs[1] - p1)
    v[1] = amp * np.sin(xs[0] - p0) * np.cos(xs[1] - p1)
    if len(n) == 3:
        mod = 1.0 + 0.3 * np.cos(xs[2])
        v[0] *= mod
        v[1] *= mod
    return v


def synth_velocity(name, n, rng, dtype=np.float64):
    d = len(n)
    xs = [np.broadcast_to(c, n) for c in np.meshgrid(*[axis_nodes(ni) for ni in n], indexing="ij",
                                                        sparse=True)]
    if name == "translation":
        shift = rng.uniform(0.3, 0.7, size=d) * rng.choice((-1.0, 1.0), size=d)
        v = np.empty((d, *n), dtype=dtype)
        for i in range(d):
            v[i].fill(shift[i])
        return v
    if name == "rotation":
        return _vortex(n, 0.7, dtype=dtype)
    if name == "swirl":
        amp = 0.6
        v = _vortex(n, amp, tuple(rng.uniform(-np.pi, np.pi, size=2)), dtype)
        q0, q1 = rng.uniform(-np.pi, np.pi, size=2)
        b = 0.5 * amp
        v[0] += -b * 0.5 * np.cos(2.0 * (xs[0] - q0)) * np.sin(xs[1] - q1)
        v[1] += b * np.sin(2.0 * (xs[0] - q0)) * np.cos(xs[1] - q1)
        return v
    if name == "compress":
        v = np.zeros((d, *n), dtype=dtype)
        v[0] = 3.0 * np.sin(xs[0])
        return v
    raise ValueError(f"unknown synthetic case {name!r}")


def synth_case(name, n, seed=0, d=2, ref_steps=64):
    """synth.py:88-118 — (m0, m1, v_true) in f64."""
    if n < 32 or (n & (n - 1)) != 0:
        raise ValueError("n must be a power of two >= 32")
    rng = np.random.default_rng(seed)
    shape = (n,) * d
    m0 = _bump(shape, rng)
    v = synth_velocity(name, shape, rng)
    y = departure(v, 1.0 / ref_steps, "cubic")
    m1 = solve_state(m0, y, ref_steps, "cubic")[-1]
    return m0, m1, v
