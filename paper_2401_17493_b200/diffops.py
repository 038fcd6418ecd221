"""Spectral and finite-difference differential operators on the device.

Mirrors flowreg.diffops (/root/reference/pkg/src/flowreg/diffops.py:1-366):
FD8 first derivatives (periodic, +h neighbour at index j-1), pseudo-spectral
derivatives (-i m, Nyquist zeroed), Sobolev regularisation symbols and their
inverse / inverse square root (zero symbol -> 1), the Leray / near-
incompressible body-force projection, band filters and spectral
restriction / prolongation.  FD8 runs in a fused stencil kernel; spectral
operators run as cuFFT R2C/C2R transforms bracketed by fused pointwise
kernels in libflowreg_b200.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .fields import Grid, ScalarField, VectorField

__all__ = [
    "RegOperatorSpec",
    "IncompressibilityMode",
    "spectral_gradient",
    "fd8_gradient",
    "gradient",
    "divergence",
    "laplacian",
    "apply_reg_operator",
    "apply_inv_reg_operator",
    "apply_inv_sqrt_reg_operator",
    "reg_symbol",
    "incompressibility_multiplier",
    "project_body_force",
    "restrict",
    "prolong",
    "low_pass",
    "high_pass",
    "low_pass_mask",
    "jacobian",
    "restrict_vector",
    "prolong_vector",
    "low_pass_vector",
    "high_pass_vector",
]


@dataclass(frozen=True)
class RegOperatorSpec:
    """diffops.py:150-164."""

    order: int = 1
    seminorm: bool = True

    def __post_init__(self):
        if self.order not in (1, 2, 3):
            raise ValueError(f"order must be 1, 2 or 3, got {self.order}")


@dataclass(frozen=True)
class IncompressibilityMode:
    """diffops.py:208-219."""

    mode: str = "none"
    beta: float = 1e-4

    def __post_init__(self):
        if self.mode not in ("none", "incompressible", "near-incompressible"):
            raise ValueError(f"unknown incompressibility mode {self.mode!r}")
        if self.mode == "near-incompressible" and self.beta <= 0:
            raise ValueError("beta must be positive for the relaxed mode")


def frg_reg(spec: RegOperatorSpec = RegOperatorSpec(), alpha: float = 1.0,
            incomp: IncompressibilityMode = IncompressibilityMode()) -> L.FrgReg:
    return L.FrgReg(float(alpha), int(spec.order), int(bool(spec.seminorm)), L.INCOMP[incomp.mode],
                    float(incomp.beta))


def _dt(t: torch.Tensor) -> int:
    return L.dtype_code(t.dtype)


def _check_fd8(grid: Grid):
    for ni in grid.n:
        if ni < 9:
            raise ValueError(f"8th-order stencil needs n_i >= 9, got {ni}")


def fd8_gradient(u: ScalarField) -> VectorField:
    """diffops.py:98-106."""
    grid = u.grid
    _check_fd8(grid)
    out = torch.empty((grid.d, *grid.n), dtype=u.values.dtype, device="cuda")
    L.check(L.lib().frg_fd8_gradient(L.n3(grid.n), grid.d, _dt(u.values), 1, L.ptr(u.values), L.ptr(out),
                                     L.stream()), "fd8_gradient")
    return VectorField._wrap(grid, out)


def spectral_gradient(u: ScalarField) -> VectorField:
    """diffops.py:67-73."""
    grid = u.grid
    out = torch.empty((grid.d, *grid.n), dtype=u.values.dtype, device="cuda")
    L.check(L.lib().frg_spectral_gradient(L.n3(grid.n), grid.d, _dt(u.values), L.ptr(u.values), L.ptr(out),
                                          L.stream()), "spectral_gradient")
    return VectorField._wrap(grid, out)


def gradient(u: ScalarField, scheme: str = "fd8") -> VectorField:
    """diffops.py:109-114."""
    if scheme == "fd8":
        return fd8_gradient(u)
    if scheme == "spectral":
        return spectral_gradient(u)
    raise ValueError(f"unknown derivative scheme {scheme!r}")


def divergence(v: VectorField, scheme: str = "spectral") -> ScalarField:
    """diffops.py:117-129."""
    grid = v.grid
    out = torch.empty(grid.n, dtype=v.data.dtype, device="cuda")
    if scheme == "spectral":
        L.check(L.lib().frg_spectral_divergence(L.n3(grid.n), grid.d, _dt(v.data), L.ptr(v.data), L.ptr(out),
                                                L.stream()), "spectral_divergence")
    elif scheme == "fd8":
        _check_fd8(grid)
        L.check(L.lib().frg_fd8_divergence(L.n3(grid.n), grid.d, _dt(v.data), L.ptr(v.data), L.ptr(out),
                                           L.stream()), "fd8_divergence")
    else:
        raise ValueError(f"unknown derivative scheme {scheme!r}")
    return ScalarField._wrap(grid, out)


def jacobian(v: VectorField, scheme: str = "fd8") -> torch.Tensor:
    """diffops.py:132-139 — J[i, j] = d v_i / d x_j, shape (d, d, *n)."""
    grid = v.grid
    if scheme == "fd8":
        _check_fd8(grid)
        out = torch.empty((grid.d, grid.d, *grid.n), dtype=v.data.dtype, device="cuda")
        L.check(L.lib().frg_fd8_gradient(L.n3(grid.n), grid.d, _dt(v.data), grid.d, L.ptr(v.data), L.ptr(out),
                                         L.stream()), "jacobian")
        return out
    return torch.stack([gradient(ScalarField._wrap(grid, v.data[i].contiguous()), scheme).data
                        for i in range(grid.d)])


def _spectral(x: torch.Tensor, grid: Grid, ncomp: int, symbol: str, reg: L.FrgReg | None = None) -> torch.Tensor:
    out = torch.empty_like(x)
    L.check(L.lib().frg_spectral_apply(L.n3(grid.n), grid.d, _dt(x), ncomp, L.ptr(x), L.ptr(out), L.SYM[symbol],
                                       L.ctypes.byref(reg) if reg is not None else None, L.stream()), symbol)
    return out


def laplacian(u: ScalarField) -> ScalarField:
    """diffops.py:142-147."""
    return ScalarField._wrap(u.grid, _spectral(u.values, u.grid, 1, "laplacian"))


def reg_symbol(grid: Grid, spec: RegOperatorSpec) -> np.ndarray:
    """diffops.py:167-173 (host array, for inspection)."""
    freqs = np.meshgrid(*[np.fft.fftfreq(ni, d=1.0 / ni) for ni in grid.n], indexing="ij", sparse=True)
    ksq = np.broadcast_to(sum(f * f for f in freqs), grid.n)
    return ksq ** spec.order if spec.seminorm else (1.0 + ksq) ** spec.order


def apply_reg_operator(v: VectorField, spec: RegOperatorSpec, alpha: float) -> VectorField:
    """diffops.py:184-187."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    return VectorField._wrap(v.grid, _spectral(v.data, v.grid, v.grid.d, "reg", frg_reg(spec, alpha)))


def apply_inv_reg_operator(b: VectorField, spec: RegOperatorSpec, alpha: float) -> VectorField:
    """diffops.py:190-196."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    return VectorField._wrap(b.grid, _spectral(b.data, b.grid, b.grid.d, "reg_inv", frg_reg(spec, alpha)))


def apply_inv_sqrt_reg_operator(b: VectorField, spec: RegOperatorSpec, alpha: float) -> VectorField:
    """diffops.py:199-205."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    return VectorField._wrap(b.grid, _spectral(b.data, b.grid, b.grid.d, "reg_inv_sqrt", frg_reg(spec, alpha)))


def incompressibility_multiplier(ksq, mode: IncompressibilityMode, alpha: float) -> np.ndarray:
    """diffops.py:222-242 (host helper, exposed for auditing like the reference)."""
    ksq = np.asarray(ksq, dtype=np.float64)
    if mode.mode == "incompressible":
        return np.ones_like(ksq)
    if mode.mode == "near-incompressible":
        inner = mode.beta * (1.0 / ksq + 1.0)
        return 1.0 / (alpha / inner + 1.0)
    raise ValueError("no projection for mode 'none'")


def project_body_force(b: VectorField, mode: IncompressibilityMode, alpha: float) -> VectorField:
    """diffops.py:245-280."""
    if mode.mode == "none":
        return b.copy()
    out = torch.empty_like(b.data)
    reg = frg_reg(RegOperatorSpec(), alpha, mode)
    L.check(L.lib().frg_project(L.n3(b.grid.n), b.grid.d, _dt(b.data), L.ptr(b.data), L.ptr(out),
                                L.ctypes.byref(reg), L.stream()), "project")
    return VectorField._wrap(b.grid, out)


def low_pass_mask(grid: Grid) -> np.ndarray:
    """diffops.py:283-289 (host array)."""
    freqs = np.meshgrid(*[np.fft.fftfreq(ni, d=1.0 / ni) for ni in grid.n], indexing="ij", sparse=True)
    mask = np.ones(grid.n, dtype=bool)
    for i, f in enumerate(freqs):
        mask &= np.broadcast_to(np.abs(f) < grid.n[i] / 4, grid.n)
    return mask


def low_pass(u: ScalarField) -> ScalarField:
    return ScalarField._wrap(u.grid, _spectral(u.values, u.grid, 1, "lowpass"))


def high_pass(u: ScalarField) -> ScalarField:
    return ScalarField._wrap(u.grid, _spectral(u.values, u.grid, 1, "highpass"))


def low_pass_vector(v: VectorField) -> VectorField:
    return VectorField._wrap(v.grid, _spectral(v.data, v.grid, v.grid.d, "lowpass"))


def high_pass_vector(v: VectorField) -> VectorField:
    return VectorField._wrap(v.grid, _spectral(v.data, v.grid, v.grid.d, "highpass"))


def restrict(u: ScalarField) -> ScalarField:
    """diffops.py:312-326."""
    cg = u.grid.coarsen()
    out = torch.empty(cg.n, dtype=u.values.dtype, device="cuda")
    L.check(L.lib().frg_restrict(L.n3(u.grid.n), _dt(u.values), L.ptr(u.values), L.ptr(out), L.stream()), "restrict")
    return ScalarField._wrap(cg, out)


def prolong(u: ScalarField, fine_grid: Grid) -> ScalarField:
    """diffops.py:329-340."""
    if tuple(2 * ni for ni in u.grid.n) != fine_grid.n:
        raise ValueError("prolongation target must have exactly twice the resolution")
    out = torch.empty(fine_grid.n, dtype=u.values.dtype, device="cuda")
    L.check(L.lib().frg_prolong(L.n3(fine_grid.n), _dt(u.values), L.ptr(u.values), L.ptr(out), L.stream()),
            "prolong")
    return ScalarField._wrap(fine_grid, out)


def restrict_vector(v: VectorField) -> VectorField:
    return VectorField.from_components([restrict(ScalarField._wrap(v.grid, v.data[i].contiguous()))
                                        for i in range(v.grid.d)])


def prolong_vector(v: VectorField, fine_grid: Grid) -> VectorField:
    return VectorField.from_components([prolong(ScalarField._wrap(v.grid, v.data[i].contiguous()), fine_grid)
                                        for i in range(v.grid.d)])
