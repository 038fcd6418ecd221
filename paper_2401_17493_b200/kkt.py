"""Reduced-space objective, gradient, Gauss-Newton matvec, preconditioners.

The wide drop-in boundary: ``KktState`` has the constructor, attributes and
methods of flowreg.kkt.KktState (/root/reference/pkg/src/flowreg/kkt.py:
136-341) and the same counters (+2 PDE solves per refresh / matvec, +1 per
objective_at).  All state lives in one libflowreg_b200 context in HBM; every
method is a single C-ABI call.

Extra keyword ``transport_dtype`` (default: the grid dtype) selects the
storage of the transport fields; velocity-space vectors always use the grid
dtype.  ``KktState(..., transport_dtype=np.float32)`` on an f64 grid is the
mixed-precision mode of SURVEY.md §7 hard part 1.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .diffops import IncompressibilityMode, RegOperatorSpec, frg_reg
from .fields import Grid, ScalarField, TimeSeriesField, VectorField
from .interp import check_method
from .transport import Trajectory

__all__ = ["RegConfig", "PrecondKind", "KktState", "evaluate_objective", "evaluate_gradient",
           "hessian_matvec_gn", "apply_precond", "release_device_pool"]


@dataclass(frozen=True)
class RegConfig:
    """kkt.py:56-68."""

    alpha: float = 1e-2
    operator: RegOperatorSpec = field(default_factory=RegOperatorSpec)
    incomp: IncompressibilityMode = field(default_factory=lambda: IncompressibilityMode("near-incompressible", 1e-4))

    def __post_init__(self):
        if self.alpha <= 0:
            raise ValueError("alpha must be positive")


_PRECOND_ALIASES = {"reg": "reg", "regularization": "reg", "h0": "h0", "2level": "2level", "h0-two-level": "2level"}


@dataclass(frozen=True)
class PrecondKind:
    """kkt.py:80-92."""

    kind: str = "2level"
    inner_tol_factor: float = 0.1
    inner_max_iterations: int = 50

    def __post_init__(self):
        k = _PRECOND_ALIASES.get(self.kind)
        if k is None:
            raise ValueError(f"unknown preconditioner {self.kind!r}")
        object.__setattr__(self, "kind", k)


class KktState:
    """Velocity iterate plus every PDE byproduct needed by the optimizer (kkt.py:136-265)."""

    def __init__(self, m0: ScalarField, m1: ScalarField, reg: RegConfig, distance: str = "ssd",
                 method: str = "cubic", scheme: str = "fd8", v_init: VectorField | None = None,
                 transport_dtype=None, interp_precision: str = "fp32"):
        """``interp_precision="fp16"`` selects the north star's mixed-precision
        interpolation mode: the SL steps of the GN Hessian matvec gather fp16
        taps (fp32 weights / accumulation; tolerance 1e-3), state / adjoint /
        gradient stay fp32; needs fp32 transport."""
        if interp_precision not in ("fp32", "fp16"):
            raise ValueError(f"unknown interpolation precision {interp_precision!r}")
        if m0.grid != m1.grid:
            raise ValueError("images live on different grids")
        if distance not in L.DISTANCES:
            raise ValueError(f"unknown distance measure {distance!r}")
        if scheme not in L.SCHEMES:
            raise ValueError(f"unknown derivative scheme {scheme!r}")
        method = check_method(method)
        self.grid: Grid = m0.grid
        self.m0, self.m1 = m0, m1
        self.reg, self.distance, self.method, self.scheme = reg, distance, method, scheme
        grid = self.grid
        if scheme == "fd8":
            for ni in grid.n:
                if ni < 9:
                    raise ValueError(f"8th-order stencil needs n_i >= 9, got {ni}")
        cdt = L.dtype_code(grid.dtype)
        tdt = cdt if transport_dtype is None else L.dtype_code(np.dtype(transport_dtype))
        self.transport_dtype = torch.float64 if tdt == L.F64 else torch.float32
        cfg = L.FrgConfig()
        n = (1,) + grid.n if grid.d == 2 else grid.n
        cfg.n = (ctypes.c_int32 * 3)(*n)
        cfg.d, cfg.n_t = grid.d, grid.n_t
        cfg.method, cfg.scheme, cfg.distance = L.METHODS[method], L.SCHEMES[scheme], L.DISTANCES[distance]
        cfg.transport_dtype, cfg.control_dtype = tdt, cdt
        cfg.reg = frg_reg(reg.operator, reg.alpha, reg.incomp)
        L.require_cuda()
        h = ctypes.c_void_p()
        L.check(L.lib().frg_kkt_create(ctypes.byref(cfg), L.stream(), ctypes.byref(h)), "kkt_create")
        self._h = h
        self.interp_precision = interp_precision
        if interp_precision == "fp16":
            L.check(L.lib().frg_kkt_set_interp_precision(h, 16), "kkt_set_interp_precision")
        L.check(L.lib().frg_kkt_set_images(h, L.ptr(m0.values), L.ptr(m1.values), cdt), "kkt_set_images")
        self.refresh(v_init if v_init is not None else VectorField.zeros(grid))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and L._lib is not None:
            try:
                L.lib().frg_kkt_destroy(h)
            except Exception:
                pass
            self._h = None

    def _call(self, name, *args):
        fn = getattr(L.lib(), name)
        L.check(fn(self._h, *args), name)

    def _vec(self, x: VectorField) -> torch.Tensor:
        if x.grid != self.grid:
            raise ValueError("velocity lives on a different grid")
        return x.data.contiguous()

    def _new(self) -> torch.Tensor:
        return torch.empty((self.grid.d, *self.grid.n), dtype=self.grid.torch_dtype, device="cuda")

    # -- counters (kkt.py:158-160) -----------------------------------------
    def _counters(self):
        c = (ctypes.c_int64 * 3)()
        self._call("frg_kkt_counters", c)
        return list(c)

    def _set_counter(self, i, value):
        c = self._counters()
        c[i] = int(value)
        self._call("frg_kkt_set_counters", (ctypes.c_int64 * 3)(*c))

    matvecs = property(lambda s: s._counters()[0], lambda s, x: s._set_counter(0, x))
    pde_solves = property(lambda s: s._counters()[1], lambda s, x: s._set_counter(1, x))
    precond_fallbacks = property(lambda s: s._counters()[2], lambda s, x: s._set_counter(2, x))

    @property
    def initial_mismatch(self) -> float:
        out = ctypes.c_double()
        self._call("frg_kkt_initial_mismatch", ctypes.byref(out))
        return out.value

    # -- state management (kkt.py:166-187) ----------------------------------
    def refresh(self, v: VectorField) -> None:
        vd = self._vec(v)
        self._call("frg_kkt_refresh", L.ptr(vd))
        self.v = v

    def _get(self, which, shape) -> torch.Tensor:
        out = torch.empty(shape, dtype=self.transport_dtype, device="cuda")
        self._call("frg_kkt_get", which, L.ptr(out))
        return out.to(self.grid.torch_dtype)

    @property
    def mseries(self) -> TimeSeriesField:
        return TimeSeriesField._wrap(self.grid, self._get(0, (self.grid.n_t + 1, *self.grid.n)))

    @property
    def lamseries(self) -> TimeSeriesField:
        return TimeSeriesField._wrap(self.grid, self._get(1, (self.grid.n_t + 1, *self.grid.n)))

    @property
    def trajectory(self) -> Trajectory:
        return Trajectory(self.grid, self._get(2, (self.grid.d, *self.grid.n)))

    @property
    def back_trajectory(self) -> Trajectory:
        return Trajectory(self.grid, self._get(3, (self.grid.d, *self.grid.n)))

    @property
    def div_v(self) -> ScalarField:
        return ScalarField._wrap(self.grid, self._get(4, self.grid.n))

    @property
    def grad_slices(self) -> list:
        g = self._get(5, (self.grid.n_t + 1, self.grid.d, *self.grid.n))
        return [VectorField._wrap(self.grid, g[j]) for j in range(self.grid.n_t + 1)]

    def deformed_image(self) -> ScalarField:
        return self.mseries.final()

    # -- objective / gradient / matvec (kkt.py:194-265) ---------------------
    def objective(self) -> float:
        out = ctypes.c_double()
        self._call("frg_kkt_objective", ctypes.byref(out))
        return out.value

    def objective_at(self, v_trial: VectorField) -> float:
        out = ctypes.c_double()
        self._call("frg_kkt_objective_at", L.ptr(self._vec(v_trial)), ctypes.byref(out))
        return out.value

    def divergence_energy(self) -> float:
        out = ctypes.c_double()
        self._call("frg_kkt_divergence_energy", ctypes.byref(out))
        return out.value

    def gradient(self) -> VectorField:
        out = self._new()
        self._call("frg_kkt_gradient", L.ptr(out))
        return VectorField._wrap(self.grid, out)

    def hessian_matvec(self, vtilde: VectorField, out: torch.Tensor | None = None) -> VectorField:
        """Gauss-Newton Hessian action; two PDE solves per call (kkt.py:237-260).

        ``vtilde`` may also be a HOST tensor (pinned, shape (d, *n)) with a
        host ``out``: then the call is asynchronous and pipelined — the
        host->device copy of call k+1 and the device->host copy of call k-1
        overlap the device work of call k (two staging slots, dedicated copy
        streams); ``out`` holds the result once the caller synchronises
        (``torch.cuda.synchronize()`` or ``wait_host_io()``)."""
        data = vtilde.data if hasattr(vtilde, "data") else vtilde
        if isinstance(data, torch.Tensor) and data.device.type == "cpu":
            return self._hessian_matvec_host(data, out)
        out = self._new() if out is None else out
        self._call("frg_kkt_hessian_matvec", L.ptr(self._vec(vtilde)), L.ptr(out))
        return VectorField._wrap(self.grid, out)

    def _hessian_matvec_host(self, host_in: torch.Tensor, host_out: torch.Tensor | None) -> VectorField:
        shape = (self.grid.d, *self.grid.n)
        if tuple(host_in.shape) != shape or host_in.dtype != self.grid.torch_dtype:
            raise ValueError(f"host v~ must be {shape} {self.grid.torch_dtype}")
        if host_out is None:
            host_out = torch.empty(shape, dtype=host_in.dtype).pin_memory()
        io = getattr(self, "_io", None)
        if io is None:
            io = self._io = {"h2d": torch.cuda.Stream(), "d2h": torch.cuda.Stream(), "k": 0,
                             "in": [self._new(), self._new()], "out": [self._new(), self._new()],
                             "ev_in": [torch.cuda.Event(), torch.cuda.Event()],
                             "ev_comp": [torch.cuda.Event(), torch.cuda.Event()],
                             "ev_out": [torch.cuda.Event(), torch.cuda.Event()], "used": [False, False]}
        s = io["k"] & 1
        io["k"] += 1
        cur = torch.cuda.current_stream()
        self._call("frg_kkt_set_stream", ctypes.c_void_p(cur.cuda_stream))
        with torch.cuda.stream(io["h2d"]):
            if io["used"][s]:
                io["h2d"].wait_event(io["ev_comp"][s])  # slot's previous matvec has consumed its input
            io["in"][s].copy_(host_in, non_blocking=True)
            io["ev_in"][s].record(io["h2d"])
        cur.wait_event(io["ev_in"][s])
        if io["used"][s]:
            cur.wait_event(io["ev_out"][s])  # slot's previous result has left the device
        self._call("frg_kkt_hessian_matvec", L.ptr(io["in"][s]), L.ptr(io["out"][s]))
        io["ev_comp"][s].record(cur)
        with torch.cuda.stream(io["d2h"]):
            io["d2h"].wait_event(io["ev_comp"][s])
            host_out.copy_(io["out"][s], non_blocking=True)
            io["ev_out"][s].record(io["d2h"])
        io["used"][s] = True
        return VectorField._wrap(self.grid, host_out)

    def wait_host_io(self) -> None:
        """Make the current stream wait for every pending host-I/O matvec copy."""
        io = getattr(self, "_io", None)
        if io is not None:
            torch.cuda.current_stream().wait_stream(io["d2h"])

    def mismatch(self) -> float:
        out = ctypes.c_double()
        self._call("frg_kkt_mismatch", ctypes.byref(out))
        return out.value

    # -- preconditioners (kkt.py:308-341) ----------------------------------
    def apply_precond(self, r: VectorField, kind: PrecondKind, outer_tol: float,
                      out: torch.Tensor | None = None) -> VectorField:
        out = self._new() if out is None else out
        fb = ctypes.c_int32(0)
        self._call("frg_kkt_apply_precond", L.PRECOND[kind.kind], float(outer_tol), float(kind.inner_tol_factor),
                   int(kind.inner_max_iterations), L.ptr(self._vec(r)), L.ptr(out), ctypes.byref(fb))
        return VectorField._wrap(self.grid, out)

    def detgrad_stats(self):
        out = (ctypes.c_double * 3)()
        self._call("frg_kkt_detgrad", out)
        return float(out[0]), float(out[1]), float(out[2])


# -- functional aliases (kkt.py:347-364) --------------------------------------


def evaluate_objective(state: KktState, v: VectorField | None = None) -> float:
    if v is None:
        return state.objective()
    return state.objective_at(v)


def evaluate_gradient(state: KktState) -> VectorField:
    return state.gradient()


def hessian_matvec_gn(state: KktState, vtilde: VectorField) -> VectorField:
    return state.hessian_matvec(vtilde)


def apply_precond(r: VectorField, kind: PrecondKind, state: KktState, outer_tol: float = 1e-6) -> VectorField:
    return state.apply_precond(r, kind, outer_tol)


def release_device_pool() -> None:
    """Free the device buffers destroyed contexts parked for reuse (the torch
    caching allocator cannot reclaim them; call before large torch
    allocations after a big solve)."""
    torch.cuda.synchronize()
    L.check(L.lib().frg_release_pool(), "release_pool")
