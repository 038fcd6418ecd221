"""Semi-Lagrangian transport solvers on the device.

Mirrors flowreg.transport (/root/reference/pkg/src/flowreg/transport.py:1-247):
RK2 departure points, homogeneous state transport, the continuity-equation
adjoint (Heun with '+'), the linearised state, the GN incremental adjoint,
the deformation tensor and the composed map.  Departure maps are kept as
index-unit displacements on the device (see csrc/transport.cu); the physical
``step_points`` of the reference ``Trajectory`` are materialised on demand.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib as L
from .diffops import divergence, gradient, jacobian
from .fields import Grid, ScalarField, TensorField, TimeSeriesField, VectorField
from .interp import check_method

__all__ = [
    "Trajectory",
    "departure_points",
    "solve_state",
    "solve_adjoint",
    "solve_inc_state",
    "solve_inc_adjoint_gn",
    "solve_deformation_tensor",
    "compose_trajectory",
    "state_gradients",
]


def _dt(t: torch.Tensor) -> int:
    return L.dtype_code(t.dtype)


def departure_disp(v: VectorField, h_t: float, method: str = "cubic") -> torch.Tensor:
    """Index-unit displacement of the RK2 feet (transport.py:37-45)."""
    grid = v.grid
    disp = torch.empty_like(v.data)
    L.check(L.lib().frg_departure(L.n3(grid.n), grid.d, _dt(disp), _dt(v.data), L.METHODS[check_method(method)],
                                  float(h_t), L.ptr(v.data), L.ptr(disp), L.stream()), "departure")
    return disp


def _to_points(grid: Grid, disp: torch.Tensor) -> torch.Tensor:
    y = torch.empty_like(disp)
    L.check(L.lib().frg_disp_to_points(L.n3(grid.n), grid.d, _dt(disp), L.ptr(disp), L.ptr(y), L.stream()),
            "disp_to_points")
    return y


def _to_disp(grid: Grid, y: torch.Tensor) -> torch.Tensor:
    disp = torch.empty_like(y)
    L.check(L.lib().frg_points_to_disp(L.n3(grid.n), grid.d, _dt(y), L.ptr(y), L.ptr(disp), L.stream()),
            "points_to_disp")
    return disp


def departure_points(v: VectorField, h_t: float, method: str = "cubic") -> VectorField:
    """transport.py:37-45 — y = x - (h_t/2)(v(x) + v(x - h_t v(x)))."""
    return VectorField._wrap(v.grid, _to_points(v.grid, departure_disp(v, h_t, method)))


@dataclass
class Trajectory:
    """transport.py:48-62 — one-step departure map of a stationary velocity."""

    grid: Grid
    disp: torch.Tensor
    composed: VectorField | None = None
    _points: VectorField | None = field(default=None, repr=False)

    @classmethod
    def compute(cls, v: VectorField, method: str = "cubic") -> "Trajectory":
        return cls(v.grid, departure_disp(v, v.grid.h_t, method))

    @classmethod
    def from_points(cls, points: VectorField) -> "Trajectory":
        return cls(points.grid, _to_disp(points.grid, points.data), _points=points)

    @property
    def step_points(self) -> VectorField:
        if self._points is None:
            self._points = VectorField._wrap(self.grid, _to_points(self.grid, self.disp))
        return self._points


def _as(t: torch.Tensor, dtype: torch.dtype) -> torch.Tensor:
    """The kernels read every operand in the series' dtype: convert mixed-dtype
    operands (the reference accepts e.g. an f32 image with an f64 velocity)
    instead of handing an f64 buffer to an f32 kernel."""
    return t if t.dtype == dtype and t.is_contiguous() else t.to(dtype).contiguous()


def _negated(v: VectorField) -> VectorField:
    return VectorField._wrap(v.grid, -v.data)


def solve_state(m0: ScalarField, v: VectorField, method: str = "cubic",
                trajectory: Trajectory | None = None) -> TimeSeriesField:
    """transport.py:83-98."""
    grid = m0.grid
    method = check_method(method)
    if trajectory is None:
        trajectory = Trajectory.compute(v, method)
    out = torch.empty((grid.n_t + 1, *grid.n), dtype=m0.values.dtype, device="cuda")
    out[0] = m0.values
    disp = _as(trajectory.disp, out.dtype)
    L.check(L.lib().frg_solve_state(L.n3(grid.n), grid.d, _dt(out), L.METHODS[method], grid.n_t,
                                    L.ptr(disp), L.ptr(out), L.stream()), "solve_state")
    return TimeSeriesField._wrap(grid, out)


def solve_adjoint(final: ScalarField, v: VectorField, method: str = "cubic", scheme: str = "fd8",
                  back_trajectory: Trajectory | None = None, div_v: ScalarField | None = None) -> TimeSeriesField:
    """transport.py:105-135 — slices ordered by t, slice n_t = final."""
    grid = final.grid
    method = check_method(method)
    if back_trajectory is None:
        back_trajectory = Trajectory.compute(_negated(v), method)
    if div_v is None:
        div_v = divergence(v, scheme=scheme)
    out = torch.empty((grid.n_t + 1, *grid.n), dtype=final.values.dtype, device="cuda")
    out[grid.n_t] = final.values
    disp, dv = _as(back_trajectory.disp, out.dtype), _as(div_v.values, out.dtype)
    L.check(L.lib().frg_solve_adjoint(L.n3(grid.n), grid.d, _dt(out), L.METHODS[method], grid.n_t,
                                      L.ptr(disp), L.ptr(dv), L.ptr(out), L.stream()),
            "solve_adjoint")
    return TimeSeriesField._wrap(grid, out)


def state_gradients(mseries: TimeSeriesField, scheme: str = "fd8") -> list:
    """transport.py:138-144."""
    grid = mseries.grid
    if scheme == "fd8":
        out = torch.empty((mseries.num_slices, grid.d, *grid.n), dtype=mseries.data.dtype, device="cuda")
        L.check(L.lib().frg_fd8_gradient(L.n3(grid.n), grid.d, _dt(out), mseries.num_slices, L.ptr(mseries.data),
                                         L.ptr(out), L.stream()), "state_gradients")
        return [VectorField._wrap(grid, out[j]) for j in range(mseries.num_slices)]
    return [gradient(ScalarField._wrap(grid, mseries.data[j].contiguous()), scheme=scheme)
            for j in range(mseries.num_slices)]


def solve_inc_state(mseries: TimeSeriesField, v: VectorField, vtilde: VectorField, method: str = "cubic",
                    scheme: str = "fd8", trajectory: Trajectory | None = None,
                    grad_slices: list | None = None) -> TimeSeriesField:
    """transport.py:147-176."""
    grid = mseries.grid
    if mseries.grid != v.grid or v.grid != vtilde.grid:
        raise ValueError("state series and velocities live on different grids")
    method = check_method(method)
    if trajectory is None:
        trajectory = Trajectory.compute(v, method)
    if grad_slices is None:
        grad_slices = state_gradients(mseries, scheme)
    if len(grad_slices) != mseries.num_slices:
        raise ValueError("need one gradient slice per state slice")
    out = torch.empty((grid.n_t + 1, *grid.n), dtype=mseries.data.dtype, device="cuda")
    grads = torch.stack([g.data for g in grad_slices]).to(out.dtype).contiguous()
    disp = _as(trajectory.disp, out.dtype)
    L.check(L.lib().frg_solve_inc_state(L.n3(grid.n), grid.d, _dt(out), _dt(vtilde.data), L.METHODS[method],
                                        grid.n_t, L.ptr(disp), L.ptr(grads), L.ptr(vtilde.data),
                                        L.ptr(out), L.stream()), "solve_inc_state")
    return TimeSeriesField._wrap(grid, out)


def solve_inc_adjoint_gn(final: ScalarField, v: VectorField, method: str = "cubic", scheme: str = "fd8",
                         back_trajectory: Trajectory | None = None,
                         div_v: ScalarField | None = None) -> TimeSeriesField:
    """transport.py:179-194 — same continuity equation as the adjoint."""
    return solve_adjoint(final, v, method=method, scheme=scheme, back_trajectory=back_trajectory, div_v=div_v)


def solve_deformation_tensor(v: VectorField, method: str = "cubic", scheme: str = "fd8",
                             trajectory: Trajectory | None = None) -> TensorField:
    """transport.py:197-221."""
    grid = v.grid
    method = check_method(method)
    if trajectory is None:
        trajectory = Trajectory.compute(v, method)
    F = torch.empty((grid.d, grid.d, *grid.n), dtype=v.data.dtype, device="cuda")
    jac = _as(jacobian(v, scheme=scheme), F.dtype)
    disp = _as(trajectory.disp, F.dtype)
    L.check(L.lib().frg_deformation_tensor(L.n3(grid.n), grid.d, _dt(F), L.METHODS[method], grid.n_t,
                                           L.ptr(disp), L.ptr(jac), L.ptr(F), L.stream()),
            "deformation_tensor")
    return TensorField._wrap(grid, F)


def compose_trajectory(v: VectorField, method: str = "cubic", trajectory: Trajectory | None = None) -> VectorField:
    """transport.py:224-247 — per-step displacement composed n_t times."""
    grid = v.grid
    method = check_method(method)
    if trajectory is None:
        trajectory = Trajectory.compute(v, method)
    out = torch.empty_like(trajectory.disp)
    L.check(L.lib().frg_compose(L.n3(grid.n), grid.d, _dt(out), L.METHODS[method], grid.n_t, L.ptr(trajectory.disp),
                                L.ptr(out), L.stream()), "compose")
    trajectory.composed = VectorField._wrap(grid, _to_points(grid, out))
    return trajectory.composed
