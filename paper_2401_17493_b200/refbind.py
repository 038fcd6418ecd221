"""Reference-side binding of the wide boundary.

``flowreg.optimizer.register`` instantiates ``KktState`` by name
(/root/reference/pkg/src/flowreg/optimizer.py:197) with the reference's own
numpy-backed containers (fields.py:160-205: ``ScalarField(grid, values)``,
``VectorField(grid, data)``, ``Grid(n, n_t, dtype)``) and then does its PCG /
Armijo vector algebra in numpy on what the state returns (optimizer.py:92-167).
This ``KktState`` accepts those containers by duck typing, runs every PDE solve
in one libflowreg_b200 context (``kkt.KktState``), and hands back objects of the
caller's own classes, so that

    import flowreg.optimizer, paper_2401_17493_b200.refbind as b200
    flowreg.optimizer.KktState = b200.KktState

swaps the hot path of an unmodified reference solve.  Per call the velocity-
space vector crosses PCIe once each way (that is the price of keeping the
reference's host-side vector algebra); transport state never leaves HBM.
``transport_dtype=np.float32`` selects the mixed-precision mode.
"""
from __future__ import annotations

import sys

import numpy as np
import torch

from . import kkt as _kkt
from .diffops import IncompressibilityMode, RegOperatorSpec
from .fields import Grid, ScalarField, VectorField

__all__ = ["KktState"]


def _grid(g) -> Grid:
    """Reference Grid (fields.py:55-80: ``n``, ``n_t``, ``dtype``) -> device Grid."""
    return Grid(tuple(int(x) for x in g.n), n_t=int(g.n_t), dtype=np.dtype(g.dtype))


def _reg(r) -> _kkt.RegConfig:
    """Reference RegConfig (kkt.py:56-68) -> device RegConfig (same fields)."""
    op = RegOperatorSpec(order=int(r.operator.order), seminorm=bool(r.operator.seminorm))
    inc = IncompressibilityMode(str(r.incomp.mode), float(r.incomp.beta))
    return _kkt.RegConfig(alpha=float(r.alpha), operator=op, incomp=inc)


def _precond(p) -> _kkt.PrecondKind:
    """Reference PrecondKind (kkt.py:80-92) -> device PrecondKind."""
    return _kkt.PrecondKind(str(p.kind), float(p.inner_tol_factor), int(p.inner_max_iterations))


def _dev(a: np.ndarray, dtype) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


class KktState:
    """Drop-in for flowreg.kkt.KktState over reference containers (kkt.py:136-341)."""

    def __init__(self, m0, m1, reg, distance: str = "ssd", method: str = "cubic", scheme: str = "fd8",
                 v_init=None, transport_dtype=None):
        if m0.grid != m1.grid:
            raise ValueError("images live on different grids")
        self.grid = m0.grid  # the caller's Grid: the optimizer builds VectorField(state.grid, ...)
        fields_mod = sys.modules[type(m0).__module__]
        self._Vec = getattr(fields_mod, "VectorField")
        self._dgrid = _grid(m0.grid)
        self._np_dtype = np.dtype(m0.grid.dtype)
        dm0 = ScalarField._wrap(self._dgrid, _dev(m0.values, self._np_dtype))
        dm1 = ScalarField._wrap(self._dgrid, _dev(m1.values, self._np_dtype))
        dv = None if v_init is None else self._to_dev(v_init)
        self._s = _kkt.KktState(dm0, dm1, _reg(reg), distance=distance, method=method, scheme=scheme, v_init=dv,
                                transport_dtype=transport_dtype)
        self.reg, self.distance, self.method, self.scheme = reg, distance, method, scheme
        self.m0, self.m1 = m0, m1
        self.v = v_init if v_init is not None else self._Vec.zeros(self.grid)

    # -- container conversion --------------------------------------------------
    def _to_dev(self, x) -> VectorField:
        if x.grid != self.grid:
            raise ValueError("velocity lives on a different grid")
        return VectorField._wrap(self._dgrid, _dev(x.data, self._np_dtype))

    def _to_ref(self, x: VectorField):
        return self._Vec(self.grid, x.data.cpu().numpy())

    # -- counters (kkt.py:158-160) --------------------------------------------
    matvecs = property(lambda s: s._s.matvecs, lambda s, x: setattr(s._s, "matvecs", x))
    pde_solves = property(lambda s: s._s.pde_solves, lambda s, x: setattr(s._s, "pde_solves", x))
    precond_fallbacks = property(lambda s: s._s.precond_fallbacks,
                                 lambda s, x: setattr(s._s, "precond_fallbacks", x))

    @property
    def initial_mismatch(self) -> float:
        return self._s.initial_mismatch

    # -- kkt.py:166-265 ---------------------------------------------------------
    def refresh(self, v) -> None:
        self._s.refresh(self._to_dev(v))
        self.v = v

    def objective(self) -> float:
        return self._s.objective()

    def objective_at(self, v_trial) -> float:
        return self._s.objective_at(self._to_dev(v_trial))

    def mismatch(self) -> float:
        return self._s.mismatch()

    def divergence_energy(self) -> float:
        return self._s.divergence_energy()

    def gradient(self):
        return self._to_ref(self._s.gradient())

    def hessian_matvec(self, vtilde):
        return self._to_ref(self._s.hessian_matvec(self._to_dev(vtilde)))

    def apply_precond(self, r, kind, outer_tol: float):
        return self._to_ref(self._s.apply_precond(self._to_dev(r), _precond(kind), outer_tol))

    def deformed_image(self):
        fields_mod = sys.modules[type(self.m0).__module__]
        return getattr(fields_mod, "ScalarField")(self.grid, self._s.deformed_image().values.cpu().numpy())
