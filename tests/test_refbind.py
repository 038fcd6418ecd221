"""The reference-side wide binding (paper_2401_17493_b200.refbind):
``flowreg.optimizer.KktState = refbind.KktState`` must accept the reference's
numpy containers (fields.py:160-205) and return the caller's own classes.

CPU: the conversions against the real reference classes (when /root/reference
is importable here) and the method surface the reference optimizer calls
(optimizer.py:92-281).  GPU: numpy stand-ins of the reference containers, a
PCG-Newton loop in numpy over the adapter, every returned vector identical to
the native device context driven the same way."""
import os
import sys
from dataclasses import dataclass, field

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"


def _import_reference():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    try:
        import flowreg  # noqa: F401
        import flowreg.kkt
        import flowreg.optimizer
    except Exception as e:  # pragma: no cover - missing numba etc.
        pytest.skip(f"reference not importable: {e}")
    return flowreg


def test_conversions_match_reference_classes():
    fr = _import_reference()
    from paper_2401_17493_b200 import refbind

    g = fr.fields.Grid((16, 12, 10), n_t=3, dtype=np.float32)
    dg = refbind._grid(g)
    assert dg.n == g.n and dg.n_t == g.n_t and dg.dtype == g.dtype
    reg = fr.kkt.RegConfig(alpha=3e-2, operator=fr.diffops.RegOperatorSpec(order=2, seminorm=False),
                           incomp=fr.diffops.IncompressibilityMode("near-incompressible", 2e-3))
    dr = refbind._reg(reg)
    assert (dr.alpha, dr.operator.order, dr.operator.seminorm, dr.incomp.mode, dr.incomp.beta) == \
        (3e-2, 2, False, "near-incompressible", 2e-3)
    p = refbind._precond(fr.kkt.PrecondKind("h0-two-level", 0.2, 7))
    assert (p.kind, p.inner_tol_factor, p.inner_max_iterations) == ("2level", 0.2, 7)


def test_adapter_covers_the_reference_state_surface():
    fr = _import_reference()
    from paper_2401_17493_b200 import refbind

    ref_public = {m for m in dir(fr.kkt.KktState) if not m.startswith("_")}
    ours = set(dir(refbind.KktState))
    assert ref_public <= ours
    # attributes register() / pcg_newton_step() read (optimizer.py:197-281)
    for a in ("matvecs", "pde_solves", "precond_fallbacks"):
        assert a in ours


# ---------------------------------------------------------------------------
# numpy stand-ins of the reference containers (fields.py:55-205 semantics)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Grid:
    n: tuple
    n_t: int = 4
    dtype: np.dtype = field(default=np.dtype(np.float64))

    @property
    def d(self):
        return len(self.n)


@dataclass
class ScalarField:
    grid: Grid
    values: np.ndarray


@dataclass
class VectorField:
    grid: Grid
    data: np.ndarray

    @classmethod
    def zeros(cls, grid):
        return cls(grid, np.zeros((grid.d, *grid.n), dtype=grid.dtype))


@dataclass(frozen=True)
class RegOperatorSpec:
    order: int = 1
    seminorm: bool = True


@dataclass(frozen=True)
class IncompressibilityMode:
    mode: str = "none"
    beta: float = 1e-4


@dataclass(frozen=True)
class RegConfig:
    alpha: float = 1e-2
    operator: RegOperatorSpec = field(default_factory=RegOperatorSpec)
    incomp: IncompressibilityMode = field(default_factory=lambda: IncompressibilityMode("near-incompressible", 1e-4))


@dataclass(frozen=True)
class PrecondKind:
    kind: str = "reg"
    inner_tol_factor: float = 0.1
    inner_max_iterations: int = 50


@pytest.mark.gpu
@pytest.mark.parametrize("tdt", [None, np.float32], ids=["f64", "mixed"])
def test_adapter_drives_a_numpy_newton_pcg_like_the_reference(tdt):
    import torch

    import paper_2401_17493_b200 as F
    from paper_2401_17493_b200 import refbind

    m0d, m1d, vtrue = F.synth_case("rotation", 32, seed=1, d=3)
    grid = Grid((32, 32, 32), n_t=4)
    m0 = ScalarField(grid, m0d.values.cpu().numpy())
    m1 = ScalarField(grid, m1d.values.cpu().numpy())
    reg = RegConfig(alpha=1e-2)
    pre = PrecondKind("2level")
    st = refbind.KktState(m0, m1, reg, method="cubic", scheme="fd8", transport_dtype=tdt)
    nat = F.KktState(m0d, m1d, F.RegConfig(alpha=1e-2), method="cubic", scheme="fd8", transport_dtype=tdt)
    assert isinstance(st.grid, Grid) and isinstance(st.v, VectorField)

    def same(ref_vec, dev_vec):
        assert isinstance(ref_vec, VectorField) and isinstance(ref_vec.data, np.ndarray)
        np.testing.assert_array_equal(ref_vec.data, dev_vec.data.cpu().numpy())

    for _ in range(2):  # two Newton steps, PCG in numpy on the adapter's results
        g = st.gradient()
        same(g, nat.gradient())
        assert st.objective() == nat.objective()
        r = VectorField(grid, -g.data)
        z = st.apply_precond(r, pre, 0.5)
        same(z, nat.apply_precond(F.VectorField._wrap(m0d.grid, torch.from_numpy(r.data).cuda()),
                                  F.PrecondKind("2level"), 0.5))
        s, vt = z, np.zeros_like(g.data)
        rz = float(np.sum(r.data * z.data))
        for _ in range(3):
            hs = st.hessian_matvec(s)
            same(hs, nat.hessian_matvec(F.VectorField._wrap(m0d.grid, torch.from_numpy(s.data).cuda())))
            kappa = rz / float(np.sum(s.data * hs.data))
            vt = vt + kappa * s.data
            r = VectorField(grid, r.data - kappa * hs.data)
            z = st.apply_precond(r, pre, 0.5)
            rz_new = float(np.sum(z.data * r.data))
            s = VectorField(grid, z.data + rz_new / rz * s.data)
            rz = rz_new
        v = VectorField(grid, st.v.data + 0.5 * vt)
        assert st.objective_at(v) == nat.objective_at(F.VectorField._wrap(m0d.grid, torch.from_numpy(v.data).cuda()))
        st.refresh(v)
        nat.refresh(F.VectorField._wrap(m0d.grid, torch.from_numpy(v.data).cuda()))
        assert st.mismatch() == nat.mismatch()
    assert (st.matvecs, st.pde_solves) == (nat.matvecs, nat.pde_solves)
    assert st.divergence_energy() == nat.divergence_energy()
