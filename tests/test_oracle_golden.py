"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/flowreg_oracle.py) is the checker for the CUDA path at
sizes beyond the fixtures; these tests prove it restates the reference.
"""
import numpy as np
import pytest

import inputs as I
from conftest import max_rel
from oracle import flowreg_oracle as O


@pytest.mark.parametrize("shape", I.SAMPLE_SHAPES)
def test_sample_matches_reference(golden, shape):
    g = golden("sample.npz")
    rng = np.random.default_rng(I.SEED)
    for s in I.SAMPLE_SHAPES:
        vals, q, labels = I.sample_inputs(s, rng)
        if s == shape:
            break
    t = f"{len(shape)}d"
    qs = [q[i] for i in range(len(shape))]
    for method in ("nearest", "linear", "cubic"):
        out = O.sample(vals, qs, method)
        assert np.array_equal(out, g[f"{t}_{method}_f64"]), method
        out32 = O.sample(vals.astype(np.float32), qs, method)
        assert out32.dtype == np.float32
        assert np.array_equal(out32, g[f"{t}_{method}_f32"]), method
        # the numpy twin restates the same arithmetic (order may differ)
        assert np.max(np.abs(O.sample_numpy(vals, qs, method) - out)) < 1e-12
    assert np.array_equal(O.sample(labels, qs, "nearest"), g[f"{t}_nearest_i32"])


def test_unknown_method_raises():
    with pytest.raises(ValueError):
        O.sample(np.zeros((8, 8)), [np.zeros(3), np.zeros(3)], "quintic")


def _diffops_inputs():
    rng = np.random.default_rng(I.SEED + 1)
    ins = {}
    for shape in I.DIFFOPS_SHAPES:
        ins[shape] = I.diffops_inputs(shape, rng)
    for shape in I.FILTER_SHAPES:
        ins[("f",) + shape] = I.filter_inputs(shape, rng)
    return ins


@pytest.mark.parametrize("shape", I.DIFFOPS_SHAPES)
def test_diffops_match_reference(golden, shape):
    g = golden("diffops.npz")
    u, v = _diffops_inputs()[shape]
    t = f"{len(shape)}d"
    tol = 1e-12
    assert max_rel(O.fd8_grad(u), g[f"{t}_fd8_grad"]) < tol
    assert max_rel(O.spectral_grad(u), g[f"{t}_spec_grad"]) < tol
    assert max_rel(O.divergence(v, "fd8"), g[f"{t}_div_fd8"]) < tol
    assert max_rel(O.divergence(v, "spectral"), g[f"{t}_div_spec"]) < tol
    assert max_rel(O.jacobian(v), g[f"{t}_jacobian"]) < tol
    assert max_rel(O.laplacian(u), g[f"{t}_laplacian"]) < tol
    for order, semi in I.REG_VARIANTS:
        k = f"{t}_o{order}{'s' if semi else 'f'}"
        assert max_rel(O.reg_apply(v, 0.03, order, semi), g[k + "_L"]) < tol
        assert max_rel(O.reg_inverse(v, 0.03, order, semi), g[k + "_Linv"]) < tol
        assert max_rel(O.reg_inv_sqrt(v, 0.03, order, semi), g[k + "_Linvsqrt"]) < tol
    assert max_rel(O.project(v, "incompressible", 1e-4, 0.01), g[f"{t}_proj_incomp"]) < tol
    assert max_rel(O.project(v, "near-incompressible", 1e-4, 0.01), g[f"{t}_proj_near"]) < tol


@pytest.mark.parametrize("shape", I.FILTER_SHAPES)
def test_filters_match_reference(golden, shape):
    g = golden("diffops.npz")
    u, uc = _diffops_inputs()[("f",) + shape]
    t = f"{len(shape)}d"
    assert max_rel(O.band_filter(u, True), g[f"{t}_lowpass"]) < 1e-12
    assert max_rel(O.band_filter(u, False), g[f"{t}_highpass"]) < 1e-12
    assert max_rel(O.restrict(u), g[f"{t}_restrict"]) < 1e-12
    assert max_rel(O.prolong(uc, shape), g[f"{t}_prolong"]) < 1e-12


@pytest.mark.parametrize("shape", I.TRANSPORT_SHAPES)
@pytest.mark.parametrize("method", ["cubic", "linear"])
def test_transport_matches_reference(golden, shape, method):
    g = golden("transport.npz")
    rng = np.random.default_rng(I.SEED + 2)
    for s in I.TRANSPORT_SHAPES:
        m0, v, vt, lam1 = I.transport_inputs(s, rng)
        if s == shape:
            break
    k = f"{I.transport_tag(shape)}_{method}"
    n_t = 4
    y = O.departure(v, 1.0 / n_t, method)
    yb = O.departure(-v, 1.0 / n_t, method)
    assert max_rel(y, g[k + "_y"]) < 1e-13
    assert max_rel(yb, g[k + "_yb"]) < 1e-13
    ms = O.solve_state(m0, y, n_t, method)
    assert max_rel(ms, g[k + "_state"]) < 1e-12
    divv = O.divergence(v, "fd8")
    assert max_rel(O.solve_adjoint(lam1, yb, divv, n_t, method), g[k + "_adjoint"]) < 1e-12
    grads = [O.fd8_grad(ms[j]) for j in range(n_t + 1)]
    assert max_rel(O.solve_inc_state(grads, y, vt, n_t, method)[-1], g[k + "_incstate"]) < 1e-12
    F = O.deformation_tensor(v, n_t, method)
    assert max_rel(O.determinant(F), g[k + "_det"]) < 1e-12
    assert max_rel(F[0, 0], g[k + "_F00"]) < 1e-12
    assert max_rel(O.compose_map(v, n_t, method), g[k + "_composed"]) < 1e-12


def _reg_of(regkw):
    return O.Reg(alpha=1e-2, order=regkw.get("order", 1), seminorm=regkw.get("seminorm", True),
                 incomp=regkw.get("incomp", "none"), beta=1e-4)


@pytest.mark.parametrize("case", I.KKT_CASES, ids=[c[0] for c in I.KKT_CASES])
def test_kkt_matches_reference(golden, case):
    g = golden("kkt.npz")
    meta = golden("kkt.json")
    rng = np.random.default_rng(I.SEED + 3)
    for c in I.KKT_CASES:
        ins = I.kkt_case_inputs(c, rng)
        if c[0] == case[0]:
            break
    name, shape, regkw, dist, method, preconds = case
    m0, m1, v, vt, r = ins
    st = O.Kkt(m0, m1, _reg_of(regkw), 4, dist, method, "fd8", v)
    p = name + "_"
    tol = 1e-11
    assert max_rel(st.mseries[-1], g[p + "m_final"]) < tol
    assert max_rel(st.lamseries[0], g[p + "lam0"]) < tol
    assert max_rel(st.gradient(), g[p + "gradient"]) < tol
    assert max_rel(st.hessian_matvec(vt), g[p + "matvec"]) < tol
    for kind in preconds:
        assert max_rel(st.apply_precond(r, kind, 0.3), g[p + "precond_" + kind]) < 1e-10, kind
    m = meta[name]
    assert st.objective() == pytest.approx(m["objective"], rel=1e-12)
    assert st.objective_at(v + 0.1 * vt) == pytest.approx(m["objective_at"], rel=1e-12)
    assert st.mismatch() == pytest.approx(m["mismatch"], rel=1e-12)
    assert st.divergence_energy() == pytest.approx(m["divergence_energy"], rel=1e-12, abs=1e-300)
    assert (st.matvecs, st.pde_solves, st.precond_fallbacks) == (
        m["matvecs"], m["pde_solves"], m["precond_fallbacks"])


def test_synth_matches_reference(golden):
    g = golden("synth.npz")
    for case in ("translation", "rotation", "swirl", "compress"):
        m0, m1, v = O.synth_case(case, 32, seed=2, d=2)
        assert max_rel(m0, g[f"{case}_m0"]) < 1e-13
        assert max_rel(v, g[f"{case}_v"]) < 1e-13
        assert max_rel(m1, g[f"{case}_m1"]) < 1e-11
    _, m1, _ = O.synth_case("rotation", 32, seed=1, d=3)
    assert max_rel(m1, g["rot3d_m1"]) < 1e-11
