"""Property tests of the device operators, restating the reference's own
behavioural suite for differential operators, interpolation, distances,
field containers and the alpha continuation (pkg/tests/test_diffops.py,
test_interp.py, test_distance.py, test_fields.py, test_continuation.py of the
reference package) in this repo's words.  Spectral / FD8 / sampling kernels
run on 2D f64 grids at the reference's tolerances and, where the kernel path
differs, on 3D fp32 grids with fp32 tolerances.
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU collection
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2401_17493_b200 as F  # noqa: E402
from paper_2401_17493_b200 import distance as Dm  # noqa: E402
from paper_2401_17493_b200.continuation import cascade_alphas  # noqa: E402
from paper_2401_17493_b200.diffops import (  # noqa: E402
    apply_inv_reg_operator,
    apply_inv_sqrt_reg_operator,
    apply_reg_operator,
    divergence,
    fd8_gradient,
    gradient,
    high_pass,
    incompressibility_multiplier,
    laplacian,
    low_pass,
    project_body_force,
    prolong,
    restrict,
    spectral_gradient,
)


def _x(g):
    return [np.broadcast_to(c, g.n).astype(np.float64) for c in g.coord_arrays()]


def _np(x):
    if isinstance(x, F.ScalarField):
        x = x.values
    return (x.data if hasattr(x, "data") else x).double().cpu().numpy()


def S(g, a):
    return F.ScalarField(g, np.ascontiguousarray(a, dtype=g.dtype))


def V(g, comps):
    return F.VectorField(g, np.ascontiguousarray(np.stack(comps), dtype=g.dtype))


def noise(g, rng):
    return S(g, rng.standard_normal(g.n))


def noise_v(g, rng):
    return F.VectorField(g, rng.standard_normal((g.d, *g.n)).astype(g.dtype))


def smooth_v(g, rng, kmax=3, modes=6):
    data = np.zeros((g.d, *g.n))
    for i in range(g.d):
        spec = np.zeros(g.n, dtype=complex)
        for _ in range(modes):
            spec[tuple(int(rng.integers(0, kmax + 1)) for _ in range(g.d))] = rng.standard_normal() + 1j
        data[i] = np.fft.ifftn(spec).real * g.num_voxels
    return F.VectorField(g, data.astype(g.dtype))


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


G2 = F.Grid((16, 16))
G3F = F.Grid((16, 16, 64), dtype=np.float32)

# ---------------------------------------------------------------------------
# gradients, divergence (reference diffops.py:56-147)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("g,tol", [(G2, 1e-12), (G3F, 2e-5)])
def test_spectral_gradient_of_a_mode(g, tol):
    x = _x(g)
    ph = 2 * x[0] + x[1] + (x[2] if g.d == 3 else 0.0)
    got = _np(spectral_gradient(S(g, np.sin(ph))))
    k = (2, 1, 1)[: g.d]
    for i in range(g.d):
        assert np.max(np.abs(got[i] - k[i] * np.cos(ph))) < tol


@pytest.mark.parametrize("g", [G2, G3F])
def test_constant_has_zero_gradient(g):
    c = F.ScalarField.full(g, 1.7)
    assert float(fd8_gradient(c).data.abs().max()) == 0.0  # antisymmetric stencil: exact
    assert np.max(np.abs(_np(spectral_gradient(c)))) < (1e-13 if g.dtype == np.float64 else 1e-5)


@pytest.mark.parametrize("g", [G2, G3F])
def test_fd8_axis_independence(g):
    x = _x(g)
    got = _np(fd8_gradient(S(g, np.sin(x[0]) + 0.0 * x[-1])))
    for i in range(1, g.d):
        assert np.max(np.abs(got[i])) == 0.0


def test_fd8_observed_order_at_least_seven():
    errs = []
    for n in (32, 64):
        g = F.Grid((n, n))
        x = _x(g)
        got = _np(fd8_gradient(S(g, np.sin(x[0]))))[0]
        errs.append(np.max(np.abs(got - np.cos(x[0]))))
    assert errs[0] / errs[1] >= 2 ** 7


def test_fd8_rejects_grids_below_the_stencil():
    g = F.Grid((8, 16))
    with pytest.raises(ValueError):
        gradient(F.ScalarField.zeros(g), scheme="fd8")


@pytest.mark.parametrize("g,tol", [(G2, 1e-10), (G3F, 1e-4)])
def test_divergence_of_gradient_is_laplacian_on_a_mode(g, tol):
    x = _x(g)
    ph = 2 * x[0] + 3 * x[1]
    u = S(g, np.cos(ph))
    div = _np(divergence(spectral_gradient(u), scheme="spectral"))
    assert np.max(np.abs(div + 13.0 * np.cos(ph))) < tol * 13
    assert np.max(np.abs(_np(laplacian(u)) + 13.0 * np.cos(ph))) < tol * 13


def test_divergence_free_and_zero_fields():
    g = F.Grid((32, 32))
    x = _x(g)
    v = V(g, [-np.cos(x[0]) * np.sin(x[1]), np.sin(x[0]) * np.cos(x[1])])
    assert np.max(np.abs(_np(divergence(v, scheme="spectral")))) < 1e-12
    assert np.max(np.abs(_np(divergence(v, scheme="fd8")))) < 1e-6
    assert float(divergence(F.VectorField.zeros(g)).values.abs().max()) == 0.0


def test_spectral_divergence_is_minus_adjoint_of_gradient(rng):
    g = F.Grid((16, 16))
    u, v = noise(g, rng), noise_v(g, rng)
    lhs = F.l2_inner(spectral_gradient(u), v)
    rhs = -F.l2_inner(u, divergence(v, scheme="spectral"))
    assert lhs == pytest.approx(rhs, rel=1e-11, abs=1e-11)


# ---------------------------------------------------------------------------
# regularisation operator (reference diffops.py:150-205)
# ---------------------------------------------------------------------------


def test_unit_mode_is_a_fixed_point_and_constants_are_its_kernel():
    x = _x(G2)
    v = V(G2, [np.sin(x[0]), np.zeros(G2.n)])
    assert np.max(np.abs(_np(apply_reg_operator(v, F.RegOperatorSpec(), 1.0)) - _np(v))) < 1e-12
    c = F.VectorField.constant(G2, (2.0, -1.0))
    assert np.max(np.abs(_np(apply_reg_operator(c, F.RegOperatorSpec(), 3.0)))) < 1e-13


@pytest.mark.parametrize("order", [2, 3])
def test_higher_order_symbol_on_a_mixed_mode(order):
    g = F.Grid((32, 32))
    x = _x(g)
    u = np.cos(2 * x[0] + 3 * x[1])
    v = V(g, [u, np.zeros(g.n)])
    got = _np(apply_reg_operator(v, F.RegOperatorSpec(order), 0.5))[0]
    want = 0.5 * 13.0 ** order * u
    # the FFT's ~1e-16 roundoff in the empty high bins is amplified by
    # alpha |k|^(2 order) (|k|^2 <= 512 here): ~1e-11 relative for H3
    assert np.max(np.abs(got - want)) < (1e-12 if order == 2 else 1e-10) * np.max(np.abs(want))


@pytest.mark.parametrize("g,tol", [(G2, 1e-10), (G3F, 1e-4)])
def test_inverse_pair_off_the_kernel(g, tol, rng):
    w = smooth_v(g, rng)
    w = F.VectorField._wrap(g, w.data - w.data.mean(dim=tuple(range(1, g.d + 1)), keepdim=True))
    back = apply_inv_reg_operator(apply_reg_operator(w, F.RegOperatorSpec(), 1e-2), F.RegOperatorSpec(), 1e-2)
    assert np.max(np.abs(_np(back) - _np(w))) < tol


def test_inverse_divides_constants_by_alpha_and_scales_modes():
    b = F.VectorField.constant(G2, (1.0, 2.0))
    out = _np(apply_inv_reg_operator(b, F.RegOperatorSpec(), 0.25))
    assert np.allclose(out[0], 4.0, rtol=1e-13) and np.allclose(out[1], 8.0, rtol=1e-13)
    x = _x(G2)
    u = np.sin(2 * x[0])
    got = _np(apply_inv_reg_operator(V(G2, [u, np.zeros(G2.n)]), F.RegOperatorSpec(), 0.1))[0]
    assert np.max(np.abs(got - u / 0.4)) < 1e-12


def test_reg_operator_self_adjoint_positive_and_inverse_square_root(rng):
    spec = F.RegOperatorSpec()
    a, b = noise_v(G2, rng), noise_v(G2, rng)
    la, lb = apply_reg_operator(a, spec, 0.3), apply_reg_operator(b, spec, 0.3)
    assert F.l2_inner(la, b) == pytest.approx(F.l2_inner(a, lb), rel=1e-12)
    assert F.l2_inner(la, a) > 0
    twice = apply_inv_sqrt_reg_operator(apply_inv_sqrt_reg_operator(a, spec, 0.3), spec, 0.3)
    once = apply_inv_reg_operator(a, spec, 0.3)
    assert np.max(np.abs(_np(twice) - _np(once))) < 1e-12 * np.max(np.abs(_np(once)))


# ---------------------------------------------------------------------------
# projections (reference diffops.py:208-280)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("g,tol", [(F.Grid((16, 16, 16)), 1e-12), (G3F, 2e-5)])
def test_leray_kills_gradients_keeps_curls_and_is_idempotent(g, tol):
    x = _x(g)
    p = np.cos(x[0] + 2 * x[1]) * np.cos(x[2])
    grad = spectral_gradient(S(g, p))
    inc = F.IncompressibilityMode("incompressible")
    assert np.max(np.abs(_np(project_body_force(grad, inc, 1.0)))) < tol * np.max(np.abs(_np(grad)))
    curl = V(g, [-np.cos(x[0]) * np.sin(x[1]), np.sin(x[0]) * np.cos(x[1]), np.zeros(g.n)])
    once = project_body_force(curl, inc, 1.0)
    assert np.max(np.abs(_np(once) - _np(curl))) < tol
    twice = project_body_force(once, inc, 1.0)
    assert np.max(np.abs(_np(twice) - _np(once))) < tol
    assert np.max(np.abs(_np(divergence(once, scheme="spectral")))) < 10 * tol


def test_relaxed_projection_matches_the_scalar_chain_on_one_wavenumber():
    g = F.Grid((32, 32))
    x = _x(g)
    alpha, beta = 1e-2, 1e-4
    b = spectral_gradient(S(g, np.cos(2 * x[0] + x[1])))  # longitudinal mode |k|^2 = 5
    out = _np(project_body_force(b, F.IncompressibilityMode("near-incompressible", beta), alpha))
    mult = 1.0 / (alpha / (beta * (1.0 / 5.0 + 1.0)) + 1.0)
    want = (1.0 - mult) * _np(b)
    assert np.max(np.abs(out - want)) < 1e-12 * max(1.0, np.max(np.abs(want)))


def test_multiplier_limits():
    m = incompressibility_multiplier(1.0, F.IncompressibilityMode("near-incompressible", 1e-4), 1e-2)
    assert 0.0 < m < 1.0
    heavy = F.IncompressibilityMode("near-incompressible", 1e6)
    assert incompressibility_multiplier(4.0, heavy, 1e-2) == pytest.approx(1.0, abs=1e-6)


def test_reg_operator_and_projection_are_linear(rng):
    a, b = noise_v(G2, rng), noise_v(G2, rng)
    ab = F.VectorField._wrap(G2, 2.0 * a.data - 3.0 * b.data)
    for op in (lambda v: apply_reg_operator(v, F.RegOperatorSpec(), 0.1),
               lambda v: project_body_force(v, F.IncompressibilityMode("near-incompressible", 1e-3), 0.1)):
        lhs = _np(op(ab))
        rhs = 2.0 * _np(op(a)) - 3.0 * _np(op(b))
        assert np.max(np.abs(lhs - rhs)) < 1e-11 * max(1.0, np.max(np.abs(rhs)))


# ---------------------------------------------------------------------------
# band filters and grid transfer (reference diffops.py:283-366)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("g", [G2, F.Grid((16, 16, 16))])
def test_band_filters_partition_the_spectrum(g, rng):
    u = noise(g, rng)
    lo, hi = _np(low_pass(u)), _np(high_pass(u))
    assert np.max(np.abs(lo + hi - _np(u.values))) < 1e-13
    assert abs(F.l2_inner(low_pass(u), high_pass(u))) < 1e-10
    assert np.max(np.abs(_np(high_pass(F.ScalarField._wrap(g, low_pass(u).values))))) < 1e-13


@pytest.mark.parametrize("g", [G2, F.Grid((16, 16, 16))])
def test_prolong_restrict_reproduce_bandlimited_fields(g):
    x = _x(g)
    u = S(g, np.cos(x[0] + 2 * x[1]) + 0.5 * np.sin(3 * x[-1]))
    back = prolong(restrict(u), g)
    assert np.max(np.abs(_np(back) - _np(u.values))) < 1e-12


def test_restriction_and_prolongation_are_an_adjoint_pair(rng):
    g = F.Grid((16, 16))
    gc = g.coarsen()
    u, w = noise(g, rng), noise(gc, rng)
    assert F.l2_inner(restrict(u), w) == pytest.approx(F.l2_inner(u, prolong(w, g)), rel=1e-12, abs=1e-12)


def test_nyquist_band_restricts_to_zero():
    g = F.Grid((16, 16))
    x = _x(g)
    u = S(g, np.cos(4 * x[0]))  # |k| = n/4: outside the coarse grid's retained band
    assert np.max(np.abs(_np(restrict(u)))) < 1e-13


# ---------------------------------------------------------------------------
# sampling (reference interp.py / _kernels.py:222-251)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("method", ["nearest", "linear", "cubic"])
@pytest.mark.parametrize("shape,dt", [((12, 10), torch.float64), ((12, 16, 64), torch.float32)])
def test_nodes_reproduce_values(method, shape, dt, rng):
    vals = torch.as_tensor(rng.standard_normal(shape), dtype=dt, device="cuda")
    idx = np.stack(np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")).reshape(len(shape), -1)
    out = F.sample_nd(vals, [torch.as_tensor(i, dtype=torch.float64) for i in idx], method)
    assert torch.equal(out.reshape(shape), vals)


def test_linear_axis_midpoint_is_the_mean(rng):
    vals = rng.standard_normal((10, 12))
    q0 = np.arange(10) + 0.5
    q1 = np.full(10, 3.0)
    out = F.sample_nd(vals, [q0, q1], "linear")
    want = 0.5 * (vals[:, 3] + np.roll(vals[:, 3], -1))
    assert np.max(np.abs(out - want)) < 1e-15


def test_cubic_fourth_order_against_analytic():
    errs = []
    rng = np.random.default_rng(3)
    pts = rng.uniform(0, 1, size=(2, 400))
    for n in (32, 64):
        i = np.arange(n)
        x0, x1 = np.meshgrid(2 * np.pi * i / n, 2 * np.pi * i / n, indexing="ij")
        f = np.sin(x0) * np.cos(2 * x1)
        q = pts * n
        out = F.sample_nd(f, [q[0], q[1]], "cubic")
        want = np.sin(2 * np.pi * pts[0]) * np.cos(4 * np.pi * pts[1])
        errs.append(np.max(np.abs(out - want)))
    assert math.log2(errs[0] / errs[1]) >= 3.7


@pytest.mark.parametrize("method", ["nearest", "linear", "cubic"])
def test_periodic_wrap_matches_in_box_points(method, rng):
    vals = rng.standard_normal((10, 12))
    q = [rng.uniform(0, 10, 50), rng.uniform(0, 12, 50)]
    base = F.sample_nd(vals, q, method)
    for s0, s1 in ((10, 0), (-20, 12), (30, -36)):
        shifted = F.sample_nd(vals, [q[0] + s0, q[1] + s1], method)
        assert np.max(np.abs(shifted - base)) < 1e-12


def test_unknown_method_raises():
    with pytest.raises(ValueError):
        F.sample_nd(np.zeros((4, 4)), [np.zeros(1), np.zeros(1)], "quintic")


# ---------------------------------------------------------------------------
# distances (reference distance.py:43-91)
# ---------------------------------------------------------------------------


def _bump(g, c):
    x = _x(g)
    v = np.ones(g.n)
    for xi, ci in zip(x, c):
        v = v * np.exp(2.0 * (np.cos(xi - ci) - 1.0))
    return S(g, v)


def test_distance_values():
    g = F.Grid((32, 32))
    a, b = _bump(g, (0.3, -0.2)), _bump(g, (-0.4, 0.5))
    for kind in ("ssd", "ncc"):
        assert Dm.dist_value(a, a, kind) == pytest.approx(0.0, abs=1e-14)
    a2 = F.ScalarField._wrap(g, 2.0 * a.values)
    assert Dm.dist_value(a2, b, "ncc") == pytest.approx(Dm.dist_value(a, b, "ncc"), rel=1e-12)
    assert Dm.dist_value(a2, b, "ssd") != pytest.approx(Dm.dist_value(a, b, "ssd"), rel=1e-3)
    one, zero = F.ScalarField.full(g, 0.5), F.ScalarField.zeros(g)
    assert Dm.dist_value(one, zero, "ssd") == pytest.approx(0.5 * 0.25 * (2 * np.pi) ** 2, rel=1e-13)
    assert 0.0 <= Dm.dist_value(a, b, "ncc") <= 1.0
    with pytest.raises(Dm.ZeroNormError):
        Dm.dist_value(zero, b, "ncc")


@pytest.mark.parametrize("kind", ["ssd", "ncc"])
def test_final_conditions(kind, rng):
    g = F.Grid((32, 32))
    a, b = _bump(g, (0.3, -0.2)), _bump(g, (-0.4, 0.5))
    # zero at a perfect match, zero for a zero perturbation, linear in it
    assert np.max(np.abs(_np(Dm.adjoint_final(a, a, kind)))) < 1e-14
    assert np.max(np.abs(_np(Dm.incremental_final_gn(F.ScalarField.zeros(g), a, b, kind)))) == 0.0
    mt = noise(g, rng)
    one = _np(Dm.incremental_final_gn(mt, a, b, kind))
    two = _np(Dm.incremental_final_gn(F.ScalarField._wrap(g, 2.0 * mt.values), a, b, kind))
    assert np.max(np.abs(two - 2.0 * one)) < 1e-12 * np.max(np.abs(one))
    # adjoint final condition = -dJ/dm_def (per unit cell volume), by central FD on a few voxels
    lam = _np(Dm.adjoint_final(a, b, kind))
    av = _np(a.values)
    for (i, j) in ((3, 5), (17, 9), (28, 30)):
        e = 1e-6
        ap, am = av.copy(), av.copy()
        ap[i, j] += e
        am[i, j] -= e
        fd = (Dm.dist_value(S(g, ap), b, kind) - Dm.dist_value(S(g, am), b, kind)) / (2 * e)
        assert -fd / g.cell_volume == pytest.approx(lam[i, j], rel=1e-5, abs=1e-9)


# ---------------------------------------------------------------------------
# grid, inner products, time integral, containers (reference fields.py)
# ---------------------------------------------------------------------------


def test_grid_geometry_and_validation():
    g = F.Grid((16, 32, 8))
    for h, n in zip(g.h, g.n):
        assert h * n == pytest.approx(2 * np.pi, rel=1e-15)
    assert g.axis_coords(1)[0] == pytest.approx(np.pi - g.h[1], rel=1e-15)
    assert np.all(np.diff(g.axis_coords(0)) < 0)
    for bad in ((15, 16), (6, 16)):
        with pytest.raises(ValueError):
            F.Grid(bad)
    assert np.allclose(F.mesh_coordinates(g, (8, 16, 4)), 0.0)
    assert F.mesh_coordinates(g, (16, 32, 8)) == pytest.approx([-np.pi] * 3)
    with pytest.raises(IndexError):
        F.mesh_coordinates(g, (0, 1, 1))


def test_l2_inner_properties(rng):
    g = F.Grid((16, 16))
    c = F.ScalarField.full(g, 1.5)
    assert F.l2_inner(c, c) == pytest.approx(2.25 * (2 * np.pi) ** 2, rel=1e-13)
    x = _x(g)
    assert abs(F.l2_inner(S(g, np.sin(x[0])), S(g, np.sin(2 * x[0])))) < 1e-13
    a, b = noise(g, rng), noise(g, rng)
    assert F.l2_inner(a, b) == F.l2_inner(b, a)
    assert F.l2_inner(a, a) > 0
    with pytest.raises(ValueError):
        F.l2_inner(a, F.ScalarField.zeros(F.Grid((16, 32))))


def test_time_integral_is_the_trapezoid_rule():
    g = F.Grid((8, 8))
    for m in (2, 3, 5):
        ts = np.linspace(0.0, 1.0, m)
        const = F.time_integral([F.ScalarField.full(g, 2.0) for _ in ts])
        assert np.allclose(_np(const.values), 2.0, rtol=1e-15)
        lin = F.time_integral([F.ScalarField.full(g, 3.0 * t + 1.0) for t in ts])
        assert np.allclose(_np(lin.values), 2.5, rtol=1e-14)
        quad = F.time_integral([F.ScalarField.full(g, t * t) for t in ts])
        h = 1.0 / (m - 1)
        assert np.allclose(_np(quad.values), 1.0 / 3.0 + h * h / 6.0, rtol=1e-14)
    vec = F.time_integral([F.VectorField.constant(g, (1.0, -2.0)) for _ in range(3)])
    assert isinstance(vec, F.VectorField) and np.allclose(_np(vec)[1], -2.0)
    with pytest.raises(ValueError):
        F.time_integral([F.ScalarField.zeros(g)])


def test_containers_reject_bad_data():
    g = F.Grid((8, 8))
    bad = np.zeros(g.n)
    bad[1, 2] = np.nan
    with pytest.raises(ValueError):
        F.ScalarField(g, bad)
    with pytest.raises(ValueError):
        F.ScalarField(g, np.zeros((8, 10)))
    with pytest.raises(ValueError):
        F.VectorField(g, np.zeros((3, 8, 8)))


# ---------------------------------------------------------------------------
# det F bounds and the alpha continuation (reference continuation.py)
# ---------------------------------------------------------------------------


def test_det_bounds_at_rest_and_under_translation():
    ok, dmin, dmax, dmean = F.det_bounds_ok(F.VectorField.zeros(F.Grid((16, 16), n_t=2)), 0.1)
    assert ok and dmin == dmax == dmean == 1.0
    ok, dmin, dmax, _ = F.det_bounds_ok(F.VectorField.constant(F.Grid((32, 32)), (0.7, -0.5)), 0.1)
    assert ok and dmin == pytest.approx(1.0, abs=1e-12) and dmax == pytest.approx(1.0, abs=1e-12)


def test_compressive_field_violates_the_det_bound():
    _, _, v = F.synth_case("compress", 32, seed=0)
    ok, dmin, _, _ = F.det_bounds_ok(v, 0.1)
    assert not ok and dmin < 0.1


def test_search_identical_images_is_one_trial():
    g = F.Grid((32, 32))
    m = _bump(g, (0.0, 0.0))
    res = F.search_alpha(m, m, reg=F.RegConfig(alpha=1.0, incomp=F.IncompressibilityMode("none")))
    assert res.status == "ok" and res.alpha == 1.0 and len(res.trials) == 1
    assert float(res.velocity.data.abs().max()) == 0.0


def test_cascade_schedule_and_single_stage_target():
    got = cascade_alphas(1.773437e-3)
    assert got[:4] == [1.0, 0.1, 0.01, 0.001] and got[4] == pytest.approx(1.773437e-3, rel=1e-12)
    assert cascade_alphas(1.0) == [1.0] and cascade_alphas(1e-2) == [1.0, 0.1, 0.01]
    m0, m1, _ = F.synth_case("rotation", 32, seed=2)
    plain = F.RegConfig(alpha=1.0, incomp=F.IncompressibilityMode("none"))
    _, direct = F.register(m0, m1, reg=plain)
    _, rep, stages = F.continuation_solve(m0, m1, 1.0, reg=plain)
    assert len(stages) == 1 and rep.mismatch == pytest.approx(direct.mismatch, rel=1e-12)
    with pytest.raises(ValueError):
        F.continuation_solve(m0, m1, 0.0)


def _plain(alpha=1.0):
    return F.RegConfig(alpha=alpha, incomp=F.IncompressibilityMode("none"))


def test_search_brackets_the_compress_pair_and_passes(tmp_path):
    from paper_2401_17493_b200.continuation import write_trials_csv

    m0, m1, _ = F.synth_case("compress", 64, seed=0)
    cfg = F.SearchConfig(bisection_depth=4)
    res = F.search_alpha(m0, m1, cfg=cfg, reg=_plain(), precond=F.PrecondKind("h0"))
    assert res.status == "ok" and res.alpha is not None
    assert F.det_bounds_ok(res.velocity, cfg.eps_det)[0]
    assert res.anomalies == []
    largest_fail = max(t.alpha for t in res.trials if not t.passed)
    assert all(t.passed for t in res.trials if t.alpha > largest_fail)
    assert all(t.warm_started or t.alpha == 1.0 or t.warm_start_dropped for t in res.trials)
    sweep = [t for t in res.trials if t.phase == "sweep"]
    assert not sweep[-1].passed and all(t.passed for t in sweep[:-1])
    write_trials_csv(tmp_path / "trials.csv", res.trials)
    assert (tmp_path / "trials.csv").read_text().splitlines()[0].startswith("alpha,passed,det_min,det_max")


def test_search_edge_cases():
    m0, m1, _ = F.synth_case("rotation", 32, seed=2)
    res = F.search_alpha(m0, m1, cfg=F.SearchConfig(eps_det=0.999999, bisection_depth=2), reg=_plain())
    assert res.status == "violated_at_start" and res.alpha is None
    assert len(res.trials) == 1 and not res.trials[0].passed
    res = F.search_alpha(m0, m1, cfg=F.SearchConfig(alpha_floor=1e-2), reg=_plain(), precond=F.PrecondKind("h0"))
    assert res.status == "floor_reached" and res.alpha == pytest.approx(1e-2)
    assert all(t.passed for t in res.trials)


def test_warm_cascade_at_least_as_good_as_cold():
    m0, m1, _ = F.synth_case("swirl", 64, seed=1)
    _, cold = F.register(m0, m1, reg=_plain(1e-2), precond=F.PrecondKind("h0"))
    _, rep, stages = F.continuation_solve(m0, m1, 1e-2, reg=_plain(), precond=F.PrecondKind("h0"))
    assert len(stages) == 3 and rep.mismatch <= cold.mismatch * 1.05
    assert rep.pde_solves == sum(s.pde_solves for s in stages)
    assert rep.iterations == sum(s.iterations for s in stages)


def test_preconditioner_iteration_ordering_at_small_alpha():
    from paper_2401_17493_b200.optimizer import OptimizerConfig, pcg_newton_step

    m0, m1, _ = F.synth_case("swirl", 64, seed=1)
    reg = _plain(1e-3)
    v, _ = F.register(m0, m1, reg=reg, precond=F.PrecondKind("h0"))
    counts = {}
    for kind in ("2level", "h0", "reg"):
        st = F.KktState(m0, m1, reg)
        st.refresh(v)
        _, n, info = pcg_newton_step(st, st.gradient(), F.PrecondKind(kind), 1e-6,
                                     OptimizerConfig(pcg_max_iterations=2000))
        assert info["flag"] == "converged"
        counts[kind] = n
    assert counts["2level"] <= counts["h0"] <= counts["reg"]


def test_mesh_coordinates_tile_the_box_and_containers_copy():
    g3 = F.Grid((8, 8, 8))
    assert np.allclose(F.mesh_coordinates(g3, (3, 4, 5)), (np.pi / 4, 0.0, -np.pi / 4))
    g = F.Grid((8, 10))
    with pytest.raises(IndexError):
        F.mesh_coordinates(g, (3, 11))
    raw = [F.mesh_coordinates(g, (a, b)) for a in range(1, 9) for b in range(1, 11)]
    assert all(-np.pi <= p[0] < np.pi and -np.pi <= p[1] < np.pi for p in raw)
    pts = {tuple(np.round(p, 12)) for p in raw}
    assert len(pts) == 80
    assert np.allclose(np.diff(sorted({p[0] for p in pts})), g.h[0])
    gt = F.Grid((8, 8), n_t=2)
    s = F.ScalarField.zeros(gt)
    ts = F.TimeSeriesField.from_slices(gt, [s, s, s])
    ts.slice(0).values[0, 0] = 99.0
    assert float(ts.data[0, 0, 0]) == 0.0
    s.values[0, 0] = 7.0
    assert float(ts.data[0, 0, 0]) == 0.0
    with pytest.raises(ValueError):
        F.VectorField.from_components([F.ScalarField.zeros(F.Grid((8, 8))), F.ScalarField.zeros(F.Grid((16, 16)))])
