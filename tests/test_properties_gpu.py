"""Property tests of the device solvers, restating the reference's own
behavioural test suite (tests/test_transport.py, test_kkt.py,
test_optimizer.py of the reference package) in this repo's words:
exactness on trivial inputs (zero / constant velocity, zero directions,
identical images), analytic solutions (translations, closed forms at rest),
convergence orders against an RK4 characteristic integrator, conservation,
linearisation checks by finite differences, SPD / symmetry, counters and
short-circuits.

Each property runs twice where the engine differs: on 2D f64 grids (the
generic staged engine, the reference's own tolerances) and on 3D fp32 grids
whose every axis reaches the TMA box (>= 12 x 16 x 64; the engine bench.py
times: TMA boxes, tile plans, periodic patches), with fp32 tolerances.
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU collection
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2401_17493_b200 as F  # noqa: E402
from paper_2401_17493_b200 import transport as T  # noqa: E402
from paper_2401_17493_b200.diffops import (  # noqa: E402
    apply_inv_reg_operator,
    apply_reg_operator,
    gradient,
    project_body_force,
)
from paper_2401_17493_b200.optimizer import DescentDirectionError, armijo_line_search, pcg_newton_step  # noqa: E402

# ---------------------------------------------------------------------------
# fixtures of the properties (smooth periodic images / velocities)
# ---------------------------------------------------------------------------


def _coords(g):
    return [np.broadcast_to(c, g.n).astype(np.float64) for c in g.coord_arrays()]


def _mesh(g):
    return np.stack(_coords(g))


def bump(g, kappa=2.0, centers=None):
    centers = centers or [0.0] * g.d
    vals = np.ones(g.n)
    for c, x in zip(centers, _coords(g)):
        vals = vals * np.exp(kappa * (np.cos(x - c) - 1.0))
    return F.ScalarField(g, vals.astype(g.dtype))


def vortex(g, amp=1.0):
    """Divergence-free cell vortex in the first two axes (stream function
    cos x0 cos x1); the third component, if any, is zero."""
    x = _coords(g)
    data = np.zeros((g.d, *g.n))
    data[0] = -amp * np.cos(x[0]) * np.sin(x[1])
    data[1] = amp * np.sin(x[0]) * np.cos(x[1])
    return F.VectorField(g, data.astype(g.dtype))


def bandlimited(g, rng, amp=1.0, kmax=3, modes=6):
    data = np.zeros((g.d, *g.n))
    for i in range(g.d):
        spec = np.zeros(g.n, dtype=complex)
        for _ in range(modes):
            k = tuple(int(rng.integers(0, kmax + 1)) for _ in range(g.d))
            spec[k] = rng.standard_normal() + 1j * rng.standard_normal()
        f = np.fft.ifftn(spec).real
        if np.abs(f).max() > 0:
            f /= np.abs(f).max()
        data[i] = amp * f
    return F.VectorField(g, data.astype(g.dtype))


def rk4_flow(points, v, t_total, steps):
    """Characteristics dy/dt = v(y) by RK4 at small steps, the velocity read
    with the (reference-pinned) cubic sample_nd; f64 on the device."""
    from paper_2401_17493_b200.interp import fractional_index

    g = v.grid
    vd = v.data.to(torch.float64)
    y = torch.as_tensor(points, dtype=torch.float64, device="cuda").clone()
    dt = t_total / steps

    def vel(p):
        qs = fractional_index(g, p)
        return torch.stack([F.sample_nd(vd[i], qs, "cubic") for i in range(g.d)]).reshape(p.shape)

    for _ in range(steps):
        k1 = vel(y)
        k2 = vel(y + 0.5 * dt * k1)
        k3 = vel(y + 0.5 * dt * k2)
        k4 = vel(y + dt * k3)
        y = y + (dt / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)
    return y.cpu().numpy()


def _np(x):
    return (x.data if hasattr(x, "data") else x).double().cpu().numpy()


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


# the two engines: (grid factory, exactness tolerance scale)
F64_2D = "f64-2d"
F32_3D = "f32-3d-tma"
ENGINES = [F64_2D, F32_3D]


def grid_of(engine, n2d=16, n_t=4):
    if engine == F64_2D:
        return F.Grid((n2d, n2d), n_t=n_t)
    return F.Grid((16, 16, 64), n_t=n_t, dtype=np.float32)


def tol(engine, f64, f32):
    return f64 if engine == F64_2D else f32


# ---------------------------------------------------------------------------
# departure points (reference transport.py:37-45)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("engine", ENGINES)
def test_departure_zero_velocity_is_identity(engine):
    g = grid_of(engine)
    disp = T.departure_disp(F.VectorField.zeros(g), g.h_t)
    assert float(disp.abs().max()) == 0.0
    y = T.departure_points(F.VectorField.zeros(g), g.h_t)
    assert np.max(np.abs(_np(y) - _mesh(g))) <= tol(engine, 1e-14, 1e-5)


@pytest.mark.parametrize("engine", ENGINES)
def test_departure_constant_velocity_exact(engine):
    g = grid_of(engine)
    c = (0.3, -0.2) if g.d == 2 else (0.3, -0.2, 0.45)
    v = F.VectorField.constant(g, c)
    y = T.departure_points(v, g.h_t)
    want = _mesh(g) - g.h_t * np.asarray(c).reshape((g.d,) + (1,) * g.d)
    assert np.max(np.abs(_np(y) - want)) < tol(engine, 1e-14, 2e-6)


def test_departure_third_order_against_rk4():
    g = F.Grid((128, 128), n_t=1)
    v = vortex(g, amp=1.0)
    x = _mesh(g).reshape(2, -1)
    neg = F.VectorField._wrap(g, -v.data)
    errs = {}
    for h_t in (0.5, 0.25, 0.125):
        y = _np(T.departure_points(v, h_t)).reshape(2, -1)
        errs[h_t] = np.max(np.abs(y - rk4_flow(x, neg, h_t, 50)))
    assert math.log2(errs[0.5] / errs[0.25]) > 2.5
    assert math.log2(errs[0.25] / errs[0.125]) > 2.5


# ---------------------------------------------------------------------------
# state equation (reference transport.py:83-98)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("engine", ENGINES)
def test_state_zero_velocity_keeps_every_slice(engine, rng):
    g = grid_of(engine, n_t=3)
    m0 = F.ScalarField(g, rng.standard_normal(g.n).astype(g.dtype))
    out = T.solve_state(m0, F.VectorField.zeros(g))
    for j in range(g.n_t + 1):
        assert torch.equal(out.data[j], m0.values)


@pytest.mark.parametrize("engine", ENGINES)
def test_state_constant_field_is_invariant(engine):
    g = grid_of(engine)
    m0 = F.ScalarField.full(g, 0.75)
    c = (0.4, 0.1) if g.d == 2 else (0.4, 0.1, -0.7)
    out = T.solve_state(m0, F.VectorField.constant(g, c))
    assert np.max(np.abs(_np(out) - 0.75)) < tol(engine, 1e-13, 2e-6)


@pytest.mark.parametrize("engine", ENGINES)
def test_state_translation_matches_analytic_shift(engine):
    g = F.Grid((128, 128), n_t=4) if engine == F64_2D else F.Grid((64, 64, 64), n_t=4, dtype=np.float32)
    x = _coords(g)
    c = (0.6, -0.4) if g.d == 2 else (0.6, -0.4, 0.5)
    out = T.solve_state(bump(g, 2.0), F.VectorField.constant(g, c)).final()
    want = np.ones(g.n)
    for xi, ci in zip(x, c):
        want = want * np.exp(2.0 * (np.cos(xi - ci) - 1.0))
    assert np.max(np.abs(_np(out.values) - want)) < tol(engine, 1e-3, 2e-3)


@pytest.mark.parametrize("engine", ENGINES)
def test_state_linear_interpolation_min_max_principle(engine, rng):
    g = grid_of(engine, n2d=32)
    m0 = F.ScalarField(g, rng.standard_normal(g.n).astype(g.dtype))
    out = _np(T.solve_state(m0, vortex(g, 1.2), method="linear"))
    mv = _np(m0.values)
    eps = 4 * np.finfo(g.dtype).eps * max(1.0, np.abs(mv).max())
    assert out.min() >= mv.min() - eps
    assert out.max() <= mv.max() + eps


def test_state_time_refinement_order_on_invariant_problem():
    # data constant along the vortex's streamlines: the exact solution does
    # not move, the error left is the RK2 characteristics' (2nd order)
    errs = {}
    for n_t in (1, 2, 4):
        g = F.Grid((128, 128), n_t=n_t)
        x = _coords(g)
        m0 = F.ScalarField(g, np.exp(1.5 * (np.cos(x[0]) * np.cos(x[1]) - 1.0)))
        errs[n_t] = np.max(np.abs(_np(T.solve_state(m0, vortex(g, 1.0)).final().values) - _np(m0.values)))
    assert math.log2(errs[1] / errs[2]) >= 1.5
    assert math.log2(errs[2] / errs[4]) >= 1.5


# ---------------------------------------------------------------------------
# adjoint / incremental adjoint (reference transport.py:105-135,179-194)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("solver", [T.solve_adjoint, T.solve_inc_adjoint_gn])
@pytest.mark.parametrize("engine", ENGINES)
def test_adjoint_zero_final_condition(engine, solver):
    g = grid_of(engine)
    out = solver(F.ScalarField.zeros(g), vortex(g, 0.5))
    assert float(out.data.abs().max()) == 0.0


@pytest.mark.parametrize("solver", [T.solve_adjoint, T.solve_inc_adjoint_gn])
@pytest.mark.parametrize("engine", ENGINES)
def test_adjoint_zero_velocity_keeps_final(engine, solver, rng):
    g = grid_of(engine)
    fin = F.ScalarField(g, rng.standard_normal(g.n).astype(g.dtype))
    out = solver(fin, F.VectorField.zeros(g))
    for j in range(g.n_t + 1):
        assert torch.equal(out.data[j], fin.values)


@pytest.mark.parametrize("engine", ENGINES)
def test_adjoint_divergence_free_is_backward_advection(engine):
    g = F.Grid((64, 64), n_t=4) if engine == F64_2D else F.Grid((32, 32, 64), n_t=4, dtype=np.float32)
    v = vortex(g, 0.8)
    fin = bump(g, 2.0, centers=[0.5, -0.3] + [0.0] * (g.d - 2))
    lam = T.solve_adjoint(fin, v)
    back = T.solve_state(fin, F.VectorField._wrap(g, -v.data))
    for j in range(g.n_t + 1):
        assert np.max(np.abs(_np(lam.data[j]) - _np(back.data[g.n_t - j]))) < tol(engine, 1e-10, 2e-5)


def test_adjoint_mass_conserved_and_converges_in_time():
    g = F.Grid((64, 64), n_t=4)
    v = vortex(g, 0.8)
    fin = bump(g, 2.0, centers=[0.5, -0.3])
    lam = T.solve_adjoint(fin, v)
    one = F.ScalarField.full(g, 1.0)
    masses = [F.l2_inner(lam.slice(j), one) for j in range(g.n_t + 1)]
    assert max(abs(m - masses[-1]) for m in masses) / abs(masses[-1]) < 1e-3
    gf = g.with_time_steps(64)
    ref = T.solve_adjoint(F.ScalarField(gf, fin.values), F.VectorField(gf, v.data))
    gap = np.max(np.abs(_np(lam.data[0]) - _np(ref.data[0]))) / np.max(np.abs(_np(ref.data[0])))
    assert gap < 5e-3


# ---------------------------------------------------------------------------
# incremental state (reference transport.py:147-176)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("engine", ENGINES)
def test_inc_state_zero_direction_is_zero(engine):
    g = grid_of(engine)
    v = vortex(g, 0.5)
    ms = T.solve_state(bump(g, 1.5), v)
    out = T.solve_inc_state(ms, v, F.VectorField.zeros(g))
    assert float(out.data.abs().max()) == 0.0


@pytest.mark.parametrize("engine", ENGINES)
def test_inc_state_zero_velocity_closed_form(engine, rng):
    # at rest every Heun source is -grad m0 . v~ and the characteristics stand
    # still, so m~(1) = -grad m0 . v~
    g = F.Grid((64, 64), n_t=4) if engine == F64_2D else F.Grid((16, 32, 64), n_t=4, dtype=np.float32)
    m0 = bump(g, 2.0)
    vt = bandlimited(g, rng, amp=0.7)
    ms = T.solve_state(m0, F.VectorField.zeros(g))
    out = _np(T.solve_inc_state(ms, F.VectorField.zeros(g), vt).final().values)
    want = -np.sum(_np(gradient(m0, scheme="fd8")) * _np(vt), axis=0)
    assert np.max(np.abs(out - want)) < tol(engine, 1e-12, 2e-6 * max(1.0, np.abs(want).max()))


def test_inc_state_linearises_the_mismatch(rng):
    g = F.Grid((64, 64), n_t=4)
    m0 = bump(g, 2.0, centers=[0.3, -0.2])
    m1 = bump(g, 2.0, centers=[-0.4, 0.5])
    v = bandlimited(g, rng, amp=0.3, kmax=2)
    vt = bandlimited(g, rng, amp=0.5, kmax=2)
    ms = T.solve_state(m0, v)
    mt1 = T.solve_inc_state(ms, v, vt).final()

    def dist(vel):
        r = T.solve_state(m0, vel).final().values - m1.values
        return 0.5 * F.l2_inner(F.ScalarField._wrap(g, r), F.ScalarField._wrap(g, r))

    pred = F.l2_inner(F.ScalarField._wrap(g, ms.final().values - m1.values), mt1)
    best = min(abs((dist(F.VectorField._wrap(g, v.data + e * vt.data)) -
                    dist(F.VectorField._wrap(g, v.data - e * vt.data))) / (2 * e) - pred) / abs(pred)
               for e in (1e-2, 3e-3, 1e-3, 3e-4))
    assert best < 1e-2


def test_state_linearisation_pairs_with_the_gradient_data_term(rng):
    # <m~(1), -lam(1)> = <v~, int lam grad m dt> up to the scheme's
    # discrete inconsistency (the reference's own loose bound)
    g = F.Grid((64, 64), n_t=4)
    m0 = bump(g, 2.0, centers=[0.3, -0.2])
    m1 = bump(g, 2.0, centers=[-0.4, 0.5])
    v = bandlimited(g, rng, amp=0.3, kmax=2)
    vt = bandlimited(g, rng, amp=0.5, kmax=2)
    ms = T.solve_state(m0, v)
    grads = T.state_gradients(ms)
    mt1 = T.solve_inc_state(ms, v, vt, grad_slices=grads).final()
    lam_fin = F.ScalarField._wrap(g, -(ms.final().values - m1.values))
    lam = T.solve_adjoint(lam_fin, v)
    lhs = F.l2_inner(mt1, F.ScalarField._wrap(g, -lam_fin.values))
    body = F.time_integral([F.VectorField._wrap(g, lam.data[j] * grads[j].data) for j in range(g.n_t + 1)])
    rhs = F.l2_inner(vt, body)
    assert abs(lhs - rhs) / max(abs(lhs), abs(rhs)) <= 5e-2


# ---------------------------------------------------------------------------
# deformation tensor and composed map (reference transport.py:197-247)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("engine", ENGINES)
def test_deformation_zero_velocity_is_identity(engine):
    g = grid_of(engine)
    det = _np(T.solve_deformation_tensor(F.VectorField.zeros(g)).determinant().values)
    assert np.max(np.abs(det - 1.0)) == 0.0


@pytest.mark.parametrize("engine", ENGINES)
def test_deformation_translation_keeps_identity(engine):
    g = grid_of(engine, n2d=32)
    c = (0.5, -0.3) if g.d == 2 else (0.5, -0.3, 0.2)
    det = _np(T.solve_deformation_tensor(F.VectorField.constant(g, c)).determinant().values)
    assert np.max(np.abs(det - 1.0)) < tol(engine, 1e-12, 1e-6)


def test_deformation_determinant_against_flow_map(rng):
    g = F.Grid((32, 32), n_t=4)
    v = bandlimited(g, rng, amp=0.5, kmax=2)
    det = _np(T.solve_deformation_tensor(v).determinant().values)
    x = _mesh(g).reshape(2, -1)
    neg = F.VectorField._wrap(g, -v.data)
    x0 = rk4_flow(x, neg, 1.0, 200)
    dlt = 1e-4
    jac = np.zeros((2, 2, x.shape[1]))
    for j in range(2):
        e = np.zeros((2, 1))
        e[j] = dlt
        jac[:, j, :] = (rk4_flow(x0 + e, v, 1.0, 200) - rk4_flow(x0 - e, v, 1.0, 200)) / (2 * dlt)
    ref = (jac[0, 0] * jac[1, 1] - jac[0, 1] * jac[1, 0]).reshape(g.n)
    assert np.max(np.abs(det - ref)) / np.max(np.abs(ref)) < 1e-2


@pytest.mark.parametrize("engine", ENGINES)
def test_composed_map_zero_and_constant_velocity(engine):
    g = grid_of(engine)
    out0 = _np(T.compose_trajectory(F.VectorField.zeros(g)))
    assert np.max(np.abs(out0 - _mesh(g))) <= tol(engine, 1e-14, 1e-5)
    c = (0.5, -0.25) if g.d == 2 else (0.5, -0.25, 0.3)
    out = _np(T.compose_trajectory(F.VectorField.constant(g, c)))
    want = _mesh(g) - np.asarray(c).reshape((g.d,) + (1,) * g.d)
    assert np.max(np.abs(out - want)) < tol(engine, 1e-13, 1e-5)


def test_composed_map_carries_the_template_like_the_state_solver(rng):
    g = F.Grid((32, 32), n_t=4)
    v = bandlimited(g, rng, amp=0.5, kmax=2)
    m0 = bump(g, 2.0, centers=[0.4, 0.2])
    mf = _np(T.solve_state(m0, v).final().values)
    from paper_2401_17493_b200.interp import interpolate

    via_map = _np(interpolate(m0, T.compose_trajectory(v)).values)
    assert np.max(np.abs(via_map - mf)) < 2e-2


# ---------------------------------------------------------------------------
# KKT state (reference kkt.py:136-341)
# ---------------------------------------------------------------------------


def plain(alpha):
    return F.RegConfig(alpha=alpha, incomp=F.IncompressibilityMode("none"))


KKT_MODES = ["f64-2d", "mixed-3d-tma"]


def kkt_case(mode, seed=3, n=32):
    if mode == "f64-2d":
        m0, m1, _ = F.synth_case("rotation", n, seed=seed)
        return m0, m1, None
    m0, m1, _ = F.synth_case("rotation", 64, seed=seed, d=3)
    return m0, m1, np.float32


def test_objective_and_gradient_vanish_for_identical_images_at_rest():
    g = F.Grid((32, 32), n_t=4)
    m = bump(g, 1.5)
    st = F.KktState(m, m, plain(1e-2))
    assert abs(st.objective()) <= 1e-14
    assert float(st.gradient().data.abs().max()) < 1e-14


@pytest.mark.parametrize("mode", KKT_MODES)
def test_gradient_at_rest_closed_form(mode):
    # at rest the dual is constant in time: g = -(m0 - m1) grad m0
    m0, m1, tdt = kkt_case(mode, seed=2)
    st = F.KktState(m0, m1, plain(1e-2), transport_dtype=tdt)
    gm = _np(gradient(m0, scheme="fd8"))
    want = -(_np(m0.values) - _np(m1.values)) * gm
    err = np.max(np.abs(_np(st.gradient()) - want))
    assert err < (1e-12 if tdt is None else 1e-5 * np.abs(want).max())


@pytest.mark.parametrize("mode", KKT_MODES)
def test_gradient_directional_derivative_matches_fd(mode, rng):
    m0, m1, tdt = kkt_case(mode, seed=5, n=64)
    st = F.KktState(m0, m1, plain(1e-2), transport_dtype=tdt)
    g = st.grid
    v0 = bandlimited(g, rng, amp=0.3, kmax=2)
    st.refresh(v0)
    grad = st.gradient()
    vt = bandlimited(g, rng, amp=1.0, kmax=2)
    slope = F.l2_inner(grad, vt)
    eps_list = (1e-2, 3e-3, 1e-3, 3e-4, 1e-4) if tdt is None else (3e-2, 1e-2, 3e-3)
    best = min(abs((st.objective_at(F.VectorField._wrap(g, v0.data + e * vt.data)) -
                    st.objective_at(F.VectorField._wrap(g, v0.data - e * vt.data))) / (2 * e) - slope) / abs(slope)
               for e in eps_list)
    assert best < 5e-2


@pytest.mark.parametrize("mode", KKT_MODES)
@pytest.mark.parametrize("incomp", ["none", "near-incompressible"])
def test_matvec_at_rest_matches_closed_form(mode, incomp, rng):
    # at rest H v~ = alpha L v~ + P((grad m0 . v~) grad m0)
    m0, m1, tdt = kkt_case(mode, seed=3)
    im = F.IncompressibilityMode(incomp, 1e-4) if incomp != "none" else F.IncompressibilityMode("none")
    st = F.KktState(m0, m1, F.RegConfig(alpha=1e-2, incomp=im), transport_dtype=tdt)
    g = st.grid
    vt = bandlimited(g, rng, amp=0.6, kmax=2)
    out = _np(st.hessian_matvec(vt))
    gm = gradient(m0, scheme="fd8")
    body = F.VectorField._wrap(g, (gm.data * vt.data).sum(0) * gm.data)
    if incomp != "none":
        body = project_body_force(body, im, 1e-2)
    want = _np(apply_reg_operator(vt, F.RegOperatorSpec(), 1e-2)) + _np(body)
    assert np.max(np.abs(out - want)) / np.max(np.abs(want)) < (1e-12 if tdt is None else 1e-5)


@pytest.mark.parametrize("mode", KKT_MODES)
def test_matvec_zero_direction_and_symmetry(mode, rng):
    m0, m1, tdt = kkt_case(mode, seed=5, n=64)
    st = F.KktState(m0, m1, plain(1e-2), transport_dtype=tdt)
    g = st.grid
    st.refresh(bandlimited(g, rng, amp=0.3, kmax=2))
    assert float(st.hessian_matvec(F.VectorField.zeros(g)).data.abs().max()) < 1e-14
    for _ in range(3):
        a, b = bandlimited(g, rng), bandlimited(g, rng)
        ha, hb = st.hessian_matvec(a), st.hessian_matvec(b)
        rel = abs(F.l2_inner(ha, b) - F.l2_inner(a, hb)) / (F.norm_l2(ha) * F.norm_l2(b))
        assert rel < 1e-3


def test_counters_track_pde_solves():
    m0, m1, _ = F.synth_case("rotation", 32, seed=3)
    st = F.KktState(m0, m1, plain(1e-2))
    assert (st.matvecs, st.pde_solves) == (0, 2)
    st.hessian_matvec(F.VectorField.zeros(st.grid))
    assert (st.matvecs, st.pde_solves) == (1, 4)
    st.refresh(F.VectorField.zeros(st.grid))
    assert st.pde_solves == 6
    st.objective_at(F.VectorField.zeros(st.grid))
    assert st.pde_solves == 7


@pytest.mark.parametrize("kind", ["h0", "2level"])
def test_h0_preconditioners_reduce_to_reg_inverse_for_a_flat_image(kind, rng):
    g = F.Grid((32, 32), n_t=2)
    const = F.ScalarField.full(g, 0.5)
    st = F.KktState(const, const, plain(1e-2))
    r = bandlimited(g, rng)
    got = _np(st.apply_precond(r, F.PrecondKind(kind), 1e-6))
    want = _np(apply_inv_reg_operator(r, F.RegOperatorSpec(), 1e-2))
    assert np.max(np.abs(got - want)) < 1e-10


@pytest.mark.parametrize("kind", ["reg", "h0", "2level"])
def test_preconditioners_are_spd_with_tight_inner_tolerance(kind, rng):
    m0, m1, _ = F.synth_case("swirl", 64, seed=1)
    st = F.KktState(m0, m1, plain(1e-2))
    pk = F.PrecondKind(kind, inner_tol_factor=1e-10, inner_max_iterations=400)
    for _ in range(3):
        r, s = bandlimited(st.grid, rng), bandlimited(st.grid, rng)
        mr, ms = st.apply_precond(r, pk, 1.0), st.apply_precond(s, pk, 1.0)
        assert F.l2_inner(mr, r) > 0.0
        assert abs(F.l2_inner(mr, s) - F.l2_inner(r, ms)) / (F.norm_l2(mr) * F.norm_l2(s)) < 1e-3


def test_two_level_matches_fine_h0_on_smooth_residuals(rng):
    m0, m1, _ = F.synth_case("rotation", 64, seed=4)
    st = F.KktState(m0, m1, plain(1e-2))
    r = bandlimited(st.grid, rng, amp=1.0, kmax=3)
    tight = dict(inner_tol_factor=1e-8, inner_max_iterations=800)
    two = _np(st.apply_precond(r, F.PrecondKind("2level", **tight), 1.0))
    fine = _np(st.apply_precond(r, F.PrecondKind("h0", **tight), 1.0))
    assert np.max(np.abs(two - fine)) / np.max(np.abs(fine)) < 1e-2


def test_unknown_preconditioner_rejected():
    with pytest.raises(ValueError):
        F.PrecondKind("jacobi")


# ---------------------------------------------------------------------------
# Newton-Krylov control (reference optimizer.py:81-281)
# ---------------------------------------------------------------------------


def test_pcg_zero_gradient_returns_zero_without_iterations():
    g = F.Grid((16, 16), n_t=2)
    m = bump(g, 1.5)
    st = F.KktState(m, m, plain(1e-2))
    vt, iters, _ = pcg_newton_step(st, F.VectorField.zeros(g), F.PrecondKind("reg"), 0.5)
    assert iters == 0
    assert float(vt.data.abs().max()) == 0.0


def test_pcg_pure_regularisation_converges_in_one_iteration(rng):
    # constant images: H = alpha L, inverted exactly by the 'reg' preconditioner
    g = F.Grid((32, 32), n_t=2)
    const = F.ScalarField.full(g, 0.4)
    st = F.KktState(const, const, plain(0.05))
    v = bandlimited(g, rng, amp=0.5)
    v = F.VectorField._wrap(g, v.data - v.data.mean(dim=(1, 2), keepdim=True))
    st.refresh(v)
    grad = st.gradient()
    vt, iters, _ = pcg_newton_step(st, grad, F.PrecondKind("reg"), 1e-8)
    assert iters == 1
    res = F.VectorField._wrap(g, st.hessian_matvec(vt).data + grad.data)
    assert F.norm_l2(res) <= 1e-8 * F.norm_l2(grad)


def test_armijo_rejects_an_ascent_direction():
    m0, m1, _ = F.synth_case("rotation", 32, seed=2)
    st = F.KktState(m0, m1, plain(1e-2))
    grad = st.gradient()
    with pytest.raises(DescentDirectionError):
        armijo_line_search(st, grad, grad)


@pytest.mark.parametrize("tdt", [None, np.float32])
def test_register_identical_images_short_circuit(tdt):
    g = F.Grid((32, 32), n_t=4) if tdt is None else F.Grid((16, 16, 64), n_t=4)
    m = bump(g, 2.0)
    v, rep = F.register(m, m, reg=plain(1e-2), transport_dtype=tdt)
    assert rep.iterations == 0
    assert rep.status == "converged"
    assert rep.mismatch == 0.0
    assert float(v.data.abs().max()) == 0.0
    assert rep.pde_solves == 2


def test_register_warm_start_resumes():
    m0, m1, _ = F.synth_case("rotation", 32, seed=2)
    v, r1 = F.register(m0, m1, reg=plain(1e-2), precond=F.PrecondKind("h0"))
    _, r2 = F.register(m0, m1, reg=plain(1e-2), precond=F.PrecondKind("h0"), v0=v)
    assert r2.trace[0]["objective"] == pytest.approx(r1.trace[-1]["objective"], rel=1e-12)
    assert r2.mismatch <= r1.mismatch * 1.05


def test_pcg_residual_meets_the_forcing_tolerance():
    m0, m1, _ = F.synth_case("rotation", 32, seed=2)
    st = F.KktState(m0, m1, plain(1e-2))
    grad = st.gradient()
    vt, _, info = pcg_newton_step(st, grad, F.PrecondKind("reg"), 0.1)
    res = F.VectorField._wrap(st.grid, st.hessian_matvec(vt).data + grad.data)
    assert F.norm_l2(res) <= 0.1 * F.norm_l2(grad)
    assert info["flag"] == "converged"


class _Quadratic:
    """J(v) = 0.5 |v|^2: the slice of the state API the line search uses."""

    def __init__(self, g, v):
        self.grid, self.v = g, v

    def objective(self):
        return 0.5 * F.l2_inner(self.v, self.v)

    def objective_at(self, v):
        return 0.5 * F.l2_inner(v, v)


def test_armijo_full_step_and_backtracking_on_a_quadratic(rng):
    from paper_2401_17493_b200.optimizer import OptimizerConfig

    g = F.Grid((16, 16), n_t=1)
    model = _Quadratic(g, F.VectorField(g, rng.standard_normal((2, *g.n))))
    grad = model.v
    gamma, trials, _ = armijo_line_search(model, F.VectorField._wrap(g, -grad.data), grad)
    assert gamma == 1.0 and trials == 1
    cfg = OptimizerConfig()
    far = F.VectorField._wrap(g, -100.0 * grad.data)
    gamma, _, j_new = armijo_line_search(model, far, grad, cfg)
    assert gamma is not None and gamma < 1.0
    assert j_new <= model.objective() + cfg.armijo_c1 * gamma * F.l2_inner(grad, far)


def test_objective_and_pure_distance_at_rest():
    from paper_2401_17493_b200.distance import dist_value

    m0, m1, _ = F.synth_case("translation", 32, seed=0)
    st = F.KktState(m0, m1, plain(1e-2))
    assert st.objective() == pytest.approx(dist_value(m0, m1, "ssd"), rel=1e-14)
    g = F.Grid((32, 32), n_t=2)
    const = F.ScalarField.full(g, 0.5)
    st = F.KktState(const, const, plain(0.3))
    v = F.VectorField(g, np.stack([np.sin(2 * _coords(g)[0]), np.zeros(g.n)]))
    st.refresh(v)
    # a single mode k = (2, 0): (alpha / 2) |k|^2 <v, v>
    assert st.objective() == pytest.approx(0.5 * 0.3 * 4.0 * F.l2_inner(v, v), rel=1e-12)


def test_functional_aliases_delegate_to_the_state(rng):
    from paper_2401_17493_b200 import kkt as K

    m0, m1, _ = F.synth_case("rotation", 32, seed=3)
    st = F.KktState(m0, m1, plain(1e-2))
    assert K.evaluate_objective(st) == st.objective()
    vt = bandlimited(st.grid, rng, amp=0.4)
    assert K.evaluate_objective(st, vt) == pytest.approx(st.objective_at(vt), rel=1e-14)
    assert torch.equal(K.evaluate_gradient(st).data, st.gradient().data)
    assert float((K.hessian_matvec_gn(st, vt).data - st.hessian_matvec(vt).data).abs().max()) < 1e-14
    r = bandlimited(st.grid, rng)
    assert torch.equal(K.apply_precond(r, F.PrecondKind("reg"), st).data,
                       apply_inv_reg_operator(r, F.RegOperatorSpec(), 1e-2).data)


def test_register_objective_monotone_and_counter_identity():
    m0, m1, _ = F.synth_case("rotation", 64, seed=2)
    _, rep = F.register(m0, m1, reg=plain(1e-2), precond=F.PrecondKind("reg"))
    obj = [row["objective"] for row in rep.trace]
    assert all(b <= a + 1e-12 for a, b in zip(obj, obj[1:]))
    assert rep.pde_solves == 2 * (rep.iterations + 1) + 2 * rep.matvecs + rep.line_search_evals
    assert len(rep.trace) == rep.iterations + 1


def test_register_reports_are_deterministic():
    m0, m1, _ = F.synth_case("translation", 32, seed=3)
    d1 = F.register(m0, m1, reg=plain(1e-2))[1].to_dict()
    d2 = F.register(m0, m1, reg=plain(1e-2))[1].to_dict()
    d1.pop("runtime"), d2.pop("runtime")
    for row in d1["trace"] + d2["trace"]:
        row.pop("time", None)
    assert d1 == d2


@pytest.mark.parametrize("tdt", [None, np.float32])
def test_register_variants_converge(tdt):
    # NCC on a translation, 3D, the all-spectral derivative scheme
    m0, m1, _ = F.synth_case("translation", 64, seed=0)
    _, rep = F.register(m0, m1, reg=plain(1e-2), distance="ncc", precond=F.PrecondKind("h0"), transport_dtype=tdt)
    assert rep.mismatch <= 0.1
    m0, m1, _ = F.synth_case("rotation", 32, seed=1, d=3)
    _, rep = F.register(m0, m1, reg=plain(1e-2), precond=F.PrecondKind("h0"), transport_dtype=tdt)
    assert rep.status == "converged" and rep.mismatch <= 0.2 and rep.detgrad_min > 0.0
    m0, m1, _ = F.synth_case("rotation", 32, seed=2)
    _, rep = F.register(m0, m1, reg=plain(1e-2), precond=F.PrecondKind("h0"), scheme="spectral",
                        transport_dtype=tdt)
    assert rep.status == "converged" and rep.mismatch <= 0.1


def test_divergence_control_tightens_volume_change():
    m0, m1, _ = F.synth_case("swirl", 64, seed=1)
    _, free = F.register(m0, m1, reg=plain(1e-2), precond=F.PrecondKind("h0"))
    hard_reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("incompressible"))
    _, hard = F.register(m0, m1, reg=hard_reg, precond=F.PrecondKind("h0"))
    assert hard.status == "converged" and hard.mismatch <= 0.15
    assert hard.detgrad_min > 0.9 and hard.detgrad_max < 1.1
    assert hard.detgrad_max - hard.detgrad_min < free.detgrad_max - free.detgrad_min
    assert free.divergence_energy == 0.0
    soft_reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
    _, soft = F.register(m0, m1, reg=soft_reg, precond=F.PrecondKind("h0"))
    assert soft.divergence_energy > 0.0
