"""Cubic B-spline interpolation (north-star extension, method "bspline").

The reference package has no B-spline path, so parity cannot
be pinned to the reference; it is pinned to an independent published
implementation instead — scipy.ndimage.map_coordinates(order=3,
mode="grid-wrap", prefilter=True) (scipy 1.x, the periodic cubic B-spline
interpolant with the same prefilter) — and by the interpolant's defining
properties:
* oracle.sample_bspline == scipy and CUDA sample_nd("bspline") == scipy at
  random points (f64 1e-12);
* interpolation condition — the interpolant reproduces the samples at every
  node (prefilter exactness);
* 4th-order accuracy on a smooth periodic function;
* CUDA sample_nd("bspline") == oracle at random points (f64 1e-12, f32 1e-5);
* fp32 TMA SL engine with B-spline weights == f64 generic engine (1e-5).
"""
import numpy as np
import pytest

from oracle import flowreg_oracle as O


def test_oracle_bspline_matches_scipy():
    ndimage = pytest.importorskip("scipy.ndimage")
    rng = np.random.default_rng(7)
    for shape in ((12, 10, 16), (20, 24)):
        u = rng.standard_normal(shape)
        qs = [rng.uniform(-5, n + 5, 800) for n in shape]
        ref = ndimage.map_coordinates(u, np.array(qs), order=3, mode="grid-wrap", prefilter=True)
        got = O.sample_bspline(u, qs)
        assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-13


def test_oracle_bspline_interpolates_nodes():
    rng = np.random.default_rng(0)
    u = rng.standard_normal((12, 10, 16))
    qs = [g.ravel().astype(np.float64) for g in np.meshgrid(*[np.arange(n) for n in u.shape], indexing="ij")]
    got = O.sample_bspline(u, qs).reshape(u.shape)
    assert np.max(np.abs(got - u)) < 1e-12


def test_oracle_bspline_fourth_order():
    errs = []
    for n in (16, 32, 64):
        x = 2 * np.pi * np.arange(n) / n
        u = np.sin(x)[:, None] * np.cos(2 * x)[None, :]
        q0 = np.linspace(0, n, 97, endpoint=False) + 0.37
        q1 = np.linspace(0, n, 97, endpoint=False) + 0.61
        exact = np.sin(2 * np.pi * q0 / n) * np.cos(4 * np.pi * q1 / n)
        errs.append(np.max(np.abs(O.sample_bspline(u, [q0, q1]) - exact)))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates > 3.7), (errs, rates)


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch


@pytest.mark.gpu
def test_sample_nd_bspline_matches_scipy():
    _gpu()
    ndimage = pytest.importorskip("scipy.ndimage")
    from paper_2401_17493_b200._kernels import sample_nd

    rng = np.random.default_rng(3)
    u = rng.standard_normal((16, 24, 32))
    qs = [rng.uniform(-5, n + 5, 4000) for n in u.shape]
    ref = ndimage.map_coordinates(u, np.array(qs), order=3, mode="grid-wrap", prefilter=True)
    got = sample_nd(u, qs, "bspline")
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
def test_sample_nd_bspline_matches_oracle(dtype, tol):
    _gpu()
    from paper_2401_17493_b200._kernels import sample_nd

    rng = np.random.default_rng(1)
    u = rng.standard_normal((16, 24, 32)).astype(dtype)
    qs = [rng.uniform(-5, n + 5, 4000) for n in u.shape]
    got = sample_nd(u, qs, "bspline")
    ref = O.sample_bspline(u.astype(np.float64), qs)
    assert got.dtype == dtype
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < tol


@pytest.mark.gpu
def test_bspline_sl_engine_fp32_matches_f64():
    """SL state transport with B-spline: fp32 TMA engine vs f64 generic engine."""
    torch = _gpu()
    import paper_2401_17493_b200 as F
    from paper_2401_17493_b200 import transport

    n = 64
    m0, _, vtrue = F.synth_case("rotation", n, seed=1, d=3)
    v = F.VectorField._wrap(m0.grid, 0.5 * vtrue.data)
    r64 = transport.solve_state(m0, v, method="bspline").final().values
    g32 = m0.grid.with_dtype(np.float32)
    m32 = F.ScalarField._wrap(g32, m0.values.float())
    v32 = F.VectorField._wrap(g32, v.data.float())
    r32 = transport.solve_state(m32, v32, method="bspline").final().values
    rel = float((r32.double() - r64).norm() / r64.norm())
    assert rel < 1e-5, rel
    # and it is a different (smoother) interpolant than cubic Lagrange
    rl = transport.solve_state(m0, v, method="cubic").final().values
    assert float((rl - r64).norm() / r64.norm()) > 1e-7


@pytest.mark.gpu
def test_bspline_registration_converges():
    _gpu()
    import paper_2401_17493_b200 as F

    m0, m1, _ = F.synth_case("rotation", 32, seed=1, d=3)
    reg = F.RegConfig(alpha=1e-2)
    _, rep = F.register(m0, m1, reg=reg, precond=F.PrecondKind("reg"), method="bspline", transport_dtype=np.float32)
    assert rep.status == "converged" and rep.mismatch < 0.5, rep


@pytest.mark.gpu
@pytest.mark.parametrize("shape,dtype,tol", [((72, 68, 80), np.float64, 1e-12), ((40, 48, 64), np.float32, 1e-5),
                                             ((40, 96), np.float32, 1e-5),
                                             # fused axes-2+1 kernel (n2 in {128, 256, 512}, n1 % 32 == 0)
                                             ((36, 64, 128), np.float32, 1e-5), ((34, 32, 256), np.float32, 1e-5),
                                             # axes shorter than a column tile (8 Q R + 2K rows)
                                             ((64, 64, 64), np.float32, 1e-5)])
def test_fir_prefilter_matches_oracle(shape, dtype, tol):
    """Grids whose axes are all >= 2K + 2 take the separable FIR prefilter
    (csrc/bspline.cu) instead of the spectral round trip: same interpolant
    as the oracle's spectral restatement, and as the library's own spectral
    path (FRG_BSPLINE_SPECTRAL=1) to rounding."""
    import os

    _gpu()
    from paper_2401_17493_b200._kernels import sample_nd

    rng = np.random.default_rng(5)
    u = rng.standard_normal(shape).astype(dtype)
    qs = [rng.uniform(-5, n + 5, 6000) for n in u.shape]
    got = sample_nd(u, qs, "bspline")
    ref = O.sample_bspline(u.astype(np.float64), qs)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < tol
    os.environ["FRG_BSPLINE_SPECTRAL"] = "1"
    try:
        spec = sample_nd(u, qs, "bspline")
    finally:
        del os.environ["FRG_BSPLINE_SPECTRAL"]
    assert np.max(np.abs(got - spec)) / np.max(np.abs(spec)) < (1e-13 if dtype == np.float64 else 2e-6)
