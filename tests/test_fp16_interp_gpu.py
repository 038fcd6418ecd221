"""Mixed-precision fp16 interpolation mode (north star: 1e-3 vs the f64
reference).  The f64 context is pinned to the reference (test_gpu_parity.py,
<= 1e-10), so the fp16-tap context is checked against it at 64^3 / 128^3,
where the fp16 TMA engine is active (rows of >= 64 columns)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2401_17493_b200 as F  # noqa: E402


def _rel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm())


@pytest.mark.parametrize("method,order", [("cubic", 1), ("linear", 2)])
def test_fp16_interp_matches_f64(method, order):
    n = 64
    m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
    reg = F.RegConfig(alpha=1e-2, operator=F.RegOperatorSpec(order, True))
    v = F.VectorField._wrap(m0.grid, 0.5 * vtrue.data)
    ref = F.KktState(m0, m1, reg, method=method, v_init=v)
    h16 = F.KktState(m0, m1, reg, method=method, v_init=v, transport_dtype=np.float32, interp_precision="fp16")
    h32 = F.KktState(m0, m1, reg, method=method, v_init=v, transport_dtype=np.float32)
    gen = torch.Generator(device="cuda").manual_seed(0)
    vt = F.VectorField._wrap(m0.grid, 0.1 * torch.randn((3, n, n, n), generator=gen, dtype=torch.float64,
                                                       device="cuda"))
    r = ref.hessian_matvec(vt).data
    o16 = h16.hessian_matvec(vt).data
    o32 = h32.hessian_matvec(vt).data
    e16, e32 = _rel(o16, r), _rel(o32, r)
    print(f"fp16 interpolation ({method}): matvec rel-L2 {e16:.2e} vs f64 (fp32: {e32:.2e})")
    assert e16 < 1e-3, e16
    assert e32 < 1e-5, e32
    # the fp16 taps are really used (with H2 the alpha L part dominates the
    # random direction's matvec, so the transport difference can sit below the
    # fp32 inverse-FFT rounding in e16 vs e32)
    assert not torch.equal(o16, o32)
    # state / adjoint / gradient keep fp32 taps: identical to the fp32 context
    assert torch.equal(h16.gradient().data, h32.gradient().data)
    assert h16.objective() == h32.objective()


def test_fp16_interp_registration():
    m0, m1, _ = F.synth_case("rotation", 64, seed=1, d=3)
    reg = F.RegConfig(alpha=1e-2)
    _, r16 = F.register(m0, m1, reg=reg, precond=F.PrecondKind("reg"), transport_dtype=np.float32,
                        interp_precision="fp16", compute_detgrad=False)
    _, r64 = F.register(m0, m1, reg=reg, precond=F.PrecondKind("reg"), compute_detgrad=False)
    assert r16.status == "converged" and r16.iterations == r64.iterations, (r16, r64)
    assert abs(r16.mismatch - r64.mismatch) < 1e-3 * max(r64.mismatch, 1e-3) * 10
