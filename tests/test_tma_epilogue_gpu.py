"""The TMA-fed IncFirstOp epilogue (csrc/transport_inc.cu) and the
programmatic dependent launches of the SL steps at the bench's engine path
(64^3: every axis reaches the TMA box), for every n_t parity of the epilogue
rounds (two time levels per round): bit-identical to the per-element
cp.async epilogue (FRG_NO_TMA_EPILOGUE=1, same arithmetic order) and within
the north-star fp32 bar of the f64 context."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _rel(a, b):
    return float((a - b).norm() / b.norm())


@pytest.mark.parametrize("n_t", [1, 3, 4, 5])
def test_tma_epilogue_matches_cp_async_and_f64(n_t):
    import paper_2401_17493_b200 as F

    n = 64
    m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3, n_t=n_t)
    reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
    v = F.VectorField._wrap(m0.grid, 0.5 * vtrue.data)
    gen = torch.Generator(device="cuda").manual_seed(0)
    vt = F.VectorField._wrap(m0.grid, 0.1 * torch.randn((3, n, n, n), generator=gen, dtype=torch.float64,
                                                          device="cuda"))
    mixed = F.KktState(m0, m1, reg, v_init=v, transport_dtype=np.float32)
    h_tma = mixed.hessian_matvec(vt).data.clone()
    os.environ["FRG_NO_TMA_EPILOGUE"] = "1"
    try:
        h_cp = mixed.hessian_matvec(vt).data.clone()
    finally:
        del os.environ["FRG_NO_TMA_EPILOGUE"]
    assert torch.equal(h_tma, h_cp)
    ref = F.KktState(m0, m1, reg, v_init=v)
    assert _rel(h_tma, ref.hessian_matvec(vt).data) < 1e-5
