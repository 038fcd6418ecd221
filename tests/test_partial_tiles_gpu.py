"""The TMA engine on grids whose extents are not multiples of its 32 x 8 x 4
voxel tiles (even extents, as fields.py:54-80 requires; partial tiles on
every axis: masked voxels, tile plans of edge tiles, the IncFirst TMA
epilogue's out-of-range boxes, periodic patches on non-power-of-two axes)
against the CPU oracle (oracle/flowreg_oracle.py, kkt.py:136-265): mixed
precision within the north-star fp32 bar (rel-L2 1e-5), f64 within 1e-10,
and a grid below the TMA box (cp.async staging) for the same checks."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
from inputs import bump, smooth_scalar, smooth_vector  # noqa: E402


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("shape", [(14, 18, 68), (18, 22, 100), (10, 14, 36)],
                         ids=["tma-14x18x68", "tma-18x22x100", "staged-10x14x36"])
@pytest.mark.parametrize("method", ["cubic", "linear"])
def test_partial_tiles_match_oracle(shape, method):
    import paper_2401_17493_b200 as F
    from oracle import flowreg_oracle as O

    rng = np.random.default_rng(7)
    m0 = bump(shape, rng.uniform(-1, 1, size=3)) + 0.05 * smooth_scalar(rng, shape)
    v_true = smooth_vector(rng, shape, 2.0, kmax=3)  # feet several cells away: boxes wrap every face
    y = O.departure(v_true, 1.0 / 16, "cubic")
    m1 = O.solve_state(m0, y, 16, "cubic")[-1]
    v = 0.5 * v_true
    vt = smooth_vector(rng, shape, 0.1, kmax=4)

    ok = O.Kkt(m0, m1, O.Reg(alpha=1e-2, incomp="near-incompressible", beta=1e-4), 4, "ssd", method, "fd8", v)
    ref_h, ref_g, ref_j = ok.hessian_matvec(vt), ok.gradient(), ok.objective()

    grid = F.Grid(shape, n_t=4)
    reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
    for tdt, tol in ((np.float32, 1e-5), (None, 1e-10)):
        st = F.KktState(F.ScalarField(grid, m0), F.ScalarField(grid, m1), reg, method=method,
                        v_init=F.VectorField(grid, v), transport_dtype=tdt)
        for _ in range(3):  # eager, capture, replay on small grids
            h = st.hessian_matvec(F.VectorField(grid, vt)).data.cpu().numpy()
            assert _rel(h, ref_h) < tol, (shape, method, tdt, _rel(h, ref_h))
        g = st.gradient().data.cpu().numpy()
        assert _rel(g, ref_g) < tol, (shape, method, tdt, _rel(g, ref_g))
        assert abs(st.objective() - ref_j) <= 10 * tol * abs(ref_j)

