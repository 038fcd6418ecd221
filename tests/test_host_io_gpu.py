"""KktState.hessian_matvec with host (pinned) buffers: the pipelined
H2D / matvec / D2H path returns exactly the device-path result, also when
several calls are in flight on the two staging slots."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2401_17493_b200 as F  # noqa: E402


def test_host_io_matvec_matches_device():
    m0, m1, vtrue = F.synth_case("rotation", 32, seed=1, d=3)
    st = F.KktState(m0, m1, F.RegConfig(alpha=1e-2), v_init=F.VectorField._wrap(m0.grid, 0.5 * vtrue.data),
                    transport_dtype=np.float32)
    gen = torch.Generator(device="cuda").manual_seed(3)
    vts = [0.1 * torch.randn((3, 32, 32, 32), generator=gen, dtype=torch.float64, device="cuda") for _ in range(5)]
    ref = [st.hessian_matvec(F.VectorField._wrap(m0.grid, v)).data.cpu() for v in vts]
    host_in = [v.cpu().pin_memory() for v in vts]
    host_out = [torch.empty_like(h).pin_memory() for h in host_in]
    for hi, ho in zip(host_in, host_out):
        st.hessian_matvec(hi, out=ho)
    st.wait_host_io()
    torch.cuda.synchronize()
    for r, ho in zip(ref, host_out):
        assert torch.equal(r, ho)
