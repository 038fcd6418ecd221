"""KktState lifecycle on the bench's engine path (64^3, and 32^3 where the
small-grid CUDA graph replays the matvec): the grad m_j(y) cache the GN
matvec reads is gathered lazily by the first matvec after each refresh
(csrc/kkt.cu ensure_grads_y), so a context that is refreshed to a new
velocity — with or without matvecs, gradients, Armijo trials and
preconditioner calls in between — must give bit-identical results to a fresh
context created at that velocity (kkt.py:166-265 semantics: every query
answers for the current v)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.mark.parametrize("n", [32, 64])
@pytest.mark.parametrize("tdt", [np.float32, None], ids=["mixed", "f64"])
def test_refreshed_context_equals_fresh_context(n, tdt):
    import paper_2401_17493_b200 as F

    m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
    grid = m0.grid
    reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
    gen = torch.Generator(device="cuda").manual_seed(3)
    vt = F.VectorField._wrap(grid, 0.1 * torch.randn((3, n, n, n), generator=gen, dtype=torch.float64,
                                                     device="cuda"))
    v1 = F.VectorField._wrap(grid, 0.3 * vtrue.data)
    v2 = F.VectorField._wrap(grid, 0.6 * vtrue.data)
    v3 = F.VectorField._wrap(grid, 0.45 * vtrue.data)

    st = F.KktState(m0, m1, reg, v_init=v1, transport_dtype=tdt)
    for _ in range(3):  # past the graph-capture threshold on small grids
        st.hessian_matvec(vt)
    st.refresh(v2)  # no matvec at v2: the cache stays stale until v3's first matvec
    st.gradient()
    st.objective_at(v1)
    st.apply_precond(vt, F.PrecondKind("reg"), 0.5)
    st.refresh(v3)
    got = [st.hessian_matvec(vt).data.clone() for _ in range(3)]
    g_got = st.gradient().data.clone()

    fresh = F.KktState(m0, m1, reg, v_init=v3, transport_dtype=tdt)
    want = fresh.hessian_matvec(vt).data
    assert all(torch.equal(h, want) for h in got)
    assert torch.equal(g_got, fresh.gradient().data)
    assert st.objective() == fresh.objective()


@pytest.mark.parametrize("n", [32, 64])
def test_refresh_at_the_accepted_trial_reuses_its_map_bit_for_bit(n):
    """A refresh at the velocity of the last objective_at (the accepted Armijo
    trial) takes that trial's departure map instead of rebuilding it (mixed
    precision; csrc/kkt.cu trial_map_matches); a matvec in between, or a
    different velocity, falls back to building it.  Either way the state is
    bit-identical to a fresh context's."""
    import paper_2401_17493_b200 as F

    m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
    grid = m0.grid
    reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
    gen = torch.Generator(device="cuda").manual_seed(5)
    vt = F.VectorField._wrap(grid, 0.1 * torch.randn((3, n, n, n), generator=gen, dtype=torch.float64,
                                                     device="cuda"))
    v1 = F.VectorField._wrap(grid, 0.3 * vtrue.data)
    v2 = F.VectorField._wrap(grid, 0.55 * vtrue.data)
    st = F.KktState(m0, m1, reg, v_init=v1, transport_dtype=np.float32)
    for sequence in ("accepted", "matvec-between", "other-velocity"):
        st.objective_at(v2)
        if sequence == "matvec-between":
            st.hessian_matvec(vt)
        target = v2 if sequence != "other-velocity" else v1
        st.refresh(target)
        fresh = F.KktState(m0, m1, reg, v_init=target, transport_dtype=np.float32)
        assert torch.equal(st.gradient().data, fresh.gradient().data), sequence
        assert torch.equal(st.hessian_matvec(vt).data, fresh.hessian_matvec(vt).data), sequence
        assert st.objective() == fresh.objective(), sequence
        st.refresh(v1)
