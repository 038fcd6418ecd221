"""BASELINE.json configs pinned directly against the reference.

* C2 (brain-like 128^3, H2 seminorm, linear interpolation, near-incompressible,
  alpha 1e-3, reg preconditioner): the reference itself registered the pair at
  f64 (tests/golden/make_golden.py gen_c2: 3 Newton iterations, 11 matvecs,
  33 PDE solves, PCG 1/3/7).  The device generator (synth.brain_arrays + the
  64-step cubic transport) must reproduce the reference's m1, and the device
  solve must reproduce the reference's counts in f64, in the mixed (bench)
  precision and in the fp16-tap precision (north star: 1e-3 tolerance there).
* C3 (256^3): the mixed-precision gradient and GN matvec against the CPU
  oracle port (f64) at rel-L2 1e-5 (the north-star fp32 bar).
"""
import numpy as np
import pytest

import inputs as I
from conftest import rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2401_17493_b200 as F  # noqa: E402


def _reg(kw):
    return F.RegConfig(alpha=kw.get("alpha", 1e-2), operator=F.RegOperatorSpec(kw.get("order", 1), True),
                       incomp=F.IncompressibilityMode(kw.get("incomp", "none"), 1e-4))


@pytest.fixture(scope="module")
def c2_pair():
    name, (n, seed), regkw, pre, method = I.C2_CASES[0]
    m0, m1, _ = F.synth_case(F.BRAIN_CASE, n, seed=seed, d=3)
    return m0, m1


def test_c2_generator_matches_reference(golden, c2_pair):
    name = I.C2_CASES[0][0]
    meta = golden("c2.json")[name]
    m0, m1 = c2_pair
    assert float(m0.values.sum()) == pytest.approx(meta["m0_sum"], rel=1e-12)
    assert float(m1.values.sum()) == pytest.approx(meta["m1_sum"], rel=1e-10)
    assert float((m1.values * m1.values).sum()) == pytest.approx(meta["m1_sumsq"], rel=1e-10)
    sub = m1.values[::4, ::4, ::4].cpu().numpy()
    assert np.max(np.abs(sub - golden("c2.npz")[name + "_m1_sub"])) < 1e-9


@pytest.mark.parametrize("mode", ["f64", "mixed", "fp16"])
def test_c2_registration_matches_reference(golden, c2_pair, mode):
    name, _, regkw, pre, method = I.C2_CASES[0]
    meta = golden("c2.json")[name]
    m0, m1 = c2_pair
    kw = {} if mode == "f64" else dict(transport_dtype=np.float32)
    if mode == "fp16":
        kw["interp_precision"] = "fp16"
    v, rep = F.register(m0, m1, reg=_reg(regkw), precond=F.PrecondKind(pre), method=method, scheme="fd8", **kw)
    print(f"C2 {mode}: iterations {rep.iterations} matvecs {rep.matvecs} pde {rep.pde_solves} "
          f"pcg {[t['pcg_iterations'] for t in rep.trace]} mismatch {rep.mismatch:.8f} "
          f"(reference {meta['mismatch']:.8f}) runtime {rep.runtime:.3f} s")
    assert rep.status == meta["status"] and rep.exit_reason == meta["exit_reason"]
    assert (rep.iterations, rep.matvecs, rep.pde_solves, rep.line_search_evals) == \
        (meta["iterations"], meta["matvecs"], meta["pde_solves"], meta["line_search_evals"])
    assert [t["pcg_iterations"] for t in rep.trace] == [t["pcg_iterations"] for t in meta["trace"]]
    rt = {"f64": 1e-6, "mixed": 1e-5, "fp16": 1e-3}[mode]
    assert rep.mismatch == pytest.approx(meta["mismatch"], rel=rt)
    assert rep.detgrad_min == pytest.approx(meta["detgrad_min"], rel=rt)
    vsub = v.data[:, ::4, ::4, ::4].cpu().numpy()
    assert rel_l2(vsub, golden("c2.npz")[name + "_v_sub"]) < max(rt, 1e-5)


def test_c3_mixed_matches_oracle_at_256():
    """One 256^3 mixed-precision gradient + GN matvec (the bench's unit of work)
    against the f64 CPU oracle port on the same inputs."""
    from oracle import flowreg_oracle as O

    n = 256
    m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3)
    reg = F.RegConfig(alpha=1e-2, operator=F.RegOperatorSpec(1, True),
                      incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
    v = F.VectorField._wrap(m0.grid, 0.5 * vtrue.data)
    rng = np.random.default_rng(0)
    vt = 0.1 * rng.standard_normal((3, n, n, n))
    st = F.KktState(m0, m1, reg, v_init=v, transport_dtype=np.float32)
    g = st.gradient().data.cpu().numpy()
    h = st.hessian_matvec(F.VectorField(m0.grid, vt)).data.cpu().numpy()
    obj = st.objective()
    del st
    m0n, m1n, vn = m0.values.cpu().numpy(), m1.values.cpu().numpy(), v.data.cpu().numpy()
    ok = O.Kkt(m0n, m1n, O.Reg(alpha=1e-2, incomp="near-incompressible", beta=1e-4), 4, "ssd", "cubic", "fd8", vn)
    eg = rel_l2(g, ok.gradient())
    eh = rel_l2(h, ok.hessian_matvec(vt))
    print(f"256^3 mixed vs oracle: gradient rel-L2 {eg:.2e}, matvec rel-L2 {eh:.2e}")
    assert eg < 1e-5 and eh < 1e-5
    assert obj == pytest.approx(ok.objective(), rel=1e-6)
