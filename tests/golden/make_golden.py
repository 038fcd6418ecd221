#!/usr/bin/env python3
"""Generate golden vectors by running the REFERENCE flowreg package itself.

Run in the build container (the reference tree exists only here):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py [sections...]

Inputs come from the seeded generators in ``inputs.py`` (re-run by the tests);
only the reference's outputs are written (small .npz / .json files next to
this script).  They pin the CPU oracle (oracle/flowreg_oracle.py) and the
CUDA path.  Nothing at test or bench time reads /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_cache")

import inputs as I  # noqa: E402
from flowreg import _kernels, diffops, kkt, optimizer, synth, transport  # noqa: E402
from flowreg.continuation import cascade_alphas, det_bounds_ok  # noqa: E402
from flowreg.fields import Grid, ScalarField, VectorField  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, out):
    np.savez_compressed(os.path.join(OUT, name), **out)


def gen_sample():
    rng = np.random.default_rng(I.SEED)
    out = {}
    for shape in I.SAMPLE_SHAPES:
        t = f"{len(shape)}d"
        vals, q, labels = I.sample_inputs(shape, rng)
        qs = [np.ascontiguousarray(q[i]) for i in range(len(shape))]
        for method in ("nearest", "linear", "cubic"):
            out[f"{t}_{method}_f64"] = _kernels.sample_nd(vals, qs, method)
            out[f"{t}_{method}_f32"] = _kernels.sample_nd(vals.astype(np.float32), qs, method)
        out[f"{t}_nearest_i32"] = _kernels.sample_nd(labels, qs, "nearest")
    save("sample.npz", out)


def gen_diffops():
    rng = np.random.default_rng(I.SEED + 1)
    out = {}
    for shape in I.DIFFOPS_SHAPES:
        t = f"{len(shape)}d"
        g = Grid(shape)
        u, v = I.diffops_inputs(shape, rng)
        U, V = ScalarField(g, u), VectorField(g, v)
        out[f"{t}_fd8_grad"] = diffops.fd8_gradient(U).data
        out[f"{t}_spec_grad"] = diffops.spectral_gradient(U).data
        out[f"{t}_div_fd8"] = diffops.divergence(V, "fd8").values
        out[f"{t}_div_spec"] = diffops.divergence(V, "spectral").values
        out[f"{t}_jacobian"] = diffops.jacobian(V, "fd8")
        out[f"{t}_laplacian"] = diffops.laplacian(U).values
        for order, semi in I.REG_VARIANTS:
            spec = diffops.RegOperatorSpec(order, semi)
            k = f"{t}_o{order}{'s' if semi else 'f'}"
            out[k + "_L"] = diffops.apply_reg_operator(V, spec, 0.03).data
            out[k + "_Linv"] = diffops.apply_inv_reg_operator(V, spec, 0.03).data
            out[k + "_Linvsqrt"] = diffops.apply_inv_sqrt_reg_operator(V, spec, 0.03).data
        out[f"{t}_proj_incomp"] = diffops.project_body_force(
            V, diffops.IncompressibilityMode("incompressible"), 0.01).data
        out[f"{t}_proj_near"] = diffops.project_body_force(
            V, diffops.IncompressibilityMode("near-incompressible", 1e-4), 0.01).data
    for shape in I.FILTER_SHAPES:
        t = f"{len(shape)}d"
        g = Grid(shape)
        u, uc = I.filter_inputs(shape, rng)
        U = ScalarField(g, u)
        out[f"{t}_lowpass"] = diffops.low_pass(U).values
        out[f"{t}_highpass"] = diffops.high_pass(U).values
        out[f"{t}_restrict"] = diffops.restrict(U).values
        out[f"{t}_prolong"] = diffops.prolong(ScalarField(g.coarsen(), uc), g).values
    save("diffops.npz", out)


def gen_transport():
    rng = np.random.default_rng(I.SEED + 2)
    out = {}
    for shape in I.TRANSPORT_SHAPES:
        t = I.transport_tag(shape)
        g = Grid(shape, n_t=4)
        m0, v, vt, lam1 = I.transport_inputs(shape, rng)
        V = VectorField(g, v)
        for method in ("cubic", "linear"):
            k = f"{t}_{method}"
            traj = transport.Trajectory.compute(V, method)
            back = transport.Trajectory.compute(VectorField(g, -v), method)
            out[k + "_y"] = traj.step_points.data
            out[k + "_yb"] = back.step_points.data
            ms = transport.solve_state(ScalarField(g, m0), V, method, traj)
            out[k + "_state"] = ms.data
            out[k + "_adjoint"] = transport.solve_adjoint(ScalarField(g, lam1), V, method, "fd8", back).data
            out[k + "_incstate"] = transport.solve_inc_state(ms, V, VectorField(g, vt), method, "fd8",
                                                             traj).data[-1]
            F = transport.solve_deformation_tensor(V, method, "fd8", traj)
            out[k + "_det"] = F.determinant().values
            out[k + "_F00"] = F.data[0, 0]
            out[k + "_composed"] = transport.compose_trajectory(V, method).data
    save("transport.npz", out)


def make_reg(order=1, seminorm=True, incomp="none", alpha=1e-2, beta=1e-4):
    return kkt.RegConfig(alpha=alpha, operator=diffops.RegOperatorSpec(order, seminorm),
                         incomp=diffops.IncompressibilityMode(incomp, beta))


def gen_kkt():
    rng = np.random.default_rng(I.SEED + 3)
    out, meta = {}, {}
    for case in I.KKT_CASES:
        name, shape, regkw, dist, method, preconds = case
        g = Grid(shape, n_t=4)
        m0, m1, v, vt, r = I.kkt_case_inputs(case, rng)
        st = kkt.KktState(ScalarField(g, m0), ScalarField(g, m1), make_reg(**regkw), distance=dist,
                          method=method, scheme="fd8", v_init=VectorField(g, v))
        p = name + "_"
        out[p + "m_final"] = st.mseries.data[-1]
        out[p + "lam0"] = st.lamseries.data[0]
        out[p + "gradient"] = st.gradient().data
        out[p + "matvec"] = st.hessian_matvec(VectorField(g, vt)).data
        for kind in preconds:
            out[p + "precond_" + kind] = st.apply_precond(VectorField(g, r), kkt.PrecondKind(kind), 0.3).data
        meta[name] = dict(
            objective=st.objective(), objective_at=st.objective_at(VectorField(g, v + 0.1 * vt)),
            mismatch=st.mismatch(), divergence_energy=st.divergence_energy(),
            matvecs=st.matvecs, pde_solves=st.pde_solves, precond_fallbacks=st.precond_fallbacks,
        )
    save("kkt.npz", out)
    with open(os.path.join(OUT, "kkt.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def gen_register():
    out, meta = {}, {}
    for name, (case, n, seed, d), regkw, pre, method, store_v in I.REGISTER_CASES:
        m0, m1, _ = synth.synth_case(case, n, seed=seed, d=d)
        v, rep = optimizer.register(m0, m1, reg=make_reg(**regkw), precond=kkt.PrecondKind(pre),
                                    method=method, scheme="fd8")
        r = rep.to_dict()
        r.pop("runtime")
        meta[name] = r
        if store_v:
            out[name + "_v"] = v.data.astype(np.float32)
        print(name, r["iterations"], r["matvecs"], r["pde_solves"], r["status"], flush=True)
    save("register.npz", out)
    with open(os.path.join(OUT, "register.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def gen_synth():
    out = {}
    for case in ("translation", "rotation", "swirl", "compress"):
        m0, m1, v = synth.synth_case(case, 32, seed=2, d=2)
        out[f"{case}_m0"], out[f"{case}_m1"], out[f"{case}_v"] = m0.values, m1.values, v.data
    m0, m1, v = synth.synth_case("rotation", 32, seed=1, d=3)
    out["rot3d_m1"] = m1.values
    ok, dmin, dmax, dmean = det_bounds_ok(VectorField(Grid((32, 32)), out["compress_v"]), 0.1)
    meta = dict(cascade=cascade_alphas(1.773437e-3), compress_det=[bool(ok), dmin, dmax, dmean])
    save("synth.npz", out)
    with open(os.path.join(OUT, "misc.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def gen_c2():
    """BASELINE config C2: the brain-like 128^3 pair (inputs from the package's
    pure-torch generator run on the CPU, m1 from the reference's own 64-step
    cubic solve_state as synth.py:113-117 does), registered by the reference
    at f64 with H2 / linear / near-incompressible / reg preconditioner."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from paper_2401_17493_b200.synth import brain_arrays

    meta, out = {}, {}
    for name, (n, seed), regkw, pre, method in I.C2_CASES:
        vals, vtrue = brain_arrays(n, seed, 3, device="cpu")
        vals, vtrue = vals.numpy(), vtrue.numpy()
        g = Grid((n,) * 3, n_t=4)
        fine = g.with_time_steps(64)
        m1 = transport.solve_state(ScalarField(fine, vals), VectorField(fine, vtrue), method="cubic").final().values
        v, rep = optimizer.register(ScalarField(g, vals), ScalarField(g, m1), reg=make_reg(**regkw),
                                    precond=kkt.PrecondKind(pre), method=method, scheme="fd8")
        r = rep.to_dict()
        r.pop("runtime")
        r["m0_sum"], r["m1_sum"], r["m1_sumsq"] = float(vals.sum()), float(m1.sum()), float((m1 * m1).sum())
        meta[name] = r
        out[name + "_m1_sub"] = m1[::4, ::4, ::4].copy()
        out[name + "_v_sub"] = v.data[:, ::4, ::4, ::4].astype(np.float32)
        print(name, r["iterations"], r["matvecs"], r["pde_solves"], r["status"], flush=True)
    save("c2.npz", out)
    with open(os.path.join(OUT, "c2.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def main():
    which = sys.argv[1:] or ["sample", "diffops", "transport", "kkt", "synth", "register", "c2"]
    for w in which:
        globals()["gen_" + w]()


if __name__ == "__main__":
    main()
