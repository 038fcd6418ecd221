"""Deterministic input generators shared by make_golden.py and the tests.

Golden fixtures store only reference OUTPUTS; the inputs are regenerated from
these seeded generators (numpy default_rng + ifftn) on both sides.
"""
from __future__ import annotations

import math

import numpy as np

SEED = 20240817


def axis_nodes(n_i):
    h = 2.0 * math.pi / n_i
    return ((n_i // 2) - (np.arange(n_i, dtype=np.float64) + 1.0)) * h


def smooth_scalar(rng, n, kmax=3, modes=8):
    spec = np.zeros(n, dtype=complex)
    for _ in range(modes):
        k = tuple(int(rng.integers(-kmax, kmax + 1)) % ni for ni in n)
        spec[k] += rng.standard_normal() + 1j * rng.standard_normal()
    f = np.fft.ifftn(spec).real
    return f / max(np.abs(f).max(), 1e-30)


def smooth_vector(rng, n, amp, kmax=3):
    return np.stack([amp * smooth_scalar(rng, n, kmax) for _ in range(len(n))])


def bump(n, centers, kappa=1.5):
    xs = np.meshgrid(*[axis_nodes(ni) for ni in n], indexing="ij", sparse=True)
    out = np.ones(n)
    for c, x in zip(centers, xs):
        out = out * np.exp(kappa * (np.cos(x - c) - 1.0))
    return out


# -- per-fixture input sets ---------------------------------------------------

SAMPLE_SHAPES = [(16, 12, 10), (16, 12)]


def sample_inputs(shape, rng):
    d = len(shape)
    vals = rng.standard_normal(shape)
    q = rng.uniform(-30.0, 30.0, size=(d, 700))
    q[:, :40] = np.round(q[:, :40])  # exact integers
    q[:, 40:80] = np.round(q[:, 40:80]) + 0.5  # half-integers (nearest ties)
    q[:, 80:90] = -0.5
    labels = rng.integers(0, 7, size=shape).astype(np.int32)
    return vals, q, labels


DIFFOPS_SHAPES = [(16, 12, 12), (16, 12)]
FILTER_SHAPES = [(16, 20, 24), (16, 20)]
REG_VARIANTS = [(1, True), (2, True), (3, False)]


def diffops_inputs(shape, rng):
    d = len(shape)
    u = smooth_scalar(rng, shape, kmax=5) + 0.1 * rng.standard_normal(shape)
    v = smooth_vector(rng, shape, 0.7, kmax=5) + 0.05 * rng.standard_normal((d, *shape))
    return u, v


def filter_inputs(shape, rng):
    u = smooth_scalar(rng, shape, kmax=6) + 0.1 * rng.standard_normal(shape)
    uc = smooth_scalar(rng, tuple(s // 2 for s in shape), kmax=2)
    return u, uc


# (12, 16, 64): every axis >= the fp32 TMA engine's box edge (csrc/sl_fast.cuh
# tma_grid_ok), so the f32 transports run the TMA box + periodic patch path
TRANSPORT_SHAPES = [(16, 12, 12), (16, 12), (12, 16, 64)]


def transport_tag(shape):
    """Fixture key prefix of a transport shape."""
    return "3d_tma" if shape == (12, 16, 64) else f"{len(shape)}d"


def transport_inputs(shape, rng):
    d = len(shape)
    m0 = bump(shape, rng.uniform(-1, 1, size=d)) + 0.05 * smooth_scalar(rng, shape)
    v = smooth_vector(rng, shape, 0.8, kmax=2)
    vt = smooth_vector(rng, shape, 1.0, kmax=3)
    lam1 = smooth_scalar(rng, shape, kmax=3)
    return m0, v, vt, lam1


# name, shape, reg kwargs, distance, method, preconds to record
KKT_CASES = [
    ("h1_none_ssd_cubic", (16, 12, 12), dict(order=1, incomp="none"), "ssd", "cubic", ("reg", "h0")),
    ("h1_near_ssd_cubic", (20, 20, 24), dict(order=1, incomp="near-incompressible"), "ssd", "cubic",
     ("reg", "h0", "2level")),
    ("h2_incomp_ssd_linear", (16, 12, 12), dict(order=2, incomp="incompressible"), "ssd", "linear",
     ("reg",)),
    ("h1_none_ncc_cubic", (16, 12, 12), dict(order=1, incomp="none"), "ncc", "cubic", ("reg",)),
    ("h3f_near_ssd_cubic_2d", (24, 20), dict(order=3, seminorm=False, incomp="near-incompressible"),
     "ssd", "cubic", ("reg", "h0", "2level")),
    # shapes on which the mixed / f32 contexts run the bench's engine: TMA
    # boxes, per-map tile plans, periodic patches on every face (n0 = 12 is
    # one box deep, so every tile wraps along axis 0)
    ("tma_h1_near_ssd_cubic", (12, 16, 64), dict(order=1, incomp="near-incompressible"), "ssd", "cubic",
     ("reg",)),
    ("tma_h2_near_ssd_linear", (12, 16, 96), dict(order=2, incomp="near-incompressible"), "ssd", "linear",
     ("reg",)),
    # 20x the velocity: departure displacements of up to ~19 columns / 6 rows /
    # 4 planes whose spread inside a tile overflows the fixed TMA box, so part
    # of the tiles take the global-memory fallback (global_interp)
    ("tma_wide_h1_none_ssd_cubic", (12, 16, 64), dict(order=1, incomp="none"), "ssd", "cubic", ("reg",)),
]
KKT_VSCALE = {"tma_wide_h1_none_ssd_cubic": 20.0}


def kkt_case_inputs(case, rng):
    """Inputs of one KKT_CASES entry (consumes ``rng`` in case order)."""
    return kkt_inputs(case[1], rng, KKT_VSCALE.get(case[0], 1.0))


def kkt_inputs(shape, rng, vscale=1.0):
    d = len(shape)
    m0 = bump(shape, rng.uniform(-1, 1, size=d)) + 0.2
    m1 = bump(shape, rng.uniform(-1, 1, size=d)) + 0.2
    v = smooth_vector(rng, shape, 0.5 * vscale, kmax=2)
    vt = smooth_vector(rng, shape, 1.0, kmax=3)
    r = smooth_vector(rng, shape, 1.0, kmax=4)
    return m0, m1, v, vt, r


# name, synth (case, n, seed, d), reg kwargs, precond, method, store_v
REGISTER_CASES = [
    ("swirl2d_reg", ("swirl", 32, 1, 2), dict(order=1, incomp="none"), "reg", "cubic", True),
    ("swirl2d_2level_near", ("swirl", 32, 1, 2), dict(order=1, incomp="near-incompressible"),
     "2level", "cubic", True),
    ("rot2d_h2_linear_h0", ("rotation", 64, 3, 2), dict(order=2, incomp="none"), "h0", "linear", True),
    ("rot3d_reg", ("rotation", 32, 1, 3), dict(order=1, incomp="none"), "reg", "cubic", True),
    ("c1_rot64_reg", ("rotation", 64, 1, 3), dict(order=1, incomp="none"), "reg", "cubic", False),
]

# BASELINE.json config C2: brain-like 128^3 (paper_2401_17493_b200.synth.
# brain_arrays), H2 seminorm, linear interpolation, near-incompressible
# (beta 1e-4), alpha 1e-3, spectral (reg) preconditioner.
# name, (n, seed), reg kwargs, precond, method
C2_CASES = [
    ("c2_brain128_h2_linear", (128, 1), dict(order=2, incomp="near-incompressible", alpha=1e-3), "reg", "linear"),
]
