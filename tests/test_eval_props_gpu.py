"""Property tests of the post-solve evaluation, the synthetic generator and
the CLF1 container, restating the reference's behavioural suite
(pkg/tests/test_metrics.py, test_synth.py, test_volio.py of the reference
package) in this repo's words: Dice counting, label transport (identity,
lattice translations = cyclic shifts, no new ids, agreement with the
thresholded linear transport), det F statistics, relative mismatch, the
synthetic pairs' design properties, CLF1 round trips and header errors.
"""
import csv
import struct

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU collection
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2401_17493_b200 as F  # noqa: E402
from paper_2401_17493_b200 import transport as T  # noqa: E402
from paper_2401_17493_b200 import volio  # noqa: E402
from paper_2401_17493_b200.distance import dist_value  # noqa: E402
from paper_2401_17493_b200.metrics import write_dice_csv  # noqa: E402
from paper_2401_17493_b200.synth import SYNTH_CASES  # noqa: E402


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def _lab(x):
    return x.labels.cpu().numpy() if isinstance(x.labels, torch.Tensor) else np.asarray(x.labels)


def _vals(x):
    t = x.values if isinstance(x, F.ScalarField) else x.data
    return t.cpu().numpy()


def half_plane(g, frac):
    lab = np.zeros(g.n, dtype=np.int32)
    lab[: int(g.n[0] * frac)] = 1
    return F.LabelVolume(g, lab)


def random_labels(g, rng, k):
    return F.LabelVolume(g, rng.integers(0, k, size=g.n).astype(np.int32))


def bandlimited(g, rng, amp=0.5, kmax=2, modes=6):
    data = np.zeros((g.d, *g.n))
    for i in range(g.d):
        spec = np.zeros(g.n, dtype=complex)
        for _ in range(modes):
            spec[tuple(int(rng.integers(0, kmax + 1)) for _ in range(g.d))] = \
                rng.standard_normal() + 1j * rng.standard_normal()
        f = np.fft.ifftn(spec).real
        data[i] = amp * f / np.abs(f).max()
    return F.VectorField(g, data)


# ---------------------------------------------------------------------------
# Dice (reference metrics.py:56-87)
# ---------------------------------------------------------------------------


def test_dice_identity_disjoint_and_half_overlap(rng):
    g = F.Grid((16, 16))
    lab = random_labels(g, rng, 4)
    res = F.dice(lab, lab)
    assert all(v == 1.0 for v in res.per_id.values()) and res.union == 1.0
    a = half_plane(g, 0.5)
    b = F.LabelVolume(g, np.flip(_lab(half_plane(g, 0.5)), axis=0).copy())
    res = F.dice(a, b)
    assert res.per_id[1] == 0.0 and res.union == 0.0
    res = F.dice(half_plane(g, 0.5), half_plane(g, 1.0))
    assert res.per_id[1] == pytest.approx(2.0 / 3.0, rel=1e-15)


def test_dice_empty_ids_flagged_symmetric_and_bounded(rng):
    g = F.Grid((16, 16))
    res = F.dice(half_plane(g, 0.5), half_plane(g, 0.5), ids=(1, 7))
    assert res.per_id[7] == 1.0 and res.empty_ids == (7,)
    a, b = random_labels(g, rng, 3), random_labels(g, rng, 3)
    assert F.dice(a, b).per_id == F.dice(b, a).per_id
    a, b = random_labels(g, rng, 5), random_labels(g, rng, 5)
    res = F.dice(a, b)
    assert all(0.0 <= v <= 1.0 for v in res.per_id.values()) and 0.0 <= res.union <= 1.0


# ---------------------------------------------------------------------------
# label transport (reference metrics.py:90-104, transport.py:224-247)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("shape", [(16, 16), (16, 16, 64)])
def test_label_transport_rest_is_identity_and_lattice_shift_is_cyclic(shape, rng):
    g = F.Grid(shape, n_t=4)
    lab = random_labels(g, rng, 4)
    assert np.array_equal(_lab(F.transport_labels(lab, F.VectorField.zeros(g))), _lab(lab))
    steps = (3, -2, 5)[: g.d]
    c = tuple(s * h for s, h in zip(steps, g.h))
    out = _lab(F.transport_labels(lab, F.VectorField.constant(g, c)))
    # coordinates decrease with index: x - c lands `steps` indices ahead
    assert np.array_equal(out, np.roll(_lab(lab), tuple(-s for s in steps), axis=tuple(range(g.d))))


def test_label_transport_creates_no_new_ids(rng):
    g = F.Grid((32, 32), n_t=4)
    lab = random_labels(g, rng, 5)
    out = F.transport_labels(lab, bandlimited(g, rng))
    assert set(np.unique(_lab(out))) <= set(np.unique(_lab(lab)))


def test_label_transport_agrees_with_thresholded_linear_transport(rng):
    g = F.Grid((64, 64), n_t=4)
    x = [np.broadcast_to(c, g.n) for c in g.coord_arrays()]
    bump = np.exp(1.5 * (np.cos(x[0] - 0.4) - 1.0)) * np.exp(1.5 * (np.cos(x[1] + 0.2) - 1.0))
    binary = (bump > 0.5).astype(np.int32)
    v = bandlimited(g, rng)
    moved = _lab(F.transport_labels(F.LabelVolume(g, binary), v)) == 1
    smooth = _vals(T.solve_state(F.ScalarField(g, binary.astype(np.float64)), v, method="linear").final()) >= 0.5
    assert np.logical_and(moved, smooth).sum() >= 0.95 * moved.sum()


# ---------------------------------------------------------------------------
# det F statistics, relative mismatch (reference metrics.py:107-155)
# ---------------------------------------------------------------------------


def test_detgrad_stats_rest_translation_and_ordering(rng):
    g = F.Grid((16, 16), n_t=2)
    assert F.detgrad_stats(F.VectorField.zeros(g)) == (1.0, 1.0, 1.0)
    dmin, _, dmax = F.detgrad_stats(F.VectorField.constant(g, (0.4, 0.2)))
    assert dmin == pytest.approx(1.0, abs=1e-12) and dmax == pytest.approx(1.0, abs=1e-12)
    dmin, dmean, dmax = F.detgrad_stats(bandlimited(F.Grid((32, 32)), rng, amp=0.6))
    assert dmin <= dmean <= dmax


def test_relative_mismatch_rest_identical_and_solver_report():
    m0, m1, _ = F.synth_case("rotation", 32, seed=1)
    res = F.relative_mismatch(m0, m1, F.VectorField.zeros(m0.grid))
    assert res.value == pytest.approx(1.0, rel=1e-12) and not res.degenerate
    g = F.Grid((16, 16), n_t=2)
    m = F.ScalarField.full(g, 0.3)
    assert tuple(F.relative_mismatch(m, m, F.VectorField.zeros(g))) == (0.0, True)
    reg = F.RegConfig(alpha=1e-2, incomp=F.IncompressibilityMode("none"))
    v, rep = F.register(m0, m1, reg=reg)
    assert F.relative_mismatch(m0, m1, v).value == rep.mismatch


def test_dice_csv_per_label_statistics(tmp_path):
    path = tmp_path / "dice.csv"
    write_dice_csv(path, {1: [0.5, 0.7], 2: [1.0]})
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["label_id", "mean", "stdev", "min", "max", "median", "q25", "q75"]
    assert len(rows) == 3 and float(rows[1][1]) == pytest.approx(0.6) and float(rows[2][2]) == 0.0


# ---------------------------------------------------------------------------
# synthetic pairs (reference synth.py:28-118)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", SYNTH_CASES)
def test_synthetic_pairs_are_nondegenerate(name):
    m0, m1, _ = F.synth_case(name, 32, seed=0)
    assert dist_value(m0, m1, "ssd") > 0.0
    vals = _vals(m0)
    assert 0.0 <= vals.min() and vals.max() <= 1.0


def test_synthetic_pairs_are_deterministic_per_seed():
    a, b, c = (F.synth_case("swirl", 32, seed=s) for s in (7, 7, 8))
    for x, y in zip(a, b):
        assert torch.equal(x.values if isinstance(x, F.ScalarField) else x.data,
                           y.values if isinstance(y, F.ScalarField) else y.data)
    assert not torch.equal(a[0].values, c[0].values)


def test_translation_pair_is_a_spectral_shift():
    m0, m1, v = F.synth_case("translation", 128, seed=0)
    c = [float(v.data[i].flatten()[0]) for i in range(2)]
    fq = [np.fft.fftfreq(n, d=1.0 / n) for n in m0.grid.n]
    phase = np.exp(1j * (fq[0][:, None] * c[0] + fq[1][None, :] * c[1]))
    shifted = np.fft.ifftn(np.fft.fftn(_vals(m0)) * phase).real
    assert np.max(np.abs(_vals(m1) - shifted)) <= 1e-4


def test_synthetic_velocities_respect_or_violate_det_bounds_by_design():
    for name in ("rotation", "swirl"):
        assert F.det_bounds_ok(F.synth_case(name, 64, seed=0)[2], 0.1)[0], name
    ok, dmin, _, _ = F.det_bounds_ok(F.synth_case("compress", 64, seed=0)[2], 0.1)
    assert not ok and dmin < 0.1


def test_synthetic_3d_case_and_size_validation():
    m0, m1, _ = F.synth_case("rotation", 32, seed=1, d=3)
    assert m0.grid.d == 3 and dist_value(m0, m1, "ssd") > 0.0
    for args in (("swirl", 48), ("swirl", 16), ("vortexsheet", 32)):
        with pytest.raises(ValueError):
            F.synth_case(*args)


# ---------------------------------------------------------------------------
# CLF1 container (reference volio.py:59-131)
# ---------------------------------------------------------------------------


def test_clf1_round_trips_bit_for_bit(rng, tmp_path):
    g = F.Grid((16, 24))
    u = F.ScalarField(g, rng.standard_normal(g.n))
    F.write_volume(u, tmp_path / "u.clf")
    back = F.read_volume(tmp_path / "u.clf", n_t=g.n_t)
    assert isinstance(back, F.ScalarField) and back.grid.n == g.n and np.array_equal(_vals(back), _vals(u))
    g3 = F.Grid((8, 8, 8))
    v = F.VectorField(g3, rng.standard_normal((3, *g3.n)))
    F.write_volume(v, tmp_path / "v.clf")
    back = F.read_volume(tmp_path / "v.clf")
    assert isinstance(back, F.VectorField) and np.array_equal(_vals(back), _vals(v))
    g32 = F.Grid((8, 8), dtype=np.float32)
    u32 = F.ScalarField(g32, rng.standard_normal(g32.n).astype(np.float32))
    F.write_volume(u32, tmp_path / "u32.clf")
    back = F.read_volume(tmp_path / "u32.clf")
    assert back.grid.dtype == np.dtype(np.float32) and np.array_equal(_vals(back), _vals(u32))
    lab = random_labels(F.Grid((16, 16)), rng, 9)
    F.write_volume(lab, tmp_path / "lab.clf")
    back = F.read_volume(tmp_path / "lab.clf")
    assert isinstance(back, F.LabelVolume) and np.array_equal(_lab(back), _lab(lab))


def _valid_bytes(rng):
    header = b"CLF1" + struct.pack("<BBBB", 1, 2, 2, 1) + struct.pack("<2I", 8, 8)
    return header + rng.standard_normal((8, 8)).astype("<f8").tobytes()


def test_clf1_header_errors(rng, tmp_path):
    data = _valid_bytes(rng)
    p = tmp_path / "x.clf"
    p.write_bytes(b"XXXX" + data[4:])
    with pytest.raises(volio.BadMagicError):
        F.read_volume(p)
    p.write_bytes(data[:-17])
    with pytest.raises(volio.TruncatedPayloadError):
        F.read_volume(p)
    bad = bytearray(data)
    bad[5] = 9
    p.write_bytes(bytes(bad))
    with pytest.raises(volio.DtypeMismatchError):
        F.read_volume(p)
    bad = bytearray(data)
    bad[4] = 2
    p.write_bytes(bytes(bad))
    with pytest.raises(volio.VolumeFormatError):
        F.read_volume(p)
    # dims written big-endian: the reserved most-significant byte is nonzero
    header = b"CLF1" + struct.pack("<BBBB", 1, 2, 2, 1) + struct.pack(">2I", 128, 128)
    p.write_bytes(header + rng.standard_normal((128, 128)).astype(">f8").tobytes())
    with pytest.raises(volio.VolumeFormatError, match="reserved"):
        F.read_volume(p)
