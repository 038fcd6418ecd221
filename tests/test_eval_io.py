"""Evaluation / I/O layer against fixtures written
by the reference itself (tests/golden/make_eval_golden.py): CLF1 bytes,
Dice, dice.csv, error classes, CLI usage exit code; GPU: float volume round
trips, label transport and relative mismatch vs the reference's own outputs,
CLI end to end."""
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

from paper_2401_17493_b200 import cli, metrics, volio  # noqa: E402

EV = os.path.join(GOLDEN, "eval")


def _labels(name):
    return volio.read_volume(os.path.join(EV, name))


def test_clf1_labels_round_trip_bytes(tmp_path):
    for name in ("labels_a.clf", "labels_b.clf"):
        lv = _labels(name)
        assert isinstance(lv, metrics.LabelVolume) and tuple(lv.labels.shape) == (10, 12, 16)
        out = tmp_path / name
        volio.write_volume(lv, out)
        assert out.read_bytes() == open(os.path.join(EV, name), "rb").read()


def test_dice_matches_reference():
    ref = json.load(open(os.path.join(EV, "dice.json")))
    res = metrics.dice(_labels("labels_a.clf"), _labels("labels_b.clf"), ids=[1, 2, 3, 4, 5, 7])
    assert {str(k): v for k, v in res.per_id.items()} == ref["per_id"]
    assert res.union == ref["union"] and list(res.empty_ids) == ref["empty_ids"]


def test_dice_csv_bytes(tmp_path):
    metrics.write_dice_csv(tmp_path / "d.csv", {1: [0.5, 0.75, 0.9], 3: [0.25], 2: []})
    assert (tmp_path / "d.csv").read_bytes() == open(os.path.join(EV, "dice.csv"), "rb").read()


def test_clf1_errors(tmp_path):
    raw = open(os.path.join(EV, "labels_a.clf"), "rb").read()
    cases = {"magic": (b"XLF1" + raw[4:], volio.BadMagicError),
             "trunc": (raw[:-3], volio.TruncatedPayloadError),
             "dtype": (raw[:5] + bytes([9]) + raw[6:], volio.DtypeMismatchError),
             "endian": (raw[:8] + raw[8:12][::-1] + raw[12:], volio.VolumeFormatError)}
    for name, (blob, exc) in cases.items():
        p = tmp_path / f"{name}.clf"
        p.write_bytes(blob)
        with pytest.raises(exc):
            volio.read_volume(p)


def test_cli_usage_exit_code():
    assert cli.main(["register"]) == cli.EXIT_USAGE
    assert cli.main(["frobnicate"]) == cli.EXIT_USAGE


def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.gpu
def test_clf1_float_round_trip_bytes(tmp_path):
    _gpu()
    for name in ("scalar_f32.clf", "vector2d_f64.clf"):
        f = volio.read_volume(os.path.join(EV, name))
        volio.write_volume(f, tmp_path / name)
        assert (tmp_path / name).read_bytes() == open(os.path.join(EV, name), "rb").read()


@pytest.mark.gpu
def test_transport_labels_matches_reference():
    """metrics.py:90-104: the reference's own moved labels (golden). Labels are
    index work, so the bar is bit-exact; the only admissible differences are
    voxels whose composed departure coordinate sits on a nearest-rounding tie
    (within 1e-9 of k + 1/2, where the last f64 bit of the composed map — FMA
    contraction vs numba — decides the label). Their count is reported."""
    _gpu()
    import paper_2401_17493_b200 as F
    from oracle import flowreg_oracle as O

    n = 32
    _, _, vtrue = F.synth_case("rotation", n, seed=1, d=3)
    lab = np.random.default_rng(3).integers(0, 4, size=(n, n, n)).astype(np.int32)
    moved = metrics.transport_labels(metrics.LabelVolume(vtrue.grid, lab), vtrue).labels.cpu().numpy()
    ref = np.load(os.path.join(EV, "labels_moved.npz"))["moved"].astype(np.int32)
    diff = moved != ref
    q = np.stack(O.frac_index((n, n, n), O.compose_map(vtrue.data.cpu().numpy(), vtrue.grid.n_t)))
    tie = np.any(np.abs(q - np.floor(q) - 0.5) < 1e-9, axis=0).reshape(n, n, n)
    print(f"label transport: {int(diff.sum())} of {diff.size} voxels differ from the reference, "
          f"{int(tie.sum())} voxels on rounding ties")
    assert not np.any(diff & ~tie)


@pytest.mark.gpu
def test_relative_mismatch_matches_reference():
    """metrics.py:111-129 (ssd, ncc, and the degenerate m0 == m1 flag)."""
    _gpu()
    import paper_2401_17493_b200 as F

    ref = json.load(open(os.path.join(EV, "mismatch.json")))
    m0, m1, vtrue = F.synth_case("rotation", 32, seed=1, d=3)
    half = F.VectorField._wrap(vtrue.grid, 0.5 * vtrue.data)
    for dist in ("ssd", "ncc"):
        val, degen = metrics.relative_mismatch(m0, m1, half, distance=dist)
        assert val == pytest.approx(ref[dist][0], rel=1e-10) and degen == ref[dist][1], dist
    assert tuple(metrics.relative_mismatch(m0, m0, half)) == tuple(ref["zero"])


@pytest.mark.gpu
def test_cli_synth_register_transport_dice(tmp_path):
    _gpu()
    d = str(tmp_path)
    assert cli.main(["synth", "rotation", "32", "3", "--out-dir", d]) == cli.EXIT_OK
    rc = cli.main(["register", "--template", f"{d}/m0.clf", "--reference", f"{d}/m1.clf", "--precond", "reg",
                   "--out-dir", d])
    assert rc == cli.EXIT_OK
    rep = json.load(open(f"{d}/report.json"))
    assert rep["status"] == "converged" and {"config", "intensity", "iterations", "matvecs"} <= set(rep)
    for f in ("velocity.clf", "deformed.clf", "residual-before.clf", "residual-after.clf"):
        assert os.path.getsize(f"{d}/{f}") > 0
    assert cli.main(["detgrad", f"{d}/velocity.clf", "--out-dir", d]) == cli.EXIT_OK
    assert cli.main(["transport", f"{d}/m0.clf", f"{d}/velocity.clf", "--out-dir", d]) == cli.EXIT_OK
    assert cli.main(["register", "--template", f"{d}/missing.clf", "--reference", f"{d}/m1.clf",
                     "--out-dir", d]) == cli.EXIT_DATA
