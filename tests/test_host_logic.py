"""Host-side control logic that runs without a GPU (CPU suite): the pieces
of the reference's optimizer / continuation / fields / diffops / metrics
tests that are pure host arithmetic or validation (reference
optimizer.py:81-89, continuation.py:35-47,225-236, fields.py:54-133,
diffops.py:150-242, metrics.py:132-155, cli.py:40-57)."""
import csv

import numpy as np
import pytest

import paper_2401_17493_b200 as F
from paper_2401_17493_b200.cli import JobConfig
from paper_2401_17493_b200.continuation import cascade_alphas
from paper_2401_17493_b200.diffops import incompressibility_multiplier, reg_symbol
from paper_2401_17493_b200.metrics import write_dice_csv
from paper_2401_17493_b200.optimizer import forcing_tolerance


def test_forcing_tolerance():
    assert forcing_tolerance(0.04, "superlinear") == pytest.approx(0.2, rel=1e-15)
    assert forcing_tolerance(1.0, "superlinear") == 0.5
    assert forcing_tolerance(9.0, "quadratic") == 0.5
    assert forcing_tolerance(1e-6, "quadratic") == pytest.approx(1e-6, rel=1e-15)
    for bad in ((-1.0, "superlinear"), (0.1, "cubic")):
        with pytest.raises(ValueError):
            forcing_tolerance(*bad)


def test_cascade_schedule():
    got = cascade_alphas(1.773437e-3)
    assert got[:4] == [1.0, 0.1, 0.01, 0.001] and got[4] == pytest.approx(1.773437e-3, rel=1e-12)
    assert cascade_alphas(1.0) == [1.0] and cascade_alphas(1e-2) == [1.0, 0.1, 0.01]
    for bad in (0.0, -1.0, 1.5):
        with pytest.raises(ValueError):
            cascade_alphas(bad)


def test_configuration_validation():
    with pytest.raises(ValueError):
        F.SearchConfig(eps_det=1.0)
    with pytest.raises(ValueError):
        F.SearchConfig(decade_factor=1.0)
    with pytest.raises(ValueError):
        F.RegConfig(alpha=0.0)
    with pytest.raises(ValueError):
        F.PrecondKind("ilu")
    assert F.PrecondKind("h0-two-level").kind == "2level" and F.PrecondKind("regularization").kind == "reg"
    with pytest.raises(ValueError):
        F.IncompressibilityMode("divergence-free")
    with pytest.raises(ValueError):
        F.IncompressibilityMode("near-incompressible", 0.0)
    with pytest.raises(ValueError):
        F.RegOperatorSpec(4)
    cfg = JobConfig()
    assert (cfg.n_t, cfg.tol, cfg.beta, cfg.eps_det, cfg.interp, cfg.forcing, cfg.precision) == (
        4, 5e-2, 1e-4, 0.1, "cubic", "superlinear", "f64")


def test_grid_and_mesh_coordinates():
    g = F.Grid((16, 32, 8))
    assert all(h * n == pytest.approx(2 * np.pi, rel=1e-15) for h, n in zip(g.h, g.n))
    assert g.axis_coords(0)[0] == pytest.approx(np.pi - g.h[0], rel=1e-15)
    assert g.cell_volume == pytest.approx(np.prod(g.h), rel=1e-15) and g.num_voxels == 16 * 32 * 8
    assert F.Grid((16, 32, 16)).coarsen().n == (8, 16, 8) and g.with_time_steps(7).n_t == 7
    for bad in ((15, 16), (6, 16), (8,), (8, 8, 8, 8)):
        with pytest.raises(ValueError):
            F.Grid(bad)
    with pytest.raises(ValueError):
        F.Grid((8, 8), n_t=0)
    with pytest.raises(ValueError):
        F.Grid((8, 8), dtype=np.int32)
    with pytest.raises(ValueError):
        F.Grid((8, 12)).coarsen()
    assert np.allclose(F.mesh_coordinates(F.Grid((8, 8, 8)), (3, 4, 5)), (np.pi / 4, 0.0, -np.pi / 4))
    for bad in ((0, 3), (3, 9)):
        with pytest.raises(IndexError):
            F.mesh_coordinates(F.Grid((8, 8)), bad)


def test_regularisation_symbols_and_multiplier():
    g = F.Grid((8, 8))
    h1 = reg_symbol(g, F.RegOperatorSpec(1))
    assert h1[0, 0] == 0.0 and h1[1, 2] == 5.0 and h1[-1, -2] == 5.0
    assert reg_symbol(g, F.RegOperatorSpec(2))[1, 2] == 25.0
    assert reg_symbol(g, F.RegOperatorSpec(1, seminorm=False))[0, 0] == 1.0
    m = incompressibility_multiplier(1.0, F.IncompressibilityMode("near-incompressible", 1e-4), 1e-2)
    assert 0.0 < m < 1.0
    heavy = F.IncompressibilityMode("near-incompressible", 1e6)
    assert incompressibility_multiplier(4.0, heavy, 1e-2) == pytest.approx(1.0, abs=1e-6)
    assert incompressibility_multiplier(4.0, F.IncompressibilityMode("incompressible"), 1e-2) == 1.0
    with pytest.raises(ValueError):
        incompressibility_multiplier(4.0, F.IncompressibilityMode("none"), 1e-2)


def test_dice_csv_statistics(tmp_path):
    path = tmp_path / "dice.csv"
    write_dice_csv(path, {1: [0.5, 0.7], 2: [1.0]})
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["label_id", "mean", "stdev", "min", "max", "median", "q25", "q75"]
    assert len(rows) == 3 and float(rows[1][1]) == pytest.approx(0.6) and float(rows[2][2]) == 0.0
