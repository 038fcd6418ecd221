"""Golden fixtures for the evaluation / I/O layer,
produced by the REFERENCE package itself (run in the build container):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_eval_golden.py

Writes tests/golden/eval/: CLF1 files of a label volume, an f32 scalar and an
f64 vector field (the reference's writer), the reference's Dice result of two
label volumes and its dice.csv bytes.
"""
import json
import os

import numpy as np
from flowreg.fields import Grid, ScalarField, VectorField
from flowreg.metrics import LabelVolume, dice, write_dice_csv
from flowreg.volio import write_volume

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "eval")
os.makedirs(OUT, exist_ok=True)
rng = np.random.default_rng(7)
n = (10, 12, 16)
la = rng.integers(0, 5, size=n).astype(np.int32)
lb = np.where(rng.random(n) < 0.8, la, rng.integers(0, 6, size=n)).astype(np.int32)
lb[lb == 4] = 0  # id 4 only in a; id 5 only in b
write_volume(LabelVolume(Grid(n), la), os.path.join(OUT, "labels_a.clf"))
write_volume(LabelVolume(Grid(n), lb), os.path.join(OUT, "labels_b.clf"))
g32 = Grid(n, dtype=np.float32)
write_volume(ScalarField(g32, rng.standard_normal(n).astype(np.float32)), os.path.join(OUT, "scalar_f32.clf"))
g64 = Grid((12, 16), dtype=np.float64)
write_volume(VectorField(g64, rng.standard_normal((2, 12, 16))), os.path.join(OUT, "vector2d_f64.clf"))
res = dice(LabelVolume(Grid(n), la), LabelVolume(Grid(n), lb), ids=[1, 2, 3, 4, 5, 7])
with open(os.path.join(OUT, "dice.json"), "w") as fh:
    json.dump({"per_id": {str(k): v for k, v in res.per_id.items()}, "union": res.union,
               "empty_ids": list(res.empty_ids)}, fh, indent=1)
write_dice_csv(os.path.join(OUT, "dice.csv"), {1: [0.5, 0.75, 0.9], 3: [0.25], 2: []})
print("wrote", sorted(os.listdir(OUT)))

# label transport + relative mismatch (metrics.py:90-129) on the 3D rotation
# case: the reference's moved labels and its mismatch values
from flowreg.metrics import relative_mismatch, transport_labels  # noqa: E402
from flowreg.synth import synth_case  # noqa: E402

m0, m1, vtrue = synth_case("rotation", 32, seed=1, d=3)
lab = np.random.default_rng(3).integers(0, 4, size=(32, 32, 32)).astype(np.int32)
moved = transport_labels(LabelVolume(vtrue.grid, lab), vtrue).labels
np.savez_compressed(os.path.join(OUT, "labels_moved.npz"), moved=moved.astype(np.int8))
half = VectorField(vtrue.grid, 0.5 * vtrue.data)
mm = {d: list(relative_mismatch(m0, m1, half, distance=d)) for d in ("ssd", "ncc")}
mm["zero"] = list(relative_mismatch(m0, m0, half))
with open(os.path.join(OUT, "mismatch.json"), "w") as fh:
    json.dump(mm, fh, indent=1)
print("wrote labels_moved.npz / mismatch.json", mm)
