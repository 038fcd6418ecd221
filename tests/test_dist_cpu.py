"""Host logic of the slab decomposition (dist.py) on CPU: plane ownership,
halo widths, and the ring / all-to-all / all-reduce exchanges of SlabComm
with the gloo backend at world sizes 2 and 3 (no GPU needed)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2401_17493_b200.dist import SlabComm, halo_width, slab_bounds  # noqa: E402


def test_slab_bounds_and_halo_width():
    assert [slab_bounds(64, 4, r) for r in range(4)] == [(0, 16), (16, 32), (32, 48), (48, 64)]
    with pytest.raises(ValueError):
        slab_bounds(64, 3, 0)
    # cubic stencil planes floor(d) - 1 .. floor(d) + 2
    assert halo_width(0.0) == 2 and halo_width(0.5) == 3 and halo_width(3.0) == 5
    assert halo_width(0.5, "linear") == 2
    assert halo_width(0.5, "bspline") == halo_width(0.5, "cubic")  # same 4-point support


def test_run_search_control_flow():
    """continuation.run_search — the sweep / bisection of continuation.py:144-207
    shared by search_alpha and dist_search_alpha — on a mock trial that passes
    iff alpha >= 3e-3: decades 1, 0.1, 0.01 pass, 1e-3 fails, then bisection
    between 1e-3 and 1e-2 with warm starts from the previous trial."""
    from paper_2401_17493_b200.continuation import SearchConfig, TrialRecord, run_search

    seen = []

    def trial(alpha, v_warm, phase):
        seen.append((alpha, v_warm, phase))
        ok = alpha >= 3e-3
        return f"v{len(seen)}", TrialRecord(alpha, ok, 0.5, 1.5, 1.0, 0.1, 3, v_warm is not None, False, phase)

    res = run_search(SearchConfig(bisection_depth=3), trial, lambda v: False)
    alphas = [a for a, _, _ in seen]
    assert np.allclose(alphas, [1.0, 0.1, 0.01, 0.001, 0.0055, 0.00325, 0.002125])
    assert [ph for _, _, ph in seen] == ["sweep"] * 4 + ["bisection"] * 3
    assert [w for _, w, _ in seen] == [None, "v1", "v2", "v3", "v4", "v5", "v6"]
    assert res.status == "ok" and np.isclose(res.alpha, 0.00325) and res.velocity == "v6"
    assert res.anomalies == []
    # failing at the first alpha, and running into the floor
    r0 = run_search(SearchConfig(), lambda a, w, ph: (None, TrialRecord(a, False, 0, 0, 0, 0, 1, False, False, ph)),
                    lambda v: False)
    assert r0.status == "violated_at_start" and r0.alpha is None and len(r0.trials) == 1
    r1 = run_search(SearchConfig(alpha_floor=1e-3),
                    lambda a, w, ph: ("v", TrialRecord(a, True, 1, 1, 1, 0, 1, False, False, ph)), lambda v: False)
    assert r1.status == "floor_reached" and np.isclose(r1.alpha, 1e-3) and len(r1.trials) == 4


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as tdist

    tdist.init_process_group("gloo", rank=rank, world_size=size)
    comm = SlabComm()
    n0, n1, n2, W = 6 * size, 3, 4, 2
    glob = torch.arange(2 * n0 * n1 * n2, dtype=torch.float64).reshape(2, n0, n1, n2)
    lo, hi = slab_bounds(n0, size, rank)
    ext = torch.zeros((2, hi - lo + 2 * W, n1, n2), dtype=torch.float64)
    ext[:, W:W + hi - lo] = glob[:, lo:hi]
    comm.halo(ext, W)
    idx = [(p % n0) for p in range(lo - W, hi + W)]
    ok_halo = bool(torch.equal(ext, glob[:, idx]))
    # all-to-all: chunk q of rank r -> chunk r of rank q
    inp = torch.stack([torch.full((3,), 100.0 * rank + q) for q in range(size)])
    out = torch.empty_like(inp)
    comm.all_to_all(out, inp)
    ok_a2a = bool(torch.equal(out[:, 0], torch.tensor([100.0 * q + rank for q in range(size)])))
    ok_red = comm.all_reduce(rank + 1.0) == size * (size + 1) / 2 and comm.all_reduce(float(rank), "max") == size - 1
    np.save(os.path.join(outdir, f"r{rank}.npy"), np.array([ok_halo, ok_a2a, ok_red]))
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("size", [2, 3])
def test_slab_comm_exchanges_gloo(size, tmp_path):
    import torch.multiprocessing as mp

    mp.start_processes(_worker, args=(size, _port(), str(tmp_path)), nprocs=size, start_method="spawn", join=True)
    for r in range(size):
        assert np.load(os.path.join(tmp_path, f"r{r}.npy")).all(), r
