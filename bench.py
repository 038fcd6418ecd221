#!/usr/bin/env python3
"""Benchmark: Gauss-Newton Hessian matvecs/s at 256^3 (+ time-to-solution and
interpolation GB/s vs the HBM roofline) — BASELINE.json metric, config C3.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A "step" is one ``KktState.hessian_matvec`` (kkt.py:237-260) at 256^3, d = 3,
n_t = 4, cubic Lagrange SL, FD8, H1 seminorm, near-incompressible beta=1e-4,
alpha = 1e-2, SSD, state fixed at v = v_true / 2 of synth_case("rotation",
256, seed=1); v~ = 0.1 N(0, 1) (seed 0).  Transport in fp32, velocity-space
vectors in fp64 (SURVEY.md §7 hard part 1).  Synthetic data generated on the
device.  Every matvec touches several GB, far above the 126 MB L2, so no L2
flush is needed between steps.

Multi-GPU (torchrun, one rank per GPU): the headline is ONE slab-decomposed
problem (dist.py) — config C4, 512^3 at N = 2 / 4, config C5's 1024^3 at
N = 8 (``--slab-n`` overrides) — generated slab by slab on the ranks
(dist.slab_synth), GN Hessian matvecs/s of that problem (strong scaling,
NCCL all-to-all FFT transposes + ghost-plane exchanges), its time to
solution (SPMD dist_register) and its e2e rate with host buffers.  A slab
failure exits non-zero.  ``--slab`` runs the same path at N = 1 (P = 1).
The barrier + max-over-ranks timing uses NCCL.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port, oracle/flowreg_oracle.py: C/OpenMP gathers + pocketfft) on the
host cores for the same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Hessian matvecs/s and time-to-solution at 256^3; interp GB/s vs HBM peak"
UNIT = "matvec/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--precision", default="mixed", choices=["mixed", "f64", "f32"])
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-solution run")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--slab", action="store_true", help="slab-decomposed headline at N = 1 too (P = 1)")
    ap.add_argument("--slab-n", type=int, default=0,
                    help="grid of the slab-decomposed headline (default 512, 1024 at N = 8)")
    return ap.parse_args()


def config(n, precision):
    return {"workload": f"C3: GN Hessian matvec, synth rotation {n}^3, nt=4, cubic-Lagrange SL, FD8, "
                        "H1 alpha=1e-2, near-incompressible beta=1e-4, SSD",
            "grid": [n, n, n], "n_t": 4, "interp": "cubic", "precision": precision,
            "l2": "inputs > L2 (working set several GB per matvec, no flush needed)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a few hundred ms to start sampling: wait for its
            # first row so that the samples kept (from here on) cover the timed region
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        self.start = len(self.rows)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = self.rows[self.start:] or self.rows[-1:]  # samples taken during the timed region
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.rows = rows
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, val in zip(names, r[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def profile_traffic():
    """dram bytes per launch of the gather kernel from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(a):
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one rank per GPU over NCCL; FRG_DIST_BACKEND=gloo lets several ranks share
    # one GPU to exercise the multi-rank path (exchanges staged through host)
    backend = os.environ.get("FRG_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2401_17493_b200 as F
    from paper_2401_17493_b200 import _lib as L

    if world > 1 or a.slab:
        return run_slab(a, F, L, world, rank, local, backend)

    n = a.n
    dtype = np.float32 if a.precision == "f32" else np.float64
    tdt = np.float32 if a.precision in ("mixed", "f32") else None
    m0, m1, vtrue = F.synth_case("rotation", n, seed=1, d=3, dtype=dtype)
    grid = m0.grid
    reg = F.RegConfig(alpha=1e-2, operator=F.RegOperatorSpec(1, True),
                      incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
    v = F.VectorField._wrap(grid, 0.5 * vtrue.data)
    st = F.KktState(m0, m1, reg, distance="ssd", method="cubic", scheme="fd8", v_init=v, transport_dtype=tdt)
    gen = torch.Generator(device="cuda").manual_seed(0)
    vt = F.VectorField._wrap(grid, 0.1 * torch.randn((3, n, n, n), generator=gen, dtype=grid.torch_dtype,
                                                     device="cuda"))
    out = torch.empty_like(vt.data)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.current_stream()
    for _ in range(a.warmup):
        st.hessian_matvec(vt, out=out)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0 = st.matvecs
    # the dominant kernel (IncFirstOp: 3-field gather of v~ at the feet + all
    # Heun sources, 22% of the step) timed live: CUDA events on its own stream
    # bracket each of its launches inside the timed matvecs (frg_probe_*)
    L.check(L.lib().frg_probe_arm(1), "probe_arm")
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(a.steps):
            st.hessian_matvec(vt, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
    L.check(L.lib().frg_probe_arm(0), "probe_arm")
    probe_ms, probe_n = ctypes.c_double(), ctypes.c_int64()
    L.check(L.lib().frg_probe_read(ctypes.byref(probe_ms), ctypes.byref(probe_n)), "probe_read")
    barrier()
    torch.cuda.synchronize()
    assert st.matvecs - c0 == a.steps
    t_ms = max_over_ranks(e0.elapsed_time(e1))
    ms_per_step = t_ms / a.steps
    value = world * a.steps / (t_ms / 1e3)

    # launches of OUR kernels per matvec (host call sequence of kkt_hessian_matvec,
    # profiles/r01_launches_matvec_final_summary.txt): v~ f64->f32 convert 1,
    # inc-state 4 (IncFirst + 3 IncStep), adjoint 4, body force 1, spectral
    # combine 1, f32->f64 output convert 1 (+ 9 cuFFT transforms, not counted)
    launches_per_matvec = 1 + 4 + 4 + 1 + 1 + 1
    gpu_launches = launches_per_matvec * a.steps

    # --- dominant kernel roofline: one cubic SL gather step (k_gather) -------
    N = n ** 3
    disp = st.trajectory.disp.to(torch.float32) if tdt is not None or dtype == np.float32 else st.trajectory.disp
    fdt = disp.dtype
    f = torch.randn((n, n, n), generator=gen, dtype=fdt, device="cuda")
    g_out = torch.empty_like(f)
    ins = (ctypes.c_void_p * 1)(f.data_ptr())
    outs = (ctypes.c_void_p * 1)(g_out.data_ptr())
    nn = L.n3((n, n, n))
    fcode = L.dtype_code(fdt)
    sp = ctypes.c_void_p(stream.cuda_stream)
    # the gather as the matvec runs it: fp32 with the map's tile plan
    planned = fdt == torch.float32
    if planned:
        plan = torch.empty((L.lib().frg_tile_plan_count(nn), 4), dtype=torch.int32, device="cuda")
        L.check(L.lib().frg_tile_plan(nn, 3, 2, ctypes.c_void_p(disp.data_ptr()), L.ptr(plan), sp), "tile_plan")

    def gather_once():
        if planned:
            L.check(L.lib().frg_gather_planned(nn, 3, 2, ctypes.c_void_p(disp.data_ptr()), L.ptr(plan), 1, ins, outs,
                                               sp), "gather")
        else:
            L.check(L.lib().frg_gather(nn, 3, fcode, 2, ctypes.c_void_p(disp.data_ptr()), 1, ins, outs, sp),
                    "gather")

    for _ in range(3):
        gather_once()
    reps = 50
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(reps):
        gather_once()
    g1.record(stream)
    torch.cuda.synchronize()
    t_gather = g0.elapsed_time(g1) / reps / 1e3
    es = 4 if fdt == torch.float32 else 8
    alg_bytes = N * (3 * es + es + es)  # coordinates + field (once) + output
    peak, peak_src = peaks()
    achieved = alg_bytes / t_gather / 1e9
    traffic = profile_traffic().get("k_gather_cubic_f32_bytes_per_launch")
    # IncFirstOp algorithmic bytes per voxel (fp32, d = 3): disp 12 + v~ 12 (gather
    # source and the x-side Heun term read the same array: counted once) +
    # grad m_j(y) n_t*12 + grad m_{j+1}(x) n_t*12, writes m~_1 4 + S_1..S_{n_t-1} 4 (n_t - 1)
    nt_ = 4
    inc_bytes = N * (12 + 12 + 12 * nt_ + 12 * nt_ + 4 + 4 * (nt_ - 1))
    t_inc = probe_ms.value / 1e3 / max(probe_n.value, 1)

    # whole-matvec roofline with the canonical field-pass count (174 F)
    canon = 174 * 4 * N
    matvec_roofline = {"canonical_bytes": canon, "achieved_gbs": canon / (ms_per_step / 1e3) / 1e9,
                       "peak_gbs": peak, "frac": canon / (ms_per_step / 1e3) / 1e9 / peak,
                       "note": "SURVEY.md §8d canonical 174 fp32 field passes per matvec"}

    # --- e2e through the public API with host buffers -----------------------
    e2e_steps = max(10, min(a.steps, 30))  # steady state: pipeline fill / drain is ~2 steps of copies
    host_in = torch.empty_like(vt.data, device="cpu").pin_memory()
    host_in.copy_(vt.data)
    host_out = torch.empty_like(host_in).pin_memory()
    dev_in = torch.empty_like(vt.data)
    for _ in range(max(a.warmup, 3)):  # the host path's first call allocates its device slots and copy streams
        st.hessian_matvec(host_in, out=host_out)
    st.wait_host_io()
    torch.cuda.synchronize()
    barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record(stream)
    for _ in range(e2e_steps):
        # public API with host buffers: H2D of v~, the matvec, D2H of the result
        # every step (pipelined across steps by KktState's copy streams)
        st.hessian_matvec(host_in, out=host_out)
    st.wait_host_io()
    x1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_e2e = max_over_ranks(x0.elapsed_time(x1)) / 1e3
    # the same call with no overlap between calls (one PCG iteration's view:
    # H2D, matvec, D2H, then the host has the result before the next call)
    lat_steps = 5
    z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    z0.record(stream)
    for _ in range(lat_steps):
        st.hessian_matvec(host_in, out=host_out)
        st.wait_host_io()
        torch.cuda.synchronize()  # the host holds this call's result before issuing the next
    z1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_lat = max_over_ranks(z0.elapsed_time(z1)) / 1e3 / lat_steps
    # the host link's own ceiling for this step: H2D of v~ and D2H of a result
    # at once on two copy streams, no compute
    s_h, s_d = torch.cuda.Stream(), torch.cuda.Stream()
    y0, y1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    y0.record(stream)
    s_h.wait_stream(stream)
    s_d.wait_stream(stream)
    for _ in range(3):
        with torch.cuda.stream(s_h):
            dev_in.copy_(host_in, non_blocking=True)
        with torch.cuda.stream(s_d):
            host_out.copy_(out, non_blocking=True)
    stream.wait_stream(s_h)
    stream.wait_stream(s_d)
    y1.record(stream)
    torch.cuda.synchronize()
    t_link = y0.elapsed_time(y1) / 3e3
    e2e = {"value": world * e2e_steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": host_in.numel() * host_in.element_size(),
           "d2h_bytes_per_step": host_out.numel() * host_out.element_size(),
           "steps": e2e_steps,
           "link_ceiling": {"value": world / t_link, "unit": UNIT,
                            "gbs_per_direction": host_in.numel() * host_in.element_size() / t_link / 1e9,
                            "note": "concurrent pinned H2D + D2H of one step's buffers, no compute"},
           "path": "pinned host v~ -> KktState.hessian_matvec(host tensor) (H2D, C-ABI frg_kkt_hessian_matvec, D2H; "
                   "copies of neighbouring steps overlap the device work on dedicated copy streams) -> pinned host",
           "latency": {"value": world / t_lat, "unit": UNIT, "ms_per_call": 1e3 * t_lat, "steps": lat_steps,
                       "note": "each call's H2D, matvec and D2H complete before the next call (no overlap "
                               "between calls): the per-iteration view of a host-side PCG"}}

    # --- time to solution (C3: register at 256^3, reg preconditioner) --------
    tts = None
    if not a.no_tts:
        del st
        torch.cuda.synchronize()
        barrier()
        # one untimed solve creates the cuFFT plans (process-wide cache), then four timed
        # solves (best of: the host-side loop syncs on every reduction, so it is noisy)
        walls = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            vsol, rep = F.register(m0, m1, reg=reg, precond=F.PrecondKind("reg"), method="cubic", scheme="fd8",
                                   transport_dtype=tdt)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        wall = max_over_ranks(min(walls[1:]))
        tts = {"seconds": wall, "first_call_seconds": walls[0], "iterations": rep.iterations,
               "matvecs": rep.matvecs, "pde_solves": rep.pde_solves, "status": rep.status, "mismatch": rep.mismatch,
               "gradient": rep.gradient, "precond": "reg", "detgrad_min": rep.detgrad_min,
               "includes": "KktState creation, all refresh/gradient/PCG/Armijo work and det(F) stats; "
                           "excludes synthetic-data generation"}

    # --- the other single-GPU configs of BASELINE.json (parity-test cases;
    # reported for completeness, not the headline) -------------------------
    other = None
    if world == 1 and n == 256 and not a.no_tts:
        other = []
        for tag, nn_, order, meth in (("C1", 64, 1, "cubic"), ("C2", 128, 2, "linear"), ("C3-bspline", 256, 1,
                                                                                          "bspline")):
            mm0, mm1, vv = F.synth_case("rotation", nn_, seed=1, d=3)
            rg = F.RegConfig(alpha=1e-2, operator=F.RegOperatorSpec(order, True),
                             incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
            s2 = F.KktState(mm0, mm1, rg, method=meth, v_init=F.VectorField._wrap(mm0.grid, 0.5 * vv.data),
                            transport_dtype=np.float32)
            vt2 = F.VectorField._wrap(mm0.grid, 0.1 * torch.randn((3, nn_, nn_, nn_), generator=gen,
                                                                  dtype=torch.float64, device="cuda"))
            o2 = torch.empty_like(vt2.data)
            for _ in range(3):
                s2.hessian_matvec(vt2, out=o2)
            torch.cuda.synchronize()
            c0_, c1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            c0_.record(stream)
            for _ in range(reps):
                s2.hessian_matvec(vt2, out=o2)
            c1_.record(stream)
            torch.cuda.synchronize()
            mv_s = reps / (c0_.elapsed_time(c1_) / 1e3)
            canon = 174 * 4 * nn_ ** 3  # SURVEY §8d canonical fp32 field passes per matvec
            rec = {"config": tag, "grid": [nn_] * 3, "reg": f"H{order} seminorm", "interp": meth,
                   "precision": "mixed (fp32 transport, fp64 control)", "matvec_per_s": mv_s,
                   "matvec_roofline": {"canonical_bytes": canon, "achieved_gbs": canon * mv_s / 1e9,
                                       "frac": canon * mv_s / 1e9 / peak}}
            del s2
            if tag == "C3-bspline":
                # BASELINE.json C3 as written: B-spline interpolation + spectral (reg) preconditioner
                walls = []
                for _ in range(2):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    _, rp = F.register(mm0, mm1, reg=reg, precond=F.PrecondKind("reg"), method="bspline",
                                       scheme="fd8", transport_dtype=tdt)
                    torch.cuda.synchronize()
                    walls.append(time.perf_counter() - t0)
                rec["time_to_solution"] = {"seconds": walls[-1], "first_call_seconds": walls[0],
                                           "iterations": rp.iterations, "matvecs": rp.matvecs,
                                           "pde_solves": rp.pde_solves, "status": rp.status,
                                           "mismatch": rp.mismatch, "precond": "reg",
                                           "reg": "H1 alpha=1e-2, near-incompressible beta=1e-4 (as the headline)"}
            other.append(rec)

    if world > 1:
        dist.barrier()
    result = None
    if rank == 0:
        cpu = None if (a.no_cpu or world > 1) else cpu_baseline(a, m0, m1, vtrue, vt)
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 transport / f64 control" if a.precision == "mixed" else a.precision,
            "data": "synthetic (synth_case rotation, generated on device)",
            "config": dict(config(n, a.precision), parallelism="single GPU"),
            "e2e": e2e, "gpu_launches": gpu_launches,
            "roofline": {"bound": "hbm", "achieved": inc_bytes / t_inc / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": inc_bytes / t_inc / 1e9 / peak,
                         "traffic": profile_traffic().get("k_incfirst_bytes_per_launch"),
                         "kernel": "k_slf<CUBIC,3,IncFirstOp<float,3>>: the step's dominant kernel (fused 3-field "
                                   "gather of v~ at the feet + every Heun source S_j), timed live inside the timed "
                                   "matvecs (CUDA events on its stream, frg_probe_*)",
                         "algorithmic_bytes_per_launch": inc_bytes, "bytes_per_voxel": inc_bytes // N,
                         "launch_s": t_inc, "launches_timed": probe_n.value, "peak_source": peak_src},
            "gather_roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                                "frac": achieved / peak, "traffic": traffic,
                                "kernel": "k_slf<CUBIC,1,GatherOp<float,1>> (one TMA-staged SL gather step with its "
                                          "tile plan, frg_gather_planned; the 7 single-field SL steps of the matvec "
                                          "run this engine; shared-memory bound, DESIGN.md §5)",
                                "algorithmic_bytes_per_launch": alg_bytes, "launch_s": t_gather,
                                "peak_source": peak_src},
            "matvec_roofline": matvec_roofline,
            "time_to_solution": tts,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        if other:
            result["other_configs"] = other
        print(json.dumps(result))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def run_slab(a, F, L, world, rank, local, backend):
    """C4 / C5 headline: ONE slab-decomposed registration problem over the N
    ranks (dist.py: all-to-all FFT transposes + ghost-plane exchanges)."""
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2401_17493_b200 import dist as D

    if world == 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29571")
        dist.init_process_group("gloo", rank=0, world_size=1)
    n = a.slab_n or (1024 if world >= 8 else 512)
    comm = D.SlabComm()
    staged = comm.staged

    def barrier():
        dist.barrier()

    def max_over_ranks(x):
        return comm.all_reduce(x, "max")

    m0, m1, vtrue = D.slab_synth("rotation", n, comm)
    reg = F.RegConfig(alpha=1e-2, operator=F.RegOperatorSpec(1, True),
                      incomp=F.IncompressibilityMode("near-incompressible", 1e-4))
    v = (0.5 * vtrue).contiguous()
    st = D.DistKktState(m0, m1, reg, comm, (n, n, n), v_init=v)
    gen = torch.Generator(device="cuda").manual_seed(rank)
    n0l = n // world
    vt = 0.1 * torch.randn((3, n0l, n, n), generator=gen, dtype=torch.float64, device="cuda")
    out = torch.empty_like(vt)
    stream = torch.cuda.current_stream()
    for _ in range(max(a.warmup, 3)):
        st.hessian_matvec(vt, out=out)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    b0 = comm.bytes_sent
    c0 = st.matvecs
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    L.check(L.lib().frg_probe_arm(1), "probe_arm")  # the dominant kernel (slab IncFirstOp), live
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(a.steps):
            st.hessian_matvec(vt, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
    L.check(L.lib().frg_probe_arm(0), "probe_arm")
    probe_ms, probe_n = ctypes.c_double(), ctypes.c_int64()
    L.check(L.lib().frg_probe_read(ctypes.byref(probe_ms), ctypes.byref(probe_n)), "probe_read")
    t_inc = max_over_ranks(probe_ms.value / 1e3 / max(probe_n.value, 1))
    inc_bytes = n0l * n * n * (12 + 12 + 48 + 48 + 4 + 12)  # IncFirstOp, 136 B/voxel (see run_b200)
    barrier()
    torch.cuda.synchronize()
    assert st.matvecs - c0 == a.steps
    t = max_over_ranks(e0.elapsed_time(e1)) / 1e3
    ms = 1e3 * t / a.steps
    value = a.steps / t
    sent = (comm.bytes_sent - b0) / a.steps  # payload each rank sent per matvec (halo + all-to-all chunks)
    peak, peak_src = peaks()
    canon = 174 * 4 * n ** 3 / world

    # dominant kernel: one planned single-field SL gather step on this rank's slab
    src = torch.randn((1, n0l, n, n), generator=gen, dtype=torch.float32, device="cuda")
    ext = st._src(src, st.Wf)  # ghost-extended, or (peer mode) a published peer window
    g_out = torch.empty((n0l, n, n), dtype=torch.float32, device="cuda")
    st._bind()
    for _ in range(3):
        st._gather(st.disp_f, st.Wf, [ext[0]], [g_out])
    torch.cuda.synchronize()
    reps = 20
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(reps):
        st._gather(st.disp_f, st.Wf, [ext[0]], [g_out])
    g1.record(stream)
    torch.cuda.synchronize()
    t_gather = g0.elapsed_time(g1) / reps / 1e3
    alg_bytes = n0l * n * n * 20

    # e2e: this rank's v~ slab from pinned host, the matvec, the result back, every step
    host_in = torch.empty(vt.shape, dtype=vt.dtype).pin_memory()
    host_in.copy_(vt)
    host_out = torch.empty_like(host_in).pin_memory()
    dev_in = torch.empty_like(vt)
    e2e_steps = max(3, min(a.steps, 10))
    barrier()
    torch.cuda.synchronize()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record(stream)
    for _ in range(e2e_steps):
        dev_in.copy_(host_in, non_blocking=True)
        st.hessian_matvec(dev_in, out=out)
        host_out.copy_(out, non_blocking=True)
    x1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_e2e = max_over_ranks(x0.elapsed_time(x1)) / 1e3
    # the same call with no overlap between calls (one PCG iteration's view:
    # H2D, matvec, D2H, then the host has the result before the next call)
    lat_steps = 5
    z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    z0.record(stream)
    for _ in range(lat_steps):
        dev_in.copy_(host_in, non_blocking=True)
        st.hessian_matvec(dev_in, out=out)
        host_out.copy_(out, non_blocking=True)
        torch.cuda.synchronize()  # the host holds this call's result before issuing the next
    z1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_lat = max_over_ranks(z0.elapsed_time(z1)) / 1e3 / lat_steps

    # time to solution of the same problem: SPMD dist_register (reg preconditioner)
    tts = None
    halo = [st.Wf, st.Wb]
    if not a.no_tts:
        del st
        torch.cuda.synchronize()
        barrier()
        walls = []
        for _ in range(2):  # the first solve creates the cuFFT plans
            torch.cuda.synchronize()
            barrier()
            w0 = time.perf_counter()
            _, rep = D.dist_register(m0, m1, comm, (n, n, n), reg=reg)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - w0)
        tts = {"seconds": max_over_ranks(walls[-1]), "first_call_seconds": max_over_ranks(walls[0]),
               "iterations": rep.iterations, "matvecs": rep.matvecs, "pde_solves": rep.pde_solves,
               "status": rep.status, "mismatch": rep.mismatch, "precond": "reg", "detgrad_min": rep.detgrad_min,
               "includes": "DistKktState creation, all refresh/gradient/PCG/Armijo work and det(F) stats over the "
                           "slabs; excludes synthetic-data generation"}

    # launches of our kernels per slab matvec: 3 converts, IncFirst, n_t-1 IncStep, n_t adjoint steps, body
    # force, 2D/1D spectra (2 forward + 1 inverse: 3 x (fft2 + fft1) are cuFFT, not counted), transposes
    # (4 at P > 1), combine, widening convert
    launches = 3 + 1 + 3 + 4 + 1 + (4 if world > 1 else 0) + 1 + 1
    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 transport / f64 control", "data": "synthetic (dist.slab_synth rotation, generated slab by "
                                                            "slab on the ranks, fp32 64-step reference transport)",
            "config": {"workload": f"{'C5' if n >= 1024 else 'C4'}: ONE {n}^3 GN Hessian matvec slab-decomposed "
                                   f"over {world} rank(s), nt=4, cubic-Lagrange SL, FD8, H1 alpha=1e-2, "
                                   "near-incompressible beta=1e-4, SSD",
                       "grid": [n, n, n], "n_t": 4, "interp": "cubic", "precision": "mixed",
                       "parallelism": f"slab along axis 0 x{world} ({'gloo-staged' if staged else 'NCCL'} "
                                      "all-to-all FFT transposes, " +
                                      ("off-rank stencil planes read from the owners' CUDA-IPC peer windows "
                                       "(FRG_SLAB_PEER=1)" if os.environ.get("FRG_SLAB_PEER") == "1"
                                       else "ghost-plane send/recv") + ")",
                       "halo_planes": halo,
                       "l2": "inputs > L2 (GB-scale working set per matvec, no flush needed)"},
            "e2e": {"value": e2e_steps / t_e2e, "unit": UNIT,
                    "h2d_bytes_per_step": host_in.numel() * host_in.element_size() * world,
                    "d2h_bytes_per_step": host_out.numel() * host_out.element_size() * world,
                    "steps": e2e_steps, "path": "pinned host v~ slab per rank -> DistKktState.hessian_matvec -> "
                                                "pinned host, serial per step",
                    "latency": {"value": 1.0 / t_lat, "unit": UNIT, "ms_per_call": 1e3 * t_lat, "steps": lat_steps,
                                "note": "each call's H2D, matvec and D2H complete on the host before the next "
                                        "call"}},
            "gpu_launches": launches * a.steps,
            "roofline": {"bound": "hbm", "achieved": inc_bytes / t_inc / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": inc_bytes / t_inc / 1e9 / peak, "traffic": None,
                         "kernel": "k_slf<CUBIC,3,IncFirstOp<float,3>> on this rank's slab (the matvec's dominant "
                                   "kernel, timed live inside the timed matvecs, max over ranks)",
                         "algorithmic_bytes_per_launch": inc_bytes, "launch_s": t_inc,
                         "launches_timed": probe_n.value, "peak_source": peak_src},
            "gather_roofline": {"bound": "hbm", "achieved": alg_bytes / t_gather / 1e9, "peak": peak,
                                "unit": "GB/s", "frac": alg_bytes / t_gather / 1e9 / peak, "traffic": None,
                                "kernel": "k_slf<CUBIC,1,GatherOp<float,1>> on this rank's slab (frg_slab_gather, "
                                          "tile plan)", "algorithmic_bytes_per_launch": alg_bytes,
                                "launch_s": t_gather, "peak_source": peak_src},
            "matvec_roofline": {"canonical_bytes_per_rank": canon, "achieved_gbs": canon / (t / a.steps) / 1e9,
                                "peak_gbs": peak, "frac": canon / (t / a.steps) / 1e9 / peak,
                                "note": "SURVEY.md §8d canonical 174 fp32 field passes per matvec, per rank"},
            "nvlink": {"bytes_per_step_per_rank": sent, "achieved_gbs": sent / (t / a.steps) / 1e9,
                       "peak_gbs": 900.0, "frac": sent / (t / a.steps) / 900e9,
                       "note": "payload each rank sends per matvec (halo planes + off-rank all-to-all chunks) / "
                               "step time; 0 at P = 1"},
            "time_to_solution": tts,
            "clocks": clk.summary(),
            "cpu_baseline": None,
        }
        print(json.dumps(res))
    barrier()
    dist.destroy_process_group()
    return None


def host_info():
    """lscpu-equivalent facts from /proc/cpuinfo + the threading the port uses."""
    model, phys, logical = "unknown", set(), 0
    try:
        cur = {}
        for line in open("/proc/cpuinfo"):
            if ":" not in line:
                if cur:
                    phys.add((cur.get("physical id", "0"), cur.get("core id", str(logical))))
                    cur = {}
                continue
            k, v = (x.strip() for x in line.split(":", 1))
            if k == "processor":
                logical += 1
            if k == "model name":
                model = v
            if k in ("physical id", "core id"):
                cur[k] = v
        if cur:
            phys.add((cur.get("physical id", "0"), cur.get("core id", str(logical))))
    except OSError:
        pass
    threads = os.cpu_count() or 1
    return {"cpu_model": model, "logical_cpus": logical or threads, "physical_cores": len(phys) or None,
            "threading": f"OpenMP gathers (oracle/csrc/gather_ref.c, OMP default = {threads} threads) + "
                         f"scipy.fft pocketfft workers={threads}; numpy single-threaded elsewhere"}


# the reference itself (numba, pkg/src/flowreg) cannot travel to the GPU box
# (/root/reference is absent there); BASELINE.md §3 measured it in the survey
# container (1 socket x 8 cores): C1 register 10.1 s, 64^3 matvec 0.341 s,
# 128^3 near-incompressible matvec 4.36 s.  The port runs C1 in 5.6 s on an
# 8-core container of the same kind, so GPU / port ratios understate GPU /
# reference by ~1.8x.
PORT_VS_NUMBA = {"numba_reference_c1_register_s_8cores": 10.1, "port_c1_register_s_8cores": 5.6,
                 "source": "BASELINE.md §3 (survey container) and this repo's build container"}


def all_host_threads() -> int:
    """Let the CPU arms use every host thread: torchrun exports
    OMP_NUM_THREADS=1 to its ranks, which would pin the oracle's OpenMP
    gathers to one core (scipy.fft takes its worker count explicitly)."""
    import ctypes

    cores = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(cores)
    try:  # an OpenMP runtime already initialised in this process keeps its ICV: set it too
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(cores)
    except OSError:
        pass
    return cores


def cpu_c1_register():
    """The oracle port's full C1 solve (64^3 rotation, H1, reg precond, cubic, fd8,
    f64) on the host cores — BASELINE.md §2 item 3; synth excluded."""
    from oracle import flowreg_oracle as O

    m0, m1, _ = O.synth_case("rotation", 64, seed=1, d=3, ref_steps=64)
    t0 = time.perf_counter()
    _, rep = O.register(m0, m1, O.Reg(alpha=1e-2, incomp="none"), precond="reg", method="cubic", scheme="fd8")
    dt = time.perf_counter() - t0
    return {"config": "C1: 64^3 rotation, H1 alpha=1e-2, reg precond, cubic, fd8, f64 (oracle port)",
            "seconds": dt, "iterations": rep["iterations"], "matvecs": rep["matvecs"],
            "pde_solves": rep["pde_solves"], "status": rep["status"]}


def cpu_baseline(a, m0, m1, vtrue, vt):
    """Oracle port on the host cores: one full 256^3 matvec (refresh untimed)
    plus a full C1 registration."""
    import numpy as np

    from oracle import flowreg_oracle as O

    cores = all_host_threads()
    M0 = m0.values.double().cpu().numpy()
    M1 = m1.values.double().cpu().numpy()
    V = 0.5 * vtrue.data.double().cpu().numpy()
    VT = vt.data.double().cpu().numpy()
    st = O.Kkt(M0, M1, O.Reg(alpha=1e-2, incomp="near-incompressible", beta=1e-4), 4, "ssd", "cubic", "fd8", V)
    t0 = time.perf_counter()
    st.hessian_matvec(VT)
    dt = time.perf_counter() - t0
    del st
    return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"1 Hessian matvec at {a.n}^3 f64 (oracle/flowreg_oracle.py, C/OpenMP gathers + "
                      f"scipy pocketfft, {cores} threads); refresh excluded",
            "host": host_info(), "time_to_solution_c1": cpu_c1_register(), "port_vs_numba": PORT_VS_NUMBA}


# ---------------------------------------------------------------------------
# reference arm (CPU oracle port)
# ---------------------------------------------------------------------------
def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import numpy as np

    from oracle import flowreg_oracle as O

    n = a.n
    cores = all_host_threads()
    # inputs: the oracle's own synth (64-step cubic transport); bounded run
    m0, m1, vtrue = O.synth_case("rotation", n, seed=1, d=3, ref_steps=64)
    st = O.Kkt(m0, m1, O.Reg(alpha=1e-2, incomp="near-incompressible", beta=1e-4), 4, "ssd", "cubic", "fd8",
               0.5 * vtrue)
    vt = 0.1 * np.random.default_rng(0).standard_normal(vtrue.shape)
    warm = min(a.warmup, 1)
    steps = max(1, min(a.steps, 2))
    for _ in range(warm):
        st.hessian_matvec(vt)
    t0 = time.perf_counter()
    for _ in range(steps):
        st.hessian_matvec(vt)
    dt = time.perf_counter() - t0
    value = steps / dt
    sample = (f"{steps} timed + {warm} warm-up Hessian matvecs at {n}^3 (f64 oracle port, {cores} host threads); "
              f"bounded from --steps {a.steps} --warmup {a.warmup} to keep the run within minutes")
    del st
    tts = cpu_c1_register()
    res = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": steps,
           "warmup": warm, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (oracle synth_case rotation)",
           "config": config(n, "f64"),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                            "host": host_info(), "port_vs_numba": PORT_VS_NUMBA},
           "time_to_solution": tts,
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res))
    return res


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
