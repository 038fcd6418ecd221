"""Slab-decomposed multi-GPU GN-Krylov core.

The reference package is single-process (pkg/src/flowreg has no MPI/NCCL);
CLAIRE's distributed design is described in PAPER.md:500-545: slabs along
the slowest axis, FFT transposes by all-to-all, off-rank departure points.
This module is that layer for one node of B200s, one process per GPU:

* rank r owns planes [r n0/P, (r+1) n0/P) of every field (axis 0, the
  slowest C-order axis = the paper's x1);
* SL steps and FD8 read GHOST PLANES: before each gather the source field's
  W nearest planes are exchanged with the two ring neighbours
  (``SlabComm.halo``: NCCL send/recv), W = ceil(max |disp_0|) + 2 for cubic,
  computed once per displacement map and max-reduced over ranks, then the
  fp32 TMA gather kernel runs on the owned planes with h0 = W (no axis-0
  wrap).  This replaces routing every off-rank departure point by a
  CFL-bounded halo: 3-5x the bytes of routing on the bench maps
  (profiles/r02_halo_vs_routing_*.json) but one contiguous send/recv per
  neighbour, no compaction, count exchange or remote-gather pass
  (DESIGN.md §8);
* spectral operators run as batched 2D R2C over the owned planes, a packed
  all-to-all to an axis-1 split, a batched 1D C2C along axis 0, the fused
  pointwise operator with global frequencies, and the inverse chain
  (``SlabFFT``);
* reductions are local fused kernels + one all-reduce of a scalar.

Host control (PCG / Armijo / Newton) is replicated SPMD: every rank runs the
same ``optimizer`` code on identical all-reduced scalars
(``dist_register``).  The exchange uses torch.distributed — NCCL on the GPU
box; with the gloo backend (CPU tests, or several ranks sharing one GPU)
buffers are staged through host memory.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as tdist

from . import _lib as L
from .diffops import frg_reg
from .kkt import PrecondKind, RegConfig

__all__ = ["SlabComm", "SlabGrid", "SlabFFT", "DistKktState", "dist_register", "dist_continuation_solve",
           "dist_search_alpha", "slab_bounds", "halo_width", "slab_synth"]

TWO_PI = 2.0 * math.pi


def slab_bounds(n0: int, nranks: int, rank: int) -> tuple[int, int]:
    """Owned plane range [lo, hi) of ``rank`` (n0 must split evenly)."""
    if n0 % nranks != 0:
        raise ValueError(f"n0 = {n0} does not split over {nranks} ranks")
    m = n0 // nranks
    return rank * m, (rank + 1) * m


def halo_width(max_abs_disp0: float, method: str = "cubic") -> int:
    """Ghost planes a gather needs for axis-0 displacements |d0| <= max_abs_disp0
    (index units): stencil planes floor(d0) - 1 .. floor(d0) + 2 for cubic,
    floor(d0) .. floor(d0) + 1 for linear (B-spline: the cubic support)."""
    extra = 1 if method == "linear" else 2
    return int(math.ceil(max(float(max_abs_disp0), 0.0))) + extra


class SlabComm:
    """Ring / all-to-all / all-reduce exchanges of the slab decomposition.

    NCCL moves device tensors directly; any other backend stages through
    host memory (gloo tests, several ranks on one GPU)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = tdist.get_rank(group)
        self.size = tdist.get_world_size(group)
        self.staged = tdist.get_backend(group) != "nccl"
        self.bytes_sent = 0  # payload this rank sent (halo planes + all-to-all chunks to other ranks)

    # -- scalars -----------------------------------------------------------
    def all_reduce(self, value: float, op: str = "sum") -> float:
        if self.size == 1:
            return float(value)
        dev = "cpu" if self.staged else torch.device("cuda", torch.cuda.current_device())
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        ops = {"sum": tdist.ReduceOp.SUM, "max": tdist.ReduceOp.MAX, "min": tdist.ReduceOp.MIN}
        tdist.all_reduce(t, op=ops[op], group=self.group)
        return float(t.item())

    # -- all-to-all with equal chunks along dim 0 -------------------------
    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        if self.size == 1:
            out.copy_(inp)
            return
        if out.is_complex():  # NCCL has no complex type: move the (re, im) pairs as reals
            out, inp = torch.view_as_real(out), torch.view_as_real(inp)
        self.bytes_sent += inp.numel() * inp.element_size() * (self.size - 1) // self.size
        if self.staged:
            o = torch.empty(out.shape, dtype=out.dtype)
            tdist.all_to_all_single(o, inp.cpu(), group=self.group)
            out.copy_(o)
        else:
            tdist.all_to_all_single(out, inp, group=self.group)

    def device_barrier(self) -> None:
        """Order every rank's prior device work before every rank's next
        kernel: a one-element NCCL all-reduce on the current stream (gloo:
        synchronise the device, then a host barrier)."""
        if self.size == 1:
            return
        if self.staged:
            torch.cuda.synchronize()
            tdist.barrier(group=self.group)
            return
        if getattr(self, "_bar", None) is None:
            self._bar = torch.zeros(1, dtype=torch.float32, device="cuda")
        tdist.all_reduce(self._bar, group=self.group)

    # -- ghost planes ----------------------------------------------------
    def halo(self, ext: torch.Tensor, W: int) -> None:
        """ext (C, n0_loc + 2W, n1, n2) with the owned planes at [W, W + n0_loc):
        fill the W ghost planes on each side from the periodic ring neighbours."""
        if W == 0:
            return
        n0l = ext.shape[1] - 2 * W
        if W > n0l and self.size > 1:
            raise ValueError(f"halo of {W} planes exceeds the {n0l}-plane slab; use fewer ranks")
        if self.size == 1:
            ext[:, :W].copy_(ext[:, n0l:n0l + W])
            ext[:, n0l + W:].copy_(ext[:, W:2 * W])
            return
        prev, nxt = (self.rank - 1) % self.size, (self.rank + 1) % self.size
        send_lo = ext[:, W:2 * W].contiguous()          # my first planes -> prev's upper ghosts
        send_hi = ext[:, n0l:n0l + W].contiguous()      # my last planes  -> next's lower ghosts
        self.bytes_sent += 2 * send_lo.numel() * send_lo.element_size()
        recv_hi = torch.empty_like(send_lo)
        recv_lo = torch.empty_like(send_hi)
        if self.staged:
            send_lo, send_hi = send_lo.cpu(), send_hi.cpu()
            recv_hi, recv_lo = recv_hi.cpu(), recv_lo.cpu()
        # identical op order on every rank: with P = 2 both messages share a
        # peer and match in issue order (send_lo <-> recv_hi, send_hi <-> recv_lo)
        ops = [tdist.P2POp(tdist.isend, send_lo, prev, self.group),
               tdist.P2POp(tdist.irecv, recv_hi, nxt, self.group),
               tdist.P2POp(tdist.isend, send_hi, nxt, self.group),
               tdist.P2POp(tdist.irecv, recv_lo, prev, self.group)]
        for req in tdist.batch_isend_irecv(ops):
            req.wait()
        ext[:, :W].copy_(recv_lo)
        ext[:, n0l + W:].copy_(recv_hi)


class _CudaArray:
    """__cuda_array_interface__ of a raw fp32 device buffer (torch.as_tensor wraps it, zero copy)."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": "<f4",
                                         "data": (int(ptr), False), "version": 2}


class PeerWindows:
    """Peer mode of the slab path (no ghost planes): NBLK blocks of
    (C, n0_loc, n1, n2) fp32 per rank, exported with CUDA IPC, mapped into
    every other rank and registered per component with the library
    (frg_peer_register), so that a slab SL call whose sources are window
    components reads the stencil planes owned by other ranks straight from
    their windows — TMA / P2P loads over NVLink — instead of exchanging
    CFL-wide ghost slabs (the north star's off-rank departure points,
    PAPER.md:545).  Blocks alternate between gathers: one device barrier per
    gather (after filling the next block) orders every rank's fill before
    every peer's reads and every peer's reads of a block before its refill."""

    NBLK = 2
    _cache: dict = {}

    @classmethod
    def get(cls, comm: SlabComm, shape) -> "PeerWindows":
        """One set of windows per (communicator, shape) for the life of the
        process: freeing a window while a peer may still read it would need a
        collective in a destructor; states of the same grid share the ring."""
        key = (id(comm.group), comm.rank, comm.size, tuple(int(x) for x in shape))
        w = cls._cache.get(key)
        if w is None:
            w = cls._cache[key] = cls(comm, shape)
        else:
            w.comm = comm
        return w

    def __init__(self, comm: SlabComm, shape):
        self.comm, self.shape = comm, tuple(int(x) for x in shape)
        P, rank = comm.size, comm.rank
        C = self.shape[0]
        comp = int(np.prod(self.shape[1:]))
        self._own, self._opened, self.blocks = [], [], []
        n3 = L.n3(self.shape[1:])
        for _ in range(self.NBLK):
            ptr, h = ctypes.c_void_p(), (ctypes.c_ubyte * 64)()
            L.check(L.lib().frg_peer_alloc(4 * C * comp, ctypes.byref(ptr), h), "peer_alloc")
            self._own.append(ptr.value)
            handles = [None] * P
            tdist.all_gather_object(handles, bytes(h), group=comm.group)
            bases = []
            for r in range(P):
                if r == rank:
                    bases.append(ptr.value)
                    continue
                q = ctypes.c_void_p()
                hb = (ctypes.c_ubyte * 64).from_buffer_copy(handles[r])
                L.check(L.lib().frg_peer_open(hb, ctypes.byref(q)), "peer_open")
                self._opened.append(q.value)
                bases.append(q.value)
            for c in range(C):
                off = 4 * c * comp
                arr = (ctypes.c_void_p * P)(*[b + off for b in bases])
                L.check(L.lib().frg_peer_register(ctypes.c_void_p(ptr.value + off), n3, P, rank, arr),
                        "peer_register")
            self.blocks.append(torch.as_tensor(_CudaArray(ptr.value, self.shape), device="cuda"))
        self._k = 0
        comm.device_barrier()

    def next(self, C: int) -> torch.Tensor:
        """The next block's first C components (the caller fills them, then calls publish())."""
        if C > self.shape[0]:
            raise ValueError(f"{C} fields exceed the {self.shape[0]}-component peer windows")
        blk = self.blocks[self._k % self.NBLK]
        self._k += 1
        return blk[:C]

    def publish(self) -> None:
        self.comm.device_barrier()

    def close(self):
        lib = L._lib
        if lib is None:
            return
        try:
            torch.cuda.synchronize()
            comp = int(np.prod(self.shape[1:]))
            for p in self._own:
                for c in range(self.shape[0]):
                    lib.frg_peer_unregister(ctypes.c_void_p(p + 4 * c * comp))
            for q in self._opened:
                lib.frg_peer_close(ctypes.c_void_p(q))
            for p in self._own:
                lib.frg_peer_free(ctypes.c_void_p(p))
        except Exception:
            pass
        self._own, self._opened = [], []


@dataclass(frozen=True)
class SlabGrid:
    """Global grid + this rank's slab.  Quacks like fields.Grid for the host
    control code (cell_volume, d, n_t, dtype; ``n`` is the LOCAL shape)."""

    n_glob: tuple
    rank: int
    size: int
    n_t: int = 4
    dtype: np.dtype = np.dtype(np.float64)

    @property
    def lo(self) -> int:
        return slab_bounds(self.n_glob[0], self.size, self.rank)[0]

    @property
    def n0_loc(self) -> int:
        return self.n_glob[0] // self.size

    @property
    def n(self) -> tuple:
        return (self.n0_loc, self.n_glob[1], self.n_glob[2])

    @property
    def d(self) -> int:
        return 3

    @property
    def h(self) -> tuple:
        return tuple(TWO_PI / ni for ni in self.n_glob)

    @property
    def h_t(self) -> float:
        return 1.0 / self.n_t

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.h))

    @property
    def torch_dtype(self):
        return torch.float64 if np.dtype(self.dtype) == np.float64 else torch.float32


def _c(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


class SlabFFT:
    """Distributed real FFT of slab fields (see module docstring)."""

    def __init__(self, grid: SlabGrid, comm: SlabComm):
        n0, n1, n2 = grid.n_glob
        if n0 % comm.size or n1 % comm.size:
            raise ValueError("n0 and n1 must both split over the ranks")
        self.g, self.comm = grid, comm
        self.nh = n2 // 2 + 1
        self.n1l = n1 // comm.size
        self.i1_off = comm.rank * self.n1l
        self.nloc = L.n3(grid.n)
        self.nglob = L.n3(grid.n_glob)

    def spectrum(self, ncomp: int, dtype: torch.dtype) -> torch.Tensor:
        cdt = torch.complex128 if dtype == torch.float64 else torch.complex64
        return torch.empty((ncomp, self.g.n_glob[0], self.n1l, self.nh), dtype=cdt, device="cuda")

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x real (C, n0_loc, n1, n2) -> axis-1 split spectrum (C, n0, n1/P, nh)."""
        C = x.shape[0]
        dt = L.dtype_code(x.dtype)
        cdt = torch.complex128 if x.dtype == torch.float64 else torch.complex64
        n0l, n1, _ = self.g.n
        P = self.comm.size
        y = torch.empty((C, n0l, n1, self.nh), dtype=cdt, device="cuda")
        L.check(L.lib().frg_slab_fft2(self.nloc, dt, C, 1, _c(x), _c(y), L.stream()), "slab_fft2")
        if P == 1:  # the axis-1 split is the whole axis: no transpose, no exchange
            L.check(L.lib().frg_slab_fft1(self.g.n_glob[0], self.n1l, self.g.n_glob[2], dt, C, 1, _c(y), L.stream()),
                    "slab_fft1")
            return y
        packed = torch.empty((C, P, n0l, self.n1l, self.nh), dtype=cdt, device="cuda")
        L.check(L.lib().frg_slab_transpose(1, P, self.nloc, dt, C, _c(y), _c(packed), L.stream()), "slab_transpose")
        spec = self.spectrum(C, x.dtype)
        for c in range(C):
            self.comm.all_to_all(spec[c].view(P, n0l, self.n1l, self.nh), packed[c])
        L.check(L.lib().frg_slab_fft1(self.g.n_glob[0], self.n1l, self.g.n_glob[2], dt, C, 1, _c(spec), L.stream()),
                "slab_fft1")
        return spec

    def inverse(self, spec: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """(C, n0, n1/P, nh) -> real (C, n0_loc, n1, n2), unnormalised; spec is consumed."""
        C = spec.shape[0]
        dt = L.dtype_code(out.dtype)
        n0l, n1, _ = self.g.n
        P = self.comm.size
        L.check(L.lib().frg_slab_fft1(self.g.n_glob[0], self.n1l, self.g.n_glob[2], dt, C, -1, _c(spec), L.stream()),
                "slab_fft1")
        if P == 1:
            L.check(L.lib().frg_slab_fft2(self.nloc, dt, C, -1, _c(spec), _c(out), L.stream()), "slab_fft2")
            return out
        packed = torch.empty((C, P, n0l, self.n1l, self.nh), dtype=spec.dtype, device="cuda")
        for c in range(C):
            self.comm.all_to_all(packed[c], spec[c].view(P, n0l, self.n1l, self.nh))
        y = torch.empty((C, n0l, n1, self.nh), dtype=spec.dtype, device="cuda")
        L.check(L.lib().frg_slab_transpose(-1, P, self.nloc, dt, C, _c(packed), _c(y), L.stream()), "slab_transpose")
        L.check(L.lib().frg_slab_fft2(self.nloc, dt, C, -1, _c(y), _c(out), L.stream()), "slab_fft2")
        return out

    def apply(self, x: torch.Tensor, kind: str, reg, out: torch.Tensor | None = None) -> torch.Tensor:
        """real(ifft(symbol * fft(x))) for the symbols of frg_slab_spec_apply."""
        spec = self.forward(x)
        L.check(L.lib().frg_slab_spec_apply(self.nglob, self.i1_off, self.n1l, L.dtype_code(x.dtype), x.shape[0],
                                            _c(spec), L.SYM[kind], ctypes.byref(reg), L.stream()), "slab_spec_apply")
        out = torch.empty_like(x) if out is None else out
        return self.inverse(spec, out)

    def reg_plus_project(self, a: torch.Tensor | None, b: torch.Tensor, reg, project: bool,
                         out: torch.Tensor) -> torch.Tensor:
        """out = alpha L a + P(b) (a may be None: P(b) only); a, b, out same dtype."""
        sb = self.forward(b)
        sa = self.forward(a) if a is not None else sb
        L.check(L.lib().frg_slab_spec_combine(self.nglob, self.i1_off, self.n1l, L.dtype_code(b.dtype), _c(sa),
                                              _c(sb), ctypes.byref(reg), int(project), L.stream()),
                "slab_spec_combine")
        return self.inverse(sa, out)


class _Vec:
    """Minimal VectorField stand-in for the host control code (.grid, .data)."""

    __slots__ = ("grid", "data")

    def __init__(self, grid, data):
        self.grid, self.data = grid, data


class DistKktState:
    """Slab-decomposed counterpart of kkt.KktState (kkt.py:136-341) for SSD,
    FD8, linear / cubic / B-spline fp32 transport, fp64 control vectors.
    B-spline: every gathered field is first prefiltered globally (slab FFT,
    symbol 1 / prod_a (4 + 2 cos(2 pi m_a / n_a)) / 6) and its coefficients
    exchanged; nodal values stay where the kernels read them locally.

    Same methods and counters as KktState (refresh, gradient, hessian_matvec,
    apply_precond('reg'), objective, objective_at, mismatch), each a sequence
    of per-rank slab kernels and exchanges; all ranks call them in lockstep."""

    def __init__(self, m0: torch.Tensor, m1: torch.Tensor, reg: RegConfig, comm: SlabComm, n_glob, n_t: int = 4,
                 method: str = "cubic", v_init: torch.Tensor | None = None, peer: bool | None = None,
                 distance: str = "ssd"):
        """``peer=True`` (default: env FRG_SLAB_PEER=1): SL gathers read off-rank
        stencil planes from the owners' peer windows (PeerWindows) instead of
        exchanging ghost slabs of width ceil(max |disp_0|) + 2; FD8 keeps its
        4 ghost planes."""
        if method not in ("linear", "cubic", "bspline"):
            raise ValueError("slab transport supports linear / cubic / bspline interpolation")
        if distance not in ("ssd", "ncc"):
            raise ValueError(f"unknown distance measure {distance!r}")
        self.distance = distance
        self.comm = comm
        self.grid = SlabGrid(tuple(int(v) for v in n_glob), comm.rank, comm.size, n_t=n_t)
        self.peer = (os.environ.get("FRG_SLAB_PEER") == "1") if peer is None else bool(peer)
        self._win = PeerWindows.get(comm, (9, *self.grid.n)) if self.peer else None
        self.reg = reg
        self.method = method
        self._m = L.METHODS[method]
        self._bs = method == "bspline"
        self._reg = frg_reg(reg.operator, reg.alpha, reg.incomp)
        self._project = reg.incomp.mode != "none"
        # spectral operators on f64 spectra: fp32 rounding of a smooth field is
        # amplified by alpha |k|^2 at high frequencies (4x per grid doubling,
        # 3.6e-4 rel-L2 on a 256^3 gradient), see kkt.cu mixed_spectral
        self._spec_dt = torch.float64
        self.fft = SlabFFT(self.grid, comm)
        g = self.grid
        self.n_loc = L.n3(g.n)
        self.N = int(np.prod(g.n))
        self.m0 = m0.to(device="cuda", dtype=torch.float32).contiguous()
        self.m1 = m1.to(device="cuda", dtype=torch.float32).contiguous()
        if tuple(self.m0.shape) != g.n or tuple(self.m1.shape) != g.n:
            raise ValueError(f"slab images must be {g.n}")
        self.matvecs = 0
        self.pde_solves = 0
        self.precond_fallbacks = 0
        self._init_mismatch = self._dist_value(self.m0)
        v0 = torch.zeros((3, *g.n), dtype=torch.float64, device="cuda") if v_init is None else v_init
        self.refresh(v0)

    # -- helpers -----------------------------------------------------------
    def _ext(self, x: torch.Tensor, W: int) -> torch.Tensor:
        """(C, n0_loc, n1, n2) -> (C, n0_loc + 2W, n1, n2) with exchanged ghost planes."""
        x = x if x.dim() == 4 else x.unsqueeze(0)
        C, n0l = x.shape[0], x.shape[1]
        ext = torch.empty((C, n0l + 2 * W, *x.shape[2:]), dtype=x.dtype, device=x.device)
        ext[:, W:W + n0l].copy_(x)
        self.comm.halo(ext, W)
        return ext

    def _coef(self, x: torch.Tensor) -> torch.Tensor:
        """What a gather reads of field x: x itself, or (B-spline) its global
        prefilter coefficients."""
        if not self._bs:
            return x
        xx = x if x.dim() == 4 else x.unsqueeze(0)
        return self.fft.apply(xx.contiguous(), "bspline_prefilter", self._reg).view(x.shape)

    def _src(self, x: torch.Tensor, W: int) -> torch.Tensor:
        """Ghost-extended gather source of x (coefficients for B-spline); in
        peer mode (W == 0) the next published peer-window block."""
        if self.peer:
            c = self._coef(x)
            c = c if c.dim() == 4 else c.unsqueeze(0)
            blk = self._win.next(c.shape[0])
            blk.copy_(c)
            self._win.publish()
            return blk
        return self._ext(self._coef(x), W)

    def _plan(self, disp: torch.Tensor) -> torch.Tensor:
        """Tile plan of a slab displacement map (the SL steps issue their TMA
        from it instead of reducing the stencil box per tile)."""
        plan = torch.empty((L.lib().frg_tile_plan_count(self.n_loc), 4), dtype=torch.int32, device="cuda")
        L.check(L.lib().frg_tile_plan(self.n_loc, 3, self._m, _c(disp), _c(plan), L.stream()), "tile_plan")
        return plan

    def _bind(self):
        """Bind disp_f / disp_b to their plans for the calls that follow."""
        L.check(L.lib().frg_bind_plan(0, _c(self.disp_f), _c(self.plan_f), self._m), "bind_plan")
        L.check(L.lib().frg_bind_plan(1, _c(self.disp_b), _c(self.plan_b), self._m), "bind_plan")

    def __del__(self):
        # drop this state's plan bindings (their maps are about to be freed)
        try:
            if L._lib is not None:
                L.lib().frg_clear_plans()
        except Exception:
            pass

    def _absmax(self, a: torch.Tensor) -> float:
        """Global max |a| (one fused reduction + one scalar all-reduce; the
        host needs it to size the ghost planes, once per displacement map)."""
        out = ctypes.c_double()
        L.check(L.lib().frg_norm_inf(L.dtype_code(a.dtype), L.ptr(a), a.numel(), ctypes.byref(out), L.stream()),
                "norm_inf")
        return self.comm.all_reduce(out.value, "max")

    def _halo_of(self, disp: torch.Tensor) -> int:
        if self.peer:
            return 0
        return max(halo_width(self._absmax(disp[0]), self.method), 1)

    def dot(self, a: torch.Tensor, b: torch.Tensor) -> float:
        """Global sum(a * b) (unweighted), fused local kernel + all-reduce."""
        out = ctypes.c_double()
        L.check(L.lib().frg_dot(L.dtype_code(a.dtype), L.ptr(a), L.ptr(b), a.numel(), ctypes.byref(out), L.stream()),
                "dot")
        return self.comm.all_reduce(out.value)

    def norm_inf(self, a: torch.Tensor) -> float:
        out = ctypes.c_double()
        L.check(L.lib().frg_norm_inf(L.dtype_code(a.dtype), L.ptr(a), a.numel(), ctypes.byref(out), L.stream()),
                "norm_inf")
        return self.comm.all_reduce(out.value, "max")

    def _ssd(self, md: torch.Tensor) -> float:
        r = md - self.m1
        return 0.5 * self.dot(r, r) * self.grid.cell_volume

    # -- distance measures (distance.py:34-91), global moments all-reduced ----
    def _ncc_moments(self, md: torch.Tensor):
        cv = self.grid.cell_volume
        a, b, c = self.dot(self.m1, md) * cv, self.dot(md, md) * cv, self.dot(self.m1, self.m1) * cv
        if b <= 0.0 or c <= 0.0:
            from .distance import ZeroNormError

            raise ZeroNormError("normalized cross correlation needs nonzero images")
        return a, b, c

    def _dist_value(self, md: torch.Tensor) -> float:
        if self.distance == "ssd":
            return self._ssd(md)
        a, b, c = self._ncc_moments(md)
        return 1.0 - (a * a) / (b * c)

    def _adjoint_final(self, md: torch.Tensor, out: torch.Tensor) -> None:
        """lambda(1) = minus the mismatch gradient in md (distance.py:58-68)."""
        if self.distance == "ssd":
            torch.sub(self.m1, md, out=out)
            return
        a, b, c = self._ncc_moments(md)
        f = -2.0 * a / (b * c)
        torch.mul(md, f * a / b, out=out)
        out.add_(self.m1, alpha=-f)

    def _incremental_final(self, mt: torch.Tensor, out: torch.Tensor) -> None:
        """lambda~(1), the GN final condition of the incremental dual
        (distance.py:71-91; SSD is fused into the last incremental step)."""
        md = self.mseries[-1]
        a, b, c = self._ncc_moments(md)
        cv = self.grid.cell_volume
        mm, rm = self.dot(md, mt) * cv, self.dot(self.m1, mt) * cv
        q1 = 2.0 * a * mm / b ** 2 - rm / b
        q2 = 4.0 * a * a * mm / b ** 3 - 2.0 * a * rm / b ** 2
        q3 = a * a / b ** 2
        torch.mul(self.m1, -2.0 * q1 / c, out=out)
        out.add_(md, alpha=2.0 * q2 / c).add_(mt, alpha=-2.0 * q3 / c)

    def _gather(self, disp, W, srcs, outs):
        ins = (ctypes.c_void_p * len(srcs))(*[s.data_ptr() for s in srcs])
        ous = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        L.check(L.lib().frg_slab_gather(self.n_loc, self.grid.n_glob[0], W, self._m, _c(disp), len(srcs), ins, ous,
                                        L.stream()), "slab_gather")

    def _departure(self, v32: torch.Tensor, sign: float) -> torch.Tensor:
        vs = v32 if sign > 0 else -v32
        h0 = TWO_PI / self.grid.n_glob[0]
        Wv = 0 if self.peer else max(halo_width(self._absmax(v32[0]) * self.grid.h_t / h0, self.method), 4)
        v_ext = self._src(vs, Wv)
        disp = torch.empty_like(vs)
        L.check(L.lib().frg_slab_departure(self.n_loc, self.grid.n_glob[0], Wv, self._m, self.grid.h_t, _c(v_ext),
                                           _c(vs), _c(disp), L.stream()), "slab_departure")
        return disp, v_ext, Wv

    def _state_solve(self, disp, W, keep: bool, m0: torch.Tensor | None = None):
        g = self.grid
        m = self.m0 if m0 is None else m0
        series = [m] if keep else None
        for _ in range(g.n_t):
            nxt = torch.empty_like(m)
            self._gather(disp, W, [self._src(m, W)], [nxt])
            m = nxt
            if keep:
                series.append(m)
        return series if keep else m

    def _spectral_out(self, a64: torch.Tensor | None, b32: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """out (fp64) = alpha L a + P(b), the single-GPU mixed arithmetic
        (kkt.cu reg_plus_project_mixed): the f64 spectrum of a, the fp32
        spectrum of b, an fp32 combine per bin, an fp32 inverse, one widening
        pass into out — half the all-to-all bytes of f64 b spectra."""
        sb = self.fft.forward(b32)
        sa = self.fft.forward(a64) if a64 is not None else None
        L.check(L.lib().frg_slab_spec_combine_mixed(self.fft.nglob, self.fft.i1_off, self.fft.n1l,
                                                    None if sa is None else _c(sa), _c(sb), ctypes.byref(self._reg),
                                                    int(self._project), L.stream()), "slab_spec_combine_mixed")
        res = torch.empty(b32.shape, dtype=torch.float32, device="cuda")
        self.fft.inverse(sb, res)
        L.check(L.lib().frg_convert(L.F32, _c(res), L.F64, _c(out), res.numel(), L.stream()), "convert")
        return out

    def _body_force(self, lam):
        g = self.grid
        b = torch.empty((3, *g.n), dtype=torch.float32, device="cuda")
        L.check(L.lib().frg_body_force(self.n_loc, 3, L.F32, g.n_t, _c(lam), _c(self.grads), _c(b), L.stream()),
                "body_force")
        return b

    # -- KktState surface ------------------------------------------------
    def refresh(self, v: torch.Tensor) -> None:
        """kkt.py:166-186 on the slab."""
        g = self.grid
        self.v = _Vec(g, v.to(device="cuda", dtype=torch.float64).contiguous())
        v32 = self.v.data.float()
        self.disp_f, v_ext, Wv = self._departure(v32, 1.0)
        self.disp_b, _, _ = self._departure(v32, -1.0)
        self.Wf, self.Wb = self._halo_of(self.disp_f), self._halo_of(self.disp_b)
        self.plan_f, self.plan_b = self._plan(self.disp_f), self._plan(self.disp_b)
        self._bind()
        divv = torch.empty(g.n, dtype=torch.float32, device="cuda")
        self.divv = divv
        if self._bs or self.peer:  # FD8 needs the nodal values with >= 4 ghost planes
            Wv = max(Wv, 4)
            v_ext = self._ext(v32, Wv)
        L.check(L.lib().frg_slab_fd8_divergence(self.n_loc, g.n_glob[0], Wv, _c(v_ext), _c(divv), L.stream()),
                "slab_fd8_divergence")
        self.mseries = self._state_solve(self.disp_f, self.Wf, keep=True)
        Wg = max(self.Wf, 4)
        self.grads = torch.empty((g.n_t + 1, 3, *g.n), dtype=torch.float32, device="cuda")
        for j, mj in enumerate(self.mseries):
            L.check(L.lib().frg_slab_fd8_gradient(self.n_loc, g.n_glob[0], Wg, 1, _c(self._ext(mj, Wg)),
                                                  _c(self.grads[j]), L.stream()), "slab_fd8_gradient")
        self.grads_y = torch.empty((g.n_t, 3, *g.n), dtype=torch.float32, device="cuda")
        for j in range(g.n_t):
            ext = self._src(self.grads[j], self.Wf)
            self._gather(self.disp_f, self.Wf, [ext[c] for c in range(3)], [self.grads_y[j, c] for c in range(3)])
        self.cmul = torch.empty(g.n, dtype=torch.float32, device="cuda")
        L.check(L.lib().frg_slab_adjoint_multiplier(self.n_loc, g.n_glob[0], self.Wb, self._m, g.h_t,
                                                    _c(self.disp_b), _c(self._src(divv, self.Wb)), _c(divv),
                                                    _c(self.cmul), L.stream()), "slab_adjoint_multiplier")
        self.lam = torch.empty((g.n_t + 1, *g.n), dtype=torch.float32, device="cuda")
        self._adjoint_final(self.mseries[-1], self.lam[g.n_t])
        self._adjoint(self.lam)
        self.pde_solves += 2
        self._dist = None
        self._h0_grad = None

    def _adjoint(self, series):
        g = self.grid
        for j in range(g.n_t, 0, -1):
            L.check(L.lib().frg_slab_adjoint_step(self.n_loc, g.n_glob[0], self.Wb, self._m, _c(self.disp_b),
                                                  _c(self.cmul), _c(self._src(series[j], self.Wb)),
                                                  _c(series[j - 1]), L.stream()), "slab_adjoint_step")

    def gradient(self) -> _Vec:
        out = torch.empty((3, *self.grid.n), dtype=torch.float64, device="cuda")
        self._spectral_out(self.v.data, self._body_force(self.lam), out)
        return _Vec(self.grid, out)

    def hessian_matvec(self, vtilde, out: torch.Tensor | None = None) -> _Vec:
        """kkt.py:237-260 (GN, SSD) on the slab.  The incremental state and
        adjoint series are stored with W ghost planes around every slice, so
        each step writes the owned planes of the next step's source in place
        and the exchange only fills the ghosts (no interior copy)."""
        g = self.grid
        self._bind()
        n0l, plane = g.n0_loc, g.n_glob[1] * g.n_glob[2]
        Wf, Wb = self.Wf, self.Wb
        vt = vtilde.data if hasattr(vtilde, "data") else vtilde
        if self._bs:  # gathers read exchanged coefficients; the Heun terms the nodal v~
            vt_loc = vt.to(torch.float32).contiguous()
            vt_ext, vt_loc_p = self._src(vt_loc, Wf), _c(vt_loc)
        else:
            vt_ext = (self._win.next(3) if self.peer else
                      torch.empty((3, n0l + 2 * Wf, *g.n[1:]), dtype=torch.float32, device="cuda"))
            vt64 = vt.to(torch.float64).contiguous()
            for c in range(3):  # f64 -> f32 straight into the owned planes (vectorised convert)
                L.check(L.lib().frg_convert(L.F64, _c(vt64[c]), L.F32, _c(vt_ext[c, Wf:Wf + n0l]), self.N,
                                            L.stream()), "convert")
            if self.peer:
                self._win.publish()
            else:
                self.comm.halo(vt_ext, Wf)
            vt_loc_p = None
        mt = torch.empty((g.n_t + 1, n0l + 2 * Wf, *g.n[1:]), dtype=torch.float32, device="cuda")
        S = torch.empty((max(g.n_t - 1, 1), *g.n), dtype=torch.float32, device="cuda")
        own_f = lambda j: mt[j, Wf:Wf + n0l]  # noqa: E731
        L.check(L.lib().frg_slab_inc_first(self.n_loc, g.n_glob[0], Wf, self._m, g.n_t, _c(self.disp_f),
                                           _c(self.grads), _c(self.grads_y), _c(vt_ext), vt_loc_p, _c(own_f(1)),
                                           _c(S), L.stream()), "slab_inc_first")

        def source(series, j, W):  # ghost-extended gather source of slice j
            if self._bs or self.peer:
                return self._src(series[j, W:W + n0l], W)[0]
            self.comm.halo(series[j:j + 1], W)
            return series[j]

        lt = torch.empty((g.n_t + 1, n0l + 2 * Wb, *g.n[1:]), dtype=torch.float32, device="cuda")
        ssd = self.distance == "ssd"
        for j in range(1, g.n_t):
            src = source(mt, j, Wf)
            # SSD: the last step writes lam~(1) = -m~(1) straight into the adjoint series
            last = ssd and j == g.n_t - 1
            L.check(L.lib().frg_slab_inc_step(self.n_loc, g.n_glob[0], Wf, self._m, _c(self.disp_f), _c(src),
                                              _c(S[j - 1]), None if last else _c(own_f(j + 1)),
                                              _c(lt[g.n_t, Wb:Wb + n0l]) if last else None, -1.0, L.stream()),
                    "slab_inc_step")
        if not ssd:
            self._incremental_final(own_f(g.n_t), lt[g.n_t, Wb:Wb + n0l])
        elif g.n_t == 1:
            torch.neg(own_f(1), out=lt[1, Wb:Wb + n0l])
        for j in range(g.n_t, 0, -1):
            src = source(lt, j, Wb)
            L.check(L.lib().frg_slab_adjoint_step(self.n_loc, g.n_glob[0], Wb, self._m, _c(self.disp_b),
                                                  _c(self.cmul), _c(src), _c(lt[j - 1, Wb:Wb + n0l]),
                                                  L.stream()), "slab_adjoint_step")
        self.matvecs += 1
        self.pde_solves += 2
        b = torch.empty((3, *g.n), dtype=torch.float32, device="cuda")
        L.check(L.lib().frg_slab_body_force(self.n_loc, g.n_t, _c(lt[0, Wb:Wb + n0l]), (n0l + 2 * Wb) * plane,
                                            _c(self.grads), _c(b), L.stream()), "slab_body_force")
        out = torch.empty((3, *g.n), dtype=torch.float64, device="cuda") if out is None else out
        self._spectral_out(vt, b, out)
        return _Vec(g, out)

    def apply_precond(self, r, kind: PrecondKind | None = None, outer_tol: float = 0.0,
                      out: torch.Tensor | None = None) -> _Vec:
        """kkt.py:308-324: 'reg' (the spectral inverse of alpha L) and 'h0'
        (nested PCG on the zero-velocity Hessian surrogate, 'reg'
        preconditioned; breakdown falls back to 'reg' and counts)."""
        rd = (r.data if hasattr(r, "data") else r).to(self._spec_dt).contiguous()
        if kind is not None and kind.kind == "2level":
            res = self._two_level(rd, kind, outer_tol)
            if res is not None:
                if out is None:
                    return _Vec(self.grid, res)
                out.copy_(res)
                return _Vec(self.grid, out)
            self.precond_fallbacks += 1
        elif kind is not None and kind.kind == "h0":
            sol, broke = self._inner_pcg(self._apply_h0, rd, kind.inner_tol_factor * outer_tol,
                                         kind.inner_max_iterations)
            if not broke:
                if out is None:
                    return _Vec(self.grid, sol)
                out.copy_(sol)
                return _Vec(self.grid, out)
            self.precond_fallbacks += 1
        out = torch.empty_like(rd) if out is None else out
        self.fft.apply(rd, "reg_inv", self._reg, out=out)
        return _Vec(self.grid, out)

    # -- two-level preconditioner (kkt.py:291-306,325-341) -------------------
    # The coarse problem (n/2 per axis, 1/8 of the unknowns) is solved
    # redundantly on every rank: restrict = the slab forward spectrum's bins
    # |k_i| < n_i/4 (diffops.py:304-327), placed by their owners into a zeroed
    # full coarse half-spectrum and summed over ranks (one all-reduce); the
    # coarse PCG runs with single-GPU kernels and rank-local inner products
    # (identical on every rank); prolong = the coarse spectrum written back
    # into each rank's fine spectrum rows + a slab inverse (diffops.py:330-343).
    def _coarse_maps(self):
        if getattr(self, "_cmaps", None) is None:
            n0, n1, n2 = self.grid.n_glob

            def kept(n):  # diffops.py:304-310: fine bins kept, their coarse bins
                nc = n // 2
                f = list(range(0, nc // 2)) + list(range(n - nc // 2 + 1, n))
                c = list(range(0, nc // 2)) + list(range(nc - nc // 2 + 1, nc))
                return f, c

            f0, c0 = kept(n0)
            f1, c1 = kept(n1)
            lo, hi = self.fft.i1_off, self.fft.i1_off + self.fft.n1l
            mine = [(a, b) for a, b in zip(f1, c1) if lo <= a < hi]
            dev = lambda v: torch.tensor(v, dtype=torch.long, device="cuda")  # noqa: E731
            self._cmaps = {"f0": dev(f0), "c0": dev(c0), "f1": dev([a - lo for a, _ in mine]),
                           "c1": dev([b for _, b in mine]), "k2": n2 // 4, "nc": (n0 // 2, n1 // 2, n2 // 2)}
        return self._cmaps

    def _restrict(self, x: torch.Tensor) -> torch.Tensor:
        """(C, n0_loc, n1, n2) slab -> (C, n0/2, n1/2, n2/2) full coarse field on every rank."""
        cm = self._coarse_maps()
        nc0, nc1, nc2 = cm["nc"]
        C = x.shape[0]
        spec = self.fft.forward(x.to(torch.float64).contiguous())
        ch = torch.zeros((C, nc0, nc1, nc2 // 2 + 1), dtype=torch.complex128, device="cuda")
        if cm["f1"].numel():
            blk = spec.index_select(1, cm["f0"]).index_select(2, cm["f1"])[..., :cm["k2"]]
            tmp = torch.zeros((C, nc0, cm["f1"].numel(), cm["k2"]), dtype=torch.complex128, device="cuda")
            tmp.index_copy_(1, cm["c0"], blk)
            ch[:, :, :, :cm["k2"]].index_copy_(2, cm["c1"], tmp)
        if self.comm.size > 1:
            rv = torch.view_as_real(ch)
            if self.comm.staged:
                h = rv.cpu()
                tdist.all_reduce(h, group=self.comm.group)
                rv.copy_(h)
            else:
                tdist.all_reduce(rv, group=self.comm.group)
        nf, nc = float(np.prod(self.grid.n_glob)), float(nc0 * nc1 * nc2)
        return torch.fft.irfftn(ch * (nc / nf), s=(nc0, nc1, nc2), dim=(1, 2, 3))

    def _prolong(self, xc: torch.Tensor) -> torch.Tensor:
        """(C, n0/2, n1/2, n2/2) full coarse field -> (C, n0_loc, n1, n2) slab (zero padding)."""
        cm = self._coarse_maps()
        nc0, nc1, nc2 = cm["nc"]
        C = xc.shape[0]
        ch = torch.fft.rfftn(xc, dim=(1, 2, 3))
        spec = torch.zeros((C, self.grid.n_glob[0], self.fft.n1l, self.fft.nh), dtype=torch.complex128,
                           device="cuda")
        if cm["f1"].numel():
            blk = ch.index_select(1, cm["c0"]).index_select(2, cm["c1"])[..., :cm["k2"]] / float(nc0 * nc1 * nc2)
            tmp = torch.zeros((C, self.grid.n_glob[0], cm["f1"].numel(), cm["k2"]), dtype=torch.complex128,
                              device="cuda")
            tmp.index_copy_(1, cm["f0"], blk)
            spec[:, :, :, :cm["k2"]].index_copy_(2, cm["f1"], tmp)
        out = torch.empty((C, *self.grid.n), dtype=torch.float64, device="cuda")
        return self.fft.inverse(spec, out)

    def _coarse_ops(self):
        if getattr(self, "_coarse", None) is None or self._coarse[0] is not self.mseries[-1]:
            cm = self._coarse_maps()
            mc = self._restrict(self.mseries[-1].unsqueeze(0))[0].contiguous()
            gc = torch.empty((3, *cm["nc"]), dtype=torch.float64, device="cuda")
            L.check(L.lib().frg_fd8_gradient(L.n3(cm["nc"]), 3, L.F64, 1, _c(mc), _c(gc), L.stream()), "fd8_coarse")
            self._coarse = (self.mseries[-1], gc)
        return self._coarse[1]

    def _coarse_inv_sqrt(self, w: torch.Tensor) -> torch.Tensor:
        cm = self._coarse_maps()
        out = torch.empty_like(w)
        L.check(L.lib().frg_spectral_apply(L.n3(cm["nc"]), 3, L.F64, 3, _c(w), _c(out), L.SYM["reg_inv_sqrt"],
                                           ctypes.byref(self._reg), L.stream()), "coarse_inv_sqrt")
        return out

    def _two_level(self, r: torch.Tensor, kind: PrecondKind, outer_tol: float):
        """kkt.py:325-341; None on a coarse PCG breakdown (caller falls back)."""
        u = self.fft.apply(r, "reg_inv_sqrt", self._reg)
        u_low = self._restrict(u)  # restrict(low_pass(u)) == restrict(u): both keep |k_i| < n_i/4
        gc = self._coarse_ops()

        def op(w):  # kkt.py:297-306: w + R^-1/2 ((g_c . R^-1/2 w) g_c)
            sw = self._coarse_inv_sqrt(w)
            return w + self._coarse_inv_sqrt((gc * sw).sum(0) * gc)

        sol, broke = self._pcg_local(op, u_low, kind.inner_tol_factor * outer_tol, kind.inner_max_iterations)
        if broke:
            return None
        s = self._prolong(sol) + self.fft.apply(u, "highpass", self._reg)  # low_pass(prolong(.)) == prolong(.)
        return self.fft.apply(s, "reg_inv_sqrt", self._reg)

    @staticmethod
    def _pcg_local(apply_op, rhs: torch.Tensor, tol_rel: float, max_it: int):
        """kkt.py:99-133 with the identity preconditioner on a replicated
        coarse problem (rank-local inner products, identical on every rank)."""
        dot = lambda a, b: float((a * b).sum())  # noqa: E731
        x = torch.zeros_like(rhs)
        r = rhs.clone()
        rhs_norm = math.sqrt(max(dot(rhs, rhs), 0.0))
        if rhs_norm == 0.0:
            return x, False
        s = r.clone()
        rz = dot(r, r)
        it = 0
        while it < max_it:
            op_s = apply_op(s)
            s_op_s = dot(s, op_s)
            if not math.isfinite(s_op_s) or s_op_s <= 0.0:
                return x, True
            kappa = rz / s_op_s
            x.add_(s, alpha=kappa)
            r.add_(op_s, alpha=-kappa)
            it += 1
            if math.sqrt(max(dot(r, r), 0.0)) <= tol_rel * rhs_norm:
                break
            rz_new = dot(r, r)
            if not math.isfinite(rz_new) or rz_new <= 0.0:
                return x, True
            mu = rz_new / rz
            rz = rz_new
            s = r.clone().add_(s, alpha=mu)
        return x, False

    def _apply_h0(self, s64: torch.Tensor) -> torch.Tensor:
        """kkt.py:275-289: alpha L (zero symbol -> 1) s + (grad m(1) . s) grad m(1),
        grad = FD8 of the deformed image (the refresh's last gradient slice)."""
        if self._h0_grad is None:
            self._h0_grad = self.grads[self.grid.n_t].to(torch.float64)
        gm = self._h0_grad
        out = self.fft.apply(s64, "reg_kc", self._reg)
        out += (gm * s64).sum(0) * gm
        return out

    def _inner_pcg(self, apply_op, rhs: torch.Tensor, tol_rel: float, max_it: int):
        """kkt.py:99-133 with global (all-reduced) inner products; 'reg'
        preconditioned.  Returns (solution, breakdown)."""
        x = torch.zeros_like(rhs)
        r = rhs.clone()
        rhs_norm = math.sqrt(max(self.dot(rhs, rhs), 0.0))
        if rhs_norm == 0.0:
            return x, False
        z = self.fft.apply(r, "reg_inv", self._reg)
        s = z.clone()
        rz = self.dot(r, z)
        it = 0
        while it < max_it:
            op_s = apply_op(s)
            s_op_s = self.dot(s, op_s)
            if not math.isfinite(s_op_s) or s_op_s <= 0.0:
                return x, True
            kappa = rz / s_op_s
            x.add_(s, alpha=kappa)
            r.add_(op_s, alpha=-kappa)
            it += 1
            if math.sqrt(max(self.dot(r, r), 0.0)) <= tol_rel * rhs_norm:
                break
            z = self.fft.apply(r, "reg_inv", self._reg)
            rz_new = self.dot(r, z)
            if not math.isfinite(rz_new) or rz_new <= 0.0:
                return x, True
            mu = rz_new / rz
            rz = rz_new
            s = z.add_(s, alpha=mu)
        return x, False

    def _reg_energy(self, v64: torch.Tensor) -> float:
        lv = self.fft.apply(v64.to(self._spec_dt), "reg", self._reg).to(torch.float64)
        return 0.5 * self.dot(v64, lv) * self.grid.cell_volume

    def objective(self) -> float:
        if self._dist is None:
            self._dist = self._dist_value(self.mseries[-1])
        return self._dist + self._reg_energy(self.v.data)

    def objective_at(self, v_trial) -> float:
        vt = (v_trial.data if hasattr(v_trial, "data") else v_trial).to(torch.float64)
        disp, _, _ = self._departure(vt.float(), 1.0)
        plan = self._plan(disp)
        L.check(L.lib().frg_bind_plan(0, _c(disp), _c(plan), self._m), "bind_plan")
        m = self._state_solve(disp, self._halo_of(disp), keep=False)
        self._bind()
        self.pde_solves += 1
        return self._dist_value(m) + self._reg_energy(vt)

    def mismatch(self) -> float:
        if self._init_mismatch == 0.0:
            return 0.0
        if self._dist is None:
            self._dist = self._dist_value(self.mseries[-1])
        return self._dist / self._init_mismatch

    def divergence_energy(self) -> float:
        """kkt.py:207-218: 0.5 beta (<div v, div v> + <grad div v, grad div v>)
        (spectral gradient) in the near-incompressible mode, else 0 — the
        gradient energy from this rank's share of the slab spectrum
        (frg_slab_grad_energy), all-reduced."""
        if self.reg.incomp.mode != "near-incompressible":
            return 0.0
        cv = self.grid.cell_volume
        w = self.divv
        ww = self.dot(w, w) * cv
        spec = self.fft.forward(w.to(torch.float64).unsqueeze(0).contiguous())
        out = ctypes.c_double()
        L.check(L.lib().frg_slab_grad_energy(self.fft.nglob, self.fft.i1_off, self.fft.n1l, _c(spec),
                                             ctypes.byref(out), L.stream()), "slab_grad_energy")
        gg = self.comm.all_reduce(out.value) * cv
        return 0.5 * self.reg.incomp.beta * (ww + gg)

    def detgrad_stats(self):
        """(min, mean, max) of det F(1) over the whole grid (kkt.py
        detgrad, transport.py:197-221 on the slab): jac = FD8 grad v, its
        gather at the feet, n_t Heun steps of d_t F = (grad v) F (9-field
        slab gathers of F + the pointwise update), det, all-reduced."""
        g = self.grid
        n0l = g.n0_loc
        W = max(self.Wf, 4)
        v32 = self.v.data.float()
        jac = torch.empty((3, 3, *g.n), dtype=torch.float32, device="cuda")
        L.check(L.lib().frg_slab_fd8_gradient(self.n_loc, g.n_glob[0], W, 3, _c(self._ext(v32, W)), _c(jac),
                                              L.stream()), "slab_fd8_gradient")
        jac9 = jac.view(9, *g.n)
        jac_y = torch.empty_like(jac9)
        ext = self._src(jac9, self.Wf)
        self._bind()
        self._gather(self.disp_f, self.Wf, [ext[e] for e in range(9)], [jac_y[e] for e in range(9)])
        F = torch.empty_like(jac9)
        L.check(L.lib().frg_deform_update(self.n_loc, L.F32, g.h_t, 1, _c(jac_y), _c(jac9), _c(F), L.stream()),
                "deform_update")
        for _ in range(1, g.n_t):
            ext = self._src(F, self.Wf)
            self._gather(self.disp_f, self.Wf, [ext[e] for e in range(9)], [F[e] for e in range(9)])
            L.check(L.lib().frg_deform_update(self.n_loc, L.F32, g.h_t, 0, _c(jac_y), _c(jac9), _c(F), L.stream()),
                    "deform_update")
        det = torch.empty(g.n, dtype=torch.float32, device="cuda")
        L.check(L.lib().frg_determinant(self.n_loc, 3, L.F32, _c(F), _c(det), L.stream()), "determinant")
        mms = (ctypes.c_double * 3)()
        L.check(L.lib().frg_min_max_sum(L.F32, _c(det), det.numel(), mms, L.stream()), "min_max_sum")
        dmin = self.comm.all_reduce(float(mms[0]), "min")
        dmax = self.comm.all_reduce(float(mms[1]), "max")
        dsum = self.comm.all_reduce(float(mms[2]))
        return dmin, dsum / float(np.prod(g.n_glob)), dmax


def dist_register(m0: torch.Tensor, m1: torch.Tensor, comm: SlabComm, n_glob, config=None, reg: RegConfig | None = None,
                  n_t: int = 4, method: str = "cubic", v0: torch.Tensor | None = None, compute_detgrad: bool = True,
                  distance: str = "ssd", precond: PrecondKind | None = None):
    """optimizer.register (optimizer.py:174-281) on the slab decomposition:
    the same host control, SPMD on every rank, reductions all-reduced
    (SSD / NCC; 'reg' or 'h0' preconditioner)."""
    from .optimizer import OptimizerConfig, solve

    reg = reg or RegConfig()
    state = DistKktState(m0, m1, reg, comm, n_glob, n_t=n_t, method=method, v_init=v0, distance=distance)
    return solve(state, config or OptimizerConfig(), precond or PrecondKind("reg"), compute_detgrad=compute_detgrad)


def dist_search_alpha(m0: torch.Tensor, m1: torch.Tensor, comm: SlabComm, n_glob, cfg=None,
                      reg: RegConfig | None = None, opt=None, n_t: int = 4, method: str = "cubic",
                      distance: str = "ssd", precond: PrecondKind | None = None):
    """continuation.search_alpha (continuation.py:87-207) on the slab
    decomposition: the same sweep / bisection (continuation.run_search), every
    trial a SPMD dist_register warm-started from the previous trial unless the
    warm objective exceeds the cold one; det F(1) bounds from the slab
    deformation solve (DistKktState.detgrad_stats).  Returns a SearchResult
    whose velocities are this rank's slabs."""
    from dataclasses import replace

    from .continuation import SearchConfig, TrialRecord, run_search
    from .optimizer import OptimizerConfig

    cfg = cfg or SearchConfig()
    reg = reg or RegConfig()
    opt = opt or OptimizerConfig()

    def trial(alpha, v_warm, phase):
        reg_a = replace(reg, alpha=alpha)
        v0, warm_started, dropped = (None if v_warm is None else v_warm.data), v_warm is not None, False
        if v_warm is not None:  # continuation.py:98-108: drop a warm start worse than v = 0
            st = DistKktState(m0, m1, reg_a, comm, n_glob, n_t=n_t, method=method, v_init=v0, distance=distance)
            if st.objective() > st._init_mismatch:
                v0, warm_started, dropped = None, False, True
            del st
        v, rep = dist_register(m0, m1, comm, n_glob, config=opt, reg=reg_a, n_t=n_t, method=method, v0=v0,
                               distance=distance, precond=precond)
        ok = rep.detgrad_min > cfg.eps_det and rep.detgrad_max < 1.0 / cfg.eps_det
        rec = TrialRecord(alpha=alpha, passed=ok, det_min=rep.detgrad_min, det_max=rep.detgrad_max,
                          det_mean=rep.detgrad_mean, mismatch=rep.mismatch, iterations=rep.iterations,
                          warm_started=warm_started, warm_start_dropped=dropped, phase=phase)
        return v, rec

    def is_zero(v):
        out = ctypes.c_double()
        L.check(L.lib().frg_norm_inf(L.F64, L.ptr(v.data), v.data.numel(), ctypes.byref(out), L.stream()),
                "norm_inf")
        return comm.all_reduce(out.value, "max") == 0.0

    return run_search(cfg, trial, is_zero)


def dist_continuation_solve(m0: torch.Tensor, m1: torch.Tensor, comm: SlabComm, n_glob, alpha_target: float,
                            reg: RegConfig | None = None, opt=None, n_t: int = 4, method: str = "cubic",
                            distance: str = "ssd", precond: PrecondKind | None = None):
    """continuation.continuation_solve (continuation.py:239-293) on the slab
    decomposition — config C5's alpha cascade 1, 0.1, ..., alpha_target with
    warm starts, every stage a SPMD dist_register.  Returns (velocity slab,
    aggregate report, per-stage reports); det F(1) statistics of the last
    stage as in continuation_solve."""
    from dataclasses import replace

    from .continuation import cascade_alphas
    from .optimizer import OptimizerConfig, SolveReport

    reg = reg or RegConfig()
    opt = opt or OptimizerConfig()
    v, stages, total = None, [], SolveReport()
    alphas = cascade_alphas(alpha_target)
    for a in alphas:
        vv, rep = dist_register(m0, m1, comm, n_glob, config=opt, reg=replace(reg, alpha=a), n_t=n_t, method=method,
                                v0=None if v is None else v.data, compute_detgrad=(a == alphas[-1]),
                                distance=distance, precond=precond)
        v = vv
        stages.append(rep)
        total.iterations += rep.iterations
        total.matvecs += rep.matvecs
        total.pde_solves += rep.pde_solves
        total.line_search_evals += rep.line_search_evals
        total.precond_fallbacks += rep.precond_fallbacks
        total.runtime += rep.runtime
    last = stages[-1]
    total.mismatch, total.gradient = last.mismatch, last.gradient
    total.status, total.exit_reason = last.status, last.exit_reason
    total.detgrad_min, total.detgrad_mean, total.detgrad_max = last.detgrad_min, last.detgrad_mean, last.detgrad_max
    total.trace = [row for rep in stages for row in rep.trace]
    return v, total, stages



class _SlabTransport(DistKktState):
    """The slab transport machinery of DistKktState (departure maps, tile
    plans, ghost-plane gathers) without images or KKT state."""

    def __init__(self, comm: SlabComm, n_glob, n_t: int, method: str = "cubic"):
        self.comm = comm
        self.grid = SlabGrid(tuple(int(v) for v in n_glob), comm.rank, comm.size, n_t=n_t)
        self.method, self._m, self._bs = method, L.METHODS[method], method == "bspline"
        self.reg = RegConfig()
        self._reg = frg_reg(self.reg.operator, self.reg.alpha, self.reg.incomp)
        self.fft = SlabFFT(self.grid, comm)
        self.n_loc = L.n3(self.grid.n)
        self.N = int(np.prod(self.grid.n))
        self.peer = os.environ.get("FRG_SLAB_PEER") == "1"
        self._win = PeerWindows.get(comm, (9, *self.grid.n)) if self.peer else None


def slab_synth(name: str, n: int, comm: SlabComm, seed: int = 1, amp: float = 0.7, ref_steps: int = 64):
    """synth.synth_case for configs C4 / C5 generated slab by slab: this rank's
    planes of the bump template (synth.py:28-43, global min / max
    normalisation all-reduced) and of the rotation velocity (synth.py:46-63),
    and the reference image from a ``ref_steps``-step cubic SL transport run
    by the slab path itself (synth.py:113-117) — no rank ever holds the whole
    grid, so 1024^3 over 8 GPUs fits.  Transport in fp32 (the slab path's
    precision; the single-GPU generator is f64).  Returns (m0, m1) fp32 and v
    f64, each (.., n/P, n, n)."""
    if name != "rotation":
        raise ValueError("slab_synth implements the rotation case")
    lo, hi = slab_bounds(n, comm.size, comm.rank)
    rng = np.random.default_rng(seed)
    hh = TWO_PI / n
    ax = ((n // 2) - (torch.arange(n, dtype=torch.float64, device="cuda") + 1.0)) * hh
    x0 = ax[lo:hi].view(-1, 1, 1)
    x1 = ax.view(1, -1, 1)
    x2 = ax.view(1, 1, -1)
    vals = torch.zeros((hi - lo, n, n), dtype=torch.float64, device="cuda")
    for _ in range(6):
        c = rng.uniform(-np.pi, np.pi, size=3)
        kappa = rng.uniform(1.0, 2.5)
        a = rng.uniform(0.4, 1.0)
        vals += a * (torch.exp(kappa * (torch.cos(x0 - c[0]) - 1.0)) * torch.exp(kappa * (torch.cos(x1 - c[1]) - 1.0))
                     * torch.exp(kappa * (torch.cos(x2 - c[2]) - 1.0)))
    vmin = -comm.all_reduce(-float(vals.min()), "max")
    vals -= vmin
    vmax = comm.all_reduce(float(vals.max()), "max")
    if vmax > 0:
        vals /= vmax
    mod = 1.0 + 0.3 * torch.cos(x2)
    v = torch.zeros((3, hi - lo, n, n), dtype=torch.float64, device="cuda")
    v[0] = -amp * torch.cos(x0) * torch.sin(x1) * mod
    v[1] = amp * torch.sin(x0) * torch.cos(x1) * mod
    m0 = vals.float().contiguous()
    tr = _SlabTransport(comm, (n, n, n), ref_steps, "cubic")
    disp, _, _ = tr._departure(v.float(), 1.0)
    plan = tr._plan(disp)
    L.check(L.lib().frg_bind_plan(0, _c(disp), _c(plan), tr._m), "bind_plan")
    m1 = tr._state_solve(disp, tr._halo_of(disp), keep=False, m0=m0)
    L.check(L.lib().frg_clear_plans(), "clear_plans")
    return m0, m1.contiguous(), v
