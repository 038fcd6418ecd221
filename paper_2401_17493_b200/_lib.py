"""ctypes binding of libflowreg_b200.so (include/flowreg_b200.h).

The product path has NO CPU fallback: importing an operator without the
built library, or calling one without a CUDA device, raises immediately.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FRG_LIB", os.path.join(HERE, "libflowreg_b200.so"))

F32, F64, I32 = 0, 1, 2
METHODS = {"nearest": 0, "linear": 1, "cubic": 2, "bspline": 3}
SCHEMES = {"fd8": 0, "spectral": 1}
DISTANCES = {"ssd": 0, "ncc": 1}
INCOMP = {"none": 0, "incompressible": 1, "near-incompressible": 2}
SYM = {"reg": 0, "reg_inv": 1, "reg_inv_sqrt": 2, "reg_kc": 3, "laplacian": 4, "lowpass": 5, "highpass": 6,
       "bspline_prefilter": 7}
PRECOND = {"reg": 0, "h0": 1, "2level": 2}

STATUS = {0: "ok", -1: "invalid argument", -2: "non-finite data", -3: "CUDA error", -4: "cuFFT error",
          -5: "invalid state"}


class FrgReg(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("order", ctypes.c_int32), ("seminorm", ctypes.c_int32),
                ("incomp", ctypes.c_int32), ("beta", ctypes.c_double)]


class FrgConfig(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32 * 3), ("d", ctypes.c_int32), ("n_t", ctypes.c_int32),
                ("method", ctypes.c_int32), ("scheme", ctypes.c_int32), ("distance", ctypes.c_int32),
                ("transport_dtype", ctypes.c_int32), ("control_dtype", ctypes.c_int32), ("reg", FrgReg)]


class FlowregError(RuntimeError):
    """A libflowreg_b200 call failed (CUDA / cuFFT / state error)."""


_P = ctypes.c_void_p
_I = ctypes.c_int32
_L = ctypes.c_int64
_D = ctypes.c_double
_N3 = ctypes.POINTER(ctypes.c_int32)
_DP = ctypes.POINTER(ctypes.c_double)

# name -> argtypes (all return int status)
PROTOTYPES = {
    "frg_sample": [_P, _I, _N3, _P, _P, _P, _L, _I, _P, _P],
    "frg_departure": [_N3, _I, _I, _I, _I, _D, _P, _P, _P],
    "frg_disp_to_points": [_N3, _I, _I, _P, _P, _P],
    "frg_points_to_disp": [_N3, _I, _I, _P, _P, _P],
    "frg_gather": [_N3, _I, _I, _I, _P, _I, ctypes.POINTER(_P), ctypes.POINTER(_P), _P],
    "frg_tile_plan": [_N3, _I, _I, _P, _P, _P],
    "frg_gather_planned": [_N3, _I, _I, _P, _P, _I, ctypes.POINTER(_P), ctypes.POINTER(_P), _P],
    "frg_solve_state": [_N3, _I, _I, _I, _I, _P, _P, _P],
    "frg_solve_adjoint": [_N3, _I, _I, _I, _I, _P, _P, _P, _P],
    "frg_solve_inc_state": [_N3, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "frg_body_force": [_N3, _I, _I, _I, _P, _P, _P, _P],
    "frg_deformation_tensor": [_N3, _I, _I, _I, _I, _P, _P, _P, _P],
    "frg_determinant": [_N3, _I, _I, _P, _P, _P],
    "frg_deform_update": [_N3, _I, ctypes.c_double, _I, _P, _P, _P, _P],
    "frg_compose": [_N3, _I, _I, _I, _I, _P, _P, _P],
    "frg_fd8_gradient": [_N3, _I, _I, _I, _P, _P, _P],
    "frg_fd8_divergence": [_N3, _I, _I, _P, _P, _P],
    "frg_spectral_gradient": [_N3, _I, _I, _P, _P, _P],
    "frg_spectral_divergence": [_N3, _I, _I, _P, _P, _P],
    "frg_spectral_apply": [_N3, _I, _I, _I, _P, _P, _I, ctypes.POINTER(FrgReg), _P],
    "frg_project": [_N3, _I, _I, _P, _P, ctypes.POINTER(FrgReg), _P],
    "frg_restrict": [_N3, _I, _P, _P, _P],
    "frg_prolong": [_N3, _I, _P, _P, _P],
    "frg_dot": [_I, _P, _P, _L, _DP, _P],
    "frg_release_pool": [],
    "frg_probe_arm": [_I],
    "frg_probe_read": [_DP, ctypes.POINTER(_L)],
    "frg_peer_alloc": [_L, ctypes.POINTER(_P), _P],
    "frg_peer_free": [_P],
    "frg_peer_open": [_P, ctypes.POINTER(_P)],
    "frg_peer_close": [_P],
    "frg_peer_register": [_P, _N3, _I, _I, ctypes.POINTER(_P)],
    "frg_peer_unregister": [_P],
    "frg_norm_inf": [_I, _P, _L, _DP, _P],
    "frg_min_max_sum": [_I, _P, _L, _DP, _P],
    "frg_all_finite": [_I, _P, _L, ctypes.POINTER(ctypes.c_int32), _P],
    "frg_axpby": [_I, _D, _P, _D, _P, _L, _P],
    "frg_pcg_update": [_I, _D, _P, _P, _P, _P, _L, _DP, _P],
    "frg_kkt_create": [ctypes.POINTER(FrgConfig), _P, ctypes.POINTER(_P)],
    "frg_kkt_destroy": [_P],
    "frg_kkt_set_stream": [_P, _P],
    "frg_kkt_set_images": [_P, _P, _P, _I],
    "frg_kkt_set_interp_precision": [_P, _I],
    "frg_kkt_refresh": [_P, _P],
    "frg_kkt_objective": [_P, _DP],
    "frg_kkt_objective_at": [_P, _P, _DP],
    "frg_kkt_gradient": [_P, _P],
    "frg_kkt_hessian_matvec": [_P, _P, _P],
    "frg_kkt_apply_precond": [_P, _I, _D, _D, _I, _P, _P, ctypes.POINTER(ctypes.c_int32)],
    "frg_kkt_mismatch": [_P, _DP],
    "frg_kkt_initial_mismatch": [_P, _DP],
    "frg_kkt_divergence_energy": [_P, _DP],
    "frg_kkt_counters": [_P, ctypes.POINTER(_L)],
    "frg_kkt_set_counters": [_P, ctypes.POINTER(_L)],
    "frg_kkt_get": [_P, _I, _P],
    "frg_kkt_detgrad": [_P, _DP],
    "frg_bind_plan": [_I, _P, _P, _I],
    "frg_clear_plans": [],
    "frg_slab_body_force": [_N3, _I, _P, _L, _P, _P, _P],
    # slab decomposition (multi-GPU, dist.py)
    "frg_slab_departure": [_N3, _I, _I, _I, _D, _P, _P, _P, _P],
    "frg_slab_gather": [_N3, _I, _I, _I, _P, _I, ctypes.POINTER(_P), ctypes.POINTER(_P), _P],
    "frg_slab_adjoint_multiplier": [_N3, _I, _I, _I, _D, _P, _P, _P, _P, _P],
    "frg_slab_adjoint_step": [_N3, _I, _I, _I, _P, _P, _P, _P, _P],
    "frg_slab_inc_first": [_N3, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "frg_slab_inc_step": [_N3, _I, _I, _I, _P, _P, _P, _P, _P, ctypes.c_double, _P],
    "frg_slab_spec_combine_mixed": [_N3, _I, _I, _P, _P, ctypes.POINTER(FrgReg), _I, _P],
    "frg_slab_grad_energy": [_N3, _I, _I, _P, _DP, _P],
    "frg_convert": [_I, _P, _I, _P, _L, _P],
    "frg_slab_fd8_gradient": [_N3, _I, _I, _I, _P, _P, _P],
    "frg_slab_fd8_divergence": [_N3, _I, _I, _P, _P, _P],
    "frg_slab_fft2": [_N3, _I, _I, _I, _P, _P, _P],
    "frg_slab_fft1": [_I, _I, _I, _I, _I, _I, _P, _P],
    "frg_slab_transpose": [_I, _I, _N3, _I, _I, _P, _P, _P],
    "frg_slab_spec_apply": [_N3, _I, _I, _I, _I, _P, _I, ctypes.POINTER(FrgReg), _P],
    "frg_slab_spec_combine": [_N3, _I, _I, _I, _P, _P, ctypes.POINTER(FrgReg), _I, _P],
}

_lib = None


def load(path: str = LIB_PATH):
    """Load the C-ABI library (no GPU needed to load it)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(
                f"libflowreg_b200.so not found at {path}; build it with "
                "`python -m paper_2401_17493_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, args in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        lib.frg_last_error.restype = ctypes.c_char_p
        lib.frg_last_error.argtypes = []
        lib.frg_tile_plan_count.restype = ctypes.c_int64
        lib.frg_tile_plan_count.argtypes = [_N3]
        lib.frg_version.restype = ctypes.c_char_p
        lib.frg_version.argtypes = []
        _lib = lib
    return _lib


def lib():
    return load()


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = lib().frg_last_error().decode(errors="replace")
        if rc == -1:
            if msg.startswith("ZeroNormError"):
                from .distance import ZeroNormError

                raise ZeroNormError(msg)
            raise ValueError(msg)
        raise FlowregError(f"{what}: {STATUS.get(rc, rc)}: {msg}")


def require_cuda():
    if not torch.cuda.is_available():
        raise FlowregError("libflowreg_b200 needs a CUDA device (B200); there is no CPU fallback")


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def dtype_code(dt) -> int:
    if dt in (torch.float64, np.float64) or dt == np.dtype(np.float64):
        return F64
    if dt in (torch.float32, np.float32) or dt == np.dtype(np.float32):
        return F32
    if dt in (torch.int32, np.int32) or dt == np.dtype(np.int32):
        return I32
    raise ValueError(f"unsupported dtype {dt}")


def n3(shape) -> ctypes.Array:
    """Grid shape -> C int32[3] with the 2D embedding (1, n0, n1)."""
    shape = tuple(int(s) for s in shape)
    if len(shape) == 2:
        shape = (1,) + shape
    return (ctypes.c_int32 * 3)(*shape)


def ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())
