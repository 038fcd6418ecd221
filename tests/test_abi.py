"""CPU checks of the C-ABI boundary: the library builds, loads, and exports
every entry point declared in include/flowreg_b200.h (no compute calls)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "flowreg_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(frg_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2401_17493_b200 import build

    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_core_entry_points():
    syms = declared_symbols()
    for core in ("frg_sample", "frg_kkt_create", "frg_kkt_refresh", "frg_kkt_hessian_matvec",
                 "frg_kkt_gradient", "frg_kkt_apply_precond", "frg_dot"):
        assert core in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_prototypes_cover_header():
    from paper_2401_17493_b200 import _lib as L

    syms = set(declared_symbols()) - {"frg_last_error", "frg_version"}
    assert syms == set(L.PROTOTYPES), syms ^ set(L.PROTOTYPES)


def test_version_and_error_strings(lib):
    lib.frg_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.frg_version()
    lib.frg_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.frg_last_error(), bytes)


def test_invalid_arguments_rejected_without_gpu(lib):
    # argument validation happens before any device work
    n = (ctypes.c_int32 * 3)(1, 16, 16)
    rc = lib.frg_sample(None, 0, n, None, None, None, ctypes.c_int64(4), 7, None, None)
    assert rc == -1
    lib.frg_last_error.restype = ctypes.c_char_p
    assert b"method" in lib.frg_last_error()


def test_sass_is_sm100a(lib):
    """The shipped cubin targets sm_100a (cuobjdump lists the arch)."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", lib._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out
