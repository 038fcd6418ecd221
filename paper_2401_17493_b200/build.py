"""Build libflowreg_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2401_17493_b200.build [--force] [--verbose]

The shared library is the product's C-ABI (include/flowreg_b200.h); it is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libflowreg_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + [
        os.path.join(ROOT, "include", "flowreg_b200.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, extra=(), out: str | None = None) -> str:
    """Compile every csrc/*.cu and link libflowreg_b200.so (``out`` + ``extra``
    flags build an experimental variant elsewhere)."""
    lib = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    # variants compile into their own object directory (never the default's)
    objdir = (os.path.join(os.path.dirname(lib), "_build_" + os.path.basename(lib).replace(".so", "")) if out
              else os.path.join(HERE, "_build"))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
              "-I", os.path.join(ROOT, "include"), *extra]
    headers = [p for p in deps() if not p.endswith(".cu")]
    newest_header = max(os.path.getmtime(p) for p in headers)
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        # incremental: an object is reused when it is newer than its source and
        # every header (and the build flags did not change: variants use --force)
        if (not force and out is None and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(src), newest_header)):
            continue
        cmd = common + ["-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = False
    for cmd, p in procs:
        log, _ = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(" ".join(cmd) + "\n" + log + "\n")
        elif verbose and log:
            sys.stderr.write(log)
    if failed:
        raise RuntimeError("nvcc failed building libflowreg_b200")
    tmp = lib + ".tmp"
    link = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcufft", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    subprocess.check_call(link)
    os.replace(tmp, lib)
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None, help="variant output path")
    ap.add_argument("-D", action="append", default=[], help="extra -D defines for a variant")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, extra=[f"-D{d}" for d in a.D], out=a.out))


if __name__ == "__main__":
    main()
