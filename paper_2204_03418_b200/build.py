"""Native build of libco_b200.so (in-tree, sm_100a only).

Each ``csrc/*.cu`` is compiled by nvcc for ``-gencode arch=compute_100a,code=sm_100a``
(with ``-lineinfo`` so ncu's source page maps to our code) into ``build/``, in
parallel, and linked into ``paper_2204_03418_b200/libco_b200.so`` with the CUDA
runtime linked statically (the library then loads on a CPU-only box for the
ABI symbol checks; CUDA is only touched on the first device call).

Usage: ``python -m paper_2204_03418_b200.build [--force] [-v]``
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "co_b200")
LIB = os.path.join(PKG, "libco_b200.so")
HEADERS = [os.path.join(ROOT, "include", "co.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
                     "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + HEADERS


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def _compile(src: str, force: bool, verbose: bool, bdir: str = BUILD, extra=()) -> str:
    obj = os.path.join(bdir, os.path.basename(src) + ".o")
    if force or _newer([src] + _deps(), obj):
        cmd = [nvcc()] + NVCC_FLAGS + list(extra) + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(bdir, os.path.basename(src) + ".log")
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
        if verbose:
            sys.stdout.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build libco_b200.so; `variant` + `defines` build an experiment copy
    libco_b200_<variant>.so (loaded when CO_LIB_VARIANT=<variant>)."""
    bdir = BUILD + (f"_{variant}" if variant else "")
    lib = LIB if not variant else LIB.replace(".so", f"_{variant}.so")
    extra = [f"-D{d}" for d in defines]
    os.makedirs(bdir, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose, bdir, extra), srcs))
    if force or _newer(objs, lib):
        tmp = lib + f".{os.getpid()}.tmp"
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + ["-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("--define", action="append", default=[])
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.variant, a.define))
