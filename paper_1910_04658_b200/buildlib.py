"""Build libbinsketch.so (the C-ABI library) in-tree for sm_100a with nvcc.

    python -m paper_1910_04658_b200.buildlib [--force] [--verbose]

Every translation unit is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17
pairs.cu (the fp64 estimator epilogue) additionally with -fmad=false, so no
FMA contraction can alter the canonical recipe's rounding (DESIGN.md R-C3).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libbinsketch.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
                 "-I", os.path.join(ROOT, "include"), "-I", CSRC]
UNITS = {
    "api.cu": [],
    "build.cu": [],
    "pairs.cu": ["-fmad=false"],
    "tc.cu": ["-fmad=false"],
    "join.cu": ["-fmad=false"],
}
HEADERS = ["bsk_internal.cuh", "bsk_device.cuh", "bsk_estimator.cuh"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "binsketch.h")]
    objs = []
    for unit, extra in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(OBJ, unit.replace(".cu", ".o"))
        objs.append(obj)
        defines = os.environ.get("BSK_NVCC_DEFINES", "").split()   # dev-only instrumentation builds
        if force or defines or _stale(obj, [src, __file__] + hdrs):
            cmd = [NVCC, "-c", src, "-o", obj] + COMMON + extra + defines
            if verbose:
                cmd += ["-Xptxas", "-v"]
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
    if force or os.environ.get("BSK_NVCC_DEFINES") or _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-o", LIB] + objs + ARCH
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
