"""Seeded synthetic CSR inputs shared by the oracle and the CUDA path.

Test/bench input infrastructure only: no BinSketch arithmetic lives here
(see synth.cpp for the recipe). Both ``oracle/`` and
``paper_1910_04658_b200`` consume the arrays this module returns; neither
imports the other.

The workload presets mirror BASELINE.json ``configs``; the
paper's UCI corpora are not available and these synthetic
Zipf-feature corpora stand in for them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
                               "-ffp-contract=off", src, "-o", _SO])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.synth_row_nnz.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p]
        lib.synth_row_nnz.restype = None
        lib.synth_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_int64, ctypes.c_double, ctypes.c_int,
                                   ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_fill.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclass(frozen=True)
class CSRSpec:
    """One synthetic corpus: n rows over d features."""
    n: int
    d: int
    kind: int          # 0: nnz uniform on {p1..p2}; 1: lognormal(mean=p1, sigma=p2), capped at cap
    p1: float
    p2: float
    cap: int
    zipf_s: float
    seed: int
    perm: int = 1      # 1: seeded rank->id permutation (default); 0: identity


def make_csr(spec: CSRSpec):
    """Return (indptr int64[n+1], indices int32[nnz]) as numpy arrays."""
    lib = _load()
    counts = np.empty(spec.n, dtype=np.int64)
    lib.synth_row_nnz(spec.n, spec.d, spec.kind, spec.p1, spec.p2, spec.cap, spec.seed,
                      counts.ctypes.data)
    indptr = np.zeros(spec.n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    indices = np.empty(int(indptr[-1]), dtype=np.int32)
    bad = lib.synth_fill(spec.n, spec.d, spec.kind, spec.p1, spec.p2, spec.cap, spec.zipf_s,
                         spec.perm, spec.seed, indptr.ctypes.data, indices.ctypes.data)
    if bad:
        raise RuntimeError("synth_fill: inconsistent indptr")
    return indptr, indices


# --- BASELINE.json configs (seeds as proposed there) ---
PI_SEED = 1
SIGMA = 1.0

TINY = CSRSpec(n=1000, d=5000, kind=0, p1=20, p2=100, cap=100, zipf_s=1.1, seed=1)
TINY_N = 1224                      # Theorem 1 with psi=100, rho=0.1

MEDIUM = CSRSpec(n=10_000, d=28_102, kind=1, p1=160, p2=SIGMA, cap=1000, zipf_s=1.1, seed=2)
MEDIUM_NS = (1000, 2000, 5000)

RANKING_DB = CSRSpec(n=100_000, d=102_660, kind=1, p1=230, p2=SIGMA, cap=900, zipf_s=1.05, seed=3)
RANKING_Q = CSRSpec(n=1000, d=102_660, kind=1, p1=230, p2=SIGMA, cap=900, zipf_s=1.05, seed=4)
RANKING_N = 4096
RANKING_K = 100

BUILD_ONLY = CSRSpec(n=10_000_000, d=1 << 20, kind=1, p1=64, p2=SIGMA, cap=2048, zipf_s=1.1, seed=5)
BUILD_ONLY_N = 1024

LARGE = CSRSpec(n=200_000, d=500_000, kind=1, p1=100, p2=SIGMA, cap=2048, zipf_s=1.1, seed=6)
LARGE_N = 1024
LARGE_K = 50


def scaled(spec: CSRSpec, n: int, seed: int | None = None) -> CSRSpec:
    """Same distribution, fewer rows (parity cases the oracle finishes quickly)."""
    return CSRSpec(n=n, d=spec.d, kind=spec.kind, p1=spec.p1, p2=spec.p2, cap=spec.cap,
                   zipf_s=spec.zipf_s, seed=spec.seed if seed is None else seed, perm=spec.perm)
