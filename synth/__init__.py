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


# --- Experiment 2 inputs: near-duplicate structure + 90/10 split ---
def plant_near_duplicates(indptr, indices, d: int, frac: float, seed: int, keep_lo: float = 0.5):
    """Replace a seeded fraction of rows by perturbed copies of earlier rows.

    Real corpora have near-duplicate documents; i.i.d. Zipf rows do not, so a
    threshold join at the paper's high thresholds (0.95 ... 0.5) would be empty.
    Row i (chosen with probability ``frac``, i >= 1) becomes a copy of a random
    earlier row in which each feature is kept with probability ``keep`` ~
    U[keep_lo, 1] and otherwise replaced by a uniform feature in [0, d); the
    result is deduplicated and sorted. Input preparation only (no method
    arithmetic). Returns new (indptr, indices).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    n = len(indptr) - 1
    rows = [indices[indptr[i]:indptr[i + 1]] for i in range(n)]
    pick = rng.random(n) < frac
    src = (rng.random(n) * np.arange(n)).astype(np.int64)
    keep = keep_lo + (1.0 - keep_lo) * rng.random(n)
    for i in range(1, n):
        if not pick[i]:
            continue
        s = rows[src[i]]
        k = rng.random(len(s)) < keep[i]
        fresh = rng.integers(0, d, size=int((~k).sum()), dtype=np.int64).astype(np.int32)
        r = np.unique(np.concatenate([s[k], fresh]))
        rows[i] = r if len(r) else s[:1].copy()
    counts = np.array([len(r) for r in rows], dtype=np.int64)
    out_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=out_ptr[1:])
    out_idx = np.concatenate(rows).astype(np.int32) if n else np.zeros(0, dtype=np.int32)
    return out_ptr, out_idx


def split_rows(n: int, frac_query: float, seed: int):
    """Seeded random partition of row ids into (training, querying) parts, each sorted
    ("randomly, partition the dataset into two parts -- 90% and 10%")."""
    rng = np.random.Generator(np.random.PCG64(seed))
    p = rng.permutation(n)
    nq = int(round(n * frac_query))
    return np.sort(p[nq:]), np.sort(p[:nq])


def take_rows(indptr, indices, rows):
    """CSR of the selected rows, in the given order."""
    rows = np.asarray(rows, dtype=np.int64)
    counts = indptr[rows + 1] - indptr[rows]
    out_ptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(counts, out=out_ptr[1:])
    out_idx = np.empty(int(out_ptr[-1]), dtype=np.int32)
    for t, r in enumerate(rows):
        out_idx[out_ptr[t]:out_ptr[t + 1]] = indices[indptr[r]:indptr[r + 1]]
    return out_ptr, out_idx


# Exp. 2 workload: the Ranking corpus distribution (NYTimes-like d), 101,000 rows with
# 30% planted near-duplicates, split 90/10 into training (db) and querying parts.
EXP2 = CSRSpec(n=101_000, d=102_660, kind=1, p1=230, p2=SIGMA, cap=900, zipf_s=1.05, seed=7)
EXP2_N = 4096
EXP2_DUP_FRAC = 0.3
EXP2_DUP_SEED = 8
EXP2_SPLIT_SEED = 9
EXP2_THRESHOLDS = (0.95, 0.9, 0.85, 0.8, 0.6, 0.5, 0.2, 0.1)


# --- categorical inputs: label-encoded table [n][c] ---
def make_categorical(n: int, cards, seed: int, dup_frac: float = 0.3, flip: float = 0.2):
    """Seeded label-encoded table: column k uniform over [0, cards[k]) (Zipf-free), with a
    fraction of rows copied from an earlier row with each column re-drawn w.p. ``flip``
    (so small categorical distances occur). Input preparation only."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cards = np.asarray(cards, dtype=np.int64)
    n = int(n)
    X = (rng.random((n, len(cards))) * cards[None, :]).astype(np.int32)
    for i in range(1, n):
        if rng.random() < dup_frac:
            s = int(rng.integers(0, i))
            re = rng.random(len(cards)) < flip
            X[i] = np.where(re, X[i], X[s])
    return X
