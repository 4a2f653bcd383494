"""CPU oracle for the BinSketch hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The
product path (``paper_1910_04658_b200``) must never import it, and shares no
code with it (tests/test_abi_host.py::test_product_shares_no_code_with_oracle checks this).

``liboracle.so`` is built from ``oracle.cpp`` (plain C++17, fp64, no FMA
contraction, OpenMP over rows). ``definitional.py`` is the per-bit
pure-Python oracle for tiny inputs that pins it.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

IP, HAM, JS, COS = 1, 2, 4, 8
MEASURES = {"ip": IP, "ham": HAM, "js": JS, "cos": COS}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
                               "-ffp-contract=off", src, "-o", _SO])
    return _SO


def _lib_():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        u64, u32, i32, vp, dbl, i64 = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32,
                                       ctypes.c_void_p, ctypes.c_double, ctypes.c_int64)
        L.orc_mix64.argtypes = [u64]; L.orc_mix64.restype = u64
        L.orc_make_pi.argtypes = [u64, u64, u32, vp]; L.orc_make_pi.restype = None
        L.orc_recommended_N.argtypes = [u32, dbl]; L.orc_recommended_N.restype = u32
        L.orc_sketch.argtypes = [vp, u64, u32, vp, vp, u64, vp]; L.orc_sketch.restype = ctypes.c_int
        L.orc_popcount.argtypes = [vp, u64, u32, vp]; L.orc_popcount.restype = None
        L.orc_andpopc.argtypes = [vp, u64, vp, u64, u32, vp]; L.orc_andpopc.restype = None
        L.orc_card_table.argtypes = [u32, u64, vp]; L.orc_card_table.restype = None
        L.orc_estimate_pair.argtypes = [i32, i32, i32, u32, vp, vp]; L.orc_estimate_pair.restype = None
        L.orc_estimate_literal.argtypes = [i32, i32, i32, u32, u64, vp]
        L.orc_estimate_literal.restype = None
        L.orc_estimate.argtypes = [vp, u64, vp, u64, u32, u64, u32, vp]; L.orc_estimate.restype = None
        L.orc_topk.argtypes = [vp, u64, vp, u64, u32, u64, u32, u32, u32, vp, vp, ctypes.c_int]
        L.orc_topk.restype = None
        L.orc_exact.argtypes = [vp, i64, vp, i64, vp]; L.orc_exact.restype = None
        L.orc_join.argtypes = [vp, u64, vp, u64, u32, u64, u32, vp, u32, u32, vp]
        L.orc_join.restype = None
        L.orc_join_exact.argtypes = [vp, vp, u64, vp, vp, u64, u32, vp, u32, u32, vp]
        L.orc_join_exact.restype = None
        L.orc_bcs_sketch.argtypes = [vp, u64, u32, vp, vp, u64, vp]; L.orc_bcs_sketch.restype = ctypes.c_int
        L.orc_bcs_table.argtypes = [u32, u64, vp]; L.orc_bcs_table.restype = None
        L.orc_bcs_estimate_pair.argtypes = [i32, i32, i32, u64, vp, vp]; L.orc_bcs_estimate_pair.restype = None
        L.orc_bcs_estimate.argtypes = [vp, u64, vp, u64, u32, u64, u32, vp]; L.orc_bcs_estimate.restype = None
        L.orc_mse.argtypes = [vp, u64, u32, u64, vp, vp, u32, vp, u32, u32, vp, vp]; L.orc_mse.restype = None
        L.orc_onehot.argtypes = [vp, u64, u32, vp, vp, vp]; L.orc_onehot.restype = ctypes.c_int
        L.orc_categorical_distance.argtypes = [vp, u64, vp, u64, u32, vp]; L.orc_categorical_distance.restype = None
        L.orc_categorical_estimate.argtypes = [vp, u64, vp, u64, u32, u64, vp]
        L.orc_categorical_estimate.restype = None
        L.orc_enumerate.argtypes = [u32, u32, vp, i64, vp, i64, vp, vp]
        L.orc_enumerate.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def words(N: int) -> int:
    return (N + 31) // 32


def mix64(z: int) -> int:
    return int(_lib_().orc_mix64(z))


def make_pi(seed: int, d: int, N: int) -> np.ndarray:
    pi = np.empty(d, dtype=np.uint32)
    _lib_().orc_make_pi(seed, d, N, _p(pi))
    return pi


def recommended_N(psi: int, rho: float) -> int:
    return int(_lib_().orc_recommended_N(psi, rho))


def sketch(pi: np.ndarray, d: int, N: int, indptr: np.ndarray, indices: np.ndarray):
    """Returns (uint32[n][W], status)."""
    n = len(indptr) - 1
    out = np.empty((n, words(N)), dtype=np.uint32)
    st = _lib_().orc_sketch(_p(np.ascontiguousarray(pi, dtype=np.uint32)), d, N,
                            _p(np.ascontiguousarray(indptr, dtype=np.int64)),
                            _p(np.ascontiguousarray(indices, dtype=np.int32)), n, _p(out))
    return out, int(st)


def popcount(sk: np.ndarray, N: int) -> np.ndarray:
    sk = np.ascontiguousarray(sk, dtype=np.uint32)
    out = np.empty(sk.shape[0], dtype=np.int32)
    _lib_().orc_popcount(_p(sk), sk.shape[0], N, _p(out))
    return out


def andpopc(A: np.ndarray, B: np.ndarray, N: int) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint32)
    B = np.ascontiguousarray(B, dtype=np.uint32)
    out = np.empty((A.shape[0], B.shape[0]), dtype=np.int32)
    _lib_().orc_andpopc(_p(A), A.shape[0], _p(B), B.shape[0], N, _p(out))
    return out


def card_table(N: int, d: int) -> np.ndarray:
    L = np.empty(N + 1, dtype=np.float64)
    _lib_().orc_card_table(N, d, _p(L))
    return L


def estimate_pair(pa: int, pb: int, pab: int, N: int, L: np.ndarray) -> np.ndarray:
    out = np.empty(4, dtype=np.float64)
    _lib_().orc_estimate_pair(pa, pb, pab, N, _p(L), _p(out))
    return out


def estimate_literal(pa: int, pb: int, pab: int, N: int, d: int) -> np.ndarray:
    tr = np.empty(9, dtype=np.float64)
    _lib_().orc_estimate_literal(pa, pb, pab, N, d, _p(tr))
    return tr


def estimate(A: np.ndarray, B: np.ndarray, N: int, d: int, measure: int) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint32)
    B = np.ascontiguousarray(B, dtype=np.uint32)
    planes = bin(measure & 15).count("1")
    out = np.empty((planes, A.shape[0], B.shape[0]), dtype=np.float32)
    _lib_().orc_estimate(_p(A), A.shape[0], _p(B), B.shape[0], N, d, measure, _p(out))
    return out


def topk(Q: np.ndarray, D: np.ndarray, N: int, d: int, measure: int, k: int,
         exclude_self: bool = False, nthreads: int = 0):
    Q = np.ascontiguousarray(Q, dtype=np.uint32)
    D = np.ascontiguousarray(D, dtype=np.uint32)
    idx = np.empty((Q.shape[0], k), dtype=np.int32)
    sc = np.empty((Q.shape[0], k), dtype=np.float32)
    _lib_().orc_topk(_p(Q), Q.shape[0], _p(D), D.shape[0], N, d, measure, k,
                     1 if exclude_self else 0, _p(idx), _p(sc), nthreads)
    return idx, sc


def exact(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.int32)
    out = np.empty(4, dtype=np.float64)
    _lib_().orc_exact(_p(a), len(a), _p(b), len(b), _p(out))
    return out


def join(Q: np.ndarray, D: np.ndarray, N: int, d: int, measure: int, thresholds,
         exclude_self: bool = False) -> np.ndarray:
    """Threshold join from sketches (Exp. 2's O'; reading R-J1).

    Returns uint32 bits [nthr][nq][ceil(ndb/32)].
    """
    Q = np.ascontiguousarray(Q, dtype=np.uint32)
    D = np.ascontiguousarray(D, dtype=np.uint32)
    thr = np.ascontiguousarray(np.atleast_1d(np.asarray(thresholds, dtype=np.float64)))
    out = np.empty((len(thr), Q.shape[0], (D.shape[0] + 31) // 32), dtype=np.uint32)
    _lib_().orc_join(_p(Q), Q.shape[0], _p(D), D.shape[0], N, d, measure, _p(thr), len(thr),
                     1 if exclude_self else 0, _p(out))
    return out


def join_exact(qptr, qidx, dptr, didx, measure: int, thresholds, exclude_self: bool = False) -> np.ndarray:
    """Threshold join on the uncompressed rows (Exp. 2's ground truth O). CSR, sorted supports."""
    qptr = np.ascontiguousarray(qptr, dtype=np.int64)
    qidx = np.ascontiguousarray(qidx, dtype=np.int32)
    dptr = np.ascontiguousarray(dptr, dtype=np.int64)
    didx = np.ascontiguousarray(didx, dtype=np.int32)
    thr = np.ascontiguousarray(np.atleast_1d(np.asarray(thresholds, dtype=np.float64)))
    nq, ndb = len(qptr) - 1, len(dptr) - 1
    out = np.empty((len(thr), nq, (ndb + 31) // 32), dtype=np.uint32)
    _lib_().orc_join_exact(_p(qptr), _p(qidx), nq, _p(dptr), _p(didx), ndb, measure, _p(thr), len(thr),
                           1 if exclude_self else 0, _p(out))
    return out


def bits_to_sets(bits: np.ndarray, ndb: int) -> list[set]:
    """Rows of a [nq][ceil(ndb/32)] bit matrix as Python sets of column indices."""
    out = []
    for row in np.asarray(bits, dtype=np.uint32):
        cols = np.nonzero(np.unpackbits(row.view(np.uint8), bitorder="little")[:ndb])[0]
        out.append(set(int(c) for c in cols))
    return out


def ranking_metrics(O: list[set], Op: list[set]) -> dict:
    """Experiment 2's measures per query, macro-averaged.

    accuracy = |O ∩ O'| / |O ∪ O'|, precision = |O ∩ O'| / |O'|,
    recall = |O ∩ O'| / |O|, F1 = 2 p r / (p + r). Queries with O = O' = ∅ are
    skipped; a 0/0 precision or recall counts as 0 and F1 = 0 when
    p + r = 0 (reading R-J2).
    """
    acc, pre, rec, f1 = [], [], [], []
    skipped = 0
    for o, op in zip(O, Op):
        u = len(o | op)
        if u == 0:
            skipped += 1
            continue
        i = len(o & op)
        p = i / len(op) if op else 0.0
        r = i / len(o) if o else 0.0
        acc.append(i / u)
        pre.append(p)
        rec.append(r)
        f1.append(2 * p * r / (p + r) if p + r > 0 else 0.0)
    mean = (lambda v: float(np.mean(v)) if v else float("nan"))
    return {"accuracy": mean(acc), "precision": mean(pre), "recall": mean(rec), "f1": mean(f1),
            "query_count": len(acc), "skipped_queries": skipped}


def bcs_sketch(pi: np.ndarray, d: int, N: int, indptr: np.ndarray, indices: np.ndarray):
    """BCS parity sketches: (uint32[n][W], status)."""
    n = len(indptr) - 1
    out = np.empty((n, words(N)), dtype=np.uint32)
    st = _lib_().orc_bcs_sketch(_p(np.ascontiguousarray(pi, dtype=np.uint32)), d, N,
                                _p(np.ascontiguousarray(indptr, dtype=np.int64)),
                                _p(np.ascontiguousarray(indices, dtype=np.int32)), n, _p(out))
    return out, int(st)


def bcs_table(N: int, d: int) -> np.ndarray:
    B = np.empty(N + 1, dtype=np.float64)
    _lib_().orc_bcs_table(N, d, _p(B))
    return B


def bcs_estimate_pair(pa: int, pb: int, m: int, d: int, B: np.ndarray) -> np.ndarray:
    out = np.empty(4, dtype=np.float64)
    _lib_().orc_bcs_estimate_pair(pa, pb, m, d, _p(B), _p(out))
    return out


def bcs_estimate(A: np.ndarray, B: np.ndarray, N: int, d: int, measure: int) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint32)
    B = np.ascontiguousarray(B, dtype=np.uint32)
    planes = bin(measure & 15).count("1")
    out = np.empty((planes, A.shape[0], B.shape[0]), dtype=np.float32)
    _lib_().orc_bcs_estimate(_p(A), A.shape[0], _p(B), B.shape[0], N, d, measure, _p(out))
    return out


def mse(S: np.ndarray, N: int, d: int, indptr, indices, measure: int, thresholds, bcs: bool = False):
    """Experiment 1 sums (R-M1): (sse float64[nthr], count uint64[nthr]) over pairs
    i < j whose exact similarity reaches each threshold; est from the sketches S (BCS if bcs)."""
    S = np.ascontiguousarray(S, dtype=np.uint32)
    thr = np.ascontiguousarray(np.atleast_1d(np.asarray(thresholds, dtype=np.float64)))
    sse = np.empty(len(thr), dtype=np.float64)
    cnt = np.empty(len(thr), dtype=np.uint64)
    _lib_().orc_mse(_p(S), S.shape[0], N, d, _p(np.ascontiguousarray(indptr, dtype=np.int64)),
                    _p(np.ascontiguousarray(indices, dtype=np.int32)), measure, _p(thr), len(thr),
                    1 if bcs else 0, _p(sse), _p(cnt))
    return sse, cnt


def mse_report(sse: np.ndarray, count: np.ndarray, measure: int) -> list[dict]:
    """MSE per threshold and, for JS / COS, -ln(MSE); empty sets -> absent."""
    out = []
    for s, c in zip(sse, count):
        if c == 0:
            out.append(None)
            continue
        v = float(s) / float(c)
        r = {"pairs": int(c), "mse": v}
        if measure in (JS, COS):
            r["neg_log_mse"] = -math.log(v) if v > 0 else math.inf
        out.append(r)
    return out


def onehot(codes: np.ndarray, cards) -> tuple:
    """Categorical extension: label codes [n][c] -> one-hot CSR.
    Returns (indptr, indices, d, status)."""
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    n, c = codes.shape
    offsets = np.zeros(c + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(np.asarray(cards, dtype=np.int64))
    indptr = np.empty(n + 1, dtype=np.int64)
    indices = np.empty(n * c, dtype=np.int32)
    st = _lib_().orc_onehot(_p(codes), n, c, _p(offsets), _p(indptr), _p(indices))
    return indptr, indices, int(offsets[-1]), int(st)


def categorical_distance(U: np.ndarray, V: np.ndarray) -> np.ndarray:
    U = np.ascontiguousarray(U, dtype=np.int32)
    V = np.ascontiguousarray(V, dtype=np.int32)
    out = np.empty((U.shape[0], V.shape[0]), dtype=np.int32)
    _lib_().orc_categorical_distance(_p(U), U.shape[0], _p(V), V.shape[0], U.shape[1], _p(out))
    return out


def categorical_estimate(A: np.ndarray, B: np.ndarray, N: int, d: int) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint32)
    B = np.ascontiguousarray(B, dtype=np.uint32)
    out = np.empty((A.shape[0], B.shape[0]), dtype=np.float32)
    _lib_().orc_categorical_estimate(_p(A), A.shape[0], _p(B), B.shape[0], N, d, _p(out))
    return out


def enumerate_expectations(d: int, N: int, a, b):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.int32))
    m1 = ctypes.c_double()
    m2 = ctypes.c_double()
    rc = _lib_().orc_enumerate(d, N, _p(a), len(a), _p(b), len(b), ctypes.byref(m1), ctypes.byref(m2))
    if rc != 0:
        raise ValueError("instance too large to enumerate")
    return m1.value, m2.value
