"""Pins for the oracle's all-pairs planes and top-k (CPU only).

The pin is an independent per-pair evaluation in pure Python (definitional
per-bit popcounts + the canonical recipe re-implemented in Python floats)
followed by Python's own sort under (key desc, index asc) (reading R-G17).
"""
import math
import random

import numpy as np
import pytest

import oracle
from oracle import definitional as D


def _bits(row, N):
    return [(int(row[j // 32]) >> (j % 32)) & 1 for j in range(N)]


def _rand_sketches(rng, n, N, density):
    W = oracle.words(N)
    out = np.zeros((n, W), dtype=np.uint32)
    for i in range(n):
        for j in range(N):
            if rng.random() < density:
                out[i, j // 32] |= np.uint32(1 << (j % 32))
    return out


@pytest.mark.parametrize("N", [5, 33, 100])
def test_estimate_planes_vs_python(N):
    rng = random.Random(N)
    d = 3 * N
    A = _rand_sketches(rng, 9, N, 0.3)
    B = _rand_sketches(rng, 7, N, 0.5)
    A[0] = 0                     # empty row
    B[1] = A[2]                  # identical pair
    B[2] = np.uint32(0)
    for j in range(N):           # a saturated row
        B[3, j // 32] |= np.uint32(1 << (j % 32))
    L = D.card_table(N, d)
    planes = oracle.estimate(A, B, N, d, 15)
    for i in range(9):
        ba = _bits(A[i], N)
        for j in range(7):
            bb = _bits(B[j], N)
            e = D.estimate_canonical(D.popcount_bits(ba), D.popcount_bits(bb), D.and_popcount_bits(ba, bb), N, L)
            for p in range(4):
                assert planes[p, i, j] == np.float32(e[p])
    # plane selection and order: IP, HAM, JS, COS
    sel = oracle.estimate(A, B, N, d, oracle.JS | oracle.IP)
    assert (sel[0] == planes[0]).all() and (sel[1] == planes[2]).all()


@pytest.mark.parametrize("measure", [1, 2, 4, 8])
@pytest.mark.parametrize("exclude_self", [False, True])
def test_topk_vs_bruteforce(measure, exclude_self):
    rng = random.Random(measure * 10 + exclude_self)
    N, d = 40, 500
    nq, ndb = 6, 30
    DB = _rand_sketches(rng, ndb, N, 0.25)
    DB[5] = DB[7]                               # exact ties -> lower index first
    DB[11] = DB[7]
    Q = DB[:nq].copy() if exclude_self else _rand_sketches(rng, nq, N, 0.25)
    Q[0] = DB[7]
    L = D.card_table(N, d)
    m = [1, 2, 4, 8].index(measure)
    for k in (1, 5, 30, 40):
        idx, sc = oracle.topk(Q, DB, N, d, measure, k, exclude_self=exclude_self)
        for i in range(nq):
            bq = _bits(Q[i], N)
            vals, keys = [], []
            for j in range(ndb):
                bd = _bits(DB[j], N)
                e = D.estimate_canonical(D.popcount_bits(bq), D.popcount_bits(bd), D.and_popcount_bits(bq, bd), N, L)
                vals.append(e[m])
                keys.append(-e[m] if measure == 2 else e[m])
            want = D.topk_bruteforce(keys, k, exclude=i if exclude_self else None)
            got = idx[i].tolist()
            assert got[:len(want)] == want
            assert all(x == -1 for x in got[len(want):])
            assert all(math.isnan(x) for x in sc[i, len(want):])
            assert sc[i, :len(want)].tolist() == [float(np.float32(vals[j])) for j in want]
