"""Pins for the oracle's BCS parity sketch and its estimates (CPU only).

BCS is the paper's comparison sketch (Definition 2); the paper gives no
estimator, so the estimates follow readings R-B2 / R-B3 (SPEC.md:240-243's inverted
parity-collision law). Pins that share no code with oracle.cpp: the literal Definition-2
sum mod 2 over dense vectors, GF(2) linearity, SPEC.md:239's forced examples, and an
EXHAUSTIVE enumeration over all N^d maps of the collision law the estimator inverts.
"""
import itertools
import math
import random

import numpy as np
import pytest

import oracle
from oracle import definitional as D


def _bits(row, N):
    return [(int(row[j // 32]) >> (j % 32)) & 1 for j in range(N)]


def _csr(rows):
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(r) for r in rows])
    indices = np.array([i for r in rows for i in r], dtype=np.int32)
    return indptr, indices


@pytest.mark.parametrize("N", [2, 3, 5, 33, 64])
def test_bcs_sketch_vs_definition(N):
    rng = random.Random(N)
    d = 40
    b_map = [rng.randrange(N) for _ in range(d)]
    rows = [sorted(rng.sample(range(d), rng.randrange(0, 15))) for _ in range(20)] + [[]]
    indptr, indices = _csr(rows)
    got, st = oracle.bcs_sketch(np.array(b_map, dtype=np.uint32), d, N, indptr, indices)
    assert st == 0
    for r, row in enumerate(rows):
        dense = D.dense(row, d)
        assert _bits(got[r], N) == D.bcs_sketch_bits(dense, b_map, N)


def test_bcs_spec_examples_and_multiset_reading():
    table = np.array([0, 1, 0, 1], dtype=np.uint32)          # SPEC.md:239, N = 2
    for rows, want in (([[0, 2]], 0), ([[]], 0), ([[0]], 1), ([[1, 3]], 0), ([[0, 1]], 3)):
        sk, st = oracle.bcs_sketch(table, 4, 2, *_csr(rows))
        assert st == 0 and int(sk[0, 0]) == want
    # R-B1: a repeated entry toggles twice (cancels); OR-sketch of the same row keeps it
    sk, _ = oracle.bcs_sketch(table, 4, 2, *_csr([[1, 1, 0]]))
    assert int(sk[0, 0]) == 1
    # bad index -> status
    _, st = oracle.bcs_sketch(table, 4, 2, *_csr([[4]]))
    assert st == 1


def test_bcs_gf2_linearity():
    rng = random.Random(5)
    d, N = 300, 97
    pi = oracle.make_pi(3, d, N)
    for _ in range(30):
        a = set(rng.sample(range(d), rng.randrange(0, 60)))
        b = set(rng.sample(range(d), rng.randrange(0, 60)))
        sk, _ = oracle.bcs_sketch(pi, d, N, *_csr([sorted(a), sorted(b), sorted(a ^ b)]))
        assert (sk[2] == (sk[0] ^ sk[1])).all()


@pytest.mark.parametrize("d,N", [(4, 2), (5, 3), (5, 4), (4, 5)])
def test_bcs_collision_law_exhaustive(d, N):
    """Mean over ALL N^d maps: E|a_s XOR b_s| = N(1-(1-2/N)^h)/2 with h = |a XOR b|, and
    E|a_s| = N(1-(1-2/N)^|a|)/2 — the law R-B2's table inverts."""
    cases = [({0, 1}, {1, 2}), ({0, 1, 2}, {3}), ({0}, {0}), (set(range(d)), set()), ({0, 2}, {1, 3})]
    for a, b in cases:
        da, db = D.dense(sorted(a), d), D.dense(sorted(b), d)
        tot_x = tot_a = 0
        count = 0
        for m in itertools.product(range(N), repeat=d):
            sa, sb = D.bcs_sketch_bits(da, list(m), N), D.bcs_sketch_bits(db, list(m), N)
            tot_x += sum(x ^ y for x, y in zip(sa, sb))
            tot_a += sum(sa)
            count += 1
        h = len(a ^ b)
        assert math.isclose(tot_x / count, N * (1 - (1 - 2 / N) ** h) / 2, rel_tol=1e-12, abs_tol=1e-12)
        assert math.isclose(tot_a / count, N * (1 - (1 - 2 / N) ** len(a)) / 2, rel_tol=1e-12, abs_tol=1e-12)


@pytest.mark.parametrize("N,d", [(2, 10), (7, 100), (1024, 50_000), (4097, 10)])
def test_bcs_table(N, d):
    B = oracle.bcs_table(N, d)
    assert B.tobytes() == np.array(D.bcs_table(N, d)).tobytes()
    assert B[0] == 0.0
    for x in range(1, N + 1):
        if 2 * x >= N:
            assert B[x] == float(d)
        else:
            assert B[x] > B[x - 1]
    # the table inverts the collision law: B at the expected XOR count of h differences is h
    if N > 2:
        for h in (1, 2, 5, 40):
            x = N * (1 - (1 - 2 / N) ** h) / 2
            if 2 * x < N - 1:
                inv = math.log1p(-2 * x / N) / math.log1p(-2 / N)
                assert math.isclose(inv, h, rel_tol=1e-9)


def test_bcs_estimate_pair_vs_python_and_conventions():
    N, d = 64, 500
    B = oracle.bcs_table(N, d)
    Bp = D.bcs_table(N, d)
    for pa in range(0, N + 1, 3):
        for pb in range(0, N + 1, 5):
            for pab in range(max(0, pa + pb - N), min(pa, pb) + 1, 2):   # feasible pairs: m <= N
                m = pa + pb - 2 * pab
                got = oracle.bcs_estimate_pair(pa, pb, m, d, B)
                want = D.bcs_estimate(pa, pb, m, d, Bp)
                assert got.tobytes() == np.array(want).tobytes(), (pa, pb, pab)
    e = oracle.bcs_estimate_pair(0, 0, 0, d, B)
    assert tuple(e) == (0.0, 0.0, 1.0, 0.0)          # both empty: JS = 1, COS = 0 (R-G15)
    e = oracle.bcs_estimate_pair(5, 5, 0, d, B)       # identical sketches: HAM 0, JS = COS = 1
    assert e[1] == 0.0 and e[2] == 1.0 and e[3] == 1.0 and e[0] == B[5]


def test_bcs_estimates_near_exact_at_large_N():
    """N >> h^2: buckets rarely collide, so every estimate is within 1 % of the exact value
    (a wrong sign, factor 2 or dropped term fails)."""
    rng = random.Random(11)
    d, N = 100_000, 1 << 18
    pi = oracle.make_pi(9, d, N)
    for _ in range(20):
        a = sorted(rng.sample(range(d), rng.randrange(10, 40)))
        b = sorted(set(rng.sample(a, rng.randrange(1, len(a)))) | set(rng.sample(range(d), rng.randrange(1, 30))))
        sk, _ = oracle.bcs_sketch(pi, d, N, *_csr([a, b]))
        est = oracle.bcs_estimate(sk[:1], sk[1:], N, d, 15)[:, 0, 0]
        ex = oracle.exact(np.array(a), np.array(b))
        for p in range(4):
            assert abs(est[p] - ex[p]) <= 0.01 * max(1.0, ex[p]), (p, est, ex)


def test_bcs_estimate_planes_vs_python():
    rng = random.Random(3)
    N, d = 45, 400
    W = oracle.words(N)
    A = np.zeros((6, W), dtype=np.uint32)
    Bm = np.zeros((8, W), dtype=np.uint32)
    for M in (A, Bm):
        for i in range(M.shape[0]):
            for j in range(N):
                if rng.random() < 0.3:
                    M[i, j // 32] |= np.uint32(1 << (j % 32))
    A[0] = 0
    Bm[2] = A[3]
    T = D.bcs_table(N, d)
    planes = oracle.bcs_estimate(A, Bm, N, d, 15)
    for i in range(6):
        ba = _bits(A[i], N)
        for j in range(8):
            bb = _bits(Bm[j], N)
            m = sum(x ^ y for x, y in zip(ba, bb))
            want = D.bcs_estimate(sum(ba), sum(bb), m, d, T)
            for p in range(4):
                assert planes[p, i, j] == np.float32(want[p])
