"""Pins for the oracle's threshold join and Experiment-2 measures (CPU only).

The join (reading R-J1) is pinned two ways that share no code
with oracle.cpp: (1) per pair, the definitional per-bit popcounts and the
canonical recipe in pure Python (estimate side); (2) the exact side against a
dense 0/1 numpy matmul (a library routine for |a ∩ b|) and numpy's own fp64
division / sqrt. The Exp.-2 measures are pinned by SPEC.md:404's worked
examples and by hand-derived special cases.
"""
import math
import random

import numpy as np
import pytest

import oracle
import synth
from oracle import definitional as D

THR = [0.95, 0.9, 0.8, 0.5, 0.2, 0.1, 0.0]


def _bits(row, N):
    return [(int(row[j // 32]) >> (j % 32)) & 1 for j in range(N)]


def _rand_sketches(rng, n, N, density):
    out = np.zeros((n, oracle.words(N)), dtype=np.uint32)
    for i in range(n):
        for j in range(N):
            if rng.random() < density:
                out[i, j // 32] |= np.uint32(1 << (j % 32))
    return out


def _pack(mask_rows, ndb):
    """bool [nq][ndb] -> uint32 [nq][ceil(ndb/32)] (bit j%32 of word j/32)."""
    wpr = (ndb + 31) // 32
    out = np.zeros((len(mask_rows), wpr), dtype=np.uint32)
    for i, row in enumerate(mask_rows):
        for j in np.nonzero(row)[0]:
            out[i, j // 32] |= np.uint32(1 << (int(j) % 32))
    return out


def _key(m, e):
    v = e[{1: 0, 2: 1, 4: 2, 8: 3}[m]]
    return -v if m == 2 else v


@pytest.mark.parametrize("measure", [1, 2, 4, 8])
@pytest.mark.parametrize("exclude_self", [False, True])
def test_join_vs_python_bruteforce(measure, exclude_self):
    rng = random.Random(100 + measure * 2 + exclude_self)
    N, d = 40, 300
    Q = _rand_sketches(rng, 11, N, 0.3)
    Dm = _rand_sketches(rng, 37, N, 0.35)   # ragged: 37 columns -> 2 words, 27 tail bits
    Q[0] = 0
    Dm[3] = Q[1]
    Dm[5] = 0
    L = D.card_table(N, d)
    thr = [t * (60.0 if measure in (1, 2) else 1.0) for t in THR]
    got = oracle.join(Q, Dm, N, d, measure, thr, exclude_self)
    assert got.shape == (len(thr), 11, 2)
    for t, th in enumerate(thr):
        tk = -th if measure == 2 else th
        mask = np.zeros((11, 37), dtype=bool)
        for i in range(11):
            ba = _bits(Q[i], N)
            for j in range(37):
                if exclude_self and i == j:
                    continue
                bb = _bits(Dm[j], N)
                e = D.estimate_canonical(D.popcount_bits(ba), D.popcount_bits(bb), D.and_popcount_bits(ba, bb), N, L)
                mask[i, j] = _key(measure, e) >= tk
        assert (got[t] == _pack(mask, 37)).all(), (t, th)


def _dense(indptr, indices, d):
    n = len(indptr) - 1
    X = np.zeros((n, d), dtype=np.int64)
    for i in range(n):
        X[i, indices[indptr[i]:indptr[i + 1]]] = 1
    return X


@pytest.mark.parametrize("measure", [1, 2, 4, 8])
def test_join_exact_vs_dense_matmul(measure):
    ip_, ix_ = synth.make_csr(synth.scaled(synth.TINY, 150, seed=21))
    ip_, ix_ = synth.plant_near_duplicates(ip_, ix_, synth.TINY.d, 0.4, seed=22)
    tr, q = synth.split_rows(150, 0.2, seed=23)
    qp, qi = synth.take_rows(ip_, ix_, q)
    dp, di = synth.take_rows(ip_, ix_, tr)
    A, B = _dense(qp, qi, synth.TINY.d), _dense(dp, di, synth.TINY.d)
    inter = (A @ B.T).astype(np.float64)
    na = A.sum(1).astype(np.float64)[:, None]
    nb = B.sum(1).astype(np.float64)[None, :]
    if measure == 1:
        val = inter
    elif measure == 2:
        val = na + nb - 2.0 * inter
    elif measure == 4:
        val = inter / (na + nb - inter)
    else:
        val = inter / np.sqrt(na * nb)
    thr = [t * (40.0 if measure in (1, 2) else 1.0) for t in THR] + ([0.5] if measure == 4 else [])
    got = oracle.join_exact(qp, qi, dp, di, measure, thr)
    for t, th in enumerate(thr):
        mask = val <= th if measure == 2 else val >= th
        assert (got[t] == _pack(mask, B.shape[0])).all(), (t, th)
    # the planted duplicates make the high thresholds non-trivial
    if measure in (4, 8):
        assert 0 < np.count_nonzero(val >= 0.8) < val.size // 10


def test_join_thresholds_nested_and_trivial():
    rng = random.Random(7)
    N, d = 64, 400
    Q = _rand_sketches(rng, 9, N, 0.25)
    Dm = _rand_sketches(rng, 45, N, 0.25)
    for m in (1, 4, 8):
        planes = oracle.join(Q, Dm, N, d, m, [0.9, 0.5, 0.2, 0.0])
        for t in range(3):   # a higher threshold selects a subset
            assert ((planes[t] & ~planes[t + 1]) == 0).all()
        # every estimate of IP / JS / COS is >= 0: threshold 0 selects all 45 pairs per row
        full = np.array([0xFFFFFFFF, (1 << 13) - 1], dtype=np.uint32)
        assert (planes[3] == full).all()
        ex = oracle.join(Q, Dm, N, d, m, [0.0], exclude_self=True)[0]
        for i in range(9):
            want = full.copy()
            want[i // 32] &= np.uint32(~(1 << (i % 32)) & 0xFFFFFFFF)
            assert (ex[i] == want).all()
    # Hamming: distance <= huge selects everything, < 0 nothing
    assert (oracle.join(Q, Dm, N, d, 2, [1e9])[0] == np.array([0xFFFFFFFF, (1 << 13) - 1], dtype=np.uint32)).all()
    assert (oracle.join(Q, Dm, N, d, 2, [-1.0])[0] == 0).all()


def test_join_exact_identical_rows():
    # exact JS >= 1 and exact COS >= 1 select exactly the identical rows; Hamming <= 0 too
    qp = np.array([0, 3, 5, 5], dtype=np.int64)
    qi = np.array([1, 4, 9, 2, 3], dtype=np.int32)            # {1,4,9}, {2,3}, {}
    dp = np.array([0, 2, 5, 8, 8, 10], dtype=np.int64)
    di = np.array([2, 3, 1, 4, 9, 1, 4, 8, 2, 3], dtype=np.int32)   # {2,3},{1,4,9},{1,4,8},{},{2,3}
    js = oracle.join_exact(qp, qi, dp, di, 4, [1.0])[0]
    assert [int(w) for w in js[:, 0]] == [0b00010, 0b10001, 0b01000]   # empty-empty JS = 1 (R-G3)
    cs = oracle.join_exact(qp, qi, dp, di, 8, [1.0])[0]
    assert [int(w) for w in cs[:, 0]] == [0b00010, 0b10001, 0]          # COS with an empty side = 0
    hm = oracle.join_exact(qp, qi, dp, di, 2, [0.0])[0]
    assert [int(w) for w in hm[:, 0]] == [0b00010, 0b10001, 0b01000]
    ip = oracle.join_exact(qp, qi, dp, di, 1, [2.0])[0]                 # |a ∩ b| >= 2
    assert [int(w) for w in ip[:, 0]] == [0b00110, 0b10001, 0]


def test_ranking_metrics_spec_examples():
    r = oracle.ranking_metrics([{1, 2, 3}], [{2, 3, 4}])
    assert r["accuracy"] == 0.5
    assert math.isclose(r["precision"], 2 / 3) and math.isclose(r["recall"], 2 / 3)
    assert math.isclose(r["f1"], 2 / 3)
    r = oracle.ranking_metrics([{5, 7}, {1}], [{5, 7}, {1}])         # O' = O
    assert r == {"accuracy": 1.0, "precision": 1.0, "recall": 1.0, "f1": 1.0, "query_count": 2,
                 "skipped_queries": 0}
    # O = O' = ∅ skipped; O' = ∅ with O ≠ ∅ scores 0 (R-J2); macro average over queries
    r = oracle.ranking_metrics([set(), {1, 2}, {3}], [set(), set(), {3, 4}])
    assert r["skipped_queries"] == 1 and r["query_count"] == 2
    assert r["accuracy"] == 0.25 and r["precision"] == 0.25 and r["recall"] == 0.5
    assert math.isclose(r["f1"], (0 + 2 * 0.5 * 1 / 1.5) / 2)


def test_bits_to_sets_roundtrip():
    m = np.zeros((3, 70), dtype=bool)
    m[0, [0, 31, 32, 69]] = True
    m[2, 5] = True
    assert oracle.bits_to_sets(_pack(m, 70), 70) == [{0, 31, 32, 69}, set(), {5}]


def test_exp2_estimate_tracks_exact_at_large_N():
    """Statistical: with N >> psi the sketch join recovers the exact join (F1 near 1 at
    J = 0.8 JS), and F1 grows with N (SPEC.md:484 trend, one instance)."""
    d = 20000
    ip_, ix_ = synth.make_csr(synth.CSRSpec(n=400, d=d, kind=0, p1=20, p2=60, cap=60, zipf_s=1.05, seed=31))
    ip_, ix_ = synth.plant_near_duplicates(ip_, ix_, d, 0.5, seed=32)
    tr, q = synth.split_rows(400, 0.1, seed=33)
    qp, qi = synth.take_rows(ip_, ix_, q)
    dp, di = synth.take_rows(ip_, ix_, tr)
    O = oracle.bits_to_sets(oracle.join_exact(qp, qi, dp, di, 4, [0.8])[0], len(tr))
    f1 = {}
    for N in (64, 4096):
        pi = oracle.make_pi(1, d, N)
        Qs, _ = oracle.sketch(pi, d, N, qp, qi)
        Ds, _ = oracle.sketch(pi, d, N, dp, di)
        Op = oracle.bits_to_sets(oracle.join(Qs, Ds, N, d, 4, [0.8])[0], len(tr))
        f1[N] = oracle.ranking_metrics(O, Op)["f1"]
    assert sum(len(o) for o in O) >= 10
    assert f1[4096] > 0.9 and f1[4096] > f1[64]
