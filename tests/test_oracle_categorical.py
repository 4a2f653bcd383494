"""Pins for the oracle's categorical extension (CPU only).

The one-hot encoding is pinned by SPEC.md:305-309's forced examples, a decode round trip and the
identity binary-Hamming(encode(u), encode(v)) = 2 D(u, v) (SPEC.md:312 — the paper says "equal",
reading R-C1 takes the factor 2 and estimates D as HAM/2); the estimate by the definitional
recipe in pure Python and near-exactness at large N.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import definitional as D


def _rows(indptr, indices):
    return [indices[indptr[i]:indptr[i + 1]].tolist() for i in range(len(indptr) - 1)]


def test_onehot_spec_examples():
    # (red, hot), (blue, hot): label codes in first-appearance order, cardinalities (2, 1)
    ip, ix, d, st = oracle.onehot(np.array([[0, 0], [1, 0]]), [2, 1])
    assert st == 0 and d == 3
    assert _rows(ip, ix) == [[0, 2], [1, 2]]
    ex = oracle.exact(ix[0:2], ix[2:4])
    assert ex[1] == 2.0 == 2 * oracle.categorical_distance(np.array([[0, 0]]), np.array([[1, 0]]))[0, 0]
    # single column, single category: every vector {0}, D = 0
    ip, ix, d, st = oracle.onehot(np.zeros((5, 1), dtype=np.int32), [1])
    assert d == 1 and _rows(ip, ix) == [[0]] * 5
    assert (oracle.categorical_distance(np.zeros((5, 1)), np.zeros((5, 1))) == 0).all()
    # code outside [0, m_k) -> status
    assert oracle.onehot(np.array([[2, 0]]), [2, 1])[3] == 1
    assert oracle.onehot(np.array([[-1, 0]]), [2, 1])[3] == 1


def test_onehot_round_trip_and_hamming_identity():
    cards = [3, 7, 2, 12, 5]
    X = synth.make_categorical(200, cards, seed=4)
    ip, ix, d, st = oracle.onehot(X, cards)
    assert st == 0 and d == sum(cards)
    off = np.concatenate([[0], np.cumsum(cards)])
    rows = _rows(ip, ix)
    for r, row in enumerate(rows):            # decode: exactly one bit per column block
        assert len(row) == len(cards)
        for k, v in enumerate(row):
            assert off[k] <= v < off[k + 1] and v - off[k] == X[r, k]
    Dm = oracle.categorical_distance(X, X)
    for i in range(0, 200, 7):
        for j in range(0, 200, 11):
            assert oracle.exact(np.array(rows[i]), np.array(rows[j]))[1] == 2 * Dm[i, j]


def test_categorical_estimate_vs_python():
    cards = [4, 9, 3, 20]
    X = synth.make_categorical(30, cards, seed=8)
    ip, ix, d, _ = oracle.onehot(X, cards)
    N = 48
    pi = oracle.make_pi(6, d, N)
    S, _ = oracle.sketch(pi, d, N, ip, ix)
    got = oracle.categorical_estimate(S, S, N, d)
    L = D.card_table(N, d)
    for i in range(30):
        bi = [(int(S[i, j // 32]) >> (j % 32)) & 1 for j in range(N)]
        for j in range(30):
            bj = [(int(S[j, t // 32]) >> (t % 32)) & 1 for t in range(N)]
            e = D.estimate_canonical(sum(bi), sum(bj), D.and_popcount_bits(bi, bj), N, L)
            assert got[i, j] == np.float32(e[1] * 0.5)


def test_categorical_estimate_near_exact_at_large_N():
    cards = [50] * 12
    X = synth.make_categorical(40, cards, seed=9)
    ip, ix, d, _ = oracle.onehot(X, cards)
    N = 1 << 16
    S, _ = oracle.sketch(oracle.make_pi(2, d, N), d, N, ip, ix)
    est = oracle.categorical_estimate(S, S, N, d)
    Dm = oracle.categorical_distance(X, X)
    err = np.abs(est - Dm)
    # a rare bucket collision between the two rows' 24 one-hot bits costs at most one unit of D
    assert err.max() <= 1.01 and err.mean() <= 0.02
    assert (np.diag(est) == 0).all()
