"""Pins for the oracle's pi map, sketch and popcounts (CPU only).

Every pin is something other than the oracle itself: published test vectors,
the brute-force preimage-OR definition evaluated per bit on a
dense vector, SPEC's forced examples, and algebraic invariants.
"""
import random

import numpy as np
import pytest

import oracle
from oracle import definitional as D
from bsk_helpers import golden_lines


def _csr(rows):
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    for r, s in enumerate(rows):
        indptr[r + 1] = indptr[r] + len(s)
    idx = np.array([i for s in rows for i in s], dtype=np.int32)
    return indptr, idx


# ---------------------------------------------------------------- pi -------
def test_pi_golden():
    for f in golden_lines("pi_splitmix64.txt"):
        if f[0] == "first_raw":
            assert oracle.mix64(0x9E3779B97F4A7C15) == int(f[1], 16)
            assert D.mix64(0x9E3779B97F4A7C15) == int(f[1], 16)
        else:
            seed, d, N = (int(x.split("=")[1]) for x in f[1:4])
            want = [int(x) for x in f[4:]]
            assert oracle.make_pi(seed, d, N).tolist() == want


def test_pi_python_vs_cpp():
    for seed in (0, 1, 7, 2**63 + 5):
        for N in (2, 3, 31, 1000, 1224, 4096, 65537):
            assert oracle.make_pi(seed, 64, N).tolist() == D.make_pi(seed, 64, N)


def test_pi_range_and_uniformity():
    pi = oracle.make_pi(3, 160_000, 16)
    assert pi.max() < 16
    counts = np.bincount(pi, minlength=16)
    chi2 = ((counts - 10_000) ** 2 / 10_000).sum()
    assert chi2 < 45  # 15 dof, p ~ 1e-4
    assert set(oracle.make_pi(9, 100, 2).tolist()) == {0, 1}
    assert (oracle.make_pi(5, 1000, 77) == oracle.make_pi(5, 1000, 77)).all()


def test_recommended_N():
    # Theorem 1
    assert oracle.recommended_N(100, 0.1) == 1224
    assert oracle.recommended_N(20, 0.1) == 110
    assert oracle.recommended_N(1, 0.999999) == 2
    assert oracle.recommended_N(0, 0.1) == 0
    assert oracle.recommended_N(10, 0.0) == 0
    assert oracle.recommended_N(10, 1.0) == 0


# ------------------------------------------------------------ sketch -------
def test_sketch_spec_examples():
    # explicit table [0,1,0,1] (d=4, N=2)
    pi = np.array([0, 1, 0, 1], dtype=np.uint32)
    indptr, idx = _csr([[0, 2], [0, 1, 2, 3], []])
    sk, st = oracle.sketch(pi, 4, 2, indptr, idx)
    assert st == 0
    assert sk[:, 0].tolist() == [0b01, 0b11, 0]
    assert oracle.popcount(sk, 2).tolist() == [1, 2, 0]


@pytest.mark.parametrize("N", [2, 3, 31, 32, 33, 63, 64, 65])
def test_sketch_vs_bruteforce_preimage_or(N):
    rng = random.Random(1000 + N)
    for trial in range(40):
        d = rng.randint(1, 64)
        if trial % 3 == 0:
            pi = [rng.randrange(N) for _ in range(d)]        # explicit table, forced collisions
        else:
            pi = D.make_pi(rng.randrange(2**64), d, N)
        rows = []
        for _ in range(5):
            m = rng.randint(0, d)
            rows.append(sorted(rng.sample(range(d), m)))
        indptr, idx = _csr(rows)
        sk, st = oracle.sketch(np.array(pi, dtype=np.uint32), d, N, indptr, idx)
        assert st == 0
        for r, s in enumerate(rows):
            bits = D.sketch_bits(D.dense(s, d), pi, N)
            assert sk[r].tolist() == D.pack_bits(bits)
            assert oracle.popcount(sk[r:r + 1], N)[0] == D.popcount_bits(bits)


def test_sketch_invariants():
    rng = random.Random(7)
    N, d = 45, 300
    pi = oracle.make_pi(11, d, N)
    W = oracle.words(N)
    for _ in range(50):
        a = sorted(rng.sample(range(d), rng.randint(0, 80)))
        b = sorted(rng.sample(range(d), rng.randint(0, 80)))
        u = sorted(set(a) | set(b))
        sub = sorted(rng.sample(a, len(a) // 2))
        indptr, idx = _csr([a, b, u, sub])
        sk, _ = oracle.sketch(pi, d, N, indptr, idx)
        assert (sk[2] == (sk[0] | sk[1])).all()                 # OR-homomorphism
        assert ((sk[3] & ~sk[0]) == 0).all()                     # monotonicity
        pc = oracle.popcount(sk, N)
        assert pc[0] <= min(N, len(a))                           # cardinality cap
        tail = N % 32
        if tail:
            assert (sk[:, W - 1] >> tail == 0).all()             # tail bits zero


def test_sketch_duplicates_unsorted_and_bad_index():
    pi = oracle.make_pi(2, 50, 40)
    indptr, idx = _csr([[3, 9, 17], [17, 3, 3, 9, 9]])
    sk, st = oracle.sketch(pi, 50, 40, indptr, idx)
    assert st == 0 and (sk[0] == sk[1]).all()
    indptr, idx = _csr([[3, 50]])
    _, st = oracle.sketch(pi, 50, 40, indptr, idx)
    assert st == 2
    indptr, idx = _csr([[-1]])
    _, st = oracle.sketch(pi, 50, 40, indptr, idx)
    assert st == 2


def test_popcount_and_andpopc():
    # SPEC.md:81, 87
    N = 64
    z = np.zeros((1, 2), dtype=np.uint32)
    ones = np.full((1, 2), 0xFFFFFFFF, dtype=np.uint32)
    assert oracle.popcount(z, N)[0] == 0 and oracle.popcount(ones, N)[0] == 64
    x = np.array([[0b011, 0]], dtype=np.uint32)
    y = np.array([[0b110, 0]], dtype=np.uint32)
    assert oracle.andpopc(x, y, N)[0, 0] == 1
    assert oracle.andpopc(x, x, N)[0, 0] == 2
    assert oracle.andpopc(x, np.array([[0b100, 1]], dtype=np.uint32), N)[0, 0] == 0
    rng = np.random.default_rng(0)
    A = rng.integers(0, 2**32, size=(7, 3), dtype=np.uint32)
    B = rng.integers(0, 2**32, size=(5, 3), dtype=np.uint32)
    M = oracle.andpopc(A, B, 96)
    pa, pb = oracle.popcount(A, 96), oracle.popcount(B, 96)
    for i in range(7):
        for j in range(5):
            bits_a = [(int(A[i, w]) >> t) & 1 for w in range(3) for t in range(32)]
            bits_b = [(int(B[j, w]) >> t) & 1 for w in range(3) for t in range(32)]
            assert M[i, j] == D.and_popcount_bits(bits_a, bits_b)
            assert M[i, j] <= min(pa[i], pb[j])
    assert (oracle.andpopc(B, A, 96) == M.T).all()               # symmetry
