"""Pins for the oracle's estimators (Alg. 1-4), Lemma 1 and the concentration lemmas.

Pins: SPEC's worked examples (tests/golden/estimator_examples.txt), the literal
pow/log Algorithm 1 text vs the canonical recipe, exhaustive enumeration of
Lemma 1 over all N^d maps, the textbook balls-in-bins occupancy moments,
near-exactness when N >> psi^2 (which a dropped term or a flipped sign
breaks), the paper's concentration bounds, and a committed bias band.
"""
import json
import math
import os
import random

import numpy as np
import pytest

import oracle
from oracle import definitional as D
from bsk_helpers import GOLDEN, golden_lines
from tools.mc_pairs import ensemble


def test_card_table_pins():
    for f in golden_lines("estimator_examples.txt"):
        if f[0] == "card":
            N, k, d, want = int(f[1]), int(f[2]), int(f[3]), float(f[4])
            L = oracle.card_table(N, d)
            if k == 95:
                assert L[k] == want                       # SPEC.md:136 / SURVEY C5 (log1p form)
            else:
                assert L[k] == want                       # exact (0 and the N=2 identity ratio)
    for N in (2, 3, 33, 1000, 1224, 5000):
        L = oracle.card_table(N, 77)
        assert L[0] == 0.0 and L[N] == 77.0
        assert (np.diff(L[:N]) > 0).all()                 # strictly increasing
        assert L.tolist() == D.card_table(N, 77)          # Python re-evaluation, bit-identical
        # L[k] -> k for k << N (ln(1-k/N)/ln(1-1/N) ~ k): the estimate of |a| is ~|a_s|
        assert abs(L[1] - 1.0) < 1e-12


def test_ip_worked_examples():
    for f in golden_lines("estimator_examples.txt"):
        if f[0] == "ipraw":
            N, d, pa, pb, pab, want = (int(f[1]), int(f[2]), int(f[3]), int(f[4]), int(f[5]), float(f[6]))
            raw = D.estimate_literal(pa, pb, pab, N, d)[0]
            assert raw == pytest.approx(want, abs=1e-15)
            tr = oracle.estimate_literal(pa, pb, pab, N, d)
            assert tr[5] == max(0.0, want)
        if f[0] == "all":
            N, d, pa, pb, pab = (int(x) for x in f[1:6])
            want = [float(x) for x in f[6:10]]
            L = oracle.card_table(N, d)
            assert oracle.estimate_pair(pa, pb, pab, N, L).tolist() == want
            assert list(oracle.estimate_literal(pa, pb, pab, N, d)[5:9]) == want


def test_identity_map_worked_example_end_to_end():
    # d=4, N=4, identity pi, a={0}, b={1}
    pi = np.arange(4, dtype=np.uint32)
    sk, _ = oracle.sketch(pi, 4, 4, np.array([0, 1, 2], dtype=np.int64), np.array([0, 1], dtype=np.int32))
    pa, pb = oracle.popcount(sk, 4)
    pab = oracle.andpopc(sk[:1], sk[1:], 4)[0, 0]
    est = oracle.estimate_pair(pa, pb, pab, 4, oracle.card_table(4, 4))
    assert est.tolist() == [0.0, 2.0, 0.0, 0.0]


@pytest.mark.parametrize("N,d", [(2, 10), (3, 5), (64, 1000), (1224, 5000), (1000, 28102), (4096, 102660)])
def test_canonical_vs_literal(N, d):
    """R-C2 identity: canonical recipe == literal Alg. 1-4 (pow/log) to 1e-12 relative."""
    L = oracle.card_table(N, d)
    rng = random.Random(N)
    cases = [(0, 0, 0), (N, N, N), (N, 0, 0), (0, N, 0), (1, 1, 1), (N - 1, N - 1, N - 2)]
    for _ in range(3000):
        pa = rng.randint(0, N)
        pb = rng.randint(0, N)
        lo = max(0, pa + pb - N)
        pab = rng.randint(lo, min(pa, pb))
        cases.append((pa, pb, pab))
    for pa, pb, pab in cases:
        can = oracle.estimate_pair(pa, pb, pab, N, L)
        lit = oracle.estimate_literal(pa, pb, pab, N, d)[5:9]
        py = D.estimate_canonical(pa, pb, pab, N, L.tolist())
        assert can.tolist() == list(py)                         # bit-identical re-implementation
        # The literal form evaluates ln(arg) with arg = q^na + q^nb + pab/N - 1, which cancels
        # catastrophically when arg is small (e.g. a saturated sketch): its own rounding error
        # is ~ 3 eps / (arg |ln q|). Allow that conditioning on top of 1e-12 relative.
        q = 1.0 - 1.0 / N
        arg = q ** L[pa] + q ** L[pb] + pab / N - 1.0
        cond = 3 * 2.2e-16 / (max(arg, 1e-300) * abs(math.log(q))) if arg > 0 else 0.0
        for c, l_ in zip(can, lit):
            scale = max(1.0, abs(c), abs(l_))
            tol = 1e-12 * scale * max(1.0, L[pa] + L[pb]) + 20 * cond
            assert abs(c - l_) <= tol, (pa, pb, pab, can, lit)


@pytest.mark.parametrize("N", [2, 7, 1224, 4096])
def test_self_similarity_exact(N):
    """(a, a) -> IP = n_a, HAM = 0, JS = 1, COS = 1 exactly."""
    L = oracle.card_table(N, 3 * N)
    for p in range(1, N + 1):
        ip, ham, js, cs = oracle.estimate_pair(p, p, p, N, L)
        assert ip == L[p] and ham == 0.0 and js == 1.0 and cs == 1.0


def test_empty_conventions():
    L = oracle.card_table(100, 1000)
    assert oracle.estimate_pair(0, 0, 0, 100, L).tolist() == [0.0, 0.0, 1.0, 0.0]
    ip, ham, js, cs = oracle.estimate_pair(0, 7, 0, 100, L)
    assert ip == 0.0 and ham == L[7] and js == 0.0 and cs == 0.0


def test_lemma1_worked_enumerations():
    for f in golden_lines("lemma1_examples.txt"):
        d, N = int(f[0]), int(f[1])
        a = [int(x) for x in f[2].split(",")]
        b = [int(x) for x in f[3].split(",")]
        m1, m2 = oracle.enumerate_expectations(d, N, a, b)
        assert m1 == float(f[4]) and m2 == float(f[5])


def test_lemma1_exhaustive_closed_form():
    """Acceptance #1: 50 random pairs, d <= 6, N = 3, all N^d maps.

    E|a_s| = N(1 - q^|a|), E<a_s,b_s> = N(1 - q^|a| - q^|b| + q^(|a|+|b|-IP))
    (PAPER.md:361-389 with the exponent sign of its own proof, reading R-G1).
    """
    rng = random.Random(42)
    N = 3
    q = 1 - 1 / N
    for _ in range(50):
        d = rng.randint(1, 6)
        a = sorted(rng.sample(range(d), rng.randint(0, d)))
        b = sorted(rng.sample(range(d), rng.randint(0, d)))
        ip = len(set(a) & set(b))
        m1, m2 = oracle.enumerate_expectations(d, N, a, b)
        assert abs(m1 - N * (1 - q ** len(a))) < 1e-9
        assert abs(m2 - N * (1 - q ** len(a) - q ** len(b) + q ** (len(a) + len(b) - ip))) < 1e-9
        if 0 < ip:
            # the printed "+IP" exponent is refuted by enumeration
            plus = N * (1 - q ** len(a) - q ** len(b) + q ** (len(a) + len(b) + ip))
            assert abs(m2 - plus) > 1e-6


def test_occupancy_moments_balls_in_bins():
    """|a_s| is the number of non-empty bins when |a| balls go into N bins.

    Textbook: E = N(1 - q^m); Var(#empty) = N q^m + N(N-1)(1-2/N)^m - N^2 q^{2m}.
    """
    m, N, T = 100, 1224, 4000
    d = m
    indptr = np.array([0, m], dtype=np.int64)
    idx = np.arange(m, dtype=np.int32)
    vals = []
    for t in range(T):
        sk, _ = oracle.sketch(oracle.make_pi(777 + t, d, N), d, N, indptr, idx)
        vals.append(int(oracle.popcount(sk, N)[0]))
    vals = np.array(vals, dtype=np.float64)
    q = 1 - 1 / N
    mean = N * (1 - q ** m)
    var = N * q ** m + N * (N - 1) * (1 - 2 / N) ** m - N * N * q ** (2 * m)
    assert abs(vals.mean() - mean) < 4 * math.sqrt(var / T)
    assert abs(vals.var() - var) < 0.15 * var


def test_near_exact_when_N_large():
    """N >> psi^2: collisions vanish, so every estimator must approach the exact value.

    Catches a dropped term / flipped sign in Alg. 1-4 (a wrong HAM sign, R-G2, fails here).
    """
    rng = random.Random(5)
    N, d = 1 << 20, 5000
    pi = oracle.make_pi(99, d, N)
    L = oracle.card_table(N, d)
    errs = []
    for _ in range(200):
        a = sorted(rng.sample(range(d), rng.randint(1, 60)))
        b = sorted(set(rng.sample(a, rng.randint(0, len(a)))) | set(rng.sample(range(d), rng.randint(1, 60))))
        indptr = np.array([0, len(a), len(a) + len(b)], dtype=np.int64)
        sk, _ = oracle.sketch(pi, d, N, indptr, np.array(a + b, dtype=np.int32))
        pa, pb = (int(x) for x in oracle.popcount(sk, N))
        pab = int(oracle.andpopc(sk[:1], sk[1:], N)[0, 0])
        est = oracle.estimate_pair(pa, pb, pab, N, L)
        ex = oracle.exact(np.array(a), np.array(b))
        errs.append(np.abs(est - ex))
    errs = np.array(errs)
    assert errs[:, 0].max() < 0.05 and errs[:, 1].max() < 0.1
    assert errs[:, 2].max() < 0.002 and errs[:, 3].max() < 0.002


def test_concentration_lemmas_and_theorem1():
    """Acceptance #2 with readings R-G4/R-G7: psi=100, delta=rho=0.1, N=1224.

    Lemma `lemma:1`: |n_as - E|a_s|| < sqrt(psi/2 ln 2/delta) w.p. >= 1-delta.
    Lemma `lemma:2`: ||a| - n_a| < 4 sqrt(psi/2 ln 2/delta) w.p. >= 1-delta.
    Lemma `lemma:IP_estimation`: |IP - n_ab| < 14 sqrt(...) w.p. >= 1-3 delta.
    Theorem 1 with the lemma constant: 14 sqrt(psi/2 ln 6/rho) w.p. >= 1-rho.
    """
    psi, delta = 100, 0.1
    N = oracle.recommended_N(psi, delta)
    assert N == 1224
    eps = math.sqrt(psi / 2 * math.log(2 / delta))
    q = 1 - 1 / N
    for o in (0, 25, 50, 75, 100):
        E = ensemble(psi, o, N, 400, 900_000 + o)
        e_as = N * (1 - q ** psi)
        assert np.mean(np.abs(E[:, 0] - e_as) >= eps) <= delta
        assert np.mean(np.abs(E[:, 3] - psi) >= 4 * eps) <= delta
        assert np.mean(np.abs(E[:, 5] - o) >= 14 * eps) <= 3 * delta
        assert np.mean(np.abs(E[:, 5] - o) >= 14 * math.sqrt(psi / 2 * math.log(6 / delta))) <= delta
        # the bound is vacuous in practice: the much tighter eps itself holds on >= 90%
        assert np.mean(np.abs(E[:, 5] - o) >= eps) <= delta


def test_bias_regression_band():
    """the committed band (tests/golden/mc_band.json, tools/gen_mc_band.py)."""
    with open(os.path.join(GOLDEN, "mc_band.json")) as f:
        band = json.load(f)
    for o, ref in band["overlaps"].items():
        o = int(o)
        E = ensemble(band["m"], o, band["N"], band["pairs"], band["seed"] + 100_000 * o)
        err = E[:, 5] - o
        assert abs(err.mean() - ref["mean_err"]) < 1e-9
        assert abs(err.std() - ref["sd_err"]) < 1e-9
        # sanity of the band itself: unbiased except the clamp at IP=0, sd ~ 2 at N=1224
        assert abs(ref["mean_err"]) < (2.0 if o == 0 else 0.3)
        assert 1.0 < ref["sd_err"] < 3.0


def test_exact_similarities_examples():
    # SPEC.md:343
    assert oracle.exact(np.arange(5), np.arange(5)).tolist() == [5, 0, 1, 1]
    assert oracle.exact(np.array([0, 1]), np.array([2, 3, 4])).tolist() == [0, 5, 0, 0]
    ip, ham, js, cs = oracle.exact(np.array([0, 1, 2]), np.array([1, 2, 3]))
    assert (ip, ham, js) == (2, 2, 0.5) and abs(cs - 2 / 3) < 1e-15
