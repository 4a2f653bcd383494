"""Pins for the oracle's Experiment-1 sums (fidelity of the estimate; CPU only).

Independent of oracle.cpp: a pure-Python pass (set intersections for the truth, definitional
per-bit popcounts + canonical recipe for the estimate) summed in the same order (per row, then
over rows); pair counts against a dense numpy matmul; SPEC.md:413's worked arithmetic; near-exactness at huge N;
and SPEC.md:484's trend (MSE non-increasing in N, averaged over seeds).
"""
import math
import random

import numpy as np
import pytest

import oracle
import synth
from oracle import definitional as D


def _bits(row, N):
    return [(int(row[j // 32]) >> (j % 32)) & 1 for j in range(N)]


def _corpus(n, d, seed, lo=10, hi=40, frac=0.5):
    ip, ix = synth.make_csr(synth.CSRSpec(n=n, d=d, kind=0, p1=lo, p2=hi, cap=hi, zipf_s=1.05, seed=seed))
    return synth.plant_near_duplicates(ip, ix, d, frac, seed=seed + 1)


@pytest.mark.parametrize("measure", [1, 2, 4, 8])
@pytest.mark.parametrize("bcs", [False, True])
def test_mse_vs_python(measure, bcs):
    d, N, n = 300, 64, 25
    ip, ix = _corpus(n, d, seed=3 + measure)
    pi = oracle.make_pi(2, d, N)
    S, _ = (oracle.bcs_sketch if bcs else oracle.sketch)(pi, d, N, ip, ix)
    thr = {1: [1.0, 5.0, 12.0], 2: [5.0, 20.0, 60.0], 4: [0.2, 0.5, 0.9], 8: [0.3, 0.6, 0.95]}[measure]
    sse, cnt = oracle.mse(S, N, d, ip, ix, measure, thr, bcs=bcs)
    T = D.bcs_table(N, d) if bcs else D.card_table(N, d)
    rows = [set(ix[ip[i]:ip[i + 1]].tolist()) for i in range(n)]
    bits = [_bits(S[i], N) for i in range(n)]
    k = {1: 0, 2: 1, 4: 2, 8: 3}[measure]
    want_s = [0.0] * len(thr)
    want_c = [0] * len(thr)
    for i in range(n):
        row_s = [0.0] * len(thr)              # summation order: per row over j, then over rows
        for j in range(i + 1, n):
            a, b = rows[i], rows[j]
            inter = len(a & b)
            tru = [float(inter), float(len(a) + len(b) - 2 * inter),
                   inter / len(a | b) if a | b else 1.0,
                   inter / math.sqrt(len(a) * len(b)) if a and b else 0.0][k]
            pa, pb = sum(bits[i]), sum(bits[j])
            if bcs:
                est = D.bcs_estimate(pa, pb, sum(x ^ y for x, y in zip(bits[i], bits[j])), d, T)[k]
            else:
                est = D.estimate_canonical(pa, pb, D.and_popcount_bits(bits[i], bits[j]), N, T)[k]
            for t, th in enumerate(thr):
                if (tru <= th) if measure == 2 else (tru >= th):
                    row_s[t] += (est - tru) * (est - tru)
                    want_c[t] += 1
        for t in range(len(thr)):
            want_s[t] += row_s[t]
    assert list(cnt) == want_c
    assert all(s == w for s, w in zip(sse, want_s)), (sse, want_s)
    assert want_c[0] > 0


def test_mse_counts_vs_dense_matmul():
    d, n = 2000, 120
    ip, ix = _corpus(n, d, seed=41)
    X = np.zeros((n, d), dtype=np.int64)
    for i in range(n):
        X[i, ix[ip[i]:ip[i + 1]]] = 1
    G = (X @ X.T).astype(np.float64)
    sz = X.sum(1).astype(np.float64)
    js = G / (sz[:, None] + sz[None, :] - G)
    iu = np.triu_indices(n, 1)
    pi = oracle.make_pi(1, d, 512)
    S, _ = oracle.sketch(pi, d, 512, ip, ix)
    thr = [0.95, 0.8, 0.5, 0.2, 0.0]
    _, cnt = oracle.mse(S, 512, d, ip, ix, 4, thr)
    assert [int(c) for c in cnt] == [int(np.count_nonzero(js[iu] >= t)) for t in thr]
    assert cnt[-1] == n * (n - 1) // 2


def test_mse_report_spec_example():
    r = oracle.mse_report(np.array([0.1 ** 2 + 0.2 ** 2]), np.array([2], dtype=np.uint64), 4)[0]
    assert math.isclose(r["mse"], 0.025) and math.isclose(r["neg_log_mse"], 3.6888794541139363)
    assert oracle.mse_report(np.array([0.0]), np.array([0], dtype=np.uint64), 4) == [None]   # empty set: absent
    assert "neg_log_mse" not in oracle.mse_report(np.array([4.0]), np.array([2], dtype=np.uint64), 1)[0]   # IP: raw


def test_mse_near_zero_at_huge_N():
    d, n = 100_000, 60
    ip, ix = _corpus(n, d, seed=7, lo=10, hi=30)
    N = 1 << 20
    S, _ = oracle.sketch(oracle.make_pi(5, d, N), d, N, ip, ix)
    sse, cnt = oracle.mse(S, N, d, ip, ix, 4, [0.0])
    assert cnt[0] == n * (n - 1) // 2 and sse[0] / cnt[0] < 1e-6


def test_mse_trend_in_N():
    """SPEC.md:484 (reduced): mean JS MSE over seeds at threshold 0.5 is non-increasing in N,
    allowing one adjacent inversion within one standard error."""
    d = 10_000
    Ns = [256, 512, 1024, 2048, 4096]
    per_N = {N: [] for N in Ns}
    for seed in range(8):
        ip, ix = _corpus(150, d, seed=100 + 10 * seed, lo=60, hi=140, frac=0.6)
        for N in Ns:
            S, _ = oracle.sketch(oracle.make_pi(seed + 1, d, N), d, N, ip, ix)
            sse, cnt = oracle.mse(S, N, d, ip, ix, 4, [0.5])
            assert cnt[0] > 0
            per_N[N].append(sse[0] / cnt[0])
    means = [np.mean(per_N[N]) for N in Ns]
    ses = [np.std(per_N[N], ddof=1) / np.sqrt(len(per_N[N])) for N in Ns]
    inversions = [(a, b) for a, b in zip(range(len(Ns)), range(1, len(Ns))) if means[b] > means[a]]
    assert len(inversions) <= 1
    for a, b in inversions:
        assert means[b] - means[a] <= ses[a] + ses[b]
    assert means[-1] < means[0] / 4
