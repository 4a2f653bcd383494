"""Monte-Carlo ensemble over random maps pi (test infrastructure; calls only oracle/).

For each overlap o, `pairs` random maps pi (seed = base + t) are drawn and the
fixed pair a = {0..m-1}, b = {m-o .. 2m-o-1} (|a| = |b| = m, IP = o) is
sketched and estimated with the oracle. Used by tests/test_oracle_estimators.py
(concentration lemmas, Theorem 1, bias regression band) and by
tools/gen_mc_band.py, which writes tests/golden/mc_band.json.
"""
from __future__ import annotations

import numpy as np

import oracle


def ensemble(m: int, overlap: int, N: int, pairs: int, base_seed: int):
    d = 2 * m
    a = np.arange(0, m, dtype=np.int32)
    b = np.arange(m - overlap, 2 * m - overlap, dtype=np.int32)
    indptr = np.array([0, m, 2 * m], dtype=np.int64)
    idx = np.concatenate([a, b])
    L = oracle.card_table(N, d)
    rows = []
    for t in range(pairs):
        pi = oracle.make_pi(base_seed + t, d, N)
        sk, st = oracle.sketch(pi, d, N, indptr, idx)
        assert st == 0
        pa, pb = (int(x) for x in oracle.popcount(sk, N))
        pab = int(oracle.andpopc(sk[0:1], sk[1:2], N)[0, 0])
        est = oracle.estimate_pair(pa, pb, pab, N, L)
        rows.append((pa, pb, pab, L[pa], L[pb], est[0], est[1], est[2], est[3]))
    return np.array(rows, dtype=np.float64)
