"""Categorical extension on one B200: one-hot encoding + sketch build throughput and
the estimated categorical distance (HAM^/2) all-pairs throughput, with sampled parity.

    python tools/bench_categorical.py [--rows 2000000] [--cols 32] [--N 1024]

Workload: a seeded label-encoded table (synth.make_categorical) with 32 columns of cardinalities
2 .. 1000 (d = sum of cardinalities), 30 % near-duplicate rows.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import synth
from paper_1910_04658_b200 import binsketch as bs

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=2_000_000)
ap.add_argument("--cols", type=int, default=32)
ap.add_argument("--N", type=int, default=1024)
ap.add_argument("--pairs_rows", type=int, default=10_000)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
rng = np.random.default_rng(0)
cards = np.unique(np.geomspace(2, 1000, a.cols).astype(np.int64))
cards = np.concatenate([cards, rng.integers(2, 1000, a.cols - len(cards))])[: a.cols]
X = synth.make_categorical(a.rows, cards, seed=5)
off = np.zeros(len(cards) + 1, dtype=np.int64)
off[1:] = np.cumsum(cards)
d, n, c, N = int(off[-1]), a.rows, len(cards), a.N
Xd, offd = torch.from_numpy(X).cuda(), torch.from_numpy(off).cuda()
indptr = torch.empty(n + 1, dtype=torch.int64, device="cuda")
indices = torch.empty(n * c, dtype=torch.int32, device="cuda")
out = torch.empty((n, bs.words(N)), dtype=torch.int32, device="cuda")


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return statistics.median(ts)


def onehot_build():
    lib = bs._lib()
    bs._check("binsketch_onehot", lib.binsketch_onehot(bs._dev(Xd, torch.int32, "codes"), n, c,
                                                       bs._dev(offd, torch.int64, "offsets"),
                                                       bs._dev(indptr, torch.int64, "indptr"),
                                                       bs._dev(indices, torch.int32, "indices"), bs._stream()))
    bs.build_seeded(synth.PI_SEED, d, N, indptr, indices, out=out)


t_b = timed(onehot_build, a.iters)
bs.device_status()
# bytes: codes read (4 B x c), indices written + read (4 B x c), indptr (8 B), sketch written (4 W)
alg = n * (4 * c + 4 * c * 2 + 8 + 4 * bs.words(N))
rows = np.sort(rng.choice(n, 500, replace=False))
ipo, ixo, _, _ = oracle.onehot(X[rows], cards)
ref, _ = oracle.sketch(oracle.make_pi(synth.PI_SEED, d, N), d, N, ipo, ixo)
ok = bool(np.array_equal(out[torch.from_numpy(rows).cuda()].cpu().numpy().view(np.uint32), ref))
print(json.dumps({"kind": "onehot+build", "rows": n, "cols": c, "d": d, "N": N, "ms": t_b * 1e3, "rows_per_s": n / t_b,
                  "GBps": alg / t_b / 1e9, "parity_sampled_500": ok}), flush=True)
m = a.pairs_rows
S = out[:m]
res = torch.empty((m, m), dtype=torch.float32, device="cuda")
ws = torch.empty(bs.workspace_bytes(bs.OP_BCS_ESTIMATE, m, m, N), dtype=torch.uint8, device="cuda")
t_e = timed(lambda: bs.categorical_estimate(S, S, N, d, out=res, ws=ws), a.iters)
sub = rows[rows < m][:32] if (rows < m).any() else np.arange(32)
sk = out[:m].cpu().numpy().view(np.uint32)
refc = oracle.categorical_estimate(sk[sub], sk, N, d)
okc = bool(np.array_equal(res[torch.from_numpy(sub).cuda()].cpu().numpy().view(np.uint32), refc.view(np.uint32)))
Dm = oracle.categorical_distance(X[sub], X[:m])
print(json.dumps({"kind": "categorical_estimate", "rows": m, "pairs": m * m, "ms": t_e * 1e3,
                  "pairs_per_s": m * m / t_e, "out_GBps": 4.0 * m * m / t_e / 1e9, "parity_sampled_rows": okc,
                  "mean_abs_err_vs_true_D": float(np.mean(np.abs(refc - Dm)))}), flush=True)
