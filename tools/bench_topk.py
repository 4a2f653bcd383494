"""Top-k / estimate kernel timing on a BASELINE config (sketches built on the GPU).
    python tools/bench_topk.py [--config large|ranking|medium1000|medium2000|medium5000] [--iters K] [--rows R]
--rows R limits the queries (all db rows kept) for quick ncu captures.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1910_04658_b200 import binsketch as bs

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--k", type=int, default=0, help="override k (top-k configs)")
ap.add_argument("--measure", default="", help="override the measure: ip | ham | js | cos")
a = ap.parse_args()

if a.config == "large":
    db, q, N, k, m, excl = synth.LARGE, None, synth.LARGE_N, synth.LARGE_K, bs.IP, True
elif a.config == "ranking":
    db, q, N, k, m, excl = synth.RANKING_DB, synth.RANKING_Q, synth.RANKING_N, synth.RANKING_K, bs.JS, False
else:
    db, q, N, k, m, excl = synth.MEDIUM, None, int(a.config[6:]), 0, 15, False
ip, ix = (torch.from_numpy(x).cuda() for x in synth.make_csr(db))
D = bs.build_seeded(synth.PI_SEED, db.d, N, ip, ix)
if q is not None:
    qp, qx = (torch.from_numpy(x).cuda() for x in synth.make_csr(q))
    Q = bs.build_seeded(synth.PI_SEED, db.d, N, qp, qx)
else:
    Q = D
if a.k and k:
    k = a.k
if a.measure:
    m = {"ip": bs.IP, "ham": bs.HAM, "js": bs.JS, "cos": bs.COS}[a.measure]
if a.rows:
    Q = Q[: a.rows]
nq, ndb, W = Q.shape[0], D.shape[0], (N + 31) // 32
if k:
    ws = torch.empty(max(1, bs.workspace_bytes(bs.OP_TOPK, nq, ndb, N, k)), dtype=torch.uint8, device="cuda")
    oi = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    osc = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    fn = lambda: bs.topk(Q, D, N, db.d, m, k, exclude_self=excl, out_idx=oi, out_score=osc, ws=ws)
else:
    ws = torch.empty(max(1, bs.workspace_bytes(bs.OP_ESTIMATE, nq, ndb, N)), dtype=torch.uint8, device="cuda")
    out = torch.empty((4, nq, ndb), dtype=torch.float32, device="cuda")
    fn = lambda: bs.estimate(Q, D, N, db.d, 15, out=out, ws=ws)
for _ in range(a.warmup):
    fn()
torch.cuda.synchronize()
ts = []
for _ in range(a.iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e-3)
bs.device_status()
t = statistics.median(ts)
pairs = nq * ndb
print(json.dumps({"config": a.config, "nq": nq, "ndb": ndb, "N": N, "k": k, "ms": t * 1e3, "pairs_per_s": pairs / t,
                  "word_ops_per_s": pairs * W / t,
                  "frac_popc16_1965": pairs * W / t / (148 * 16 * 1.965e9),
                  "frac_k9_24p1_1965": pairs * W / t / (148 * 24.1 * 1.965e9)}), flush=True)
