"""Experiment 1 at configs[1] (Medium) size on one B200: binsketch_mse timing and
the -ln(MSE) table for BinSketch and BCS per N and threshold.

    python tools/bench_mse.py [--Ns 1000,2000,5000] [--measures js,cos,ip] [--rows 10000]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1910_04658_b200 import binsketch as bs
from paper_1910_04658_b200 import exp1, exp2

ap = argparse.ArgumentParser()
ap.add_argument("--Ns", default="1000,2000,5000")
ap.add_argument("--measures", default="js,cos,ip")
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
spec = synth.MEDIUM if not a.rows else synth.scaled(synth.MEDIUM, a.rows)
ip_h, ix_h = synth.make_csr(spec)
ip_h, ix_h = synth.plant_near_duplicates(ip_h, ix_h, spec.d, 0.3, seed=12)
d, n = spec.d, spec.n
ip, ix = torch.from_numpy(ip_h).cuda(), torch.from_numpy(ix_h).cuda()
X = exp2.exact_vectors(ip, ix, d)
thr_rel = exp1.PAPER_THRESHOLDS
maxip = None
for mname in a.measures.split(","):
    m = bs.MEASURES[mname]
    if m == bs.IP:
        if maxip is None:
            # largest exact IP over pairs i != j (R-J3 style thresholds for IP)
            best = 0
            for r0 in range(0, n, 2048):
                P = bs.andpopc(X[r0:r0 + 2048], X, d)
                idx = torch.arange(P.shape[0], device="cuda")
                P[idx, idx + r0] = 0
                best = max(best, int(P.max().item()))
                del P
            maxip = best
        thr = [t * maxip for t in thr_rel]
    else:
        thr = list(thr_rel)
    for N in [int(x) for x in a.Ns.split(",")]:
        for bcs in (False, True):
            S = (bs.bcs_build_seeded if bcs else bs.build_seeded)(synth.PI_SEED, d, N, ip, ix)
            ws = torch.empty(bs.workspace_bytes(bs.OP_MSE, n, d, N), dtype=torch.uint8, device="cuda")
            fn = lambda: bs.mse(S, X, N, d, m, thr, bcs=bcs, ws=ws)   # noqa: E731
            fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); sse, cnt = fn(); e1.record(); e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            bs.device_status()
            t = statistics.median(ts)
            sse, cnt = sse.cpu().numpy(), cnt.cpu().numpy()
            rows = []
            for th, s, c in zip(thr, sse, cnt):
                r = {"t": th, "pairs": int(c)}
                if c:
                    r["mse"] = float(s / c)
                    if m != bs.IP:
                        r["neg_log_mse"] = float(-np.log(s / c)) if s > 0 else None
                rows.append(r)
            pairs = n * (n - 1) // 2
            print(json.dumps({"config": "medium", "n": n, "d": d, "N": N, "measure": mname,
                              "sketch": "bcs" if bcs else "binsketch", "ms": t * 1e3,
                              "pairs_per_s": pairs / t, "rows": rows}), flush=True)
            del ws
