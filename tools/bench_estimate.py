"""All-pairs estimation on configs[1] (Medium: 1e4 x 1e4 pairs, 4 planes) — BinSketch on the
tensor-core and CUDA-core engines, and BCS — with sampled parity against the oracle.

    python tools/bench_estimate.py [--iters 10] [--Ns 1000,2000,5000]

Algorithmic bytes per call = 16 B per pair written (4 float planes) + the sketches read;
the write stream is the HBM bound (1.6 GB -> 0.25 ms at 6.5 TB/s).
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
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--Ns", default="1000,2000,5000")
a = ap.parse_args()
spec = synth.MEDIUM
ip_h, ix_h = synth.make_csr(spec)
n, d = spec.n, spec.d
ip, ix = torch.from_numpy(ip_h).cuda(), torch.from_numpy(ix_h).cuda()
pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = pk.get("hbm_gbs", 6530.3)
rng = np.random.default_rng(0)
rows = np.sort(rng.choice(n, 64, replace=False))
cols = np.sort(rng.choice(n, 64, replace=False))
for N in [int(x) for x in a.Ns.split(",")]:
    W = (N + 31) // 32
    pi_h = oracle.make_pi(synth.PI_SEED, d, N)
    pi = bs.make_pi(synth.PI_SEED, d, N)
    out = torch.empty((4, n, n), dtype=torch.float32, device="cuda")
    for kind in ("binsketch-pab", "binsketch-tc", "binsketch-cuda", "bcs-pab", "bcs-tc"):
        # pab: tensor-core AND-popcount table + elementwise recipe kernel; tc: the fused epilogue
        os.environ["BINSKETCH_ENGINE"] = "cuda" if kind == "binsketch-cuda" else "tc"
        os.environ["BINSKETCH_EST_PAB"] = "1" if kind.endswith("pab") else "0"
        bcs = kind.startswith("bcs")
        sk = (bs.bcs_build if bcs else bs.build)(pi, d, N, ip, ix)
        op = bs.OP_BCS_ESTIMATE if bcs else bs.OP_ESTIMATE
        ws = torch.empty(max(1, bs.workspace_bytes(op, n, n, N)), dtype=torch.uint8, device="cuda")
        est = bs.bcs_estimate if bcs else bs.estimate
        fn = lambda: est(sk, sk, N, d, 15, out=out, ws=ws)   # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        bs.device_status()
        t = statistics.median(ts)
        # sampled parity: 64 x 64 block against the oracle
        sub = lambda idx: (np.concatenate([[0], np.cumsum(ip_h[idx + 1] - ip_h[idx])]).astype(np.int64),   # noqa: E731
                           np.concatenate([ix_h[ip_h[r]:ip_h[r + 1]] for r in idx]))
        ska, _ = (oracle.bcs_sketch if bcs else oracle.sketch)(pi_h, d, N, *sub(rows))
        skb, _ = (oracle.bcs_sketch if bcs else oracle.sketch)(pi_h, d, N, *sub(cols))
        ref = (oracle.bcs_estimate if bcs else oracle.estimate)(ska, skb, N, d, 15)
        got = out[:, torch.from_numpy(rows).cuda()][:, :, torch.from_numpy(cols).cuda()].cpu().numpy()
        ok = bool(np.array_equal(got.view(np.uint32), ref.view(np.uint32)))
        byts = 16.0 * n * n + 2 * 4.0 * W * n
        print(json.dumps({"config": "medium", "N": N, "kind": kind, "ms": t * 1e3, "pairs_per_s": n * n / t,
                          "out_GBps": byts / t / 1e9, "frac_hbm": byts / t / 1e9 / hbm,
                          "int8_TOPS": 2.0 * n * n * N / t / 1e12, "parity_sampled_64x64": ok}), flush=True)
        del ws
