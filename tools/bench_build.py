"""Build-kernel A/B timing on configs[3] (Build-only) and friends; parity-checks sampled rows.
    python tools/bench_build.py [--config buildonly|large|ranking|medium] [--modes global,cache,seeded,auto]
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
ap.add_argument("--config", default="buildonly")
ap.add_argument("--modes", default="auto,global,cache,seeded")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--bcs", action="store_true", help="BCS parity sketch (XOR) instead of BinSketch (OR)")
ap.add_argument("--perm", type=int, default=1,
                help="1: seeded Zipf rank -> id permutation (default); 0: identity (hot ids first: the "
                     "cache-sensitivity row of SURVEY.md 8(d))")
a = ap.parse_args()
spec, N = {"buildonly": (synth.BUILD_ONLY, synth.BUILD_ONLY_N), "large": (synth.LARGE, synth.LARGE_N),
           "ranking": (synth.RANKING_DB, synth.RANKING_N), "medium": (synth.MEDIUM, 1000)}[a.config]
import dataclasses
spec = dataclasses.replace(spec, perm=a.perm)
ip_h, ix_h = synth.make_csr(spec)
n, d, W, nnz = spec.n, spec.d, (N + 31) // 32, int(ip_h[-1])
ip, ix = torch.from_numpy(ip_h).cuda(), torch.from_numpy(ix_h).cuda()
pi = bs.make_pi(synth.PI_SEED, d, N)
out = torch.empty((n, W), dtype=torch.int32, device="cuda")
alg = 4 * nnz + 8 * (n + 1) + 4 * W * n + 4 * d
rows = np.sort(np.random.default_rng(0).choice(n, min(n, 5000), replace=False))
sub_ptr = np.zeros(len(rows) + 1, dtype=np.int64)
sub_ptr[1:] = np.cumsum(ip_h[rows + 1] - ip_h[rows])
sub_idx = np.concatenate([ix_h[ip_h[r]:ip_h[r + 1]] for r in rows])
ref, _ = (oracle.bcs_sketch if a.bcs else oracle.sketch)(oracle.make_pi(synth.PI_SEED, d, N), d, N, sub_ptr, sub_idx)
build_t, build_s = (bs.bcs_build, bs.bcs_build_seeded) if a.bcs else (bs.build, bs.build_seeded)
for mode in a.modes.split(","):
    if mode in ("global", "cache", "smem16"):
        os.environ["BINSKETCH_BUILD_MODE"] = mode
    else:
        os.environ.pop("BINSKETCH_BUILD_MODE", None)
    fn = (lambda: build_s(synth.PI_SEED, d, N, ip, ix, out=out)) if mode == "seeded" else \
         (lambda: build_t(pi, d, N, ip, ix, out=out))
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    bs.device_status()
    ok = np.array_equal(out[torch.from_numpy(rows).cuda()].cpu().numpy().view(np.uint32), ref)
    t = statistics.median(ts)
    print(json.dumps({"config": a.config, "perm": a.perm, "sketch": "bcs" if a.bcs else "binsketch", "mode": mode, "ms": t * 1e3, "rows_per_s": n / t,
                      "alg_GBps": alg / t / 1e9, "frac_hbm_6555": alg / t / 6555.2e9, "parity_sampled": ok}), flush=True)
