"""Experiment 2 at full size on one B200: threshold-join throughput and the
paper's accuracy / precision / recall / F1 per threshold.

    python tools/bench_join.py [--steps 5] [--warmup 3] [--N 4096] [--measures js,cos]

Workload: synth.EXP2 — 101,000 rows from the Ranking corpus distribution
(d = 102,660) with 30 % planted near-duplicates, split 90/10 into 90,900 training rows (db) and
10,100 queries. Timed (CUDA events on the launching stream, L2 flushed between reps):
  sketch join  binsketch_join on the N-bit sketches, all 8 paper thresholds in one pass
  exact join   binsketch_join with BINSKETCH_JOIN_EXACT on the uncompressed rows (N = d)
Prints one JSON line per (measure, kind) and one with the Exp.-2 table.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--N", type=int, default=0)
    ap.add_argument("--measures", default="js,cos")
    ap.add_argument("--rows", type=int, default=0, help="scale the corpus down (rows)")
    ap.add_argument("--no-exact", action="store_true")
    args = ap.parse_args()

    import numpy as np
    import torch

    import synth
    from paper_1910_04658_b200 import binsketch as bs
    from paper_1910_04658_b200 import exp2

    spec = synth.EXP2 if not args.rows else synth.scaled(synth.EXP2, args.rows)
    N = args.N or synth.EXP2_N
    d = spec.d
    t0 = time.time()
    ip, ix = synth.make_csr(spec)
    ip, ix = synth.plant_near_duplicates(ip, ix, d, synth.EXP2_DUP_FRAC, synth.EXP2_DUP_SEED)
    tr, q = synth.split_rows(spec.n, 0.1, synth.EXP2_SPLIT_SEED)
    (qp, qi), (tp, ti) = synth.take_rows(ip, ix, q), synth.take_rows(ip, ix, tr)
    gen_s = time.time() - t0
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()   # noqa: E731
    qp_d, qi_d, tp_d, ti_d = dev(qp), dev(qi), dev(tp), dev(ti)
    nq, ndb = len(q), len(tr)
    Qs = bs.build_seeded(synth.PI_SEED, d, N, qp_d, qi_d)
    Ds = bs.build_seeded(synth.PI_SEED, d, N, tp_d, ti_d)
    Qx = None if args.no_exact else exp2.exact_vectors(qp_d, qi_d, d)
    Dx = None if args.no_exact else exp2.exact_vectors(tp_d, ti_d, d)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    thr = list(synth.EXP2_THRESHOLDS)
    stream = torch.cuda.current_stream()
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    int8_peak = 2.0 * pk.get("bf16_tflops_sustained", 1394.3)
    pairs = nq * ndb

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        l0 = bs.launch_count()
        ts = []
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        bs.device_status()
        return float(np.median(ts)), (bs.launch_count() - l0) // args.steps

    table = []
    for mname in args.measures.split(","):
        m = bs.MEASURES[mname]
        out_e = torch.empty((len(thr), nq, (ndb + 31) // 32), dtype=torch.int32, device="cuda")
        ws_e = torch.empty(bs.workspace_bytes(bs.OP_JOIN, nq, ndb, N), dtype=torch.uint8, device="cuda")
        t_e, l_e = timed(lambda: bs.join(Qs, Ds, N, d, m, thr, out=out_e, ws=ws_e))
        Kp = (N + 127) // 128 * 128
        line = {"kind": "sketch_join", "measure": mname, "N": N, "nq": nq, "ndb": ndb, "thresholds": thr,
                "ms": t_e * 1e3, "pairs_per_s": pairs / t_e, "launches_per_call": int(l_e),
                "roofline": {"bound": "tensor", "achieved": 2.0 * pairs * N / t_e / 1e12, "peak": int8_peak,
                             "unit": "TOPS (int8)", "frac": 2.0 * pairs * N / t_e / 1e12 / int8_peak,
                             "padded_K": Kp,
                             "time_basis": "whole binsketch_join call (popcounts, sort, expand, memset, TC join)"}}
        print(json.dumps(line), flush=True)
        if args.no_exact:
            continue
        del ws_e
        out_x = torch.empty_like(out_e)
        ws_x = torch.empty(bs.workspace_bytes(bs.OP_JOIN, nq, ndb, d), dtype=torch.uint8, device="cuda")
        t_x, l_x = timed(lambda: bs.join(Qx, Dx, d, d, m, thr, exact=True, out=out_x, ws=ws_x))
        line = {"kind": "exact_join", "measure": mname, "d": d, "nq": nq, "ndb": ndb, "ms": t_x * 1e3,
                "pairs_per_s": pairs / t_x, "launches_per_call": int(l_x),
                "roofline": {"bound": "tensor", "achieved": 2.0 * pairs * d / t_x / 1e12, "peak": int8_peak,
                             "unit": "TOPS (int8)", "frac": 2.0 * pairs * d / t_x / 1e12 / int8_peak}}
        print(json.dumps(line), flush=True)
        del ws_x
        for t in range(len(thr)):
            conf = bs.join_confusion(out_e[t], out_x[t], ndb).cpu().numpy()
            r = exp2.metrics_from_counts(conf)
            r.update({"measure": mname, "N": N, "threshold": thr[t], "O_total": int(conf[1].sum()),
                      "Oprime_total": int(conf[0].sum())})
            table.append(r)
        del out_x
    if table:
        print(json.dumps({"kind": "exp2_table", "corpus": {"rows": spec.n, "d": d, "nnz": int(ip[-1]),
                                                            "gen_s": gen_s}, "rows": table}), flush=True)


if __name__ == "__main__":
    main()
