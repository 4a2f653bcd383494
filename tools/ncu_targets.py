"""Single-launch targets for ncu captures (run the same command without ncu first).
    python tools/ncu_targets.py build_table | estimate_medium_cuda | join_exact
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1910_04658_b200 import binsketch as bs

what = sys.argv[1]
if what == "build_table":
    spec, N = synth.BUILD_ONLY, synth.BUILD_ONLY_N
    ip, ix = synth.make_csr(spec)
    ipd, ixd = torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda()
    pi = bs.make_pi(synth.PI_SEED, spec.d, N)
    out = torch.empty((spec.n, bs.words(N)), dtype=torch.int32, device="cuda")
    for _ in range(2):
        bs.build(pi, spec.d, N, ipd, ixd, out=out)
elif what == "estimate_medium_cuda":
    spec, N = synth.MEDIUM, 1000
    ip, ix = synth.make_csr(spec)
    sk = bs.build_seeded(synth.PI_SEED, spec.d, N, torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda())
    out = torch.empty((4, spec.n, spec.n), dtype=torch.float32, device="cuda")
    for _ in range(2):
        bs.estimate(sk, sk, N, spec.d, 15, out=out)
elif what == "join_exact":   # Exp. 2 ground truth: exact rows (identity map, N = d), CTA-pair engine
    spec = synth.EXP2
    ip, ix = synth.make_csr(spec)
    ip, ix = synth.plant_near_duplicates(ip, ix, spec.d, synth.EXP2_DUP_FRAC, seed=synth.EXP2_DUP_SEED)
    tr, q = synth.split_rows(spec.n, 0.1, seed=synth.EXP2_SPLIT_SEED)
    (qp, qx), (tp, tx) = synth.take_rows(ip, ix, q), synth.take_rows(ip, ix, tr)
    from paper_1910_04658_b200 import exp2
    Q = exp2.exact_vectors(torch.from_numpy(qp).cuda(), torch.from_numpy(qx).cuda(), spec.d)
    D = exp2.exact_vectors(torch.from_numpy(tp).cuda(), torch.from_numpy(tx).cuda(), spec.d)
    for _ in range(2):
        bs.join(Q, D, spec.d, spec.d, bs.JS, list(synth.EXP2_THRESHOLDS), exact=True)
torch.cuda.synchronize()
bs.device_status()
print("ok", what)
