"""Single-launch targets for ncu captures (run the same command without ncu first).
    python tools/ncu_targets.py build_table | estimate_medium_cuda
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
torch.cuda.synchronize()
bs.device_status()
print("ok", what)
