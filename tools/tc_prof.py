"""One tensor-core top-k (self-join IP top-50 on a scaled Large db) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1910_04658_b200 import binsketch as bs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = synth.scaled(synth.LARGE, n)
ip, ix = synth.make_csr(spec)
pi = bs.make_pi(1, spec.d, 1024)
sk = bs.build(pi, spec.d, 1024, torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda())
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); bs.topk(sk, sk, 1024, spec.d, m, 50, exclude_self=True); e1.record(); e1.synchronize()
    print("topk ms", e0.elapsed_time(e1), flush=True)
