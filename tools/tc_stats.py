import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1910_04658_b200 import binsketch as bs
os.environ["BINSKETCH_TC_STATS"] = "1"
spec = synth.scaled(synth.LARGE, int(sys.argv[1]) if len(sys.argv) > 1 else 20000)
ip, ix = synth.make_csr(spec)
pi = bs.make_pi(1, spec.d, 1024)
sk = bs.build(pi, spec.d, 1024, torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda())
for m in (1, 4):
    bs.topk(sk, sk, 1024, spec.d, m, 50, exclude_self=True)
    torch.cuda.synchronize()
