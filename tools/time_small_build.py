"""Dev: build time of Ranking's query set (1000 rows) and db (100,000 rows) per pi source."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1910_04658_b200 import binsketch as bs
N = synth.RANKING_N
for name, spec in (("queries", synth.RANKING_Q), ("db", synth.RANKING_DB)):
    ip, ix = (torch.from_numpy(x).cuda() for x in synth.make_csr(spec))
    pi = bs.make_pi(synth.PI_SEED, spec.d, N)
    for mode in ("auto", "global", "cache"):
        if mode == "auto": os.environ.pop("BINSKETCH_BUILD_MODE", None)
        else: os.environ["BINSKETCH_BUILD_MODE"] = mode
        out = bs.build(pi, spec.d, N, ip, ix)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): bs.build(pi, spec.d, N, ip, ix, out=out)
        e1.record(); e1.synchronize()
        print(json.dumps({"set": name, "rows": spec.n, "mode": mode, "ms": e0.elapsed_time(e1) / 20}), flush=True)
