"""Dev: fused tensor-core vs CUDA-core top-k for query-vs-db shapes under the small-call threshold."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1910_04658_b200 import binsketch as bs

db_spec = synth.scaled(synth.LARGE, 100_000, seed=7)
ip, ix = (torch.from_numpy(x).cuda() for x in synth.make_csr(db_spec))
Dall = bs.build_seeded(synth.PI_SEED, db_spec.d, 1024, ip, ix)
for nq, ndb, m, k in [(100, 100_000, bs.IP, 10), (100, 100_000, bs.JS, 10), (300, 100_000, bs.IP, 50),
                      (1000, 30_000, bs.IP, 50), (1000, 30_000, bs.JS, 10), (30, 100_000, bs.COS, 64)]:
    Q, D = Dall[:nq].clone(), Dall[:ndb]
    res = {}
    for eng in ("tc", "cuda"):
        os.environ["BINSKETCH_ENGINE"] = eng
        for _ in range(3):
            o = bs.topk(Q, D, 1024, db_spec.d, m, k)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); o = bs.topk(Q, D, 1024, db_spec.d, m, k); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        res[eng] = (ts[5], o[0].cpu())
    print(json.dumps({"nq": nq, "ndb": ndb, "measure": int(m), "k": k, "tc_ms": res["tc"][0], "cuda_ms": res["cuda"][0],
                      "identical_lists": torch.equal(res["tc"][1], res["cuda"][1])}), flush=True)
