"""Dev: fused tensor-core top-k vs the CUDA-core top-k on small self-joins (the engine crossover).
    python tools/topk_engine_sweep.py  -> one JSON line per (n, N, measure, k, engine)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1910_04658_b200 import binsketch as bs

for n, N, spec, m, k in [(1000, 1224, synth.TINY, bs.JS, 10), (2000, 1224, synth.TINY, bs.JS, 10),
                         (4000, 1224, synth.TINY, bs.JS, 10), (8000, 1224, synth.TINY, bs.JS, 10),
                         (1000, 1024, synth.LARGE, bs.IP, 50), (4000, 1024, synth.LARGE, bs.IP, 50),
                         (16000, 1024, synth.LARGE, bs.IP, 50), (32000, 1024, synth.LARGE, bs.IP, 50)]:
    sp = synth.scaled(spec, n, seed=5)
    ip, ix = (torch.from_numpy(x).cuda() for x in synth.make_csr(sp))
    D = bs.build_seeded(synth.PI_SEED, sp.d, N, ip, ix)
    res = {}
    for eng in ("tc", "cuda"):
        os.environ["BINSKETCH_ENGINE"] = eng
        out = None
        for _ in range(3):
            out = bs.topk(D, D, N, sp.d, m, k, exclude_self=True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); o = bs.topk(D, D, N, sp.d, m, k, exclude_self=True); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        res[eng] = (ts[len(ts) // 2], o[0].cpu())
    same = torch.equal(res["tc"][1], res["cuda"][1])
    print(json.dumps({"n": n, "N": N, "measure": int(m), "k": k, "tc_ms": res["tc"][0], "cuda_ms": res["cuda"][0],
                      "identical_lists": same}), flush=True)
