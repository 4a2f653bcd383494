"""A/B timing of the pair engines (tensor-core kind::i8 vs CUDA-core POPC) on andpopc.
    python tools/bench_pairs.py
"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1910_04658_b200 import binsketch as bs

def run(N, na, nb, engine, iters=5):
    os.environ["BINSKETCH_ENGINE"] = engine
    W = (N + 31) // 32
    g = torch.Generator(device="cuda").manual_seed(N)
    A = torch.randint(-2**31, 2**31 - 1, (na, W), dtype=torch.int32, device="cuda", generator=g)
    B = torch.randint(-2**31, 2**31 - 1, (nb, W), dtype=torch.int32, device="cuda", generator=g)
    out = torch.empty((na, nb), dtype=torch.int32, device="cuda")
    ws = torch.empty(max(1, bs.workspace_bytes(bs.OP_ANDPOPC, na, nb, N)), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        bs.andpopc(A, B, N, out=out, ws=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); bs.andpopc(A, B, N, out=out, ws=ws); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = statistics.median(ts)
    kp = ((N + 127) // 128) * 128
    chk = int(out[na // 3, nb // 5].item())
    return {"N": N, "na": na, "nb": nb, "engine": engine, "ms": t * 1e3, "pairs_per_s": na * nb / t,
            "int8_TOPS": 2.0 * na * nb * kp / t / 1e12, "out_GBps": na * nb * 4 / t / 1e9, "check": chk}

for (N, na, nb) in [(1024, 16384, 16384), (8192, 8192, 8192), (4096, 1024, 100000)]:
    r = [run(N, na, nb, e) for e in ("tc", "cuda")]
    assert r[0]["check"] == r[1]["check"]
    for x in r:
        print(json.dumps(x), flush=True)
