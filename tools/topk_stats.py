"""Dev: epilogue statistics of the fused top-k (needs a -DBSK_TOPK_STATS variant library).
    BINSKETCH_LIB_VARIANT=variants/libbinsketch_stats.so python tools/topk_stats.py [--k K] [--measure ip]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1910_04658_b200 import binsketch as bs

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=synth.LARGE_K)
ap.add_argument("--measure", default="ip")
a = ap.parse_args()
db, N = synth.LARGE, synth.LARGE_N
ip, ix = (torch.from_numpy(x).cuda() for x in synth.make_csr(db))
D = bs.build_seeded(synth.PI_SEED, db.d, N, ip, ix)
m = bs.MEASURES[a.measure]
lib = bs._lib()
lib.bsk_topk_stats.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 16)()
bs.topk(D, D, N, db.d, m, a.k, exclude_self=True)
torch.cuda.synchronize()
lib.bsk_topk_stats(buf)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
bs.topk(D, D, N, db.d, m, a.k, exclude_self=True)
e1.record()
e1.synchronize()
lib.bsk_topk_stats(buf)
names = ["warp_tiles", "skippable_warp_tiles", "passing_chunks", "survivors", "direct_warp_tiles", "candidates",
         "epi_wait_tfull", "epi_filter", "epi_score", "epi_setup", "mma_wait_tempty", "mma_wait_full", "prod_wait_empty",
         "epi_setup_loads", "mma_total", "pmin_recomputes"]
out = {n: int(buf[i]) for i, n in enumerate(names)}
out.update(k=a.k, measure=a.measure, qsort=os.environ.get("BINSKETCH_TC_QSORT", "default"), ms=e0.elapsed_time(e1))
print(json.dumps(out), flush=True)
