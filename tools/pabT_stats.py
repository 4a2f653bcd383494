"""Dev: counters of the pab-table top-k (needs a -DBSK_PABT_STATS variant library).
    BINSKETCH_LIB_VARIANT=variants/libbinsketch_pabt.so python tools/pabT_stats.py
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1910_04658_b200 import binsketch as bs

db, q, N, k = synth.RANKING_DB, synth.RANKING_Q, synth.RANKING_N, synth.RANKING_K
ip, ix = (torch.from_numpy(x).cuda() for x in synth.make_csr(db))
qp, qx = (torch.from_numpy(x).cuda() for x in synth.make_csr(q))
pi = bs.make_pi(synth.PI_SEED, db.d, N)
D = bs.build(pi, db.d, N, ip, ix)
Q = bs.build(pi, db.d, N, qp, qx)
lib = bs._lib()
stats = hasattr(lib, "bsk_pabt_stats")
buf = (ctypes.c_ulonglong * 16)()
if stats:
    lib.bsk_pabt_stats.argtypes = [ctypes.c_void_p]
mask = int(os.environ.get("MASK", "12"))
bs.topk(Q, D, N, db.d, mask, k)
torch.cuda.synchronize()
if stats:
    lib.bsk_pabt_stats(buf)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
bs.topk(Q, D, N, db.d, mask, k)
e1.record()
e1.synchronize()
out = {"ms": e0.elapsed_time(e1), "mask": mask}
if stats:
    lib.bsk_pabt_stats(buf)
    names = ["queries", "entries", "keys_ge_ts", "final_buf", "x4", "cyc_passA", "cyc_select", "cyc_passB", "cyc_ovf", "cyc_final", "thr_hist", "thr_select", "thr_T", "thr_suffix"]
    out.update({n: int(buf[i]) for i, n in enumerate(names)})
print(json.dumps(out), flush=True)
