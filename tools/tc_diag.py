"""Diagnose tensor-core AND-popcount mismatches vs the oracle (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
from paper_1910_04658_b200 import binsketch as bs

def sk(spec, N):
    ip, ix = synth.make_csr(spec)
    return oracle.sketch(oracle.make_pi(1, spec.d, N), spec.d, N, ip, ix)[0]

cases = [(1024, 128, 256, None), (1024, 256, 256, None), (1024, 128, 512, None), (1024, 129, 256, None),
         (1024, 333, 517, None), (1024, 333, 517, "1"), (1024, 256, 256, "1"), (1024, 128, 256 + 32, None),
         (1024, 128, 300, None), (1024, 128, 260, None)]
for N, na, nb, grid in cases:
    if grid: os.environ["BINSKETCH_TC_GRID"] = grid
    else: os.environ.pop("BINSKETCH_TC_GRID", None)
    A = sk(synth.scaled(synth.LARGE, na, seed=5), N); B = sk(synth.scaled(synth.LARGE, nb, seed=6), N)
    ref = oracle.andpopc(A, B, N)
    out = torch.full((na, nb), -7, dtype=torch.int32, device="cuda")
    got = bs.andpopc(torch.from_numpy(A.view(np.int32)).cuda(), torch.from_numpy(B.view(np.int32)).cuda(), N, out=out).cpu().numpy()
    bad = np.argwhere(got != ref)
    print(N, na, nb, "grid", grid, "mismatches", len(bad), "of", ref.size, "unwritten", int((got == -7).sum()))
    if len(bad):
        rows = np.unique(bad[:, 0]); cols = np.unique(bad[:, 1])
        print("  rows", rows[:24], len(rows), " cols", cols[:24], len(cols))
        for r, c in bad[:4]:
            print("  ", r, c, "got", got[r, c], "ref", ref[r, c])
