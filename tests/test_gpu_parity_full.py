"""Whole-output parity of the headline configuration (BASELINE.json configs[4], Large): every one
of the 200,000 top-50 lists (IP, self excluded) against the CPU oracle, in the bench's launch
configuration. About 4 CPU-minutes on 16 cores, so it runs only on request:

    BSK_FULL_PARITY=1 python -m pytest tests/test_gpu_parity_full.py -m gpu -s

(the committed log of a run: profiles/r02_parity_large_full.log).
"""
import os
import time

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1910_04658_b200 import binsketch as bs

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(os.environ.get("BSK_FULL_PARITY") != "1", reason="set BSK_FULL_PARITY=1")]


def test_full_large_every_list():
    spec, N, k = synth.LARGE, synth.LARGE_N, synth.LARGE_K
    indptr, indices = synth.make_csr(spec)
    pi = oracle.make_pi(synth.PI_SEED, spec.d, N)
    ip = torch.from_numpy(indptr).cuda()
    ix = torch.from_numpy(indices).cuda()
    sk = bs.build(bs.make_pi(synth.PI_SEED, spec.d, N), spec.d, N, ip, ix)
    gi, gs = bs.topk(sk, sk, N, spec.d, bs.IP, k, exclude_self=True)
    bs.device_status()
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    skh = sk.cpu().numpy().view(np.uint32)
    ref_sk, st = oracle.sketch(pi, spec.d, N, indptr, indices)
    assert st == 0 and np.array_equal(skh, ref_sk)
    print(f"sketches: {spec.n} rows bit-identical to the oracle", flush=True)
    bad_idx = bad_score = 0
    t0 = time.perf_counter()
    B = 10_000
    for r0 in range(0, spec.n, B):
        rows = np.arange(r0, min(spec.n, r0 + B))
        # exclude-self list of row r = its top-(k+1) over all db rows with r removed (or the first k)
        i1, s1 = oracle.topk(skh[rows], skh, N, spec.d, bs.IP, k + 1)
        keep = i1 != rows[:, None]
        ri = np.stack([i1[t][keep[t]][:k] for t in range(len(rows))])
        rs = np.stack([s1[t][keep[t]][:k] for t in range(len(rows))])
        bad_idx += int(np.sum(np.any(gi[rows] != ri, axis=1)))
        bad_score += int(np.sum(np.any(gs[rows].view(np.uint32) != rs.astype(np.float32).view(np.uint32), axis=1)))
        print(f"rows {r0}..{rows[-1]}: index lists differing so far {bad_idx}, scores differing {bad_score} "
              f"({time.perf_counter() - t0:.0f} s)", flush=True)
    print(f"RESULT: {spec.n - bad_idx}/{spec.n} top-{k} index lists identical, "
          f"{spec.n - bad_score}/{spec.n} score lists bit-identical", flush=True)
    assert bad_idx == 0 and bad_score == 0
