"""Experiment 1 of the paper (fidelity of the estimate) on the GPU path.

Per (measure, N): sketches by binsketch_build_seeded (or binsketch_bcs_build_seeded for the BCS
comparison), the uncompressed rows by binsketch_build with the identity map, and the squared-error
sums over the pairs whose exact similarity reaches each threshold by binsketch_mse (tensor-core
AND-popcount tables + a fixed-order fp64 reduction). The host only divides: MSE = sse / count,
reported as -ln(MSE) for JS / COS and as is for IP. Product code: no oracle import.
"""
from __future__ import annotations

import math

import torch

from . import binsketch as bs
from .exp2 import exact_vectors

PAPER_THRESHOLDS = (0.95, 0.9, 0.85, 0.8, 0.6, 0.5, 0.2, 0.1)


def fidelity(indptr: torch.Tensor, indices: torch.Tensor, d: int, N: int, measure: int,
             thresholds=PAPER_THRESHOLDS, pi_seed: int = 1, bcs: bool = False, exact: torch.Tensor | None = None):
    S = (bs.bcs_build_seeded if bcs else bs.build_seeded)(pi_seed, d, N, indptr, indices)
    X = exact if exact is not None else exact_vectors(indptr, indices, d)
    sse, cnt = bs.mse(S, X, N, d, measure, list(thresholds), bcs=bcs)
    sse, cnt = sse.cpu().tolist(), cnt.cpu().tolist()
    out = []
    for t, s, c in zip(thresholds, sse, cnt):
        r = {"threshold": t, "pairs": int(c), "sse": s}
        if c:
            r["mse"] = s / c
            if measure in (bs.JS, bs.COS):
                r["neg_log_mse"] = -math.log(r["mse"]) if r["mse"] > 0 else math.inf
        out.append(r)
    return out
