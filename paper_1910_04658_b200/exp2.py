"""Experiment 2 of the paper (ranking by threshold) on the GPU path.

Every per-pair step runs in the library's kernels through the C ABI:
  sketches        binsketch_build_seeded (or binsketch_build with a pi table)
  exact vectors   binsketch_build with the identity map and N = d (the uncompressed rows)
  O', O           binsketch_join on the sketches / with BINSKETCH_JOIN_EXACT on the exact vectors
  |O'|,|O|,|O∩O'| binsketch_join_confusion
The host only turns the per-query counts into the paper's ratios (reading R-J2) and, for
inner product, picks the thresholds from the maximum exact IP (R-J3, a protocol parameter).
Product code: no oracle import; no CPU fallback.
"""
from __future__ import annotations

import numpy as np
import torch

from . import binsketch as bs

PAPER_THRESHOLDS = (0.95, 0.9, 0.85, 0.8, 0.6, 0.5, 0.2, 0.1)


def identity_pi(d: int) -> torch.Tensor:
    """The identity map [d] -> [d]: building with it (N = d) yields the uncompressed bit vectors."""
    return torch.arange(d, dtype=torch.int32, device="cuda")


def exact_vectors(indptr: torch.Tensor, indices: torch.Tensor, d: int) -> torch.Tensor:
    out = torch.empty((indptr.numel() - 1, bs.words(d)), dtype=torch.int32, device="cuda")
    return bs.build(identity_pi(d), d, d, indptr, indices, out=out)


def metrics_from_counts(conf: np.ndarray) -> dict:
    """conf int64 [3][nq] = |O'|, |O|, |O' ∩ O| -> macro-averaged accuracy / precision /
    recall / F1 over queries with O ∪ O' non-empty (R-J2)."""
    est, tru, both = (np.asarray(conf[i], dtype=np.float64) for i in range(3))
    union = est + tru - both
    use = union > 0
    n = int(use.sum())
    if n == 0:
        return {"accuracy": float("nan"), "precision": float("nan"), "recall": float("nan"), "f1": float("nan"),
                "query_count": 0, "skipped_queries": int(len(union))}
    e, t, b, u = est[use], tru[use], both[use], union[use]
    p = np.where(e > 0, b / np.where(e > 0, e, 1), 0.0)
    r = np.where(t > 0, b / np.where(t > 0, t, 1), 0.0)
    f1 = np.where(p + r > 0, 2 * p * r / np.where(p + r > 0, p + r, 1), 0.0)
    return {"accuracy": float(np.mean(b / u)), "precision": float(np.mean(p)), "recall": float(np.mean(r)),
            "f1": float(np.mean(f1)), "query_count": n, "skipped_queries": int(len(union) - n)}


def max_exact_ip(Qx: torch.Tensor, Dx: torch.Tensor, d: int, block: int = 2048) -> int:
    """Largest |a ∩ b| over query x training pairs (R-J3), via binsketch_andpopc on the exact vectors."""
    best = 0
    ws = None
    for q0 in range(0, Qx.shape[0], block):
        q = Qx[q0:q0 + block]
        ws = torch.empty(max(1, bs.workspace_bytes(bs.OP_ANDPOPC, q.shape[0], Dx.shape[0], d)), dtype=torch.uint8,
                         device="cuda") if ws is None or q.shape[0] != block else ws
        best = max(best, int(bs.andpopc(q, Dx, d, ws=ws).max().item()))
    return best


def ranking(train: tuple, query: tuple, d: int, N: int, measure: int, thresholds=PAPER_THRESHOLDS,
            pi_seed: int = 1, relative_ip: bool = True) -> list[dict]:
    """Run Exp. 2 for one (measure, N): train / query are device CSR (indptr int64, indices int32).

    Returns one dict per threshold: the threshold, the paper's four measures, query counts
    and |O|, |O'| totals.
    """
    (tp, ti), (qp, qi) = train, query
    Ds = bs.build_seeded(pi_seed, d, N, tp, ti)
    Qs = bs.build_seeded(pi_seed, d, N, qp, qi)
    Dx = exact_vectors(tp, ti, d)
    Qx = exact_vectors(qp, qi, d)
    thr = list(thresholds)
    if measure == bs.IP and relative_ip:
        top = max_exact_ip(Qx, Dx, d)
        thr = [t * top for t in thr]
    ndb = Ds.shape[0]
    est = bs.join(Qs, Ds, N, d, measure, thr)
    tru = bs.join(Qx, Dx, d, d, measure, thr, exact=True)
    out = []
    for t in range(len(thr)):
        conf = bs.join_confusion(est[t], tru[t], ndb).cpu().numpy()
        m = metrics_from_counts(conf)
        m.update({"threshold": thr[t], "O_total": int(conf[1].sum()), "Oprime_total": int(conf[0].sum())})
        out.append(m)
    return out
