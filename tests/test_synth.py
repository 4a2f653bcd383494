"""The seeded input generator: determinism, structure, distribution shape (CPU only)."""
import os
import subprocess
import sys

import numpy as np

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _check_structure(spec, indptr, indices):
    assert indptr[0] == 0 and len(indptr) == spec.n + 1
    nnz = np.diff(indptr)
    assert (nnz >= 1).all()
    assert (indices >= 0).all() and (indices < spec.d).all()
    rows = np.repeat(np.arange(spec.n), nnz)
    same = rows[1:] == rows[:-1]
    assert (np.diff(indices.astype(np.int64))[same] > 0).all()     # sorted, distinct within a row
    return nnz


def test_tiny_structure():
    indptr, indices = synth.make_csr(synth.TINY)
    nnz = _check_structure(synth.TINY, indptr, indices)
    assert nnz.min() >= 20 and nnz.max() <= 100
    assert abs(nnz.mean() - 60) < 3


def test_lognormal_mean_and_cap():
    spec = synth.scaled(synth.MEDIUM, 5000)
    indptr, indices = synth.make_csr(spec)
    nnz = _check_structure(spec, indptr, indices)
    assert nnz.max() <= 1000
    assert 140 < nnz.mean() < 165          # mean 160 before the cap at 1000 trims the tail


def test_zipf_head_heavier_than_tail():
    spec = synth.CSRSpec(n=2000, d=10_000, kind=0, p1=10, p2=30, cap=30, zipf_s=1.1, seed=9, perm=0)
    _, indices = synth.make_csr(spec)
    counts = np.bincount(indices, minlength=spec.d)
    assert counts[:10].mean() > 20 * counts[5000:].mean()     # identity rank->id: head is ids 0..9
    spec_p = synth.CSRSpec(**{**spec.__dict__, "perm": 1})
    _, ind_p = synth.make_csr(spec_p)
    c2 = np.sort(np.bincount(ind_p, minlength=spec.d))[::-1]
    c1 = np.sort(counts)[::-1]
    assert abs(c2[:10].mean() - c1[:10].mean()) < 0.1 * c1[:10].mean()   # same frequency profile
    assert counts[:10].mean() > 5 * np.bincount(ind_p, minlength=spec.d)[:10].mean()   # permuted: head scattered


def test_determinism_independent_of_threads():
    code = ("import sys; sys.path.insert(0, %r); import synth, hashlib;"
            "p, i = synth.make_csr(synth.scaled(synth.LARGE, 3000));"
            "print(hashlib.sha256(p.tobytes() + i.tobytes()).hexdigest())") % ROOT
    outs = []
    for t in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env).strip())
    assert outs[0] == outs[1]
