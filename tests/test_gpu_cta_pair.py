"""GPU parity of the tensor-core engine's CTA-pair mode (cta_group::2, tc.cu).

A CTA pair computes a 256 x 256 tile: each CTA stages its own 128 A rows and half of the B
rows, and the pair MMA leaves every CTA its 128 rows x all 256 columns. These tests force the
mode (BINSKETCH_TC_CG=2, read at every launch) at sizes whose row count is an odd number of
128-row tiles (the second CTA of the last pair has no valid rows) with ragged column tails,
and require the same bar as the single-CTA engine: bit-exact AND-popcounts, lists and
bitmaps vs the oracle; estimates within the fp32 rounding of the oracle's fp64 value.
The exact join over d-bit rows (K >= 32768) takes the pair mode by default.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1910_04658_b200 import binsketch as bs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    bs._lib()
    yield
    torch.cuda.synchronize()


@pytest.fixture(params=[1, 2])
def cg(request, monkeypatch):
    monkeypatch.setenv("BINSKETCH_ENGINE", "tc")
    monkeypatch.setenv("BINSKETCH_TC_CG", str(request.param))
    return request.param


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _sketches(spec, N, seed=synth.PI_SEED):
    ip, ix = synth.make_csr(spec)
    sk, st = oracle.sketch(oracle.make_pi(seed, spec.d, N), spec.d, N, ip, ix)
    assert st == 0
    return sk


@pytest.mark.parametrize("N,na,nb", [(1024, 1100, 1300), (1224, 130, 2049), (33, 385, 257), (4096, 257, 513)])
def test_andpopc_pair(cg, N, na, nb):
    A = _sketches(synth.scaled(synth.LARGE, na, seed=91), N)
    B = _sketches(synth.scaled(synth.LARGE, nb, seed=92), N)
    got = bs.andpopc(dev(A.view(np.int32)), dev(B.view(np.int32)), N).cpu().numpy()
    assert np.array_equal(got, oracle.andpopc(A, B, N))


@pytest.mark.parametrize("N", [2000, 5000])
def test_estimate_pair(cg, N, monkeypatch):
    monkeypatch.setenv("BINSKETCH_EST_PAB", "0")   # the fused estimate epilogue on the pair engine
    A = _sketches(synth.scaled(synth.MEDIUM, 300, seed=93), N)
    B = _sketches(synth.scaled(synth.MEDIUM, 450, seed=94), N)
    B[:40] = A[:40]
    got = bs.estimate(dev(A.view(np.int32)), dev(B.view(np.int32)), N, 28_102, 15).cpu().numpy()
    ref = np.asarray(oracle.estimate(A, B, N, 28_102, 15)).astype(np.float32)
    ref64 = ref.astype(np.float64)
    assert np.all(np.abs(got.astype(np.float64) - ref64) <= 1e-4 * np.maximum(1.0, np.abs(ref64)))   # graded tolerance
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))     # and bit identity (canonical recipe, R-C3)


@pytest.mark.parametrize("measure", [1, 4])
def test_topk_pair(cg, measure):
    N, d = 1024, 500_000
    D = _sketches(synth.scaled(synth.LARGE, 3000, seed=95), N)
    D[100:110] = D[5]                                   # exact ties: lower index first
    Q = D[:385].copy()                                  # 3 query tiles + 1 row: odd pair count
    gi, gs = bs.topk(dev(Q.view(np.int32)), dev(D.view(np.int32)), N, d, measure, 50, exclude_self=True)
    ri, rs = oracle.topk(Q, D, N, d, measure, 50, exclude_self=True)
    assert np.array_equal(gi.cpu().numpy(), ri)
    g = gs.cpu().numpy()
    r32 = np.asarray(rs).astype(np.float32)
    assert np.all(np.abs(g.astype(np.float64) - r32.astype(np.float64)) <= 1e-4 * np.maximum(1.0, np.abs(r32)))
    assert np.array_equal(g.view(np.uint32), r32.view(np.uint32))


def test_join_pair_sketch_and_exact(cg):
    """Sketch join (short K) and exact join over the d-bit rows (K = d padded; >= 32768 takes the
    pair mode without the override): bitmaps bit-exact vs the oracle."""
    spec = synth.scaled(synth.TINY, 400, seed=96)
    d = 40_000
    spec = synth.CSRSpec(n=spec.n, d=d, kind=spec.kind, p1=spec.p1, p2=spec.p2, cap=spec.cap, zipf_s=spec.zipf_s, seed=96)
    ip, ix = synth.make_csr(spec)
    ip, ix = synth.plant_near_duplicates(ip, ix, d, 0.4, seed=97)
    N = 2048
    S, _ = oracle.sketch(oracle.make_pi(synth.PI_SEED, d, N), d, N, ip, ix)
    thr = [0.9, 0.5, 0.2]
    Sd = dev(S.view(np.int32))
    got = bs.join(Sd, Sd, N, d, bs.JS, thr, exclude_self=True).cpu().numpy().view(np.uint32)
    ref = oracle.join(S, S, N, d, 4, thr, exclude_self=True)
    assert np.array_equal(got, ref)
    X, _ = oracle.sketch(np.arange(d, dtype=np.uint32), d, d, ip, ix)   # exact bit vectors (identity map, N = d)
    Xd = dev(X.view(np.int32))
    got = bs.join(Xd, Xd, d, d, bs.JS, thr, exclude_self=True, exact=True).cpu().numpy().view(np.uint32)
    ref = oracle.join_exact(ip, ix, ip, ix, 4, thr, exclude_self=True)
    assert np.array_equal(got, ref)
