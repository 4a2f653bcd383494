"""GPU parity for the BCS parity sketch and its estimates, through the C ABI.

Bar: sketches bit-exact (integer work); estimate planes within |delta| <= 1e-4 * max(1, |ref|)
and, under the shared fp64 recipe (R-B2, R-B3), bit-identical.
"""
import os

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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("spec,N", [(synth.TINY, synth.TINY_N), (synth.scaled(synth.MEDIUM, 3000), 1000),
                                    (synth.scaled(synth.LARGE, 5000), 1024),
                                    (synth.scaled(synth.RANKING_DB, 2000), 4096),
                                    (synth.scaled(synth.TINY, 300), 5000)])
@pytest.mark.parametrize("mode", ["seeded", "auto", "global", "cache"])
def test_bcs_build_bit_exact(spec, N, mode, monkeypatch):
    indptr, indices = synth.make_csr(spec)
    d = spec.d
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    want, st = oracle.bcs_sketch(pi, d, N, indptr, indices)
    assert st == 0
    ip, ix = dev(indptr), dev(indices)
    if mode == "seeded":
        got = bs.bcs_build_seeded(synth.PI_SEED, d, N, ip, ix)
    else:
        if mode != "auto":
            monkeypatch.setenv("BINSKETCH_BUILD_MODE", mode)
        got = bs.bcs_build(dev(pi.view(np.int32)), d, N, ip, ix)
    bs.device_status()
    assert np.array_equal(u32(got), want)
    # BCS differs from the OR sketch exactly where a bucket received an even count >= 2
    orsk, _ = oracle.sketch(pi, d, N, indptr, indices)
    assert ((u32(got) & ~orsk) == 0).all()


def test_bcs_build_duplicates_cancel_and_ragged_rows():
    # hand-built CSR: duplicate entries (R-B1), empty rows, a long row spanning chunks
    rng = np.random.default_rng(1)
    d, N = 3000, 1000
    rows = [[], [5, 5], [1, 2, 3, 2], list(rng.integers(0, d, 5000)), [], [7]] + \
           [list(rng.integers(0, d, int(rng.integers(0, 40)))) for _ in range(200)]
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(r) for r in rows])
    indices = np.array([i for r in rows for i in r], dtype=np.int32)
    pi = oracle.make_pi(4, d, N)
    want, _ = oracle.bcs_sketch(pi, d, N, indptr, indices)
    got = bs.bcs_build(dev(pi.view(np.int32)), d, N, dev(indptr), dev(indices))
    assert np.array_equal(u32(got), want)
    assert not want[1].any()                     # {5, 5} cancels
    got2 = bs.bcs_build_seeded(4, d, N, dev(indptr), dev(indices))
    assert np.array_equal(u32(got2), want)


@pytest.mark.parametrize("na,nb,N", [(300, 700, synth.TINY_N), (129, 257, 1024), (1, 1, 64), (70, 513, 4096),
                                     (200, 200, 33)])
@pytest.mark.parametrize("path", ["pab", "fused"])
def test_bcs_estimate_planes(na, nb, N, path, monkeypatch):
    """pab: tensor-core AND-popcount table + elementwise recipe kernel; fused: the estimate epilogue."""
    monkeypatch.setenv("BINSKETCH_EST_PAB", "1" if path == "pab" else "0")
    spec = synth.scaled(synth.TINY, na + nb, seed=17)
    indptr, indices = synth.make_csr(spec)
    d = spec.d
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    sk, _ = oracle.bcs_sketch(pi, d, N, indptr, indices)
    A, B = sk[:na], sk[na:]
    B[0] = 0
    if nb > 3:
        B[3] = A[0]
    want = oracle.bcs_estimate(A, B, N, d, 15)
    got = bs.bcs_estimate(dev(A.view(np.int32)), dev(B.view(np.int32)), N, d, 15).cpu().numpy()
    ref64 = want.astype(np.float64)
    assert np.all(np.abs(got.astype(np.float64) - ref64) <= 1e-4 * np.maximum(1.0, np.abs(ref64)))
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # plane selection (JS only) and self-pairs (queries == db)
    js = bs.bcs_estimate(dev(A.view(np.int32)), dev(B.view(np.int32)), N, d, bs.JS).cpu().numpy()
    assert np.array_equal(js[0].view(np.uint32), want[2].view(np.uint32))
    Ad = dev(A.view(np.int32))
    selfp = bs.bcs_estimate(Ad, Ad, N, d, bs.HAM).cpu().numpy()[0]
    assert np.array_equal(selfp.view(np.uint32), oracle.bcs_estimate(A, A, N, d, bs.HAM)[0].view(np.uint32))
    assert (np.diag(selfp) == 0).all()


def test_bcs_table_matches_oracle():
    for N, d in ((2, 10), (1224, 5000), (4096, 102_660)):
        assert bs.bcs_table(N, d).tobytes() == oracle.bcs_table(N, d).tobytes()
