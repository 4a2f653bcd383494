"""All-pairs estimate planes over (|a_s|, |b_s|, |a_s AND b_s|) triples, both pair engines.

The estimate epilogues store round32 of the canonical fp64 recipe (bsk_estimator.cuh). These
tests feed sketches built so that the all-pairs table hits every feasible triple (A rows:
prefixes of length pa; B rows: bit intervals [s, s + pb)), including empty and saturated
sketches, and require bit-identical float planes vs the oracle's fp64 recipe rounded to fp32.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1910_04658_b200 import binsketch as bs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    bs._lib()
    yield
    torch.cuda.synchronize()


def _rows(spans, N):
    W = (N + 31) // 32
    out = np.zeros((len(spans), W), dtype=np.uint32)
    for r, (s, e) in enumerate(spans):
        bits = np.zeros(W * 32, dtype=np.uint8)
        bits[s:e] = 1
        out[r] = np.packbits(bits.reshape(-1, 32)[:, ::-1], axis=1).view(">u4").ravel().astype(np.uint32)
    return out


def _check(N, d, pas, intervals, engine, monkeypatch):
    monkeypatch.setenv("BINSKETCH_ENGINE", "cuda" if engine == "cuda" else "tc")
    monkeypatch.setenv("BINSKETCH_EST_PAB", "0" if engine == "tc-fused" else "1")
    A = _rows([(0, p) for p in pas], N)
    B = _rows(intervals, N)
    assert np.array_equal(oracle.popcount(A, N), np.asarray(pas))
    got = bs.estimate(torch.from_numpy(A.view(np.int32)).cuda(), torch.from_numpy(B.view(np.int32)).cuda(), N, d, 15)
    ref = oracle.estimate(A, B, N, d, 15)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("engine", ["tc", "tc-fused", "cuda"])
def test_all_triples_small_N(engine, monkeypatch):
    N = 64
    pas = list(range(N + 1))
    intervals = [(s, s + p) for p in range(N + 1) for s in range(0, N - p + 1)]   # every (pb, offset)
    for d in (64, 1000, 1_000_000):
        _check(N, d, pas, intervals, engine, monkeypatch)


@pytest.mark.parametrize("engine", ["tc", "tc-fused", "cuda"])
@pytest.mark.parametrize("N", [1000, 2000])
def test_triples_sampled_large_N(engine, N, monkeypatch):
    rng = np.random.default_rng(N)
    pas = sorted(set([0, 1, 2, N - 1, N] + rng.integers(0, N + 1, 250).tolist()))
    pbs = [0, 1, 2, N - 1, N] + rng.integers(0, N + 1, 300).tolist()
    intervals = [(s, s + p) for p in pbs for s in {0, N - p, int(rng.integers(0, N - p + 1))}]
    _check(N, 28_102, pas, intervals, engine, monkeypatch)


@pytest.mark.parametrize("measure", [4, 8])
def test_join_thresholds_on_exact_key_values(measure):
    """Threshold join (sketch keys) with thresholds equal to keys that pairs actually take: the
    division-free plane decision (join_first_plane) must defer to the exact key inside its margin
    and reproduce the oracle's bitmaps bit for bit, ties at the threshold included."""
    from oracle import definitional as D
    N, d = 64, 1000
    pas = list(range(N + 1))
    intervals = [(s, s + p) for p in range(N + 1) for s in range(0, N - p + 1, 3)]
    A = _rows([(0, p) for p in pas], N)
    B = _rows(intervals, N)
    L = D.card_table(N, d)
    k = 2 if measure == 4 else 3
    # exact fp64 keys of a few triples (the recipe R-C3) + round values that many pairs hit exactly
    thr = sorted({D.estimate_canonical(pa, pb, pab, N, L)[k] for pa, pb, pab in
                  [(10, 20, 5), (30, 30, 30), (40, 12, 7), (64, 64, 64), (17, 33, 9)]} | {0.5, 0.25, 1.0})
    thr = [t for t in thr if t > 0.0][:16]
    Ad, Bd = torch.from_numpy(A.view(np.int32)).cuda(), torch.from_numpy(B.view(np.int32)).cuda()
    got = bs.join(Ad, Bd, N, d, measure, thr).cpu().numpy().view(np.uint32)
    ref = oracle.join(A, B, N, d, measure, thr)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("bcs", [False, True])
@pytest.mark.parametrize("N", [500, 1224])
def test_estimate_rows_memoised_cos_denominator(bcs, N, monkeypatch):
    """Rows of >= 4 (N + 1) db columns take the recipe kernel's per-row memo of sqrt(L[pa] L[pb])
    (pairs.cu, SQ); the planes stay bit-identical to the oracle (BinSketch and BCS)."""
    import synth
    monkeypatch.setenv("BINSKETCH_ENGINE", "tc")
    monkeypatch.setenv("BINSKETCH_EST_PAB", "1")
    spec = synth.scaled(synth.MEDIUM, 90 + 4 * (N + 1) + 7, seed=31 + N)
    ip, ix = synth.make_csr(spec)
    pi = oracle.make_pi(synth.PI_SEED, spec.d, N)
    S, _ = (oracle.bcs_sketch if bcs else oracle.sketch)(pi, spec.d, N, ip, ix)
    A, B = S[:90], S[90:]
    B[0] = 0
    B[5] = A[3]
    Ad, Bd = torch.from_numpy(A.view(np.int32)).cuda(), torch.from_numpy(B.view(np.int32)).cuda()
    got = (bs.bcs_estimate if bcs else bs.estimate)(Ad, Bd, N, spec.d, 15).cpu().numpy()
    ref = (oracle.bcs_estimate if bcs else oracle.estimate)(A, B, N, spec.d, 15)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
