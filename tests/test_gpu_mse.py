"""GPU parity for Experiment 1 (binsketch_mse) against the oracle.

Bar: pair counts bit-exact (integer); sums of squared errors within 1e-9 relative — both sides
add the same fp64 squares but in different orders (the oracle sequentially in (i, j) order, the
GPU in a fixed tree), so the bound is the fp64 summation error, n_pairs * 2^-53 << 1e-9 here.
The GPU result itself is bit-identical run to run (fixed grid), asserted too.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1910_04658_b200 import binsketch as bs
from paper_1910_04658_b200 import exp1

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


THR = {1: [2.0, 5.0, 10.0, 20.0], 2: [10.0, 40.0, 80.0, 150.0], 4: [0.95, 0.8, 0.5, 0.2, 0.1, 0.0],
       8: [0.95, 0.9, 0.6, 0.3, 0.0]}


@pytest.mark.parametrize("measure", [1, 2, 4, 8])
@pytest.mark.parametrize("bcs", [False, True])
@pytest.mark.parametrize("n,N", [(700, synth.TINY_N), (4500, 256)])   # 4500 rows: two row blocks + ragged
def test_mse_parity(measure, bcs, n, N):
    if n > 1000 and (measure in (1, 2) or bcs):
        pytest.skip("large case run for JS / COS BinSketch only (oracle time)")
    spec = synth.scaled(synth.TINY, n, seed=90 + n)
    ip, ix = synth.make_csr(spec)
    ip, ix = synth.plant_near_duplicates(ip, ix, spec.d, 0.4, seed=91)
    d = spec.d
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    S, _ = (oracle.bcs_sketch if bcs else oracle.sketch)(pi, d, N, ip, ix)
    X, _ = oracle.sketch(np.arange(d, dtype=np.uint32), d, d, ip, ix)
    thr = THR[measure]
    sse_ref, cnt_ref = oracle.mse(S, N, d, ip, ix, measure, thr, bcs=bcs)
    sse, cnt = bs.mse(dev(S.view(np.int32)), dev(X.view(np.int32)), N, d, measure, thr, bcs=bcs)
    sse, cnt = sse.cpu().numpy(), cnt.cpu().numpy()
    assert np.array_equal(cnt.astype(np.uint64), cnt_ref)
    assert np.all(np.abs(sse - sse_ref) <= 1e-9 * np.maximum(1e-300, np.abs(sse_ref)))
    sse2, cnt2 = bs.mse(dev(S.view(np.int32)), dev(X.view(np.int32)), N, d, measure, thr, bcs=bcs)
    assert sse2.cpu().numpy().tobytes() == sse.tobytes()
    assert cnt_ref[0] > 0


def test_mse_edge_cases():
    d, N = 100, 64
    X = torch.zeros((1, bs.words(d)), dtype=torch.int32, device="cuda")
    S = torch.zeros((1, bs.words(N)), dtype=torch.int32, device="cuda")
    sse, cnt = bs.mse(S, X, N, d, bs.JS, [0.5])          # one row: no pairs
    assert cnt.item() == 0 and sse.item() == 0.0
    with pytest.raises(bs.BinSketchError, match="EINVAL"):
        bs.mse(S, X, N, d, bs.JS | bs.IP, [0.5])


def test_exp1_driver_matches_oracle():
    spec = synth.scaled(synth.TINY, 600, seed=5)
    ip, ix = synth.make_csr(spec)
    ip, ix = synth.plant_near_duplicates(ip, ix, spec.d, 0.5, seed=6)
    d, N = spec.d, 512
    rows = exp1.fidelity(dev(ip), dev(ix), d, N, bs.JS, [0.9, 0.5], pi_seed=3)
    S, _ = oracle.sketch(oracle.make_pi(3, d, N), d, N, ip, ix)
    sse, cnt = oracle.mse(S, N, d, ip, ix, bs.JS, [0.9, 0.5])
    rep = oracle.mse_report(sse, cnt, bs.JS)
    for r, w in zip(rows, rep):
        assert r["pairs"] == w["pairs"]
        assert abs(r["neg_log_mse"] - w["neg_log_mse"]) <= 1e-9 * abs(w["neg_log_mse"])


def test_mse_sixteen_thresholds():
    spec = synth.scaled(synth.TINY, 400, seed=77)
    ip, ix = synth.make_csr(spec)
    d, N = spec.d, 700
    S, _ = oracle.sketch(oracle.make_pi(2, d, N), d, N, ip, ix)
    X, _ = oracle.sketch(np.arange(d, dtype=np.uint32), d, d, ip, ix)
    thr = list(np.linspace(0.0, 0.9, 16))
    sse_ref, cnt_ref = oracle.mse(S, N, d, ip, ix, bs.COS, thr)
    sse, cnt = bs.mse(dev(S.view(np.int32)), dev(X.view(np.int32)), N, d, bs.COS, thr)
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), cnt_ref)
    assert np.all(np.abs(sse.cpu().numpy() - sse_ref) <= 1e-9 * np.maximum(1e-300, np.abs(sse_ref)))
