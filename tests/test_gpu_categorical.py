"""GPU parity for the categorical extension through the C ABI.

Bar: one-hot CSR and sketches bit-exact; estimated categorical distance (HAM^/2, reading R-C1)
bit-identical to the oracle's fp64 recipe (and within 1e-4 relative).
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _offsets(cards):
    off = np.zeros(len(cards) + 1, dtype=np.int64)
    off[1:] = np.cumsum(cards)
    return off


@pytest.mark.parametrize("n,cards", [(1, [2]), (1000, [3, 7, 2, 12, 5]), (5000, [40] * 25), (300, [1, 1000, 2])])
def test_onehot_and_build_bit_exact(n, cards):
    X = synth.make_categorical(n, cards, seed=n)
    ip_ref, ix_ref, d, st = oracle.onehot(X, cards)
    assert st == 0
    ip, ix = bs.onehot(dev(X), dev(_offsets(cards)))
    bs.device_status()
    assert np.array_equal(ip.cpu().numpy(), ip_ref) and np.array_equal(ix.cpu().numpy(), ix_ref)
    N = 256
    pi = oracle.make_pi(3, d, N)
    sk = bs.build(dev(pi.view(np.int32)), d, N, ip, ix)
    ref, _ = oracle.sketch(pi, d, N, ip_ref, ix_ref)
    assert np.array_equal(sk.cpu().numpy().view(np.uint32), ref)


def test_onehot_bad_code_latched():
    X = np.array([[0, 1], [2, 0]], dtype=np.int32)      # 2 is outside column 0's [0, 2)
    bs.onehot(dev(X), dev(_offsets([2, 3])))
    with pytest.raises(bs.BinSketchError, match="EINDEX"):
        bs.device_status()
    bs.device_status()                                   # cleared


@pytest.mark.parametrize("na,nb,N", [(700, 700, 512), (129, 300, 1224), (1, 1, 64)])
@pytest.mark.parametrize("path", ["pab", "fused"])
def test_categorical_estimate_bit_exact(na, nb, N, path, monkeypatch):
    monkeypatch.setenv("BINSKETCH_EST_PAB", "1" if path == "pab" else "0")
    cards = [5, 11, 3, 30, 8, 2]
    X = synth.make_categorical(na + nb, cards, seed=na + nb)
    ip, ix, d, _ = oracle.onehot(X, cards)
    S, _ = oracle.sketch(oracle.make_pi(1, d, N), d, N, ip, ix)
    A, B = S[:na], S[na:]
    want = oracle.categorical_estimate(A, B, N, d)
    got = bs.categorical_estimate(dev(A.view(np.int32)), dev(B.view(np.int32)), N, d).cpu().numpy()
    assert np.all(np.abs(got.astype(np.float64) - want) <= 1e-4 * np.maximum(1.0, np.abs(want)))
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_onehot_zero_columns_and_zero_rows():
    ip, ix = bs.onehot(torch.zeros((5, 0), dtype=torch.int32, device="cuda"), torch.zeros(1, dtype=torch.int64, device="cuda"))
    assert ip.cpu().tolist() == [0] * 6 and ix.numel() == 0
    ip, ix = bs.onehot(torch.zeros((0, 3), dtype=torch.int32, device="cuda"), dev(_offsets([2, 2, 2])))
    assert ix.numel() == 0
