"""GPU parity for the threshold join (Experiment 2) through the C ABI.

Bar: bit-exact match bitmaps (a set of (query, db row) pairs, decided in fp64 on both
sides by the same recipe; R-J1), exact list order (db index ascending) and bit-identical
float scores, exact per-query confusion counts. All inputs come from synth/ + oracle/;
the sketches and exact bit vectors fed to both sides are the oracle's.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1910_04658_b200 import binsketch as bs
from paper_1910_04658_b200 import exp2

pytestmark = pytest.mark.gpu

JS_THR = list(synth.EXP2_THRESHOLDS)


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


def _corpus(n, seed, spec=synth.TINY, frac=0.4):
    ip, ix = synth.make_csr(synth.scaled(spec, n, seed=seed))
    ip, ix = synth.plant_near_duplicates(ip, ix, spec.d, frac, seed=seed + 1)
    tr, q = synth.split_rows(n, 0.1, seed=seed + 2)
    return synth.take_rows(ip, ix, q), synth.take_rows(ip, ix, tr)


def _thresholds(measure, scale):
    if measure in (bs.JS, bs.COS):
        return JS_THR
    if measure == bs.IP:
        return [t * scale for t in JS_THR]
    return [t * scale for t in (0.02, 0.05, 0.1, 0.2, 0.4, 0.8, 1.2, 2.0)]   # Hamming: distance <= t


def _sketch(csr, d, N):
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    sk, st = oracle.sketch(pi, d, N, *csr)
    assert st == 0
    return sk


@pytest.mark.parametrize("measure", [bs.IP, bs.HAM, bs.JS, bs.COS])
@pytest.mark.parametrize("N", [synth.TINY_N, 4096])
def test_join_sketch_parity(measure, N):
    (q, t) = _corpus(3000, seed=40)          # 300 queries x 2700 db rows: 11 n-tiles + ragged tail
    d = synth.TINY.d
    Qs, Ds = _sketch(q, d, N), _sketch(t, d, N)
    thr = _thresholds(measure, 60.0)
    ref = oracle.join(Qs, Ds, N, d, measure, thr)
    got = u32(bs.join(dev(Qs.view(np.int32)), dev(Ds.view(np.int32)), N, d, measure, thr))
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)
    # the workload is not trivial: some planes non-empty, some pairs rejected
    nbits = lambda a: int(np.unpackbits(a.view(np.uint8)).sum())   # noqa: E731
    assert 0 < nbits(ref[0]) and nbits(ref[-1]) < Qs.shape[0] * Ds.shape[0]


@pytest.mark.parametrize("measure", [bs.IP, bs.HAM, bs.JS, bs.COS])
def test_join_exact_parity(measure):
    (q, t) = _corpus(1500, seed=50)
    d = synth.TINY.d
    # exact bit vectors: the oracle's sketch with the identity map and N = d
    ident = np.arange(d, dtype=np.uint32)
    Qx, _ = oracle.sketch(ident, d, d, *q)
    Dx, _ = oracle.sketch(ident, d, d, *t)
    thr = _thresholds(measure, 40.0)
    ref = oracle.join_exact(q[0], q[1], t[0], t[1], measure, thr)
    got = u32(bs.join(dev(Qx.view(np.int32)), dev(Dx.view(np.int32)), d, d, measure, thr, exact=True))
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("exact", [False, True])
def test_join_self_exclusion_and_unsorted_thresholds(exact):
    (q, t) = _corpus(1200, seed=60)
    d = synth.TINY.d
    N = d if exact else 2048
    pi = np.arange(d, dtype=np.uint32) if exact else oracle.make_pi(synth.PI_SEED, d, N)
    Ds, _ = oracle.sketch(pi, d, N, *t)
    thr = [0.5, 0.95, 0.1, 0.8]                       # any order; planes follow the argument order
    Dd = dev(Ds.view(np.int32))
    got = u32(bs.join(Dd, Dd, N, d, bs.JS, thr, exclude_self=True, exact=exact))
    if exact:
        ref = oracle.join_exact(t[0], t[1], t[0], t[1], bs.JS, thr, exclude_self=True)
    else:
        ref = oracle.join(Ds, Ds, N, d, bs.JS, thr, exclude_self=True)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("nq,ndb", [(1, 1), (1, 31), (5, 32), (129, 33), (7, 257), (200, 0)])
def test_join_edge_shapes(nq, ndb):
    rng = np.random.default_rng(nq * 1000 + ndb)
    N, d = 1000, 3000
    Q = (rng.random((nq, bs.words(N))) < 0.5).astype(np.uint32) * rng.integers(0, 2**32, (nq, bs.words(N)), dtype=np.uint32)
    D = (rng.random((ndb, bs.words(N))) < 0.5).astype(np.uint32) * rng.integers(0, 2**32, (ndb, bs.words(N)), dtype=np.uint32)
    Q[:, -1] &= np.uint32((1 << (N % 32)) - 1)
    D[:, -1] &= np.uint32((1 << (N % 32)) - 1)
    if ndb:
        D[0] = 0
    for m, thr in ((bs.IP, [0.0, 100.0, 1e9]), (bs.COS, [0.0, 0.3, 2.0]), (bs.HAM, [-1.0, 500.0, float("inf")])):
        got = u32(bs.join(dev(Q.view(np.int32)), dev(D.view(np.int32)), N, d, m, thr))
        ref = oracle.join(Q, D, N, d, m, thr)
        assert np.array_equal(got, ref), (m, thr)


def test_join_invalid_arguments():
    Q = torch.zeros((4, 32), dtype=torch.int32, device="cuda")
    with pytest.raises(bs.BinSketchError, match="EINVAL"):
        bs.join(Q, Q, 1024, 5000, bs.JS, [float("nan")])
    with pytest.raises(bs.BinSketchError, match="EINVAL"):
        bs.join(Q, Q, 1024, 5000, bs.JS, [0.5] * 17)
    with pytest.raises(bs.BinSketchError, match="EINVAL"):
        bs.join(Q, Q, 1024, 5000, bs.JS | bs.COS, [0.5])


@pytest.mark.parametrize("measure,exact", [(bs.JS, False), (bs.IP, False), (bs.HAM, True), (bs.COS, True)])
def test_join_list_parity(measure, exact):
    (q, t) = _corpus(2000, seed=70)
    d = synth.TINY.d
    N = d if exact else synth.TINY_N
    pi = np.arange(d, dtype=np.uint32) if exact else oracle.make_pi(synth.PI_SEED, d, N)
    Qs, _ = oracle.sketch(pi, d, N, *q)
    Ds, _ = oracle.sketch(pi, d, N, *t)
    thr = _thresholds(measure, 40.0)[3]
    ref_bits = (oracle.join_exact(q[0], q[1], t[0], t[1], measure, [thr]) if exact
                else oracle.join(Qs, Ds, N, d, measure, [thr]))[0]
    Qd, Dd = dev(Qs.view(np.int32)), dev(Ds.view(np.int32))
    bits = bs.join(Qd, Dd, N, d, measure, [thr], exact=exact)[0]
    row_ptr, cols, scores = bs.join_list(bits, Qd, Dd, N, d, measure, exact=exact)
    row_ptr, cols, scores = row_ptr.cpu().numpy(), cols.cpu().numpy(), scores.cpu().numpy()
    sets = oracle.bits_to_sets(ref_bits, Ds.shape[0])
    assert row_ptr[0] == 0 and np.array_equal(np.diff(row_ptr), [len(s) for s in sets])
    assert row_ptr[-1] > 0
    if not exact:
        planes = oracle.estimate(Qs, Ds, N, d, measure)[0]
    for i, s in enumerate(sets):
        js = cols[row_ptr[i]:row_ptr[i + 1]]
        assert list(js) == sorted(s)
        for j, sc in zip(js, scores[row_ptr[i]:row_ptr[i + 1]]):
            if exact:
                e = oracle.exact(q[1][q[0][i]:q[0][i + 1]], t[1][t[0][j]:t[0][j + 1]])
                want = np.float32(e[{1: 0, 2: 1, 4: 2, 8: 3}[measure]])
            else:
                want = planes[i, j]
            assert np.float32(sc).view(np.uint32) == np.float32(want).view(np.uint32)


def test_join_confusion_and_exp2_metrics():
    (q, t) = _corpus(2000, seed=80)
    d = synth.TINY.d
    N = 512
    thr = [0.9, 0.5]
    qd = (dev(q[0]), dev(q[1]))
    td = (dev(t[0]), dev(t[1]))
    res = exp2.ranking(td, qd, d, N, bs.JS, thr, pi_seed=synth.PI_SEED)
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    Qs, _ = oracle.sketch(pi, d, N, *q)
    Ds, _ = oracle.sketch(pi, d, N, *t)
    est = oracle.join(Qs, Ds, N, d, bs.JS, thr)
    tru = oracle.join_exact(q[0], q[1], t[0], t[1], bs.JS, thr)
    ndb = len(t[0]) - 1
    for k in range(len(thr)):
        want = oracle.ranking_metrics(oracle.bits_to_sets(tru[k], ndb), oracle.bits_to_sets(est[k], ndb))
        got = res[k]
        assert got["query_count"] == want["query_count"] and got["skipped_queries"] == want["skipped_queries"]
        for key in ("accuracy", "precision", "recall", "f1"):
            assert abs(got[key] - want[key]) <= 1e-12, (k, key)
        # raw counts against numpy popcounts of the oracle's bitmaps
        conf = bs.join_confusion(dev(est[k].view(np.int32)), dev(tru[k].view(np.int32)), ndb).cpu().numpy()
        pc = lambda a: np.unpackbits(a.view(np.uint8), axis=1).sum(1)   # noqa: E731
        assert np.array_equal(conf[0], pc(est[k])) and np.array_equal(conf[1], pc(tru[k]))
        assert np.array_equal(conf[2], pc(est[k] & tru[k]))


def test_join_list_capacity_truncation_and_exact_row_ptr():
    (q, t) = _corpus(1500, seed=90)
    d, N = synth.TINY.d, synth.TINY_N
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    Qs, _ = oracle.sketch(pi, d, N, *q)
    Ds, _ = oracle.sketch(pi, d, N, *t)
    Qd, Dd = dev(Qs.view(np.int32)), dev(Ds.view(np.int32))
    bits = bs.join(Qd, Dd, N, d, bs.JS, [0.2])[0]
    row_ptr, cols, scores = bs.join_list(bits, Qd, Dd, N, d, bs.JS)
    total = int(row_ptr[-1].item())
    assert total > 10
    # raw ABI call with a capacity below the total: row_ptr still exact, the first `cap` entries identical
    cap = total // 3
    rp = torch.empty(Qd.shape[0] + 1, dtype=torch.int64, device="cuda")
    oj = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
    osc = torch.empty(cap, dtype=torch.float32, device="cuda")
    nws = bs.workspace_bytes(bs.OP_JOIN_LIST, Qd.shape[0], Dd.shape[0], N)
    ws = torch.empty(max(1, nws), dtype=torch.uint8, device="cuda")
    code = bs._lib().binsketch_join_list(bs._words_tensor(bits, "b"), bs._words_tensor(Qd, "q"), Qd.shape[0],
                                         bs._words_tensor(Dd, "d"), Dd.shape[0], N, d, bs.JS, 0,
                                         bs._dev(rp, torch.int64, "rp"), bs._dev(oj, torch.int32, "oj"),
                                         bs._dev(osc, torch.float32, "os"), cap, bs.ctypes.c_void_p(ws.data_ptr()),
                                         ws.numel(), bs._stream())
    assert code == 0
    assert torch.equal(rp, row_ptr)
    assert torch.equal(oj, cols[:cap]) and torch.equal(osc.view(torch.int32), scores[:cap].view(torch.int32))


def test_join_sixteen_thresholds():
    (q, t) = _corpus(1200, seed=91)
    d, N = synth.TINY.d, 2048
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    Qs, _ = oracle.sketch(pi, d, N, *q)
    Ds, _ = oracle.sketch(pi, d, N, *t)
    thr = list(np.linspace(0.02, 0.98, 16))
    got = u32(bs.join(dev(Qs.view(np.int32)), dev(Ds.view(np.int32)), N, d, bs.COS, thr))
    assert np.array_equal(got, oracle.join(Qs, Ds, N, d, bs.COS, thr))
