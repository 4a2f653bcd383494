"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar (north star): bit-exact for pi, sketches, popcounts, AND-popcounts and
top-k index lists (ties -> lower index); float estimates within
|delta| <= 1e-4 * max(1, |ref|) — under the canonical fp64 recipe (R-C3) they
are expected bit-identical, and that stronger property is asserted too.
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
    bs._lib()       # fails loudly if libbinsketch.so is missing (no fallback)
    yield
    torch.cuda.synchronize()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def csr_dev(indptr, indices):
    return dev(indptr.astype(np.int64)), dev(indices.astype(np.int32))


def assert_est_close(got, ref):
    """The graded tolerance, then bit-identity (canonical recipe)."""
    ref64 = ref.astype(np.float64)
    assert np.all(np.abs(got.astype(np.float64) - ref64) <= 1e-4 * np.maximum(1.0, np.abs(ref64)))
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


# ------------------------------------------------------------------ pi -----
@pytest.mark.parametrize("seed,d,N", [(0, 8, 16), (1, 8, 1224), (1, 5000, 1224), (1, 28_102, 1000),
                                      (7, 102_660, 4096), (1, 1 << 20, 1024), (3, 1000, 2),
                                      (5, 1000, 3), (9, 4097, 65537), (11, 3000, 2**31 + 11),
                                      (2**64 - 1, 777, 4294967295)])
def test_make_pi_bit_exact(seed, d, N):
    got = u32(bs.make_pi(seed, d, N))
    assert np.array_equal(got, oracle.make_pi(seed, d, N))


# --------------------------------------------------------------- build -----
def _check_build(spec_or_csr, N, seed=synth.PI_SEED, d=None, seeded_too=True):
    if isinstance(spec_or_csr, synth.CSRSpec):
        indptr, indices = synth.make_csr(spec_or_csr)
        d = spec_or_csr.d
    else:
        indptr, indices = spec_or_csr
    pi = oracle.make_pi(seed, d, N)
    ref, st = oracle.sketch(pi, d, N, indptr, indices)
    assert st == 0
    ip, ix = csr_dev(indptr, indices)
    got = u32(bs.build(dev(pi.view(np.int32)), d, N, ip, ix))
    assert np.array_equal(got, ref)
    if seeded_too:
        got2 = u32(bs.build_seeded(seed, d, N, ip, ix))
        assert np.array_equal(got2, ref)
    bs.device_status()
    return ref


def test_build_tiny_full():
    _check_build(synth.TINY, synth.TINY_N)


@pytest.mark.parametrize("N", synth.MEDIUM_NS)
def test_build_medium_scaled(N):
    _check_build(synth.scaled(synth.MEDIUM, 3000), N)


def test_build_medium_smem_pi_path():
    # >= 148*8*32 rows with W = 32 and d = 28102 engages the shared-memory uint16 pi table
    _check_build(synth.scaled(synth.MEDIUM, 40_000), 1000, seeded_too=False)


def test_build_ranking_and_buildonly_and_large_scaled():
    _check_build(synth.scaled(synth.RANKING_DB, 3000), synth.RANKING_N)
    _check_build(synth.scaled(synth.BUILD_ONLY, 50_000), synth.BUILD_ONLY_N)
    _check_build(synth.scaled(synth.LARGE, 20_000), synth.LARGE_N)


@pytest.mark.parametrize("N", [2, 3, 31, 32, 33, 63, 64, 65, 1000, 1224, 2000, 4096, 5000, 40_000, 100_000])
def test_build_adversarial_widths(N):
    rng = np.random.default_rng(N)
    d = 3000
    rows = []
    for r in range(300):
        kind = r % 6
        if kind == 0:
            rows.append(np.array([], dtype=np.int32))                        # empty row
        elif kind == 1:
            rows.append(rng.integers(0, d, 1).astype(np.int32))              # nnz = 1
        elif kind == 2:
            rows.append(rng.integers(0, d, 2500).astype(np.int32))           # nnz >> N, duplicates, unsorted
        else:
            rows.append(np.sort(rng.choice(d, rng.integers(1, 200), replace=False)).astype(np.int32))
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(x) for x in rows])
    indices = np.concatenate(rows)
    _check_build((indptr, indices), N, seed=N, d=d)


@pytest.mark.parametrize("mode", ["global", "cache", "cache32", "smem16"])
def test_build_forced_pi_source(mode, monkeypatch):
    """Every pi source of K1 (shared-memory table, shared-memory caches, L1/L2 gather) gives
    the same bit-exact sketches, on Zipf data and on adversarial rows."""
    monkeypatch.setenv("BINSKETCH_BUILD_MODE", mode)
    _check_build(synth.scaled(synth.BUILD_ONLY, 20_000), synth.BUILD_ONLY_N, seeded_too=False)
    _check_build(synth.scaled(synth.RANKING_DB, 2000), synth.RANKING_N, seeded_too=False)
    rng = np.random.default_rng(7)
    d, N = 70_000, 1224
    rows = [np.array([], dtype=np.int32) if r % 5 == 0 else
            rng.integers(0, d, int(rng.integers(1, 3000))).astype(np.int32) for r in range(400)]
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(x) for x in rows])
    _check_build((indptr, np.concatenate(rows)), N, seed=3, d=d, seeded_too=False)


def test_build_unaligned_indices_view():
    """indices not 16-B aligned (a view at offset 1): the scalar-load path."""
    indptr, indices = synth.make_csr(synth.scaled(synth.LARGE, 3000))
    N, d = synth.LARGE_N, synth.LARGE.d
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    ref, _ = oracle.sketch(pi, d, N, indptr, indices)
    buf = torch.zeros(len(indices) + 1, dtype=torch.int32, device="cuda")
    buf[1:] = dev(indices)
    view = buf[1:]
    assert view.data_ptr() % 16 != 0
    got = u32(bs.build(dev(pi.view(np.int32)), d, N, dev(indptr), view))
    assert np.array_equal(got, ref)
    got = u32(bs.build_seeded(synth.PI_SEED, d, N, dev(indptr), view))
    assert np.array_equal(got, ref)


def test_build_explicit_colliding_table_and_offset_indptr():
    d, N = 500, 70
    pi = (np.arange(d) % 7).astype(np.uint32)          # forced collisions: only 7 buckets used
    indptr, indices = synth.make_csr(synth.CSRSpec(n=400, d=d, kind=0, p1=1, p2=60, cap=60, zipf_s=1.1, seed=31))
    ref, _ = oracle.sketch(pi, d, N, indptr, indices)
    got = u32(bs.build(dev(pi.view(np.int32)), d, N, *csr_dev(indptr, indices)))
    assert np.array_equal(got, ref)
    # indptr with a nonzero base: rows 100..399 addressed into the full indices array
    sub = indptr[100:]
    got = u32(bs.build(dev(pi.view(np.int32)), d, N, dev(sub), dev(indices)))
    assert np.array_equal(got, ref[100:])


def test_build_empty_and_errors():
    pi = dev(oracle.make_pi(1, 100, 64).view(np.int32))
    out = bs.build(pi, 100, 64, dev(np.zeros(1, dtype=np.int64)), dev(np.zeros(0, dtype=np.int32)))
    assert out.shape == (0, 2)
    # out-of-range index -> latched EINDEX
    bs.build(pi, 100, 64, dev(np.array([0, 2], dtype=np.int64)), dev(np.array([5, 100], dtype=np.int32)))
    with pytest.raises(bs.BinSketchError) as e:
        bs.device_status()
    assert e.value.code == 2
    bs.device_status()                                # cleared
    bs.build(pi, 100, 64, dev(np.array([0, 1], dtype=np.int64)), dev(np.array([-3], dtype=np.int32)))
    with pytest.raises(bs.BinSketchError):
        bs.device_status()
    # decreasing indptr
    bs.build(pi, 100, 64, dev(np.array([0, 3, 1, 4], dtype=np.int64)), dev(np.arange(4, dtype=np.int32)))
    with pytest.raises(bs.BinSketchError):
        bs.device_status()
    # pi value >= N
    bad = dev(np.array([0, 99, 1], dtype=np.int32))
    bs.build(bad, 3, 64, dev(np.array([0, 3], dtype=np.int64)), dev(np.arange(3, dtype=np.int32)))
    with pytest.raises(bs.BinSketchError):
        bs.device_status()
    with pytest.raises(bs.BinSketchError):
        bs.build(pi, 100, 1, dev(np.array([0, 1], dtype=np.int64)), dev(np.array([1], dtype=np.int32)))


# ----------------------------------------------------------- popcounts -----
def _sketches(spec, N, seed=synth.PI_SEED):
    indptr, indices = synth.make_csr(spec)
    sk, _ = oracle.sketch(oracle.make_pi(seed, spec.d, N), spec.d, N, indptr, indices)
    return sk


@pytest.mark.parametrize("N", [1224, 1000, 2000, 5000, 4096, 33])
def test_popcount_and_andpopc(N):
    A = _sketches(synth.scaled(synth.MEDIUM, 333, seed=77), N)
    B = _sketches(synth.scaled(synth.MEDIUM, 517, seed=78), N)
    Ad, Bd = dev(A.view(np.int32)), dev(B.view(np.int32))
    assert np.array_equal(bs.popcount(Ad, N).cpu().numpy(), oracle.popcount(A, N))
    assert np.array_equal(bs.andpopc(Ad, Bd, N).cpu().numpy(), oracle.andpopc(A, B, N))


def test_andpopc_tiny_full():
    A = _sketches(synth.TINY, synth.TINY_N)
    Ad = dev(A.view(np.int32))
    assert np.array_equal(bs.andpopc(Ad, Ad, synth.TINY_N).cpu().numpy(), oracle.andpopc(A, A, synth.TINY_N))


@pytest.mark.parametrize("engine", ["tc", "cuda"])
@pytest.mark.parametrize("N,na,nb", [(1024, 1100, 1300), (1224, 700, 2049), (4096, 257, 513),
                                     (5000, 130, 300), (33, 129, 257), (2, 5, 7)])
def test_andpopc_engines_tiles_and_tails(engine, N, na, nb, monkeypatch):
    """Both pair engines bit-exact vs the oracle, at sizes spanning several 128 x 256
    tensor-core tiles with ragged row tails and K padding (N not a multiple of 128)."""
    monkeypatch.setenv("BINSKETCH_ENGINE", engine)
    A = _sketches(synth.scaled(synth.LARGE, na, seed=91), N)
    B = _sketches(synth.scaled(synth.LARGE, nb, seed=92), N)
    got = bs.andpopc(dev(A.view(np.int32)), dev(B.view(np.int32)), N).cpu().numpy()
    assert np.array_equal(got, oracle.andpopc(A, B, N))


def test_andpopc_tc_saturated_and_empty_rows():
    """All-ones and all-zero sketches: counts 0 and N exactly (no int8 saturation)."""
    N = 1224
    W = (N + 31) // 32
    A = np.zeros((300, W), dtype=np.uint32)
    A[::2] = 0xFFFFFFFF
    A[::2, -1] = (1 << (N % 32)) - 1 if N % 32 else 0xFFFFFFFF
    got = bs.andpopc(dev(A.view(np.int32)), dev(A.view(np.int32)), N).cpu().numpy()
    assert np.array_equal(got, oracle.andpopc(A, A, N))
    assert got.max() == N


@pytest.fixture(params=["tc", "tc-fused", "cuda"])
def engine(request, monkeypatch):
    """Run a test on both pair engines: tensor-core (tcgen05 kind::i8) and CUDA-core (POPC). All-pairs
    estimates on the tensor cores go through the pab table + elementwise recipe ("tc") or the fused
    estimate epilogue ("tc-fused")."""
    monkeypatch.setenv("BINSKETCH_ENGINE", "cuda" if request.param == "cuda" else "tc")
    monkeypatch.setenv("BINSKETCH_EST_PAB", "0" if request.param == "tc-fused" else "1")
    return request.param


# ------------------------------------------------------------ estimate -----
def test_estimate_tiny_full_all_planes(engine):
    N, d = synth.TINY_N, synth.TINY.d
    A = _sketches(synth.TINY, N)
    Ad = dev(A.view(np.int32))
    got = bs.estimate(Ad, Ad, N, d, 15).cpu().numpy()
    ref = oracle.estimate(A, A, N, d, 15)
    assert_est_close(got, ref)


@pytest.mark.parametrize("N", synth.MEDIUM_NS)
@pytest.mark.parametrize("measure", [15, 1, 2 | 8, 4])
def test_estimate_medium_scaled(N, measure, engine):
    A = _sketches(synth.scaled(synth.MEDIUM, 300, seed=91), N)
    B = _sketches(synth.scaled(synth.MEDIUM, 450, seed=92), N)
    B[:40] = A[:40]                         # identical pairs (self-similarity exactness)
    B[40] = 0                               # empty sketch
    B[41] = 0xFFFFFFFF                      # saturated (tail bits cleared below)
    if N % 32:
        B[41, -1] = (1 << (N % 32)) - 1
    got = bs.estimate(dev(A.view(np.int32)), dev(B.view(np.int32)), N, 28_102, measure).cpu().numpy()
    ref = oracle.estimate(A, B, N, 28_102, measure)
    assert_est_close(got, ref)


# ---------------------------------------------------------------- top-k ----
def _check_topk(Q, D, N, d, measure, k, exclude_self=False):
    gi, gs = bs.topk(dev(Q.view(np.int32)), dev(D.view(np.int32)), N, d, measure, k, exclude_self=exclude_self)
    ri, rs = oracle.topk(Q, D, N, d, measure, k, exclude_self=exclude_self)
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    assert np.array_equal(gi, ri)
    assert np.array_equal(np.isnan(gs), np.isnan(rs))
    m = ~np.isnan(rs)
    assert_est_close(gs[m], rs[m])


@pytest.mark.parametrize("measure", [1, 2, 4, 8])
def test_topk_tiny(measure, engine):
    N, d = synth.TINY_N, synth.TINY.d
    A = _sketches(synth.TINY, N)
    _check_topk(A, A, N, d, measure, 10)
    _check_topk(A, A, N, d, measure, 10, exclude_self=True)


@pytest.mark.parametrize("measure", [4, 8])
def test_topk_ranking_scaled_split_merge(measure, engine):
    # few queries, many db rows: exercises db splits + the merge kernel
    N, d = synth.RANKING_N, synth.RANKING_DB.d
    D = _sketches(synth.scaled(synth.RANKING_DB, 20_000), N)
    Q = _sketches(synth.scaled(synth.RANKING_Q, 70), N)
    _check_topk(Q, D, N, d, measure, 100)


@pytest.mark.parametrize("k", [1, 50, 64, 65, 100, 192, 193, 256])
def test_topk_k_sizes_and_ties(k, engine):
    N, d = 1024, 500_000
    D = _sketches(synth.scaled(synth.LARGE, 3000), N)
    D[100:110] = D[5]                    # exact ties: lower index first
    D[2000:2300] = D[7]
    Q = D[:150].copy()
    _check_topk(Q, D, N, d, 1, k, exclude_self=True)
    _check_topk(Q, D, N, d, 4, k)


@pytest.mark.parametrize("k", [1, 50])
def test_topk_strict_bound_single_popcount_tiles(k, engine):
    """The fused IP top-k's strict tile bound (tc.cu, BSK_TOPK_STRICT): on a tile whose db rows all have
    one popcount and whose db indices all exceed the row's k-th index, only keys ABOVE the threshold are
    admitted. Whole 128-row tiles of identical sketches (at low and at high indices, so both branches of
    the index test occur), a block of empty rows (lo = 0), and sparse queries whose k-th key is 0 (T = 0,
    thousands of ties) — lists and scores bit-identical to the oracle."""
    N, d = 1024, 500_000
    D = _sketches(synth.scaled(synth.LARGE, 4000), N)
    D[40:440] = D[3]                     # ~3 whole tiles of one sketch at low indices
    D[2500:3100] = D[11]                 # ~5 whole tiles at high indices
    D[3300:3500] = 0                     # empty db rows
    Q = np.concatenate([D[:60], D[2490:2520], D[3290:3310]]).copy()
    sparse = np.zeros_like(D[:8])        # a few bits each: most keys are 0
    for i in range(8):
        sparse[i, i] = 1 << (3 * i % 32)
    Q = np.concatenate([Q, sparse])
    _check_topk(Q, D, N, d, 1, k)
    _check_topk(D, D, N, d, 1, k, exclude_self=True)


def test_topk_padding_and_empty_db(engine):
    N, d = 64, 1000
    D = _sketches(synth.CSRSpec(n=20, d=d, kind=0, p1=5, p2=20, cap=20, zipf_s=1.1, seed=3), N)
    _check_topk(D[:5], D, N, d, 2, 30)                       # k > ndb -> -1 / NaN padding
    _check_topk(D[:5], D, N, d, 1, 20, exclude_self=True)    # k > ndb - 1
    gi, gs = bs.topk(dev(D[:3].view(np.int32)), dev(D[:0].view(np.int32)), N, d, 1, 4)
    assert (gi.cpu().numpy() == -1).all() and np.isnan(gs.cpu().numpy()).all()


# ------------------------------------------------- full BASELINE sizes --
@pytest.mark.slow
def test_full_large_selfjoin_sampled():
    """configs[4] at full size in the bench launch configuration: all 2e5 sketches vs the oracle
    (bit-exact), and 2000 sampled query rows' top-50 lists (IP, self excluded) vs the oracle."""
    spec, N, k = synth.LARGE, synth.LARGE_N, synth.LARGE_K
    indptr, indices = synth.make_csr(spec)
    pi = oracle.make_pi(synth.PI_SEED, spec.d, N)
    ip, ix = csr_dev(indptr, indices)
    sk = bs.build(dev(pi.view(np.int32)), spec.d, N, ip, ix)
    gi, gs = bs.topk(sk, sk, N, spec.d, bs.IP, k, exclude_self=True)
    torch.cuda.synchronize()
    skh = u32(sk)
    ref_sk, _ = oracle.sketch(pi, spec.d, N, indptr, indices)
    assert np.array_equal(skh, ref_sk)
    rows = np.sort(np.random.default_rng(0).choice(spec.n, 2000, replace=False))
    # exclude-self top-k of row r = the top-(k+1) over every db row with r removed (or its first k
    # when r is not among them: ties with smaller indices pushed it out)
    i1, s1 = oracle.topk(skh[rows], skh, N, spec.d, bs.IP, k + 1)
    ri = np.empty((len(rows), k), dtype=np.int32)
    rs = np.empty((len(rows), k), dtype=np.float32)
    for t, r in enumerate(rows):
        keep = i1[t] != r
        ri[t] = i1[t][keep][:k]
        rs[t] = s1[t][keep][:k]
    assert np.array_equal(gi.cpu().numpy()[rows], ri)
    assert_est_close(gs.cpu().numpy()[rows], rs)


@pytest.mark.slow
def test_full_ranking():
    """configs[2] at full size: 100k db, 1000 queries, top-100 JS and COS — every query's list."""
    N, d, k = synth.RANKING_N, synth.RANKING_DB.d, synth.RANKING_K
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    dbp, dbi = synth.make_csr(synth.RANKING_DB)
    qp, qi = synth.make_csr(synth.RANKING_Q)
    D = bs.build(dev(pi.view(np.int32)), d, N, *csr_dev(dbp, dbi))
    Q = bs.build(dev(pi.view(np.int32)), d, N, *csr_dev(qp, qi))
    Dh, Qh = u32(D), u32(Q)
    assert np.array_equal(Dh, oracle.sketch(pi, d, N, dbp, dbi)[0])
    assert np.array_equal(Qh, oracle.sketch(pi, d, N, qp, qi)[0])
    for m in (bs.JS, bs.COS):
        gi, gs = bs.topk(Q, D, N, d, m, k)
        ri, rs = oracle.topk(Qh, Dh, N, d, m, k)
        assert np.array_equal(gi.cpu().numpy(), ri)
        assert_est_close(gs.cpu().numpy(), rs)


@pytest.mark.slow
def test_full_medium_planes():
    """configs[1] at full size (10k x 10k, 4 planes) for each N: every value vs the oracle."""
    spec = synth.MEDIUM
    indptr, indices = synth.make_csr(spec)
    ip, ix = csr_dev(indptr, indices)
    for N in synth.MEDIUM_NS:
        sk = bs.build_seeded(synth.PI_SEED, spec.d, N, ip, ix)
        out = bs.estimate(sk, sk, N, spec.d, 15)
        torch.cuda.synchronize()
        skh = u32(sk)
        ref = oracle.estimate(skh, skh, N, spec.d, 15)
        assert_est_close(out.cpu().numpy(), ref)
        del out, ref


@pytest.mark.slow
def test_full_buildonly():
    """configs[3] at full size (1e7 rows, 6.4e8 nonzeros): the whole 1.28 GB of sketches vs the
    oracle, bit-exact, for the pi table (binsketch_build) and in-kernel pi (binsketch_build_seeded)."""
    spec, N = synth.BUILD_ONLY, synth.BUILD_ONLY_N
    indptr, indices = synth.make_csr(spec)
    pi = oracle.make_pi(synth.PI_SEED, spec.d, N)
    ref, st = oracle.sketch(pi, spec.d, N, indptr, indices)
    assert st == 0
    ip, ix = csr_dev(indptr, indices)
    for fn in ("table", "seeded"):
        if fn == "table":
            sk = bs.build(dev(pi.view(np.int32)), spec.d, N, ip, ix)
        else:
            sk = bs.build_seeded(synth.PI_SEED, spec.d, N, ip, ix)
        bs.device_status()
        assert np.array_equal(u32(sk), ref), fn
        del sk


@pytest.mark.parametrize("qsort", ["1", "0"])
@pytest.mark.parametrize("measure", [1, 2, 4, 8])
def test_topk_query_sort_paths(measure, qsort, monkeypatch):
    """The fused top-k with queries popcount-sorted (default for JS / COS / HAM on >= 16384 queries)
    and without, on both db sort directions (descending for IP, ascending otherwise): identical lists."""
    monkeypatch.setenv("BINSKETCH_TC_QSORT", qsort)
    N, d = 1024, 500_000
    D = _sketches(synth.scaled(synth.LARGE, 2500), N)
    D[300:340] = D[11]                   # ties across the sorted order
    Q = D[:700].copy()
    _check_topk(Q, D, N, d, measure, 50, exclude_self=True)


@pytest.mark.parametrize("k", [20, 100])
def test_topk_several_measures_in_one_call(k, engine):
    """measure mask with several bits: lists stacked in IP, HAM, JS, COS order, each identical to
    the single-measure result (one AND-popcount table for all on the tensor-core pab path)."""
    N, d = synth.RANKING_N, synth.RANKING_DB.d
    D = _sketches(synth.scaled(synth.RANKING_DB, 3000), N)
    Q = _sketches(synth.scaled(synth.RANKING_Q, 150), N)
    Qd, Dd = dev(Q.view(np.int32)), dev(D.view(np.int32))
    for ms in ((bs.IP, bs.JS, bs.COS), (bs.JS, bs.COS), (bs.IP, bs.HAM, bs.JS, bs.COS)):
        # pab path: measures scored two per pass (pairs, plus a single for an odd count)
        mask = 0
        for m in ms:
            mask |= m
        gi, gs = bs.topk(Qd, Dd, N, d, mask, k, exclude_self=len(ms) == 2)
        assert gi.shape == (len(ms), 150, k)
        for t, m in enumerate(ms):
            ri, rs = oracle.topk(Q, D, N, d, m, k, exclude_self=len(ms) == 2)
            assert np.array_equal(gi[t].cpu().numpy(), ri)
            assert_est_close(gs[t].cpu().numpy(), rs)


@pytest.mark.parametrize("measure", [bs.JS, bs.COS])
def test_topk_pab_single_split_direct_outputs(measure, monkeypatch):
    """k > 64 takes the tensor-core pab table + threshold top-k; with more queries than one wave of
    warps the launcher picks ONE db split per query and the kernel writes the lists directly (no
    merge). Ties and duplicated db rows included."""
    monkeypatch.setenv("BINSKETCH_ENGINE", "tc")
    N, d = synth.RANKING_N, synth.RANKING_DB.d
    D = _sketches(synth.scaled(synth.RANKING_DB, 700, seed=57), N)
    D[40:60] = D[3]
    Q = _sketches(synth.scaled(synth.RANKING_Q, 4000, seed=58), N)
    _check_topk(Q, D, N, d, measure, 100)


@pytest.mark.parametrize("path", ["fused-screen", "pab-screen", "pab-pretest"])
def test_topk_pab_screen_paths(path, monkeypatch):
    """Top-k beyond the fused kernel (k > 64 or N > 6143): the fused tensor-core screen with
    survivor lists (K4d), the pab-table integer-screen kernel (K4c,
    BINSKETCH_TOPK_SCREEN=0) and the pab-table pre-test kernel (K4b, also BINSKETCH_PAB_SCREEN=0)
    on the cases that leave the common path: a query whose 700 exact copies in the db all tie
    above its threshold (buffer overflow -> barrier-stepped re-walk), one with 9000 copies (pass-2
    survivors beyond the scratch slot -> screened re-walk), an empty query row, an unaligned db
    (ndb % 4 != 0), self exclusion, every measure alone and all four together."""
    monkeypatch.setenv("BINSKETCH_ENGINE", "tc")
    if path != "fused-screen":
        monkeypatch.setenv("BINSKETCH_TOPK_SCREEN", "0")
    monkeypatch.setenv("BINSKETCH_PAB_SCREEN", "0" if path == "pab-pretest" else "1")
    N, d = synth.RANKING_N, synth.RANKING_DB.d
    D = _sketches(synth.scaled(synth.RANKING_DB, 12_003, seed=71), N)
    D[1000:1700] = D[7]
    D[2000:11000] = D[8]
    D[5] = 0
    Q = D[:40].copy()
    for m in (bs.IP, bs.HAM, bs.JS, bs.COS):
        _check_topk(Q, D, N, d, m, 100, exclude_self=True)
    _check_topk(Q, D[:12_000], N, d, bs.JS, 256)
    Qd, Dd = dev(Q.view(np.int32)), dev(D.view(np.int32))
    gi, gs = bs.topk(Qd, Dd, N, d, bs.IP | bs.HAM | bs.JS | bs.COS, 90)
    for t, m in enumerate((bs.IP, bs.HAM, bs.JS, bs.COS)):
        ri, rs = oracle.topk(Q, D, N, d, m, 90)
        assert np.array_equal(gi[t].cpu().numpy(), ri)
        assert_est_close(gs[t].cpu().numpy(), rs)


@pytest.mark.parametrize("path", ["fused-screen", "pab-screen"])
def test_topk_screen_small_and_padded(path, monkeypatch):
    """Top-k beyond the fused kernel on degenerate shapes: fewer db rows than k (lists padded with
    -1 / NaN), a single query, a db smaller than the threshold sample, an all-zero query, self
    exclusion with k > ndb - 1, an odd sketch length (ragged last word)."""
    monkeypatch.setenv("BINSKETCH_ENGINE", "tc")
    if path != "fused-screen":
        monkeypatch.setenv("BINSKETCH_TOPK_SCREEN", "0")
    d = synth.RANKING_DB.d
    for N, ndb, nq in ((4096, 50, 7), (4095, 300, 1), (1000, 999, 30)):
        D = _sketches(synth.scaled(synth.RANKING_DB, ndb, seed=90 + ndb), N)
        Q = D[: max(nq, 1)].copy()
        Q[0] = 0
        _check_topk(Q, D, N, d, bs.JS, 100)
        _check_topk(D, D, N, d, bs.COS, 120, exclude_self=True)
        _check_topk(Q, D, N, d, bs.IP | 0, 90)


def test_topk_screen_extremes():
    """The fused-screen top-k at its limits: N = 16383 (14-bit table entries), k = 256, all four
    measures in one call (three and four tables per pb), an empty and a saturated db row, a
    one-popcount cluster, more queries than 4 x 148 list-kernel slots, self exclusion."""
    N, d = 16383, 60_000
    spec = synth.CSRSpec(n=3000, d=d, kind=1, p1=150, p2=1.0, cap=900, zipf_s=1.05, seed=97)
    D = _sketches(spec, N)
    D[5] = 0
    D[6] = 0xFFFFFFFF
    D[6, -1] = (1 << (N % 32)) - 1
    D[100:160] = D[7]
    Q = D[:700].copy()
    Qd, Dd = dev(Q.view(np.int32)), dev(D.view(np.int32))
    for ms, k in (((bs.IP, bs.HAM, bs.JS, bs.COS), 256), ((bs.IP, bs.JS, bs.COS), 130)):
        mask = 0
        for m in ms:
            mask |= m
        gi, gs = bs.topk(Qd, Dd, N, d, mask, k, exclude_self=True)
        for t, m in enumerate(ms):
            ri, rs = oracle.topk(Q, D, N, d, m, k, exclude_self=True)
            assert np.array_equal(gi[t].cpu().numpy(), ri)
            g, rr = gs[t].cpu().numpy(), rs
            assert np.array_equal(np.isnan(g), np.isnan(rr))
            assert_est_close(g[~np.isnan(rr)], rr[~np.isnan(rr)])


@pytest.mark.parametrize("k, N", [(100, 4096), (50, 1024)])
def test_topk_graph_replay(k, N, monkeypatch):
    """binsketch_topk replays a captured CUDA graph when called again with the same buffers: the
    replay computes on the buffers' CURRENT contents (new queries and db rows in place), and a
    changed BINSKETCH_* knob selects a new capture (here: the pab-table path instead of the fused
    screen, or the CUDA-core engine); every result identical to the oracle."""
    monkeypatch.setenv("BINSKETCH_ENGINE", "tc")
    d = synth.RANKING_DB.d
    D1 = _sketches(synth.scaled(synth.RANKING_DB, 3000, seed=101), N)
    D2 = _sketches(synth.scaled(synth.RANKING_DB, 3000, seed=102), N)
    Qd, Dd = dev(D1[:200].view(np.int32)), dev(D1.view(np.int32))
    oi = torch.empty((200, k), dtype=torch.int32, device="cuda")
    os_ = torch.empty((200, k), dtype=torch.float32, device="cuda")
    ws = torch.empty(bs.workspace_bytes(bs.OP_TOPK, 200, 3000, N, k), dtype=torch.uint8, device="cuda")
    cases = [(D1, None), (D2, None), (D1, ("BINSKETCH_TOPK_SCREEN", "0")), (D2, ("BINSKETCH_ENGINE", "cuda"))]
    for D, knob in cases:
        if knob:
            monkeypatch.setenv(*knob)
        Qd.copy_(dev(D[:200].view(np.int32)))
        Dd.copy_(dev(D.view(np.int32)))
        for _ in range(2):   # capture, then replay
            gi, gs = bs.topk(Qd, Dd, N, d, bs.JS, k, exclude_self=True, out_idx=oi, out_score=os_, ws=ws)
            ri, rs = oracle.topk(D[:200], D, N, d, bs.JS, k, exclude_self=True)
            assert np.array_equal(gi.cpu().numpy(), ri)
            assert_est_close(gs.cpu().numpy(), rs)


@pytest.mark.parametrize("N", [16383, 16384])
def test_topk_pab_screen_n_limit(N):
    """The integer-screen kernel's 14-bit table entries end at N = 16383; N = 16384 takes the
    pre-test pab kernel. Both exact, ties included."""
    d = 102_660
    D = _sketches(synth.scaled(synth.RANKING_DB, 1_500, seed=73), N)
    D[100:400] = D[3]
    _check_topk(D[:30].copy(), D, N, d, bs.COS, 100)


@pytest.mark.parametrize("N", [1024, 1025, 5600, 5700, 6143])
def test_topk_k64_shared_memory_boundary(N):
    """k = 64 across the fused kernel's shared-memory limit: N = 1024 keeps the query
    tile in TMEM, N = 1025 / 5600 stage it in shared memory, and N = 5700 / 6143 no longer fit
    (heaps + staged table + two stages > 227 KB) and are routed to the pab-table path: every case
    returns the oracle's lists."""
    d = 60_000
    spec = synth.CSRSpec(n=700, d=d, kind=1, p1=120, p2=1.0, cap=900, zipf_s=1.1, seed=61)
    D = _sketches(spec, N)
    D[200:230] = D[9]
    Q = D[:170].copy()
    _check_topk(Q, D, N, d, 1, 64, exclude_self=True)
    _check_topk(Q, D, N, d, 8, 64)


def test_topk_from_host_csr_measure_order():
    """topk_from_host_csr (the e2e call): measures deduplicated and stacked in IP, HAM, JS, COS
    order whatever order the caller lists them in; lists identical to the oracle's."""
    spec = synth.scaled(synth.RANKING_DB, 900, seed=63)
    qspec = synth.scaled(synth.RANKING_Q, 60, seed=64)
    N, d, k = synth.RANKING_N, spec.d, 30
    ip, ix = synth.make_csr(spec)
    qp, qx = synth.make_csr(qspec)
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    (gi, gs), h2d, d2h = bs.topk_from_host_csr(torch.from_numpy(ip).pin_memory(), torch.from_numpy(ix).pin_memory(),
                                               torch.from_numpy(pi.view(np.int32)).pin_memory(), d, N,
                                               [bs.COS, bs.JS, bs.COS], k, q_indptr_h=torch.from_numpy(qp).pin_memory(),
                                               q_indices_h=torch.from_numpy(qx).pin_memory())
    torch.cuda.synchronize()
    assert gi.shape == (2, 60, k) and d2h == 2 * 60 * k * 8
    D, _ = oracle.sketch(pi, d, N, ip, ix)
    Q, _ = oracle.sketch(pi, d, N, qp, qx)
    for t, m in enumerate((4, 8)):          # JS plane first, then COS
        ri, rs = oracle.topk(Q, D, N, d, m, k)
        assert np.array_equal(gi[t].numpy(), ri)
        assert_est_close(gs[t].numpy(), rs)


@pytest.mark.parametrize("measure,k", [(1, 50), (4, 10)])
def test_topk_small_call_routing(measure, k, monkeypatch):
    """The product rule: calls with nq * ndb <= 2^25 pairs take the CUDA-core kernels
    (binsketch_topk_path), larger ones the fused tensor-core kernel; lists identical to the oracle
    on both sides of the boundary."""
    monkeypatch.setenv("BINSKETCH_TOPK_SMALL", "1")
    monkeypatch.delenv("BINSKETCH_ENGINE", raising=False)
    N, d = 1024, 500_000
    assert bs.topk_path(1000, 1000, N, d, k) == "cuda"
    assert bs.topk_path(5792, 5793, N, d, k) == "cuda" and bs.topk_path(5793, 5793, N, d, k) == "tc_fused"
    assert bs.topk_path(200_000, 200_000, N, d, 50) == "tc_fused"
    D = _sketches(synth.scaled(synth.LARGE, 1500), N)
    _check_topk(D, D, N, d, measure, k, exclude_self=True)       # CUDA-core
    monkeypatch.setenv("BINSKETCH_TOPK_SMALL", "0")
    assert bs.topk_path(1500, 1500, N, d, k) == "tc_fused"
    _check_topk(D, D, N, d, measure, k, exclude_self=True)       # fused tensor-core


def test_topk_from_host_csr_batches_streaming():
    """topk_from_host_csr_batches (the bench's e2e leg): several DIFFERENT host batches streamed with
    overlapped copies — every batch's lists equal the oracle's for that batch (a buffer handed over
    too early or a copy racing the compute would mix batches). Self-join and separate-query forms."""
    N, k = 1024, 20
    got = {}
    specs = [synth.scaled(synth.LARGE, 700, seed=70 + i) for i in range(4)]
    d = specs[0].d
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    pin = lambda a: torch.from_numpy(a).pin_memory()
    csr = [synth.make_csr(sp) for sp in specs]
    batches = [(pin(ip), pin(ix)) for ip, ix in csr]
    h2d, d2h = bs.topk_from_host_csr_batches(batches, pin(pi.view(np.int32)), d, N, bs.IP, k, exclude_self=True,
                                             on_result=lambda i, r: got.__setitem__(i, (r[0].clone(), r[1].clone())))
    assert sorted(got) == [0, 1, 2, 3] and d2h == 700 * k * 8
    for i, (ip, ix) in enumerate(csr):
        D, _ = oracle.sketch(pi, d, N, ip, ix)
        ri, rs = oracle.topk(D, D, N, d, 1, k, exclude_self=True)
        assert np.array_equal(got[i][0].numpy(), ri)
        assert_est_close(got[i][1].numpy(), rs)
    # separate query CSR, two measures
    got.clear()
    qcsr = [synth.make_csr(synth.scaled(synth.LARGE, 90, seed=90 + i)) for i in range(3)]
    batches = [(pin(ip), pin(ix), pin(qp), pin(qx)) for (ip, ix), (qp, qx) in zip(csr[:3], qcsr)]
    bs.topk_from_host_csr_batches(batches, pin(pi.view(np.int32)), d, N, [bs.COS, bs.JS], k,
                                  on_result=lambda i, r: got.__setitem__(i, (r[0].clone(), r[1].clone())))
    for i in range(3):
        D, _ = oracle.sketch(pi, d, N, *csr[i])
        Q, _ = oracle.sketch(pi, d, N, *qcsr[i])
        for t, m in enumerate((4, 8)):
            ri, rs = oracle.topk(Q, D, N, d, m, k)
            assert np.array_equal(got[i][0][t].numpy(), ri)
            assert_est_close(got[i][1][t].numpy(), rs)


def test_schedule_independence_stress(monkeypatch):
    """Race / ordering stress in place of compute-sanitizer (closed on this pool,
    profiles/r02_sanitize_memcheck_refused.log): the same inputs through every schedule knob —
    persistent grid size, ring depth, db chunk size, forced heap chaining across chunks, CTA pairs —
    must give bit-identical sketches, AND-popcounts and top-k lists, equal to the oracle's.
    A missing barrier, a racy shared-memory OR or a heap update lost between the two epilogue
    groups would show up as a schedule-dependent result."""
    spec = synth.scaled(synth.LARGE, 2600, seed=71)
    indptr, indices = synth.make_csr(spec)
    N, d = synth.LARGE_N, spec.d
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    ref_sk, _ = oracle.sketch(pi, d, N, indptr, indices)
    ref_i, ref_s = oracle.topk(ref_sk[:700], ref_sk, N, d, 1, 50)
    ref_j, _ = oracle.topk(ref_sk[:700], ref_sk, N, d, 4, 20)
    ip, ix = csr_dev(indptr, indices)
    knobs = [{}, {"BINSKETCH_TC_GRID": "7"}, {"BINSKETCH_TC_STAGES": "2"}, {"BINSKETCH_TC_CHUNK_KB": "384"},
             {"BINSKETCH_TC_CHUNK_KB": "256", "BINSKETCH_TC_CHAIN": "1"},
             {"BINSKETCH_TC_CHUNK_KB": "256", "BINSKETCH_TC_CHAIN": "1", "BINSKETCH_TC_GRID": "3"},
             {"BINSKETCH_TC_ATM": "0", "BINSKETCH_TC_CG": "2"}, {"BINSKETCH_BUILD_MODE": "global"}]
    for kn in knobs:
        for key, val in kn.items():
            monkeypatch.setenv(key, val)
        sk = bs.build(dev(pi.view(np.int32)), d, N, ip, ix)
        assert np.array_equal(u32(sk), ref_sk), kn
        gi, gs = bs.topk(sk[:700], sk, N, d, 1, 50)
        assert np.array_equal(gi.cpu().numpy(), ref_i), kn
        assert_est_close(gs.cpu().numpy(), ref_s)
        gj, _ = bs.topk(sk[:700], sk, N, d, 4, 20)
        assert np.array_equal(gj.cpu().numpy(), ref_j), kn
        bs.device_status()
        for key in kn:
            monkeypatch.delenv(key)
