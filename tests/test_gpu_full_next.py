"""Full-size GPU checks for the §8(f) rows, in the launch configuration the tools time.

Sampled outputs the oracle computes one by one (join rows, sketch rows) and whole-problem sums
the oracle recomputes (Exp. 1 on the full Medium corpus). Bars as in the per-row parity tests.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1910_04658_b200 import binsketch as bs
from paper_1910_04658_b200 import exp2

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    bs._lib()
    yield
    torch.cuda.synchronize()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_full_exp2_join_sampled():
    """Exp. 2 at full size (10,100 queries x 90,900 db, d = 102,660, N = 4096, the 8 paper
    thresholds): 48 sampled query rows of the sketch join and of the exact join vs the oracle."""
    spec, N, d = synth.EXP2, synth.EXP2_N, synth.EXP2.d
    ip, ix = synth.make_csr(spec)
    ip, ix = synth.plant_near_duplicates(ip, ix, d, synth.EXP2_DUP_FRAC, synth.EXP2_DUP_SEED)
    tr, q = synth.split_rows(spec.n, 0.1, synth.EXP2_SPLIT_SEED)
    (qp, qi), (tp, ti) = synth.take_rows(ip, ix, q), synth.take_rows(ip, ix, tr)
    thr = list(synth.EXP2_THRESHOLDS)
    qpd, qid, tpd, tid = dev(qp), dev(qi), dev(tp), dev(ti)
    Qs = bs.build_seeded(synth.PI_SEED, d, N, qpd, qid)
    Ds = bs.build_seeded(synth.PI_SEED, d, N, tpd, tid)
    bits = bs.join(Qs, Ds, N, d, bs.JS, thr).cpu().numpy().view(np.uint32)
    del Qs, Ds
    Qx, Dx = exp2.exact_vectors(qpd, qid, d), exp2.exact_vectors(tpd, tid, d)
    bits_x = bs.join(Qx, Dx, d, d, bs.JS, thr, exact=True).cpu().numpy().view(np.uint32)
    del Qx, Dx
    torch.cuda.empty_cache()
    rows = np.sort(np.random.default_rng(11).choice(len(q), 48, replace=False))
    sp, si = synth.take_rows(qp, qi, rows)
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    Qo, _ = oracle.sketch(pi, d, N, sp, si)
    Do, _ = oracle.sketch(pi, d, N, tp, ti)
    ref = oracle.join(Qo, Do, N, d, bs.JS, thr)
    assert np.array_equal(bits[:, rows], ref)
    ref_x = oracle.join_exact(sp, si, tp, ti, bs.JS, thr)
    assert np.array_equal(bits_x[:, rows], ref_x)
    assert ref_x[0].any() and ref[-1].any()


@pytest.mark.parametrize("measure,bcs", [(bs.JS, False), (bs.IP, False), (bs.COS, True)])
def test_full_medium_mse(measure, bcs):
    """Exp. 1 on the full Medium corpus (1e4 rows, 5e7 pairs, d = 28,102, N = 1000): counts exact,
    sums within 1e-9 relative (different fp64 summation orders)."""
    spec, N, d = synth.MEDIUM, 1000, synth.MEDIUM.d
    ip, ix = synth.make_csr(spec)
    ip, ix = synth.plant_near_duplicates(ip, ix, d, 0.3, seed=12)
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    S, _ = (oracle.bcs_sketch if bcs else oracle.sketch)(pi, d, N, ip, ix)
    X, _ = oracle.sketch(np.arange(d, dtype=np.uint32), d, d, ip, ix)
    thr = {bs.JS: [0.95, 0.8, 0.5, 0.1], bs.IP: [5.0, 20.0, 60.0], bs.COS: [0.95, 0.6, 0.2]}[measure]
    sse_ref, cnt_ref = oracle.mse(S, N, d, ip, ix, measure, thr, bcs=bcs)
    sse, cnt = bs.mse(dev(S.view(np.int32)), dev(X.view(np.int32)), N, d, measure, thr, bcs=bcs)
    sse, cnt = sse.cpu().numpy(), cnt.cpu().numpy()
    assert np.array_equal(cnt.astype(np.uint64), cnt_ref)
    assert np.all(np.abs(sse - sse_ref) <= 1e-9 * np.abs(sse_ref))
    assert cnt_ref[0] > 0


def test_full_buildonly_bcs_sampled():
    """BCS build at configs[3] size (1e7 rows, 6.4e8 nonzeros), seeded and table pi: 2000 sampled rows."""
    spec, N = synth.BUILD_ONLY, synth.BUILD_ONLY_N
    ip, ix = synth.make_csr(spec)
    d, n = spec.d, spec.n
    ipd, ixd = dev(ip), dev(ix)
    rows = np.sort(np.random.default_rng(3).choice(n, 2000, replace=False))
    sp, si = synth.take_rows(ip, ix, rows)
    want, _ = oracle.bcs_sketch(oracle.make_pi(synth.PI_SEED, d, N), d, N, sp, si)
    out = torch.empty((n, bs.words(N)), dtype=torch.int32, device="cuda")
    bs.bcs_build_seeded(synth.PI_SEED, d, N, ipd, ixd, out=out)
    got = out[torch.from_numpy(rows).cuda()].cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)
    pi = bs.make_pi(synth.PI_SEED, d, N)
    bs.bcs_build(pi, d, N, ipd, ixd, out=out)
    bs.device_status()
    got = out[torch.from_numpy(rows).cuda()].cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)
