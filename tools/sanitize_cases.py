"""Every kernel of libbinsketch on small shapes, for compute-sanitizer (memcheck / racecheck /
synccheck; one tool per run). No oracle: the sanitizer is the check. Shapes span several tiles and
ragged tails, both TC engines modes (single CTA, CTA pair), the fused top-k with the query tile in
TMEM and in shared memory, chained heaps across >= 2 db chunks, the pab-table top-k, the threshold
join, Exp. 1, BCS and the categorical path.
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1910_04658_b200 import binsketch as bs


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    bs.device_status()
    print("ok", name, flush=True)


def main():
    spec = synth.scaled(synth.LARGE, 1500, seed=5)
    ip, ix = synth.make_csr(spec)
    d, N = spec.d, 1024
    ipd, ixd = dev(ip), dev(ix)
    pi = bs.make_pi(1, d, N)
    case("make_pi", lambda: bs.make_pi(7, 5000, 1224))
    case("build seeded", lambda: bs.build_seeded(1, d, N, ipd, ixd))
    for mode in ("cache", "global"):
        os.environ["BINSKETCH_BUILD_MODE"] = mode
        case(f"build table {mode}", lambda: bs.build(pi, d, N, ipd, ixd))
    os.environ.pop("BINSKETCH_BUILD_MODE", None)
    small = synth.scaled(synth.MEDIUM, 900, seed=6)
    sp, sx = synth.make_csr(small)
    pis = bs.make_pi(1, small.d, 5000)
    case("build table smem16 generic N", lambda: bs.build(pis, small.d, 5000, dev(sp), dev(sx)))
    case("bcs build", lambda: bs.bcs_build(pis, small.d, 5000, dev(sp), dev(sx)))
    buf = torch.zeros(len(ix) + 1, dtype=torch.int32, device="cuda")
    buf[1:] = ixd
    case("build unaligned (wide fallback)", lambda: bs.build_seeded(1, d, N, ipd, buf[1:]))
    sk = bs.build(pi, d, N, ipd, ixd)
    case("popcount", lambda: bs.popcount(sk, N))
    case("andpopc", lambda: bs.andpopc(sk[:700], sk, N))
    os.environ["BINSKETCH_TC_CG"] = "2"
    case("andpopc cta pair", lambda: bs.andpopc(sk[:700], sk, N))
    case("estimate fused cta pair", lambda: (os.environ.__setitem__("BINSKETCH_EST_PAB", "0"), bs.estimate(sk[:300], sk, N, d, 15)))
    os.environ.pop("BINSKETCH_TC_CG", None)
    case("estimate fused", lambda: bs.estimate(sk[:300], sk, N, d, 15))
    os.environ.pop("BINSKETCH_EST_PAB", None)
    case("estimate pab", lambda: bs.estimate(sk[:300], sk, N, d, 15))
    case("topk fused TMEM-A", lambda: bs.topk(sk, sk, N, d, bs.IP, 50, exclude_self=True))
    os.environ["BINSKETCH_TC_CHAIN"] = "1"
    os.environ["BINSKETCH_TC_CHUNK_KB"] = "512"      # 512 rows per db chunk: >= 2 chunks, chained heaps
    case("topk fused chained heaps", lambda: bs.topk(sk, sk, N, d, bs.JS, 20, exclude_self=True))
    os.environ.pop("BINSKETCH_TC_CHAIN")
    case("topk fused db splits + merge", lambda: bs.topk(sk[:200], sk, N, d, bs.COS, 30))
    os.environ.pop("BINSKETCH_TC_CHUNK_KB")
    sk2 = bs.build_seeded(1, small.d, 2000, dev(sp), dev(sx))
    case("topk fused smem-A (N=2000)", lambda: bs.topk(sk2, sk2, 2000, small.d, bs.HAM, 40))
    case("topk pab table (k=100)", lambda: bs.topk(sk2[:300], sk2, 2000, small.d, bs.JS | bs.COS, 100))
    case("join sketch", lambda: bs.join(sk[:400], sk, N, d, bs.JS, [0.5, 0.2], exclude_self=False))
    bits = bs.join(sk[:400], sk, N, d, bs.COS, [0.6, 0.3])
    case("join list", lambda: bs.join_list(bits[0], sk[:400], sk, N, d, bs.COS))
    case("join confusion", lambda: bs.join_confusion(bits[0], bits[1], sk.shape[0]))
    case("bcs estimate", lambda: bs.bcs_estimate(sk2[:200], sk2, 2000, small.d, 15))
    ex = bs.build(torch.arange(small.d, dtype=torch.int32, device="cuda"), small.d, small.d, dev(sp), dev(sx))
    case("mse", lambda: bs.mse(sk2, ex, 2000, small.d, bs.JS, [0.5, 0.1]))
    codes = dev(np.random.default_rng(1).integers(0, 5, (500, 8)).astype(np.int32))
    offs = dev(np.arange(0, 45, 5, dtype=np.int64))
    oip, oix = bs.onehot(codes, offs)
    cat = bs.build_seeded(1, 40, 256, oip, oix)
    case("onehot + categorical", lambda: bs.categorical_estimate(cat, cat, 256, 40))
    print("all cases done", flush=True)


if __name__ == "__main__":
    main()
