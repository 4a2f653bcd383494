"""Pure-Python definitional oracle for TINY inputs (test infrastructure only).

Written straight from the paper's definitions, per bit, with no packing
tricks, so that a reader can check it against PAPER.md by eye. It is used to
pin the C++ oracle (oracle.cpp) — never by the product path.

* sketch: PAPER.md:340-344, evaluated as a brute-force preimage OR over a
  DENSE 0/1 vector: for every bucket j, OR of a[i] over all i with pi(i) = j.
* popcounts: per-bit loops (Alg. 1 lines 1-2).
* estimators: the canonical fp64 recipe (DESIGN.md R-C3) re-implemented in
  Python floats (IEEE binary64, no FMA) and the literal Alg. 1-4 with
  math.pow / math.log.
"""
from __future__ import annotations

import math

MASK64 = (1 << 64) - 1


def mix64(z: int) -> int:
    """splitmix64 finalizer, SPEC.md:63 (64-bit wrapping)."""
    z &= MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    z ^= z >> 31
    return z


def make_pi(seed: int, d: int, N: int) -> list[int]:
    """pi(i) = mix64(seed + (i+1)*gamma) mod N, i in [0,d) (R-G8)."""
    return [mix64(seed + (i + 1) * 0x9E3779B97F4A7C15) % N for i in range(d)]


def dense(support, d: int) -> list[int]:
    a = [0] * d
    for i in support:
        a[i] = 1
    return a


def sketch_bits(a_dense: list[int], pi: list[int], N: int) -> list[int]:
    """a_s[j] = OR_{i : pi(i) = j} a[i], as a list of N bits."""
    out = []
    for j in range(N):
        bit = 0
        for i in range(len(a_dense)):
            if pi[i] == j and a_dense[i] == 1:
                bit = 1
        out.append(bit)
    return out


def pack_bits(bits: list[int]) -> list[int]:
    """LSB-first uint32 words, W = ceil(N/32), tail zero (reading R-G10)."""
    W = (len(bits) + 31) // 32
    words = [0] * W
    for j, b in enumerate(bits):
        if b:
            words[j // 32] |= 1 << (j % 32)
    return words


def popcount_bits(bits: list[int]) -> int:
    return sum(1 for b in bits if b)


def and_popcount_bits(x: list[int], y: list[int]) -> int:
    return sum(1 for u, v in zip(x, y) if u and v)


def card_table(N: int, d: int) -> list[float]:
    """L[k] = log1p(-k/N)/log1p(-1/N), L[N] = d (Alg. 1 line 3; R-G11, R-G12)."""
    c = math.log1p(-1.0 / N)
    return [math.log1p(-float(k) / float(N)) / c for k in range(N)] + [float(d)]


def estimate_canonical(pa: int, pb: int, pab: int, N: int, L: list[float]):
    """(IP, HAM, JS, COS) by the canonical recipe R-C3, same operation order as oracle.cpp."""
    pu = pa + pb - pab
    La, Lb = L[pa], L[pb]
    S = La + Lb
    if pu == N and pa < N and pb < N:
        ip = 0.0
    else:
        ip = min(max(S - L[pu], 0.0), min(La, Lb))
    ham = min(max(S - 2.0 * ip, 0.0), S)
    js = 1.0 if (pa == 0 and pb == 0) else min(max(ip / (S - ip), 0.0), 1.0)
    cs = 0.0 if (pa == 0 or pb == 0) else min(max(ip / math.sqrt(La * Lb), 0.0), 1.0)
    return ip, ham, js, cs


def estimate_literal(n_as: int, n_bs: int, n_asbs: int, N: int, d: int):
    """Algorithm 1 with pow/log, then Alg. 2-4 (R-G2, R-G3, R-G15).

    Returns (raw_ip, IP, HAM, JS, COS); raw_ip is the unclamped line-4 value
    (-inf when the log argument is <= 0).
    """
    q = 1.0 - 1.0 / N

    def card(k):
        return float(d) if k == N else math.log(1.0 - k / N) / math.log(q)

    n_a, n_b = card(n_as), card(n_bs)
    arg = q ** n_a + q ** n_b + n_asbs / N - 1.0
    raw = -math.inf if arg <= 0 else n_a + n_b - math.log(arg) / math.log(q)
    ip = 0.0 if arg <= 0 else min(max(raw, 0.0), min(n_a, n_b))
    ham = min(max(n_a + n_b - 2.0 * ip, 0.0), n_a + n_b)
    if n_as == 0 and n_bs == 0:
        js = 1.0
    else:
        u = n_a + n_b - ip
        js = 0.0 if u <= 0 else min(max(ip / u, 0.0), 1.0)
    cs = 0.0 if (n_as == 0 or n_bs == 0) else min(max(ip / math.sqrt(n_a * n_b), 0.0), 1.0)
    return raw, ip, ham, js, cs


def topk_bruteforce(keys: list[float], k: int, exclude: int | None = None):
    """Indices of the k best keys under (key desc, index asc) (reading R-G17)."""
    order = sorted((j for j in range(len(keys)) if j != exclude), key=lambda j: (-keys[j], j))
    return order[:k]


# ---- BCS (Definition 2) ----
def bcs_sketch_bits(a_dense: list[int], b_map: list[int], N: int) -> list[int]:
    """u_s[j] = sum_{i : b(i) = j} u[i] mod 2, literally."""
    return [sum(a_dense[i] for i in range(len(a_dense)) if b_map[i] == j) % 2 for j in range(N)]


def bcs_table(N: int, d: int) -> list[float]:
    """B[x] = ln(1-2x/N)/ln(1-2/N) (log1p form), B[0] = 0, d once 2x >= N (R-B2)."""
    return [0.0] + [float(d) if 2 * x >= N else math.log1p(-2.0 * x / N) / math.log1p(-2.0 / N)
                    for x in range(1, N + 1)]


def bcs_estimate(pa: int, pb: int, m: int, d: int, B: list[float]):
    """(IP, HAM, JS, COS) from BCS popcounts (R-B2, R-B3), same operation order as oracle.cpp."""
    na, nb = B[pa], B[pb]
    ham = min(B[m], float(d))
    S = na + nb
    ip = min(max((S - ham) * 0.5, 0.0), min(na, nb))
    js = 1.0 if (pa == 0 and pb == 0) else min(max(ip / (S - ip), 0.0), 1.0)
    cs = 0.0 if (pa == 0 or pb == 0) else min(max(ip / math.sqrt(na * nb), 0.0), 1.0)
    return ip, ham, js, cs
