// bsk_estimator.cuh — the canonical fp64 estimator recipe (DESIGN.md R-C3) and the
// top-k order, shared by the CUDA-core (pairs.cu) and tensor-core (tc.cu) pair engines.
// Every fp64 operation is an explicit round-to-nearest intrinsic, and both units are
// compiled with -fmad=false, so no contraction can change a bit relative to the oracle.
#pragma once
#include <cstdint>

namespace bsk {

// ----------------------------------------------------------- estimator ----
struct Est {
  double ip, ham, js, cs;
};

// The canonical recipe; `need` is the measure mask actually consumed.
__device__ __forceinline__ Est estimate_pair(int pa, int pb, int pab, int N, const double* __restrict__ L,
                                             uint32_t need) {
  Est r;
  const int pu = pa + pb - pab;
  const double La = L[pa];
  const double Lb = L[pb];
  const double S = __dadd_rn(La, Lb);
  double ip;
  if (pu == N && pa < N && pb < N) {
    ip = 0.0;
  } else {
    double raw = __dsub_rn(S, L[pu]);
    double lo = raw > 0.0 ? raw : 0.0;
    double cap = La < Lb ? La : Lb;
    ip = lo < cap ? lo : cap;
  }
  r.ip = ip;
  r.ham = 0.0;
  r.js = 0.0;
  r.cs = 0.0;
  if (need & 2u) {
    double h = __dsub_rn(S, __dmul_rn(2.0, ip));
    h = h > 0.0 ? h : 0.0;
    r.ham = h < S ? h : S;
  }
  if (need & 4u) {
    if (pa == 0 && pb == 0) {
      r.js = 1.0;
    } else {
      double v = __ddiv_rn(ip, __dsub_rn(S, ip));
      v = v > 0.0 ? v : 0.0;
      r.js = v < 1.0 ? v : 1.0;
    }
  }
  if (need & 8u) {
    if (pa == 0 || pb == 0) {
      r.cs = 0.0;
    } else {
      double v = __ddiv_rn(ip, __dsqrt_rn(__dmul_rn(La, Lb)));
      v = v > 0.0 ? v : 0.0;
      r.cs = v < 1.0 ? v : 1.0;
    }
  }
  return r;
}


// BCS (Definition 2) estimates from parity sketches (readings R-B2, R-B3;
// the paper gives the sketch, not an estimator): a bucket's parity differs between a_s and
// b_s with probability (1 - (1-2/N)^h)/2 for h = |a XOR b|, so with the table
// B[x] = log1p(-2x/N)/log1p(-2/N) (B[0] = 0, B[x] = d once 2x >= N) and
// m = |a_s XOR b_s| = pa + pb - 2 pab:
//   HAM = min(B[m], d);  n_a = B[pa], n_b = B[pb] (the same law for |a|);  S = n_a + n_b
//   IP  = min(max((S - HAM)/2, 0), min(n_a, n_b));  JS / COS as in the BinSketch recipe.
__device__ __forceinline__ Est bcs_estimate_pair(int pa, int pb, int pab, double dcap, const double* __restrict__ B,
                                                 uint32_t need) {
  Est r;
  const double na = B[pa], nb = B[pb];
  const double h = B[pa + pb - 2 * pab];
  const double ham = h < dcap ? h : dcap;
  const double S = __dadd_rn(na, nb);
  double ip = __dmul_rn(__dsub_rn(S, ham), 0.5);
  ip = ip > 0.0 ? ip : 0.0;
  const double cap = na < nb ? na : nb;
  ip = ip < cap ? ip : cap;
  r.ip = ip;
  r.ham = ham;
  r.js = 0.0;
  r.cs = 0.0;
  if (need & 4u) {
    if (pa == 0 && pb == 0) {
      r.js = 1.0;
    } else {
      double v = __ddiv_rn(ip, __dsub_rn(S, ip));
      v = v > 0.0 ? v : 0.0;
      r.js = v < 1.0 ? v : 1.0;
    }
  }
  if (need & 8u) {
    if (pa == 0 || pb == 0) {
      r.cs = 0.0;
    } else {
      double v = __ddiv_rn(ip, __dsqrt_rn(__dmul_rn(na, nb)));
      v = v > 0.0 ? v : 0.0;
      r.cs = v < 1.0 ? v : 1.0;
    }
  }
  return r;
}

// Necessary condition for measure_key(estimate_pair(...)) >= t (t finite), evaluated without
// the division / square root of the JS and COS keys; the 1e-9 relative margins absorb every
// rounding difference, so a pair it rejects is certainly below t.
__device__ __forceinline__ bool pretest_keep(int pa, int pb, int pab, int N, const double* __restrict__ L, uint32_t m,
                                             double t) {
  const int pu = pa + pb - pab;
  const double La = L[pa], Lb = L[pb];
  const double S = La + Lb;
  double ip;
  if (pu == N && pa < N && pb < N) {
    ip = 0.0;
  } else {
    ip = S - L[pu];
    ip = ip > 0.0 ? ip : 0.0;
    ip = fmin(ip, fmin(La, Lb));
  }
  const double eps = 1e-9;
  if (m == 1u) return ip >= t - eps * fmax(1.0, fabs(t));
  if (m == 2u) return 2.0 * ip - S >= t - eps * fmax(1.0, fabs(t));
  if (t <= 0.0) return true;
  if (m == 4u) {
    if (pa == 0 && pb == 0) return true;
    return ip * (1.0 + t) * (1.0 + eps) >= t * S;        // JS = ip/(S-ip) >= t
  }
  if (pa == 0 || pb == 0) return true;
  return ip * ip * (1.0 + eps) >= t * t * (La * Lb);      // COS = ip/sqrt(La Lb) >= t
}

// Exact similarity key of two uncompressed rows from (|a|, |b|, |a AND b|) — the threshold
// join's ground truth (Exp. 2's O): the recipe above with L = identity
// (no estimation), keys as in measure_key (-HAM for Hamming). Integers up to 2^31 are exact
// in fp64, so IP and HAM are exact and JS / COS are one correctly rounded division.
__device__ __forceinline__ double exact_key(int pa, int pb, int pab, uint32_t m) {
  const double ip = (double)pab;
  const double S = __dadd_rn((double)pa, (double)pb);
  if (m == 1u) return ip;
  if (m == 2u) return -__dsub_rn(S, __dmul_rn(2.0, ip));
  if (m == 4u) return (pa == 0 && pb == 0) ? 1.0 : __ddiv_rn(ip, __dsub_rn(S, ip));
  return (pa == 0 || pb == 0) ? 0.0 : __ddiv_rn(ip, __dsqrt_rn(__dmul_rn((double)pa, (double)pb)));
}

// Order (reading R-G17): a before b iff a.key > b.key, or equal keys and
// a.idx < b.idx. Sentinel (key = -inf, idx = INT_MAX) sorts last.
__device__ __forceinline__ bool before(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

constexpr int kSentinelIdx = 0x7fffffff;

__device__ __forceinline__ double measure_key(const Est& e, uint32_t m) {
  return m == 1u ? e.ip : m == 2u ? -e.ham : m == 4u ? e.js : e.cs;
}
__device__ __forceinline__ float key_to_score(double key, uint32_t m) {
  return __double2float_rn(m == 2u ? -key : key);
}


// First plane of the threshold join (thresholds as keys, descending: planes t >= t0 have
// key >= tkey[t]) for the estimated JS or COS key, deciding each threshold division-free where
// that is certain: with the recipe's IP part (the same fp64 operations as estimate_pair),
// JS >= t <=> ip (1 + t) >= t S and COS >= t <=> ip^2 >= t^2 La Lb (t in (0, 1]); a 1e-12
// relative margin on both sides covers every rounding of the recipe's quotient, and a threshold
// inside the margin is settled by the exact key (measure_key(estimate_pair)). Returns the same
// t0 as scanning with the exact key.
__device__ __forceinline__ uint32_t join_first_plane(int pa, int pb, int pab, int N, const double* __restrict__ L,
                                                     uint32_t m, const double* tkey, uint32_t nthr) {
  const int pu = pa + pb - pab;
  const double La = L[pa], Lb = L[pb];
  const double S = __dadd_rn(La, Lb);
  double ip;
  if (pu == N && pa < N && pb < N) {
    ip = 0.0;
  } else {
    const double raw = __dsub_rn(S, L[pu]);
    const double lo = raw > 0.0 ? raw : 0.0;
    const double cap = La < Lb ? La : Lb;
    ip = lo < cap ? lo : cap;
  }
  bool special = (m == 4u) ? (pa == 0 && pb == 0) || !(__dsub_rn(S, ip) > 0.0) : (pa == 0 || pb == 0);
  const double lhs_c = m == 4u ? ip : __dmul_rn(ip, ip);
  const double q = m == 4u ? S : __dmul_rn(La, Lb);
  uint32_t t0 = nthr;
  while (t0 > 0 && !special) {
    const double t = tkey[t0 - 1];
    if (t <= 0.0) { --t0; continue; }          // keys are clamped to [0, 1]
    if (t > 1.0) break;
    double lhs, rhs;
    if (m == 4u) { lhs = __dmul_rn(lhs_c, __dadd_rn(1.0, t)); rhs = __dmul_rn(t, q); }
    else { lhs = lhs_c; rhs = __dmul_rn(__dmul_rn(t, t), q); }
    if (lhs >= __dmul_rn(rhs, 1.0 + 1e-12)) { --t0; continue; }   // certainly key >= t
    if (lhs <= __dmul_rn(rhs, 1.0 - 1e-12)) break;                 // certainly key < t
    special = true;                                                // within the margin: exact key
  }
  if (special) {
    const double key = measure_key(estimate_pair(pa, pb, pab, N, L, m), m);
    while (t0 > 0 && key >= tkey[t0 - 1]) --t0;
  }
  return t0;
}

}  // namespace bsk
