// oracle.cpp — plain, slow, obviously-correct CPU oracle for the BinSketch hot path.
//
// *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library. The
// product path (paper_1910_04658_b200/) never calls, links or imports it, and
// this file shares no code, header, table or constant generator with it.
//
// Paper: Pratap, Bera, Revanuru, "Efficient Sketching Algorithm for Sparse
// Binary Data" (arXiv 1910.04658) = /root/reference/PAPER.md. Citations are
// PAPER.md line numbers; SPEC.md lines are cited where the paper is silent
// and SPEC's reading is adopted.
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fopenmp (no fast-math, no FMA
// contraction: the canonical estimator recipe is a fixed sequence of IEEE
// fp64 operations, DESIGN.md R-C3).
//
// Parity status per function: every function below is pinned by a
// `-m "not gpu"` test (tests/test_oracle_*.py); none is "parity unpinned".
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <utility>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

// ---------------------------------------------------------------------------
// Random map pi : [d] -> [N]   (PAPER.md:341 Definition "Let pi be a random
// mapping"; generator fixed by SPEC.md:63, reading R-G8: 0-based, mod-N).
//   pi(i) = mix64(seed + (i+1) * 0x9E3779B97F4A7C15) mod N
//   mix64(z): z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
//             z *= 0x94D049BB133111EB; z ^= z>>31      (64-bit wrapping)
// ---------------------------------------------------------------------------
uint64_t orc_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

void orc_make_pi(uint64_t seed, uint64_t d, uint32_t N, uint32_t* pi) {
  for (uint64_t i = 0; i < d; ++i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    pi[i] = (uint32_t)(orc_mix64(z) % (uint64_t)N);
  }
}

// Theorem 1 sizing rule, PAPER.md:79 (N = psi * sqrt(psi/2 * ln(2/rho))),
// made an integer as in SPEC.md:54 (reading R-G5): max(2, ceil(.)).
// Returns 0 on a domain error (psi = 0 or rho not in (0,1)).
uint32_t orc_recommended_N(uint32_t psi, double rho) {
  if (psi == 0 || !(rho > 0.0 && rho < 1.0)) return 0;
  double p = (double)psi;
  double v = p * std::sqrt(p / 2.0 * std::log(2.0 / rho));
  double c = std::ceil(v);
  if (c < 2.0) c = 2.0;
  if (c > 4294967295.0) return 0;
  return (uint32_t)c;
}

uint32_t orc_words(uint32_t N) { return (N + 31u) / 32u; }

// ---------------------------------------------------------------------------
// BinSketch definition:  a_s[j] = OR_{i : pi(i) = j} a[i].
// A row is the set of its nonzero indices, stored CSR.
// Bit j of the sketch lives in word j/32 at bit position j%32 (reading R-G10,
// LSB-first uint32, W = ceil(N/32) words per row, tail bits 0).
// Returns 0, or 2 if an index is outside [0,d) / pi value outside [0,N) /
// indptr is non-monotone (the row is then left all-zero).
// ---------------------------------------------------------------------------
int orc_sketch(const uint32_t* pi, uint64_t d, uint32_t N, const int64_t* indptr,
               const int32_t* indices, uint64_t n, uint32_t* out) {
  const uint64_t W = orc_words(N);
  int status = 0;
  for (uint64_t r = 0; r < n; ++r) {
    uint32_t* row = out + r * W;
    for (uint64_t w = 0; w < W; ++w) row[w] = 0u;
    int64_t b = indptr[r], e = indptr[r + 1];
    if (e < b) { status = 2; continue; }
    for (int64_t t = b; t < e; ++t) {
      int64_t i = indices[t];
      if (i < 0 || (uint64_t)i >= d) { status = 2; continue; }
      uint32_t j = pi[i];
      if (j >= N) { status = 2; continue; }
      row[j / 32u] |= (1u << (j % 32u));   // OR of a[i] into bucket pi(i)
    }
  }
  return status;
}

// Algorithm 1 line 1: n_as = |a_s|, the number of set bits.
static int popc32(uint32_t x) {
  int c = 0;
  for (int b = 0; b < 32; ++b) c += (int)((x >> b) & 1u);
  return c;
}
static int popc_fast(uint32_t x) { return __builtin_popcount(x); }

void orc_popcount(const uint32_t* sk, uint64_t n, uint32_t N, int32_t* out) {
  const uint64_t W = orc_words(N);
  for (uint64_t r = 0; r < n; ++r) {
    int c = 0;
    for (uint64_t w = 0; w < W; ++w) c += popc32(sk[r * W + w]);
    out[r] = c;
  }
}

// Algorithm 1 line 2: n_{as,bs} = <a_s, b_s> = |a_s AND b_s|.
void orc_andpopc(const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb, uint32_t N,
                 int32_t* out) {
  const uint64_t W = orc_words(N);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)na; ++i)
    for (uint64_t j = 0; j < nb; ++j) {
      int c = 0;
      for (uint64_t w = 0; w < W; ++w) c += popc_fast(A[i * W + w] & B[j * W + w]);
      out[(uint64_t)i * nb + j] = c;
    }
}

// ---------------------------------------------------------------------------
// Cardinality table, Algorithm 1 line 3:
//   n_a = ln(1 - n_as/N) / ln(q),  q = 1 - 1/N  (paper's "n"; R-G22)
// evaluated as L[k] = log1p(-k/N) / log1p(-1/N)   (reading R-G11: log1p form)
// with saturation L[N] = d (reading R-G12).
// ---------------------------------------------------------------------------
void orc_card_table(uint32_t N, uint64_t d, double* L) {
  const double c = std::log1p(-1.0 / (double)N);
  for (uint32_t k = 0; k < N; ++k) L[k] = std::log1p(-(double)k / (double)N) / c;
  L[N] = (double)d;
}

// ---------------------------------------------------------------------------
// Canonical estimator recipe (DESIGN.md R-C3). With
// n_a = L[pa], Algorithm 1 line 4 becomes
//   arg = q^{n_a} + q^{n_b} + pab/N - 1 = 1 - pu/N,  pu = pa + pb - pab,
// so n_ab = L[pa] + L[pb] - L[pu] (identity R-C2). Clamps: SPEC.md:140
// (IP into [0, min(n_a,n_b)], log-arg <= 0 -> 0), Alg. 2 with the sign
// reading R-G2 (HAM = n_a + n_b - 2 n_ab), Alg. 3 with R-G3
// (JS = n_ab/(n_a+n_b-n_ab)), Alg. 4,
// empty-set conventions R-G15.
// out[0..3] = IP, HAM, JS, COS (fp64).
// ---------------------------------------------------------------------------
void orc_estimate_pair(int32_t pa, int32_t pb, int32_t pab, uint32_t N, const double* L,
                       double* out) {
  const int32_t pu = pa + pb - pab;
  const double La = L[pa];
  const double Lb = L[pb];
  const double S = La + Lb;
  double ip;
  if (pu == (int32_t)N && pa < (int32_t)N && pb < (int32_t)N) {
    ip = 0.0;                                   // ln(0): raw -> -inf, clamped to 0
  } else {
    double raw = S - L[pu];
    double lo = raw > 0.0 ? raw : 0.0;           // max(raw, 0)
    double cap = La < Lb ? La : Lb;              // min(n_a, n_b)
    ip = lo < cap ? lo : cap;
  }
  double two_ip = 2.0 * ip;
  double h = S - two_ip;
  h = h > 0.0 ? h : 0.0;
  double ham = h < S ? h : S;
  double js;
  if (pa == 0 && pb == 0) {
    js = 1.0;
  } else {
    double v = ip / (S - ip);
    v = v > 0.0 ? v : 0.0;
    js = v < 1.0 ? v : 1.0;
  }
  double cs;
  if (pa == 0 || pb == 0) {
    cs = 0.0;
  } else {
    double v = ip / std::sqrt(La * Lb);
    v = v > 0.0 ? v : 0.0;
    cs = v < 1.0 ? v : 1.0;
  }
  out[0] = ip;
  out[1] = ham;
  out[2] = js;
  out[3] = cs;
}

// ---------------------------------------------------------------------------
// The literal Algorithm 1-4 text (PAPER.md:398-407, 575-582, 595-602,
// 615-621) with pow/log, plus SPEC's corrections (R-G2, R-G3) and clamps.
// Used only as a cross-check of the canonical recipe (agreement <= 1e-12
// relative); the canonical recipe alone defines the bits.
// trace[0..8] = n_as, n_bs, n_asbs, n_a, n_b, n_ab, ham, js, cos.
// ---------------------------------------------------------------------------
void orc_estimate_literal(int32_t n_as, int32_t n_bs, int32_t n_asbs, uint32_t N, uint64_t d,
                          double* trace) {
  const double Nd = (double)N;
  const double q = 1.0 - 1.0 / Nd;
  auto card = [&](int32_t k) -> double {                        // Alg. 1 line 3
    if ((uint32_t)k == N) return (double)d;
    return std::log(1.0 - (double)k / Nd) / std::log(q);
  };
  const double n_a = card(n_as), n_b = card(n_bs);
  double arg = std::pow(q, n_a) + std::pow(q, n_b) + (double)n_asbs / Nd - 1.0;  // Alg. 1 line 4
  double n_ab;
  if (arg <= 0.0) {
    n_ab = 0.0;
  } else {
    n_ab = n_a + n_b - std::log(arg) / std::log(q);
    n_ab = std::min(std::max(n_ab, 0.0), std::min(n_a, n_b));
  }
  double ham = std::min(std::max(n_a + n_b - 2.0 * n_ab, 0.0), n_a + n_b);  // Alg. 2, R-G2
  double js;
  if (n_as == 0 && n_bs == 0) js = 1.0;                         // R-G15
  else {
    double u = n_a + n_b - n_ab;                                // = n_ab + ham (Alg. 3, R-G3)
    js = u <= 0.0 ? 0.0 : std::min(std::max(n_ab / u, 0.0), 1.0);
  }
  double cs = (n_as == 0 || n_bs == 0) ? 0.0
                                       : std::min(std::max(n_ab / std::sqrt(n_a * n_b), 0.0), 1.0);
  trace[0] = n_as; trace[1] = n_bs; trace[2] = n_asbs;
  trace[3] = n_a; trace[4] = n_b; trace[5] = n_ab;
  trace[6] = ham; trace[7] = js; trace[8] = cs;
}

static int popcount_row(const uint32_t* x, uint64_t W) {
  int c = 0;
  for (uint64_t w = 0; w < W; ++w) c += popc_fast(x[w]);
  return c;
}

// All-pairs estimation (north star binsketch_estimate): planes in order
// IP, HAM, JS, COS for the bits set in `measure` (1, 2, 4, 8); out is
// float[planes][na][nb], each value (float)fp64 (round to nearest).
void orc_estimate(const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb, uint32_t N,
                  uint64_t d, uint32_t measure, float* out) {
  const uint64_t W = orc_words(N);
  std::vector<double> L(N + 1);
  orc_card_table(N, d, L.data());
  std::vector<int32_t> pa(na), pb(nb);
  for (uint64_t i = 0; i < na; ++i) pa[i] = popcount_row(A + i * W, W);
  for (uint64_t j = 0; j < nb; ++j) pb[j] = popcount_row(B + j * W, W);
  int planes[4], np = 0;
  for (int m = 0; m < 4; ++m)
    if (measure & (1u << m)) planes[np++] = m;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)na; ++i)
    for (uint64_t j = 0; j < nb; ++j) {
      int pab = 0;
      for (uint64_t w = 0; w < W; ++w) pab += popc_fast(A[i * W + w] & B[j * W + w]);
      double e[4];
      orc_estimate_pair(pa[i], pb[j], pab, N, L.data(), e);
      for (int p = 0; p < np; ++p)
        out[((uint64_t)p * na + (uint64_t)i) * nb + j] = (float)e[planes[p]];
    }
}

// ---------------------------------------------------------------------------
// Top-k per query (north star; reading R-G17): a full sort of all db rows by
// (key descending, index ascending), truncated to k. key = IP / JS / COS as
// is, key = -HAM for Hamming. flags & 1 (EXCLUDE_SELF): db row j == query
// row i is skipped (self-join, R-G18). Slots beyond the available count hold
// idx = -1, score = NaN. score = (float) of the measure's value (not the key).
// nthreads <= 0: all available.
// ---------------------------------------------------------------------------
void orc_topk(const uint32_t* Q, uint64_t nq, const uint32_t* D, uint64_t ndb, uint32_t N,
              uint64_t d, uint32_t measure, uint32_t k, uint32_t flags, int32_t* out_idx,
              float* out_score, int nthreads) {
  const uint64_t W = orc_words(N);
  int m = 0;
  while (m < 4 && measure != (1u << m)) ++m;
  if (m == 4) return;
  std::vector<double> L(N + 1);
  orc_card_table(N, d, L.data());
  std::vector<int32_t> pd(ndb);
  for (uint64_t j = 0; j < ndb; ++j) pd[j] = popcount_row(D + j * W, W);
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
  nthreads = 1;
#endif
#pragma omp parallel num_threads(nthreads)
  {
    std::vector<std::pair<double, int64_t>> keys;
    std::vector<double> vals(ndb);
#pragma omp for schedule(dynamic, 1)
    for (int64_t i = 0; i < (int64_t)nq; ++i) {
      const uint32_t* qi = Q + (uint64_t)i * W;
      int pq = popcount_row(qi, W);
      keys.clear();
      for (uint64_t j = 0; j < ndb; ++j) {
        if ((flags & 1u) && (int64_t)j == i) continue;
        int pab = 0;
        for (uint64_t w = 0; w < W; ++w) pab += popc_fast(qi[w] & D[j * W + w]);
        double e[4];
        orc_estimate_pair(pq, pd[j], pab, N, L.data(), e);
        vals[j] = e[m];
        double key = (m == 1) ? -e[m] : e[m];
        keys.emplace_back(key, (int64_t)j);
      }
      auto better = [](const std::pair<double, int64_t>& a, const std::pair<double, int64_t>& b) {
        if (a.first != b.first) return a.first > b.first;
        return a.second < b.second;
      };
      uint64_t kk = std::min<uint64_t>(k, keys.size());
      std::partial_sort(keys.begin(), keys.begin() + kk, keys.end(), better);
      for (uint64_t t = 0; t < k; ++t) {
        if (t < kk) {
          out_idx[(uint64_t)i * k + t] = (int32_t)keys[t].second;
          out_score[(uint64_t)i * k + t] = (float)vals[keys[t].second];
        } else {
          out_idx[(uint64_t)i * k + t] = -1;
          out_score[(uint64_t)i * k + t] = __builtin_nanf("");
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Exact similarities of two sparse binary vectors (sorted supports), for the
// statistical tests only (Hamming per R-G2).
// out[0..3] = IP, HAM, JS, COS.
// ---------------------------------------------------------------------------
void orc_exact(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, double* out) {
  int64_t i = 0, j = 0, ip = 0;
  while (i < na && j < nb) {
    if (a[i] == b[j]) { ++ip; ++i; ++j; }
    else if (a[i] < b[j]) ++i;
    else ++j;
  }
  out[0] = (double)ip;
  out[1] = (double)(na + nb - 2 * ip);
  out[2] = (na + nb - ip) > 0 ? (double)ip / (double)(na + nb - ip) : 1.0;
  out[3] = (na > 0 && nb > 0) ? (double)ip / std::sqrt((double)na * (double)nb) : 0.0;
}

// ---------------------------------------------------------------------------
// Threshold similarity join, the retrieval step of Experiment 2 (PAPER.md:
// 690-700: "compute the points in the training partition whose similarities
// are higher than a certain threshold"; thresholds PAPER.md:697). Reading
// R-J1: pair (i, j) is reported at threshold t iff key(i,j) >= key(t), with
// key = the measure's value for IP / JS / COS and -HAM for Hamming (distance
// at most t), evaluated in fp64 exactly as top-k keys are (R-G17).
// out_bits: uint32 [nthr][nq][ceil(ndb/32)], bit j%32 of word j/32 of row i
// (LSB first, tail bits 0), plane t for thresholds[t]. flags & 1: skip j == i.
//
// orc_join: estimates from sketches by the canonical recipe (orc_estimate_pair).
// orc_join_exact: exact similarities of the uncompressed sparse rows (CSR,
// sorted supports) by the merge walk of orc_exact — the ground truth O.
// ---------------------------------------------------------------------------
static void join_set(uint32_t* out_bits, uint64_t nq, uint64_t ndb, uint32_t nthr, int m, const double* thr,
                     uint64_t i, uint64_t j, const double* e) {
  const uint64_t wpr = (ndb + 31) / 32;
  const double key = (m == 1) ? -e[m] : e[m];
  for (uint32_t t = 0; t < nthr; ++t) {
    const double tk = (m == 1) ? -thr[t] : thr[t];
    if (key >= tk) out_bits[((uint64_t)t * nq + i) * wpr + j / 32] |= 1u << (j % 32);
  }
}

void orc_join(const uint32_t* Q, uint64_t nq, const uint32_t* D, uint64_t ndb, uint32_t N, uint64_t d,
              uint32_t measure, const double* thr, uint32_t nthr, uint32_t flags, uint32_t* out_bits) {
  const uint64_t W = orc_words(N), wpr = (ndb + 31) / 32;
  int m = 0;
  while (m < 4 && measure != (1u << m)) ++m;
  std::memset(out_bits, 0, (size_t)nthr * nq * wpr * 4);
  if (m == 4) return;
  std::vector<double> L(N + 1);
  orc_card_table(N, d, L.data());
  std::vector<int32_t> pd(ndb);
  for (uint64_t j = 0; j < ndb; ++j) pd[j] = popcount_row(D + j * W, W);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < (int64_t)nq; ++i) {
    const uint32_t* qi = Q + (uint64_t)i * W;
    const int pq = popcount_row(qi, W);
    for (uint64_t j = 0; j < ndb; ++j) {
      if ((flags & 1u) && (int64_t)j == i) continue;
      int pab = 0;
      for (uint64_t w = 0; w < W; ++w) pab += popc_fast(qi[w] & D[j * W + w]);
      double e[4];
      orc_estimate_pair(pq, pd[j], pab, N, L.data(), e);
      join_set(out_bits, nq, ndb, nthr, m, thr, (uint64_t)i, j, e);
    }
  }
}

void orc_join_exact(const int64_t* qptr, const int32_t* qidx, uint64_t nq, const int64_t* dptr,
                    const int32_t* didx, uint64_t ndb, uint32_t measure, const double* thr, uint32_t nthr,
                    uint32_t flags, uint32_t* out_bits) {
  const uint64_t wpr = (ndb + 31) / 32;
  int m = 0;
  while (m < 4 && measure != (1u << m)) ++m;
  std::memset(out_bits, 0, (size_t)nthr * nq * wpr * 4);
  if (m == 4) return;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < (int64_t)nq; ++i) {
    for (uint64_t j = 0; j < ndb; ++j) {
      if ((flags & 1u) && (int64_t)j == i) continue;
      double e[4];
      orc_exact(qidx + qptr[i], qptr[i + 1] - qptr[i], didx + dptr[j], dptr[j + 1] - dptr[j], e);
      join_set(out_bits, nq, ndb, nthr, m, thr, (uint64_t)i, j, e);
    }
  }
}

// ---------------------------------------------------------------------------
// BCS parity sketch, PAPER.md:321-331 (Definition 2):
//   u_s[j] = sum_{i : b(i) = j} u[i]  (mod 2),  b = the same random map pi.
// A CSR row is read as the multiset of its entries (reading R-B1): each entry
// toggles its bucket, so a repeated index cancels.
// ---------------------------------------------------------------------------
int orc_bcs_sketch(const uint32_t* pi, uint64_t d, uint32_t N, const int64_t* indptr, const int32_t* indices,
                   uint64_t n, uint32_t* out) {
  const uint64_t W = orc_words(N);
  int status = 0;
  for (uint64_t r = 0; r < n; ++r) {
    uint32_t* row = out + r * W;
    for (uint64_t w = 0; w < W; ++w) row[w] = 0;
    if (indptr[r + 1] < indptr[r]) { status = 1; continue; }
    for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e) {
      const int64_t i = indices[e - indptr[0]];
      if (i < 0 || (uint64_t)i >= d || pi[i] >= N) { status = 1; continue; }
      const uint32_t j = pi[i];
      row[j / 32] ^= 1u << (j % 32);
    }
  }
  return status;
}

// BCS estimator table (R-B2, SPEC.md:240-243 inverted parity-collision law):
//   B[0] = 0;  B[x] = d if 2x >= N, else ln(1 - 2x/N) / ln(1 - 2/N)  (log1p form, as R-G11)
void orc_bcs_table(uint32_t N, uint64_t d, double* B) {
  B[0] = 0.0;
  for (uint32_t x = 1; x <= N; ++x)
    B[x] = (2.0 * (double)x >= (double)N) ? (double)d : std::log1p(-2.0 * (double)x / (double)N) / std::log1p(-2.0 / (double)N);
}

// BCS estimates (R-B2, R-B3) from pa = |a_s|, pb = |b_s| and m = |a_s XOR b_s|:
//   HAM = min(B[m], d); n_a = B[pa]; n_b = B[pb]; S = n_a + n_b
//   IP = min(max((S - HAM) * 0.5, 0), min(n_a, n_b))
//   JS = (pa == 0 && pb == 0) ? 1 : clamp(IP / (S - IP), 0, 1)
//   COS = (pa == 0 || pb == 0) ? 0 : clamp(IP / sqrt(n_a * n_b), 0, 1)
// out = {IP, HAM, JS, COS}.
void orc_bcs_estimate_pair(int32_t pa, int32_t pb, int32_t m, uint64_t d, const double* B, double* out) {
  const double na = B[pa], nb = B[pb];
  const double h = B[m];
  const double ham = std::min(h, (double)d);
  const double S = na + nb;
  const double ip = std::min(std::max((S - ham) * 0.5, 0.0), std::min(na, nb));
  double js, cs;
  if (pa == 0 && pb == 0) js = 1.0;
  else js = std::min(std::max(ip / (S - ip), 0.0), 1.0);
  if (pa == 0 || pb == 0) cs = 0.0;
  else cs = std::min(std::max(ip / std::sqrt(na * nb), 0.0), 1.0);
  out[0] = ip; out[1] = ham; out[2] = js; out[3] = cs;
}

// All pairs from BCS sketches; m from the XOR popcount of the words (planes as orc_estimate).
void orc_bcs_estimate(const uint32_t* A, uint64_t na, const uint32_t* Bm, uint64_t nb, uint32_t N, uint64_t d,
                      uint32_t measure, float* out) {
  const uint64_t W = orc_words(N);
  std::vector<double> T(N + 1);
  orc_bcs_table(N, d, T.data());
  int planes[4], np = 0;
  for (int m = 0; m < 4; ++m)
    if (measure & (1u << m)) planes[np++] = m;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)na; ++i) {
    const int pa = popcount_row(A + (uint64_t)i * W, W);
    for (uint64_t j = 0; j < nb; ++j) {
      const int pb = popcount_row(Bm + j * W, W);
      int x = 0;
      for (uint64_t w = 0; w < W; ++w) x += popc_fast(A[(uint64_t)i * W + w] ^ Bm[j * W + w]);
      double e[4];
      orc_bcs_estimate_pair(pa, pb, x, d, T.data(), e);
      for (int p = 0; p < np; ++p) out[((uint64_t)p * na + (uint64_t)i) * nb + j] = (float)e[planes[p]];
    }
  }
}

// ---------------------------------------------------------------------------
// Experiment 1, fidelity of the estimate: over every unordered pair
// i < j of one corpus whose TRUE similarity is at least the threshold ("we considered
// only those pairs whose similarities are higher than 0.95"; reading R-M1: >=, and for
// Hamming a distance <= t), the squared difference between the estimate and the truth:
//   count[t] = #{i<j : true(i,j) selects t},  sse[t] = sum (est(i,j) - true(i,j))^2
// (MSE = sse / count, reported as -ln MSE for JS / COS and as is for IP).
// est: the canonical BinSketch recipe from the sketches (flags & 1: BCS estimates from
// BCS sketches, R-B2); true: exact similarities of the CSR rows (orc_exact). Sums: per row i
// sequentially over j, then over i in order (fp64, independent of the thread count).
// ---------------------------------------------------------------------------
void orc_mse(const uint32_t* S, uint64_t n, uint32_t N, uint64_t d, const int64_t* indptr, const int32_t* indices,
             uint32_t measure, const double* thr, uint32_t nthr, uint32_t flags, double* sse, uint64_t* count) {
  const uint64_t W = orc_words(N);
  int m = 0;
  while (m < 4 && measure != (1u << m)) ++m;
  for (uint32_t t = 0; t < nthr; ++t) { sse[t] = 0.0; count[t] = 0; }
  if (m == 4) return;
  std::vector<double> T(N + 1);
  if (flags & 1u) orc_bcs_table(N, d, T.data()); else orc_card_table(N, d, T.data());
  std::vector<int32_t> pc(n);
  for (uint64_t i = 0; i < n; ++i) pc[i] = popcount_row(S + i * W, W);
  // per-row partial sums (each a sequential sum over j), then a sequential sum over i: the
  // same fixed order whatever the thread count
  std::vector<double> rs((size_t)n * nthr, 0.0);
  std::vector<uint64_t> rc((size_t)n * nthr, 0);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t ii = 0; ii < (int64_t)n; ++ii) {
    const uint64_t i = (uint64_t)ii;
    for (uint64_t j = i + 1; j < n; ++j) {
      double tr[4], es[4];
      orc_exact(indices + (indptr[i] - indptr[0]), indptr[i + 1] - indptr[i], indices + (indptr[j] - indptr[0]),
                indptr[j + 1] - indptr[j], tr);
      int pab = 0, px = 0;
      for (uint64_t w = 0; w < W; ++w) {
        pab += popc_fast(S[i * W + w] & S[j * W + w]);
        px += popc_fast(S[i * W + w] ^ S[j * W + w]);
      }
      if (flags & 1u) orc_bcs_estimate_pair(pc[i], pc[j], px, d, T.data(), es);
      else orc_estimate_pair(pc[i], pc[j], pab, N, T.data(), es);
      for (uint32_t t = 0; t < nthr; ++t) {
        const bool sel = (m == 1) ? (tr[m] <= thr[t]) : (tr[m] >= thr[t]);
        if (sel) {
          const double e = es[m] - tr[m];
          rs[i * nthr + t] += e * e;
          rc[i * nthr + t] += 1;
        }
      }
    }
  }
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t t = 0; t < nthr; ++t) { sse[t] += rs[i * nthr + t]; count[t] += rc[i * nthr + t]; }
}

// ---------------------------------------------------------------------------
// Categorical extension: label-encoded features (codes[r][k] in
// [0, m_k)) are one-hot encoded as the binary vector with ones at offsets[k] + codes[r][k],
// offsets = prefix sums of the cardinalities m_k (d = offsets[c]); the distance
// D(u, v) = #{k : u[k] != v[k]}. Returns 1 on a code outside [0, m_k).
// ---------------------------------------------------------------------------
int orc_onehot(const int32_t* codes, uint64_t n, uint32_t c, const int64_t* offsets, int64_t* indptr,
               int32_t* indices) {
  int status = 0;
  for (uint64_t r = 0; r <= n; ++r) indptr[r] = (int64_t)(r * c);
  for (uint64_t r = 0; r < n; ++r)
    for (uint32_t k = 0; k < c; ++k) {
      const int64_t v = codes[r * c + k];
      if (v < 0 || v >= offsets[k + 1] - offsets[k]) { status = 1; indices[r * c + k] = (int32_t)offsets[k]; continue; }
      indices[r * c + k] = (int32_t)(offsets[k] + v);
    }
  return status;
}

// D(u, v) for all pairs (the categorical distance, literally).
void orc_categorical_distance(const int32_t* U, uint64_t nu, const int32_t* V, uint64_t nv, uint32_t c, int32_t* out) {
  for (uint64_t i = 0; i < nu; ++i)
    for (uint64_t j = 0; j < nv; ++j) {
      int32_t dd = 0;
      for (uint32_t k = 0; k < c; ++k) dd += U[i * c + k] != V[j * c + k] ? 1 : 0;
      out[i * nv + j] = dd;
    }
}

// Estimated categorical distance (reading R-C1): D^ = HAM^ / 2 with HAM^ the canonical
// recipe's Hamming estimate from the one-hot sketches (the one-hot Hamming distance is
// exactly 2 D); out float[na][nb] = (float)(HAM^ * 0.5).
void orc_categorical_estimate(const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb, uint32_t N, uint64_t d,
                              float* out) {
  const uint64_t W = orc_words(N);
  std::vector<double> L(N + 1);
  orc_card_table(N, d, L.data());
  for (uint64_t i = 0; i < na; ++i) {
    const int pa = popcount_row(A + i * W, W);
    for (uint64_t j = 0; j < nb; ++j) {
      const int pb = popcount_row(B + j * W, W);
      int pab = 0;
      for (uint64_t w = 0; w < W; ++w) pab += popc_fast(A[i * W + w] & B[j * W + w]);
      double e[4];
      orc_estimate_pair(pa, pb, pab, N, L.data(), e);
      out[i * nb + j] = (float)(e[1] * 0.5);
    }
  }
}

// ---------------------------------------------------------------------------
// Exhaustive enumeration of Lemma 1's expectations: the
// mean of |a_s| and of <a_s,b_s> over ALL N^d maps pi, computed by sketching
// with every map (orc_sketch) and counting bits. a, b are sorted supports in
// [0,d). Returns -1 if N^d > 1e7.
// ---------------------------------------------------------------------------
int orc_enumerate(uint32_t d, uint32_t N, const int32_t* a, int64_t na, const int32_t* b,
                  int64_t nb, double* mean_as, double* mean_asbs) {
  double total = std::pow((double)N, (double)d);
  if (total > 1e7) return -1;
  const uint64_t W = orc_words(N);
  std::vector<uint32_t> pi(d, 0), sa(W), sb(W);
  int64_t ipa[2] = {0, na}, ipb[2] = {0, nb};
  double s1 = 0, s2 = 0;
  uint64_t count = 0;
  while (true) {
    orc_sketch(pi.data(), d, N, ipa, a, 1, sa.data());
    orc_sketch(pi.data(), d, N, ipb, b, 1, sb.data());
    int pa_, pab_;
    orc_popcount(sa.data(), 1, N, &pa_);
    orc_andpopc(sa.data(), 1, sb.data(), 1, N, &pab_);
    s1 += pa_;
    s2 += pab_;
    ++count;
    // next map in lexicographic order
    uint32_t t = 0;
    while (t < d) {
      if (++pi[t] < N) break;
      pi[t] = 0;
      ++t;
    }
    if (t == d) break;
  }
  *mean_as = s1 / (double)count;
  *mean_asbs = s2 / (double)count;
  return 0;
}

}  // extern "C"
