// synth.cpp — seeded synthetic sparse-binary CSR generator.
//
// TEST/BENCH INPUT INFRASTRUCTURE. This module holds none of BinSketch's
// arithmetic (no random map pi, no sketching, no estimator). It only produces
// the CSR inputs that both the CPU oracle (oracle/) and the CUDA path
// (paper_1910_04658_b200/) consume, so that both sides see identical data.
//
// Recipe (SURVEY.md §8(d) "Synthetic inputs"):
//   * counter-based RNG: one splitmix64-style stream per row, keyed by
//     (data_seed, row) -> output independent of thread count / scheduling;
//   * feature popularity Zipf(s) over ranks r = 1..d, P(r) ∝ r^-s, sampled by
//     inverse CDF (fp64 prefix sums in fixed order + guide table + scan);
//   * rank -> feature id through a seeded Fisher–Yates permutation (perm=1,
//     default: ids uncorrelated with frequency, like a real vocabulary) or the
//     identity id = r-1 (perm=0);
//   * nnz per row: uniform on {lo..hi} (kind 0) or
//     clamp(round(exp(mu + sigma Z)), 1, cap) with mu = ln(mean) - sigma^2/2
//     (kind 1, lognormal);
//   * exactly nnz DISTINCT indices per row (draw until distinct), sorted
//     ascending; int64 indptr, int32 indices.
// The stand-in for the paper's UCI bag-of-words corpora,
// which are not available here.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

// A generic 64-bit counter-based stream (splitmix64 construction). This is the
// data generator's own RNG; the method's pi map is implemented separately and
// independently on each side (oracle/ and the CUDA library).
struct Stream {
  uint64_t s;
  static uint64_t fin(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  Stream(uint64_t seed, uint64_t ctr) : s(fin(seed * 0xD1342543DE82EF95ULL + fin(ctr + 0x632BE59BD9B4E019ULL))) {}
  uint64_t next() { s += 0x9E3779B97F4A7C15ULL; return fin(s); }
  double u01() { return (double)(next() >> 11) * 0x1.0p-53; }           // [0,1)
  double u01_open() { return ((double)(next() >> 11) + 0.5) * 0x1.0p-53; } // (0,1)
};

struct Zipf {
  std::vector<double> cdf;     // cdf[r] = sum_{t<=r+1} t^-s, r = 0..d-1
  std::vector<uint32_t> guide; // guide[g] = first r with cdf[r] > g/G*total
  double total = 0;
  void init(uint64_t d, double s) {
    cdf.resize(d);
    double acc = 0;
    for (uint64_t r = 0; r < d; ++r) { acc += std::pow((double)(r + 1), -s); cdf[r] = acc; }
    total = acc;
    uint64_t G = d;
    guide.resize(G + 1);
    uint64_t r = 0;
    for (uint64_t g = 0; g <= G; ++g) {
      double thr = (double)g / (double)G * total;
      while (r + 1 < d && cdf[r] <= thr) ++r;
      guide[g] = (uint32_t)r;
    }
  }
  uint32_t sample(Stream& st) const {
    double u = st.u01() * total;
    uint64_t G = guide.size() - 1;
    uint64_t g = (uint64_t)(u / total * (double)G);
    if (g > G) g = G;
    uint64_t r = guide[g];
    // guide[g] is a lower bound; scan forward (and guard backwards for rounding)
    while (r > 0 && cdf[r - 1] > u) --r;
    while (r + 1 < cdf.size() && cdf[r] <= u) ++r;
    return (uint32_t)r;
  }
};

int64_t row_nnz(Stream& st, int kind, double p1, double p2, int64_t cap, uint64_t d) {
  int64_t m;
  if (kind == 0) {
    int64_t lo = (int64_t)p1, hi = (int64_t)p2;
    m = lo + (int64_t)(st.next() % (uint64_t)(hi - lo + 1));
  } else {
    double sigma = p2, mu = std::log(p1) - 0.5 * sigma * sigma;
    double u1 = st.u01_open(), u2 = st.u01();
    double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    double v = std::exp(mu + sigma * z);
    m = (int64_t)std::llround(v);
    if (m < 1) m = 1;
    if (m > cap) m = cap;
  }
  if (m > (int64_t)d) m = (int64_t)d;
  if (m < 0) m = 0;
  return m;
}

}  // namespace

extern "C" {

// Phase 1: nnz of every row (int64 counts). kind: 0 uniform{p1..p2}, 1 lognormal(mean p1, sigma p2, cap).
void synth_row_nnz(uint64_t n, uint64_t d, int kind, double p1, double p2, int64_t cap,
                   uint64_t data_seed, int64_t* counts) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)n; ++r) {
    Stream st(data_seed, (uint64_t)r);
    counts[r] = row_nnz(st, kind, p1, p2, cap, d);
  }
}

// Phase 2: fill indices given indptr (prefix sums of synth_row_nnz). perm: 0 identity, 1 seeded permutation.
int synth_fill(uint64_t n, uint64_t d, int kind, double p1, double p2, int64_t cap, double zipf_s,
               int perm, uint64_t data_seed, const int64_t* indptr, int32_t* indices) {
  if (d == 0 || d > 0x7fffffffULL) return 1;
  Zipf z;
  z.init(d, zipf_s);
  std::vector<uint32_t> id(d);
  for (uint64_t i = 0; i < d; ++i) id[i] = (uint32_t)i;
  if (perm) {
    Stream ps(data_seed ^ 0xA5A5A5A5DEADBEEFULL, 0xFFFFFFFFFFFFULL);
    for (uint64_t i = d - 1; i > 0; --i) {
      uint64_t j = ps.next() % (i + 1);
      std::swap(id[i], id[j]);
    }
  }
  int bad = 0;
#pragma omp parallel
  {
    std::vector<uint32_t> buf;
#pragma omp for schedule(dynamic, 256) reduction(| : bad)
    for (int64_t r = 0; r < (int64_t)n; ++r) {
      Stream st(data_seed, (uint64_t)r);
      int64_t m = row_nnz(st, kind, p1, p2, cap, d);
      if (indptr[r + 1] - indptr[r] != m) { bad |= 1; continue; }
      buf.clear();
      while ((int64_t)buf.size() < m) {
        int64_t need = m - (int64_t)buf.size();
        for (int64_t t = 0; t < need; ++t) buf.push_back(id[z.sample(st)]);
        std::sort(buf.begin(), buf.end());
        buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
      }
      int32_t* dst = indices + indptr[r];
      for (int64_t t = 0; t < m; ++t) dst[t] = (int32_t)buf[t];
    }
  }
  return bad;
}

}  // extern "C"
