// api.cu — host side of the C ABI declared in include/binsketch.h:
// argument validation, the fp64 cardinality table (built with the host C
// library's log1p, cached per (N, d) in pinned memory and uploaded into the
// caller's workspace), workspace layout, and kernel dispatch on the caller's
// stream. Product code; shares nothing with oracle/.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <unistd.h>   // environ
#include <utility>

#include "binsketch.h"
#include "bsk_internal.cuh"

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// Cardinality table, Algorithm 1 line 3 with q = 1 - 1/N
// (PAPER.md:358): L[k] = ln(1-k/N)/ln(q) evaluated as log1p(-k/N)/log1p(-1/N)
// (reading R-G11); L[N] = d (saturation, R-G12).
// BCS table (R-B2): B[x] = log1p(-2x/N)/log1p(-2/N) for 0 < 2x < N, B[0] = 0, B[x] = d once
// 2x >= N (the parity-collision law inverted; cached under kind 1).
struct TableCache {
  std::mutex mu;
  std::map<std::tuple<uint32_t, uint64_t, int>, double*> tables;
  std::map<std::pair<uint32_t, uint64_t>, bool> convex_;

  // L non-decreasing with non-decreasing increments (to 1e-9 relative): the condition
  // under which the tensor-core top-k prefilter bound holds (K10). False e.g.
  // when the saturation value L[N] = d is below L[N-1].
  bool convex(uint32_t N, uint64_t d) {
    const double* t = get(N, d);
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(N, d);
    auto it = convex_.find(key);
    if (it != convex_.end()) return it->second;
    bool ok = t != nullptr;
    for (uint32_t k = 0; ok && k < N; ++k) {
      const double inc = t[k + 1] - t[k];
      if (inc < 0.0) ok = false;
      if (k > 0) {
        const double prev = t[k] - t[k - 1];
        if (inc < prev - 1e-9 * std::fabs(prev)) ok = false;
      }
    }
    convex_.emplace(key, ok);
    return ok;
  }

  // L non-decreasing on [0, N): every estimator key is then non-decreasing in pab for fixed
  // (pa, pb) — the condition of the pab-table top-k's integer screen (K4c).
  bool monotone(uint32_t N, uint64_t d) {
    const double* t = get(N, d);
    if (!t) return false;
    for (uint32_t k = 0; k + 1 < N; ++k)
      if (t[k + 1] < t[k]) return false;
    return true;
  }

  const double* get(uint32_t N, uint64_t d, int kind = 0) {
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_tuple(N, d, kind);
    auto it = tables.find(key);
    if (it != tables.end()) return it->second;
    double* t = nullptr;
    if (cudaHostAlloc(reinterpret_cast<void**>(&t), (size_t)(N + 1) * sizeof(double), cudaHostAllocDefault) !=
        cudaSuccess) {
      cudaGetLastError();  // clear; fall back to pageable memory (host-only use, no GPU)
      t = static_cast<double*>(std::malloc((size_t)(N + 1) * sizeof(double)));
      if (!t) return nullptr;
    }
    if (kind == 0) {
      const double c = std::log1p(-1.0 / (double)N);
      for (uint32_t k = 0; k < N; ++k) t[k] = std::log1p(-(double)k / (double)N) / c;
      t[N] = (double)d;
    } else {
      const double c = std::log1p(-2.0 / (double)N);
      t[0] = 0.0;
      for (uint32_t k = 1; k <= N; ++k)
        t[k] = (2.0 * (double)k >= (double)N) ? (double)d : std::log1p(-2.0 * (double)k / (double)N) / c;
    }
    tables.emplace(key, t);
    return t;
  }
};

TableCache& cache() {
  static TableCache* c = new TableCache();  // never destroyed: pinned buffers may back in-flight copies
  return *c;
}

struct Layout {
  size_t tmeta = 0, L = 0, pa = 0, pb = 0, pkey = 0, pidx = 0, a8 = 0, b8 = 0, bins = 0, perm = 0, spb = 0, qperm = 0, qspb = 0,
         ctr = 0, done = 0, pab = 0, cnt = 0, x8 = 0, px = 0, pabx = 0, part = 0, range = 0, scratch = 0, s8 = 0, pabs = 0, ts = 0, tsuf = 0,
         lcnt = 0, total = 0;
  uint32_t splits = 1;
};

// Pair engine: tensor cores (tcgen05 kind::i8 on {0,1}-byte operands, tc.cu) or CUDA
// cores (LOP3 + POPC, pairs.cu). BINSKETCH_ENGINE=cuda|tc overrides (A/B measurement).
bool engine_cuda() {
  const char* e = std::getenv("BINSKETCH_ENGINE");
  return e && !std::strcmp(e, "cuda");
}
bool engine_tc() {
  const char* e = std::getenv("BINSKETCH_ENGINE");
  return e && !std::strcmp(e, "tc");
}
bool fused_topk_ok(uint32_t N, uint32_t k) {
  return k <= bsk::tc_topk_max_k() && N <= bsk::tc_topk_max_n() && bsk::tc_topk_fits(N, k);
}
// Small top-k calls (nq * ndb <= 2^25 pairs) go to the CUDA-core kernels: the fused tensor-core
// kernel then has fewer tiles than SMs and every tile is a heap-filling one (measured, self-joins:
// 1000 rows JS k = 10 0.158 vs 0.336 ms, 4000 rows IP k = 50 1.19 vs 1.78 ms; 16000 rows IP
// 7.1 vs 5.1 ms; profiles/r02_topk_engine_sweep.jsonl). BINSKETCH_ENGINE=tc forces the fused kernel.
constexpr uint64_t kSmallTopkPairs = uint64_t(1) << 25;
bool small_topk(uint64_t nq, uint64_t ndb) {
  if (const char* e = std::getenv("BINSKETCH_TOPK_SMALL"))   // "0": no small-call rule (test / A-B knob)
    if (!std::strcmp(e, "0")) return false;
  return !engine_tc() && nq <= kSmallTopkPairs && ndb <= kSmallTopkPairs && nq * ndb <= kSmallTopkPairs;
}
bool use_tc(int op, uint32_t N, uint32_t k = 0, uint64_t nq = ~uint64_t(0), uint64_t ndb = ~uint64_t(0)) {
  if (engine_cuda()) return false;
  if (op == BINSKETCH_OP_TOPK) return fused_topk_ok(N, k) && !small_topk(nq, ndb);
  // all-pairs estimate: the epilogue (fp64 recipe, 16 B of planes per pair) dominates; at W <= 32
  // the CUDA-core kernel's 32 POPCs per pair are cheaper than the tensor-core pipeline around it
  // (Medium, 1e8 pairs x 4 planes: N = 1000 1.28 vs 1.49 ms; N = 2000 1.87 vs 1.56 ms)
  if (op == BINSKETCH_OP_ESTIMATE && !engine_tc()) return (N + 31) / 32 > 32;
  return true;
}
// Top-k beyond the fused kernel's limits (k > 64 or N > 6143): tensor-core AND-popcount into a
// workspace table pab[nq][ndb], then the CUDA-core threshold top-k reading it — when the table
// fits the budget; otherwise the CUDA-core kernels end to end.
constexpr size_t kPabBudget = size_t(4) << 30;
bool use_tc_pab(uint32_t N, uint64_t nq, uint64_t ndb, uint32_t k) {
  return !engine_cuda() && !fused_topk_ok(N, k) && nq * ndb * 4 <= kPabBudget;
}

// Top-k through the fused tensor-core screen (K4d): sample thresholds and minimum-pab
// tables, the AND-popcount with the screen in its epilogue (survivor lists, no table), the exact
// ranking of the survivors. Sizes that allow it (the lists take 8 B per pair, in the budget);
// the call also needs L non-decreasing on [0, N) (checked per (N, d)). BINSKETCH_TOPK_SCREEN=0
// selects the pab-table kernels instead (dev A/B).
constexpr uint64_t kScreenSample = 4096;   // db rows [0, S) sampled for the thresholds

// A second stream (and fork / join events) per host thread and device, for the fused screen's
// independent branches (never destroyed: they may back in-flight work at exit).
struct Fork {
  cudaStream_t s2 = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
Fork* fork_for_device() {
  constexpr int kMaxDev = 64;
  thread_local Fork f[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  Fork& x = f[dev];
  if (!x.s2) {
    if (cudaStreamCreateWithFlags(&x.s2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      x = Fork{};
      return nullptr;
    }
  }
  return &x;
}
bool screen_size_ok(uint32_t N, uint64_t nq, uint64_t ndb, uint32_t k) {
  if (const char* e = std::getenv("BINSKETCH_TOPK_SCREEN")) if (!std::strcmp(e, "0")) return false;
  return N <= 16383 && k >= 1 && k <= 256 && bsk::tc_sortable(N) && nq * ndb * 8 <= kPabBudget;
}

// All-pairs estimate planes through a pab table: tensor-core AND-popcount into pab[na][nb], then the
// elementwise recipe kernel at full occupancy (K10 estimate). BINSKETCH_EST_PAB=0|1
// overrides (dev A/B); the CUDA-core engine override disables it.
bool use_est_pab(uint64_t na, uint64_t nb) {
  if (engine_cuda()) return false;
  if (const char* e = std::getenv("BINSKETCH_EST_PAB")) return std::strcmp(e, "0") != 0 && na * nb * 4 <= kPabBudget;
  return na * nb * 4 <= kPabBudget;
}

constexpr uint64_t kMseRows = 4096;   // Experiment-1 row block (two [rows][n] int32 tables)

Layout layout(int op, uint64_t na, uint64_t nb, uint32_t N, uint32_t k) {
  Layout l;
  size_t off = 0;
  if (op == BINSKETCH_OP_MSE) {   // na = n rows, nb = d (width of the exact rows)
    const uint64_t n = na, d = nb, R = std::min<uint64_t>(n, kMseRows);
    l.L = off; off += align_up((size_t)(N + 1) * 8);
    l.pa = off; off += align_up((size_t)n * 4);
    l.px = off; off += align_up((size_t)n * 4);
    l.ctr = off; off += kAlign;
    l.a8 = off; off += align_up((size_t)n * bsk::tc_kpad(N));
    l.x8 = off; off += align_up((size_t)n * bsk::tc_kpad((uint32_t)std::min<uint64_t>(d, 0xffffff80ull)));
    l.pab = off; off += align_up((size_t)R * n * 4);
    l.pabx = off; off += align_up((size_t)R * n * 4);
    l.part = off; off += align_up(bsk::mse_partial_bytes());
    l.total = off;
    return l;
  }
  if (op == BINSKETCH_OP_ANDPOPC) {   // only the tensor-core engine needs scratch: expanded operands
    l.ctr = off; off += kAlign;
    l.a8 = off; off += align_up((size_t)na * bsk::tc_kpad(N));
    l.b8 = off; off += align_up((size_t)nb * bsk::tc_kpad(N));
    l.total = off;
    return l;
  }
  l.L = off; off += align_up((size_t)(N + 1) * 8);
  l.pa = off; off += align_up((size_t)na * 4);
  l.pb = off; off += align_up((size_t)nb * 4);
  if (op == BINSKETCH_OP_JOIN) {   // tensor-core join: widened operands
    l.ctr = off; off += kAlign;
    l.a8 = off; off += align_up((size_t)na * bsk::tc_kpad(N));
    l.b8 = off; off += align_up((size_t)nb * bsk::tc_kpad(N));
    l.total = off;
    return l;
  }
  if (op == BINSKETCH_OP_BCS_ESTIMATE) {   // always the tensor-core engine
    l.ctr = off; off += kAlign;
    l.a8 = off; off += align_up((size_t)na * bsk::tc_kpad(N));
    l.b8 = off; off += align_up((size_t)nb * bsk::tc_kpad(N));
    if (use_est_pab(na, nb)) { l.pab = off; off += align_up((size_t)na * nb * 4); }
    l.total = off;
    return l;
  }
  if (op == BINSKETCH_OP_JOIN_LIST) {
    l.cnt = off; off += align_up((size_t)na * 4);
    l.total = off;
    return l;
  }
  const bool ep = op == BINSKETCH_OP_ESTIMATE && use_est_pab(na, nb);
  const bool tc = !ep && use_tc(op, N, k, na, nb);
  const bool tcp = (op == BINSKETCH_OP_TOPK && use_tc_pab(N, na, nb, k)) || ep;
  if (tcp) {
    l.ctr = off; off += kAlign;
    l.a8 = off; off += align_up((size_t)na * bsk::tc_kpad(N));
    l.b8 = off; off += align_up((size_t)nb * bsk::tc_kpad(N));
    // the pab table, or (fused-screen top-k) the survivor lists [na][nb] uint2 in the same place
    const bool scr = op == BINSKETCH_OP_TOPK && screen_size_ok(N, na, nb, k);
    l.pab = off; off += align_up((size_t)na * nb * (scr ? 8 : 4));
    if (op == BINSKETCH_OP_TOPK) {   // pab-table top-k: db popcount range, pass-2 survivor scratch
      l.range = off; off += kAlign;
      l.scratch = off; off += align_up(bsk::topk_pab3_scratch_bytes(15u));
    }
    if (scr) {   // fused screen: sample operand + table, thresholds, tables, list counts, db sort
      const uint64_t S = std::min<uint64_t>(nb, kScreenSample);
      l.s8 = off; off += align_up((size_t)S * bsk::tc_kpad(N));
      l.pabs = off; off += align_up((size_t)na * S * 4);
      l.ts = off; off += align_up((size_t)na * 4 * 8);
      l.tsuf = off; off += align_up((size_t)na * (N + 1) * 4 * 2);
      l.lcnt = off; off += align_up((size_t)na * ((nb + 255) / 256) * 4);   // [na][db chunks]
      l.bins = off; off += align_up((size_t)(N + 1) * 4);
      l.perm = off; off += align_up((size_t)nb * 4);
      l.spb = off; off += align_up((size_t)nb * 4);
    }
  }
  if (tc) {
    l.ctr = off; off += kAlign;
    l.a8 = off; off += align_up((size_t)na * bsk::tc_kpad(N));
    l.b8 = off; off += align_up((size_t)nb * bsk::tc_kpad(N));
  }
  if (op == BINSKETCH_OP_TOPK && tc && bsk::tc_sortable(N)) {
    l.bins = off; off += align_up((size_t)(N + 1) * 4);
    l.perm = off; off += align_up((size_t)nb * 4);
    l.spb = off; off += align_up((size_t)nb * 4);
    l.qperm = off; off += align_up((size_t)na * 4);
    l.qspb = off; off += align_up((size_t)na * 4);
    l.tmeta = off; off += align_up((size_t)((nb + 255) / 256) * 256 * 8 +     // per-tile db metadata
                                   (size_t)((nb + 255) / 256) * 2 * 4);        // + per-tile smallest db index
  }
  if (op == BINSKETCH_OP_TOPK) {
    l.splits = tc ? bsk::tc_topk_splits(na, nb, N, k) : bsk::topk_splits(na, nb, k);
    if (tc) { l.done = off; off += align_up(((na + 127) / 128) * 4); }
    if (l.splits > 1 || tc) {
      l.pkey = off; off += align_up((size_t)na * l.splits * k * 8);
      l.pidx = off; off += align_up((size_t)na * l.splits * k * 4);
    }
  }
  l.total = off;
  return l;
}

inline binsketch_status cuda_status(cudaError_t e) { return e == cudaSuccess ? BINSKETCH_OK : BINSKETCH_ECUDA; }

inline bool one_bit(uint32_t m) { return m == 1u || m == 2u || m == 4u || m == 8u; }

binsketch_status upload_table(uint32_t N, uint64_t d, void* ws, const Layout& l, cudaStream_t s, int kind = 0) {
  const double* t = cache().get(N, d, kind);
  if (!t) return BINSKETCH_ECUDA;
  return cuda_status(cudaMemcpyAsync(static_cast<char*>(ws) + l.L, t, (size_t)(N + 1) * 8,
                                     cudaMemcpyHostToDevice, s));
}

}  // namespace

extern "C" {

uint32_t binsketch_words(uint32_t N) { return (uint32_t)(((uint64_t)N + 31u) / 32u); }

uint32_t binsketch_recommended_N(uint32_t psi, double rho) {
  // Theorem 1: N = psi * sqrt(psi/2 * ln(2/rho)); max(2, ceil(.)) (R-G5).
  if (psi == 0 || !(rho > 0.0 && rho < 1.0)) return 0;
  const double p = (double)psi;
  double v = std::ceil(p * std::sqrt(0.5 * p * std::log(2.0 / rho)));
  if (v < 2.0) v = 2.0;
  if (v > 4294967295.0) return 0;
  return (uint32_t)v;
}

binsketch_status binsketch_make_pi(uint64_t seed, uint64_t d, uint32_t N, uint32_t* pi, binsketch_stream_t stream) {
  if (N < 2 || (d > 0 && pi == nullptr)) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_BUILD) return BINSKETCH_EUNSUPPORTED;
  return cuda_status(bsk::launch_make_pi(seed, d, N, pi, reinterpret_cast<cudaStream_t>(stream)));
}

static binsketch_status build_common(const uint32_t* pi, uint64_t seed, uint64_t d, uint32_t N,
                                     const int64_t* indptr, const int32_t* indices, uint64_t n,
                                     uint32_t* out, binsketch_stream_t stream, bool parity = false) {
  if (N < 2) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_BUILD) return BINSKETCH_EUNSUPPORTED;
  if (n == 0) return BINSKETCH_OK;
  if (d == 0 || indptr == nullptr || indices == nullptr || out == nullptr) return BINSKETCH_EINVAL;
  if (d > 0x80000000ull) return BINSKETCH_EINVAL;  // int32 indices cannot address more
  if (!bsk::status_ptr()) return BINSKETCH_ECUDA;
  return cuda_status(bsk::launch_build(pi, seed, d, N, indptr, indices, n, out,
                                       reinterpret_cast<cudaStream_t>(stream), parity));
}

binsketch_status binsketch_build(const uint32_t* pi, uint64_t d, uint32_t N, const int64_t* indptr,
                                 const int32_t* indices, uint64_t n, uint32_t* out_words,
                                 binsketch_stream_t stream) {
  if (n > 0 && pi == nullptr) return BINSKETCH_EINVAL;
  return build_common(pi, 0, d, N, indptr, indices, n, out_words, stream);
}

binsketch_status binsketch_build_seeded(uint64_t seed, uint64_t d, uint32_t N, const int64_t* indptr,
                                        const int32_t* indices, uint64_t n, uint32_t* out_words,
                                        binsketch_stream_t stream) {
  return build_common(nullptr, seed, d, N, indptr, indices, n, out_words, stream);
}

binsketch_status binsketch_bcs_build(const uint32_t* pi, uint64_t d, uint32_t N, const int64_t* indptr,
                                     const int32_t* indices, uint64_t n, uint32_t* out_words,
                                     binsketch_stream_t stream) {
  if (n > 0 && pi == nullptr) return BINSKETCH_EINVAL;
  return build_common(pi, 0, d, N, indptr, indices, n, out_words, stream, true);
}

binsketch_status binsketch_bcs_build_seeded(uint64_t seed, uint64_t d, uint32_t N, const int64_t* indptr,
                                            const int32_t* indices, uint64_t n, uint32_t* out_words,
                                            binsketch_stream_t stream) {
  return build_common(nullptr, seed, d, N, indptr, indices, n, out_words, stream, true);
}

binsketch_status binsketch_popcount(const uint32_t* sk, uint64_t n, uint32_t N, int32_t* out,
                                    binsketch_stream_t stream) {
  if (N < 2) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_BUILD) return BINSKETCH_EUNSUPPORTED;
  if (n == 0) return BINSKETCH_OK;
  if (!sk || !out) return BINSKETCH_EINVAL;
  return cuda_status(bsk::launch_popcount(sk, n, binsketch_words(N), out, reinterpret_cast<cudaStream_t>(stream)));
}

size_t binsketch_workspace_bytes(int op, uint64_t na, uint64_t nb, uint32_t N, uint32_t k) {
  if (N < 2 || N > BINSKETCH_MAX_N_PAIRS) return 0;
  return layout(op, na, nb, N, k).total;
}

binsketch_status binsketch_andpopc(const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb, uint32_t N,
                                   int32_t* out, void* ws, size_t ws_bytes, binsketch_stream_t stream) {
  if (N < 2) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  if (na == 0 || nb == 0) return BINSKETCH_OK;
  if (!A || !B || !out) return BINSKETCH_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!use_tc(BINSKETCH_OP_ANDPOPC, N))
    return cuda_status(bsk::launch_pairs(bsk::kAndPopc, A, na, B, nb, N, 0, nullptr, nullptr, nullptr, out, s));
  const Layout l = layout(BINSKETCH_OP_ANDPOPC, na, nb, N, 0);
  if (!ws || ws_bytes < l.total) return BINSKETCH_EWORKSPACE;
  uint8_t* a8 = static_cast<uint8_t*>(ws) + l.a8;
  uint8_t* b8 = static_cast<uint8_t*>(ws) + l.b8;
  cudaError_t e = bsk::launch_expand(A, na, N, a8, s);
  if (e == cudaSuccess) e = bsk::launch_expand(B, nb, N, b8, s);
  if (e == cudaSuccess)
    e = bsk::launch_tc_andpopc(a8, na, b8, nb, N, out, reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(ws) + l.ctr), s);
  return cuda_status(e);
}

// expand, tensor-core AND-popcount into the pab table, elementwise recipe (use_est_pab)
binsketch_status estimate_via_pab(const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb, uint32_t N,
                                  uint32_t measure, const int32_t* pa, const int32_t* pb, const Layout& l, char* w,
                                  float* out, cudaStream_t s, bool self, bool bcs, double dcap, double ham_scale) {
  uint8_t* a8 = reinterpret_cast<uint8_t*>(w + l.a8);
  uint8_t* b8 = self ? a8 : reinterpret_cast<uint8_t*>(w + l.b8);
  int32_t* pab = reinterpret_cast<int32_t*>(w + l.pab);
  cudaError_t e = bsk::launch_expand(A, na, N, a8, s);
  if (e == cudaSuccess && !self) e = bsk::launch_expand(B, nb, N, b8, s);
  if (e == cudaSuccess)
    e = bsk::launch_tc_andpopc(a8, na, b8, nb, N, pab, reinterpret_cast<unsigned long long*>(w + l.ctr), s);
  if (e == cudaSuccess)
    e = bsk::launch_estimate_from_pab(pab, na, nb, N, measure, pa, pb, reinterpret_cast<const double*>(w + l.L), out,
                                      s, bcs, dcap, ham_scale);
  return cuda_status(e);
}

binsketch_status binsketch_estimate(const uint32_t* sketches_a, uint64_t na, const uint32_t* sketches_b,
                                    uint64_t nb, uint32_t N, uint64_t d, uint32_t measure, float* out, void* ws,
                                    size_t ws_bytes, binsketch_stream_t stream) {
  if (N < 2 || measure == 0 || (measure & ~15u)) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  if (na == 0 || nb == 0) return BINSKETCH_OK;
  if (!sketches_a || !sketches_b || !out || d == 0) return BINSKETCH_EINVAL;
  const Layout l = layout(BINSKETCH_OP_ESTIMATE, na, nb, N, 0);
  if (!ws || ws_bytes < l.total) return BINSKETCH_EWORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  binsketch_status st = upload_table(N, d, ws, l, s);
  if (st != BINSKETCH_OK) return st;
  const uint32_t W = binsketch_words(N);
  int32_t* pa = reinterpret_cast<int32_t*>(w + l.pa);
  int32_t* pb = reinterpret_cast<int32_t*>(w + l.pb);
  cudaError_t e = bsk::launch_popcount(sketches_a, na, W, pa, s);
  const bool self = sketches_a == sketches_b && na == nb;
  if (e == cudaSuccess) e = self ? cudaMemcpyAsync(pb, pa, na * 4, cudaMemcpyDeviceToDevice, s)
                                 : bsk::launch_popcount(sketches_b, nb, W, pb, s);
  if (e != cudaSuccess) return cuda_status(e);
  if (use_est_pab(na, nb))
    return estimate_via_pab(sketches_a, na, sketches_b, nb, N, measure, pa, pb, l, w, out, s, self, false, 0.0, 1.0);
  if (use_tc(BINSKETCH_OP_ESTIMATE, N)) {
    uint8_t* a8 = reinterpret_cast<uint8_t*>(w + l.a8);
    uint8_t* b8 = self ? a8 : reinterpret_cast<uint8_t*>(w + l.b8);
    e = bsk::launch_expand(sketches_a, na, N, a8, s);
    if (e == cudaSuccess && !self) e = bsk::launch_expand(sketches_b, nb, N, b8, s);
    if (e == cudaSuccess)
      e = bsk::launch_tc_estimate(a8, na, b8, nb, N, measure, pa, pb, reinterpret_cast<const double*>(w + l.L), out,
                                  reinterpret_cast<unsigned long long*>(w + l.ctr), s);
    return cuda_status(e);
  }
  e = bsk::launch_pairs(bsk::kEstimate, sketches_a, na, sketches_b, nb, N, measure, pa, pb,
                        reinterpret_cast<const double*>(w + l.L), out, s);
  return cuda_status(e);
}

static binsketch_status topk_impl(const uint32_t* queries, uint64_t nq, const uint32_t* db, uint64_t ndb, uint32_t N,
                                  uint64_t d, uint32_t measure, uint32_t k, uint32_t flags, int32_t* out_idx,
                                  float* out_score, void* ws, size_t ws_bytes, binsketch_stream_t stream) {
  if (N < 2 || measure == 0 || (measure & ~15u) || (flags & ~1u)) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  if (nq == 0 || k == 0) return BINSKETCH_OK;
  if (k > BINSKETCH_MAX_K) return BINSKETCH_EUNSUPPORTED;
  if (!queries || !out_idx || !out_score || d == 0 || (ndb > 0 && !db)) return BINSKETCH_EINVAL;
  // several measures: lists stacked [measure][nq][k] in the order IP, HAM, JS, COS
  uint32_t mlist[4], nm = 0;
  for (uint32_t b = 1; b <= 8; b <<= 1)
    if (measure & b) mlist[nm++] = b;
  if (ndb > 0x7fffffffull) return BINSKETCH_EUNSUPPORTED;   // int32 output indices
  const Layout l = layout(BINSKETCH_OP_TOPK, nq, ndb, N, k);
  if (!ws || ws_bytes < l.total) return BINSKETCH_EWORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  binsketch_status st = upload_table(N, d, ws, l, s);
  if (st != BINSKETCH_OK) return st;
  const uint32_t W = binsketch_words(N);
  int32_t* pq = reinterpret_cast<int32_t*>(w + l.pa);
  int32_t* pd = reinterpret_cast<int32_t*>(w + l.pb);
  cudaError_t e = bsk::launch_popcount(queries, nq, W, pq, s);
  const bool self = queries == db && nq == ndb;
  if (e == cudaSuccess) e = self ? cudaMemcpyAsync(pd, pq, nq * 4, cudaMemcpyDeviceToDevice, s)
                                 : bsk::launch_popcount(db, ndb, W, pd, s);
  if (e != cudaSuccess) return cuda_status(e);
  if (ndb > 0 && use_tc(BINSKETCH_OP_TOPK, N, k, nq, ndb)) {
   for (uint32_t mi = 0; mi < nm; ++mi) {   // fused top-k: one pass per measure
    const uint32_t measure_m = mlist[mi];
    int32_t* out_idx_m = out_idx + (size_t)mi * nq * k;
    float* out_score_m = out_score + (size_t)mi * nq * k;
    // db popcount-sorted (tight per-tile prefilter). Queries popcount-sorted too for JS / COS / HAM
    // (a query tile then has a narrow |a_s| range, so its best candidates — pb near pa — arrive
    // together; Large k = 50: HAM 90 -> 65, JS 214 -> 150, COS 158 -> 119 ms) but not for IP, where
    // sorting clusters the heavy rows (large |a_s|, many candidates) into straggler tiles (53 -> 70 ms).
    // BINSKETCH_TC_QSORT=0|1 overrides (dev A/B knob).
    uint8_t* q8 = reinterpret_cast<uint8_t*>(w + l.a8);
    uint8_t* d8 = reinterpret_cast<uint8_t*>(w + l.b8);
    const bool sorted = bsk::tc_sortable(N);
    int32_t* perm = sorted ? reinterpret_cast<int32_t*>(w + l.perm) : nullptr;
    int32_t* spb = sorted ? reinterpret_cast<int32_t*>(w + l.spb) : pd;
    const char* qs = std::getenv("BINSKETCH_TC_QSORT");
    // (small query sets: the three extra sort launches would dominate a launch-bound call)
    const bool qsort = sorted && (qs ? !std::strcmp(qs, "1") : (measure_m != BINSKETCH_IP && nq >= 16384));
    int32_t* qperm = qsort ? reinterpret_cast<int32_t*>(w + l.qperm) : nullptr;
    int32_t* qspb = qsort ? reinterpret_cast<int32_t*>(w + l.qspb) : pq;
    uint32_t* bins = reinterpret_cast<uint32_t*>(w + l.bins);
    // order that raises the heaps' thresholds fastest (measured, Large k = 50): IP's best
    // candidates have large pb (descending: 53 vs 262 ms); JS / COS / HAM favour pb close to pa,
    // reached earlier from below (ascending: JS 302 -> 214, COS 260 -> 158, HAM 870 -> 90 ms)
    if (sorted) e = bsk::launch_sort_by_popcount(pd, ndb, N, bins, perm, spb, s, measure_m == BINSKETCH_IP);
    if (qsort && e == cudaSuccess) e = bsk::launch_sort_by_popcount(pq, nq, N, bins, qperm, qspb, s);
    const bool packed_q = bsk::tc_topk_packed_queries(N);   // widened in the kernel, into TMEM
    if (e == cudaSuccess && !packed_q) e = bsk::launch_expand(queries, nq, N, q8, s, qperm);
    if (e == cudaSuccess) e = bsk::launch_expand(db, ndb, N, d8, s, perm);
    if (e == cudaSuccess)
      e = bsk::launch_tc_topk(q8, queries, nq, d8, ndb, N, measure_m, k, flags, qspb, qperm, spb, perm,
                              reinterpret_cast<const double*>(w + l.L), cache().convex(N, d),
                              reinterpret_cast<double*>(w + l.pkey), reinterpret_cast<int32_t*>(w + l.pidx),
                              out_idx_m, out_score_m, reinterpret_cast<unsigned long long*>(w + l.ctr),
                              reinterpret_cast<unsigned int*>(w + l.done), reinterpret_cast<int2*>(w + l.tmeta), s);
    if (e != cudaSuccess) return cuda_status(e);
   }
    return BINSKETCH_OK;
  }
  const int32_t* pab = nullptr;
  if (ndb > 0 && use_tc_pab(N, nq, ndb, k)) {
    uint8_t* q8 = reinterpret_cast<uint8_t*>(w + l.a8);
    if (screen_size_ok(N, nq, ndb, k) && cache().monotone(N, d)) {
      // fused screen (K4d): the table region holds the survivor lists, b8 the sorted db
      uint8_t* d8 = reinterpret_cast<uint8_t*>(w + l.b8);
      uint2* lists = reinterpret_cast<uint2*>(w + l.pab);
      int32_t* perm = reinterpret_cast<int32_t*>(w + l.perm);
      int32_t* spb = reinterpret_cast<int32_t*>(w + l.spb);
      uint8_t* s8 = reinterpret_cast<uint8_t*>(w + l.s8);
      int32_t* pabs = reinterpret_cast<int32_t*>(w + l.pabs);
      double* ts = reinterpret_cast<double*>(w + l.ts);
      uint16_t* tsuf = reinterpret_cast<uint16_t*>(w + l.tsuf);
      uint32_t* lcnt = reinterpret_cast<uint32_t*>(w + l.lcnt);
      int32_t* range = reinterpret_cast<int32_t*>(w + l.range);
      unsigned long long* ctr = reinterpret_cast<unsigned long long*>(w + l.ctr);
      const double* Ld = reinterpret_cast<const double*>(w + l.L);
      const uint32_t S = (uint32_t)std::min<uint64_t>(ndb, kScreenSample);
      const uint32_t nmp = nm == 3 ? 4u : nm;
      // two independent branches until the screen: the db's popcount sort + widening on a second
      // stream (when one is available), the sample thresholds on the caller's stream
      Fork* fk = fork_for_device();
      cudaStream_t s2 = fk ? fk->s2 : s;
      if (fk) {
        e = cudaEventRecord(fk->fork, s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s2, fk->fork, 0);
        if (e != cudaSuccess) return cuda_status(e);
      }
      e = bsk::launch_sort_by_popcount(pd, ndb, N, reinterpret_cast<uint32_t*>(w + l.bins), perm, spb, s2, false);
      if (e == cudaSuccess) e = bsk::launch_expand(db, ndb, N, d8, s2, perm);
      if (fk && e == cudaSuccess) e = cudaEventRecord(fk->join, s2);
      if (e == cudaSuccess) e = bsk::launch_expand(queries, nq, N, q8, s);
      if (e == cudaSuccess) e = bsk::launch_expand(db, S, N, s8, s);
      if (e == cudaSuccess) e = bsk::launch_tc_andpopc(q8, nq, s8, S, N, pabs, ctr, s);
      if (e == cudaSuccess) e = bsk::launch_int_range(pd, ndb, range, s);
      if (e == cudaSuccess)
        e = bsk::launch_screen_threshold(pabs, nq, S, N, measure, k, flags, pq, pd, Ld, range, tsuf, ts, s);
      uint32_t splits = 0, seg_cols = 0;
      if (fk && e == cudaSuccess) e = cudaStreamWaitEvent(s, fk->join, 0);   // join before the screen
      if (e == cudaSuccess)
        e = bsk::launch_tc_screen(q8, nq, d8, ndb, N, spb, perm, tsuf, nmp, lists, lcnt, ctr, splits, seg_cols, s);
      if (e == cudaSuccess)
        e = bsk::launch_topk_list(lists, lcnt, splits, seg_cols, nq, ndb, N, measure, k, flags, pq, Ld, ts,
                                  w + l.scratch, out_idx, out_score, s);
      return cuda_status(e);
    }
    uint8_t* d8 = self ? q8 : reinterpret_cast<uint8_t*>(w + l.b8);
    int32_t* pabw = reinterpret_cast<int32_t*>(w + l.pab);
    e = bsk::launch_expand(queries, nq, N, q8, s);
    if (e == cudaSuccess && !self) e = bsk::launch_expand(db, ndb, N, d8, s);
    if (e == cudaSuccess)
      e = bsk::launch_tc_andpopc(q8, nq, d8, ndb, N, pabw, reinterpret_cast<unsigned long long*>(w + l.ctr), s);
    if (e != cudaSuccess) return cuda_status(e);
    pab = pabw;
    const char* ps = std::getenv("BINSKETCH_PAB_SCREEN");   // dev A/B knob (0: the pre-test kernel)
    if (!(ps && !std::strcmp(ps, "0")) && bsk::topk_pab3_fits(N, measure, k) && cache().monotone(N, d))
      return cuda_status(bsk::launch_topk_pab3(pab, nq, ndb, N, measure, k, flags, pq, pd,
                                               reinterpret_cast<const double*>(w + l.L),
                                               reinterpret_cast<int32_t*>(w + l.range), w + l.scratch, out_idx,
                                               out_score, s));
  }
  // the AND-popcount table (when used) serves every requested measure
  for (uint32_t mi = 0; mi < nm && e == cudaSuccess; ++mi)
    e = bsk::launch_topk(queries, nq, db, ndb, N, mlist[mi], k, flags, pq, pd,
                         reinterpret_cast<const double*>(w + l.L),
                         l.splits > 1 ? reinterpret_cast<double*>(w + l.pkey) : nullptr,
                         l.splits > 1 ? reinterpret_cast<int32_t*>(w + l.pidx) : nullptr,
                         out_idx + (size_t)mi * nq * k, out_score + (size_t)mi * nq * k, s, pab);
  return cuda_status(e);
}

// binsketch_topk replays a CUDA graph of the call when it was made before with the same arguments
// (pointers, sizes, measure, k, flags, workspace) by this host thread on this device: a call is
// 5-20 kernel launches and memsets, several of them a few microseconds long, so launch gaps are a
// visible part of small and mid-size calls. The graph is captured on an internal stream (relaxed
// mode) and launched on the caller's stream; any capture failure falls back to the direct launches.
// Nothing in the call depends on the data (no host synchronisation), so a replay is the same
// computation on the current contents of the inputs. BINSKETCH_GRAPH=0 disables (dev A/B).
namespace {
struct TopkKey {
  const void *q, *db, *oi, *os, *ws;
  uint64_t nq, ndb, d, ws_bytes;
  uint32_t N, measure, k, flags;
  int dev;
  std::string knobs;   // the BINSKETCH_* environment (the A/B knobs steer the captured path)
  bool operator<(const TopkKey& o) const {
    return std::tie(q, db, oi, os, ws, nq, ndb, d, ws_bytes, N, measure, k, flags, dev, knobs) <
           std::tie(o.q, o.db, o.oi, o.os, o.ws, o.nq, o.ndb, o.d, o.ws_bytes, o.N, o.measure, o.k, o.flags, o.dev,
                    o.knobs);
  }
};
std::string binsketch_knobs() {
  std::string r;
  for (char** e = environ; e && *e; ++e)
    if (!std::strncmp(*e, "BINSKETCH_", 10)) { r += *e; r += '\n'; }
  return r;
}
struct TopkGraph {
  cudaGraphExec_t exec = nullptr;
  uint64_t launches = 0;
};
bool graphs_enabled() {
  const char* e = std::getenv("BINSKETCH_GRAPH");
  return !(e && !std::strcmp(e, "0"));
}
}  // namespace

int binsketch_topk_path(uint64_t nq, uint64_t ndb, uint32_t N, uint64_t d, uint32_t k) {
  if (nq == 0 || ndb == 0 || k == 0 || N < 2) return BINSKETCH_PATH_NONE;
  if (use_tc(BINSKETCH_OP_TOPK, N, k, nq, ndb)) return BINSKETCH_PATH_TC_FUSED;
  if (use_tc_pab(N, nq, ndb, k))
    return (screen_size_ok(N, nq, ndb, k) && cache().monotone(N, d)) ? BINSKETCH_PATH_TC_SCREEN : BINSKETCH_PATH_TC_PAB;
  return BINSKETCH_PATH_CUDA;
}

binsketch_status binsketch_topk(const uint32_t* queries, uint64_t nq, const uint32_t* db, uint64_t ndb, uint32_t N,
                                uint64_t d, uint32_t measure, uint32_t k, uint32_t flags, int32_t* out_idx,
                                float* out_score, void* ws, size_t ws_bytes, binsketch_stream_t stream) {
  int dev = 0;
  if (!graphs_enabled() || nq == 0 || k == 0 || cudaGetDevice(&dev) != cudaSuccess)
    return topk_impl(queries, nq, db, ndb, N, d, measure, k, flags, out_idx, out_score, ws, ws_bytes, stream);
  constexpr size_t kMaxGraphs = 16;   // per host thread (oldest entries dropped)
  thread_local std::map<TopkKey, TopkGraph> graphs;
  thread_local cudaStream_t cap[64] = {};
  const TopkKey key{queries, db, out_idx, out_score, ws, nq, ndb, d, ws_bytes, N, measure, k, flags, dev,
                    binsketch_knobs()};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto it = graphs.find(key);
  if (it != graphs.end()) {
    const cudaError_t e = cudaGraphLaunch(it->second.exec, s);
    if (e == cudaSuccess) {
      bsk::count_launch(it->second.launches);
      return BINSKETCH_OK;
    }
    cudaGetLastError();
    cudaGraphExecDestroy(it->second.exec);
    graphs.erase(it);
    return topk_impl(queries, nq, db, ndb, N, d, measure, k, flags, out_idx, out_score, ws, ws_bytes, stream);
  }
  if (dev < 0 || dev >= 64 ||
      (!cap[dev] && cudaStreamCreateWithFlags(&cap[dev], cudaStreamNonBlocking) != cudaSuccess)) {
    cudaGetLastError();
    return topk_impl(queries, nq, db, ndb, N, d, measure, k, flags, out_idx, out_score, ws, ws_bytes, stream);
  }
  const uint64_t before = bsk::launch_count();
  cudaGraph_t g = nullptr;
  binsketch_status st = BINSKETCH_ECUDA;
  if (cudaStreamBeginCapture(cap[dev], cudaStreamCaptureModeRelaxed) == cudaSuccess) {
    st = topk_impl(queries, nq, db, ndb, N, d, measure, k, flags, out_idx, out_score, ws, ws_bytes,
                   reinterpret_cast<binsketch_stream_t>(cap[dev]));
    if (cudaStreamEndCapture(cap[dev], &g) != cudaSuccess) st = BINSKETCH_ECUDA;
  }
  const uint64_t launches = bsk::launch_count() - before;
  cudaGraphExec_t exec = nullptr;
  if (st == BINSKETCH_OK && g && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess &&
      cudaGraphLaunch(exec, s) == cudaSuccess) {
    cudaGraphDestroy(g);
    if (graphs.size() >= kMaxGraphs) {
      cudaGraphExecDestroy(graphs.begin()->second.exec);
      graphs.erase(graphs.begin());
    }
    graphs[key] = TopkGraph{exec, launches};
    return BINSKETCH_OK;
  }
  // capture unavailable (or an argument error, which the direct call reports the same way)
  cudaGetLastError();
  if (exec) cudaGraphExecDestroy(exec);
  if (g) cudaGraphDestroy(g);
  return topk_impl(queries, nq, db, ndb, N, d, measure, k, flags, out_idx, out_score, ws, ws_bytes, stream);
}

binsketch_status binsketch_join(const uint32_t* queries, uint64_t nq, const uint32_t* db, uint64_t ndb, uint32_t N,
                                uint64_t d, uint32_t measure, const double* thresholds, uint32_t nthr, uint32_t flags,
                                uint32_t* out_bits, void* ws, size_t ws_bytes, binsketch_stream_t stream) {
  if (N < 2 || !one_bit(measure) || (flags & ~3u)) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  if (nthr == 0 || nthr > BINSKETCH_MAX_THRESHOLDS || !thresholds) return BINSKETCH_EINVAL;
  for (uint32_t t = 0; t < nthr; ++t)
    if (std::isnan(thresholds[t])) return BINSKETCH_EINVAL;
  if (nq == 0 || ndb == 0) return BINSKETCH_OK;
  const bool exact = (flags & BINSKETCH_JOIN_EXACT) != 0;
  if (!queries || !db || !out_bits || (!exact && d == 0)) return BINSKETCH_EINVAL;
  if (nq > 0x7fffffffull || ndb > 0x7fffffffull) return BINSKETCH_EUNSUPPORTED;
  const Layout l = layout(BINSKETCH_OP_JOIN, nq, ndb, N, 0);
  if (!ws || ws_bytes < l.total) return BINSKETCH_EWORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  if (!exact) {
    binsketch_status st = upload_table(N, d, ws, l, s);
    if (st != BINSKETCH_OK) return st;
  }
  const uint32_t W = binsketch_words(N);
  int32_t* pq = reinterpret_cast<int32_t*>(w + l.pa);
  int32_t* pd = reinterpret_cast<int32_t*>(w + l.pb);
  cudaError_t e = bsk::launch_popcount(queries, nq, W, pq, s);
  const bool self = queries == db && nq == ndb;
  if (e == cudaSuccess) e = self ? cudaMemcpyAsync(pd, pq, nq * 4, cudaMemcpyDeviceToDevice, s)
                                 : bsk::launch_popcount(db, ndb, W, pd, s);
  // db in its own order: every output word is then owned by one lane and written once with a
  // plain store (no memset, no atomics; K11)
  uint8_t* q8 = reinterpret_cast<uint8_t*>(w + l.a8);
  uint8_t* d8 = self ? q8 : reinterpret_cast<uint8_t*>(w + l.b8);
  if (e == cudaSuccess) e = bsk::launch_expand(queries, nq, N, q8, s);
  if (e == cudaSuccess && !self) e = bsk::launch_expand(db, ndb, N, d8, s);
  if (e != cudaSuccess) return cuda_status(e);
  // threshold keys (R-J1), descending; tslot maps each back to its output plane
  double tkey[BINSKETCH_MAX_THRESHOLDS];
  uint32_t tslot[BINSKETCH_MAX_THRESHOLDS];
  for (uint32_t t = 0; t < nthr; ++t) { tslot[t] = t; tkey[t] = measure == BINSKETCH_HAM ? -thresholds[t] : thresholds[t]; }
  for (uint32_t a = 1; a < nthr; ++a)
    for (uint32_t b = a; b > 0 && tkey[b] > tkey[b - 1]; --b) { std::swap(tkey[b], tkey[b - 1]); std::swap(tslot[b], tslot[b - 1]); }
  e = bsk::launch_tc_join(q8, nq, d8, ndb, N, measure, tkey, tslot, nthr, flags & BINSKETCH_JOIN_EXCLUDE_SELF, exact, pq,
                          pd, reinterpret_cast<const double*>(w + l.L), out_bits,
                          reinterpret_cast<unsigned long long*>(w + l.ctr), s);
  return cuda_status(e);
}

binsketch_status binsketch_join_list(const uint32_t* bits, const uint32_t* queries, uint64_t nq, const uint32_t* db,
                                     uint64_t ndb, uint32_t N, uint64_t d, uint32_t measure, uint32_t flags,
                                     int64_t* row_ptr, int32_t* out_j, float* out_score, uint64_t capacity, void* ws,
                                     size_t ws_bytes, binsketch_stream_t stream) {
  if (N < 2 || !one_bit(measure) || (flags & ~3u)) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  if (nq == 0) return BINSKETCH_OK;
  const bool exact = (flags & BINSKETCH_JOIN_EXACT) != 0;
  if (!row_ptr || (ndb > 0 && !bits)) return BINSKETCH_EINVAL;
  if (capacity > 0 && (!out_j || !out_score || !queries || (ndb > 0 && !db) || (!exact && d == 0)))
    return BINSKETCH_EINVAL;
  if (ndb > 0x7fffffffull) return BINSKETCH_EUNSUPPORTED;
  const Layout l = layout(BINSKETCH_OP_JOIN_LIST, nq, ndb, N, 0);
  if (!ws || ws_bytes < l.total) return BINSKETCH_EWORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  cudaError_t e = bsk::launch_join_rowptr(bits, nq, ndb, reinterpret_cast<int32_t*>(w + l.cnt), row_ptr, s);
  if (e != cudaSuccess || capacity == 0 || ndb == 0) return cuda_status(e);
  if (!exact) {
    binsketch_status st = upload_table(N, d, ws, l, s);
    if (st != BINSKETCH_OK) return st;
  }
  const uint32_t W = binsketch_words(N);
  int32_t* pq = reinterpret_cast<int32_t*>(w + l.pa);
  int32_t* pd = reinterpret_cast<int32_t*>(w + l.pb);
  e = bsk::launch_popcount(queries, nq, W, pq, s);
  if (e == cudaSuccess) e = bsk::launch_popcount(db, ndb, W, pd, s);
  if (e == cudaSuccess)
    e = bsk::launch_join_list(bits, nq, ndb, queries, db, N, pq, pd, reinterpret_cast<const double*>(w + l.L), measure,
                              exact, row_ptr, out_j, out_score, capacity, s);
  return cuda_status(e);
}

binsketch_status binsketch_join_confusion(const uint32_t* bits_est, const uint32_t* bits_true, uint64_t nq,
                                          uint64_t ndb, int64_t* out, binsketch_stream_t stream) {
  if (nq == 0) return BINSKETCH_OK;
  if (!out || (ndb > 0 && (!bits_est || !bits_true))) return BINSKETCH_EINVAL;
  return cuda_status(bsk::launch_join_confusion(bits_est, bits_true, nq, ndb, out, reinterpret_cast<cudaStream_t>(stream)));
}

binsketch_status binsketch_bcs_estimate(const uint32_t* sketches_a, uint64_t na, const uint32_t* sketches_b,
                                        uint64_t nb, uint32_t N, uint64_t d, uint32_t measure, float* out, void* ws,
                                        size_t ws_bytes, binsketch_stream_t stream) {
  if (N < 2 || measure == 0 || (measure & ~15u)) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  if (na == 0 || nb == 0) return BINSKETCH_OK;
  if (!sketches_a || !sketches_b || !out || d == 0) return BINSKETCH_EINVAL;
  const Layout l = layout(BINSKETCH_OP_BCS_ESTIMATE, na, nb, N, 0);
  if (!ws || ws_bytes < l.total) return BINSKETCH_EWORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  binsketch_status st = upload_table(N, d, ws, l, s, 1);
  if (st != BINSKETCH_OK) return st;
  const uint32_t W = binsketch_words(N);
  int32_t* pa = reinterpret_cast<int32_t*>(w + l.pa);
  int32_t* pb = reinterpret_cast<int32_t*>(w + l.pb);
  uint8_t* a8 = reinterpret_cast<uint8_t*>(w + l.a8);
  const bool self = sketches_a == sketches_b && na == nb;
  uint8_t* b8 = self ? a8 : reinterpret_cast<uint8_t*>(w + l.b8);
  cudaError_t e = bsk::launch_popcount(sketches_a, na, W, pa, s);
  if (e == cudaSuccess) e = self ? cudaMemcpyAsync(pb, pa, na * 4, cudaMemcpyDeviceToDevice, s)
                                 : bsk::launch_popcount(sketches_b, nb, W, pb, s);
  if (e != cudaSuccess) return cuda_status(e);
  if (use_est_pab(na, nb))
    return estimate_via_pab(sketches_a, na, sketches_b, nb, N, measure, pa, pb, l, w, out, s, self, true, (double)d, 1.0);
  e = bsk::launch_expand(sketches_a, na, N, a8, s);
  if (e == cudaSuccess && !self) e = bsk::launch_expand(sketches_b, nb, N, b8, s);
  if (e == cudaSuccess)
    e = bsk::launch_tc_estimate(a8, na, b8, nb, N, measure, pa, pb, reinterpret_cast<const double*>(w + l.L), out,
                                reinterpret_cast<unsigned long long*>(w + l.ctr), s, true, (double)d);
  return cuda_status(e);
}

binsketch_status binsketch_bcs_table(uint32_t N, uint64_t d, double* host_out) {
  if (N < 2 || !host_out) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  const double* t = cache().get(N, d, 1);
  if (!t) return BINSKETCH_ECUDA;
  for (uint32_t k = 0; k <= N; ++k) host_out[k] = t[k];
  return BINSKETCH_OK;
}

binsketch_status binsketch_mse(const uint32_t* sketches, const uint32_t* exact, uint64_t n, uint32_t N, uint64_t d,
                               uint32_t measure, const double* thresholds, uint32_t nthr, uint32_t flags,
                               double* out_sse, uint64_t* out_count, void* ws, size_t ws_bytes,
                               binsketch_stream_t stream) {
  if (N < 2 || !one_bit(measure) || (flags & ~1u) || d == 0) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  if (nthr == 0 || nthr > BINSKETCH_MAX_THRESHOLDS || !thresholds || !out_sse || !out_count) return BINSKETCH_EINVAL;
  for (uint32_t t = 0; t < nthr; ++t)
    if (std::isnan(thresholds[t])) return BINSKETCH_EINVAL;
  if (n > 0 && (!sketches || !exact)) return BINSKETCH_EINVAL;
  if (n > 0x7fffffffull || d > 0xffffff80ull) return BINSKETCH_EUNSUPPORTED;
  const Layout l = layout(BINSKETCH_OP_MSE, n, d, N, 0);
  if (!ws || ws_bytes < l.total) return BINSKETCH_EWORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  const bool bcs = (flags & BINSKETCH_MSE_BCS) != 0;
  double* part_sse = reinterpret_cast<double*>(w + l.part);
  unsigned long long* part_cnt = reinterpret_cast<unsigned long long*>(w + l.part + bsk::mse_partial_bytes() / 2);
  cudaError_t e = cudaMemsetAsync(w + l.part, 0, bsk::mse_partial_bytes(), s);
  if (e != cudaSuccess) return cuda_status(e);
  if (n >= 2) {
    binsketch_status st = upload_table(N, d, ws, l, s, bcs ? 1 : 0);
    if (st != BINSKETCH_OK) return st;
    int32_t* ps = reinterpret_cast<int32_t*>(w + l.pa);
    int32_t* px = reinterpret_cast<int32_t*>(w + l.px);
    uint8_t* a8 = reinterpret_cast<uint8_t*>(w + l.a8);
    uint8_t* x8 = reinterpret_cast<uint8_t*>(w + l.x8);
    const uint32_t Dw = (uint32_t)d;
    e = bsk::launch_popcount(sketches, n, binsketch_words(N), ps, s);
    if (e == cudaSuccess) e = bsk::launch_popcount(exact, n, binsketch_words(Dw), px, s);
    if (e == cudaSuccess) e = bsk::launch_expand(sketches, n, N, a8, s);
    if (e == cudaSuccess) e = bsk::launch_expand(exact, n, Dw, x8, s);
    int32_t* pab = reinterpret_cast<int32_t*>(w + l.pab);
    int32_t* pabx = reinterpret_cast<int32_t*>(w + l.pabx);
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(w + l.ctr);
    for (uint64_t r0 = 0; e == cudaSuccess && r0 + 1 < n; r0 += kMseRows) {
      const uint64_t rows = std::min<uint64_t>(kMseRows, n - r0);
      e = bsk::launch_tc_andpopc(a8 + r0 * bsk::tc_kpad(N), rows, a8, n, N, pab, ctr, s);
      if (e == cudaSuccess) e = bsk::launch_tc_andpopc(x8 + r0 * bsk::tc_kpad(Dw), rows, x8, n, Dw, pabx, ctr, s);
      if (e == cudaSuccess)
        e = bsk::launch_mse_block(pab, pabx, r0, rows, n, ps, px, reinterpret_cast<const double*>(w + l.L), N,
                                  (double)d, measure, bcs, thresholds, nthr, part_sse, part_cnt, s);
    }
  }
  if (e == cudaSuccess)
    e = bsk::launch_mse_final(part_sse, part_cnt, nthr, out_sse, reinterpret_cast<unsigned long long*>(out_count), s);
  return cuda_status(e);
}

binsketch_status binsketch_onehot(const int32_t* codes, uint64_t n, uint32_t c, const int64_t* offsets,
                                  int64_t* indptr, int32_t* indices, binsketch_stream_t stream) {
  if (n > 0 && (!indptr || (c > 0 && (!codes || !offsets || !indices)))) return BINSKETCH_EINVAL;
  if (!bsk::status_ptr()) return BINSKETCH_ECUDA;
  if (n == 0) return BINSKETCH_OK;
  if (c == 0) return cuda_status(cudaMemsetAsync(indptr, 0, (n + 1) * 8, reinterpret_cast<cudaStream_t>(stream)));
  return cuda_status(bsk::launch_onehot(codes, n, c, offsets, indptr, indices, reinterpret_cast<cudaStream_t>(stream)));
}

binsketch_status binsketch_categorical_estimate(const uint32_t* sketches_a, uint64_t na, const uint32_t* sketches_b,
                                                uint64_t nb, uint32_t N, uint64_t d, float* out, void* ws,
                                                size_t ws_bytes, binsketch_stream_t stream) {
  if (N < 2) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  if (na == 0 || nb == 0) return BINSKETCH_OK;
  if (!sketches_a || !sketches_b || !out || d == 0) return BINSKETCH_EINVAL;
  const Layout l = layout(BINSKETCH_OP_BCS_ESTIMATE, na, nb, N, 0);   // the tensor-core estimate layout
  if (!ws || ws_bytes < l.total) return BINSKETCH_EWORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(ws);
  binsketch_status st = upload_table(N, d, ws, l, s, 0);
  if (st != BINSKETCH_OK) return st;
  const uint32_t W = binsketch_words(N);
  int32_t* pa = reinterpret_cast<int32_t*>(w + l.pa);
  int32_t* pb = reinterpret_cast<int32_t*>(w + l.pb);
  uint8_t* a8 = reinterpret_cast<uint8_t*>(w + l.a8);
  const bool self = sketches_a == sketches_b && na == nb;
  uint8_t* b8 = self ? a8 : reinterpret_cast<uint8_t*>(w + l.b8);
  cudaError_t e = bsk::launch_popcount(sketches_a, na, W, pa, s);
  if (e == cudaSuccess) e = self ? cudaMemcpyAsync(pb, pa, na * 4, cudaMemcpyDeviceToDevice, s)
                                 : bsk::launch_popcount(sketches_b, nb, W, pb, s);
  if (e != cudaSuccess) return cuda_status(e);
  if (use_est_pab(na, nb))
    return estimate_via_pab(sketches_a, na, sketches_b, nb, N, BINSKETCH_HAM, pa, pb, l, w, out, s, self, false, 0.0, 0.5);
  e = bsk::launch_expand(sketches_a, na, N, a8, s);
  if (e == cudaSuccess && !self) e = bsk::launch_expand(sketches_b, nb, N, b8, s);
  if (e == cudaSuccess)
    e = bsk::launch_tc_estimate(a8, na, b8, nb, N, BINSKETCH_HAM, pa, pb, reinterpret_cast<const double*>(w + l.L), out,
                                reinterpret_cast<unsigned long long*>(w + l.ctr), s, false, 0.0, 0.5);
  return cuda_status(e);
}

binsketch_status binsketch_card_table(uint32_t N, uint64_t d, double* host_out) {
  if (N < 2 || !host_out) return BINSKETCH_EINVAL;
  if (N > BINSKETCH_MAX_N_PAIRS) return BINSKETCH_EUNSUPPORTED;
  const double* t = cache().get(N, d);
  if (!t) return BINSKETCH_ECUDA;
  for (uint32_t k = 0; k <= N; ++k) host_out[k] = t[k];
  return BINSKETCH_OK;
}

binsketch_status binsketch_device_status(binsketch_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaStreamSynchronize(s) != cudaSuccess) return BINSKETCH_ECUDA;
  unsigned int* p = bsk::status_ptr();
  if (!p) return BINSKETCH_ECUDA;
  unsigned int v = 0;
  if (cudaMemcpy(&v, p, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return BINSKETCH_ECUDA;
  if (v) {
    const unsigned int z = 0;
    if (cudaMemcpy(p, &z, sizeof(z), cudaMemcpyHostToDevice) != cudaSuccess) return BINSKETCH_ECUDA;
    return BINSKETCH_EINDEX;
  }
  return BINSKETCH_OK;
}

uint64_t binsketch_launch_count(void) { return bsk::launch_count(); }

const char* binsketch_strerror(binsketch_status status) {
  switch (status) {
    case BINSKETCH_OK: return "ok";
    case BINSKETCH_EINVAL: return "invalid argument";
    case BINSKETCH_EINDEX: return "device-detected invalid input (index out of range, pi value >= N, or decreasing indptr)";
    case BINSKETCH_ECUDA: return "CUDA runtime error";
    case BINSKETCH_EWORKSPACE: return "workspace too small";
    case BINSKETCH_EUNSUPPORTED: return "unsupported request (outside this build's limits)";
  }
  return "unknown status";
}

}  // extern "C"
