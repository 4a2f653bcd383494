// join.cu — kernels of the paper's two experiments beyond the pair engine:
//  * Experiment 2 post-processing: the per-query match list (CSR, db
//    index ascending, with scores) from a join bitmap, and the per-query confusion counts
//    |O'|, |O|, |O ∩ O'| from which accuracy / precision / recall / F1 follow
//    (PAPER.md:700-705). The bitmaps come from the tensor-core join (tc.cu, kTcJoin).
//  * Experiment 1: the squared-error reduction over the pairs whose exact
//    similarity reaches each threshold, from two AND-popcount tables (sketches, exact rows).
// Compiled with -fmad=false (the list scores use the canonical fp64 recipe, R-C3).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bsk_device.cuh"
#include "bsk_estimator.cuh"
#include "bsk_internal.cuh"

namespace bsk {

// row_ptr[0] = 0, row_ptr[i+1] = row_ptr[i] + counts[i]; one block, chunked serial scan.
__global__ void row_ptr_kernel(const int32_t* __restrict__ counts, uint64_t n, int64_t* __restrict__ row_ptr) {
  __shared__ int64_t part[1024];
  const uint32_t t = threadIdx.x;
  const uint64_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint64_t b0 = min((uint64_t)t * per, n), b1 = min(b0 + per, n);
  int64_t sum = 0;
  for (uint64_t i = b0; i < b1; ++i) sum += counts[i];
  part[t] = sum;
  __syncthreads();
  for (uint32_t o = 1; o < blockDim.x; o <<= 1) {
    const int64_t v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - sum;
  if (t == 0) row_ptr[0] = 0;
  for (uint64_t i = b0; i < b1; ++i) { run += counts[i]; row_ptr[i + 1] = run; }
}

// One warp per query row: set bits of the row in ascending column order; each match's
// score is recomputed from the sketches (AND-popcount over W words + the recipe, or the
// exact key). Entries at positions >= cap are counted in row_ptr but not written.
__global__ void join_list_kernel(const uint32_t* __restrict__ bits, uint64_t nq, uint64_t wpr,
                                 const uint32_t* __restrict__ Q, const uint32_t* __restrict__ D, uint32_t W,
                                 const int32_t* __restrict__ pq, const int32_t* __restrict__ pd,
                                 const double* __restrict__ L, uint32_t N, uint32_t m, uint32_t exact,
                                 const int64_t* __restrict__ row_ptr, int32_t* __restrict__ out_j,
                                 float* __restrict__ out_score, uint64_t cap) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = gw; i < nq; i += nwarps) {
    const uint32_t* brow = bits + i * wpr;
    const uint32_t* qrow = Q + i * W;
    const int pa = __ldg(pq + i);
    uint64_t base = (uint64_t)__ldg(row_ptr + i);
    if (base >= cap) continue;
    for (uint64_t w0 = 0; w0 < wpr; w0 += 32) {
      uint32_t word = (w0 + lane < wpr) ? __ldg(brow + w0 + lane) : 0u;
      const uint32_t c = __popc(word);
      uint32_t off = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, off, o); if (lane >= o) off += y; }
      const uint32_t total = __shfl_sync(0xffffffffu, off, 31);
      uint64_t pos = base + off - c;
      while (word && pos < cap) {
        const uint32_t b = __ffs(word) - 1;
        word &= word - 1;
        const uint64_t j = (w0 + lane) * 32 + b;
        const uint32_t* drow = D + j * W;
        int pab = 0;
        for (uint32_t w = 0; w < W; ++w) pab += __popc(__ldg(qrow + w) & __ldg(drow + w));
        const int pb = __ldg(pd + j);
        const double key = exact ? exact_key(pa, pb, pab, m) : measure_key(estimate_pair(pa, pb, pab, (int)N, L, m), m);
        out_j[pos] = (int32_t)j;
        out_score[pos] = key_to_score(key, m);
        ++pos;
      }
      base += total;
      if (base >= cap) break;
    }
  }
}

// out[0][i] = |est_i|, out[1][i] = |true_i|, out[2][i] = |est_i AND true_i| (one warp per row).
__global__ void join_confusion_kernel(const uint32_t* __restrict__ est, const uint32_t* __restrict__ tru,
                                      uint64_t nq, uint64_t wpr, int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = gw; i < nq; i += nwarps) {
    int64_t a = 0, b = 0, ab = 0;
    for (uint64_t w = lane; w < wpr; w += 32) {
      const uint32_t x = __ldg(est + i * wpr + w), y = __ldg(tru + i * wpr + w);
      a += __popc(x); b += __popc(y); ab += __popc(x & y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      ab += __shfl_xor_sync(0xffffffffu, ab, o);
    }
    if (lane == 0) { out[i] = a; out[nq + i] = b; out[2 * nq + i] = ab; }
  }
}

cudaError_t launch_join_rowptr(const uint32_t* bits, uint64_t nq, uint64_t ndb, int32_t* counts, int64_t* row_ptr,
                               cudaStream_t s) {
  const uint64_t wpr = (ndb + 31) / 32;
  cudaError_t e = launch_popcount(bits, nq, (uint32_t)wpr, counts, s);
  if (e != cudaSuccess) return e;
  row_ptr_kernel<<<1, 1024, 0, s>>>(counts, nq, row_ptr);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_join_list(const uint32_t* bits, uint64_t nq, uint64_t ndb, const uint32_t* Q, const uint32_t* D,
                             uint32_t N, const int32_t* pq, const int32_t* pd, const double* L, uint32_t measure,
                             bool exact, const int64_t* row_ptr, int32_t* out_j, float* out_score, uint64_t cap,
                             cudaStream_t s) {
  if (nq == 0 || cap == 0) return cudaSuccess;
  const uint64_t wpr = (ndb + 31) / 32;
  const uint64_t blocks = std::min<uint64_t>((nq * 32 + 255) / 256, (uint64_t)num_sms() * 16);
  join_list_kernel<<<(unsigned)blocks, 256, 0, s>>>(bits, nq, wpr, Q, D, (N + 31) / 32, pq, pd, L, N, measure,
                                                    exact ? 1u : 0u, row_ptr, out_j, out_score, cap);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_join_confusion(const uint32_t* est, const uint32_t* tru, uint64_t nq, uint64_t ndb, int64_t* out,
                                  cudaStream_t s) {
  if (nq == 0) return cudaSuccess;
  const uint64_t blocks = std::min<uint64_t>((nq * 32 + 255) / 256, (uint64_t)num_sms() * 16);
  join_confusion_kernel<<<(unsigned)blocks, 256, 0, s>>>(est, tru, nq, (ndb + 31) / 32, out);
  count_launch();
  return cudaGetLastError();
}

// ---- Experiment 1 -------------------------------------------------------------------------
// Fixed grid (kMseBlocks, device independent) so that every partial sum has a fixed owner and
// a fixed order: block b owns rows r0 + b, r0 + b + G, ... of the row block; thread t strides
// over j > i; thread sums -> warp shuffle tree -> warps in order -> partial[b][t] (+=, the
// block is its only writer; row blocks run in stream order). Result: bit-identical run to run.
constexpr uint32_t kMseBlocks = 1024, kMseThreads = 256, kMseMaxThr = 16;
struct MseThr { double v[kMseMaxThr]; };   // thresholds by value (kernel parameter space)

__global__ void __launch_bounds__(kMseThreads)
mse_block_kernel(const int32_t* __restrict__ pab_s, const int32_t* __restrict__ pab_x, uint64_t r0, uint64_t rows,
                 uint64_t n, const int32_t* __restrict__ ps, const int32_t* __restrict__ px,
                 const double* __restrict__ L, uint32_t N, double dcap, uint32_t m, uint32_t bcs,
                 const MseThr thr, uint32_t nthr, double* __restrict__ part_sse,
                 unsigned long long* __restrict__ part_cnt) {
  __shared__ double s_sse[kMseThreads / 32][kMseMaxThr];
  __shared__ unsigned long long s_cnt[kMseThreads / 32][kMseMaxThr];
  double sse[kMseMaxThr];
  unsigned long long cnt[kMseMaxThr];
#pragma unroll
  for (uint32_t t = 0; t < kMseMaxThr; ++t) { sse[t] = 0.0; cnt[t] = 0ull; }
  for (uint64_t li = blockIdx.x; li < rows; li += gridDim.x) {
    const uint64_t i = r0 + li;
    const int pa = __ldg(ps + i), xa = __ldg(px + i);
    const int32_t* rs = pab_s + li * n;
    const int32_t* rx = pab_x + li * n;
    for (uint64_t j = i + 1 + threadIdx.x; j < n; j += blockDim.x) {
      const int pb = __ldg(ps + j), xb = __ldg(px + j);
      const double key = exact_key(xa, xb, __ldg(rx + j), m);
      const double tru = m == 2u ? -key : key;
      const Est e = bcs ? bcs_estimate_pair(pa, pb, __ldg(rs + j), dcap, L, m)
                        : estimate_pair(pa, pb, __ldg(rs + j), (int)N, L, m);
      const double est = m == 1u ? e.ip : m == 2u ? e.ham : m == 4u ? e.js : e.cs;
      const double df = __dsub_rn(est, tru);
      const double sq = __dmul_rn(df, df);
#pragma unroll
      for (uint32_t t = 0; t < kMseMaxThr; ++t) {
        if (t < nthr && (m == 2u ? tru <= thr.v[t] : tru >= thr.v[t])) { sse[t] = __dadd_rn(sse[t], sq); cnt[t] += 1ull; }
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (uint32_t t = 0; t < kMseMaxThr; ++t) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sse[t] = __dadd_rn(sse[t], __shfl_down_sync(0xffffffffu, sse[t], o));
      cnt[t] += __shfl_down_sync(0xffffffffu, cnt[t], o);
    }
    if (lane == 0) { s_sse[warp][t] = sse[t]; s_cnt[warp][t] = cnt[t]; }
  }
  __syncthreads();
  if (threadIdx.x < nthr) {
    double a = 0.0;
    unsigned long long c = 0ull;
    for (int w = 0; w < (int)(kMseThreads / 32); ++w) { a = __dadd_rn(a, s_sse[w][threadIdx.x]); c += s_cnt[w][threadIdx.x]; }
    part_sse[blockIdx.x * kMseMaxThr + threadIdx.x] = __dadd_rn(part_sse[blockIdx.x * kMseMaxThr + threadIdx.x], a);
    part_cnt[blockIdx.x * kMseMaxThr + threadIdx.x] += c;
  }
}

__global__ void mse_final_kernel(const double* __restrict__ part_sse, const unsigned long long* __restrict__ part_cnt,
                                 uint32_t nthr, double* __restrict__ sse, unsigned long long* __restrict__ cnt) {
  const uint32_t t = threadIdx.x;
  if (t >= nthr) return;
  double a = 0.0;
  unsigned long long c = 0ull;
  for (uint32_t b = 0; b < kMseBlocks; ++b) { a = __dadd_rn(a, part_sse[b * kMseMaxThr + t]); c += part_cnt[b * kMseMaxThr + t]; }
  sse[t] = a;
  cnt[t] = c;
}

uint32_t mse_partial_bytes() { return kMseBlocks * kMseMaxThr * 16; }

cudaError_t launch_mse_block(const int32_t* pab_s, const int32_t* pab_x, uint64_t r0, uint64_t rows, uint64_t n,
                             const int32_t* ps, const int32_t* px, const double* L, uint32_t N, double dcap,
                             uint32_t measure, bool bcs, const double* thr, uint32_t nthr, double* part_sse,
                             unsigned long long* part_cnt, cudaStream_t s) {
  if (nthr > kMseMaxThr) return cudaErrorInvalidValue;
  MseThr t = {};
  for (uint32_t k = 0; k < nthr; ++k) t.v[k] = thr[k];   // host array
  mse_block_kernel<<<kMseBlocks, kMseThreads, 0, s>>>(pab_s, pab_x, r0, rows, n, ps, px, L, N, dcap, measure,
                                                      bcs ? 1u : 0u, t, nthr, part_sse, part_cnt);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_mse_final(const double* part_sse, const unsigned long long* part_cnt, uint32_t nthr, double* sse,
                             unsigned long long* cnt, cudaStream_t s) {
  mse_final_kernel<<<1, 32, 0, s>>>(part_sse, part_cnt, nthr, sse, cnt);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsk
