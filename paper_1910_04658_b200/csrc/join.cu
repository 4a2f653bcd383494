// join.cu — threshold-join post-processing (Experiment 2): the
// per-query match list (CSR, db index ascending, with scores) from a match bitmap, and
// the per-query confusion counts |O'|, |O|, |O ∩ O'| of two bitmaps, from which the
// paper's accuracy / precision / recall / F1 follow.
// The bitmaps themselves come from the tensor-core join (tc.cu, kTcJoin).
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

}  // namespace bsk
