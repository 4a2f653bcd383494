// pairs.cu — all-pairs AND-popcount (K3 mainloop), the fp64 estimator
// epilogue (Algorithms 1-4) and query x db top-k (K4) for sm_100a, CUDA-core
// (LOP3 + POPC) path.
//
// Mainloop: a CTA owns a BM x BN tile of (row of A, row of B) pairs; K = W
// sketch words is streamed in KC-word chunks through shared memory; every
// thread keeps a TM x TN register tile of uint32 AND-popcount accumulators
// (Alg. 1 line 2: n_{as,bs} = <a_s, b_s>).
//
// Epilogue: the canonical fp64 recipe (DESIGN.md R-C3) with the host-built
// cardinality table L (Alg. 1 line 3) staged in shared memory; every fp64
// operation is an explicit round-to-nearest intrinsic, so no FMA contraction
// can change a bit relative to the CPU oracle (this TU is also compiled with
// -fmad=false).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bsk_device.cuh"
#include "bsk_estimator.cuh"
#include "bsk_internal.cuh"

namespace bsk {

// ------------------------------------------------------------ mainloop ----
template <int BM, int BN, int TM, int TN, int KC>
struct TileCfg {
  static constexpr int kThreadsX = BN / TN;
  static constexpr int kThreadsY = BM / TM;
  static constexpr int kThreads = kThreadsX * kThreadsY;
  static constexpr int kLd = KC + 1;  // padded row stride (words): conflict-free column reads
  static constexpr size_t kSmemWords = (size_t)(BM + BN) * kLd;
};

template <int BM, int BN, int TM, int TN, int KC>
__device__ __forceinline__ void mainloop(const uint32_t* __restrict__ A, uint64_t na, uint64_t m0,
                                         const uint32_t* __restrict__ B, uint64_t nb, uint64_t n0,
                                         uint32_t W, uint32_t* As, uint32_t* Bs, uint32_t (&acc)[TM][TN]) {
  using C = TileCfg<BM, BN, TM, TN, KC>;
  const int tid = threadIdx.x;
  const int tx = tid % C::kThreadsX, ty = tid / C::kThreadsX;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0u;
  for (uint32_t k0 = 0; k0 < W; k0 += KC) {
    for (int l = tid; l < BM * KC; l += C::kThreads) {
      const int r = l / KC, kk = l % KC;
      const uint64_t gr = m0 + r;
      const uint32_t gk = k0 + kk;
      As[r * C::kLd + kk] = (gr < na && gk < W) ? __ldg(A + gr * W + gk) : 0u;
    }
    for (int l = tid; l < BN * KC; l += C::kThreads) {
      const int r = l / KC, kk = l % KC;
      const uint64_t gr = n0 + r;
      const uint32_t gk = k0 + kk;
      Bs[r * C::kLd + kk] = (gr < nb && gk < W) ? __ldg(B + gr * W + gk) : 0u;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < KC; ++kk) {
      uint32_t a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[(ty + i * C::kThreadsY) * C::kLd + kk];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[(tx + j * C::kThreadsX) * C::kLd + kk];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] += __popc(a[i] & b[j]);
    }
    __syncthreads();
  }
}

// ------------------------------------------------- all-pairs (K3) ---------
constexpr int kPBM = 64, kPBN = 64, kPTM = 4, kPTN = 4, kPKC = 32;
using PCfg = TileCfg<kPBM, kPBN, kPTM, kPTN, kPKC>;
constexpr uint32_t kMaxSmemL = 6144;   // N+1 <= 6144 doubles (48 KB) staged in smem

template <int MODE>
__global__ void __launch_bounds__(PCfg::kThreads)
pairs_kernel(const uint32_t* __restrict__ A, uint64_t na, const uint32_t* __restrict__ B, uint64_t nb,
             uint32_t N, uint32_t measure, const int32_t* __restrict__ pa, const int32_t* __restrict__ pb,
             const double* __restrict__ Lg, void* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t W = (N + 31) / 32;
  double* Ls = reinterpret_cast<double*>(smem);
  const bool l_in_smem = (MODE == kEstimate) && (N + 1 <= kMaxSmemL);
  const size_t l_bytes = l_in_smem ? (size_t)(N + 1) * 8 : 0;
  uint32_t* As = reinterpret_cast<uint32_t*>(smem + ((l_bytes + 15) / 16) * 16);
  uint32_t* Bs = As + kPBM * PCfg::kLd;
  if (l_in_smem) {
    for (uint32_t i = threadIdx.x; i <= N; i += blockDim.x) Ls[i] = Lg[i];
  }
  const double* L = l_in_smem ? Ls : Lg;

  const uint64_t ntn = (nb + kPBN - 1) / kPBN;
  const uint64_t m0 = (blockIdx.x / ntn) * kPBM, n0 = (blockIdx.x % ntn) * kPBN;
  uint32_t acc[kPTM][kPTN];
  mainloop<kPBM, kPBN, kPTM, kPTN, kPKC>(A, na, m0, B, nb, n0, W, As, Bs, acc);

  const int tx = threadIdx.x % PCfg::kThreadsX, ty = threadIdx.x / PCfg::kThreadsX;
  const uint64_t plane = na * nb;
#pragma unroll
  for (int i = 0; i < kPTM; ++i) {
    const uint64_t r = m0 + ty + i * PCfg::kThreadsY;
    if (r >= na) continue;
    const int par = (MODE == kEstimate) ? pa[r] : 0;
#pragma unroll
    for (int j = 0; j < kPTN; ++j) {
      const uint64_t c = n0 + tx + j * PCfg::kThreadsX;
      if (c >= nb) continue;
      if (MODE == kAndPopc) {
        static_cast<int32_t*>(out)[r * nb + c] = (int32_t)acc[i][j];
      } else {
        const Est e = estimate_pair(par, pb[c], (int)acc[i][j], (int)N, L, measure);
        float* o = static_cast<float*>(out) + r * nb + c;
        if (measure & 1u) { __stcs(o, __double2float_rn(e.ip)); o += plane; }
        if (measure & 2u) { __stcs(o, __double2float_rn(e.ham)); o += plane; }
        if (measure & 4u) { __stcs(o, __double2float_rn(e.js)); o += plane; }
        if (measure & 8u) { __stcs(o, __double2float_rn(e.cs)); }
      }
    }
  }
}

cudaError_t launch_pairs(int mode, const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb,
                         uint32_t N, uint32_t measure, const int32_t* pa, const int32_t* pb,
                         const double* L, void* out, cudaStream_t s) {
  if (na == 0 || nb == 0) return cudaSuccess;
  const size_t l_bytes = (mode == kEstimate && N + 1 <= kMaxSmemL) ? (((size_t)(N + 1) * 8 + 15) / 16) * 16 : 0;
  const size_t smem = l_bytes + PCfg::kSmemWords * 4;
  const uint64_t tiles = ((nb + kPBN - 1) / kPBN) * ((na + kPBM - 1) / kPBM);
  if (tiles > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  const unsigned grid = (unsigned)tiles;
  cudaError_t e;
  if (mode == kAndPopc) {
    e = cudaFuncSetAttribute(pairs_kernel<kAndPopc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    pairs_kernel<kAndPopc><<<grid, PCfg::kThreads, smem, s>>>(A, na, B, nb, N, measure, pa, pb, L, out);
    count_launch();
  } else {
    e = cudaFuncSetAttribute(pairs_kernel<kEstimate>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    pairs_kernel<kEstimate><<<grid, PCfg::kThreads, smem, s>>>(A, na, B, nb, N, measure, pa, pb, L, out);
    count_launch();
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------ top-k (K4) --
// One warp sorts n (power of two) (key, idx) entries in shared memory, best first.
__device__ void warp_bitonic_sort(double* key, int* idx, int n) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < n / 2; i += 32) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;   // "up" block: best first
        const double klo = key[lo], khi = key[hi];
        const int ilo = idx[lo], ihi = idx[hi];
        const bool sw = up ? before(khi, ihi, klo, ilo) : before(klo, ilo, khi, ihi);
        if (sw) {
          key[lo] = khi; key[hi] = klo;
          idx[lo] = ihi; idx[hi] = ilo;
        }
      }
      __syncwarp();
    }
  }
}

// Whole-block variant for the cross-split merge.
__device__ void block_bitonic_sort(double* key, int* idx, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const double klo = key[lo], khi = key[hi];
        const int ilo = idx[lo], ihi = idx[hi];
        const bool sw = up ? before(khi, ihi, klo, ilo) : before(klo, ilo, khi, ihi);
        if (sw) {
          key[lo] = khi; key[hi] = klo;
          idx[lo] = ihi; idx[hi] = ilo;
        }
      }
      __syncthreads();
    }
  }
}

constexpr int kTBN = 64, kTKC = 32;

template <int TQ, int CAP>
struct TopkCfg {
  static constexpr int TM = TQ / 16;   // 16 thread rows
  static constexpr int TN = 4;         // 16 thread cols x 4 = 64
  using C = TileCfg<TQ, kTBN, TM, TN, kTKC>;
};

// FROMPAB: the AND-popcounts come precomputed (pab[nq][ndb], from the tensor-core engine)
// instead of the LOP3+POPC mainloop.
template <int TQ, int CAP, bool FROMPAB>
__global__ void __launch_bounds__(256)
topk_kernel(const uint32_t* __restrict__ Q, uint64_t nq, const uint32_t* __restrict__ D, uint64_t ndb,
            uint32_t N, uint32_t measure, uint32_t k, uint32_t flags, const int32_t* __restrict__ pq,
            const int32_t* __restrict__ pd, const double* __restrict__ Lg, uint32_t splits,
            double* __restrict__ part_key, int32_t* __restrict__ part_idx, int32_t* __restrict__ out_idx,
            float* __restrict__ out_score, const int32_t* __restrict__ pab) {
  using Cfg = TopkCfg<TQ, CAP>;
  using C = typename Cfg::C;
  constexpr int TM = Cfg::TM, TN = Cfg::TN;
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t W = (N + 31) / 32;
  const bool l_in_smem = N + 1 <= kMaxSmemL;
  // layout: ckey[TQ][CAP] | thr[TQ] | L? | cidx[TQ][CAP] | cnt[TQ] | thr_idx[TQ] | As | Bs
  double* ckey = reinterpret_cast<double*>(smem);
  double* thr = ckey + TQ * CAP;
  double* Ls = thr + TQ;
  int* cidx = reinterpret_cast<int*>(Ls + (l_in_smem ? ((N + 2) & ~1u) : 0));
  int* cnt = cidx + TQ * CAP;
  int* thr_idx = cnt + TQ;
  uint32_t* As = reinterpret_cast<uint32_t*>(thr_idx + TQ + ((TQ & 3) ? 4 - (TQ & 3) : 0));
  uint32_t* Bs = As + TQ * C::kLd;
  if (l_in_smem)
    for (uint32_t i = threadIdx.x; i <= N; i += blockDim.x) Ls[i] = Lg[i];
  const double* L = l_in_smem ? Ls : Lg;
  for (int i = threadIdx.x; i < TQ * CAP; i += blockDim.x) {
    ckey[i] = -__longlong_as_double(0x7ff0000000000000LL);   // -inf
    cidx[i] = kSentinelIdx;
  }
  for (int i = threadIdx.x; i < TQ; i += blockDim.x) {
    cnt[i] = 0;
    thr[i] = -__longlong_as_double(0x7ff0000000000000LL);
    thr_idx[i] = kSentinelIdx;
  }
  __syncthreads();

  const uint64_t q0 = (uint64_t)blockIdx.x * TQ;
  const uint32_t s = blockIdx.y;
  const uint64_t per = ((ndb + splits - 1) / splits + kTBN - 1) / kTBN * kTBN;
  const uint64_t cb = (uint64_t)s * per;
  const uint64_t c_begin = cb < ndb ? cb : ndb;
  const uint64_t c_end = (c_begin + per) < ndb ? (c_begin + per) : ndb;
  const int tx = threadIdx.x % C::kThreadsX, ty = threadIdx.x / C::kThreadsX;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int flush_at = CAP - (int)k - kTBN;   // flush when more candidates than this are pending

  int pqr[TM];
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const uint64_t r = q0 + ty + i * C::kThreadsY;
    pqr[i] = r < nq ? pq[r] : 0;
  }

  for (uint64_t n0 = c_begin; n0 < c_end; n0 += kTBN) {
    uint32_t acc[TM][TN];
    if (FROMPAB) {
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const uint64_t r = q0 + ty + i * C::kThreadsY;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const uint64_t c = n0 + tx + j * C::kThreadsX;
          acc[i][j] = (r < nq && c < c_end) ? (uint32_t)__ldcs(pab + r * ndb + c) : 0u;
        }
      }
    } else {
      mainloop<TQ, kTBN, TM, TN, kTKC>(Q, nq, q0, D, c_end, n0, W, As, Bs, acc);
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int ql = ty + i * C::kThreadsY;
      const uint64_t r = q0 + ql;
      if (r >= nq) continue;
      const double t = thr[ql];
      const int ti = thr_idx[ql];
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const uint64_t c = n0 + tx + j * C::kThreadsX;
        if (c >= c_end) continue;
        if ((flags & 1u) && c == r) continue;
        const Est e = estimate_pair(pqr[i], pd[c], (int)acc[i][j], (int)N, L, measure);
        const double key = measure_key(e, measure);
        if (before(key, (int)c, t, ti)) {
          const int pos = atomicAdd(cnt + ql, 1);
          ckey[ql * CAP + (int)k + pos] = key;
          cidx[ql * CAP + (int)k + pos] = (int)c;
        }
      }
    }
    __syncthreads();
    const bool last = n0 + kTBN >= c_end;
    for (int ql = warp; ql < TQ; ql += 8) {
      const int c = cnt[ql];
      if (c > 0 && (last || c > flush_at)) {
        warp_bitonic_sort(ckey + ql * CAP, cidx + ql * CAP, CAP);
        for (int i = (int)k + lane; i < CAP; i += 32) {
          ckey[ql * CAP + i] = -__longlong_as_double(0x7ff0000000000000LL);
          cidx[ql * CAP + i] = kSentinelIdx;
        }
        if (lane == 0) {
          cnt[ql] = 0;
          thr[ql] = ckey[ql * CAP + k - 1];
          thr_idx[ql] = cidx[ql * CAP + k - 1];
        }
        __syncwarp();
      }
    }
    __syncthreads();
  }

  // write results: final (splits == 1) or partial lists
  for (int ql = warp; ql < TQ; ql += 8) {
    const uint64_t r = q0 + ql;
    if (r >= nq) continue;
    for (uint32_t t = lane; t < k; t += 32) {
      const double key = ckey[ql * CAP + t];
      const int id = cidx[ql * CAP + t];
      if (splits == 1) {
        const bool valid = id != kSentinelIdx;
        out_idx[r * k + t] = valid ? id : -1;
        out_score[r * k + t] = valid ? key_to_score(key, measure) : __int_as_float(0x7fc00000);
      } else {
        part_key[(r * splits + s) * k + t] = key;
        part_idx[(r * splits + s) * k + t] = id;
      }
    }
  }
}

__global__ void topk_merge_kernel(uint64_t nq, uint32_t splits, uint32_t k, uint32_t P, uint32_t measure,
                                  const double* __restrict__ part_key, const int32_t* __restrict__ part_idx,
                                  int32_t* __restrict__ out_idx, float* __restrict__ out_score) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* key = reinterpret_cast<double*>(smem);
  int* idx = reinterpret_cast<int*>(key + P);
  const uint64_t q = blockIdx.x;
  const uint32_t total = splits * k;
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
    if (i < total) {
      key[i] = part_key[q * total + i];
      idx[i] = part_idx[q * total + i];
    } else {
      key[i] = -__longlong_as_double(0x7ff0000000000000LL);
      idx[i] = kSentinelIdx;
    }
  }
  __syncthreads();
  block_bitonic_sort(key, idx, (int)P);
  for (uint32_t t = threadIdx.x; t < k; t += blockDim.x) {
    const bool valid = idx[t] != kSentinelIdx;
    out_idx[q * k + t] = valid ? idx[t] : -1;
    out_score[q * k + t] = valid ? key_to_score(key[t], measure) : __int_as_float(0x7fc00000);
  }
}

static uint32_t next_pow2(uint32_t v) {
  uint32_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

static constexpr uint32_t kMaxMergeEntries = 8192;

uint32_t topk_splits(uint64_t nq, uint64_t ndb, uint32_t k) {
  if (nq == 0 || ndb == 0 || k == 0) return 1;
  const uint32_t TQ = k <= 128 - kTBN ? 32u : 16u;   // must match launch_topk
  const uint64_t qtiles = (nq + TQ - 1) / TQ;
  const uint64_t target = 148ull * 4ull;              // fixed: workspace size is device independent
  uint64_t s = (target + qtiles - 1) / qtiles;
  s = std::min<uint64_t>(s, (ndb + 4 * kTBN - 1) / (4 * kTBN));   // >= 4 db tiles per split
  s = std::min<uint64_t>(s, kMaxMergeEntries / k);
  return (uint32_t)std::max<uint64_t>(1, s);
}

template <int TQ, int CAP, bool FROMPAB>
static cudaError_t launch_topk_t2(const uint32_t* Q, uint64_t nq, const uint32_t* D, uint64_t ndb, uint32_t N,
                                  uint32_t measure, uint32_t k, uint32_t flags, const int32_t* pq,
                                  const int32_t* pd, const double* L, uint32_t splits, double* part_key,
                                  int32_t* part_idx, int32_t* out_idx, float* out_score, const int32_t* pab,
                                  cudaStream_t s) {
  using C = typename TopkCfg<TQ, CAP>::C;
  const bool l_in_smem = N + 1 <= kMaxSmemL;
  const size_t smem = (size_t)TQ * CAP * 8 + TQ * 8 + (l_in_smem ? ((N + 2) & ~1u) * 8 : 0) +
                      (size_t)TQ * CAP * 4 + TQ * 4 * 2 + 16 + C::kSmemWords * 4;
  cudaError_t e = cudaFuncSetAttribute(topk_kernel<TQ, CAP, FROMPAB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((nq + TQ - 1) / TQ), splits);
  topk_kernel<TQ, CAP, FROMPAB><<<grid, 256, smem, s>>>(Q, nq, D, ndb, N, measure, k, flags, pq, pd, L, splits,
                                                         part_key, part_idx, out_idx, out_score, pab);
  count_launch();
  return cudaGetLastError();
}

template <int TQ, int CAP>
static cudaError_t launch_topk_t(const uint32_t* Q, uint64_t nq, const uint32_t* D, uint64_t ndb, uint32_t N,
                                 uint32_t measure, uint32_t k, uint32_t flags, const int32_t* pq,
                                 const int32_t* pd, const double* L, uint32_t splits, double* part_key,
                                 int32_t* part_idx, int32_t* out_idx, float* out_score, const int32_t* pab,
                                 cudaStream_t s) {
  return pab ? launch_topk_t2<TQ, CAP, true>(Q, nq, D, ndb, N, measure, k, flags, pq, pd, L, splits, part_key,
                                             part_idx, out_idx, out_score, pab, s)
             : launch_topk_t2<TQ, CAP, false>(Q, nq, D, ndb, N, measure, k, flags, pq, pd, L, splits, part_key,
                                              part_idx, out_idx, out_score, pab, s);
}

cudaError_t launch_topk(const uint32_t* Q, uint64_t nq, const uint32_t* D, uint64_t ndb, uint32_t N,
                        uint32_t measure, uint32_t k, uint32_t flags, const int32_t* pq, const int32_t* pd,
                        const double* L, double* part_key, int32_t* part_idx, int32_t* out_idx,
                        float* out_score, cudaStream_t s, const int32_t* pab) {
  if (nq == 0 || k == 0) return cudaSuccess;
  const uint32_t splits = topk_splits(nq, ndb, k);
  cudaError_t e;
  if (k <= 128 - kTBN)       e = launch_topk_t<32, 128>(Q, nq, D, ndb, N, measure, k, flags, pq, pd, L, splits, part_key, part_idx, out_idx, out_score, pab, s);
  else if (k <= 256 - kTBN)  e = launch_topk_t<16, 256>(Q, nq, D, ndb, N, measure, k, flags, pq, pd, L, splits, part_key, part_idx, out_idx, out_score, pab, s);
  else                       e = launch_topk_t<16, 512>(Q, nq, D, ndb, N, measure, k, flags, pq, pd, L, splits, part_key, part_idx, out_idx, out_score, pab, s);
  if (e != cudaSuccess || splits == 1) return e;
  return launch_topk_merge(nq, splits, k, measure, part_key, part_idx, out_idx, out_score, s);
}

cudaError_t launch_topk_merge(uint64_t nq, uint32_t splits, uint32_t k, uint32_t measure, const double* part_key,
                              const int32_t* part_idx, int32_t* out_idx, float* out_score, cudaStream_t s) {
  if (nq == 0 || k == 0) return cudaSuccess;
  const uint32_t P = next_pow2(splits * k);
  const size_t smem = (size_t)P * 12;
  cudaError_t e = cudaFuncSetAttribute(topk_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  topk_merge_kernel<<<(unsigned)nq, 256, smem, s>>>(nq, splits, k, P, measure, part_key, part_idx, out_idx, out_score);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsk
