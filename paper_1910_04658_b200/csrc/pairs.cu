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
#include <cstdlib>
#include <type_traits>

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
  // the all-planes call (the common one) is compiled with the measure mask as a constant
  auto epilogue = [&](auto mtag) {
    constexpr uint32_t MM = decltype(mtag)::value;
    const uint32_t mm = MM ? MM : measure;
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
          const Est e = estimate_pair(par, pb[c], (int)acc[i][j], (int)N, L, mm);
          float* o = static_cast<float*>(out) + r * nb + c;
          if (mm & 1u) { __stcs(o, __double2float_rn(e.ip)); o += plane; }
          if (mm & 2u) { __stcs(o, __double2float_rn(e.ham)); o += plane; }
          if (mm & 4u) { __stcs(o, __double2float_rn(e.js)); o += plane; }
          if (mm & 8u) { __stcs(o, __double2float_rn(e.cs)); }
        }
      }
    }
  };
  if (MODE == kEstimate && measure == 15u) epilogue(std::integral_constant<uint32_t, 15u>{});
  else epilogue(std::integral_constant<uint32_t, 0u>{});
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
        const int pbc = pd[c];
        // division-free pre-test against the row's threshold: the IP part of the recipe, then a
        // conservative (1e-9 relative margin) necessary condition for key >= t; only pairs that
        // pass pay for the exact key (division / square root)
        if (t > -1e300 && !pretest_keep(pqr[i], pbc, (int)acc[i][j], (int)N, L, measure, t)) continue;
        const Est e = estimate_pair(pqr[i], pbc, (int)acc[i][j], (int)N, L, measure);
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

// Same merge with one warp per query row (8 rows per block) for short lists (P <= 256): the
// chained tensor-core top-k hands over one k-list per row, and a 256-thread block per row
// spent most of its time in block barriers.
__global__ void topk_merge_warp_kernel(uint64_t nq, uint32_t splits, uint32_t k, uint32_t P, uint32_t measure,
                                       const double* __restrict__ part_key, const int32_t* __restrict__ part_idx,
                                       int32_t* __restrict__ out_idx, float* __restrict__ out_score) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* key = reinterpret_cast<double*>(smem) + (size_t)warp * P;
  int* idx = reinterpret_cast<int*>(reinterpret_cast<double*>(smem) + 8 * (size_t)P) + (size_t)warp * P;
  const uint64_t q = (uint64_t)blockIdx.x * 8 + warp;
  if (q >= nq) return;
  const uint32_t total = splits * k;
  for (uint32_t i = lane; i < P; i += 32) {
    if (i < total) {
      key[i] = part_key[q * total + i];
      idx[i] = part_idx[q * total + i];
    } else {
      key[i] = -__longlong_as_double(0x7ff0000000000000LL);
      idx[i] = kSentinelIdx;
    }
  }
  __syncwarp();
  warp_bitonic_sort(key, idx, (int)P);
  for (uint32_t t = lane; t < k; t += 32) {
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

// ------------------------------------------------ estimate from a pab table ---
// The all-pairs estimate split in two: the tensor-core AND-popcount writes pab[na][nb] (int32),
// then this elementwise kernel evaluates the recipe (Alg. 1-4, canonical order) for every pair
// and writes the float planes. The recipe is latency-bound fp64 work; here it runs at full
// occupancy (one row segment of 4 columns per thread, 16-B loads and stores) instead of in the
// 16 epilogue warps of the persistent tensor-core kernel. MM: the measure mask at compile time
// (15 = every plane), 0 = runtime mask (BCS / scaled Hamming variants too).
// 4 blocks per SM (64 registers): latency-bound fp64 chains need the warps (vs 3 blocks at 80 registers:
// Medium N = 1000 0.91 -> 0.89 ms, BCS 0.96 -> 0.85 ms)
// SQ: the block owns whole rows (gridDim.x == 1) and memoises the COS denominator
// sqrt(L[pa] * L[pb]) per |b_s| value in shared memory for each row — the same correctly rounded
// operations as the recipe, computed N + 1 times per row instead of once per pair.
template <int MM, bool SQ, bool BCS = false>
__global__ void __launch_bounds__(256, 4)
estimate_pab_kernel(const int32_t* __restrict__ pab, uint64_t na, uint64_t nb, uint32_t N, uint32_t measure,
                    const int32_t* __restrict__ pa, const int32_t* __restrict__ pb, const double* __restrict__ Lg,
                    uint32_t bcs, double dcap, double ham_scale, float* __restrict__ out) {
  extern __shared__ __align__(16) double Ls[];
  const bool l_in_smem = N + 1 <= kMaxSmemL;
  if (l_in_smem)
    for (uint32_t i = threadIdx.x; i <= N; i += blockDim.x) Ls[i] = Lg[i];
  __syncthreads();
  const double* L = l_in_smem ? Ls : Lg;
  double* sq = Ls + (N + 1);
  const uint32_t mm = MM ? (uint32_t)MM : measure;
  const uint64_t plane = na * nb;
  const bool vec = (nb & 3u) == 0 && (reinterpret_cast<uintptr_t>(pab) & 15u) == 0 &&
                   (reinterpret_cast<uintptr_t>(pb) & 15u) == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  const uint64_t nb4 = (nb + 3) / 4;
  for (uint64_t r = blockIdx.y; r < na; r += gridDim.y) {
    const int a = __ldg(pa + r);
    if constexpr (SQ) {
      __syncthreads();   // the previous row's denominators are no longer read
      const double La = L[a];
      for (uint32_t i = threadIdx.x; i <= N; i += blockDim.x) sq[i] = __dsqrt_rn(__dmul_rn(La, L[i]));
      __syncthreads();
    }
    for (uint64_t c4 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c4 < nb4; c4 += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t c = 4 * c4;
      int v[4], b[4];
      if (vec) {
        const int4 v4 = __ldcs(reinterpret_cast<const int4*>(pab + r * nb + c));
        const int4 b4 = __ldg(reinterpret_cast<const int4*>(pb + c));
        v[0] = v4.x; v[1] = v4.y; v[2] = v4.z; v[3] = v4.w;
        b[0] = b4.x; b[1] = b4.y; b[2] = b4.z; b[3] = b4.w;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u] = c + u < nb ? __ldcs(pab + r * nb + c + u) : 0;
          b[u] = c + u < nb ? __ldg(pb + c + u) : 0;
        }
      }
      float val[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        Est e;
        if (BCS || (MM == 0 && bcs)) e = bcs_estimate_pair(a, b[u], v[u], dcap, L, SQ ? (mm & 7u) : mm);
        else e = estimate_pair(a, b[u], v[u], (int)N, L, SQ ? (mm & 7u) : mm);
        if constexpr (SQ) {   // COS with the memoised denominator (the recipe's operations)
          if (a == 0 || b[u] == 0) {
            e.cs = 0.0;
          } else {
            double cv = __ddiv_rn(e.ip, sq[b[u]]);
            cv = cv > 0.0 ? cv : 0.0;
            e.cs = cv < 1.0 ? cv : 1.0;
          }
        }
        val[0][u] = __double2float_rn(e.ip);
        val[1][u] = __double2float_rn(MM ? e.ham : __dmul_rn(e.ham, ham_scale));
        val[2][u] = __double2float_rn(e.js);
        val[3][u] = __double2float_rn(e.cs);
      }
      float* o = out + r * nb + c;
#pragma unroll
      for (uint32_t id = 0; id < 4; ++id) {
        if (!(mm & (1u << id))) continue;
        float* oq = o + (uint64_t)__popc(mm & ((1u << id) - 1u)) * plane;
        if (vec) {
          __stcs(reinterpret_cast<float4*>(oq), make_float4(val[id][0], val[id][1], val[id][2], val[id][3]));
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c + u < nb) __stcs(oq + u, val[id][u]);
        }
      }
    }
  }
}

cudaError_t launch_estimate_from_pab(const int32_t* pab, uint64_t na, uint64_t nb, uint32_t N, uint32_t measure,
                                     const int32_t* pa, const int32_t* pb, const double* L, float* out, cudaStream_t s,
                                     bool bcs, double dcap, double ham_scale) {
  if (na == 0 || nb == 0) return cudaSuccess;
  const size_t smem = N + 1 <= kMaxSmemL ? (size_t)(N + 1) * 8 : 0;
  const uint64_t nb4 = (nb + 3) / 4;
  const unsigned gx = (unsigned)std::min<uint64_t>((nb4 + 255) / 256, 64);
  const unsigned gy = (unsigned)std::min<uint64_t>(na, std::max<uint64_t>(1, (uint64_t)num_sms() * 16 / gx));
  const bool all = measure == 15u && !bcs && ham_scale == 1.0;
  // COS denominators memoised per row while both tables fit 48 KB and a row is long enough to
  // amortise them (N + 1 square roots per row against nb pairs)
  // (BCS too: its COS is ip / sqrt(B[pa] B[pb]) over its own table, the same memo)
  const bool sqm = measure == 15u && ham_scale == 1.0 && (size_t)(N + 1) * 16 <= 48 * 1024 && nb >= 4 * (uint64_t)(N + 1);
  cudaError_t e;
  if (sqm) {
    const size_t smem2 = (size_t)(N + 1) * 16;
    const unsigned gy2 = (unsigned)std::min<uint64_t>(na, (uint64_t)num_sms() * 16);
    auto kern = bcs ? estimate_pab_kernel<15, true, true> : estimate_pab_kernel<15, true, false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    if (e != cudaSuccess) return e;
    kern<<<dim3(1, gy2), 256, smem2, s>>>(pab, na, nb, N, measure, pa, pb, L, bcs ? 1u : 0u, dcap, ham_scale, out);
  } else if (all) {
    e = cudaFuncSetAttribute(estimate_pab_kernel<15, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    estimate_pab_kernel<15, false><<<dim3(gx, gy), 256, smem, s>>>(pab, na, nb, N, measure, pa, pb, L, 0u, dcap,
                                                                  ham_scale, out);
  } else {
    e = cudaFuncSetAttribute(estimate_pab_kernel<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    estimate_pab_kernel<0, false><<<dim3(gx, gy), 256, smem, s>>>(pab, na, nb, N, measure, pa, pb, L, bcs ? 1u : 0u, dcap,
                                                                 ham_scale, out);
  }
  count_launch();
  return cudaGetLastError();
}

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

// ------------------------------------------- pab-table top-k, integer screen (K4c) --
// For fixed (pa, pb) every measure key is a non-decreasing function of pab: in estimate_pair
// pu = pa + pb - pab falls as pab rises, so L[pu] falls and ip = S - L[pu] (clamped) rises;
// JS = ip / (S - ip), COS = ip / sqrt(La Lb) and -HAM = 2 ip - S rise with ip; every fp64 step
// is correctly rounded and hence monotone. So for a query row (pa fixed) and a threshold key t,
// "key >= t" is exactly "pab >= T_t[pb]" with T_t[pb] the smallest pab whose key reaches t: the
// scan over the table is one integer compare per pair and measure against a per-query table in
// shared memory, and only the (few) pairs that pass are scored.
#ifdef BSK_PABT_STATS   // dev: counters for tools/pabT_stats.py (variant library only)
__device__ unsigned long long g_pabt[16];
#define PABT_ADD(i, v) atomicAdd(&g_pabt[i], (unsigned long long)(v))
#else
#define PABT_ADD(i, v) ((void)0)
#endif

__device__ __forceinline__ double pab_key(int pa, int pb, int pab, int N, const double* __restrict__ L, uint32_t m) {
  return measure_key(estimate_pair(pa, pb, pab, N, L, m), m);
}

// The smallest pab in [max(pa + pb - N, 0, from), min(pa, pb)] whose key reaches t, 0xFFFF if
// none (no table value exceeds N <= 16383). `from` is a known lower bound of the answer (the
// previous table value: t only rises). A guess from the inverted recipe — key >= t needs
// ip >= ipmin (IP: t; -HAM: (S + t) / 2; JS: t S / (1 + t); COS: t sqrt(La Lb)), i.e.
// L[pu] <= S - ipmin, the largest such pu by bisection of the (non-decreasing) L table, and
// pab = pa + pb - pu — is then settled by the exact key, stepping down while the key still
// reaches t and up while it does not (the guess is off by rounding only: a step or two).
__device__ uint16_t min_pab(int pa, int pb, int N, const double* __restrict__ L, uint32_t m, double t, int from) {
  const int lo = max(max(0, pa + pb - N), from);
  const int hi = min(pa, pb);
  if (lo > hi) return 0xFFFFu;
  const double La = L[pa], Lb = L[pb];
  const double S = La + Lb;
  double ipmin;
  if (m == 1u) ipmin = t;
  else if (m == 2u) ipmin = 0.5 * (S + t);
  else if (m == 4u) ipmin = t > 0.0 ? t * S / (1.0 + t) : -1.0;
  else ipmin = t > 0.0 ? t * sqrt(La * Lb) : -1.0;
  int g;   // guess
  if (!(ipmin > 0.0)) {
    g = lo;
  } else {
    // largest pu in [pa + pb - hi, pa + pb - lo] with L[pu] <= S - ipmin (pu = pa + pb - pab)
    const double y = S - ipmin;
    int plo = pa + pb - hi, phi = pa + pb - lo;
    if (L[plo] > y) {
      g = hi + 1;   // even the largest pab misses the target: check hi below
    } else {
      while (plo < phi) {
        const int mid = (plo + phi + 1) >> 1;
        if (L[mid] <= y) plo = mid;
        else phi = mid - 1;
      }
      g = pa + pb - plo;
    }
  }
  g = min(max(g, lo), hi);
  if (pab_key(pa, pb, g, N, L, m) >= t) {
    while (g > lo && pab_key(pa, pb, g - 1, N, L, m) >= t) --g;
    return (uint16_t)g;
  }
  do {
    ++g;
  } while (g <= hi && pab_key(pa, pb, g, N, L, m) < t);
  return g <= hi ? (uint16_t)g : (uint16_t)0xFFFFu;
}

// [min, max] of x[0..n) into out[0], out[1], which hold (INT_MAX-ish, INT_MIN-ish) byte patterns
// on entry (0x7f7f7f7f, 0x80808080: two memsets).
__global__ void __launch_bounds__(256) int_range_kernel(const int32_t* __restrict__ x, uint64_t n,
                                                        int32_t* __restrict__ out) {
  int lo = 0x7fffffff, hi = -0x7fffffff - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const int v = __ldg(x + i);
    lo = min(lo, v);
    hi = max(hi, v);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}

// One block per query row (grid-stride), every requested measure in the same passes over the
// row's pab values, with no per-step block barriers:
//  1. sample: exact keys of the first kPabSample columns into a kHB-bucket histogram over the
//     measure's key range; t_s = the lower edge of the highest bucket with >= k sample pairs at
//     or above it (so >= k pairs of the row have key >= t_s: a lower bound of its k-th key);
//     T = the minimum-pab table for t_s.
//  2. the whole row through the screen pab >= T[pb]; exact keys of the survivors into a
//     histogram over [t_s, key max]; t0 >= t_s the same way; T raised to t0.
//  3. the whole row through the raised screen; survivors that beat the running k-th (tk, ti)
//     are buffered. Typically they number k plus one bucket's worth and fit; on an overflow the
//     pass restarts in steps of 256 columns with a barrier each, cutting the buffer back to k
//     (block bitonic sort) whenever the next step could overflow it.
// The buffer is then sorted and its head written. Every compare is on the exact fp64 key, so
// the result is the exact top-k whatever the histograms hold; they only set the screens.
constexpr int kHB = 2048;               // histogram buckets (256 threads x 8)
constexpr uint32_t kPabSample = 4096;   // pass-1 columns
constexpr int kPab3Cap = 512;           // pass-3 buffer entries per measure (k <= 256)
constexpr uint32_t kPab3Slow = 256;     // pass-3 step after an overflow (1 column per thread)
constexpr uint32_t kPab3Keep = 8192;    // pass-2 survivors kept per (block, measure) in the scratch
constexpr uint32_t kPab3Slots = 592;    // blocks (scratch slots) at most: 4 per SM on 148 SMs
constexpr int kRing = 4;                // pab row ring: one-step chunks (256 threads x 16 B)

__device__ __forceinline__ uint4 lds_v4u(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u32u(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
#ifndef BSK_PAB3_MINB
#define BSK_PAB3_MINB 3
#endif

template <int NM>
__global__ void __launch_bounds__(256, BSK_PAB3_MINB)
topk_pab3_kernel(const int32_t* __restrict__ pab, uint64_t nq, uint64_t ndb, uint32_t N, uint32_t mask, uint32_t k,
                 uint32_t flags, const int32_t* __restrict__ pq, const int32_t* __restrict__ pd,
                 const double* __restrict__ Lg, const int32_t* __restrict__ pdr, double* __restrict__ skey,
                 int32_t* __restrict__ sidx, int32_t* __restrict__ out_idx, float* __restrict__ out_score) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int kQ = 32 + 128 * NM;   // per-warp survivor queue: < 32 waiting + one step's worth
  uint32_t ms[NM];
  {
    uint32_t mm = mask, j = 0;
#pragma unroll
    for (int i = 0; i < NM; ++i) { ms[i] = mm & (0u - mm); mm &= mm - 1; (void)j; }
  }
  const uint32_t TS = N + 1;
  const size_t lbytes = 0;   // L stays in global memory (read through L1: 8(N+1) bytes, hot)
  constexpr size_t hbytes = (size_t)NM * kHB * 4 > (size_t)NM * kPab3Cap * 12 ? (size_t)NM * kHB * 4
                                                                              : (size_t)NM * kPab3Cap * 12;
  const size_t tbytes = ((size_t)(NM == 3 ? 4 : NM) * TS * 2 + 15) & ~(size_t)15;
  const double* __restrict__ L = Lg;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + lbytes);                  // [NM][kHB] (passes 1-2)
  double* bkey = reinterpret_cast<double*>(smem + lbytes);                      // [NM][kPab3Cap] (pass 3)
  int* bidx = reinterpret_cast<int*>(smem + lbytes + (size_t)NM * kPab3Cap * 8);
  constexpr int NMP = NM == 3 ? 4 : NM;   // table entries per pb (one 2/4/8-byte load per column)
  uint16_t* T = reinterpret_cast<uint16_t*>(smem + lbytes + hbytes);            // [N + 1][NMP]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint2* queue = reinterpret_cast<uint2*>(smem + lbytes + hbytes + tbytes) + warp * kQ;   // (column, v|b<<14|mi<<28)
  __shared__ uint32_t cnt[NM];
  __shared__ double tk[NM];
  __shared__ int ti[NM];
  __shared__ double lo_s[NM], sc_s[NM], tl_s[NM];
  __shared__ uint32_t warp_sum[8];
  __shared__ int found;
  __shared__ int ovf;
  __shared__ uint32_t scnt[NM];
  __shared__ __align__(8) unsigned long long rbar[2 * kRing];   // full[kRing], empty[kRing]
  const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(rbar);
  const uint32_t ring_a = (uint32_t)__cvta_generic_to_shared(queue - warp * kQ + 8 * kQ);   // [kRing][blockDim.x * 4] int
  uint32_t g0 = 0;   // row chunks streamed through the ring so far (block-uniform)
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(bar_a + 8u * i, 1);
      mbar_init(bar_a + 8u * (kRing + i), blockDim.x / 32);
    }
    fence_proxy_async();
  }
  const double kNegInf = -__longlong_as_double(0x7ff0000000000000LL);
  const int pdlo = pdr[0], pdhi = pdr[1];
  const bool vec = (ndb & 3u) == 0 && (reinterpret_cast<uintptr_t>(pab) & 15u) == 0 &&
                   (reinterpret_cast<uintptr_t>(pd) & 15u) == 0;
  auto load = [&](const int32_t* prow, uint32_t cl, uint32_t cend, int (&v)[4], int (&b)[4]) {
    if (vec && cl + 3 < cend) {
      const int4 a4 = __ldcs(reinterpret_cast<const int4*>(prow + cl));
      const int4 p4 = __ldg(reinterpret_cast<const int4*>(pd + cl));
      v[0] = a4.x; v[1] = a4.y; v[2] = a4.z; v[3] = a4.w;
      b[0] = p4.x; b[1] = p4.y; b[2] = p4.z; b[3] = p4.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = cl + u < cend ? __ldcs(prow + cl + u) : 0;
        b[u] = cl + u < cend ? __ldg(pd + cl + u) : 0;
      }
    }
  };
  // Walk columns [c, cend) of the row (32-bit indices: ndb < 2^31), 4 per thread per step,
  // calling f(cl, v, b, ok) once per step with ok bit u set for the columns cl + u to consider
  // (inside the range, not the excluded self pair). The pab values stream through a ring of
  // kRing one-step chunks in shared memory, filled by 1-D bulk copies (TMA engine) that thread 0
  // issues kRing - 1 steps ahead (the latency x bandwidth product needs tens of KB in flight per
  // SM, far more than a register prefetch holds); the db popcounts (L2-resident) come through
  // registers one step ahead. Unaligned rows take the register path for both.
  auto walk = [&](const int32_t* prow, uint64_t r, uint32_t c, uint32_t cend, auto&& f) {
    const uint32_t stride = 4 * blockDim.x;
    const uint32_t self = (flags & 1u) ? (uint32_t)r : 0xffffffffu;
    auto okmask = [&](uint32_t c0, uint32_t cl) -> uint32_t {
      if (c0 + stride <= cend && (self < c0 || self >= c0 + stride)) return 0xfu;   // whole step inside
      uint32_t ok = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (cl + u < cend && cl + u != self) ok |= 1u << u;
      return ok;
    };
    if (c >= cend) return;
    if (!vec) {
      int va[4], ba[4], vb[4], bb[4];
      uint32_t cl = c + 4 * threadIdx.x;
      load(prow, cl, cend, va, ba);
      for (uint32_t c0 = c; c0 < cend; c0 += 2 * stride, cl += 2 * stride) {
        const bool m1 = c0 + stride < cend;
        if (m1) load(prow, cl + stride, cend, vb, bb);
        f(cl, va, ba, okmask(c0, cl));
        if (!m1) break;
        if (c0 + 2 * stride < cend) load(prow, cl + 2 * stride, cend, va, ba);
        f(cl + stride, vb, bb, okmask(c0 + stride, cl + stride));
      }
      return;
    }
    const uint32_t nch = (cend - c + stride - 1) / stride;
    // chunk j (global sequence number g0 + j) -> slot (g0 + j) % kRing; its 16-B part by bulk copy
    auto issue = [&](uint32_t j) {
      const uint32_t gj = g0 + j, slot = gj % kRing;
      const uint32_t full = bar_a + 8u * slot, empty = bar_a + 8u * (kRing + slot);
      if (gj >= kRing) mbar_wait(empty, ((gj / kRing) - 1) & 1u);   // the slot's previous chunk consumed
      fence_proxy_async();
      const uint32_t s0 = c + j * stride;
      const uint32_t nb = (min(s0 + stride, cend) - s0) * 4 & ~15u;
      if (nb > 0) {
        mbar_expect_tx(full, nb);
        bulk_load(ring_a + slot * 16u * blockDim.x, prow + s0, nb, full);
      } else {
        mbar_arrive(full);
      }
    };
    if (threadIdx.x == 0)
      for (uint32_t j = 0; j < min(nch, (uint32_t)kRing - 1); ++j) issue(j);
    int b[4], bn[4];
    uint32_t cl = c + 4 * threadIdx.x;
    {
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = cl + u < cend ? __ldg(pd + cl + u) : 0;
    }
    for (uint32_t j = 0; j < nch; ++j, cl += stride) {
      const uint32_t c0 = c + j * stride;
      const bool more = j + 1 < nch;
      if (more) {
        if (cl + stride + 3 < cend) {
          const int4 p4 = __ldg(reinterpret_cast<const int4*>(pd + cl + stride));
          bn[0] = p4.x; bn[1] = p4.y; bn[2] = p4.z; bn[3] = p4.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) bn[u] = cl + stride + u < cend ? __ldg(pd + cl + stride + u) : 0;
        }
      }
      if (threadIdx.x == 0 && j + kRing - 1 < nch) issue(j + kRing - 1);
      const uint32_t gj = g0 + j, slot = gj % kRing;
      mbar_wait(bar_a + 8u * slot, (gj / kRing) & 1u);
      int v[4];
      const uint32_t bulk_end = c0 + (((min(c0 + stride, cend) - c0) * 4 & ~15u) >> 2);
      if (cl + 3 < bulk_end) {
        const uint4 q = lds_v4u(ring_a + slot * 16u * blockDim.x + 16u * threadIdx.x);
        v[0] = (int)q.x; v[1] = (int)q.y; v[2] = (int)q.z; v[3] = (int)q.w;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = cl + u < bulk_end ? (int)lds_u32u(ring_a + slot * 16u * blockDim.x + 4u * (threadIdx.x * 4 + u))
                                   : (cl + u < cend ? __ldg(prow + cl + u) : 0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_a + 8u * (kRing + slot));   // this warp is done with the slot
      f(cl, v, b, okmask(c0, cl));
      if (more) {
#pragma unroll
        for (int u = 0; u < 4; ++u) b[u] = bn[u];
      }
    }
    g0 += nch;
  };
  // Screened walk: the (column, measure) items with pab >= T[mi][pb] go to the warp's queue;
  // every full 32 are scored by the warp's 32 lanes together (dense fp64 work instead of one
  // divergent lane per warp-step) and handed to g(column, mi, key); the rest at the end.
  auto screened = [&](const int32_t* prow, uint64_t r, auto&& g) {
    int qn = 0;   // warp-uniform
    const int pa_ = pq[r];
    auto drain = [&](int n) {   // score the top n (<= 32) queue entries
      if (lane < n) {
        const uint2 it = queue[qn - n + lane];
        const int v = (int)(it.y & 0x3fffu), b = (int)((it.y >> 14) & 0x3fffu);
        const uint32_t mi = it.y >> 28;
        uint32_t m = ms[0];
#pragma unroll
        for (int i = 1; i < NM; ++i) m = mi == (uint32_t)i ? ms[i] : m;
        g((uint64_t)it.x, mi, pab_key(pa_, b, v, (int)N, L, m));
      }
      qn -= n;
      __syncwarp();
    };
    walk(prow, r, 0, (uint32_t)ndb, [&](uint32_t cl, const int (&v)[4], const int (&b)[4], uint32_t ok) {
      uint32_t pm = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint16_t tv[NMP];
        if constexpr (NMP == 1) {
          tv[0] = T[b[u]];
        } else if constexpr (NMP == 2) {
          const ushort2 t2 = reinterpret_cast<const ushort2*>(T)[b[u]];
          tv[0] = t2.x; tv[1] = t2.y;
        } else {
          const ushort4 t4 = reinterpret_cast<const ushort4*>(T)[b[u]];
          tv[0] = t4.x; tv[1] = t4.y; tv[2] = t4.z; tv[3] = t4.w;
        }
#pragma unroll
        for (int mi = 0; mi < NM; ++mi)
          if (((ok >> u) & 1u) && v[u] >= (int)tv[mi]) pm |= 1u << (u * NM + mi);
      }
      const uint32_t n = __popc(pm);
      if (__any_sync(0xffffffffu, n != 0)) {
        uint32_t off = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, off, o); if (lane >= o) off += y; }
        const uint32_t total = __shfl_sync(0xffffffffu, off, 31);
        uint32_t pos = (uint32_t)qn + off - n;
        while (pm) {
          const int bit = __ffs(pm) - 1;
          pm &= pm - 1;
          const int u = bit / NM, mi = bit % NM;
          queue[pos++] = make_uint2((uint32_t)(cl + u), (uint32_t)v[u] | ((uint32_t)b[u] << 14) | ((uint32_t)mi << 28));
        }
        qn += (int)total;
        __syncwarp();
        while (qn >= 32) drain(32);
      }
    });
    if (qn > 0) drain(qn);
  };
  // Highest bucket h with >= k counts in buckets >= h, or -1 (block-wide; thread t owns buckets
  // [kHB - 8(t+1), kHB - 8t), scanned from the top).
  auto select = [&](const uint32_t* hm) -> int {
    const int top = kHB - 8 * (int)threadIdx.x;
    uint32_t loc = 0;
#pragma unroll
    for (int j = 1; j <= 8; ++j) loc += hm[top - j];
    uint32_t inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
    if (lane == 31) warp_sum[warp] = inc;
    if (threadIdx.x == 0) found = -1;
    __syncthreads();
    uint32_t before_w = 0;
    for (int w = 0; w < warp; ++w) before_w += warp_sum[w];
    const uint32_t excl = before_w + inc - loc;
    if (excl < k && excl + loc >= k) {
      uint32_t run = excl;
      for (int j = 1; j <= 8; ++j) {
        run += hm[top - j];
        if (run >= k) { found = top - j; break; }
      }
    }
    __syncthreads();
    const int h = found;
    __syncthreads();
    return h;
  };
  auto bucket = [&](uint32_t mi, double key) -> int {
    const double x = (key - lo_s[mi]) * sc_s[mi];
    return x <= 0.0 ? 0 : (x >= (double)(kHB - 1) ? kHB - 1 : (int)x);
  };
  // lower bound from a selected bucket (h > 0): its lower edge less a rounding margin
  auto edge = [&](uint32_t mi, int h) -> double {
    if (h <= 0 || !(sc_s[mi] > 0.0)) return kNegInf;
    const double e = lo_s[mi] + (double)h / sc_s[mi];
    return e - 1e-12 * fmax(1.0, fmax(fabs(e), fabs(lo_s[mi])));
  };
  // sort measure mi's n buffered candidates, keep the best k, raise (tk, ti) and T (block-wide)
  auto flush = [&](uint32_t mi, uint32_t n, int pa) {
    double* key = bkey + mi * kPab3Cap;
    int* idx = bidx + mi * kPab3Cap;
    uint32_t P = 2;
    while (P < n) P <<= 1;
    for (uint32_t i = n + threadIdx.x; i < P; i += blockDim.x) { key[i] = kNegInf; idx[i] = kSentinelIdx; }
    __syncthreads();
    block_bitonic_sort(key, idx, (int)P);
    const bool full = n >= k;
    const double nt = full ? key[k - 1] : kNegInf;
    const int nti = full ? idx[k - 1] : kSentinelIdx;
    const bool raise = full && nt > tl_s[mi];
    __syncthreads();
    if (threadIdx.x == 0) {
      cnt[mi] = full ? k : n;
      tk[mi] = nt;
      ti[mi] = nti;
      if (raise) tl_s[mi] = nt;
    }
    if (raise)
      for (int pb = pdlo + (int)threadIdx.x; pb <= pdhi; pb += (int)blockDim.x)
        T[pb * NMP + mi] = min_pab(pa, pb, (int)N, L, ms[mi], nt, (int)T[pb * NMP + mi]);
    __syncthreads();
  };
  // pass-3 consumer: buffer a survivor that beats the running k-th
  auto collect = [&](uint64_t c, uint32_t mi, double key) {
    PABT_ADD(3, 1);
    if (!before(key, (int)c, tk[mi], ti[mi])) return;
    const uint32_t pos = atomicAdd(&cnt[mi], 1u);
    if (pos < (uint32_t)kPab3Cap) {
      bkey[mi * kPab3Cap + pos] = key;
      bidx[mi * kPab3Cap + pos] = (int)c;
    } else {
      ovf = 1;
    }
  };
  for (uint64_t r = blockIdx.x; r < nq; r += gridDim.x) {
    const int pa = pq[r];
    const int32_t* prow = pab + r * ndb;
    const double La = L[pa];
#ifdef BSK_PABT_STATS
    long long tph = clock64();
#define PHASE(i) do { if (threadIdx.x == 0) { const long long t_ = clock64(); PABT_ADD(i, t_ - tph); tph = t_; } } while (0)
#else
#define PHASE(i) ((void)0)
#endif
    const double Lbmax = fmax(L[pdhi], L[pdhi < (int)N ? pdhi : (int)N - 1]);
    // ---- pass 1: sample histogram over each measure's whole key range
    for (uint32_t i = threadIdx.x; i < NM * kHB; i += blockDim.x) hist[i] = 0u;
    if (threadIdx.x < NM) {
      uint32_t m = ms[0];
#pragma unroll
      for (int i = 1; i < NM; ++i) m = threadIdx.x == (unsigned)i ? ms[i] : m;
      const double lo = m == 2u ? -(La + Lbmax) : 0.0;
      const double hi = m == 1u ? La : (m == 2u ? 0.0 : 1.0);
      lo_s[threadIdx.x] = lo;
      sc_s[threadIdx.x] = (hi > lo && hi - lo < 1e300) ? (double)kHB / (hi - lo) : 0.0;
    }
    __syncthreads();
    walk(prow, r, 0, (uint32_t)min(ndb, (uint64_t)kPabSample), [&](uint32_t cl, const int (&v)[4], const int (&b)[4], uint32_t ok) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if ((ok >> u) & 1u)
#pragma unroll
          for (int mi = 0; mi < NM; ++mi)
            atomicAdd(hist + mi * kHB + bucket(mi, pab_key(pa, b[u], v[u], (int)N, L, ms[mi])), 1u);
    });
    __syncthreads();
    PHASE(5);
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) {
      const double ts = edge(mi, select(hist + mi * kHB));
      if (threadIdx.x == 0) tl_s[mi] = ts;
      for (int pb = pdlo + (int)threadIdx.x; pb <= pdhi; pb += (int)blockDim.x)
        T[pb * NMP + mi] = ts == kNegInf ? (uint16_t)0 : min_pab(pa, pb, (int)N, L, ms[mi], ts, 0);
    }
    __syncthreads();
    // ---- pass 2: screened histogram over [t_s, key max]
    for (uint32_t i = threadIdx.x; i < NM * kHB; i += blockDim.x) hist[i] = 0u;
    if (threadIdx.x < NM) {
      uint32_t m = ms[0];
#pragma unroll
      for (int i = 1; i < NM; ++i) m = threadIdx.x == (unsigned)i ? ms[i] : m;
      const double hi = m == 1u ? La : (m == 2u ? 0.0 : 1.0);
      const double lo = tl_s[threadIdx.x] == kNegInf ? lo_s[threadIdx.x] : tl_s[threadIdx.x];
      lo_s[threadIdx.x] = lo;
      sc_s[threadIdx.x] = (hi > lo && hi - lo < 1e300) ? (double)kHB / (hi - lo) : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < NM) scnt[threadIdx.x] = 0;
    __syncthreads();
    PHASE(6);
    screened(prow, r, [&](uint64_t c, uint32_t mi, double key) {
      PABT_ADD(2, 1);
      atomicAdd(hist + mi * kHB + bucket(mi, key), 1u);
      const uint32_t pos = atomicAdd(&scnt[mi], 1u);   // keep it for pass 3 (this block's slot)
      if (pos < kPab3Keep) {
        skey[((size_t)blockIdx.x * NM + mi) * kPab3Keep + pos] = key;
        sidx[((size_t)blockIdx.x * NM + mi) * kPab3Keep + pos] = (int)c;
      }
    });
    __syncthreads();
    PHASE(7);
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) {
      const double t0 = edge(mi, select(hist + mi * kHB));
      const bool raise = t0 > tl_s[mi];
      __syncthreads();
      if (threadIdx.x == 0 && raise) tl_s[mi] = t0;
      if (raise)
        for (int pb = pdlo + (int)threadIdx.x; pb <= pdhi; pb += (int)blockDim.x)
          T[pb * NMP + mi] = min_pab(pa, pb, (int)N, L, ms[mi], t0, (int)T[pb * NMP + mi]);
    }
    if (threadIdx.x < NM) { cnt[threadIdx.x] = 0; tk[threadIdx.x] = kNegInf; ti[threadIdx.x] = kSentinelIdx; }
    if (threadIdx.x == 0) ovf = 0;
    __syncthreads();   // (the buffers alias the histograms: every select is done)
    PHASE(8);
    // ---- pass 3: collect the survivors of the raised screen — from the pass-2 survivors kept
    // in this block's scratch slot (key >= t0 <=> pab >= T[pb]), or by re-walking the row
    // when more survived pass 2 than the slot holds
    bool kept = true;
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) kept = kept && scnt[mi] <= kPab3Keep;
    if (kept) {
#pragma unroll
      for (int mi = 0; mi < NM; ++mi) {
        const double t0 = tl_s[mi];
        const double* sk = skey + ((size_t)blockIdx.x * NM + mi) * kPab3Keep;
        const int* si = sidx + ((size_t)blockIdx.x * NM + mi) * kPab3Keep;
        for (uint32_t i = threadIdx.x; i < scnt[mi]; i += blockDim.x) {
          const double key = sk[i];
          if (key >= t0) collect((uint64_t)si[i], mi, key);
        }
      }
    } else {
      screened(prow, r, collect);
    }
    __syncthreads();
    PHASE(9);
    if (ovf) {   // (uniform) rare: restart the pass in barrier-separated steps
      PABT_ADD(4, threadIdx.x == 0);
      if (threadIdx.x < NM) { cnt[threadIdx.x] = 0; tk[threadIdx.x] = kNegInf; ti[threadIdx.x] = kSentinelIdx; }
      __syncthreads();
      for (uint64_t c = 0; c < ndb; c += kPab3Slow) {
        const uint64_t cc = c + threadIdx.x;
        if (cc < ndb && !((flags & 1u) && cc == r)) {
          const int v = __ldcs(prow + cc), b = __ldg(pd + cc);
#pragma unroll
          for (int mi = 0; mi < NM; ++mi)
            if (v >= (int)T[b * NMP + mi]) collect(cc, mi, pab_key(pa, b, v, (int)N, L, ms[mi]));
        }
        __syncthreads();
#pragma unroll
        for (int mi = 0; mi < NM; ++mi) {
          const uint32_t n = cnt[mi];
          if (n > (uint32_t)kPab3Cap - kPab3Slow) flush(mi, n, pa);
        }
      }
    }
    // final ranking: warp mi sorts measure mi's buffer (no block barriers) and writes its head
    if (warp < NM) {
      const int mi = warp;
      uint32_t m = ms[0];
#pragma unroll
      for (int i = 1; i < NM; ++i) m = mi == i ? ms[i] : m;
      double* key = bkey + mi * kPab3Cap;
      int* idx = bidx + mi * kPab3Cap;
      const uint32_t n = min(cnt[mi], (uint32_t)kPab3Cap);
      uint32_t P = 32;
      while (P < n) P <<= 1;
      for (uint32_t i = n + lane; i < P; i += 32) { key[i] = kNegInf; idx[i] = kSentinelIdx; }
      __syncwarp();
      warp_bitonic_sort(key, idx, (int)P);
      for (uint32_t q = lane; q < k; q += 32) {
        const bool valid = q < n && idx[q] != kSentinelIdx;
        const size_t o = (size_t)mi * nq * k + r * k + q;
        out_idx[o] = valid ? idx[q] : -1;
        out_score[o] = valid ? key_to_score(key[q], m) : __int_as_float(0x7fc00000);
      }
    }
    PABT_ADD(0, threadIdx.x == 0);
    __syncthreads();
    PHASE(10);
  }
}
#undef PHASE

#ifdef BSK_PABT_STATS
}  // namespace bsk
extern "C" void bsk_pabt_stats(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, bsk::g_pabt, sizeof(bsk::g_pabt));
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(bsk::g_pabt, z, sizeof(z));
}
namespace bsk {
#endif

cudaError_t launch_int_range(const int32_t* x, uint64_t n, int32_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(out, 0x7f, 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(out + 1, 0x80, 4, s);
  if (e != cudaSuccess) return e;
  int_range_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms()), 256, 0, s>>>(x, n, out);
  count_launch();
  return cudaGetLastError();
}

static size_t topk_pab3_smem(uint32_t N, uint32_t nm) {
  const size_t h = std::max<size_t>((size_t)nm * kHB * 4, (size_t)nm * kPab3Cap * 12);
  return h + (((size_t)(nm == 3 ? 4 : nm) * (N + 1) * 2 + 15) & ~(size_t)15) +
         (size_t)8 * (32 + 128 * nm) * 8 + (size_t)kRing * 256 * 16;
}

size_t topk_pab3_scratch_bytes(uint32_t mask) {
  return (size_t)kPab3Slots * (size_t)__builtin_popcount(mask & 15u) * kPab3Keep * 12;
}

bool topk_pab3_fits(uint32_t N, uint32_t mask, uint32_t k) {
  const uint32_t nm = (uint32_t)__builtin_popcount(mask & 15u);
  return nm >= 1 && N <= 16383 && k >= 1 && k <= (uint32_t)kPab3Cap - kPab3Slow &&
         topk_pab3_smem(N, nm) <= (size_t)227 * 1024;
}

template <int NM>
static cudaError_t launch_topk_pab3_t(const int32_t* pab, uint64_t nq, uint64_t ndb, uint32_t N, uint32_t mask,
                                      uint32_t k, uint32_t flags, const int32_t* pq, const int32_t* pd, const double* L,
                                      int32_t* pd_range, unsigned char* scratch, int32_t* out_idx, float* out_score,
                                      cudaStream_t s) {
  const size_t smem = topk_pab3_smem(N, NM);
  cudaError_t e = cudaFuncSetAttribute(topk_pab3_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int bps = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, topk_pab3_kernel<NM>, 256, smem) != cudaSuccess || bps < 1)
    bps = 1;
  const uint64_t grid = std::min<uint64_t>({nq, (uint64_t)num_sms() * (uint64_t)bps, (uint64_t)kPab3Slots});
  double* skey = reinterpret_cast<double*>(scratch);
  int32_t* sidx = reinterpret_cast<int32_t*>(scratch + (size_t)kPab3Slots * NM * kPab3Keep * 8);
  topk_pab3_kernel<NM><<<(unsigned)grid, 256, smem, s>>>(pab, nq, ndb, N, mask, k, flags, pq, pd, L, pd_range, skey,
                                                         sidx, out_idx, out_score);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_topk_pab3(const int32_t* pab, uint64_t nq, uint64_t ndb, uint32_t N, uint32_t mask, uint32_t k,
                             uint32_t flags, const int32_t* pq, const int32_t* pd, const double* L, int32_t* pd_range,
                             void* scratch_v, int32_t* out_idx, float* out_score, cudaStream_t s) {
  if (nq == 0 || k == 0 || ndb == 0) return cudaSuccess;
  unsigned char* scratch = static_cast<unsigned char*>(scratch_v);
  cudaError_t e = cudaMemsetAsync(pd_range, 0x7f, 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(pd_range + 1, 0x80, 4, s);
  if (e != cudaSuccess) return e;
  int_range_kernel<<<(unsigned)std::min<uint64_t>((ndb + 255) / 256, (uint64_t)num_sms()), 256, 0, s>>>(pd, ndb,
                                                                                                        pd_range);
  count_launch();
  mask &= 15u;
  switch (__builtin_popcount(mask)) {
    case 1: return launch_topk_pab3_t<1>(pab, nq, ndb, N, mask, k, flags, pq, pd, L, pd_range, scratch, out_idx, out_score, s);
    case 2: return launch_topk_pab3_t<2>(pab, nq, ndb, N, mask, k, flags, pq, pd, L, pd_range, scratch, out_idx, out_score, s);
    case 3: return launch_topk_pab3_t<3>(pab, nq, ndb, N, mask, k, flags, pq, pd, L, pd_range, scratch, out_idx, out_score, s);
    default: return launch_topk_pab3_t<4>(pab, nq, ndb, N, mask, k, flags, pq, pd, L, pd_range, scratch, out_idx, out_score, s);
  }
}

// ------------------------------------- fused screen: thresholds + survivor lists (K4d) --
// Shared pieces of the two kernels around the tensor-core screen (tc.cu kTcScreen).
struct ListHist {   // kHB-bucket histogram of keys over [lo, lo + kHB / sc)
  __device__ static int bucket(double key, double lo, double sc) {
    const double x = (key - lo) * sc;
    return x <= 0.0 ? 0 : (x >= (double)(kHB - 1) ? kHB - 1 : (int)x);
  }
  // a lower bound of the k-th key from a selected bucket h (> 0): its lower edge less a margin
  __device__ static double edge(int h, double lo, double sc) {
    if (h <= 0 || !(sc > 0.0)) return -__longlong_as_double(0x7ff0000000000000LL);
    const double e = lo + (double)h / sc;
    return e - 1e-12 * fmax(1.0, fmax(fabs(e), fabs(lo)));
  }
};

// The recipe's IP part (estimate_pair's exact fp64 operations) and, from it, every key: IP and -HAM
// exactly, JS and COS within kApproxEps (fp32 quotient of the recipe's fp64 operands: fast
// division / reciprocal square root, keys in [0, 1]). Used only to set thresholds and to skip
// pairs that cannot reach one (with the margin); every ranked key is the exact one.
constexpr double kApproxEps = 4e-6;
__device__ __forceinline__ double approx_key(int pa, int pb, int pab, int N, const double* __restrict__ L, uint32_t m) {
  const int pu = pa + pb - pab;
  const double La = L[pa], Lb = L[pb];
  const double S = __dadd_rn(La, Lb);
  double ip = 0.0;
  if (!(pu == N && pa < N && pb < N)) {
    const double raw = __dsub_rn(S, L[pu]);
    const double lo = raw > 0.0 ? raw : 0.0;
    const double cap = La < Lb ? La : Lb;
    ip = lo < cap ? lo : cap;
  }
  if (m == 1u) return ip;
  if (m == 2u) {
    double h = __dsub_rn(S, __dmul_rn(2.0, ip));
    h = h > 0.0 ? h : 0.0;
    return -(h < S ? h : S);
  }
  float v;
  if (m == 4u) v = (pa == 0 && pb == 0) ? 1.0f : __fdividef((float)ip, (float)__dsub_rn(S, ip));
  else v = (pa == 0 || pb == 0) ? 0.0f : (float)ip * rsqrtf((float)La * (float)Lb);
  return (double)fminf(fmaxf(v, 0.0f), 1.0f);
}
__device__ __forceinline__ double approx_eps(uint32_t m) { return m >= 4u ? kApproxEps : 0.0; }

// Highest bucket h with >= k counts in buckets >= h, or -1 (block-wide, 256 threads; thread t owns
// buckets [kHB - 8(t+1), kHB - 8t), scanned from the top). warp_sum: 8 words, found: 1 word.
__device__ int block_select_bucket(const uint32_t* hm, uint32_t k, uint32_t* warp_sum, int* found) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int top = kHB - 8 * (int)threadIdx.x;
  uint32_t loc = 0;
#pragma unroll
  for (int j = 1; j <= 8; ++j) loc += hm[top - j];
  uint32_t inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
  if (lane == 31) warp_sum[warp] = inc;
  if (threadIdx.x == 0) *found = -1;
  __syncthreads();
  uint32_t before_w = 0;
  for (int w = 0; w < warp; ++w) before_w += warp_sum[w];
  const uint32_t excl = before_w + inc - loc;
  if (excl < k && excl + loc >= k) {
    uint32_t run = excl;
    for (int j = 1; j <= 8; ++j) {
      run += hm[top - j];
      if (run >= k) { *found = top - j; break; }
    }
  }
  __syncthreads();
  const int h = *found;
  __syncthreads();
  return h;
}

// Per query row (one block, grid-stride): exact keys of the sample pab row [S] (the first S db
// rows) into a kHB-bucket histogram over each measure's key range; t_s = the lower edge of the
// highest bucket with >= k sample pairs at or above it (as K4c pass 1: >= k pairs of the row reach
// it, so it is a lower bound of the row's k-th key); the minimum-pab table
// T_{t_s}[pb] over the db's popcount range, then its suffix minimum Tsuf[pb] = min_{pb' >= pb}
// T[pb'] (a tile of the popcount-sorted db with smallest |b_s| = lo holds no pair with
// pab < Tsuf[lo] whose key reaches t_s) -> tsuf[row][pb][NMP], ts[measure][row].
template <int NM>
__global__ void __launch_bounds__(256)
screen_threshold_kernel(const int32_t* __restrict__ pab_s, uint64_t nq, uint32_t S, uint32_t N, uint32_t mask,
                        uint32_t k, uint32_t flags, const int32_t* __restrict__ pq, const int32_t* __restrict__ pd,
                        const double* __restrict__ L, const int32_t* __restrict__ pdr, uint16_t* __restrict__ tsuf,
                        double* __restrict__ ts) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NMP = NM == 3 ? 4 : NM;
  uint32_t ms[NM];
  {
    uint32_t mm = mask;
#pragma unroll
    for (int i = 0; i < NM; ++i) { ms[i] = mm & (0u - mm); mm &= mm - 1; }
  }
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);                          // [NM][kHB]
  uint16_t* T = reinterpret_cast<uint16_t*>(smem + (size_t)NM * kHB * 4);       // [range][NM]
  __shared__ uint32_t warp_sum[8];
  __shared__ int found;
  __shared__ double lo_s[NM], sc_s[NM], t_s[NM];
  __shared__ uint32_t wmin[NM][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pdlo = pdr[0], pdhi = pdr[1];
  const int R = pdhi - pdlo + 1;
  const double kNegInf = -__longlong_as_double(0x7ff0000000000000LL);
  for (uint64_t r = blockIdx.x; r < nq; r += gridDim.x) {
    const int pa = pq[r];
    const double La = L[pa];
    const double Lbmax = fmax(L[pdhi], L[pdhi < (int)N ? pdhi : (int)N - 1]);
#ifdef BSK_PABT_STATS
    long long tq = clock64();
#define TPH(i) do { if (threadIdx.x == 0) { const long long t_ = clock64(); PABT_ADD(i, t_ - tq); tq = t_; } } while (0)
#else
#define TPH(i) ((void)0)
#endif
    for (uint32_t i = threadIdx.x; i < NM * kHB; i += blockDim.x) hist[i] = 0u;
    if (threadIdx.x < NM) {
      uint32_t m = ms[0];
#pragma unroll
      for (int i = 1; i < NM; ++i) m = threadIdx.x == (unsigned)i ? ms[i] : m;
      const double lo = m == 2u ? -(La + Lbmax) : 0.0;
      const double hi = m == 1u ? La : (m == 2u ? 0.0 : 1.0);
      lo_s[threadIdx.x] = lo;
      sc_s[threadIdx.x] = (hi > lo && hi - lo < 1e300) ? (double)kHB / (hi - lo) : 0.0;
    }
    __syncthreads();
    const int32_t* row = pab_s + r * S;
    // four columns per thread and step, loads and key evaluations independent (ILP), then the
    // histogram updates
    for (uint32_t c0 = threadIdx.x; c0 < S; c0 += 4 * blockDim.x) {
      int v[4], pb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t c = c0 + u * blockDim.x;
        v[u] = c < S ? __ldcs(row + c) : 0;
        pb[u] = c < S ? __ldg(pd + c) : 0;   // the sample: db rows [0, S) in their own order
      }
      int bk[4][NM];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int mi = 0; mi < NM; ++mi)
          bk[u][mi] = ListHist::bucket(approx_key(pa, pb[u], v[u], (int)N, L, ms[mi]), lo_s[mi], sc_s[mi]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t c = c0 + u * blockDim.x;
        if (c < S && !((flags & 1u) && c == r))
#pragma unroll
          for (int mi = 0; mi < NM; ++mi) atomicAdd(hist + mi * kHB + bk[u][mi], 1u);
      }
    }
    __syncthreads();
    TPH(10);
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) {
      const double t = ListHist::edge(block_select_bucket(hist + mi * kHB, k, warp_sum, &found), lo_s[mi], sc_s[mi]);
      if (threadIdx.x == 0) t_s[mi] = t - approx_eps(ms[mi]);   // (the histogram holds approximate keys)
    }
    __syncthreads();
    TPH(11);
    // T over the popcount range, then its suffix minimum: thread t owns the contiguous chunk
    // [t * per, (t+1) * per); chunk minima combined by a reverse scan across the block
    for (int i = threadIdx.x; i < R; i += blockDim.x)
#pragma unroll
      for (int mi = 0; mi < NM; ++mi)
        T[i * NM + mi] = t_s[mi] == kNegInf ? (uint16_t)0 : min_pab(pa, pdlo + i, (int)N, L, ms[mi], t_s[mi], 0);
    __syncthreads();
    TPH(12);
    const int per = (R + (int)blockDim.x - 1) / (int)blockDim.x;
    const int c0 = (int)threadIdx.x * per, c1 = min(R, c0 + per);
    uint32_t later[NM];   // min over the chunks after this thread's
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) {
      uint32_t mn = 0xFFFFu;
      for (int i = c1 - 1; i >= c0; --i) mn = min(mn, (uint32_t)T[i * NM + mi]);
      uint32_t x = mn;   // inclusive suffix minimum within the warp
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_down_sync(0xffffffffu, x, o); if (lane + o < 32) x = min(x, y); }
      if (lane == 0) wmin[mi][warp] = x;
      const uint32_t nxt = __shfl_down_sync(0xffffffffu, x, 1);
      later[mi] = lane < 31 ? nxt : 0xFFFFu;
    }
    __syncthreads();
#pragma unroll
    for (int mi = 0; mi < NM; ++mi)
      for (int w = warp + 1; w < 8; ++w) later[mi] = min(later[mi], wmin[mi][w]);
    uint16_t* out = tsuf + (size_t)r * (N + 1) * NMP;
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) {
      uint32_t run = later[mi];
      for (int i = c1 - 1; i >= c0; --i) {
        run = min(run, (uint32_t)T[i * NM + mi]);
        out[(size_t)(pdlo + i) * NMP + mi] = (uint16_t)run;
      }
    }
    if (threadIdx.x < NM) ts[(size_t)threadIdx.x * nq + r] = t_s[threadIdx.x];
    if (NMP > NM)   // (NM = 3: the fourth entry never screens anything out)
      for (int i = threadIdx.x; i < R; i += blockDim.x) out[(size_t)(pdlo + i) * NMP + 3] = 0xFFFFu;
    __syncthreads();
    TPH(13);
  }
}
#undef TPH

size_t screen_threshold_smem(uint32_t N, uint32_t nm, uint32_t S) {
  (void)S;
  return (size_t)nm * kHB * 4 + (size_t)(N + 1) * nm * 2;
}

cudaError_t launch_screen_threshold(const int32_t* pab_s, uint64_t nq, uint32_t S, uint32_t N, uint32_t mask,
                                    uint32_t k, uint32_t flags, const int32_t* pq, const int32_t* pd, const double* L,
                                    const int32_t* pd_range, uint16_t* tsuf, double* ts, cudaStream_t s) {
  if (nq == 0) return cudaSuccess;
  const uint32_t nm = (uint32_t)__builtin_popcount(mask & 15u);
  const size_t smem = screen_threshold_smem(N, nm, S);
  const unsigned grid = (unsigned)std::min<uint64_t>(nq, (uint64_t)num_sms() * 8);
  cudaError_t e = cudaSuccess;
#define BSK_SCREEN_T(NMV)                                                                                       \
  do {                                                                                                          \
    e = cudaFuncSetAttribute(screen_threshold_kernel<NMV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                             \
    screen_threshold_kernel<NMV><<<grid, 256, smem, s>>>(pab_s, nq, S, N, mask & 15u, k, flags, pq, pd, L,    \
                                                         pd_range, tsuf, ts);                                   \
  } while (0)
  switch (nm) {
    case 1: BSK_SCREEN_T(1); break;
    case 2: BSK_SCREEN_T(2); break;
    case 3: BSK_SCREEN_T(3); break;
    default: BSK_SCREEN_T(4); break;
  }
#undef BSK_SCREEN_T
  count_launch();
  return cudaGetLastError();
}

// Per query row (one block, grid-stride): its screen survivors (original db index, |b_s| << 14 |
// pab) from the tensor-core screen, ranked exactly for every measure. Pass A: each thread walks a
// contiguous run of the row's list (its segments seen as one index range), four entries at a time
// with their loads issued together; approximate keys (approx_key: IP / -HAM exact, JS / COS within
// kApproxEps) of the pairs that may reach t_s go into a histogram over [t_s, key max] and, as
// (approximate key, |b_s|:pab, index) records, into the block's scratch slot; t0 = the histogram's
// lower bound of the k-th key less the margin. Pass B: the records that may reach t0 get their
// EXACT key (fp64 recipe); those that beat the running k-th go to a 512-entry buffer, ranked at the
// end by counting (the order is strict). A slot overflow makes pass B re-score the list exactly; a
// buffer overflow restarts pass B in 256-entry steps with a barrier each, cutting back to k.
template <int NM>
__global__ void __launch_bounds__(256, 4)
topk_list_kernel(const uint2* __restrict__ lists, const uint32_t* __restrict__ lcnt, uint32_t splits,
                 uint32_t seg_cols, uint64_t nq, uint64_t ndb,
                 uint32_t N, uint32_t mask, uint32_t k, uint32_t flags, const int32_t* __restrict__ pq,
                 const double* __restrict__ L,
                 const double* __restrict__ ts, double* __restrict__ skey, int32_t* __restrict__ sidx,
                 int32_t* __restrict__ out_idx, float* __restrict__ out_score) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t ms[NM];
  {
    uint32_t mm = mask;
#pragma unroll
    for (int i = 0; i < NM; ++i) { ms[i] = mm & (0u - mm); mm &= mm - 1; }
  }
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);                        // [NM][kHB] (pass A)
  double* bkey = reinterpret_cast<double*>(smem);                            // [NM][kPab3Cap] (pass B)
  int* bidx = reinterpret_cast<int*>(smem + (size_t)NM * kPab3Cap * 8);
  const size_t hb = (size_t)NM * kHB * 4 > (size_t)NM * kPab3Cap * 12 ? (size_t)NM * kHB * 4 : (size_t)NM * kPab3Cap * 12;
  uint32_t* segp = reinterpret_cast<uint32_t*>(smem + hb);                   // [splits + 1]
  __shared__ uint32_t cnt[NM], kcnt[NM];
  __shared__ double tk[NM];
  __shared__ int ti[NM];
  __shared__ double lo_s[NM], sc_s[NM], tl_s[NM];
  __shared__ uint32_t warp_sum[8];
  __shared__ int found;
  __shared__ int ovf;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double kNegInf = -__longlong_as_double(0x7ff0000000000000LL);
  double* sk = skey + (size_t)blockIdx.x * NM * kPab3Keep;                   // this block's slot
  int32_t* si = sidx + (size_t)blockIdx.x * NM * kPab3Keep;
  for (uint64_t r = blockIdx.x; r < nq; r += gridDim.x) {
    const int pa = pq[r];
    const double La = L[pa];
    const uint2* lst = lists + r * ndb;
    const uint32_t* cnts = lcnt + r * splits;
    // the row's list segments (segment sp: up to seg_cols entries from sp * seg_cols) as one flat
    // index range: exclusive prefix sums of the segment counts in shared memory (warp 0)
    __syncthreads();
    if (warp == 0) {
      uint32_t run = 0;
      for (uint32_t b = 0; b < splits; b += 32) {
        const uint32_t x = b + lane < splits ? cnts[b + lane] : 0u;
        uint32_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
        if (b + lane < splits) segp[b + lane] = run + inc - x;
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) segp[splits] = run;
    }
    if (threadIdx.x < NM) {
      uint32_t m = ms[0];
#pragma unroll
      for (int i = 1; i < NM; ++i) m = threadIdx.x == (unsigned)i ? ms[i] : m;
      const double t = ts[(size_t)threadIdx.x * nq + r];
      const double hi = m == 1u ? La : (m == 2u ? 0.0 : 1.0);
      // (keys below lo land in bucket 0, which never yields a bound: any lo is safe)
      const double lo = t != kNegInf ? t : (m == 2u ? -(La + fmax(L[N], L[N - 1])) : 0.0);
      tl_s[threadIdx.x] = t;
      lo_s[threadIdx.x] = lo;
      sc_s[threadIdx.x] = (hi > lo && hi - lo < 1e300) ? (double)kHB / (hi - lo) : 0.0;
      kcnt[threadIdx.x] = 0;
    }
    for (uint32_t i = threadIdx.x; i < NM * kHB; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const uint32_t total = segp[splits];
#ifdef BSK_PABT_STATS
    long long tq = clock64();
    if (threadIdx.x == 0) { PABT_ADD(0, 1); PABT_ADD(1, total); }
#define LPH(i) do { if (threadIdx.x == 0) { const long long t_ = clock64(); PABT_ADD(i, t_ - tq); tq = t_; } } while (0)
#else
#define LPH(i) ((void)0)
#endif
    // thread t's run [t * per_t, ...): locate its first segment once, then step through
    const uint32_t per_t = (total + blockDim.x - 1) / blockDim.x;
    const uint32_t i0 = min(total, threadIdx.x * per_t), i1 = min(total, i0 + per_t);
    auto run_entries = [&](auto&& f) {   // f(orig, pb, pab) per entry of the run, 4 loads in flight
      if (i0 >= i1) return;
      uint32_t lo = 0, hi = splits;      // segp[lo] <= i0 < segp[hi]
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (segp[mid] <= i0) lo = mid;
        else hi = mid;
      }
      uint32_t sp = lo, off = i0 - segp[lo];
      for (uint32_t i = i0; i < i1; i += 4) {
        uint2 e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          e[u] = make_uint2(0u, 0xFFFFFFFFu);
          if (i + u < i1) {
            while (segp[sp] + off >= segp[sp + 1]) { ++sp; off = 0; }
            e[u] = lst[(size_t)sp * seg_cols + off];
            ++off;
          }
        }
        int orig[4], pb[4], v[4];   // entry: (original db index, |b_s| << 14 | pab)
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          orig[u] = (int)e[u].x;
          pb[u] = (int)(e[u].y >> 14) & 0x3FFF;
          v[u] = (int)(e[u].y & 0x3FFFu);
          ok[u] = e[u].y != 0xFFFFFFFFu && !((flags & 1u) && (uint64_t)orig[u] == r);
        }
        f(ok, orig, pb, v);
      }
    };
    // pass A on approximate keys (approx_key: IP / -HAM exact, JS / COS within kApproxEps): the
    // histogram and the kept records (approximate key, pb:pab, db index) of pairs that may reach t_s
    run_entries([&](const bool (&ok)[4], const int (&orig)[4], const int (&pb)[4], const int (&v)[4]) {
      double key[4][NM];   // all keys of the batch first (independent chains), then the updates
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int mi = 0; mi < NM; ++mi) key[u][mi] = approx_key(pa, pb[u], v[u], (int)N, L, ms[mi]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int mi = 0; mi < NM; ++mi) {
          if (key[u][mi] < tl_s[mi] - approx_eps(ms[mi])) continue;
          atomicAdd(hist + mi * kHB + ListHist::bucket(key[u][mi], lo_s[mi], sc_s[mi]), 1u);
          const uint32_t pos = atomicAdd(&kcnt[mi], 1u);
          if (pos < kPab3Keep) {
            uint32_t* rec = reinterpret_cast<uint32_t*>(sk + (size_t)mi * kPab3Keep + pos);
            rec[0] = __float_as_uint(__double2float_rd(key[u][mi]));   // (rounded down: still <= the key + eps)
            rec[1] = ((uint32_t)pb[u] << 14) | (uint32_t)v[u];       // (pb, pab <= N <= 16383)
            si[(size_t)mi * kPab3Keep + pos] = orig[u];
          }
        }
      }
    });
    __syncthreads();
    LPH(5);
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) {
      const double t0 = ListHist::edge(block_select_bucket(hist + mi * kHB, k, warp_sum, &found), lo_s[mi], sc_s[mi]) -
                        approx_eps(ms[mi]);   // (the histogram holds approximate keys)
      if (threadIdx.x == 0 && t0 > tl_s[mi]) tl_s[mi] = t0;
    }
    if (threadIdx.x < NM) { cnt[threadIdx.x] = 0; tk[threadIdx.x] = kNegInf; ti[threadIdx.x] = kSentinelIdx; }
    if (threadIdx.x == 0) ovf = 0;
    __syncthreads();   // (the buffers alias the histograms)
    LPH(6);
    auto collect = [&](int mi, int orig, double key) {
      if (key < tl_s[mi] || !before(key, orig, tk[mi], ti[mi])) return;
      const uint32_t pos = atomicAdd(&cnt[mi], 1u);
      if (pos < (uint32_t)kPab3Cap) {
        bkey[mi * kPab3Cap + pos] = key;
        bidx[mi * kPab3Cap + pos] = orig;
      } else {
        ovf = 1;
      }
    };
    auto collect_all = [&](int orig, int pb, int v) {
#pragma unroll
      for (int mi = 0; mi < NM; ++mi) collect(mi, orig, pab_key(pa, pb, v, (int)N, L, ms[mi]));
    };
    auto collect_batch = [&](const bool (&ok)[4], const int (&orig)[4], const int (&pb)[4], const int (&v)[4]) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (ok[u]) collect_all(orig[u], pb[u], v[u]);
    };
    // sort measure mi's nb buffered candidates, keep the best k, raise (tk, ti) (block-wide)
    auto flush = [&](int mi, uint32_t nb) {
      double* key = bkey + mi * kPab3Cap;
      int* idx = bidx + mi * kPab3Cap;
      uint32_t P = 2;
      while (P < nb) P <<= 1;
      for (uint32_t i = nb + threadIdx.x; i < P; i += blockDim.x) { key[i] = kNegInf; idx[i] = kSentinelIdx; }
      __syncthreads();
      block_bitonic_sort(key, idx, (int)P);
      const bool full = nb >= k;
      const double nt = full ? key[k - 1] : kNegInf;
      const int nti = full ? idx[k - 1] : kSentinelIdx;
      __syncthreads();
      if (threadIdx.x == 0) { cnt[mi] = full ? k : nb; tk[mi] = nt; ti[mi] = nti; }
      __syncthreads();
    };
    bool kept = true;
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) kept = kept && kcnt[mi] <= kPab3Keep;
    if (kept) {
#pragma unroll
      for (int mi = 0; mi < NM; ++mi) {
        const uint2* recs = reinterpret_cast<const uint2*>(sk + (size_t)mi * kPab3Keep);
        const double tcut = tl_s[mi] - approx_eps(ms[mi]);
        const uint32_t nk = kcnt[mi];
        for (uint32_t i0 = threadIdx.x; i0 < nk; i0 += 4 * blockDim.x) {
          uint2 rc[4];   // four records' loads in flight
#pragma unroll
          for (int u = 0; u < 4; ++u) rc[u] = i0 + u * blockDim.x < nk ? recs[i0 + u * blockDim.x] : make_uint2(0xFF800000u, 0u);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t i = i0 + u * blockDim.x;
            if (i >= nk || (double)__uint_as_float(rc[u].x) < tcut) continue;   // (none) / cannot reach t0
            const int pb = (int)(rc[u].y >> 14), v = (int)(rc[u].y & 0x3FFFu);
            collect(mi, si[(size_t)mi * kPab3Keep + i], pab_key(pa, pb, v, (int)N, L, ms[mi]));   // the exact key
          }
        }
      }
    } else {
      run_entries(collect_batch);
    }
    __syncthreads();
    LPH(7);
    if (ovf) {   // (uniform) rare: restart pass B in barrier-separated steps over the list
      if (threadIdx.x < NM) { cnt[threadIdx.x] = 0; tk[threadIdx.x] = kNegInf; ti[threadIdx.x] = kSentinelIdx; }
      __syncthreads();
      for (uint32_t c = 0; c < total; c += kPab3Slow) {
        const uint32_t i = c + threadIdx.x;
        if (i < total) {
          uint32_t lo = 0, hi = splits;
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (segp[mid] <= i) lo = mid;
            else hi = mid;
          }
          const uint2 e = lst[(size_t)lo * seg_cols + (i - segp[lo])];
          const int orig = (int)e.x;
          if (!((flags & 1u) && (uint64_t)orig == r)) collect_all(orig, (int)(e.y >> 14) & 0x3FFF, (int)(e.y & 0x3FFFu));
        }
        __syncthreads();
#pragma unroll
        for (int mi = 0; mi < NM; ++mi) {
          const uint32_t nb = cnt[mi];
          if (nb > (uint32_t)kPab3Cap - kPab3Slow) flush(mi, nb);
        }
      }
    }
    LPH(8);
    // final ranking: every candidate's rank in the (key desc, index asc) order by counting (the
    // order is strict: indices are distinct), written straight to its output slot; threads
    // [mi * G, (mi + 1) * G) take measure mi
    {
      constexpr int NMP = NM == 3 ? 4 : NM;
      constexpr uint32_t G = 256 / NMP;
      const int mi = (int)(threadIdx.x / G);
      if (mi < NM) {
        uint32_t m = ms[0];
#pragma unroll
        for (int i = 1; i < NM; ++i) m = mi == i ? ms[i] : m;
        const double* key = bkey + mi * kPab3Cap;
        const int* idx = bidx + mi * kPab3Cap;
        const uint32_t nb = min(cnt[mi], (uint32_t)kPab3Cap);
        if (threadIdx.x % G == 0) PABT_ADD(3, nb);
        const size_t ob = (size_t)mi * nq * k + r * k;
        for (uint32_t c = threadIdx.x % G; c < nb; c += G) {
          const double kc = key[c];
          const int ic = idx[c];
          uint32_t rank = 0;
          for (uint32_t j = 0; j < nb; ++j) rank += before(key[j], idx[j], kc, ic) ? 1u : 0u;
          if (rank < k) { out_idx[ob + rank] = ic; out_score[ob + rank] = key_to_score(kc, m); }
        }
        for (uint32_t q = nb + threadIdx.x % G; q < k; q += G) { out_idx[ob + q] = -1; out_score[ob + q] = __int_as_float(0x7fc00000); }
      }
    }
    __syncthreads();
    LPH(9);
  }
}
#undef LPH

cudaError_t launch_topk_list(const uint2* lists, const uint32_t* lcnt, uint32_t splits, uint32_t seg_cols,
                             uint64_t nq, uint64_t ndb, uint32_t N,
                             uint32_t mask, uint32_t k, uint32_t flags, const int32_t* pq, const double* L,
                             const double* ts, void* scratch_v, int32_t* out_idx, float* out_score, cudaStream_t s) {
  unsigned char* scratch = static_cast<unsigned char*>(scratch_v);   // topk_pab3_scratch_bytes(15) (slots)
  if (nq == 0 || k == 0) return cudaSuccess;
  const uint32_t nm = (uint32_t)__builtin_popcount(mask & 15u);
  const size_t smem = std::max<size_t>((size_t)nm * kHB * 4, (size_t)nm * kPab3Cap * 12) + ((size_t)splits + 1) * 4;
  int bps = 0;
  cudaError_t e = cudaSuccess;
#define BSK_LIST_T(NMV)                                                                                          \
  do {                                                                                                           \
    e = cudaFuncSetAttribute(topk_list_kernel<NMV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    if (e != cudaSuccess) return e;                                                                              \
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, topk_list_kernel<NMV>, 256, smem) != cudaSuccess ||  \
        bps < 1)                                                                                                 \
      bps = 1;                                                                                                   \
    topk_list_kernel<NMV><<<(unsigned)std::min<uint64_t>({nq, (uint64_t)num_sms() * bps, (uint64_t)kPab3Slots}),  \
                            256, smem, s>>>(lists, lcnt, splits, seg_cols, nq, ndb, N, mask & 15u, k, flags, pq, L,   \
                                            ts, reinterpret_cast<double*>(scratch),                               \
                                            reinterpret_cast<int32_t*>(scratch + (size_t)kPab3Slots * NMV * kPab3Keep * 8), \
                                            out_idx, out_score);                                                  \
  } while (0)
  switch (nm) {
    case 1: BSK_LIST_T(1); break;
    case 2: BSK_LIST_T(2); break;
    case 3: BSK_LIST_T(3); break;
    default: BSK_LIST_T(4); break;
  }
#undef BSK_LIST_T
  count_launch();
  return cudaGetLastError();
}

// Top-k from a precomputed AND-popcount table pab[nq][ndb] (tensor cores): one warp per
// (query row, db split) streams its pab row (16-B loads, 128 columns per step), keeps a running
// threshold (its current k-th best), screens every pair with the division-free pre-test, scores
// the rest exactly and appends those that beat the threshold to a per-warp buffer, which is
// sorted (warp bitonic) and cut back to k when it could overflow. No block-level barriers.
template <int CAPW>
__global__ void __launch_bounds__(256)
topk_pab_kernel(const int32_t* __restrict__ pab, uint64_t nq, uint64_t ndb, uint32_t N, uint32_t measure, uint32_t k,
                uint32_t flags, const int32_t* __restrict__ pq, const int32_t* __restrict__ pd,
                const double* __restrict__ Lg, uint32_t splits, double* __restrict__ part_key,
                int32_t* __restrict__ part_idx, int32_t* __restrict__ out_idx, float* __restrict__ out_score) {
  extern __shared__ __align__(16) unsigned char smem[];
  const bool l_in_smem = N + 1 <= kMaxSmemL;
  const size_t lbytes = l_in_smem ? (((size_t)(N + 1) * 8 + 15) & ~(size_t)15) : 0;
  double* Ls = reinterpret_cast<double*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ckey = reinterpret_cast<double*>(smem + lbytes) + warp * CAPW;
  int* cidx = reinterpret_cast<int*>(smem + lbytes + (size_t)8 * CAPW * 8) + warp * CAPW;
  if (l_in_smem)
    for (uint32_t i = threadIdx.x; i <= N; i += blockDim.x) Ls[i] = Lg[i];
  __syncthreads();
  const double* L = l_in_smem ? Ls : Lg;
  const uint64_t gw = (uint64_t)blockIdx.x * 8 + warp;
  if (gw >= nq * splits) return;
  const uint64_t r = gw / splits;
  const uint32_t sp = (uint32_t)(gw - r * splits);
  const uint64_t per = ((ndb + splits - 1) / splits + 127) / 128 * 128;
  const uint64_t c_begin = min((uint64_t)sp * per, ndb), c_end = min(c_begin + per, ndb);
  const double kNegInf = -__longlong_as_double(0x7ff0000000000000LL);
  for (int i = lane; i < CAPW; i += 32) { ckey[i] = kNegInf; cidx[i] = kSentinelIdx; }
  __syncwarp();
  double t = kNegInf;
  int ti = kSentinelIdx;
  uint32_t cnt = 0;                                     // buffered candidates beyond the first k
  const int pa = pq[r];
  const int32_t* prow = pab + r * ndb;
  const bool vec = (ndb & 3u) == 0 && (reinterpret_cast<uintptr_t>(pab) & 15u) == 0 &&
                   (reinterpret_cast<uintptr_t>(pd) & 15u) == 0;
  auto flush = [&]() {
    warp_bitonic_sort(ckey, cidx, CAPW);
    for (int i = (int)k + lane; i < CAPW; i += 32) { ckey[i] = kNegInf; cidx[i] = kSentinelIdx; }
    __syncwarp();
    t = ckey[k - 1];
    ti = cidx[k - 1];
    cnt = 0;
  };
  for (uint64_t c0 = c_begin; c0 < c_end; c0 += 128) {
    const uint64_t cl = c0 + 4 * (uint64_t)lane;
    int v[4], b[4];
    if (vec && cl + 3 < c_end) {
      const int4 a4 = __ldcs(reinterpret_cast<const int4*>(prow + cl));
      const int4 p4 = __ldg(reinterpret_cast<const int4*>(pd + cl));
      v[0] = a4.x; v[1] = a4.y; v[2] = a4.z; v[3] = a4.w;
      b[0] = p4.x; b[1] = p4.y; b[2] = p4.z; b[3] = p4.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = cl + u < c_end ? __ldcs(prow + cl + u) : 0;
        b[u] = cl + u < c_end ? __ldg(pd + cl + u) : 0;
      }
    }
    double key[4];
    bool keep[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t c = cl + u;
      keep[u] = c < c_end && !((flags & 1u) && c == r);
      if (keep[u] && t > kNegInf) keep[u] = pretest_keep(pa, b[u], v[u], (int)N, L, measure, t);
      key[u] = kNegInf;
      if (keep[u]) {
        key[u] = measure_key(estimate_pair(pa, b[u], v[u], (int)N, L, measure), measure);
        keep[u] = before(key[u], (int)c, t, ti);
      }
    }
    const uint32_t mine = (keep[0] ? 1u : 0u) + (keep[1] ? 1u : 0u) + (keep[2] ? 1u : 0u) + (keep[3] ? 1u : 0u);
    uint32_t off = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, off, o); if (lane >= o) off += y; }
    const uint32_t total = __shfl_sync(0xffffffffu, off, 31);
    if (total == 0) continue;
    if (cnt + total > (uint32_t)CAPW - k) {
      flush();   // frees CAPW - k >= 128 slots; re-screen this step's picks against the new threshold
#pragma unroll
      for (int u = 0; u < 4; ++u) keep[u] = keep[u] && before(key[u], (int)(cl + u), t, ti);
      const uint32_t m2 = (keep[0] ? 1u : 0u) + (keep[1] ? 1u : 0u) + (keep[2] ? 1u : 0u) + (keep[3] ? 1u : 0u);
      off = m2;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, off, o); if (lane >= o) off += y; }
      const uint32_t tot2 = __shfl_sync(0xffffffffu, off, 31);
      off -= m2;
      uint32_t pos = k + cnt + off;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (keep[u]) { ckey[pos] = key[u]; cidx[pos] = (int)(cl + u); ++pos; }
      cnt += tot2;
    } else {
      off -= mine;
      uint32_t pos = k + cnt + off;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (keep[u]) { ckey[pos] = key[u]; cidx[pos] = (int)(cl + u); ++pos; }
      cnt += total;
    }
    __syncwarp();
  }
  if (cnt > 0 || t == kNegInf) flush();
  for (uint32_t q = lane; q < k; q += 32) {
    const double kq = ckey[q];
    const int id = cidx[q];
    if (splits == 1) {
      const bool valid = id != kSentinelIdx;
      out_idx[r * k + q] = valid ? id : -1;
      out_score[r * k + q] = valid ? key_to_score(kq, measure) : __int_as_float(0x7fc00000);
    } else {
      part_key[(r * splits + sp) * k + q] = kq;
      part_idx[(r * splits + sp) * k + q] = id;
    }
  }
}

template <int CAPW>
static cudaError_t launch_topk_pab_t(const int32_t* pab, uint64_t nq, uint64_t ndb, uint32_t N, uint32_t measure,
                                     uint32_t k, uint32_t flags, const int32_t* pq, const int32_t* pd, const double* L,
                                     uint32_t& splits, double* part_key, int32_t* part_idx, int32_t* out_idx,
                                     float* out_score, cudaStream_t s) {
  const bool l_in_smem = N + 1 <= kMaxSmemL;
  const size_t smem = (l_in_smem ? (((size_t)(N + 1) * 8 + 15) & ~(size_t)15) : 0) + (size_t)8 * CAPW * 12;
  cudaError_t e = cudaFuncSetAttribute(topk_pab_kernel<CAPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // db splits per query: as many as fit ONE wave of resident blocks (<= the workspace bound). A
  // warp's candidate-buffer sorts grow only like k ln(n/k) with its stream length n, so longer
  // streams cost fewer sorts in total, and a partial second wave costs a whole wave (Ranking,
  // 1000 queries: 10 splits 3.48 ms, 6: 2.99, 4: 3.14, 3: 2.35 (one wave), 2: 2.58, 1: 3.60)
  int bps = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, topk_pab_kernel<CAPW>, 256, smem) != cudaSuccess || bps < 1) bps = 1;
  const uint64_t wave_warps = (uint64_t)num_sms() * (uint64_t)bps * 8;
  splits = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(splits, wave_warps / nq));
  if (const char* ev = std::getenv("BINSKETCH_PAB_SPLITS")) splits = std::max(1u, std::min<uint32_t>(splits, (uint32_t)std::atoi(ev)));   // dev A/B
  const uint64_t warps = nq * splits;
  topk_pab_kernel<CAPW><<<(unsigned)((warps + 7) / 8), 256, smem, s>>>(pab, nq, ndb, N, measure, k, flags, pq, pd, L,
                                                                       splits, part_key, part_idx, out_idx, out_score);
  count_launch();
  return cudaGetLastError();
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
  uint32_t splits = topk_splits(nq, ndb, k);   // workspace bound; the pab path may use fewer
  cudaError_t e;
  if (pab) {
    e = k <= 128 ? launch_topk_pab_t<256>(pab, nq, ndb, N, measure, k, flags, pq, pd, L, splits, part_key, part_idx,
                                          out_idx, out_score, s)
                 : launch_topk_pab_t<512>(pab, nq, ndb, N, measure, k, flags, pq, pd, L, splits, part_key, part_idx,
                                          out_idx, out_score, s);
    if (e != cudaSuccess || splits == 1) return e;
    return launch_topk_merge(nq, splits, k, measure, part_key, part_idx, out_idx, out_score, s);
  }
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
  if (P <= 256) {
    const size_t smem = (size_t)8 * P * 12;
    cudaError_t e = cudaFuncSetAttribute(topk_merge_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    topk_merge_warp_kernel<<<(unsigned)((nq + 7) / 8), 256, smem, s>>>(nq, splits, k, P, measure, part_key, part_idx,
                                                                     out_idx, out_score);
    count_launch();
    return cudaGetLastError();
  }
  const size_t smem = (size_t)P * 12;
  cudaError_t e = cudaFuncSetAttribute(topk_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  topk_merge_kernel<<<(unsigned)nq, 256, smem, s>>>(nq, splits, k, P, measure, part_key, part_idx, out_idx, out_score);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsk
