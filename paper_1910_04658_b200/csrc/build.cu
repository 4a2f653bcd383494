// build.cu — pi generation (K5), sketch construction (K1) and row popcount (K2)
// for sm_100a.
//
// K1 computes the BinSketch definition
//     a_s[j] = OR_{i : pi(i) = j} a[i]
// for every CSR row in ONE streaming pass over the nonzeros (PAPER.md:349-352,
// "Hashing a vector a involves only looking at the non-zero bits"):
//   * a warp owns RW consecutive rows (a "row tile"); their nonzeros are one
//     contiguous span of `indices`, which the 32 lanes stream with coalesced,
//     evict-first loads (each nonzero is read exactly once);
//   * each lane tracks the row of its current nonzero by walking the tile's
//     indptr slice (staged in shared memory) forward — no search;
//   * pi(i) comes from (a) a shared-memory copy of the table when it fits
//     (uint16 when N <= 65536), (b) the read-only L1/L2 path otherwise, or
//     (c) in-kernel evaluation of the splitmix64 recipe (build_seeded);
//   * bits are OR-ed into the tile's sketch rows in shared memory with
//     shared atomics (ATOMS.OR), so every output word is written exactly once,
//     as contiguous (RW*W-word) coalesced 16-byte streaming stores.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "bsk_device.cuh"
#include "bsk_internal.cuh"

namespace bsk {

__device__ unsigned int g_status = 0u;

static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

unsigned int* status_ptr() {
  static unsigned int* p = nullptr;
  if (!p) {
    void* v = nullptr;
    if (cudaGetSymbolAddress(&v, g_status) == cudaSuccess) p = static_cast<unsigned int*>(v);
  }
  return p;
}

ModN make_modn(uint32_t N) {
  ModN m;
  m.N = N;
  m.M = (N > 1) ? (~0ULL) / (uint64_t)N : 0ULL;
  return m;
}

int num_sms() {
  int dev = 0, v = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v > 0 ? v : 148;
}

// ------------------------------------------------------------------ K5 ----
__global__ void make_pi_kernel(uint64_t seed, uint64_t d, ModN m, uint32_t* __restrict__ pi) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < d;
       i += (uint64_t)gridDim.x * blockDim.x)
    pi[i] = pi_seeded(seed, i, m);
}

cudaError_t launch_make_pi(uint64_t seed, uint64_t d, uint32_t N, uint32_t* pi, cudaStream_t s) {
  if (d == 0) return cudaSuccess;
  uint64_t blocks = std::min<uint64_t>((d + 255) / 256, (uint64_t)num_sms() * 8);
  make_pi_kernel<<<(unsigned)blocks, 256, 0, s>>>(seed, d, make_modn(N), pi);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K1 ----
enum PiMode { kPiGlobal = 0, kPiSmem16 = 1, kPiSmem32 = 2, kPiSeeded = 3 };

constexpr int kBuildThreads = 256;
constexpr int kBuildWarps = kBuildThreads / 32;
constexpr uint32_t kTileWords = 1024;     // RW * W <= 1024 words (4 KB) per warp

template <int MODE>
__global__ void __launch_bounds__(kBuildThreads)
build_kernel(const uint32_t* __restrict__ pi, uint64_t seed, uint64_t d, ModN mn,
             const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, uint64_t n,
             uint32_t* __restrict__ out, uint32_t W, uint32_t RW, unsigned int* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t N = mn.N;

  size_t pi_bytes = 0;
  if (MODE == kPiSmem16) pi_bytes = ((d * 2 + 15) / 16) * 16;
  if (MODE == kPiSmem32) pi_bytes = ((d * 4 + 15) / 16) * 16;
  // per-warp: indptr slice (RW+1 int64), then the RW x W sketch tile (16-B aligned)
  const size_t ip_bytes = (((size_t)(RW + 1) * 8 + 15) / 16) * 16;
  const size_t tile_bytes = (size_t)RW * W * 4;
  unsigned char* wbase = smem + pi_bytes + (size_t)warp * (ip_bytes + ((tile_bytes + 15) / 16) * 16);
  int64_t* ip_s = reinterpret_cast<int64_t*>(wbase);
  uint32_t* tile = reinterpret_cast<uint32_t*>(wbase + ip_bytes);

  unsigned bad_bits = 0;
  if (MODE == kPiSmem16 || MODE == kPiSmem32) {
    for (uint64_t i = threadIdx.x; i < d; i += blockDim.x) {
      uint32_t v = __ldg(pi + i);
      if (v >= N) { bad_bits = kStatusIndex; v = 0; }
      if (MODE == kPiSmem16) reinterpret_cast<uint16_t*>(smem)[i] = (uint16_t)v;
      else reinterpret_cast<uint32_t*>(smem)[i] = v;
    }
    __syncthreads();
  }

  const uint64_t ntiles = (n + RW - 1) / RW;
  for (uint64_t t = (uint64_t)blockIdx.x * kBuildWarps + warp; t < ntiles;
       t += (uint64_t)gridDim.x * kBuildWarps) {
    const uint64_t r0 = t * RW;
    const uint32_t rows = (uint32_t)((n - r0) < RW ? (n - r0) : RW);
    const uint32_t nw = rows * W;
    for (uint32_t i = lane; i <= rows; i += 32) ip_s[i] = __ldg(indptr + r0 + i);
    if ((nw & 3u) == 0) {
      uint4 z = make_uint4(0, 0, 0, 0);
      for (uint32_t w = lane * 4; w < nw; w += 128) *reinterpret_cast<uint4*>(tile + w) = z;
    } else {
      for (uint32_t w = lane; w < nw; w += 32) tile[w] = 0u;
    }
    __syncwarp();
    bool mono = true;
    for (uint32_t i = lane; i < rows; i += 32) mono &= ip_s[i + 1] >= ip_s[i];
    if (__all_sync(0xffffffffu, mono)) {
      const int64_t e1 = ip_s[rows];
      uint32_t cr = 0;
      for (int64_t e = ip_s[0] + lane; e < e1; e += 32) {
        while (e >= ip_s[cr + 1]) ++cr;
        const int32_t idx = __ldcs(indices + e);
        if ((uint64_t)(uint32_t)idx >= d || idx < 0) { bad_bits = kStatusIndex; continue; }
        uint32_t j;
        if (MODE == kPiGlobal) j = __ldg(pi + idx);
        else if (MODE == kPiSmem16) j = reinterpret_cast<const uint16_t*>(smem)[idx];
        else if (MODE == kPiSmem32) j = reinterpret_cast<const uint32_t*>(smem)[idx];
        else j = pi_seeded(seed, (uint64_t)idx, mn);
        if (MODE == kPiGlobal && j >= N) { bad_bits = kStatusIndex; continue; }
        atomicOr(tile + cr * W + (j >> 5), 1u << (j & 31u));
      }
    } else {
      bad_bits = kStatusIndex;  // decreasing indptr: rows of this tile stay zero
    }
    __syncwarp();
    uint32_t* dst = out + r0 * W;
    if ((nw & 3u) == 0 && ((r0 * W) & 3u) == 0) {
      for (uint32_t w = lane * 4; w < nw; w += 128)
        __stcs(reinterpret_cast<uint4*>(dst + w), *reinterpret_cast<const uint4*>(tile + w));
    } else {
      for (uint32_t w = lane; w < nw; w += 32) __stcs(dst + w, tile[w]);
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, bad_bits != 0) && lane == 0) latch(status, kStatusIndex);
}

// Fallback for very wide sketches (RW*W tile does not fit a warp's share of
// shared memory): rows zeroed by cudaMemsetAsync, then global atomicOr.
__global__ void build_wide_kernel(const uint32_t* __restrict__ pi, uint64_t seed, uint64_t d, ModN mn,
                                  bool seeded, const int64_t* __restrict__ indptr,
                                  const int32_t* __restrict__ indices, uint64_t n,
                                  uint32_t* __restrict__ out, uint32_t W, unsigned int* status) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned bad = 0;
  for (uint64_t r = gw; r < n; r += nwarps) {
    int64_t b = indptr[r], e = indptr[r + 1];
    if (e < b) { bad = kStatusIndex; continue; }
    for (int64_t t = b + lane; t < e; t += 32) {
      int32_t idx = indices[t];
      if (idx < 0 || (uint64_t)idx >= d) { bad = kStatusIndex; continue; }
      uint32_t j = seeded ? pi_seeded(seed, (uint64_t)idx, mn) : __ldg(pi + idx);
      if (j >= mn.N) { bad = kStatusIndex; continue; }
      atomicOr(out + r * W + (j >> 5), 1u << (j & 31u));
    }
  }
  if (bad) latch(status, bad);
}

cudaError_t launch_build(const uint32_t* pi, uint64_t seed, uint64_t d, uint32_t N,
                         const int64_t* indptr, const int32_t* indices, uint64_t n,
                         uint32_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint32_t W = (N + 31) / 32;
  const ModN mn = make_modn(N);
  unsigned int* st = status_ptr();
  const int sms = num_sms();
  int dev = 0, smem_optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);

  uint32_t RW = std::max<uint32_t>(1, std::min<uint32_t>(32, kTileWords / W));
  const size_t ip_bytes = (((size_t)(RW + 1) * 8 + 15) / 16) * 16;
  const size_t tile_bytes = (((size_t)RW * W * 4 + 15) / 16) * 16;
  const size_t per_cta = kBuildWarps * (ip_bytes + tile_bytes);
  if (per_cta > (size_t)smem_optin) {
    cudaError_t e = cudaMemsetAsync(out, 0, n * (size_t)W * 4, s);
    if (e != cudaSuccess) return e;
    build_wide_kernel<<<sms * 8, 256, 0, s>>>(pi, seed, d, mn, pi == nullptr, indptr, indices, n, out, W, st);
    count_launch();
    return cudaGetLastError();
  }
  const uint64_t ntiles = (n + RW - 1) / RW;
  const uint64_t want_blocks = (ntiles + kBuildWarps - 1) / kBuildWarps;

  int mode;
  size_t pi_bytes = 0;
  if (pi == nullptr) {
    mode = kPiSeeded;
  } else if (N <= 65536 && ((d * 2 + 15) / 16) * 16 + per_cta <= (size_t)smem_optin && d * 2 <= 160 * 1024 &&
             want_blocks >= (uint64_t)sms) {
    mode = kPiSmem16;
    pi_bytes = ((d * 2 + 15) / 16) * 16;
  } else {
    mode = kPiGlobal;
  }
  const size_t smem = pi_bytes + per_cta;
  uint64_t blocks;
  if (mode == kPiSmem16) {
    blocks = std::min<uint64_t>(want_blocks, (uint64_t)sms);  // persistent: table loaded once per CTA
  } else {
    int per_sm = std::max<int>(1, (int)std::min<size_t>(8, (size_t)(smem_optin) / std::max<size_t>(smem, 1)));
    blocks = std::min<uint64_t>(want_blocks, (uint64_t)sms * per_sm);
  }
  cudaError_t e = cudaSuccess;
#define BSK_LAUNCH_BUILD(M)                                                                            \
  do {                                                                                                 \
    e = cudaFuncSetAttribute(build_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                    \
    build_kernel<M><<<(unsigned)blocks, kBuildThreads, smem, s>>>(pi, seed, d, mn, indptr, indices, n, \
                                                                  out, W, RW, st);                    \
    count_launch();                                                                                    \
  } while (0)
  switch (mode) {
    case kPiSmem16: BSK_LAUNCH_BUILD(kPiSmem16); break;
    case kPiSeeded: BSK_LAUNCH_BUILD(kPiSeeded); break;
    default: BSK_LAUNCH_BUILD(kPiGlobal); break;
  }
#undef BSK_LAUNCH_BUILD
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K2 ----
// Algorithm 1 line 1: one warp per row, lanes over words.
__global__ void popcount_kernel(const uint32_t* __restrict__ sk, uint64_t n, uint32_t W,
                                int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = gw; r < n; r += nwarps) {
    const uint32_t* row = sk + r * W;
    int c = 0;
    for (uint32_t w = lane; w < W; w += 32) c += __popc(__ldg(row + w));
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) out[r] = c;
  }
}

cudaError_t launch_popcount(const uint32_t* sk, uint64_t n, uint32_t W, int32_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t blocks = std::min<uint64_t>((n * 32 + 255) / 256, (uint64_t)num_sms() * 16);
  popcount_kernel<<<(unsigned)blocks, 256, 0, s>>>(sk, n, W, out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsk
