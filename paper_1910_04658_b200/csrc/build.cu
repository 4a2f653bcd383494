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
#include <cstdlib>
#include <cstring>
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
  m.mask = (N > 1 && (N & (N - 1)) == 0) ? N - 1 : 0u;
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
enum PiMode { kPiGlobal = 0, kPiSmem16 = 1, kPiCache = 2, kPiSeeded = 3 };

constexpr uint32_t kTileWordsMax = 1024;     // RW * W <= 1024 words (4 KB) per warp
constexpr uint32_t kCacheSlots = 32768;      // shared-memory pi cache: 32K x 4 B = 128 KB
constexpr uint32_t kCacheEmpty = 0xFFFFFFFFu;

// 32-bit shared-memory accessors (keep shared addresses in one register; no generic
// address conversion per access).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or_shared(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// K1. Modes of obtaining pi(idx):
//  kPiGlobal: read-only L1/L2 gather.   kPiSmem16: whole table in shared memory (uint16).
//  kPiSeeded: splitmix64 evaluated in-kernel (no table).
//  kPiCache:  direct-mapped software cache in shared memory, slot = idx mod 32K holding
//             (idx >> 15) << 16 | pi(idx); a miss gathers from global and fills the slot.
//             Zipf-skewed features make most lookups hits; every (tag, value) ever written
//             is correct because pi is read-only, so races between lanes are benign.
// Per lane and iteration, 8 nonzeros (two 16-B quads) are looked up branch-free (all
// loads independent), then OR-ed into the warp's shared tile with RED.OR; the next two
// quads are already in flight. Invalid indices / pi values are clamped (so no access
// leaves its array) and latched as EINDEX.
template <int MODE>
__global__ void __launch_bounds__(1024)
build_kernel(const uint32_t* __restrict__ pi, uint64_t seed, uint64_t d, ModN mn,
             const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, uint64_t n,
             uint32_t* __restrict__ out, uint32_t W, uint32_t RW, size_t pi_bytes, unsigned int* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const uint32_t N = mn.N;
  const uint32_t d32 = (uint32_t)d;   // d <= 2^31 (checked on the host)

  // per-warp: indptr slice (RW+1 int64), window-relative int32 copy, then the RW x W tile
  const size_t ip_bytes = (((size_t)(RW + 1) * 12 + 15) / 16) * 16;
  const size_t tile_bytes = (((size_t)RW * W * 4 + 15) / 16) * 16;
  unsigned char* wbase = smem + pi_bytes + (size_t)warp * (ip_bytes + tile_bytes);
  int64_t* ip_s = reinterpret_cast<int64_t*>(wbase);
  const uint32_t rel_a = smem_u32(wbase + (size_t)(RW + 1) * 8);
  int* rel_p = reinterpret_cast<int*>(wbase + (size_t)(RW + 1) * 8);
  uint32_t* tile = reinterpret_cast<uint32_t*>(wbase + ip_bytes);
  const uint32_t tile_a = smem_u32(tile);
  const uint32_t pi_a = smem_u32(smem);

  unsigned bad_bits = 0;
  if (MODE == kPiSmem16) {
    for (uint64_t i = threadIdx.x; i < d; i += blockDim.x) {
      uint32_t v = __ldg(pi + i);
      if (v >= N) { bad_bits = kStatusIndex; v = 0; }
      reinterpret_cast<uint16_t*>(smem)[i] = (uint16_t)v;
    }
  }
  if (MODE == kPiCache) {
    for (uint32_t i = threadIdx.x; i < kCacheSlots; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = kCacheEmpty;
  }
  if (MODE == kPiSmem16 || MODE == kPiCache) __syncthreads();

  uint32_t max_idx = 0, max_j = 0;   // validity, checked once at the end
  const bool vec = (reinterpret_cast<uintptr_t>(indices) & 15u) == 0;
  const uint64_t ntiles = (n + RW - 1) / RW;
  for (uint64_t t = (uint64_t)blockIdx.x * nwarps + warp; t < ntiles; t += (uint64_t)gridDim.x * nwarps) {
    const uint64_t r0 = t * RW;
    const uint32_t rows = (uint32_t)((n - r0) < RW ? (n - r0) : RW);
    const uint32_t nw = rows * W;
    for (uint32_t i = lane; i <= rows; i += 32) ip_s[i] = __ldg(indptr + r0 + i);
    {
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (uint32_t w = lane * 4; w < nw; w += 128) *reinterpret_cast<uint4*>(tile + w) = z;  // tile_bytes padded
    }
    __syncwarp();
    bool ok = ip_s[0] >= 0;
    for (uint32_t i = lane; i < rows; i += 32) ok &= ip_s[i + 1] >= ip_s[i];
    if (__all_sync(0xffffffffu, ok)) {
      const int64_t e0 = ip_s[0], e1 = ip_s[rows];
      uint32_t cr = 0;
      // The tile's nonzeros [e0, e1) are walked in windows of 2^30 elements with 32-bit
      // window-relative offsets (one window unless a tile holds > 1e9 nonzeros). Lane l
      // owns the quads at 4l + 256 it and 4l + 128 + 256 it.
      const int64_t first = vec ? (e0 & ~(int64_t)3) : e0;
      for (int64_t wb = first; wb < e1; wb += (int64_t)1 << 30) {
        const int n_el = (int)min((int64_t)1 << 30, e1 - wb);
        const int lo = (int)max((int64_t)0, e0 - wb);
        for (uint32_t i = lane; i <= rows; i += 32) {
          const int64_t x = ip_s[i] - wb;
          rel_p[i] = x > 0x7fffffff ? 0x7fffffff : (x < 0 ? 0 : (int)x);
        }
        __syncwarp();
        const int* __restrict__ src = indices + wb;
        int nxt = lds_s32(rel_a + 4 * (cr + 1));
        auto load_quad = [&](int q, int (&v)[4]) {
          if (vec && q + 4 <= n_el) {
            const int4 t4 = __ldcs(reinterpret_cast<const int4*>(src + q));
            v[0] = t4.x; v[1] = t4.y; v[2] = t4.z; v[3] = t4.w;
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = (q + u >= lo && q + u < n_el) ? __ldcs(src + q + u) : 0;
          }
        };
        int cur[2][4], nx[2][4];
        int p = 4 * lane;
        if (p < n_el) { load_quad(p, cur[0]); load_quad(p + 128, cur[1]); }
        for (; p < n_el; p += 256) {
          if (p + 256 < n_el) { load_quad(p + 256, nx[0]); load_quad(p + 384, nx[1]); }
          uint32_t idx[8], j[8];
          bool in[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = p + 128 * (u >> 2) + (u & 3);
            in[u] = (unsigned)(e - lo) < (unsigned)(n_el - lo);
            const uint32_t x = (uint32_t)cur[u >> 2][u & 3];
            max_idx = in[u] ? max(max_idx, x) : max_idx;    // negative -> huge -> flagged
            idx[u] = min(x, d32 - 1);
          }
          if (MODE == kPiGlobal) {
#pragma unroll
            for (int u = 0; u < 8; ++u) j[u] = __ldg(pi + idx[u]);
          } else if (MODE == kPiSmem16) {
#pragma unroll
            for (int u = 0; u < 8; ++u) j[u] = lds_u16(pi_a + 2 * idx[u]);
          } else if (MODE == kPiSeeded) {
#pragma unroll
            for (int u = 0; u < 8; ++u) j[u] = pi_seeded(seed, idx[u], mn);
          } else {
            uint32_t c[8], g[8];
            bool miss[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) c[u] = lds_u32(pi_a + 4 * (idx[u] & (kCacheSlots - 1)));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              miss[u] = (c[u] >> 16) != (idx[u] >> 15);
              g[u] = __ldg(pi + (miss[u] ? idx[u] : 0u));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              j[u] = miss[u] ? g[u] : (c[u] & 0xFFFFu);
              if (miss[u] && in[u] && g[u] < 65536u)
                sts_u32(pi_a + 4 * (idx[u] & (kCacheSlots - 1)), ((idx[u] >> 15) << 16) | g[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (MODE == kPiGlobal || MODE == kPiCache) {
              max_j = in[u] ? max(max_j, j[u]) : max_j;
              j[u] = min(j[u], N - 1);
            }
            if (in[u]) {
              const int e = p + 128 * (u >> 2) + (u & 3);
              while (e >= nxt) { ++cr; nxt = lds_s32(rel_a + 4 * (cr + 1)); }
              red_or_shared(tile_a + 4 * (cr * W + (j[u] >> 5)), 1u << (j[u] & 31u));
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < 4; ++u) cur[h][u] = nx[h][u];
        }
        __syncwarp();
      }
    } else {
      bad_bits = kStatusIndex;  // decreasing / negative indptr: rows of this tile stay zero
    }
    __syncwarp();
    uint32_t* dst = out + r0 * W;
    if ((nw & 3u) == 0 && ((r0 * W) & 3u) == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
      for (uint32_t w = lane * 4; w < nw; w += 128)
        __stcs(reinterpret_cast<uint4*>(dst + w), *reinterpret_cast<const uint4*>(tile + w));
    } else {
      for (uint32_t w = lane; w < nw; w += 32) __stcs(dst + w, tile[w]);
    }
    __syncwarp();
  }
  if (max_idx >= d32 || ((MODE == kPiGlobal || MODE == kPiCache) && max_j >= N)) bad_bits = kStatusIndex;
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

// Largest RW (rows per warp tile, <= 32, RW*W <= kTileWordsMax) whose per-warp shared
// memory fits `per_warp` bytes; 0 if even one row does not fit.
static uint32_t pick_rw(uint32_t W, size_t per_warp) {
  uint32_t rw = std::max<uint32_t>(1, std::min<uint32_t>(32, kTileWordsMax / W));
  for (; rw >= 1; --rw) {
    const size_t need = (((size_t)(rw + 1) * 12 + 15) / 16) * 16 + (((size_t)rw * W * 4 + 15) / 16) * 16;
    if (need <= per_warp) return rw;
  }
  return 0;
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
  const size_t optin = (size_t)smem_optin;

  int mode = kPiGlobal, threads = 256;
  size_t pi_bytes = 0;
  const size_t smem16_bytes = ((d * 2 + 15) / 16) * 16;
  if (pi == nullptr) {
    mode = kPiSeeded;
  } else if (N <= 65536 && smem16_bytes <= 96 * 1024) {
    mode = kPiSmem16; threads = 1024; pi_bytes = smem16_bytes;
  } else if (N <= 65536 && d < 0x80000000ull - 32768ull) {
    mode = kPiCache; threads = 1024; pi_bytes = (size_t)kCacheSlots * 4;
  }
  // Experiment knob (ncu A/B of the pi source): BINSKETCH_BUILD_MODE=global|cache|smem16.
  const char* force = std::getenv("BINSKETCH_BUILD_MODE");
  if (force && pi != nullptr && N <= 65536) {
    if (!std::strcmp(force, "global")) { mode = kPiGlobal; threads = 256; pi_bytes = 0; }
    if (!std::strcmp(force, "cache") && d < 0x80000000ull - 32768ull) {
      mode = kPiCache; threads = 1024; pi_bytes = (size_t)kCacheSlots * 4;
    }
    if (!std::strcmp(force, "smem16") && smem16_bytes + 32 * 1024 <= optin) {
      mode = kPiSmem16; threads = 1024; pi_bytes = smem16_bytes;
    }
  }
  uint32_t RW = pick_rw(W, (optin - pi_bytes) / (threads / 32));
  if (RW == 0 && mode != kPiSeeded && mode != kPiGlobal) {   // wide sketches: drop the smem table
    mode = kPiGlobal; threads = 256; pi_bytes = 0;
    RW = pick_rw(W, optin / (threads / 32));
  }
  if (RW == 0 || (mode == kPiSeeded && RW == 0)) RW = pick_rw(W, optin / (threads / 32));
  if (RW == 0) {
    cudaError_t e = cudaMemsetAsync(out, 0, n * (size_t)W * 4, s);
    if (e != cudaSuccess) return e;
    build_wide_kernel<<<sms * 8, 256, 0, s>>>(pi, seed, d, mn, pi == nullptr, indptr, indices, n, out, W, st);
    count_launch();
    return cudaGetLastError();
  }
  const size_t per_warp = (((size_t)(RW + 1) * 12 + 15) / 16) * 16 + (((size_t)RW * W * 4 + 15) / 16) * 16;
  const size_t smem = pi_bytes + per_warp * (threads / 32);
  const uint64_t ntiles = (n + RW - 1) / RW;
  const uint64_t want_blocks = (ntiles + (threads / 32) - 1) / (threads / 32);
  const int per_sm = std::max<int>(1, std::min<int>(2048 / threads, (int)(optin / std::max<size_t>(smem, 1))));
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>(want_blocks, (uint64_t)sms * per_sm));
  cudaError_t e = cudaSuccess;
#define BSK_LAUNCH_BUILD(M)                                                                            \
  do {                                                                                                 \
    e = cudaFuncSetAttribute(build_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                    \
    build_kernel<M><<<(unsigned)blocks, threads, smem, s>>>(pi, seed, d, mn, indptr, indices, n, out,  \
                                                            W, RW, pi_bytes, st);                      \
    count_launch();                                                                                    \
  } while (0)
  switch (mode) {
    case kPiSmem16: BSK_LAUNCH_BUILD(kPiSmem16); break;
    case kPiCache: BSK_LAUNCH_BUILD(kPiCache); break;
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
