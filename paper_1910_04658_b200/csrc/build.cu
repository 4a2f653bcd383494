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
#include <type_traits>
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

// The latched status word of the CURRENT device (a __device__ variable has one instance per
// device): its address is cached per device ordinal; racing first calls store the same value.
unsigned int* status_ptr() {
  constexpr int kMaxDev = 64;
  static std::atomic<unsigned int*> cache[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  if (dev >= 0 && dev < kMaxDev) {
    unsigned int* p = cache[dev].load(std::memory_order_acquire);
    if (p) return p;
  }
  void* v = nullptr;
  if (cudaGetSymbolAddress(&v, g_status) != cudaSuccess) return nullptr;
  unsigned int* p = static_cast<unsigned int*>(v);
  if (dev >= 0 && dev < kMaxDev) cache[dev].store(p, std::memory_order_release);
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
// Sketch construction, v5: one continuous element stream per warp.
//
// A warp owns a contiguous range of row tiles (RW rows each) and streams the range's
// nonzeros, indices[indptr[Ra] .. indptr[Rb]), as ONE sequence of stages (S elements,
// 1-D bulk copies issued by lane 0 into a per-warp shared ring, completion on an
// mbarrier) — no per-tile restart and no half-empty tail stage per tile. Stage data are
// read as 16-byte quads: lane l holds elements 4l..4l+3 (+128 h) of each 256-element half.
//
// Rows live in a per-warp shared ring of RR = 2 RW sketch rows (compact: empty rows take
// no slot). The two oldest unflushed tiles t, t+1 form the WINDOW: a stage is processed
// up to the window end (the end of tile t+1); when tile t is complete it is flushed
// (every output word written once, coalesced 16-byte streaming stores, then its ring rows
// re-zeroed) and tile t+2 enters the window. Rows of a stage that lie beyond the window
// are processed in a further pass over the same stage data (only when 2 tiles hold fewer
// than S nonzeros).
//
// Row of an element without a search: a 2048-element bitmap P (bit q: a nonempty window
// row ends at offset q) plus, per 32-bit word w, B[w] = the ring row live at the word's
// start; the row of element q is B[q/32] + popc(P[q/32] & mask_le(q)) — wrapped into the
// ring with one LOP3 (ring bytes a power of two, ring base aligned to it).
//
// pi(i) comes from (MODE): kPiSeeded (splitmix64 recipe in registers), kPiSmem16 (the whole
// table in shared memory as uint16), kPiCache16 / kPiCache32 (direct-mapped shared cache of
// the table, entry = tag:value), kPiGlobal (read-only L1/L2 gather). pi is read-only, so
// every cache entry ever written is correct and racing fills are benign.
// Bits are OR-ed (XOR for the BCS parity sketch) into the ring with shared reductions.
enum PiMode { kPiSeeded = 0, kPiSmem16 = 1, kPiCache16 = 2, kPiCache32 = 3, kPiGlobal = 4 };

constexpr int kChunk = 2048;                  // elements per row-boundary bitmap
constexpr int kChunkWords = kChunk / 32;      // 64 {P, B} pairs
constexpr uint32_t kMetaBytes = kChunkWords * 8;
constexpr uint32_t kCache16Slots = 65536;     // 128 KB
constexpr uint32_t kCache32Slots = 32768;     // 128 KB
constexpr uint32_t kFull = 0xffffffffu;
constexpr int kNS = 2;                        // stage ring depth per warp
constexpr uint32_t kAuxFixed = kMetaBytes + 16 * kNS;  // bitmap + mbarriers (per warp; + a zero row of 4W bytes)

// Per-mode launch shape. Cache / shared-table modes: one 512-thread block per SM (the table
// shared by all warps), 1 KB stages; the others: BSK_BUILD_BLOCKS blocks of BSK_BUILD_THREADS
// per SM, 4 KB stages (measured: DESIGN.md K1).
#ifndef BSK_BUILD_STAGE
#define BSK_BUILD_STAGE 1024      // elements per stage (register-pi modes)
#endif
#ifndef BSK_BUILD_THREADS
#define BSK_BUILD_THREADS 384
#endif
#ifndef BSK_BUILD_BLOCKS
#define BSK_BUILD_BLOCKS 1
#endif
#ifndef BSK_BUILD_RRMAX
#define BSK_BUILD_RRMAX 64        // ring rows cap (tiles of RR / 2 rows)
#endif
#ifndef BSK_BUILD_PI_STAGE
#define BSK_BUILD_PI_STAGE 256    // elements per stage (shared-memory pi modes)
#endif
#ifndef BSK_BUILD_FILL_STAGES
#define BSK_BUILD_FILL_STAGES 0   // cache modes: stages per warp that fill the cache on a miss (0: all, < 0: none)
#endif
#ifndef BSK_BUILD_PI_THREADS
#define BSK_BUILD_PI_THREADS 384
#endif
template <int MODE>
struct BuildCfg {
  static constexpr bool kSmemPi = !(MODE == kPiSeeded || MODE == kPiGlobal);
  static constexpr int kThreads = kSmemPi ? BSK_BUILD_PI_THREADS : BSK_BUILD_THREADS;
  static constexpr int kBlocks = kSmemPi ? 1 : BSK_BUILD_BLOCKS;
  static constexpr int kStage = kSmemPi ? BSK_BUILD_PI_STAGE : BSK_BUILD_STAGE;   // elements per stage
  static constexpr int kStageBytes = kStage * 4;
};

struct BuildParams {
  const uint32_t* pi;
  uint64_t seed;
  ModN mn;
  const int64_t* indptr;
  const int32_t* indices;
  uint64_t n;
  uint32_t* out;
  uint64_t ntiles;        // ceil(n / RW)
  uint32_t d, W, RR;      // RR: ring rows (power of two >= 4); tiles of RW = RR / 2 rows
  uint32_t pi_bytes;      // shared bytes of the pi table / cache (block-wide, first)
  uint32_t ring_align;    // alignment of the rings (RR * 4W when N is a power of two, else 16)
  uint32_t aux_bytes;     // per-warp stages + bitmap + mbarriers
  uint32_t vb;            // cache: value bits
  uint32_t out16;         // out 16-B aligned and W % 4 == 0: vector flush
  unsigned int* status;
};

// 32-bit shared-memory accessors: shared addresses stay in one register, no generic
// conversion per access. Volatile keeps them ordered among themselves (and after the
// mbarrier waits); none clobbers "memory", so global loads schedule freely around them.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v));
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void sts_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w));
}
__device__ __forceinline__ void sts_u16_if(bool pred, uint32_t a, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u16 [%0], %1;\n\t}"
               ::"r"(a), "h"((unsigned short)v), "r"((uint32_t)pred));
}
__device__ __forceinline__ void sts_u32_if(bool pred, uint32_t a, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}"
               ::"r"(a), "r"(v), "r"((uint32_t)pred));
}
// A sketch bit: OR (BinSketch) or XOR (BCS parity buckets),
// optionally predicated (no branch: the partial-stage path stays convergent).
template <bool XOR>
__device__ __forceinline__ void put_bit(uint32_t a, uint32_t v) {
  if (XOR) asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(a), "r"(v));
  else asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v));
}
template <bool XOR>
__device__ __forceinline__ void put_bit_if(bool pred, uint32_t a, uint32_t v) {
  if (XOR)
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.xor.b32 [%0], %1;\n\t}"
                 ::"r"(a), "r"(v), "r"((uint32_t)pred));
  else
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.or.b32 [%0], %1;\n\t}"
                 ::"r"(a), "r"(v), "r"((uint32_t)pred));
}
// a * b + c on the FMA pipe (IMAD): the ALU pipe is the busier one in K1's inner loop
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
// 1 << (x mod 32) in one funnel shift (shf.l.wrap takes the shift amount mod 32).
__device__ __forceinline__ uint32_t bit_of(uint32_t x) {
  uint32_t r;
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(0u), "r"(1u), "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// 64-bit x * c (mod 2^64) as exactly three 32-bit multiplies (mul.wide + 2 mad.lo).
__device__ __forceinline__ uint64_t mul64c(uint64_t x, uint32_t clo, uint32_t chi) {
  uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32), rlo, rhi;
  asm("{\n\t.reg .u64 t;\n\t"
      "mul.wide.u32 t, %2, %4;\n\t"
      "mov.b64 {%0, %1}, t;\n\t"
      "mad.lo.u32 %1, %3, %4, %1;\n\t"
      "mad.lo.u32 %1, %2, %5, %1;\n\t}"
      : "=r"(rlo), "=r"(rhi) : "r"(lo), "r"(hi), "r"(clo), "r"(chi));
  return ((uint64_t)rhi << 32) | rlo;
}

// pi(i) for a power-of-two N; seed1 = seed + gamma, so seed + (i+1)*gamma = seed1 + i*gamma
// (one wide multiply-add). Only the low log2(N) bits of the finalizer are needed. Returns
// x, the low finalizer word before masking (j = x & (N-1); x & 31 = j & 31 when N >= 32).
__device__ __forceinline__ uint32_t pi_pow2_raw(uint64_t seed1, uint32_t i) {
  uint32_t zl, zh;   // z = seed1 + i * gamma (64-bit), as a carry chain of 32-bit multiply-adds
  asm("mad.lo.cc.u32 %0, %2, %3, %4;\n\t"
      "madc.hi.u32 %1, %2, %3, %5;\n\t"
      "mad.lo.u32 %1, %2, %6, %1;"
      : "=r"(zl), "=r"(zh) : "r"(i), "r"(0x7F4A7C15u), "r"((uint32_t)seed1), "r"((uint32_t)(seed1 >> 32)),
        "r"(0x9E3779B9u));
  uint64_t z = ((uint64_t)zh << 32) | zl;
  z ^= z >> 30;
  z = mul64c(z, 0x1CE4E5B9u, 0xBF58476Du);
  z ^= z >> 27;
  z = mul64c(z, 0x133111EBu, 0x94D049BBu);
  return (uint32_t)z ^ (uint32_t)(z >> 31);
}

// Predicated read-only load (no branch): v = pred ? *p : v.
__device__ __forceinline__ uint32_t ldg_if(const uint32_t* ptr, bool pred, uint32_t v) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
      : "+r"(v) : "l"(ptr), "r"((uint32_t)pred));
  return v;
}

// One row tile in registers (warp-collective state): lane l < rows holds the end offset
// (relative to the warp's stream base) of the tile's row l; lanes >= rows hold the tile end.
struct Tile {
  int e;          // end of this lane's row (monotone across lanes)
  uint32_t ne;    // nonempty-row mask
  uint32_t c;     // compact index of the tile's first nonempty row (ring row = c mod RR)
  int tend;       // end of the tile's last row
  uint32_t rows;  // rows in the tile
};

// Checked build (-DBSK_CHECKED; a dev library, never the product): every shared-memory access of
// K1 is range-checked against the regions it may touch — the block-wide pi table / cache, or the
// warp's OWN ring / stages / bitmap / mbarriers / zero row (so no warp reads or writes another
// warp's rows: the inter-warp race a racecheck would look for) — and a violation traps the kernel.
#ifdef BSK_CHECKED
#define BSK_CHKE(a, n) (chk_ok((uint32_t)(a), (uint32_t)(n)) ? (void)0 : __trap())
#define BSK_CHK(a, n) BSK_CHKE(a, n)
#define lds_u16(a) (BSK_CHKE(a, 2), lds_u16(a))
#define lds_u32(a) (BSK_CHKE(a, 4), lds_u32(a))
#define lds_v2(a) (BSK_CHKE(a, 8), lds_v2(a))
#define lds_v4(a) (BSK_CHKE(a, 16), lds_v4(a))
#define sts_u16(a, v) (BSK_CHKE(a, 2), sts_u16(a, v))
#define sts_u32(a, v) (BSK_CHKE(a, 4), sts_u32(a, v))
#define sts_v4(a, x, y, z, w) (BSK_CHKE(a, 16), sts_v4(a, x, y, z, w))
#define sts_u16_if(q, a, v) (BSK_CHKE(a, 2), sts_u16_if(q, a, v))
#define sts_u32_if(q, a, v) (BSK_CHKE(a, 4), sts_u32_if(q, a, v))
#else
#define BSK_CHK(a, n) do {} while (0)
#endif
template <int MODE, int LOGN, bool XOR>
__global__ void __launch_bounds__(BuildCfg<MODE>::kThreads, BuildCfg<MODE>::kBlocks)
build_kernel(const BuildParams p) {
  constexpr int S = BuildCfg<MODE>::kStage, SB = BuildCfg<MODE>::kStageBytes;
  constexpr bool POW2 = LOGN > 0;
  constexpr uint32_t wmask = POW2 ? ((1u << LOGN) - 1u) & ~31u : 0u;   // j & wmask = 32 * (j / 32)
  constexpr uint32_t wsh = POW2 ? LOGN - 3 : 0;                         // log2(4W)
  constexpr uint32_t kSlots = MODE == kPiCache16 ? kCache16Slots : kCache32Slots;
  constexpr uint32_t kSlotBits = MODE == kPiCache16 ? 16 : 15;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const uint32_t N = p.mn.N, W = p.W, Wb = 4 * W, d = p.d, RR = p.RR, RW = RR >> 1;
  const uint32_t ringB = RR * Wb;
  const uint32_t pi_a = smem_u32(smem);
  const uint32_t rows0 = (pi_a + p.pi_bytes + p.ring_align - 1) & ~(p.ring_align - 1);
  const uint32_t ring_a = rows0 + (uint32_t)warp * ringB;
  const uint32_t stage_a = rows0 + (uint32_t)nwarps * ringB + (uint32_t)warp * p.aux_bytes;
  const uint32_t meta_a = stage_a + kNS * SB;
  const uint32_t mbar_a = meta_a + kMetaBytes;
  const uint32_t zero_a = mbar_a + 8 * kNS;           // one all-zero sketch row (flush of empty rows)
  const uint64_t seed1 = p.seed + 0x9E3779B97F4A7C15ULL;
  const uint32_t vb = p.vb, vmask = (1u << vb) - 1u;
#ifdef BSK_CHECKED
  auto chk_ok = [&](uint32_t a, uint32_t n) -> bool {
    const bool tab = a >= pi_a && a + n <= pi_a + p.pi_bytes;
#ifdef BSK_CHECKED_SELFTEST
    const bool ring = a >= ring_a && a + n <= ring_a + ringB - Wb;   // (the checker's own test: one ring row short)
#else
    const bool ring = a >= ring_a && a + n <= ring_a + ringB;
#endif
    const bool aux = a >= stage_a && a + n <= stage_a + p.aux_bytes;
    return (n > 16 || (a & (n - 1)) == 0) && (tab || ring || aux);   // (natural alignment of the access widths)
  };
#endif

  unsigned bad = 0;
  uint32_t maxj = 0, maxidx = 0;
  if (MODE == kPiSmem16 || MODE == kPiCache16 || MODE == kPiCache32) {
    // the shared copy of the table (whole, or its first kSlots entries as the cache's initial
    // contents: tag 0), four entries per 16-B load: this fill is a fixed cost of every launch
    // (the whole cost of a small build), so it runs at load width with four loads in flight
    const uint32_t n_fill = MODE == kPiSmem16 ? d : kSlots;
    const uint32_t n_src = min(n_fill, d);
    const bool pv = (reinterpret_cast<uintptr_t>(p.pi) & 15u) == 0;
    const uint32_t g4 = pv ? n_src / 4 : 0;   // whole 4-entry groups read as uint4
#pragma unroll 4
    for (uint32_t g = threadIdx.x; g < g4; g += blockDim.x) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(p.pi) + g);
      maxj = max(maxj, max(max(x.x, x.y), max(x.z, x.w)));
      const uint32_t a = min(x.x, N - 1), b = min(x.y, N - 1), c = min(x.z, N - 1), e = min(x.w, N - 1);
      if (MODE == kPiCache32) {
        sts_v4(pi_a + 16 * g, a, b, c, e);
      } else {
        sts_u32(pi_a + 8 * g, a | (b << 16));
        sts_u32(pi_a + 8 * g + 4, c | (e << 16));
      }
    }
    for (uint32_t s = 4 * g4 + threadIdx.x; s < n_fill; s += blockDim.x) {
      uint32_t v = s < d ? __ldg(p.pi + s) : 0u;
      maxj = max(maxj, v);
      v = min(v, N - 1);
      if (MODE == kPiCache32) sts_u32(pi_a + 4 * s, v); else sts_u16(pi_a + 2 * s, v);
    }
  }
  for (uint32_t w = 4 * lane; w < RR * W; w += 128) sts_v4(ring_a + 4 * w, 0u, 0u, 0u, 0u);
  for (uint32_t w = lane; w < W; w += 32) sts_u32(zero_a + 4 * w, 0u);
  if (lane == 0) {
    for (int s = 0; s < kNS; ++s) mbar_init(mbar_a + 8 * s, 1);
    fence_proxy_async();
  }
  __syncthreads();

  // lane constants: masks selecting bitmap-word bits <= element (4*lane + k) mod 32
  uint32_t mle[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) mle[k] = (2u << ((4 * lane + k) & 31)) - 1u;
  const uint32_t lmlt = lanemask_lt();

  // ---- this warp's tiles [t_begin, t_end) and its element stream ----
  const uint64_t G = (uint64_t)gridDim.x * nwarps, g = (uint64_t)blockIdx.x * nwarps + warp;
  const uint64_t t_begin = p.ntiles * g / G, t_end = p.ntiles * (g + 1) / G;
  if (t_begin < t_end) {
    const uint64_t Ra = t_begin * RW, Rb = min(t_end * RW, p.n);
    const int64_t S0 = __ldg(p.indptr + Ra), Send = __ldg(p.indptr + Rb), Etot = __ldg(p.indptr + p.n);
    const bool valid = S0 >= 0 && S0 <= Send && Send <= Etot;
    auto tile_rows = [&](uint64_t tt) -> uint32_t { return (uint32_t)min((uint64_t)RW, p.n - tt * RW); };
    auto out_row = [&](uint64_t r) { return p.out + r * W; };

    if (!valid || Send - S0 > 0x7ff00000ll) {
      // Invalid indptr (latched, rows zeroed) or more than 2^31 nonzeros in one warp's range:
      // a row-at-a-time loop through ring row 0 (64-bit offsets; correct, not fast).
      for (uint64_t r = Ra; r < Rb; ++r) {
        const int64_t rs = __ldg(p.indptr + r), re = __ldg(p.indptr + r + 1);
        if (!valid || rs > re || rs < 0 || re > Etot) {
          bad = 1;
        } else {
          for (int64_t q = rs + lane; q < re; q += 32) {
            const uint32_t x = (uint32_t)__ldg(p.indices + q);
            maxidx = max(maxidx, x);
            uint32_t jj;
            if (MODE == kPiSeeded) {
              jj = pi_seeded(p.seed, (uint64_t)x, p.mn);
            } else {
              jj = __ldg(p.pi + min(x, d - 1));
              maxj = max(maxj, jj);
              jj = min(jj, N - 1);
            }
            BSK_CHK(ring_a + ((jj >> 5) << 2), 4);
            put_bit<XOR>(ring_a + ((jj >> 5) << 2), 1u << (jj & 31u));
          }
        }
        __syncwarp();
        for (uint32_t w = lane; w < W; w += 32) {
          __stcs(out_row(r) + w, lds_u32(ring_a + 4 * w));
          sts_u32(ring_a + 4 * w, 0u);
        }
        __syncwarp();
      }
    } else {
      const int64_t base = S0 & ~(int64_t)3;            // 16-B aligned stream start
      const int head = (int)(S0 - base), end = (int)(Send - base), end4 = end & ~3;
      const int nst = (end + S - 1) / S;
      const int32_t* src0 = p.indices + base;

      // raw indptr ends of tile tt (prefetched one tile ahead)
      auto load_raw = [&](uint64_t tt) -> int64_t {
        return (uint32_t)lane < tile_rows(tt) ? __ldg(p.indptr + tt * RW + lane + 1) : INT64_MIN;
      };
      // clamp into [prev_end, end], make monotone (inclusive max scan), flag any change
      auto finish = [&](int64_t raw, uint32_t rows, int prev_end, uint32_t c) -> Tile {
        Tile T;
        const bool has = (uint32_t)lane < rows;
        const int64_t v = raw - base;
        int e = has ? (int)min(max(v, (int64_t)prev_end), (int64_t)end) : end;
        int st = __shfl_up_sync(kFull, e, 1);
        if (lane == 0) st = prev_end;
        if (!__all_sync(kFull, !has || (e >= st && (int64_t)e == v))) {
          // a decreasing or out-of-range indptr (latched): make the ends monotone
          bad = 1;
          if (!has) e = prev_end;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, e, o);
            if (lane >= o) e = max(e, y);
          }
          st = __shfl_up_sync(kFull, e, 1);
          if (lane == 0) st = prev_end;
        }
        T.rows = rows;
        const int last = __shfl_sync(kFull, e, rows - 1);   // (all lanes: a shuffle must not diverge)
        T.e = has ? e : last;
        T.ne = __ballot_sync(kFull, has && e > st);
        T.tend = __shfl_sync(kFull, T.e, 31);
        T.c = c;
        return T;
      };
      auto empty_tile = [&](int at, uint32_t c) -> Tile {
        Tile T;
        T.e = at; T.ne = 0u; T.tend = at; T.rows = 0u; T.c = c;
        return T;
      };
      // tile tt complete: write its rows (every output word exactly once), re-zero its ring rows
      auto flush = [&](const Tile& T, uint64_t tt) {
        const uint32_t nw = T.rows * W;
        uint32_t* dst = out_row(tt * RW);
        if (POW2 && p.out16 && LOGN <= 12) {
          // lane r: ring address of the tile's row r (an empty row reads the warp's zero row);
          // 128 words per iteration, no per-word predicate for a whole tile
          const uint32_t myra = ((T.ne >> lane) & 1u) ? ring_a + ((T.c + __popc(T.ne & lmlt)) & (RR - 1u)) * Wb : zero_a;
          constexpr uint32_t lw = LOGN > 5 ? LOGN - 5 : 0;               // log2(W)
          constexpr uint32_t rpi = lw <= 7 ? (128u >> lw) : 1u;           // rows per iteration
          const uint32_t sub = (4u * lane) >> lw, wo = 4u * ((4u * lane) & ((1u << lw) - 1u));
          uint4* d4 = reinterpret_cast<uint4*>(dst) + lane;
          if (nw == RW * W && (RW * W) % 128 == 0) {
#pragma unroll 4
            for (uint32_t i = 0; i < RW * W / 128; ++i) {
              const uint32_t a = __shfl_sync(kFull, myra, (i * rpi + sub) & 31u) + wo;
              const uint4 v = lds_v4(a);
              sts_v4(a, 0u, 0u, 0u, 0u);
              __stcs(d4 + 32 * i, v);
            }
          } else {
            for (uint32_t i = 0; 128 * i < nw; ++i) {          // warp-uniform trip count
              const uint32_t a = __shfl_sync(kFull, myra, (i * rpi + sub) & 31u) + wo;
              if (4 * lane + 128 * i < nw) {
                const uint4 v = lds_v4(a);
                sts_v4(a, 0u, 0u, 0u, 0u);
                __stcs(d4 + 32 * i, v);
              }
            }
          }
        } else if (p.out16) {
          for (uint32_t w = 4 * lane; w < nw; w += 128) {
            const uint32_t r = w / W;
            const uint32_t wi = w - r * W;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if ((T.ne >> r) & 1u) {
              const uint32_t idx = (T.c + __popc(T.ne & ((1u << r) - 1u))) & (RR - 1u);
              const uint32_t a = ring_a + idx * Wb + 4 * wi;
              v = lds_v4(a);
              sts_v4(a, 0u, 0u, 0u, 0u);
            }
            __stcs(reinterpret_cast<uint4*>(dst + w), v);
          }
        } else {
          for (uint32_t w = lane; w < nw; w += 32) {
            const uint32_t r = w / W;
            const uint32_t wi = w - r * W;
            uint32_t v = 0u;
            if ((T.ne >> r) & 1u) {
              const uint32_t idx = (T.c + __popc(T.ne & ((1u << r) - 1u))) & (RR - 1u);
              const uint32_t a = ring_a + idx * Wb + 4 * wi;
              v = lds_u32(a);
              sts_u32(a, 0u);
            }
            __stcs(dst + w, v);
          }
        }
        __syncwarp();
      };

      uint64_t t = t_begin;
      Tile T0 = finish(load_raw(t), tile_rows(t), head, 0u);
      Tile T1 = t + 1 < t_end ? finish(load_raw(t + 1), tile_rows(t + 1), T0.tend, T0.c + __popc(T0.ne))
                              : empty_tile(T0.tend, T0.c + __popc(T0.ne));
      int64_t raw2 = t + 2 < t_end ? load_raw(t + 2) : 0;
      int wend = T1.tend;
      auto advance = [&]() {
        T0 = T1;
        ++t;
        const uint32_t c = T0.c + __popc(T0.ne);
        if (t + 1 < t_end) {
          T1 = finish(raw2, tile_rows(t + 1), T0.tend, c);
          raw2 = t + 2 < t_end ? load_raw(t + 2) : 0;
        } else {
          T1 = empty_tile(T0.tend, c);
        }
        wend = T1.tend;
      };

      // stage k -> ring slot k % kNS; bulk copy of its 16-B aligned part (lane 0)
      auto issue = [&](int k) {
        if (k >= nst || lane != 0) return;
        const int s = k * S;
        const int nb = max(0, min(s + S, end4) - s) * 4;
        // (no proxy fence: the slot's previous contents were read by LDS whose results the
        // warp consumed before this point, and the mbarrier wait orders the copy's writes)
        const uint32_t slot = stage_a + (uint32_t)(k % kNS) * SB, mb = mbar_a + 8u * (uint32_t)(k % kNS);
        BSK_CHK(mb, 8);
        BSK_CHK(slot, (uint32_t)SB);
        if (nb > 0) {
          mbar_expect_tx(mb, (uint32_t)nb);
          bulk_load(slot, src0 + s, (uint32_t)nb, mb);
        } else {
          mbar_arrive(mb);
        }
      };

      // row-boundary bitmap of [b0, b0 + kChunk) for the window's rows
      auto build_bitmap = [&](int b0) {
        sts_v4(meta_a + 16 * lane, 0u, 0u, 0u, 0u);
        __syncwarp();
        int q = T0.e - b0;
        if (((T0.ne >> lane) & 1u) && q > 0 && q < kChunk) { BSK_CHK(meta_a + 8 * (uint32_t)(q >> 5), 4); put_bit<false>(meta_a + 8 * (uint32_t)(q >> 5), 1u << (q & 31)); }
        q = T1.e - b0;
        if (((T1.ne >> lane) & 1u) && q > 0 && q < kChunk) { BSK_CHK(meta_a + 8 * (uint32_t)(q >> 5), 4); put_bit<false>(meta_a + 8 * (uint32_t)(q >> 5), 1u << (q & 31)); }
        const uint32_t before = T0.c + __popc(T0.ne & __ballot_sync(kFull, T0.e <= b0)) +
                                __popc(T1.ne & __ballot_sync(kFull, T1.e <= b0));
        __syncwarp();
        const uint4 pr = lds_v4(meta_a + 16 * lane);
        const uint32_t c0 = __popc(pr.x), c = c0 + __popc(pr.z);
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += y;
        }
        const uint32_t b = before + incl - c;
        const uint32_t B0 = POW2 ? ((b & (RR - 1u)) << wsh) : (b & (RR - 1u));
        const uint32_t B1 = POW2 ? (((b + c0) & (RR - 1u)) << wsh) : ((b + c0) & (RR - 1u));
        sts_v4(meta_a + 16 * lane, pr.x, B0, pr.z, B1);
        __syncwarp();
      };

      // cache modes: misses fill the shared cache only in the warp's first kFillStages stages
      // (0: always); afterwards the cache is read-only (warp-uniform)
      bool fill_on = true;
      // one 256-element half of a stage: off = stage-relative offset of the half, wb = its
      // bitmap-relative offset; PRED: only elements at stage offsets [lo, hi) take effect
      auto half_step = [&](const uint32_t slot, const int off, const int wb, const int lo, const int hi,
                           auto pred_tag) {
        constexpr bool PRED = decltype(pred_tag)::value;
        const uint4 qa = lds_v4(slot + 4 * off + 16 * lane), qb = lds_v4(slot + 4 * off + 512 + 16 * lane);
        const uint32_t cur[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
        bool ok[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int pos = off + 128 * (u >> 2) + 4 * lane + (u & 3);
          ok[u] = !PRED || (pos >= lo && pos < hi);
        }
        const uint32_t wq = (uint32_t)(wb >> 5) + (uint32_t)(lane >> 3);
        uint32_t rowp[8];   // ring row part: byte offset (POW2) or ring index
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint2 pb = lds_v2(meta_a + 8 * (wq + 4 * h));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            rowp[4 * h + k] = POW2 ? mad_u32((uint32_t)__popc(pb.x & mle[k]), 1u << wsh, pb.y)   // FMA pipe, off the ALU
                                   : pb.y + (uint32_t)__popc(pb.x & mle[k]);
        }
        if (PRED) {
#pragma unroll
          for (int u = 0; u < 8; ++u) maxidx = max(maxidx, ok[u] ? cur[u] : 0u);
        } else {
          maxidx = __vimax3_u32(maxidx, __vimax3_u32(cur[0], cur[1], cur[2]),
                                __vimax3_u32(__vimax3_u32(cur[3], cur[4], cur[5]), cur[6], cur[7]));
        }
        uint32_t j[8], bit[8];
        if (MODE == kPiSeeded && POW2) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t x = pi_pow2_raw(seed1, cur[u]);
            j[u] = x & wmask;                         // = (j >> 5) << 5
            bit[u] = bit_of(x);                       // x & 31 = j & 31 since N >= 32
          }
        } else {
          if (MODE == kPiSeeded) {
#pragma unroll
            for (int u = 0; u < 8; ++u) j[u] = pi_seeded(p.seed, (uint64_t)cur[u], p.mn);
          } else if (MODE == kPiSmem16) {
#pragma unroll
            for (int u = 0; u < 8; ++u) j[u] = lds_u16(pi_a + 2 * min(cur[u], d - 1));
          } else if (MODE == kPiGlobal) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const uint32_t gv = __ldg(p.pi + min(cur[u], d - 1));
              maxj = max(maxj, ok[u] ? gv : 0u);
              j[u] = POW2 ? gv : min(gv, N - 1);    // POW2: the ring mask keeps any j in bounds
            }
          } else {
            // probe all 8, then issue all misses' loads (independent, predicated), then fill
            uint32_t c[8], slot_[8], x[8];
            bool miss[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              x[u] = min(cur[u], d - 1);
              slot_[u] = x[u] & (kSlots - 1);
              c[u] = MODE == kPiCache16 ? lds_u16(pi_a + 2 * slot_[u]) : lds_u32(pi_a + 4 * slot_[u]);
              miss[u] = (c[u] >> vb) != (x[u] >> kSlotBits);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) j[u] = ldg_if(p.pi + x[u], miss[u], c[u] & vmask);
            // fill every missed slot (branch-free: predicated stores) while the warp is in its
            // warm-up stages; afterwards the cache is read-only. Measured: a probabilistic
            // fill (1/4 of misses, hashed) keeps the simulated hit rate but was slower (1.75 vs 1.68 ms).
            if (fill_on) {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                maxj = max(maxj, (ok[u] && miss[u]) ? j[u] : 0u);
                if (!POW2) j[u] = min(j[u], N - 1);      // POW2: the ring mask keeps any j in bounds
                const uint32_t ent = ((x[u] >> kSlotBits) << vb) | (j[u] & vmask);
                if (MODE == kPiCache16) sts_u16_if(miss[u], pi_a + 2 * slot_[u], ent);
                else sts_u32_if(miss[u], pi_a + 4 * slot_[u], ent);
              }
            } else {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                maxj = max(maxj, (ok[u] && miss[u]) ? j[u] : 0u);
                if (!POW2) j[u] = min(j[u], N - 1);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) { bit[u] = bit_of(j[u]); j[u] &= ~31u; }
        }
        uint32_t addr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          addr[u] = POW2 ? (((rowp[u] + (j[u] >> 3)) & (ringB - 1u)) | ring_a)
                         : ring_a + (rowp[u] & (RR - 1u)) * Wb + (j[u] >> 3);
        if (PRED) {
#pragma unroll
          for (int u = 0; u < 8; ++u) { if (ok[u]) BSK_CHK(addr[u], 4); put_bit_if<XOR>(ok[u], addr[u], bit[u]); }
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) { BSK_CHK(addr[u], 4); put_bit<XOR>(addr[u], bit[u]); }
        }
      };

      for (int i = 0; i < kNS - 1; ++i) issue(i);
      int done = head;            // stream offsets < done are processed
      int b0 = 0;
      bool bm_ok = false;
      int fast_lim = 0;           // a stage [s, s + S) with done == s and s + S <= fast_lim runs unpredicated
      const int tail_k = end4 < end ? end4 / S : -1;
      // flush every complete tile; after an advance, rebuild the bitmap for the next stage
      auto retire = [&](int next_s) {
        if (t < t_end && T0.tend <= done) {
          do {
            flush(T0, t);
            advance();
          } while (t < t_end && T0.tend <= done);
          bm_ok = false;
          if (t < t_end && done == next_s && next_s < end) { build_bitmap(next_s); b0 = next_s; bm_ok = true; }
        }
        fast_lim = bm_ok ? min(min(wend, end), b0 + kChunk) : 0;
      };
      for (int k = 0; k < nst; ++k) {
        if (BSK_BUILD_FILL_STAGES != 0) fill_on = k < BSK_BUILD_FILL_STAGES;   // (< 0: never)
        issue(k + kNS - 1);
        const uint32_t slot = stage_a + (uint32_t)(k % kNS) * SB;
        mbar_wait(mbar_a + 8u * (uint32_t)(k % kNS), (uint32_t)(k / kNS) & 1u);
        const int s = k * S;
        if (k == tail_k) {   // < 4 trailing elements past the bulk copy: plain loads
          if (lane < end - end4) sts_u32(slot + 4u * (uint32_t)(end4 - s + lane), (uint32_t)__ldg(src0 + end4 + lane));
          __syncwarp();
        }
        bool full = done == s && s + S <= fast_lim;
        if (!full) {
          const int se = min(s + S, end);
          while (done < se) {
            if (t >= t_end) { done = se; break; }          // only after a latched bad indptr
            const int lim = min(se, wend);
            if (!bm_ok || s + S > b0 + kChunk) { build_bitmap(s); b0 = s; bm_ok = true; }
            if (done == s && lim == s + S) { full = true; break; }
#pragma unroll 1
            for (int h = 0; h < S / 256; ++h)
              if (256 * h + 256 > done - s && 256 * h < lim - s)
                half_step(slot, 256 * h, s - b0 + 256 * h, done - s, lim - s, std::true_type{});
            done = lim;
            __syncwarp();
            if (done < se) retire(s);
          }
        }
        if (full) {
#pragma unroll
          for (int h = 0; h < S / 256; ++h) half_step(slot, 256 * h, s - b0 + 256 * h, 0, S, std::false_type{});
          done = s + S;
        }
        __syncwarp();
        retire(s + S);
      }
      while (t < t_end) {   // tiles whose rows are all empty after the last element
        flush(T0, t);
        advance();
      }
    }
  }
  if (maxidx >= d || maxj >= N) bad = 1;
  if (__any_sync(kFull, bad != 0) && lane == 0) latch(p.status, kStatusIndex);
}

#ifdef BSK_CHECKED
#undef lds_u16
#undef lds_u32
#undef lds_v2
#undef lds_v4
#undef sts_u16
#undef sts_u32
#undef sts_v4
#undef sts_u16_if
#undef sts_u32_if
#endif
#undef BSK_CHK
#undef BSK_CHKE

// Fallback for very wide sketches (one row's W words do not fit the per-warp ring) and for
// index arrays that are not 16-B aligned (the bulk copies need it): rows zeroed by
// cudaMemsetAsync, then global atomicOr (atomicXor: BCS).
__global__ void build_wide_kernel(const uint32_t* __restrict__ pi, uint64_t seed, uint64_t d, ModN mn,
                                  bool seeded, bool parity, const int64_t* __restrict__ indptr,
                                  const int32_t* __restrict__ indices, uint64_t n,
                                  uint32_t* __restrict__ out, uint32_t W, unsigned int* status) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned bad = 0;
  for (uint64_t r = gw; r < n; r += nwarps) {
    int64_t b = indptr[r], e = indptr[r + 1];
    if (e < b || b < 0) { bad = kStatusIndex; continue; }
    for (int64_t t = b + lane; t < e; t += 32) {
      int32_t idx = indices[t];
      if (idx < 0 || (uint64_t)idx >= d) { bad = kStatusIndex; continue; }
      uint32_t j = seeded ? pi_seeded(seed, (uint64_t)idx, mn) : __ldg(pi + idx);
      if (j >= mn.N) { bad = kStatusIndex; continue; }
      if (parity) atomicXor(out + r * W + (j >> 5), 1u << (j & 31u));
      else atomicOr(out + r * W + (j >> 5), 1u << (j & 31u));
    }
  }
  if (bad) latch(status, bad);
}

static uint32_t bits_for(uint64_t v) {   // number of bits to represent 0..v
  uint32_t b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

cudaError_t launch_build(const uint32_t* pi, uint64_t seed, uint64_t d, uint32_t N,
                         const int64_t* indptr, const int32_t* indices, uint64_t n,
                         uint32_t* out, cudaStream_t s, bool parity) {
  if (n == 0) return cudaSuccess;
  const uint64_t W64 = ((uint64_t)N + 31) / 32;
  const uint32_t W = (uint32_t)W64;
  const ModN mn = make_modn(N);
  unsigned int* st = status_ptr();
  const int sms = num_sms();
  int dev = 0, smem_optin = 0, smem_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);

  auto wide = [&]() -> cudaError_t {
    cudaError_t e = cudaMemsetAsync(out, 0, n * W64 * 4, s);
    if (e != cudaSuccess) return e;
    build_wide_kernel<<<sms * 8, 256, 0, s>>>(pi, seed, d, mn, pi == nullptr, parity, indptr, indices, n, out, W, st);
    count_launch();
    return cudaGetLastError();
  };
  if ((reinterpret_cast<uintptr_t>(indices) & 15u) != 0 || W64 > 4096) return wide();

  const uint32_t vb = bits_for(N - 1);
  const uint32_t dbits = bits_for(d - 1);
  const bool c16 = N <= 65536 && (dbits > 16 ? dbits - 16 : 0) + vb <= 16;
  const bool c32 = (dbits > 15 ? dbits - 15 : 0) + vb <= 32;
  const uint64_t smem16_bytes = ((d * 2 + 15) / 16) * 16;
  int mode = kPiGlobal;
  if (pi == nullptr) mode = kPiSeeded;
  else if (N <= 65536 && smem16_bytes <= 100 * 1024) mode = kPiSmem16;
  else if (c16) mode = kPiCache16;
  else if (c32) mode = kPiCache32;
  // Experiment knob (A/B of the pi source): BINSKETCH_BUILD_MODE=global|cache|cache32|smem16.
  if (const char* f = pi != nullptr ? std::getenv("BINSKETCH_BUILD_MODE") : nullptr) {
    if (!std::strcmp(f, "global")) mode = kPiGlobal;
    if (!std::strcmp(f, "cache")) mode = c16 ? kPiCache16 : (c32 ? kPiCache32 : mode);
    if (!std::strcmp(f, "cache32") && c32) mode = kPiCache32;
    if (!std::strcmp(f, "smem16") && N <= 65536 && smem16_bytes + 64 * 1024 <= (uint64_t)smem_optin) mode = kPiSmem16;
  }
  // compiled-in sketch widths: the configs' N = 1024 (W = 32) and 4096 (W = 128); the BCS
  // parity variant for N = 1024 and the generic width
  const int logn = N == 1024 ? 10 : ((N == 4096 && !parity) ? 12 : 0);
  const uint64_t Wb = 4 * W64;

  // Shared memory per block: [pi] [align slack] [rings: nwarps x RR x Wb] [aux: nwarps x (stages + bitmap + mbar)]
  auto plan = [&](int m, uint32_t& RR, uint32_t& pi_bytes, uint32_t& align, uint32_t& aux, int& threads, int& bps,
                  size_t& smem) -> bool {
    const bool smem_pi = m == kPiSmem16 || m == kPiCache16 || m == kPiCache32;
    threads = smem_pi ? BuildCfg<kPiCache16>::kThreads : BuildCfg<kPiSeeded>::kThreads;
    bps = smem_pi ? BuildCfg<kPiCache16>::kBlocks : BuildCfg<kPiSeeded>::kBlocks;
    const uint32_t stage_bytes = smem_pi ? BuildCfg<kPiCache16>::kStageBytes : BuildCfg<kPiSeeded>::kStageBytes;
    pi_bytes = m == kPiSmem16 ? (uint32_t)smem16_bytes : (smem_pi ? 128u * 1024u : 0u);
    aux = kNS * stage_bytes + kAuxFixed + (uint32_t)((Wb + 15) / 16 * 16);   // 16-B aligned per-warp regions
    const size_t budget = std::min<size_t>((size_t)smem_optin, (size_t)smem_sm / bps - 1024);
    const int nw = threads / 32;
    for (uint32_t rr = BSK_BUILD_RRMAX; rr >= 4; rr >>= 1) {
      const uint64_t ringB = rr * Wb;
      align = logn ? (uint32_t)ringB : 16u;
      smem = pi_bytes + (size_t)(align - 16) + (size_t)nw * (ringB + aux);
      if (ringB <= (1u << 20) && smem <= budget) { RR = rr; return true; }
    }
    return false;
  };
  uint32_t RR = 0, pi_bytes = 0, align = 16, aux = 0;
  int threads = 0, bps = 0;
  size_t smem = 0;
  if (!plan(mode, RR, pi_bytes, align, aux, threads, bps, smem)) {
    if (mode == kPiSeeded || !plan(kPiGlobal, RR, pi_bytes, align, aux, threads, bps, smem)) return wide();
    mode = kPiGlobal;
  }
  BuildParams bp;
  bp.pi = pi; bp.seed = seed; bp.mn = mn; bp.indptr = indptr; bp.indices = indices; bp.n = n; bp.out = out;
  bp.d = (uint32_t)d; bp.W = W; bp.RR = RR; bp.vb = vb; bp.status = st;
  bp.pi_bytes = pi_bytes; bp.ring_align = align; bp.aux_bytes = aux;
  bp.ntiles = (n + RR / 2 - 1) / (RR / 2);
  bp.out16 = ((W & 3u) == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0) ? 1u : 0u;
  const int nw = threads / 32;
  const uint64_t want = (bp.ntiles + nw - 1) / nw;
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms * bps));
  cudaError_t e = cudaSuccess;
#define BSK_LAUNCH_BUILD3(M, LN, X)                                                                              \
  do {                                                                                                           \
    e = cudaFuncSetAttribute(build_kernel<M, LN, X>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    if (e != cudaSuccess) return e;                                                                              \
    build_kernel<M, LN, X><<<(unsigned)blocks, threads, smem, s>>>(bp);                                          \
    count_launch();                                                                                              \
  } while (0)
#define BSK_LAUNCH_BUILD(M)                                   \
  do {                                                        \
    if (logn == 10 && parity) BSK_LAUNCH_BUILD3(M, 10, true); \
    else if (logn == 10) BSK_LAUNCH_BUILD3(M, 10, false);     \
    else if (logn == 12) BSK_LAUNCH_BUILD3(M, 12, false);     \
    else if (parity) BSK_LAUNCH_BUILD3(M, 0, true);           \
    else BSK_LAUNCH_BUILD3(M, 0, false);                      \
  } while (0)
  switch (mode) {
    case kPiSeeded: BSK_LAUNCH_BUILD(kPiSeeded); break;
    case kPiSmem16: BSK_LAUNCH_BUILD(kPiSmem16); break;
    case kPiCache16: BSK_LAUNCH_BUILD(kPiCache16); break;
    case kPiCache32: BSK_LAUNCH_BUILD(kPiCache32); break;
    default: BSK_LAUNCH_BUILD(kPiGlobal); break;
  }
#undef BSK_LAUNCH_BUILD
#undef BSK_LAUNCH_BUILD3
  return cudaGetLastError();
}

// ------------------------------------------------------------- one-hot ----
// Categorical extension: label codes [n][c] -> the one-hot CSR that K1
// sketches: indptr[r] = r*c, indices[r*c+k] = offsets[k] + codes[r][k]. A code outside
// [0, offsets[k+1]-offsets[k]) or an index >= 2^31 latches kStatusIndex (the entry is then
// offsets[k], so the CSR stays well formed).
__global__ void onehot_kernel(const int32_t* __restrict__ codes, uint64_t n, uint32_t c,
                              const int64_t* __restrict__ offsets, int64_t* __restrict__ indptr,
                              int32_t* __restrict__ indices, unsigned int* status) {
  unsigned bad = 0;
  const uint64_t total = n * c;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = e / c;
    const uint32_t k = (uint32_t)(e - r * c);
    const int64_t o = __ldg(offsets + k), m = __ldg(offsets + k + 1) - o;
    const int64_t v = __ldg(codes + e);
    int64_t idx = o + v;
    if (v < 0 || v >= m || idx > 0x7fffffffll || o < 0) { bad = 1; idx = o >= 0 && o <= 0x7fffffffll ? o : 0; }
    indices[e] = (int32_t)idx;
    if (k == 0) indptr[r] = (int64_t)(r * c);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) indptr[n] = (int64_t)(n * c);
  if (bad) latch(status, kStatusIndex);
}

cudaError_t launch_onehot(const int32_t* codes, uint64_t n, uint32_t c, const int64_t* offsets, int64_t* indptr,
                          int32_t* indices, cudaStream_t s) {
  const uint64_t total = n * c;
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, (uint64_t)num_sms() * 8));
  onehot_kernel<<<(unsigned)blocks, 256, 0, s>>>(codes, n, c, offsets, indptr, indices, status_ptr());
  count_launch();
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
