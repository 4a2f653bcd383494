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
// Sketch construction, v4. A warp owns a tile of RW <= 32 consecutive rows (lane l holds
// row l's [start, end)); the tile's nonzeros are one contiguous span of `indices`, which
// the warp streams as coalesced 16-byte quads (lane l: elements 4l..4l+3 and
// 128+4l..128+4l+3 of each 256-element iteration, next iteration prefetched).
//
// Row of an element without a search: rows are compacted to the NONEMPTY ones (their
// end offsets are distinct), and for each 2048-element chunk of the span the warp builds
// in shared memory a bitmap P with bit q set iff a nonempty row ends at chunk offset q,
// plus, per 32-bit word w of P, B[w] = the tile address of the row live at the word's
// start. The row of element q is then B[q/32] + popc(P[q/32] & mask_le(q)) rows on — an
// AND, a POPC and an IMAD per element, no loop and no divergence.
//
// pi(i) comes from (MODE):
//   kPiSeeded  : the splitmix64 recipe evaluated in registers (no table);
//   kPiSmem16  : the whole table as uint16 in shared memory (d small);
//   kPiCache16 : a direct-mapped shared-memory cache of the table, 64K uint16 slots
//                entry = (i >> 16) << vb | pi(i), prefilled with slot s <- pi(s);
//   kPiCache32 : the same with 32K uint32 slots when tag + value need more than 16 bits;
//   kPiGlobal  : read-only L1/L2 gather.
// Since pi is read-only every entry ever written is correct, so racing fills are benign.
// Bits are OR-ed into the warp's shared tile (RED.OR), and the tile is written once with
// coalesced streaming stores — every output word exactly once, no memset.
enum PiMode { kPiSeeded = 0, kPiSmem16 = 1, kPiCache16 = 2, kPiCache32 = 3, kPiGlobal = 4 };

constexpr int kIter = 256;                      // elements per warp iteration (2 quads per lane)
constexpr int kChunk = 2048;                    // elements per row-boundary bitmap chunk
constexpr int kChunkWords = kChunk / 32;        // 64 {P, B} pairs
constexpr uint32_t kMetaBytes = kChunkWords * 8 + 32 * 4;   // {P,B} pairs + compact row index
constexpr uint32_t kCache16Slots = 65536;       // 128 KB
constexpr uint32_t kCache32Slots = 32768;       // 128 KB
constexpr uint32_t kFull = 0xffffffffu;

struct BuildParams {
  const uint32_t* pi;
  uint64_t seed;
  ModN mn;
  const int64_t* indptr;
  const int32_t* indices;
  uint64_t n;
  uint32_t* out;
  uint32_t d, W, RW;
  uint32_t pi_bytes;     // shared bytes before the per-warp regions
  uint32_t warp_bytes;   // per-warp region: meta (kMetaBytes), cp.async ring, RW x W tile
  uint32_t vb;           // cache: value bits
  unsigned int* status;
};

// 32-bit shared-memory accessors: shared addresses stay in one register, no generic
// conversion per access. Volatile keeps them ordered among themselves; none clobbers
// "memory", so global loads (indices, pi) schedule freely around them.
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
__device__ __forceinline__ void red_or_shared(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void red_xor_shared(uint32_t a, uint32_t v) {
  asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(a), "r"(v));
}
// A sketch bit: OR (BinSketch) or XOR (BCS parity buckets).
template <bool XOR>
__device__ __forceinline__ void put_bit(uint32_t a, uint32_t v) {
  if (XOR) red_xor_shared(a, v); else red_or_shared(a, v);
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

// pi(i) for a power-of-two N; seed1 = seed + gamma, so seed + (i+1)*gamma = seed1 + i*gamma.
// Only the low log2(N) bits of the finalizer are needed. Pipe balance (ncu): every IMAD
// form runs on the FMA-heavy pipe at half the ALU-pipe rate, so the xor-shifts stay on the
// ALU (SHF + LOP3) and the three 64-bit multiplies are the only IMADs. Returns x, the low
// finalizer word before masking (j = x & (N-1); x & 31 = j & 31 when N >= 32).
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

// Per-mode launch shape. 24 warps per SM (<= 85 registers): cache / shared-table modes as
// one 768-thread block (the cache shared by all warps), the others as two 384-thread
// blocks. kStages: depth of each warp's cp.async ring of index quads (kStages-1 iterations
// of 1 KB in flight per warp: 72 KB per SM for the seeded / global modes).
template <int MODE>
struct BuildCfg {
  static constexpr bool kSmemPi = !(MODE == kPiSeeded || MODE == kPiGlobal);
  static constexpr int kThreads = kSmemPi ? 512 : 256;     // per block
  static constexpr int kBlocks = kSmemPi ? 1 : 3;          // per SM (launch bound)
  static constexpr int kStages = 2;                        // ring depth
  static constexpr int kStage = kSmemPi ? 256 : 512;       // elements per ring stage
  static constexpr int kStageBytes = kStage * 4;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K)); }

// LOGN > 0: N = 2^LOGN >= 32 compiled in (sketch-word and row shifts become immediates);
// LOGN = 0: any N. XOR: BCS parity sketch (bits toggled instead of set).
template <int MODE, int LOGN, bool VEC, bool XOR>
__global__ void __launch_bounds__(BuildCfg<MODE>::kThreads, BuildCfg<MODE>::kBlocks)
build_kernel(const BuildParams p) {
  constexpr int NS = BuildCfg<MODE>::kStages;
  constexpr int kStage = BuildCfg<MODE>::kStage, kStageBytes = BuildCfg<MODE>::kStageBytes;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const uint32_t N = p.mn.N, W = p.W, RW = p.RW, Wb = 4 * W, d = p.d;
  const uint32_t pi_a = smem_u32(smem);
  // per-warp region: {P,B} pairs | compact row index [32] | ring [NS][kStageBytes] | tile [RW+2][W]
  const uint32_t meta_a = pi_a + p.pi_bytes + (uint32_t)warp * p.warp_bytes;
  const uint32_t crow_a = meta_a + kChunkWords * 8;
  const uint32_t ring_a = meta_a + kMetaBytes;
  const uint32_t tile_a = ring_a + NS * kStageBytes;
  const uint64_t seed1 = p.seed + 0x9E3779B97F4A7C15ULL;
  constexpr uint32_t kSlots = MODE == kPiCache16 ? kCache16Slots : kCache32Slots;
  constexpr uint32_t kSlotBits = MODE == kPiCache16 ? 16 : 15;
  const uint32_t vb = p.vb, vmask = (1u << vb) - 1u;
  constexpr bool POW2 = LOGN > 0;
  constexpr uint32_t wmask = POW2 ? ((1u << LOGN) - 1u) & ~31u : 0u;   // j & wmask = 32 * (j / 32)
  constexpr uint32_t wsh = POW2 ? LOGN - 3 : 0;                         // log2(4W)

  unsigned bad = 0;
  uint32_t maxj = 0;
  if (MODE == kPiSmem16) {
    for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
      uint32_t v = __ldg(p.pi + i);
      maxj = max(maxj, v);
      sts_u16(pi_a + 2 * i, min(v, N - 1));
    }
  } else if (MODE == kPiCache16 || MODE == kPiCache32) {
    for (uint32_t s = threadIdx.x; s < kSlots; s += blockDim.x) {
      uint32_t v = s < d ? __ldg(p.pi + s) : 0u;
      maxj = max(maxj, v);
      v = min(v, N - 1);
      if (MODE == kPiCache16) sts_u16(pi_a + 2 * s, v); else sts_u32(pi_a + 4 * s, v);
    }
  }
  if (BuildCfg<MODE>::kSmemPi) __syncthreads();

  // lane constants: masks selecting chunk-word bits <= element (4*lane + k) mod 32
  uint32_t mle[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) mle[k] = (2u << ((4 * lane + k) & 31)) - 1u;
  const uint32_t lmlt = lanemask_lt();
  uint32_t maxidx = 0;

  const uint64_t ntiles = (p.n + RW - 1) / RW;
  const uint64_t tstride = (uint64_t)gridDim.x * nwarps;
  uint64_t t = (uint64_t)blockIdx.x * nwarps + warp;

  // Row tile tt: lane l < rows holds row r0+l's [s, e).
  auto tile_rows = [&](uint64_t tt) -> uint32_t {
    return tt < ntiles ? (uint32_t)min((uint64_t)RW, p.n - tt * RW) : 0u;
  };
  auto load_info = [&](uint64_t tt, int64_t& s_, int64_t& e_) {
    s_ = 0; e_ = 0;
    if ((uint32_t)lane < tile_rows(tt)) {
      s_ = __ldg(p.indptr + tt * RW + lane);
      e_ = __ldg(p.indptr + tt * RW + lane + 1);
    }
  };
  // Streamed span of tile tt (warp-collective): [base, base + span) of `indices`, base
  // 16-B aligned when VEC (lo = E0 - base head elements belong to earlier rows). span = 0
  // for invalid tiles (bad indptr: rows stay zero) and for tiles of > 2^31 nonzeros
  // (handled by a per-row loop).
  auto span_of = [&](uint64_t tt, int64_t s_, int64_t e_, int64_t& base_, int& lo_) -> int {
    const uint32_t rows_ = tile_rows(tt);
    base_ = 0; lo_ = 0;
    if (rows_ == 0) return 0;
    const int64_t E0 = __shfl_sync(kFull, s_, 0), E1 = __shfl_sync(kFull, e_, rows_ - 1);
    const bool ok = __all_sync(kFull, (uint32_t)lane >= rows_ || s_ <= e_) && E0 >= 0;
    base_ = VEC ? (E0 & ~(int64_t)3) : E0;
    lo_ = (int)(E0 - base_);
    return (ok && E1 - base_ <= 0x7fff0000ll) ? (int)(E1 - base_) : 0;
  };

  int64_t cs, ce, ns, nE;            // current / next tile's per-lane row bounds
  load_info(t, cs, ce);
  load_info(t + tstride, ns, nE);

  // ---- producer: cp.async of 256-element iterations into the ring, NS-1 ahead, running
  // through the current tile and into the next one; group g holds stream position g.
  // Bytes past span are zero-filled (src-size); the < 4 head elements before E0 are zeroed
  // by the consumer. Out-of-range elements then land in the tile's virtual rows.
  int ptile = 0, pwb = 0, pspan, plo;   // ptile: 0 = current tile, 1 = next tile
  int64_t pbase;
  const int32_t* psrc;                  // indices + pbase + pwb + 4*lane
  uint32_t kp = 0, kc = 0;              // positions issued / consumed
  uint32_t pslot = ring_a + 16 * lane;  // ring slot of position kp (this lane's bytes)
  pspan = span_of(t, cs, ce, pbase, plo);
  psrc = p.indices + pbase + 4 * lane;
  auto issue = [&]() {
    while (pwb >= pspan) {
      if (ptile == 1 || t + tstride >= ntiles) return;   // wait for the consumer
      ptile = 1; pwb = 0;
      pspan = span_of(t + tstride, ns, nE, pbase, plo);
      psrc = p.indices + pbase + 4 * lane;
    }
    if (VEC && pwb + kStage <= pspan) {   // whole stage in range
#pragma unroll
      for (int h = 0; h < kStage / 128; ++h) cp_async16(pslot + 512 * h, psrc + 128 * h, 16u);
    } else
#pragma unroll
    for (int h = 0; h < kStage / 128; ++h) {
      const int rem = pspan - (pwb + 128 * h + 4 * lane);   // elements left from this quad on
      if (VEC) {
        cp_async16(pslot + 512 * h, psrc + 128 * h, (uint32_t)min(max(rem, 0), 4) * 4u);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) cp_async4(pslot + 512 * h + 4 * k, psrc + 128 * h + k, k < rem ? 4u : 0u);
      }
    }
    cp_async_commit();
    ++kp;
    pwb += kStage;
    psrc += kStage;
    pslot = (kp % NS == 0) ? pslot - (NS - 1) * kStageBytes : pslot + kStageBytes;
  };
  auto wait_pos = [&]() {   // wait until position kc has landed (kp - kc - 1 newer groups may stay pending)
    if (kp - kc - 1 >= NS - 1) cp_async_wait<NS - 1>();
    else cp_async_wait<0>();   // fewer newer groups (producer blocked at a tile end): drain
  };
  for (int i = 0; i < NS - 1; ++i) issue();
  uint32_t cslot = ring_a + 16 * lane;  // ring slot of position kc

  // Tile rows in shared memory: row 0 = virtual head row (elements before E0 in the first
  // aligned quad), rows 1..nne = the tile's nonempty rows in order, row nne+1 = virtual
  // tail row (zero-filled elements past E1). The virtual rows are never stored.
  for (; t < ntiles; t += tstride) {
    const uint64_t r0 = t * RW;
    const uint32_t rows = tile_rows(t);
    const bool has = (uint32_t)lane < rows;
    const int64_t s = cs, e = ce;
    const int64_t E0 = __shfl_sync(kFull, s, 0);
    const int64_t E1 = __shfl_sync(kFull, e, rows - 1);
    const bool ok = __all_sync(kFull, !has || s <= e) && E0 >= 0;
    const uint32_t nw = rows * W;
    uint32_t* dst = p.out + r0 * W;
    const bool ne = ok && has && e > s;
    const uint32_t NE = __ballot_sync(kFull, ne);
    const uint32_t crow_l = __popc(NE & lmlt) + 1u;      // tile row of this lane's row
    if (!ok) bad = 1;                // decreasing / negative indptr: rows stay zero, latched
    for (uint32_t w = 4 * lane; w < (rows + 2) * W; w += 128) sts_v4(tile_a + 4 * w, 0, 0, 0, 0);   // padded to 16 B
    if (has) sts_u32(crow_a + 4 * lane, ne ? crow_l : kFull);
    const int64_t base = VEC ? (E0 & ~(int64_t)3) : E0;
    __syncwarp();
    if (ok && E1 - base > 0x7fff0000ll) {
      // > 2^31 nonzeros in one tile: per-row loop with 64-bit offsets (correct, not fast)
      for (uint32_t r = 0; r < rows; ++r) {
        const int64_t rs = __shfl_sync(kFull, s, r), re = __shfl_sync(kFull, e, r);
        const uint32_t ra = tile_a + __shfl_sync(kFull, crow_l, r) * Wb;
        for (int64_t q = rs + lane; q < re; q += 32) {
          const uint32_t x = (uint32_t)p.indices[q];
          maxidx = max(maxidx, x);
          uint32_t jj;
          if (MODE == kPiSeeded) {
            jj = pi_seeded(p.seed, (uint64_t)x, p.mn);
          } else {
            jj = __ldg(p.pi + min(x, d - 1));
            maxj = max(maxj, jj);
            jj = min(jj, N - 1);
          }
          put_bit<XOR>(ra + ((jj >> 5) << 2), 1u << (jj & 31u));
        }
      }
    } else if (ok) {
      const int span = (int)(E1 - base);
      const int lo = (int)(E0 - base);
      const int pe = ne ? (int)(e - base) : -1;   // end offset of this lane's (nonempty) row
      for (int ws = 0; ws < span; ws += kStage) {
        issue();
        wait_pos();
        const uint32_t stage = cslot;
        ++kc;
        cslot = (kc % NS == 0) ? cslot - (NS - 1) * kStageBytes : cslot + kStageBytes;
        if ((ws & (kChunk - 1)) == 0) {
          // row-boundary bitmap for [ws, ws + kChunk): bit q set iff a row (virtual head
          // row included) ends at offset ws + q; B = tile row address at each word start
          sts_v4(meta_a + 16 * lane, 0, 0, 0, 0);
          __syncwarp();
          const int q = pe - ws;
          if (ne && q > 0 && q < kChunk) red_or_shared(meta_a + 8 * (uint32_t)(q >> 5), 1u << (q & 31));
          if (ws == 0 && lo > 0 && lane == 0) {
            red_or_shared(meta_a, 1u << lo);
            // head elements (earlier rows' data, before E0) -> index 0 (virtual head row)
            const uint4 h4 = lds_v4(stage);
            sts_v4(stage, 0u, lo > 1 ? 0u : h4.y, lo > 2 ? 0u : h4.z, h4.w);
          }
          const uint32_t before = __popc(__ballot_sync(kFull, ne && pe <= ws)) + (lo <= ws ? 1u : 0u);
          __syncwarp();
          const uint4 pr = lds_v4(meta_a + 16 * lane);
          const uint32_t c0 = __popc(pr.x), c = c0 + __popc(pr.z);
          uint32_t incl = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
          }
          const uint32_t b0 = tile_a + (before + incl - c) * Wb;
          sts_v4(meta_a + 16 * lane, pr.x, b0, pr.z, b0 + c0 * Wb);
          __syncwarp();
        }
        // one 256-element half of the stage; FULL: the whole stage lies inside the span
        auto half_step = [&](const int half, auto full_tag) {
          constexpr bool FULL = decltype(full_tag)::value;
          const int wb = ws + kIter * half;
          const uint4 qa = lds_v4(stage + 1024 * half), qb = lds_v4(stage + 1024 * half + 512);
          const uint32_t cur[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
          const uint32_t wq = (uint32_t)((wb & (kChunk - 1)) >> 5) + (uint32_t)(lane >> 3);
          uint32_t addr[8], j[8];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint2 pb = lds_v2(meta_a + 8 * (wq + 4 * h));
#pragma unroll
            for (int k = 0; k < 4; ++k)
              addr[4 * h + k] = pb.y + (POW2 ? ((uint32_t)__popc(pb.x & mle[k]) << wsh)
                                            : (uint32_t)__popc(pb.x & mle[k]) * Wb);
          }
          maxidx = __vimax3_u32(maxidx, __vimax3_u32(cur[0], cur[1], cur[2]),
                                __vimax3_u32(__vimax3_u32(cur[3], cur[4], cur[5]), cur[6], cur[7]));
          uint32_t bit[8];   // 1 << (j & 31)
          if (MODE == kPiSeeded && POW2) {
            // word offset from j & ~31 (LEA.HI); x & 31 = j & 31 since N >= 32
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const uint32_t x = pi_pow2_raw(seed1, cur[u]);
              j[u] = x & wmask;                         // = (j >> 5) << 5
              bit[u] = bit_of(x);
            }
          } else if (MODE == kPiSeeded) {
#pragma unroll
            for (int u = 0; u < 8; ++u) j[u] = pi_seeded(p.seed, (uint64_t)cur[u], p.mn);
          } else if (MODE == kPiSmem16) {
#pragma unroll
            for (int u = 0; u < 8; ++u) j[u] = lds_u16(pi_a + 2 * min(cur[u], d - 1));
          } else if (MODE == kPiGlobal) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const uint32_t g = __ldg(p.pi + min(cur[u], d - 1));
              maxj = max(maxj, g);
              j[u] = min(g, N - 1);
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
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (miss[u]) {
                maxj = max(maxj, j[u]);
                j[u] = min(j[u], N - 1);
                const uint32_t ent = ((x[u] >> kSlotBits) << vb) | j[u];
                if (MODE == kPiCache16) sts_u16(pi_a + 2 * slot_[u], ent); else sts_u32(pi_a + 4 * slot_[u], ent);
              }
            }
          }
          if (!(MODE == kPiSeeded && POW2)) {
#pragma unroll
            for (int u = 0; u < 8; ++u) { bit[u] = bit_of(j[u]); j[u] &= ~31u; }
          }
          if (FULL) {
#pragma unroll
            for (int u = 0; u < 8; ++u) put_bit<XOR>(addr[u] + (j[u] >> 3), bit[u]);
          } else {   // tile tail: skip the zero-filled elements (they would all hit one word)
            const int rem = span - wb;
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (128 * (u >> 2) + 4 * lane + (u & 3) < rem) put_bit<XOR>(addr[u] + (j[u] >> 3), bit[u]);
          }
        };
        if (ws + kStage <= span) {
#pragma unroll
          for (int h = 0; h < kStage / kIter; ++h) half_step(h, std::true_type{});
        } else {
#pragma unroll 1
          for (int h = 0; h < kStage / kIter; ++h)
            if (ws + kIter * h < span) half_step(h, std::false_type{});
        }
      }
    }
    __syncwarp();
    // write the tile: rows in order, empty rows as zeros; every output word exactly once
    const uint32_t all = rows == 32 ? kFull : ((1u << rows) - 1u);
    if (NE == all && (W & 3u) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 15u) == 0) {
      for (uint32_t w = 4 * lane; w < nw; w += 128) {
        const uint4 v = lds_v4(tile_a + Wb + 4 * w);   // tile rows 1..rows
        __stcs(reinterpret_cast<uint4*>(dst + w), v);
      }
    } else {
      for (uint32_t w = lane; w < nw; w += 32) {
        const uint32_t r = w / W;
        const uint32_t cr = lds_u32(crow_a + 4 * r);
        __stcs(dst + w, cr == kFull ? 0u : lds_u32(tile_a + 4 * (cr * W + (w - r * W))));
      }
    }
    __syncwarp();
    // advance: next becomes current; the producer follows (it is on the next tile, or done
    // with this one and must restart on the new current tile)
    cs = ns; ce = nE;
    load_info(t + 2 * tstride, ns, nE);
    if (ptile == 1) {
      ptile = 0;
    } else {
      pwb = 0;
      pspan = span_of(t + tstride, cs, ce, pbase, plo);
      psrc = p.indices + pbase + 4 * lane;
    }
  }
  cp_async_wait<0>();
  if (maxidx >= d || maxj >= N) bad = 1;
  if (__any_sync(kFull, bad != 0) && lane == 0) latch(p.status, kStatusIndex);
}

// Fallback for very wide sketches (one row's W words do not fit a warp's share of
// shared memory): rows zeroed by cudaMemsetAsync, then global atomicOr (atomicXor: BCS).
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
  const uint32_t W = (N + 31) / 32;
  const ModN mn = make_modn(N);
  unsigned int* st = status_ptr();
  const int sms = num_sms();
  int dev = 0, smem_optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t optin = (size_t)smem_optin;

  const uint32_t vb = bits_for(N - 1);
  const uint32_t dbits = bits_for(d - 1);
  const bool c16 = N <= 65536 && (dbits > 16 ? dbits - 16 : 0) + vb <= 16;
  const bool c32 = (dbits > 15 ? dbits - 15 : 0) + vb <= 32;
  const size_t smem16_bytes = ((d * 2 + 15) / 16) * 16;
  int mode = kPiGlobal;
  if (pi == nullptr) mode = kPiSeeded;
  else if (N <= 65536 && smem16_bytes <= 100 * 1024) mode = kPiSmem16;
  else if (c16) mode = kPiCache16;
  else if (c32) mode = kPiCache32;
  // Experiment knob (ncu A/B of the pi source): BINSKETCH_BUILD_MODE=global|cache|smem16.
  if (const char* f = pi != nullptr ? std::getenv("BINSKETCH_BUILD_MODE") : nullptr) {
    if (!std::strcmp(f, "global")) mode = kPiGlobal;
    if (!std::strcmp(f, "cache")) mode = c16 ? kPiCache16 : (c32 ? kPiCache32 : mode);
    if (!std::strcmp(f, "cache32") && c32) mode = kPiCache32;
    if (!std::strcmp(f, "smem16") && N <= 65536 && smem16_bytes + 64 * 1024 <= optin) mode = kPiSmem16;
  }
  // Shared memory per warp: meta + ring (kStages KB) + an RW x W tile, RW <= 32 rows.
  auto rows_fit = [&](size_t per_warp, int stages, int stage_bytes) -> uint32_t {
    const size_t fixed = kMetaBytes + (size_t)stages * stage_bytes + 16 + 8 * (size_t)W;   // + 2 virtual rows
    return per_warp > fixed ? (uint32_t)std::min<size_t>(32, (per_warp - fixed) / (4 * (size_t)W)) : 0u;
  };
  bool smem_pi = mode == kPiSmem16 || mode == kPiCache16 || mode == kPiCache32;
  uint32_t pi_bytes = mode == kPiSmem16 ? (uint32_t)smem16_bytes : (smem_pi ? 128u * 1024u : 0u);
  int threads = smem_pi ? BuildCfg<kPiCache16>::kThreads : BuildCfg<kPiSeeded>::kThreads;
  int stages = smem_pi ? BuildCfg<kPiCache16>::kStages : BuildCfg<kPiSeeded>::kStages;
  int stage_bytes = smem_pi ? BuildCfg<kPiCache16>::kStageBytes : BuildCfg<kPiSeeded>::kStageBytes;
  int bps = smem_pi ? BuildCfg<kPiCache16>::kBlocks : BuildCfg<kPiSeeded>::kBlocks;
  size_t budget = optin / bps;
  uint32_t RW = rows_fit(budget > pi_bytes ? (budget - pi_bytes) / (threads / 32) : 0, stages, stage_bytes);
  if (RW == 0 && smem_pi) {       // wide sketches: fall back to the global-gather variant
    mode = kPiGlobal; smem_pi = false; pi_bytes = 0;
    threads = BuildCfg<kPiGlobal>::kThreads; stages = BuildCfg<kPiGlobal>::kStages;
    stage_bytes = BuildCfg<kPiGlobal>::kStageBytes;
    bps = BuildCfg<kPiGlobal>::kBlocks;
    budget = optin / bps;
    RW = rows_fit(budget / (threads / 32), stages, stage_bytes);
  }
  if (RW == 0) {
    cudaError_t e = cudaMemsetAsync(out, 0, n * (size_t)W * 4, s);
    if (e != cudaSuccess) return e;
    build_wide_kernel<<<sms * 8, 256, 0, s>>>(pi, seed, d, mn, pi == nullptr, parity, indptr, indices, n, out, W, st);
    count_launch();
    return cudaGetLastError();
  }
  BuildParams bp;
  bp.pi = pi; bp.seed = seed; bp.mn = mn; bp.indptr = indptr; bp.indices = indices; bp.n = n; bp.out = out;
  bp.d = (uint32_t)d; bp.W = W; bp.RW = RW; bp.vb = vb; bp.status = st;
  bp.pi_bytes = smem_pi ? pi_bytes : 0u;
  bp.warp_bytes = kMetaBytes + (uint32_t)(stages * stage_bytes) + (uint32_t)((((size_t)(RW + 2) * W * 4) + 15) / 16 * 16);
  const size_t smem = bp.pi_bytes + (size_t)bp.warp_bytes * (threads / 32);
  const uint64_t ntiles = (n + RW - 1) / RW;
  const uint64_t want = (ntiles + (threads / 32) - 1) / (threads / 32);
  const int fit = (int)std::max<size_t>(1, std::min<size_t>((size_t)bps, optin / std::max<size_t>(smem, 1)));
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms * fit));
  // compiled-in sketch widths: the configs' N = 1024 (W = 32) and 4096 (W = 128); the BCS
  // parity variant is instantiated for the generic width only
  const int logn = parity ? 0 : (N == 1024 ? 10 : (N == 4096 ? 12 : 0));
  const bool vec = (reinterpret_cast<uintptr_t>(indices) & 15u) == 0;
  cudaError_t e = cudaSuccess;
#define BSK_LAUNCH_BUILD4(M, LN, V, X)                                                                           \
  do {                                                                                                           \
    e = cudaFuncSetAttribute(build_kernel<M, LN, V, X>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                              \
    build_kernel<M, LN, V, X><<<(unsigned)blocks, threads, smem, s>>>(bp);                                       \
    count_launch();                                                                                              \
  } while (0)
#define BSK_LAUNCH_BUILD3(M, LN, V)                       \
  do {                                                    \
    if (LN == 0 && parity) BSK_LAUNCH_BUILD4(M, 0, V, true); \
    else BSK_LAUNCH_BUILD4(M, LN, V, false);              \
  } while (0)
#define BSK_LAUNCH_BUILD2(M, LN)                 \
  do {                                           \
    if (vec) BSK_LAUNCH_BUILD3(M, LN, true);     \
    else BSK_LAUNCH_BUILD3(M, LN, false);        \
  } while (0)
#define BSK_LAUNCH_BUILD(M)                                  \
  do {                                                       \
    if (logn == 10) BSK_LAUNCH_BUILD2(M, 10);                \
    else if (logn == 12) BSK_LAUNCH_BUILD2(M, 12);           \
    else BSK_LAUNCH_BUILD2(M, 0);                            \
  } while (0)
  switch (mode) {
    case kPiSeeded: BSK_LAUNCH_BUILD(kPiSeeded); break;
    case kPiSmem16: BSK_LAUNCH_BUILD(kPiSmem16); break;
    case kPiCache16: BSK_LAUNCH_BUILD(kPiCache16); break;
    case kPiCache32: BSK_LAUNCH_BUILD(kPiCache32); break;
    default: BSK_LAUNCH_BUILD(kPiGlobal); break;
  }
#undef BSK_LAUNCH_BUILD
#undef BSK_LAUNCH_BUILD2
#undef BSK_LAUNCH_BUILD3
#undef BSK_LAUNCH_BUILD4
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
