// tc.cu — all-pairs AND-popcount on the 5th-generation tensor cores (sm_100a).
//
// Algorithm 1 line 2 needs n_{as,bs} = |a_s AND b_s| for every
// (a, b) pair. With every sketch bit widened to a {0,1} byte, that count is the
// exact integer dot product of two 0/1 vectors:
//     |a_s AND b_s| = sum_k a8[k] * b8[k]          (products are 0/1, int32 sums)
// so the all-pairs table is an unsigned-int8 GEMM  C[na][nb] = A8 * B8^T  that
// tcgen05.mma kind::i8 evaluates bit-exactly.
//
// K10 (this file):
//   expand_kernel   uint32 sketch words -> {0,1} bytes, rows padded to Kp (a
//                   multiple of 128) with zeros (zero bytes add nothing).
//   tc_pairs_kernel persistent, warp-specialised: warp 0 = TMA producer (one
//                   lane), warp 1 = MMA issuer (one lane; also owns TMEM),
//                   warps 2..5 = epilogue (one TMEM lane = one A row each).
//                   128 x 256 output tile per CTA; K streamed in 128-byte
//                   stages (A 16 KB + B 32 KB, 128B-swizzled by TMA) through a
//                   4-deep mbarrier ring; accumulators double-buffered in TMEM
//                   (2 x 256 int32 columns) so the epilogue of tile t overlaps
//                   the MMAs of tile t+1. With CG = 2 (long K) a CTA pair runs
//                   cta_group::2 MMAs over a 256 x 256 tile, each CTA staging half
//                   of the B rows. The fused top-k's per-tile db metadata comes
//                   through a producer-filled bulk-copy ring.
#include <cuda.h>
#include <type_traits>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "bsk_estimator.cuh"
#include "bsk_internal.cuh"

namespace bsk {

// ------------------------------------------------------------ PTX wrappers ---
namespace tc {

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
#ifdef BSK_MBAR_NOHINT
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(0x100000u)   // suspend-time hint (ns): sleep, do not spin
        : "memory");
#endif
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t x, int32_t y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
// 1-D bulk copy global -> shared (16-B aligned, size a multiple of 16), completing on `bar`
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// one lane of a converged warp (the same lane in every call)
__device__ __forceinline__ bool elect_one() {
  uint32_t r;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(r));
  return r != 0u;
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand tile of 128-byte rows, 128B-swizzled (as TMA writes it): 8-row
// atoms of 1 KB, SBO = 1024 B; descriptor version 1 (sm_100), layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;              // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;    // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1u << 46;              // version
  d |= (uint64_t)2u << 61;              // SWIZZLE_128B
  return d;
}

// D[tmem] (+)= A[smem] * B[smem]^T, unsigned int8 -> int32, M=128 x N=256 x K=32.
__device__ __forceinline__ void mma_u8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
// D[tmem] (+)= A[tmem] * B[smem]^T (A from tensor memory: lane = row, 4 K-bytes per column).
__device__ __forceinline__ void mma_u8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum));
}
// 32 lanes x 32 consecutive columns <- 32 registers per thread, then wait for the stores.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
      ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
        "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// ---- CTA pair (cta_group::2): one MMA over both SMs' shared memory, M = 256 ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// wait with cluster-scope acquire (the phase was completed by the peer CTA, data written remotely)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(0x100000u)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void st_cluster_u64(uint32_t cluster_addr, uint64_t v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(cluster_addr), "l"(v) : "memory");
}
// TMA into this CTA's shared memory, completing bytes on the pair leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int32_t x, int32_t y,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void mma_u8_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
// arrive on the barrier at this offset in every CTA of `mask` when the pair's MMAs complete
__device__ __forceinline__ void commit_pair(uint32_t bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
               "h"(mask)
               : "memory");
}

// 32 lanes x 32 consecutive columns of 32-bit TMEM -> 32 registers per thread. The wait
// is in the same asm statement so no output register is read before the load lands.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

// 32 lanes x 8 consecutive columns.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
      : "r"(taddr)
      : "memory");
}

// Split form for software pipelining: issue a load without waiting, and a wait that
// names the destination registers as in/out operands (so no use is scheduled before it).
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
      : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
        "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
        "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
        "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
      :
      : "memory");
}


}  // namespace tc

// Checked build (-DBSK_CHECKED, a dev library): index invariants of the top-k epilogue's shared
// structures (heap slots, survivor queue, owner lanes, metadata columns) trap when violated.
#ifdef BSK_CHECKED
#define BSK_ASSERT(c) do { if (!(c)) __trap(); } while (0)
#else
#define BSK_ASSERT(c) do {} while (0)
#endif
#ifndef BSK_PMIN_FAST
#define BSK_PMIN_FAST 1   // fused top-k: tile bound start by MUFU exp, IP refinement on the hoisted sum (A/B: DESIGN.md K10)
#endif
#ifndef BSK_TOPK_STRICT
#define BSK_TOPK_STRICT 1 // fused top-k (IP): exact strict bound on single-popcount tiles where no tie can enter
#endif
#ifndef BSK_TOPK_QCAP
#define BSK_TOPK_QCAP 256 // fused top-k: per-warp survivor queue entries
#endif
#ifdef BSK_TOPK_PROF
#define BSK_T0(v) const long long v = clock64()
#define BSK_TADD(slot, t0) (pacc[(slot) - 6] += (unsigned long long)(clock64() - (t0)))
#else
#define BSK_T0(v)
#define BSK_TADD(slot, t0)
#endif
#if defined(BSK_TOPK_STATS) || defined(BSK_TOPK_PROF)
// dev instrumentation (never in the product build): warp-tiles, all-rows-skippable warp-tiles,
// passing chunks, survivors, direct-path warp-tiles, candidates; BSK_TOPK_PROF adds clock64
// cycle sums: [6] epilogue waits tfull, [7] filter, [8] scoring, [9] tile setup (metadata wait +
// bound), [10] MMA waits tempty, [11] MMA waits full, [12] producer waits empty, [13] epilogue
// item loop, [14] MMA role total
__device__ unsigned long long g_tkstats[16];
}  // namespace bsk
extern "C" int bsk_topk_stats(unsigned long long* host8) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host8, bsk::g_tkstats, 128);
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(bsk::g_tkstats, z, 128);
  return 0;
}
namespace bsk {
#endif

// ------------------------------------------------------------- expansion ---
// out[r][b] = bit b of row r (LSB-first words), b < 32W; zero for 32W <= b < Kp.
__global__ void expand_kernel(const uint32_t* __restrict__ sk, uint64_t n, uint32_t W, uint32_t Kp,
                              const int32_t* __restrict__ perm, uint8_t* __restrict__ out) {
  const uint32_t chunks = Kp / 32;   // one 32-byte chunk per sketch word
  const uint64_t total = n * chunks;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / chunks;
    const uint32_t c = (uint32_t)(i - r * chunks);
    const uint64_t src = perm ? (uint64_t)__ldg(perm + r) : r;   // row r of the output = sketch src
    const uint32_t w = c < W ? __ldg(sk + src * W + c) : 0u;
    uint32_t b[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t nib = (w >> (4 * q)) & 0xFu;   // bytes {bit0, bit1, bit2, bit3} of this nibble
      b[q] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
    }
    uint4* o = reinterpret_cast<uint4*>(out + r * Kp + 32u * c);
    o[0] = make_uint4(b[0], b[1], b[2], b[3]);
    o[1] = make_uint4(b[4], b[5], b[6], b[7]);
  }
}

// ------------------------------------------------- db order for top-k ---
// Per-tile db metadata for the top-k epilogue: meta[i] = (|b_s|, original index) of B row i,
// padded to whole 256-row tiles with (0, -1), so the producer bulk-loads 2 KB per tile.
__global__ void tile_meta_kernel(const int32_t* __restrict__ pb, const int32_t* __restrict__ perm, uint64_t nb,
                                 uint64_t npad, int2* __restrict__ meta) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npad; i += (uint64_t)gridDim.x * blockDim.x)
    meta[i] = i < nb ? make_int2(__ldg(pb + i), perm ? __ldg(perm + i) : (int32_t)i) : make_int2(0, -1);
}

// Counting sort of the db rows by popcount (descending: bin N - pb; or ascending), so every 256-row
// tensor-core tile spans a narrow popcount range and the per-tile key bound is tight.
// Order inside a bin is arbitrary: the top-k result is the unique top-k under
// (key desc, original index asc), independent of processing order.
__global__ void pb_hist_kernel(const int32_t* __restrict__ pb, uint64_t n, uint32_t N, uint32_t desc,
                               uint32_t* __restrict__ bins) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = (uint32_t)__ldg(pb + i);
    atomicAdd(bins + (desc ? N - v : v), 1u);
  }
}

__global__ void pb_scan_kernel(uint32_t* __restrict__ bins, uint32_t nbins) {   // one block, exclusive, in place
  __shared__ uint32_t part[1024];
  const uint32_t t = threadIdx.x, per = (nbins + blockDim.x - 1) / blockDim.x;
  const uint32_t b0 = min(t * per, nbins), b1 = min(b0 + per, nbins);
  uint32_t sum = 0;
  for (uint32_t i = b0; i < b1; ++i) sum += bins[i];
  part[t] = sum;
  __syncthreads();
  for (uint32_t o = 1; o < blockDim.x; o <<= 1) {
    const uint32_t v = t >= o ? part[t - o] : 0u;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  uint32_t run = part[t] - sum;
  for (uint32_t i = b0; i < b1; ++i) { const uint32_t c = bins[i]; bins[i] = run; run += c; }
}

// Smallest original db index of each TN-row db tile (one block of TN threads per tile).
__global__ void tile_min_kernel(const int2* __restrict__ meta, int32_t* __restrict__ tmin) {
  __shared__ int32_t wm[8];
  const int2 e = meta[(uint64_t)blockIdx.x * blockDim.x + threadIdx.x];
  int32_t v = __reduce_min_sync(0xffffffffu, e.y < 0 ? 0x7fffffff : e.y);
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < blockDim.x / 32; ++w) v = min(v, wm[w]);
    tmin[blockIdx.x] = v;
  }
}
__global__ void pb_scatter_kernel(const int32_t* __restrict__ pb, uint64_t n, uint32_t N, uint32_t desc,
                                  uint32_t* __restrict__ cursor, int32_t* __restrict__ perm, int32_t* __restrict__ spb) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t v = __ldg(pb + i);
    const uint32_t pos = atomicAdd(cursor + (desc ? N - (uint32_t)v : (uint32_t)v), 1u);
    perm[pos] = (int32_t)i;
    spb[pos] = v;
  }
}

// --------------------------------------------------------- pairs kernel ---
// Output tile 128 (A rows) x 256 (B rows). K is streamed in KC-byte chunks: KC = 128
// (SWIZZLE_128B) for the plain AND-popcount, KC = 64 (SWIZZLE_64B, half-size stages, so
// deeper rings fit next to the estimator table / per-row top-k heaps) otherwise.
constexpr int kTcM = 128, kTcN = 256;
constexpr int kTcAcc = 512 / kTcN;   // TMEM accumulators (512 columns)
constexpr uint32_t kTcSmemMax = 227 * 1024;
enum TcMode { kTcAndPopc = 0, kTcEstimate = 1, kTcTopk = 2, kTcJoin = 3, kTcTopkT = 4, kTcScreen = 5 };
// kTcScreen: the AND-popcount with an integer screen in the epilogue instead of the table store:
// per (query row, 256-wide tile of the popcount-sorted db) pmin = the suffix minimum of the row's
// minimum-pab tables at the tile's smallest |b_s| (K4d), and every pair with pab >= pmin
// is appended (original db index, |b_s| << 14 | pab) to the row's survivor list.
// kTcTopkT: the fused top-k with the query tile A resident in TMEM (columns [0, Kp/4), Kp <= 1024)
// for the whole work item and 128-wide db tiles (two 128-column accumulators after it): only B
// streams through shared memory, so each MMA's operand traffic drops from A + B to B.
constexpr uint32_t kTcMaxThr = 16;   // thresholds per join launch

// Roles per mode: warp 0 TMA producer, warp 1 MMA issuer, then kEpi epilogue warps (kEpi/4 per
// TMEM lane quadrant, each owning 256/(kEpi/4) columns of the tile). The estimate epilogue (fp64
// recipe per pair, latency-bound) runs 16 warps reading 8-column chunks; the others 4 warps.
template <int MODE>
struct TcRoles {
  static constexpr int kEpi = (MODE == kTcEstimate || MODE == kTcJoin) ? 16 : (MODE == kTcTopkT ? 8 : 4);   // TMEM-reading warps
  static constexpr uint32_t kThreads = 64 + 32 * kEpi;
  static constexpr int kCW = (MODE == kTcEstimate || MODE == kTcJoin) ? 8 : 32;   // columns per TMEM load
};

// CG = 1: one CTA per 128 x 256 tile. CG = 2: a CTA pair (cluster of 2, one TPC) computes a
// 256 x 256 tile with cta_group::2 MMAs: each CTA stages its own 128 A rows and HALF of the
// 256 B rows (the MMA reads both CTAs' shared memory), and receives its 128 rows x 256 columns
// in its own TMEM. Same epilogue work per SM, two thirds of the operand bytes per MMA.
template <int KC, int CG = 1>
struct TcGeom {
  static constexpr uint32_t kABytes = kTcM * KC, kBBytes = (kTcN / CG) * KC, kStageBytes = kABytes + kBBytes;
};

// K-major operand tile of KC-byte rows, swizzled as TMA writes it: 8-row atoms of 8*KC
// bytes (SBO); descriptor version 1 (sm_100); layout SWIZZLE_128B (2) or SWIZZLE_64B (4).
template <int KC>
__device__ __forceinline__ uint64_t desc_sw(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;                          // leading byte offset (unused, swizzled K-major)
  d |= (uint64_t)((8u * KC) >> 4) << 32;            // stride byte offset
  d |= (uint64_t)1u << 46;                          // version
  d |= (uint64_t)(KC == 128 ? 2u : 4u) << 61;       // swizzle mode
  return d;
}

struct TcParams {
  uint64_t na, nb;
  uint32_t nk;            // K chunks per tile = Kp / KC
  uint32_t stages;        // ring depth
  uint32_t tiles_n;       // ceil(nb / 256)
  uint32_t splits, per;   // work item = (db chunk s, m-tile); chunk s covers n-tiles [s*per, s*per + per)
  uint64_t mtiles, nitems;
  uint32_t chain;         // kTcTopk: heaps persist across chunks in part_key/idx (one list per row)
  unsigned int* done;     // kTcTopk chained: per m-tile count of finished (chunk, epilogue warp) pairs
  int32_t* out_i32;       // kTcAndPopc: int32 [na][nb]
  const uint16_t* tsuf;   // kTcScreen: suffix-min minimum-pab tables [na][N + 1][nmp] (u16)
  uint32_t nmp;           // kTcScreen: table entries per (row, pb)
  uint2* lists;           // kTcScreen: survivors [na][nb] (original db index, |b_s| << 14 | pab)
  uint32_t* lcnt;         // kTcScreen: survivors per (row, db chunk) [na][splits]
  float* out_f32;         // kTcEstimate: float [popcount(measure)][na][nb]
  uint32_t measure, N, k, flags, prefilter;
  const int32_t* pa;      // |a_s| per A row
  const int32_t* pb;      // |b_s| per B row
  const double* L;        // cardinality table, global (kTcTopk survivors, kTcEstimate if not staged)
  double* part_key;       // kTcTopk: [na][splits][k] (unsorted partial lists)
  int32_t* part_idx;
  uint32_t l_smem;        // kTcEstimate: table staged in shared memory (bytes, 0 = not staged)
  uint32_t heap_smem;     // kTcTopk: per-row heaps + survivor scratch in shared memory (bytes)
  const int2* meta;       // kTcTopk: per db tile [256] (|b_s|, original index), padded to whole tiles
  const int32_t* tmin;    // kTcTopk: per db tile (TN rows) the smallest original index
  const int32_t* perm;    // kTcTopk: B row (sorted by |b_s|, descending for IP, else ascending) -> original db index
  uint32_t l_topk_smem;   // kTcTopk: table staged after the heaps (bytes, 0 = global)
  double lc;              // log1p(-1/N): closed-form inverse of the table for the tile bound
  const int32_t* qperm;   // kTcTopk: A row (queries sorted by |a_s| descending) -> original query index
  const uint32_t* qsk;    // kTcTopkT: the PACKED query sketches [na][qw] in their original order, widened
  uint32_t qw;            //   into TMEM per item by the epilogue warps (no widened copy in HBM)
  uint32_t kp;            // kTcTopkT: bytes per widened row (Kp <= 1024)
  unsigned long long* item_ctr;   // dynamic work queue: next item (zeroed before the launch)
  uint32_t* bits;         // kTcJoin: match bitmaps [nthr][na][wpr] (zeroed before the launch)
  uint64_t wpr;           // kTcJoin: words per bitmap row = ceil(nb / 32)
  uint32_t nthr, exact;   // kTcJoin: threshold count; exact similarities (L = identity) instead of estimates
  uint32_t bcs;           // kTcEstimate: BCS parity sketches (L = the BCS table B, dcap = d)
  double dcap;
  double ham_scale;       // kTcEstimate: Hamming plane = fp64 HAM x ham_scale (1, or 0.5 categorical)
  double tkey[kTcMaxThr];     // kTcJoin: threshold keys, descending
  uint32_t tslot[kTcMaxThr];  // kTcJoin: bitmap plane of each key
};

// Max of 32 values as a depth-4 tree of 3-input maxima (VIMNMX3), not a 31-deep chain: the
// epilogue runs one warp per scheduler, so dependent-latency chains are what it waits on.
__device__ __forceinline__ uint32_t max32(const uint32_t (&v)[32]) {
  uint32_t a[11];
#pragma unroll
  for (int i = 0; i < 10; ++i) a[i] = __vimax3_u32(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  a[10] = max(v[30], v[31]);
  const uint32_t b0 = __vimax3_u32(a[0], a[1], a[2]), b1 = __vimax3_u32(a[3], a[4], a[5]);
  const uint32_t b2 = __vimax3_u32(a[6], a[7], a[8]), b3 = max(a[9], a[10]);
  return max(__vimax3_u32(b0, b1, b2), b3);
}
// Bit j set iff v[j] >= t, built in four independent partial masks.
__device__ __forceinline__ uint32_t ge_mask32(const uint32_t (&v)[32], uint32_t t) {
  uint32_t m[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int j = 0; j < 32; ++j) m[j & 3] |= (v[j] >= t ? 1u : 0u) << j;
  return (m[0] | m[1]) | (m[2] | m[3]);
}

template <int MODE, int KC, int CG>
__global__ void __launch_bounds__(TcRoles<MODE>::kThreads, 1)
tc_pairs_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const TcParams p) {
  using G = TcGeom<KC, CG>;
  constexpr int kEpi = TcRoles<MODE>::kEpi;
  constexpr bool TOPK = MODE == kTcTopk || MODE == kTcTopkT;
  constexpr bool ATM = MODE == kTcTopkT;                    // A resident in TMEM
  constexpr int TN = ATM ? 128 : kTcN;                      // db rows per tile
  constexpr uint32_t kAB = ATM ? 0u : G::kABytes;           // A bytes per stage
  constexpr uint32_t kSB = ATM ? (uint32_t)TN * KC : G::kStageBytes;   // stage bytes
  constexpr uint32_t kAcc0 = ATM ? 256u : 0u;               // first accumulator column
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB alignment by pointer arithmetic on the shared array (keeps the shared address space,
  // so heap / table accesses compile to LDS/STS, not generic LD/ST). Both CTAs of a pair get
  // the same offset (same kernel, same dynamic size), as the pair MMA requires.
  uint8_t* smem = smem_raw + ((1024u - (tc::saddr(smem_raw) & 1023u)) & 1023u);
  const uint32_t S = p.stages;
  const uint32_t base = tc::saddr(smem);
  const uint32_t bars = base + S * kSB;
  auto full = [&](uint32_t s) { return bars + 8u * s; };
  auto empty = [&](uint32_t s) { return bars + 8u * (S + s); };
  auto tfull = [&](int a) { return bars + 8u * (2 * S + a); };
  auto tempty = [&](int a) { return bars + 8u * (2 * S + kTcAcc + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * S + 2 * kTcAcc);
  // dynamic item schedule: the producer takes items from a global counter (heaviest query
  // tiles first) and publishes them through a 4-slot ring read by the MMA and epilogue roles
  // (CG = 2: the leader's producer publishes into both CTAs' rings)
  auto ifull = [&](uint32_t k) { return bars + 8u * (2 * S + 2 * kTcAcc + 1 + k); };
  auto iempty = [&](uint32_t k) { return bars + 8u * (2 * S + 2 * kTcAcc + 5 + k); };
  const uint32_t iring = bars + 8u * (2 * S + 2 * kTcAcc + 9);   // 4 x u64 item ids
  // kTcTopk: 4-slot ring of per-tile db metadata, bulk-loaded by the producer
  // top-k: ring of per-tile db metadata (kMS slots of TN entries, 8 KB), bulk-loaded by the producer
  constexpr uint32_t kMS = ATM ? 8u : 4u;
  auto mfull = [&](uint32_t k) { return bars + 8u * (2 * S + 2 * kTcAcc + 13 + k); };
  auto mempty = [&](uint32_t k) { return bars + 8u * (2 * S + 2 * kTcAcc + 21 + k); };
  const uint32_t aready = bars + 8u * (2 * S + 2 * kTcAcc + 29);   // kTcTopkT: item's A in TMEM
  uint8_t* extra = smem + S * kSB + 1024;        // estimator table or top-k heaps
  // kTcTopk: the metadata ring [4][256] int2 after the heaps and the survivor scratch
  int2* meta_s = reinterpret_cast<int2*>(extra + (size_t)p.k * kTcM * 12 + (kEpi / 4) * 32 * kTcM * 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef BSK_TOPK_PROF
  unsigned long long pacc[9] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};   // per-lane cycle sums, slots 6..14
#endif
  const uint32_t rank = CG == 2 ? tc::cluster_rank() : 0u;
  const bool leader = rank == 0u;

  if (warp == 0 && lane == 0) {
    // CG = 2 counts: tempty one arrival per epilogue warp of both CTAs; iempty the leader's MMA
    // lane + epilogue warps and the peer's producer lane + epilogue warps (the leader's barriers)
    for (uint32_t s = 0; s < S; ++s) { tc::mbar_init(full(s), 1); tc::mbar_init(empty(s), 1); }
    // warps that read each accumulator: every epilogue warp, except top-k (one group of 4)
    constexpr int kTileWarps = TOPK ? 4 : kEpi;
    for (int a = 0; a < kTcAcc; ++a) { tc::mbar_init(tfull(a), 1); tc::mbar_init(tempty(a), CG == 1 ? 32 * kTileWarps : 2 * kTileWarps); }
    constexpr int kTake = kEpi;   // item consumers besides the MMA / producer lanes
    for (uint32_t k = 0; k < 4; ++k) { tc::mbar_init(ifull(k), 1); tc::mbar_init(iempty(k), CG == 1 ? 1 + kTake : 2 + 2 * kTake); }
    for (uint32_t k = 0; k < kMS; ++k) { tc::mbar_init(mfull(k), 1); tc::mbar_init(mempty(k), kTileWarps); }
    tc::mbar_init(aready, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tmem_slot));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tmem_slot));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  const double* L = p.L;
  double* Ls = reinterpret_cast<double*>(extra + ((TOPK || MODE == kTcJoin) ? p.heap_smem : 0u));
  if ((MODE == kTcEstimate && p.l_smem) || TOPK || (MODE == kTcJoin && p.l_topk_smem)) {   // top-k always stages the table
    for (uint32_t i = threadIdx.x; i <= p.N; i += blockDim.x) Ls[i] = p.L[i];
    L = Ls;
  }
  tc::fence_before();
  if constexpr (CG == 1) __syncthreads();
  else tc::cluster_sync();   // both CTAs' barriers initialised and TMEM allocated
  tc::fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot));

  auto publish_item = [&](uint32_t i) -> uint64_t {   // producer lane (the leader's when CG = 2)
    const uint32_t k = i & 3u, ph = (i >> 2) & 1u;
    tc::mbar_wait(iempty(k), ph ^ 1u);
    const uint64_t it = atomicAdd(p.item_ctr, 1ull);
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(iring + 8u * k), "l"(it) : "memory");
    tc::mbar_arrive(ifull(k));
    if constexpr (CG == 2) {
      tc::st_cluster_u64(tc::mapa(iring + 8u * k, 1u), it);
      tc::mbar_arrive_cluster(tc::mapa(ifull(k), 1u));   // release.cluster: orders the remote store
    }
    return it;
  };
  auto take_item = [&](uint32_t i) -> uint64_t {      // one lane per consumer warp
    const uint32_t k = i & 3u, ph = (i >> 2) & 1u;
    uint64_t it;
    if constexpr (CG == 1) {
      tc::mbar_wait(ifull(k), ph);
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(it) : "r"(iring + 8u * k) : "memory");
      tc::mbar_arrive(iempty(k));
    } else {
      tc::mbar_wait_cluster(ifull(k), ph);
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(it) : "r"(iring + 8u * k) : "memory");
      tc::mbar_arrive_cluster(tc::mapa(iempty(k), 0u));
    }
    return it;
  };
  // every role walks the same (item, n-tile) sequence
  // items are chunk-major: all query tiles against db chunk 0, then chunk 1, ... so the
  // chunk's B operand (sized to stay L2-resident) is fetched from HBM about once.
  // mt = this CTA's 128-row A tile (item m-index x CG + rank)
  auto item_range = [&](uint64_t it, uint64_t& mt, uint32_t& sp, uint32_t& nt0, uint32_t& nt1) {
    sp = (uint32_t)(it / p.mtiles);
    mt = (it - (uint64_t)sp * p.mtiles) * CG + rank;
    nt0 = sp * p.per;
    nt1 = min(nt0 + p.per, p.tiles_n);
  };
  // epilogue warp done with accumulator a (after its last TMEM load)
  auto release_acc = [&](int a) {
    tc::fence_before();
    if constexpr (CG == 1) {
      tc::mbar_arrive(tempty(a));
    } else {
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(tc::mapa(tempty(a), 0u));
    }
  };

  // Producer and MMA roles run as whole converged warps (barrier waits by every lane, the TMA /
  // MMA / commit instructions under elect.sync), so the descriptor and coordinate arithmetic
  // stays on the uniform datapath instead of a single-thread branch (ELECT + R2UR broadcasts +
  // BRA.U.ANY around every tcgen05 / TMA instruction).
  if (warp == 0) {
    {   // ---- TMA producer (both CTAs: own A rows, own half of the B rows)
      uint32_t stage = 0, phase = 0, mcount = 0;
      for (uint32_t ii = 0;; ++ii) {
        uint64_t it = 0;
        if (lane == 0) it = (CG == 1 || leader) ? publish_item(ii) : take_item(ii);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= p.nitems) break;
        uint64_t mt; uint32_t sp, nt0, nt1;
        item_range(it, mt, sp, nt0, nt1);
        // top-k: the tiles' db metadata for the epilogue, kMetaAhead tiles ahead of the B stages
        // (the epilogue derives its per-tile bound before the accumulator is ready)
        constexpr uint32_t kMetaAhead = ATM ? 3u : 0u;
        auto issue_meta = [&](uint32_t tnt) {
          const uint32_t ms = mcount % kMS;
          tc::mbar_wait(mempty(ms), ((mcount / kMS) & 1u) ^ 1u);
          if (tc::elect_one()) {
            tc::mbar_expect_tx(mfull(ms), TN * 8u);
            tc::bulk_load(tc::saddr(meta_s) + ms * TN * 8u, p.meta + (size_t)tnt * TN, TN * 8u, mfull(ms));
          }
          __syncwarp();
          ++mcount;
        };
        if constexpr (TOPK)
          for (uint32_t j = nt0; j < min(nt1, nt0 + kMetaAhead); ++j) issue_meta(j);
        for (uint32_t nt = nt0; nt < nt1; ++nt) {
          if constexpr (TOPK)
            if (nt + kMetaAhead < nt1) issue_meta(nt + kMetaAhead);
          for (uint32_t kc = 0; kc < p.nk; ++kc) {
            BSK_T0(tw2);
            tc::mbar_wait(empty(stage), phase ^ 1u);
            if (TOPK && lane == 0) BSK_TADD(12, tw2);
            const uint32_t sa = base + stage * kSB;
            if (tc::elect_one()) {
              if constexpr (ATM) {
                tc::mbar_expect_tx(full(stage), kSB);
                tc::tma_load_2d(sa, &tmB, (int32_t)(kc * KC), (int32_t)(nt * TN), full(stage));
              } else if constexpr (CG == 1) {
                tc::mbar_expect_tx(full(stage), G::kStageBytes);
                tc::tma_load_2d(sa, &tmA, (int32_t)(kc * KC), (int32_t)(mt * kTcM), full(stage));
                tc::tma_load_2d(sa + G::kABytes, &tmB, (int32_t)(kc * KC), (int32_t)(nt * kTcN), full(stage));
              } else {
                if (leader) tc::mbar_expect_tx(full(stage), 2u * G::kStageBytes);   // both CTAs' bytes
                const uint32_t fb = tc::mapa(full(stage), 0u);
                tc::tma_load_2d_pair(sa, &tmA, (int32_t)(kc * KC), (int32_t)(mt * kTcM), fb);
                tc::tma_load_2d_pair(sa + G::kABytes, &tmB, (int32_t)(kc * KC),
                                     (int32_t)(nt * kTcN + rank * (kTcN / 2)), fb);
              }
            }
            __syncwarp();
            if (++stage == S) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {   // ---- MMA issuer (the leader's, for the pair when CG = 2)
      BSK_T0(tmma);
      constexpr uint32_t idesc = (2u << 4) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)((kTcM * CG) >> 4) << 24);
      uint32_t stage = 0, phase = 0, aphase = 0;
      int acc = 0;
      for (uint32_t ii = 0;; ++ii) {
        uint64_t it = 0;
        if (lane == 0) it = take_item(ii);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= p.nitems) break;
        uint64_t mt; uint32_t sp, nt0, nt1;
        item_range(it, mt, sp, nt0, nt1);
        if constexpr (ATM) {   // this item's A rows in TMEM (written by the epilogue warps)
          tc::mbar_wait(aready, ii & 1u);
          tc::fence_after();
        }
        for (uint32_t nt = nt0; nt < nt1; ++nt) {
          BSK_T0(tw0);
          tc::mbar_wait(tempty(acc), aphase ^ 1u);
          if (TOPK && lane == 0) BSK_TADD(10, tw0);
          tc::fence_after();
          const uint32_t d = tmem + kAcc0 + (uint32_t)acc * TN;
          for (uint32_t kc = 0; kc < p.nk; ++kc) {
            BSK_T0(tw1);
            tc::mbar_wait(full(stage), phase);
            if (TOPK && lane == 0) BSK_TADD(11, tw1);
            tc::fence_after();
            const uint32_t sa = base + stage * kSB;
            const uint64_t da = desc_sw<KC>(sa), db = desc_sw<KC>(sa + kAB);
            if (tc::elect_one()) {
#pragma unroll
              for (int kk = 0; kk < KC / 32; ++kk) {   // K = 32 bytes per MMA: +2 in 16-B units
                if constexpr (ATM) tc::mma_u8_ts(d, tmem + (kc * KC + 32u * kk) / 4u, db + 2u * kk, idesc, (kc | (uint32_t)kk) != 0u);
                else if constexpr (CG == 1) tc::mma_u8(d, da + 2u * kk, db + 2u * kk, idesc, (kc | (uint32_t)kk) != 0u);
                else tc::mma_u8_pair(d, da + 2u * kk, db + 2u * kk, idesc, (kc | (uint32_t)kk) != 0u);
              }
              // frees the smem stage (both CTAs' when CG = 2) when these MMAs finish
              if constexpr (CG == 1) tc::commit(empty(stage));
              else tc::commit_pair(empty(stage), (uint16_t)3u);
            }
            __syncwarp();
            if (++stage == S) { stage = 0; phase ^= 1u; }
          }
          // accumulator ready for the epilogue (of both CTAs)
          if (tc::elect_one()) {
            if constexpr (CG == 1) tc::commit(tfull(acc));
            else tc::commit_pair(tfull(acc), (uint16_t)3u);
          }
          __syncwarp();
          if (++acc == kTcAcc) { acc = 0; aphase ^= 1u; }
        }
      }
      if (TOPK && lane == 0) BSK_TADD(14, tmma);
    }
  } else if (TOPK) {
    // ---- top-k epilogue: thread = one query row (TMEM lane), its k best (key, db index)
    // as a heap (worst at the root) in shared memory. kEpi / 4 groups of four warps (one per
    // TMEM lane quadrant) take the tiles in turn (group g: the tiles of accumulator g when
    // there are two groups), so two tiles are filtered at once; a row's heap is shared by the
    // groups under a per-row lock, and its threshold is published for the other group's
    // prefilter (index written before key, read key first: any read is a valid lower bound).
    // Per tile: a prefilter
    // bound pmin on the AND-popcount (db sorted by popcount, so the tile's pb range is
    // narrow); chunks of 32 columns whose max pab < pmin are skipped with one compare.
    // Survivors: while a row's heap fills, each lane evaluates its own columns; in steady
    // state they go through a per-warp queue and are scored lane-parallel (exact fp64
    // recipe), only the rare insertions being serialised to the owning lane.
    constexpr uint32_t NGRP = kEpi / 4;               // epilogue groups
    const uint32_t lb = 32u * (uint32_t)(warp & 3);
    const uint32_t rt = lb + (uint32_t)lane;          // row within the tile
    const uint32_t grp = (uint32_t)(warp - 2) >> 2;   // this warp's group
    const uint32_t m = p.measure, K = p.k;
    constexpr uint32_t kQCap = BSK_TOPK_QCAP;         // per-warp survivor queue entries
    // shared-memory layout (host: topk_heap_smem): heaps | per-group scratch | metadata ring |
    // per-warp queues, candidates, owner masks | per-row count, threshold, lock
    uint8_t* xp = extra;
    double* hk = reinterpret_cast<double*>(xp);                    xp += (size_t)K * kTcM * 8;
    int32_t* hi = reinterpret_cast<int32_t*>(xp);                  xp += (size_t)K * kTcM * 4;
    uint32_t* scr = reinterpret_cast<uint32_t*>(xp) + grp * 32 * kTcM;   xp += NGRP * 32 * kTcM * 4;   // [32][128] per group
    xp += 4 * kTcN * 8;                                                  // metadata ring (meta_s)
    uint2* q = reinterpret_cast<uint2*>(xp) + (size_t)(warp - 2) * kQCap;  xp += kEpi * kQCap * 8;
    uint4* cq = reinterpret_cast<uint4*>(xp) + (size_t)(warp - 2) * 32;    xp += kEpi * 32 * 16;   // per-warp candidate list
    uint32_t* own = reinterpret_cast<uint32_t*>(xp) + (size_t)(warp - 2) * 32;  xp += kEpi * 32 * 4;   // per-owner masks
    volatile uint32_t* cnt_s = reinterpret_cast<volatile uint32_t*>(xp);  xp += kTcM * 4;
    volatile double* Tp = reinterpret_cast<volatile double*>(xp);        xp += kTcM * 8;
    volatile int32_t* Tip = reinterpret_cast<volatile int32_t*>(xp);     xp += kTcM * 4;
    uint32_t* lk = reinterpret_cast<uint32_t*>(xp);
    auto hkey = [&](uint32_t i) -> double& { BSK_ASSERT(i < K); return hk[i * kTcM + rt]; };
    auto hidx = [&](uint32_t i) -> int32_t& { BSK_ASSERT(i < K); return hi[i * kTcM + rt]; };
    auto epi_bar = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpi) : "memory"); };
    uint32_t tcount = 0;   // tiles seen (every group): accumulator, metadata slot and phases
    for (uint32_t ii = 0;; ++ii) {
      uint64_t it = 0;
      if (lane == 0) it = take_item(ii);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= p.nitems) break;
      uint64_t mt; uint32_t sp, nt0, nt1;
      item_range(it, mt, sp, nt0, nt1);
      const uint64_t r = mt * kTcM + rt;               // row of the (sorted) query matrix
      const bool valid = r < p.na;
      const uint64_t rq = (valid && p.qperm) ? (uint64_t)__ldg(p.qperm + r) : r;   // original query index
      if (ATM && grp == 0) {
        // this item's 128 query rows -> TMEM columns [0, kp/4) (lane = row, 4 K-bytes per column),
        // widened here from the packed sketch (column c = nibble c: bytes {bit 4c, .., bit 4c+3},
        // the expand_kernel layout of the B operand). The previous item's MMAs are complete (this
        // warp waited on its last accumulator).
        const uint32_t* src = p.qsk + (valid ? rq : 0) * p.qw;
        for (uint32_t c0 = 0; c0 < p.kp / 4u; c0 += 32) {   // 32 columns = 4 sketch words
          uint32_t wd[4], v[32];
#pragma unroll
          for (int j = 0; j < 4; ++j) wd[j] = (valid && c0 / 8u + j < p.qw) ? __ldg(src + c0 / 8u + j) : 0u;
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const uint32_t nib = (wd[q >> 3] >> (4 * (q & 7))) & 0xFu;
            v[q] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
          }
          tc::tmem_st32(tmem + (lb << 16) + c0, v);
        }
        tc::tmem_st_wait();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(aready);
      }
      const int pa = valid ? __ldg(p.pa + r) : 0;
      const double La = Ls[pa];
      const bool filt = p.prefilter && pa > 0;
      uint32_t cnt = valid ? 0u : K, pmin = 0;   // invalid rows count as full (never insert)
      double T = -__longlong_as_double(0x7ff0000000000000LL);
      int32_t Ti = kSentinelIdx;
      if (grp == 0 && p.chain && sp > 0) {
        // resume this row's heap from the previous chunk (chunk order per query tile is
        // enforced by the done counters: 4 epilogue warps finish each chunk)
        if (lane == 0) {
          const unsigned int need = 4u * CG * sp;   // every epilogue warp of the CTA (pair)
          unsigned int v;
          do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.done + mt / CG) : "memory"); } while (v < need);
        }
        __syncwarp();
        if (valid) {
          const double* ik = p.part_key + rq * K;
          const int32_t* ii = p.part_idx + rq * K;
          cnt = 0;
          for (uint32_t i = 0; i < K; ++i) {
            const int32_t id = __ldcg(ii + i);
            hkey(i) = __ldcg(ik + i); hidx(i) = id;
            cnt += id != kSentinelIdx ? 1u : 0u;
          }
          if (cnt == K) { T = hkey(0); Ti = hidx(0); }
        }
      }
      if (grp == 0) {   // publish the row state for both groups
        cnt_s[rt] = cnt; Tip[rt] = Ti; Tp[rt] = T; lk[rt] = 0u;
      }
      epi_bar();
      // threshold of this row as published by any group (a valid lower bound of the current one)
      auto refresh = [&]() {   // (volatile shared loads issue in program order: key, then index)
        cnt = cnt_s[rt];
        if (cnt >= K) { T = Tp[rt]; Ti = Tip[rt]; }
      };
      refresh();
      auto sift_down = [&](uint32_t i) {
        for (;;) {
          const uint32_t l = 2 * i + 1, rr = l + 1;
          uint32_t w = i;
          if (l < K && before(hkey(w), hidx(w), hkey(l), hidx(l))) w = l;
          if (rr < K && before(hkey(w), hidx(w), hkey(rr), hidx(rr))) w = rr;
          if (w == i) break;
          const double tk = hkey(i); const int32_t ti = hidx(i);
          hkey(i) = hkey(w); hidx(i) = hidx(w);
          hkey(w) = tk; hidx(w) = ti;
          i = w;
        }
      };
      // offer (key, original db index) to this lane's row: under the row lock, against the
      // heap itself; republishes the threshold (index first, then key)
      auto offer = [&](double key, int32_t orig) {
        if ((p.flags & 1u) && (uint64_t)orig == rq) return;
        while (atomicCAS(lk + rt, 0u, 1u) != 0u) {}
        __threadfence_block();
        uint32_t c = cnt_s[rt];
        bool pub = false;
        if (c < K) {
          hkey(c) = key; hidx(c) = orig;
          cnt_s[rt] = ++c;
          if (c == K) {
            for (int i = (int)K / 2 - 1; i >= 0; --i) sift_down((uint32_t)i);
            pub = true;
          }
        } else if (before(key, orig, hkey(0), hidx(0))) {
          hkey(0) = key; hidx(0) = orig;
          sift_down(0);
          pub = true;
        }
        cnt = c;
        if (c >= K) { T = hkey(0); Ti = hidx(0); }
        if (pub) { Tip[rt] = Ti; __threadfence_block(); Tp[rt] = T; }
        __threadfence_block();
        atomicExch(lk + rt, 0u);
      };
      // Upper bound of the key over every pair of this row with a db row of popcount
      // pb in [lo, hi] and AND-popcount pab (K10): the IP raw value decreases
      // in pb for fixed pab (L convex), so IP <= U = min(max(La + L[lo] - L[pa+lo-pab], 0),
      // La, L[hi]); then JS <= U/(La+L[lo]-U), COS <= U/sqrt(La*L[lo]), -HAM <= min(2U-La-L[lo], 0).
      // Non-decreasing in pab.
      auto key_bound = [&](uint32_t pab, uint32_t lo, uint32_t hi_) -> double {
        const uint32_t pu = min(pa + lo - min(pab, pa + lo), p.N);
        const double Llo = Ls[lo];
        double u = La + Llo - Ls[pu];
        u = u > 0.0 ? u : 0.0;
        u = fmin(u, fmin(La, Ls[hi_]));
        if (m == 1u) return u;
        if (m == 4u) { const double den = La + Llo - u; return den > 0.0 ? fmin(u / den, 1.0) : 1.0; }
        if (m == 8u) return fmin(u / sqrt(La * Llo), 1.0);
        return fmin(2.0 * u - La - Llo, 0.0);
      };
      // smallest pab whose bound reaches the current threshold (slack for fp64 rounding)
      // smallest pab whose bound reaches the current threshold g (slack for fp64 rounding):
      // closed-form start from the inverse of L(p) = log1p(-p/N)/log1p(-1/N) with a 2-step
      // low margin, then exact refinement on the staged table (typically 1-3 evaluations)
      uint32_t c_lo = 0xFFFFFFFFu, c_hi = 0, c_pmin = 0;   // last (lo, hi, T, strict) -> pmin
      bool c_strict = false;
      double c_T = 0.0;
      // strict (IP, a single-popcount tile whose db indices all exceed the row's k-th index):
      // the bound is then the exact key (same fp64 expression) and a tie cannot enter, so the
      // smallest pab whose bound EXCEEDS the threshold is taken (no rounding slack needed)
      auto tile_pmin = [&](uint32_t lo, uint32_t hi_, bool strict) -> uint32_t {
        if (!filt || cnt < K || lo == 0) return 0u;
        strict = strict && T >= 0.0;
#ifdef BSK_PMIN_STALE
        if (lo == c_lo && hi_ == c_hi) return c_pmin;   // dev A/B: a stale (lower) threshold is conservative
#else
        if (lo == c_lo && hi_ == c_hi && T == c_T && strict == c_strict) return c_pmin;   // sorted db: runs of equal ranges
#endif
#ifdef BSK_TOPK_STATS
        atomicAdd(&g_tkstats[15], 1ull);   // (lane, tile) bound recomputations
#endif
        const double g = T - 1e-9 * fmax(1.0, fabs(T));
        const uint32_t pmax = min((uint32_t)pa, hi_);
        const double Llo = Ls[lo];
#if BSK_TOPK_STRICT
        if (strict) {   // (m == 1, lo == hi, T >= 0): U(pab) = the key, exactly; find the first U > T
          if (fmin(La, Ls[hi_]) <= T) { c_lo = lo; c_hi = hi_; c_T = T; c_strict = true; c_pmin = pmax + 1; return pmax + 1; }
          const float prs = (float)p.N * (1.0f - __expf((float)((La + Llo - T) * p.lc)));
          const float q0s = (float)pa + (float)lo - fminf(floorf(prs) + 2.0f, (float)p.N);
          uint32_t qs = q0s <= 0.0f ? 0u : min((uint32_t)q0s, pmax);
          const double sab = La + Llo;
          const uint32_t pl = pa + lo;
          for (;;) {
            bool ok[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) ok[u] = qs + u > pmax || sab - Ls[min(pl - min(qs + u, pl), p.N)] > T;
            if (ok[0] || ok[1] || ok[2] || ok[3]) { qs += ok[0] ? 0u : (ok[1] ? 1u : (ok[2] ? 2u : 3u)); break; }
            qs += 4;
          }
          qs = min(qs, pmax + 1);
          c_lo = lo; c_hi = hi_; c_T = T; c_strict = true; c_pmin = qs;
          return qs;
        }
#endif
        double t;   // U(pab) >= t  <=>  key bound >= g
        if (m == 1u) t = g;
        else if (m == 4u) t = g > -1.0 ? g * (La + Llo) / (1.0 + g) : -1.0;
        else if (m == 8u) t = g * sqrt(La * Llo);
        else t = 0.5 * (g + La + Llo);
        if (t <= 0.0) return 0u;
        if (fmin(La, Ls[hi_]) < t) return pmax + 1;               // no pair of the tile can enter
        // fp32 start (hardware exp); its error is far below the 2-step margin, and the
        // result is made exact by the table refinement below
#if BSK_PMIN_FAST
        // (MUFU exp: the absolute error of pr stays below 1e-3 for N <= 65536)
        const float pr = (float)p.N * (1.0f - __expf((float)((La + Llo - t) * p.lc)));
#else
        const float pr = -(float)p.N * expm1f((float)((La + Llo - t) * p.lc));
#endif
        const float q0 = (float)pa + (float)lo - fminf(floorf(pr) + 2.0f, (float)p.N);
        // q0 is a lower bound of the exact answer (the fp32 error of pr is < 0.01, far below the
        // 2-step margin), so only the upward refinement is needed
        uint32_t qq = q0 <= 0.0f ? 0u : min((uint32_t)q0, pmax);
        // refinement, four candidates per step evaluated independently (the answer is
        // typically within q0 + 3): the first qq with key_bound(qq) >= g
#if BSK_PMIN_FAST
        // IP: with t = g > 0 and min(La, L[hi]) >= g checked above, key_bound(pab) >= g is
        // exactly (La + L[lo]) - L[pu(pab)] >= g — the same fp64 expression, the rest hoisted
        const double sab = La + Llo;
        const uint32_t pl = pa + lo;
#endif
        for (;;) {
          bool ok[4];
#if BSK_PMIN_FAST
          if (m == 1u) {
#pragma unroll
            for (int u = 0; u < 4; ++u) ok[u] = qq + u > pmax || sab - Ls[min(pl - min(qq + u, pl), p.N)] >= g;
          } else
#endif
#pragma unroll
          for (int u = 0; u < 4; ++u) ok[u] = qq + u > pmax || key_bound(qq + u, lo, hi_) >= g;
          if (ok[0] || ok[1] || ok[2] || ok[3]) {
            qq += ok[0] ? 0u : (ok[1] ? 1u : (ok[2] ? 2u : 3u));
            break;
          }
          qq += 4;
        }
        qq = min(qq, pmax + 1);
        c_lo = lo; c_hi = hi_; c_T = T; c_strict = false; c_pmin = qq;
        return qq;
      };
      for (uint32_t nt = nt0; nt < nt1; ++nt) {
        const uint32_t my = tcount++;
        if (my % NGRP != grp) continue;                // the other group's tile
        const int acc = (int)(my % kTcAcc);
        const uint32_t aphase = (my / kTcAcc) & 1u;
        BSK_T0(te0);
#if BSK_TOPK_STRICT
        const int32_t tmin_t = m == 1u ? __ldg(p.tmin + nt) : 0;   // (consumed after the refresh and metadata wait)
#endif
        refresh();
        const uint64_t n0 = (uint64_t)nt * TN;
        // this tile's db popcounts / original indices, bulk-loaded by the producer
        const uint32_t ms = my % kMS;
        tc::mbar_wait(mfull(ms), (my / kMS) & 1u);
        const int2* tm = meta_s + ms * TN;
        const uint32_t nval = (uint32_t)min((uint64_t)TN, p.nb - n0);
        // the tile's popcount range (the db is popcount-sorted, descending or ascending)
#ifdef BSK_TOPK_PROF
        { const uint32_t x0 = (uint32_t)tm[nval - 1].x + (uint32_t)tm[0].x; if (x0 == 0xFFFFFFFFu) pmin = 1u; }
        if (lane == 0) BSK_TADD(13, te0);
#endif
        {
          const uint32_t tlo = min((uint32_t)tm[nval - 1].x, (uint32_t)tm[0].x), thi = max((uint32_t)tm[nval - 1].x, (uint32_t)tm[0].x);
          bool strict = false;
#if BSK_TOPK_STRICT
          if (m == 1u && tlo == thi) strict = tmin_t > Ti;   // (tmin_t: smallest db index of the tile)
#endif
          if (valid) pmin = tile_pmin(tlo, thi, strict);
        }
        const bool direct = __any_sync(0xffffffffu, cnt < K);
#ifdef BSK_TOPK_STATS
        {
          const uint32_t hi_ = max((uint32_t)tm[nval - 1].x, (uint32_t)tm[0].x);
          const bool skip = __all_sync(0xffffffffu, !valid || (cnt >= K && pmin > min((uint32_t)pa, hi_)));
          if (lane == 0) { atomicAdd(&g_tkstats[0], 1ull); if (skip) atomicAdd(&g_tkstats[1], 1ull); if (direct) atomicAdd(&g_tkstats[4], 1ull); }
        }
#endif
        if (lane == 0) BSK_TADD(9, te0);
        BSK_T0(te1);
        tc::mbar_wait(tfull(acc), aphase);
        if (lane == 0) BSK_TADD(6, te1);
        BSK_T0(te2);
        tc::fence_after();
        // survivors queued by this warp since the last call, scored lane-parallel (exact fp64 recipe)
        uint32_t qn = 0;
        auto score_queue = [&]() {
          __syncwarp();
          for (uint32_t b = 0; b < qn; b += 32) {
            const bool has = b + lane < qn;
            const uint2 e = has ? q[b + lane] : make_uint2(0u, 0u);
            const int owner = (int)(e.y >> 24);
            BSK_ASSERT(!has || (owner < 32 && e.x < TN));
            const int pa_o = __shfl_sync(0xffffffffu, pa, owner);
            const double T_o = __shfl_sync(0xffffffffu, T, owner);
            const int32_t Ti_o = __shfl_sync(0xffffffffu, Ti, owner);
            double key = -__longlong_as_double(0x7ff0000000000000LL);
            const int2 me = tm[e.x];
            if (has) key = measure_key(estimate_pair(pa_o, me.x, (int)(e.y & 0xFFFFFFu), (int)p.N, Ls, m), m);
            // candidates — those that would enter the owner's heap at its current threshold
            // (key, then the tie order of R-G17 on the db index, checked here lane-parallel:
            // rows with tiny sketches tie with thousands of db rows) — go back to their owners
            const bool cand = has && before(key, me.y, T_o, Ti_o);
            const uint32_t bal = __ballot_sync(0xffffffffu, cand);
#ifdef BSK_TOPK_STATS
            if (lane == 0) atomicAdd(&g_tkstats[5], (unsigned long long)__popc(bal));
#endif
            if (bal) {
              // owner-parallel insertion: candidate of evaluating lane e sits in cq[e]; the
              // lowest lane of each same-owner group publishes the group's mask to its owner,
              // and every owner walks its own candidates (rounds = max candidates per owner)
              const uint32_t grp = __match_any_sync(0xffffffffu, cand ? (uint32_t)owner : 32u + (uint32_t)lane);
              __syncwarp();
              own[lane] = 0u;
              if (cand) cq[lane] = make_uint4(e.x, (uint32_t)owner, __double2loint(key), __double2hiint(key));
              __syncwarp();
              if (cand && (grp & ((1u << lane) - 1u)) == 0u) own[owner] = grp;
              __syncwarp();
              uint32_t mine = own[lane];
              while (mine) {
                const uint32_t ee = __ffs(mine) - 1; mine &= mine - 1;
                BSK_ASSERT(ee < 32u);
                const uint4 c4 = cq[ee];
                offer(__hiloint2double((int)c4.w, (int)c4.z), tm[c4.x].y);
              }
              __syncwarp();
            }
          }
          __syncwarp();
          qn = 0;
        };
        // one 32-column chunk (values v): prefilter, then survivors
        // (V(j): the pab of column c + j of this lane's row; mx: the max of V over the chunk)
        auto chunk = [&](const uint32_t c, const uint32_t mx, auto&& V) {
          if (c >= nval) return;
          const uint32_t left = nval - c;
          const bool pass = valid && mx >= pmin;
          if (!__any_sync(0xffffffffu, pass)) return;
          // survivor mask of this lane (four independent partial masks)
          uint32_t sm = 0u;
          if (pass) {
            uint32_t mk[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int j = 0; j < 32; ++j) mk[j & 3] |= (V(j) >= pmin ? 1u : 0u) << j;
            sm = ((mk[0] | mk[1]) | (mk[2] | mk[3])) & (left >= 32 ? 0xffffffffu : ((1u << left) - 1u));
          }
          const uint32_t ns = __popc(sm);
#ifdef BSK_TOPK_STATS
          {
            const uint32_t tot = __reduce_add_sync(0xffffffffu, ns);
            if (lane == 0) { atomicAdd(&g_tkstats[2], 1ull); atomicAdd(&g_tkstats[3], (unsigned long long)tot); }
          }
#endif
          uint32_t off = ns;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, off, o); if (lane >= o) off += y; }
          const uint32_t total = __shfl_sync(0xffffffffu, off, 31);
          off -= ns;
          if (direct || total > kQCap) {
            // per-lane: each lane walks its own survivors (heap filling, or a burst)
            if (ns) {
#pragma unroll
              for (int j = 0; j < 32; ++j) scr[j * kTcM + rt] = V(j);
              uint32_t mm = sm;
              while (mm) {   // four independent fp64 evaluations in flight, then the offers
                double kk[4];
                int32_t ix[4];
                uint32_t nk = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  if (mm) {
                    const uint32_t j = __ffs(mm) - 1; mm &= mm - 1;
                    const int2 mj = tm[c + j];
                    kk[u] = measure_key(estimate_pair(pa, mj.x, (int)scr[j * kTcM + rt], (int)p.N, Ls, m), m);
                    ix[u] = mj.y;
                    nk = (uint32_t)u + 1;
                  }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  if ((uint32_t)u < nk && (cnt < K || kk[u] >= T)) offer(kk[u], ix[u]);
              }
            }
            __syncwarp();
            return;
          }
          // queue: (column in tile, owner lane << 24 | pab); scored after the accumulator is
          // released (score_queue), so the MMA never waits on survivor scoring
          if (qn + total > kQCap) score_queue();
          off += qn;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if ((sm >> j) & 1u) { BSK_ASSERT(off < kQCap && c + (uint32_t)j < TN); q[off++] = make_uint2(c + (uint32_t)j, ((uint32_t)lane << 24) | V(j)); }
          qn += total;
          __syncwarp();
                };
        // 64 columns per step: both TMEM loads in flight, one vote for the pair of chunks (the
        // prefilter rejects ~90 % of them); the whole tile is skipped without reading TMEM when
        // no row of the warp can reach its threshold in it (pmin above the row's largest pab)
        const uint32_t tb = tmem + (lb << 16) + kAcc0 + (uint32_t)acc * TN;
        const uint32_t tile_hi = max((uint32_t)tm[nval - 1].x, (uint32_t)tm[0].x);
#ifdef BSK_TOPK_NULLEPI
        if (false) {   // dev: MMA/TMA-side bound of the tiling (results are garbage)
#else
        if (__any_sync(0xffffffffu, valid && (cnt < K || pmin <= min((uint32_t)pa, tile_hi)))) {
#endif
          uint32_t va[32];
#pragma unroll 1
          for (uint32_t c = 0; c < nval; c += 32) {   // one 32-column chunk at a time (register budget)
            tc::tmem_ld32_issue(tb + c, va);
            tc::tmem_ld_wait(va);
#ifdef BSK_EPI_LDONLY
            if (va[0] == 0xdeadbeefu && va[31] == 0x12345678u) pmin = 0;   // dev: keep the loads, skip the filter
            continue;
#endif
            chunk(c, max32(va), [&](int j) { return va[j]; });
          }
        }
        release_acc(acc);
        if (lane == 0) BSK_TADD(7, te2);
        BSK_T0(te3);
        if (qn) score_queue();
        if (lane == 0) BSK_TADD(8, te3);
        __syncwarp();   // every lane done with this tile's metadata
        if (lane == 0) tc::mbar_arrive(mempty(ms));
      }
      epi_bar();   // every group done with this item's tiles
      cnt = cnt_s[rt];
      if (grp == 0 && valid) {   // partial list of this (row, chunk) — or the row's running heap when chained
        const uint64_t slot = p.chain ? rq : rq * p.splits + sp;
        double* ok = p.part_key + slot * K;
        int32_t* oi = p.part_idx + slot * K;
        for (uint32_t i = 0; i < K; ++i) {
          __stcg(ok + i, i < cnt ? hkey(i) : -__longlong_as_double(0x7ff0000000000000LL));
          __stcg(oi + i, i < cnt ? hidx(i) : kSentinelIdx);
        }
      }
      if (grp == 0 && p.chain) {
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.done + mt / CG, 1u);
      }
    }
  } else if (MODE == kTcJoin) {
    // ---- threshold-join epilogue (Exp. 2; R-J1). The db is in its own order,
    // so each lane (one query row, its TMEM lane) owns whole output words: the kEpi/4 warps of a
    // lane quadrant split the tile's columns (64 each, 8-column TMEM chunks), every pair is
    // screened by the division-free necessary condition against the LOWEST threshold key
    // (pretest_keep), the rest are scored exactly (canonical fp64 recipe, or the exact key) and
    // set their bit in every plane whose threshold they reach; each lane then stores its row's
    // two words per plane with plain stores (every output word written exactly once: no memset,
    // no atomics).
    constexpr int CW = TcRoles<MODE>::kCW, NG = TcRoles<MODE>::kEpi / 4;
    constexpr uint32_t kWC = kTcN / NG;               // columns per warp (64)
    const int ew = warp - 2;
    const uint32_t lb = 32u * (uint32_t)(warp & 3);
    const uint32_t rt = lb + (uint32_t)lane;
    const uint32_t cg0 = (uint32_t)(ew >> 2) * kWC;
    const uint32_t m = p.measure, nthr = p.nthr;
    const bool exact = p.exact != 0u;
    const double tlo = p.tkey[nthr - 1];
    const uint64_t plane = p.na * p.wpr;
    // per-warp scratch after the (optionally staged) table: output words [32 lanes][16][2],
    // the chunk's pab values [32][CW+1] and db popcounts [CW]
    uint8_t* jscr = extra + p.l_topk_smem + (size_t)ew * (32 * nthr * 2 * 4 + 32 * (CW + 1) * 4 + 64);
    uint32_t* jw = reinterpret_cast<uint32_t*>(jscr);
    uint32_t* sv = jw + 32 * nthr * 2;
    int32_t* spb_s = reinterpret_cast<int32_t*>(sv + 32 * (CW + 1));
    const uint32_t rt_w = (uint32_t)lane;
    uint32_t aphase = 0;
    int acc = 0;
    for (uint32_t ii = 0;; ++ii) {
      uint64_t it = 0;
      if (lane == 0) it = take_item(ii);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= p.nitems) break;
      uint64_t mt; uint32_t sp, nt0, nt1;
      item_range(it, mt, sp, nt0, nt1);
      const uint64_t r = mt * kTcM + rt;
      const bool valid = r < p.na;
      const int pa = valid ? __ldg(p.pa + r) : 0;
      for (uint32_t nt = nt0; nt < nt1; ++nt) {
        const uint64_t n0 = (uint64_t)nt * kTcN;
        tc::mbar_wait(tfull(acc), aphase);
        tc::fence_after();
        // this lane's output words for the tile: [plane][2] in shared memory (own lane only)
        uint32_t* wb = jw + (size_t)rt_w * (nthr * (kWC / 32));
#pragma unroll 1
        for (uint32_t t = 0; t < nthr; ++t) { wb[2 * t] = 0u; wb[2 * t + 1] = 0u; }
#pragma unroll 1
        for (uint32_t c = 0; c < kWC; c += CW) {
          uint32_t v[CW];
          if constexpr (CW == 8) tc::tmem_ld8(tmem + (lb << 16) + (uint32_t)acc * kTcN + cg0 + c, v);
          else tc::tmem_ld32(tmem + (lb << 16) + (uint32_t)acc * kTcN + cg0 + c, v);
          const uint64_t cb = n0 + cg0 + c;
          const int32_t pbl = (lane < CW && cb + lane < p.nb) ? __ldg(p.pb + cb + lane) : 0;
          // 1) screen the 8 pairs (straight-line, no per-pair branches)
          uint32_t keepm = 0;
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            const int pb = __shfl_sync(0xffffffffu, pbl, j);
            const uint64_t col = cb + j;
            bool keep = valid && col < p.nb && !((p.flags & 1u) && col == r);
            if (!exact) keep = keep && pretest_keep(pa, pb, (int)v[j], (int)p.N, L, m, tlo);
            keepm |= (keep ? 1u : 0u) << j;
            sv[lane * (CW + 1) + j] = v[j];
          }
          if (lane < CW) spb_s[lane] = pbl;
          __syncwarp();
          // 2) the survivors: exact key, then the planes it reaches (thresholds descending)
          while (keepm) {
            const uint32_t j = __ffs(keepm) - 1; keepm &= keepm - 1;
            const int pb = spb_s[j];
            const int pab = (int)sv[lane * (CW + 1) + j];
            uint32_t t0 = nthr;   // planes t >= t0 pass
            if (!exact && (m == 4u || m == 8u)) {
              t0 = join_first_plane(pa, pb, pab, (int)p.N, L, m, p.tkey, nthr);   // division-free where certain
            } else {
              const double key = exact ? exact_key(pa, pb, pab, m) : measure_key(estimate_pair(pa, pb, pab, (int)p.N, L, m), m);
              while (t0 > 0 && key >= p.tkey[t0 - 1]) --t0;
            }
            const uint32_t h = (c + j) >> 5, bit = 1u << ((c + j) & 31u);
            for (uint32_t t = t0; t < nthr; ++t) wb[2 * t + h] |= bit;
          }
          __syncwarp();
        }
        release_acc(acc);
        if (++acc == kTcAcc) { acc = 0; aphase ^= 1u; }
        if (valid) {
          const uint64_t w0 = (n0 + cg0) >> 5;
#pragma unroll 1
          for (uint32_t t = 0; t < nthr; ++t) {
            uint32_t* row = p.bits + (uint64_t)p.tslot[t] * plane + r * p.wpr;
            if (w0 < p.wpr) __stcs(row + w0, wb[2 * t]);
            if (w0 + 1 < p.wpr) __stcs(row + w0 + 1, wb[2 * t + 1]);
          }
        }
      }
    }
  } else {             // ---- andpopc / estimate epilogue: warp w reads TMEM lanes 32*(w%4) .. +31
    // Thread = one row of the tile (its TMEM lane); the kEpi/4 warps of a lane quadrant split
    // the 256 columns. Each 32 x CW chunk is transposed through a per-warp shared scratch
    // ([plane][32][CW+1], conflict-free writes) so that stores are row-contiguous.
    constexpr int CW = TcRoles<MODE>::kCW, NG = TcRoles<MODE>::kEpi / 4;
    constexpr int RPI = 32 / CW;                      // rows per store instruction
    constexpr uint32_t kTr = 32 * (CW + 1);           // one transposed plane
    constexpr uint32_t kPl = MODE == kTcAndPopc ? 1 : 4;
    const int ew = warp - 2;
    const uint32_t lb = 32u * (uint32_t)(warp & 3);
    const uint32_t rt = lb + (uint32_t)lane;          // row within the tile
    const uint32_t cg0 = (uint32_t)(ew >> 2) * (kTcN / NG), cg1 = cg0 + kTcN / NG;
    uint32_t* tr = reinterpret_cast<uint32_t*>(extra + p.l_smem) + (size_t)ew * kPl * kTr;
    uint32_t aphase = 0;
    int acc = 0;
    const uint32_t m = p.measure;
    const uint32_t nplanes = MODE == kTcEstimate ? (uint32_t)__popc(m) : 1u;
    for (uint32_t ii = 0;; ++ii) {
      uint64_t it = 0;
      if (lane == 0) it = take_item(ii);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= p.nitems) break;
      uint64_t mt; uint32_t sp, nt0, nt1;
      item_range(it, mt, sp, nt0, nt1);
      const uint64_t r = mt * kTcM + rt;
      const bool valid = r < p.na;
      const int pa = (MODE == kTcEstimate && valid) ? __ldg(p.pa + r) : 0;
      const uint64_t r0 = mt * kTcM + lb;             // first row of this warp's quadrant
      const uint32_t nrows = r0 < p.na ? (uint32_t)min((uint64_t)32, p.na - r0) : 0u;
      const bool vec_rows = (p.nb & 3u) == 0 && (reinterpret_cast<uintptr_t>(p.out_f32) & 15u) == 0;
      // kTcScreen: this row's survivors of the item's db chunk go to the list segment that starts
      // at the chunk's first column (a chunk of w columns holds at most w survivors of a row), so
      // the lane appends with a private counter — no atomics — and stores the count at item end
      uint32_t lc = 0;
      const uint64_t lbase = (uint64_t)nt0 * kTcN;
      for (uint32_t nt = nt0; nt < nt1; ++nt) {
        const uint64_t n0 = (uint64_t)nt * kTcN;
        uint32_t pmin = 0xFFFFFFFFu;   // kTcScreen: this row's screen for the tile (none for padding rows)
        int2* tmeta_w = reinterpret_cast<int2*>(extra) + (size_t)ew * kTcN;   // kTcScreen: per warp
        if constexpr (MODE == kTcScreen) {
          // the tile's (original index, |b_s|) per column into this warp's shared buffer while the
          // MMA runs (survivors then carry them: the list top-k needs no gathers)
          for (uint32_t c = (uint32_t)lane; c < kTcN; c += 32) {
            const uint64_t col = n0 + c;
            tmeta_w[c] = col < p.nb ? make_int2(__ldg(p.perm + col), __ldg(p.pb + col)) : make_int2(0, 0);
          }
          __syncwarp();
          if (valid && n0 < p.nb) {
            const uint32_t lo = (uint32_t)tmeta_w[0].y;   // the tile's smallest |b_s| (ascending sort)
            const uint16_t* t = p.tsuf + ((size_t)r * (p.N + 1) + lo) * p.nmp;
            for (uint32_t i = 0; i < p.nmp; ++i) pmin = min(pmin, (uint32_t)__ldg(t + i));
          }
        }
        tc::mbar_wait(tfull(acc), aphase);
        tc::fence_after();
#pragma unroll 1
        for (uint32_t c = cg0; c < cg1; c += CW) {
          uint32_t v[CW];
          if constexpr (CW == 32) tc::tmem_ld32(tmem + (lb << 16) + (uint32_t)acc * kTcN + c, v);
          else tc::tmem_ld8(tmem + (lb << 16) + (uint32_t)acc * kTcN + c, v);
          if (n0 + c >= p.nb || nrows == 0) continue;    // warp-uniform
          const uint64_t cb = n0 + c;
          const uint32_t left = (uint32_t)min((uint64_t)CW, p.nb - cb);
          if constexpr (MODE == kTcScreen) {
            const uint32_t sm = ge_mask32(v, pmin) & (left >= 32u ? 0xFFFFFFFFu : ((1u << left) - 1u));
            if (!__any_sync(0xffffffffu, sm != 0u)) continue;
            // the chunk's values through this warp's shared row (conflict-free: lane * 33 + j), so
            // each lane walks only its own survivors
            uint32_t* vs = reinterpret_cast<uint32_t*>(reinterpret_cast<int2*>(extra) + 4 * kTcN) + (size_t)ew * 32 * 33;
#pragma unroll
            for (int j = 0; j < CW; ++j) vs[lane * 33 + j] = v[j];
            __syncwarp();
            uint64_t pos = lbase + lc;
            lc += (uint32_t)__popc(sm);
            uint2* o = p.lists + r * p.nb;
            uint32_t mm = sm;
            while (mm) {   // (original db index, |b_s| << 14 | pab): N <= 16383
              const uint32_t j = (uint32_t)__ffs(mm) - 1u;
              mm &= mm - 1u;
              const int2 mt_ = tmeta_w[c + j];
              o[pos++] = make_uint2((uint32_t)mt_.x, ((uint32_t)mt_.y << 14) | vs[lane * 33 + j]);
            }
            __syncwarp();
            continue;
          }
          if (MODE == kTcAndPopc) {
#pragma unroll
            for (int j = 0; j < CW; ++j) tr[lane * (CW + 1) + j] = v[j];
          } else {
            const int32_t pbl = lane < (int)left ? __ldg(p.pb + cb + lane) : 0;
            // all four planes of BinSketch (the common call) compiled with the mask constant;
            // with 16-B aligned rows each lane stores its row's CW = 8 values per plane as two
            // 16-B stores (no transpose)
            auto planes = [&](auto mtag) -> bool {
              constexpr uint32_t MM = decltype(mtag)::value;
              const uint32_t mm = MM ? MM : m;
              float val[4][CW];
#pragma unroll
              for (int j = 0; j < CW; ++j) {
                const int pb = __shfl_sync(0xffffffffu, pbl, j);
                Est e;
                if (MM == 0u && p.bcs) e = bcs_estimate_pair(pa, pb, (int)v[j], p.dcap, L, mm);
                else e = estimate_pair(pa, pb, (int)v[j], (int)p.N, L, mm);
                // val[measure id][j] (static indices; the output plane of id is popc(mm & ((1<<id)-1)))
                val[0][j] = __double2float_rn(e.ip);
                val[1][j] = __double2float_rn(MM ? e.ham : __dmul_rn(e.ham, p.ham_scale));
                val[2][j] = __double2float_rn(e.js);
                val[3][j] = __double2float_rn(e.cs);
              }
              if (CW == 8 && vec_rows && left == (uint32_t)CW) {
                if (valid) {
                  const uint64_t plane = p.na * p.nb;
                  float* o = p.out_f32 + r * p.nb + cb;
#pragma unroll
                  for (uint32_t id = 0; id < 4; ++id) {
                    if (mm & (1u << id)) {
                      float* oq = o + (uint64_t)__popc(mm & ((1u << id) - 1u)) * plane;
                      __stcs(reinterpret_cast<float4*>(oq), make_float4(val[id][0], val[id][1], val[id][2], val[id][3]));
                      __stcs(reinterpret_cast<float4*>(oq + 4), make_float4(val[id][4], val[id][5], val[id][6], val[id][7]));
                    }
                  }
                }
                return true;
              }
#pragma unroll
              for (int j = 0; j < CW; ++j)
                if (valid && (uint32_t)j < left)
#pragma unroll
                  for (uint32_t id = 0; id < 4; ++id)
                    if (mm & (1u << id))
                      tr[(uint32_t)__popc(mm & ((1u << id) - 1u)) * kTr + lane * (CW + 1) + j] = __float_as_uint(val[id][j]);
              return false;
            };
            const bool done = (m == 15u && !p.bcs && p.ham_scale == 1.0) ? planes(std::integral_constant<uint32_t, 15u>{})
                                                                         : planes(std::integral_constant<uint32_t, 0u>{});
            if (done) continue;                            // warp-uniform (left, vec_rows uniform)
          }
          __syncwarp();
          {
            const uint32_t col = (uint32_t)lane % CW, rsub = (uint32_t)lane / CW;
            const uint64_t plane = p.na * p.nb;
            if (col < left) {
              for (uint32_t rr = rsub; rr < nrows; rr += RPI) {
                const uint64_t o = (r0 + rr) * p.nb + cb + col;
                if (MODE == kTcAndPopc) {
                  __stcs(p.out_i32 + o, (int32_t)tr[rr * (CW + 1) + col]);
                } else {
                  for (uint32_t q = 0; q < nplanes; ++q)
                    __stcs(reinterpret_cast<uint32_t*>(p.out_f32) + q * plane + o, tr[q * kTr + rr * (CW + 1) + col]);
                }
              }
            }
          }
          __syncwarp();
        }
        release_acc(acc);
        if (++acc == kTcAcc) { acc = 0; aphase ^= 1u; }
      }
      if constexpr (MODE == kTcScreen)
        if (valid) p.lcnt[r * p.splits + sp] = lc;
    }
  }
#ifdef BSK_TOPK_PROF
  if (lane == 0)
    for (int i = 0; i < 9; ++i)
      if (pacc[i]) atomicAdd(&g_tkstats[6 + i], pacc[i]);
#endif
  tc::fence_before();
  if constexpr (CG == 1) __syncthreads();
  else tc::cluster_sync();   // no CTA leaves while its peer may still signal its barriers / TMEM
  if (warp == 1) {
    tc::fence_after();
    if constexpr (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ------------------------------------------------------------------- host ---
namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(f);
  });
  return fn;
}

bool make_map(CUtensorMap* m, const uint8_t* ptr, uint64_t rows, uint32_t Kp, uint32_t box_rows, uint32_t kc) {
  EncodeTiled enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {Kp, rows};
  const cuuint64_t strides[1] = {Kp};
  const cuuint32_t box[2] = {kc, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, kc == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

uint32_t tc_kpad(uint32_t N) { return ((N + 127) / 128) * 128; }

cudaError_t launch_expand(const uint32_t* sk, uint64_t n, uint32_t N, uint8_t* out, cudaStream_t s,
                          const int32_t* perm) {
  if (n == 0) return cudaSuccess;
  const uint32_t W = (N + 31) / 32, Kp = tc_kpad(N);
  const uint64_t total = n * (Kp / 32);
  const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, (uint64_t)num_sms() * 16);
  expand_kernel<<<(unsigned)blocks, 256, 0, s>>>(sk, n, W, Kp, perm, out);
  count_launch();
  return cudaGetLastError();
}

// Work decomposition (device independent, so workspace sizes are pure functions):
// db chunks of <= ~40 MB of widened operand (L2-resident while every query tile visits
// them), and at least ~2 items per SM. Top-k chains its per-row heaps through the chunks
// when there are enough query tiles to keep every SM busy; otherwise it uses independent
// per-chunk partial lists merged afterwards.
struct TcSplit { uint32_t splits, chain; };
static TcSplit tc_split_rule(uint64_t na, uint64_t nb, uint32_t N, bool topk, uint32_t k = 0, uint32_t tn = kTcN) {
  const uint64_t tiles_n = (nb + tn - 1) / tn, mtiles = (na + kTcM - 1) / kTcM, sms = 148;
  uint64_t chunk_bytes = (topk ? 48ull : 40ull) << 20;   // top-k, Large: 5 chunks of 41 MB (measured: 6 x 34 MB 39.68, 5 x 41 MB 39.40, 3 x 68 MB 41.12 ms)
  // dev knobs (sanitizer / A-B runs on small shapes): db chunk size in KB, forced heap chaining.
  // Read here only, so workspace sizing and the launch always agree.
  if (const char* e = std::getenv("BINSKETCH_TC_CHUNK_KB")) chunk_bytes = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) << 10;
  uint64_t s_l2 = (nb * tc_kpad(N) + chunk_bytes - 1) / chunk_bytes;
  uint64_t s_par = (2 * sms + mtiles - 1) / mtiles;
  TcSplit r;
  r.chain = (topk && mtiles >= 2 * sms) ? 1u : 0u;
  if (const char* e = std::getenv("BINSKETCH_TC_CHAIN")) if (topk && !std::strcmp(e, "1")) r.chain = 1u;
  uint64_t splits = r.chain ? s_l2 : std::max(s_l2, s_par);
  if (topk && !r.chain && k) splits = std::min<uint64_t>(splits, std::max<uint32_t>(1, 8192 / k));   // merge capacity
  splits = std::max<uint64_t>(1, std::min<uint64_t>(splits, tiles_n));
  const uint64_t per = (tiles_n + splits - 1) / splits;
  r.splits = (uint32_t)((tiles_n + per - 1) / per);
  return r;
}

// CTA-pair mode per launch. Pairs halve each SM's share of the B operand (shared-memory and L2
// traffic per MMA), which pays when the K loop is long relative to the epilogue: the plain
// AND-popcount from K = 4096 (8192^2 x 8192: 0.46 -> 0.38 ms; Exp.-1 exact rows, K = 28160:
// 4.02 -> 3.60 ms; Ranking's table: 3.65 -> 3.59 ms) and every mode from K = 16384 (exact join,
// K = 102784: 77.7 -> 67.7 ms). With sketch-length K the coupling of the two CTAs' epilogues costs
// more than it saves (Large top-k 52.9 -> 61.7 ms; estimate / sketch join neutral to -2 %).
// BINSKETCH_TC_CG=1|2 overrides (dev A/B; K10).
template <int MODE>
static int tc_cg(uint32_t Kp) {
  if (MODE == kTcTopkT) return 1;
  if (const char* e = std::getenv("BINSKETCH_TC_CG")) return std::atoi(e) == 2 ? 2 : 1;
  return (Kp >= 16384u || ((MODE == kTcAndPopc || MODE == kTcScreen) && Kp >= 4096u)) ? 2 : 1;
}

// Shared launcher: pick ring depth from the shared memory left after `extra_bytes`, build
// the TMA maps, size the work items (>= 2 per SM when the db can be split).
template <int MODE, int KC, int CG>
static cudaError_t tc_launch_cg(const uint8_t* A8, const uint8_t* B8, TcParams& p, uint32_t N, uint32_t extra_bytes,
                                uint32_t force_splits, cudaStream_t s) {
  using G = TcGeom<KC, CG>;
  constexpr bool ATM = MODE == kTcTopkT;
  constexpr uint32_t TN = ATM ? 128u : (uint32_t)kTcN;
  constexpr uint32_t kSB = ATM ? TN * KC : G::kStageBytes;
  const uint32_t Kp = tc_kpad(N);
  if (p.na > 0x7fffffffull || p.nb > 0x7fffffffull) return cudaErrorInvalidValue;
  if (ATM && (CG != 1 || Kp > 1024u)) return cudaErrorInvalidValue;   // A must fit TMEM columns [0, 256)
  const uint32_t fixed = 1024 /* align */ + 1024 /* barriers */ + extra_bytes;
  if (fixed + 2 * kSB > kTcSmemMax) return cudaErrorInvalidConfiguration;
  p.stages = std::min<uint32_t>(ATM ? 16u : 8u, (kTcSmemMax - fixed) / kSB);
  if (const char* st = std::getenv("BINSKETCH_TC_STAGES"))   // dev A/B: cap the ring depth
    p.stages = std::max<uint32_t>(2u, std::min<uint32_t>(p.stages, (uint32_t)std::atoi(st)));
  alignas(64) CUtensorMap ma, mb;
  if (!make_map(&mb, B8, p.nb, Kp, ATM ? TN : kTcN / CG, KC)) return cudaErrorNotSupported;
  if (ATM) ma = mb;   // (A is not TMA-loaded: the epilogue widens the packed rows into TMEM)
  else if (!make_map(&ma, A8, p.na, Kp, kTcM, KC)) return cudaErrorNotSupported;
  cudaError_t e = cudaSuccess;
  p.nk = Kp / KC;
  p.tiles_n = (uint32_t)((p.nb + TN - 1) / TN);
  const uint64_t mtiles = (p.na + kTcM * CG - 1) / (kTcM * CG);   // items' m-index: 128 x CG rows
  if (force_splits) {
    p.splits = force_splits;
  } else {
    const TcSplit sc = tc_split_rule(p.na, p.nb, N, MODE == kTcTopk || ATM, 0, TN);
    p.splits = sc.splits;
    p.chain = sc.chain;
  }
  p.per = (p.tiles_n + p.splits - 1) / p.splits;
  p.splits = (p.tiles_n + p.per - 1) / p.per;                    // no empty splits
  p.mtiles = mtiles;
  p.nitems = mtiles * p.splits;
  if (p.chain && !p.done) return cudaErrorInvalidValue;
  if (p.chain) {
    e = cudaMemsetAsync(p.done, 0, mtiles * sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
  }
  const uint32_t smem = p.stages * kSB + fixed;
  auto kern = tc_pairs_kernel<MODE, KC, CG>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (!p.item_ctr) return cudaErrorInvalidValue;
  e = cudaMemsetAsync(p.item_ctr, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(TcRoles<MODE>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent: every CTA co-resident (the chained top-k waits on other CTAs' items)
  uint64_t units = (uint64_t)num_sms() / CG;
  if (CG > 1) {
    int ncl = 0;
    cfg.gridDim = dim3((unsigned)(units * CG));
    if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) == cudaSuccess && ncl > 0) units = std::min<uint64_t>(units, (uint64_t)ncl);
    (void)cudaGetLastError();
  }
  uint64_t grid = std::min<uint64_t>(p.nitems, units);
  if (const char* g = std::getenv("BINSKETCH_TC_GRID"))
    grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, std::strtoull(g, nullptr, 10) / CG));
  cfg.gridDim = dim3((unsigned)(grid * CG));
  e = cudaLaunchKernelEx(&cfg, kern, ma, mb, p);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int MODE, int KC>
static cudaError_t tc_launch(const uint8_t* A8, const uint8_t* B8, TcParams& p, uint32_t N, uint32_t extra_bytes,
                             uint32_t force_splits, cudaStream_t s) {
  return tc_cg<MODE>(tc_kpad(N)) == 2 ? tc_launch_cg<MODE, KC, 2>(A8, B8, p, N, extra_bytes, force_splits, s)
                            : tc_launch_cg<MODE, KC, 1>(A8, B8, p, N, extra_bytes, force_splits, s);
}

cudaError_t launch_tc_andpopc(const uint8_t* A8, uint64_t na, const uint8_t* B8, uint64_t nb, uint32_t N,
                              int32_t* out, unsigned long long* ctr, cudaStream_t s) {
  if (na == 0 || nb == 0) return cudaSuccess;
  TcParams p = {};
  p.na = na; p.nb = nb; p.N = N; p.out_i32 = out; p.item_ctr = ctr;
  return tc_launch<kTcAndPopc, 128>(A8, B8, p, N, TcRoles<kTcAndPopc>::kEpi * 4 * 32 * (TcRoles<kTcAndPopc>::kCW + 1), 0, s);   // transposes
}

cudaError_t launch_tc_screen(const uint8_t* A8, uint64_t na, const uint8_t* B8, uint64_t nb, uint32_t N,
                             const int32_t* spb, const int32_t* perm, const uint16_t* tsuf, uint32_t nmp, uint2* lists,
                             uint32_t* lcnt, unsigned long long* ctr, uint32_t& splits, uint32_t& seg_cols,
                             cudaStream_t s) {
  splits = 0;
  seg_cols = 0;
  if (na == 0 || nb == 0) return cudaSuccess;
  TcParams p = {};
  p.na = na; p.nb = nb; p.N = N; p.pb = spb; p.perm = perm; p.tsuf = tsuf; p.nmp = nmp; p.lists = lists;
  p.lcnt = lcnt;
  p.item_ctr = ctr;
  // per epilogue warp: the tile's metadata (kTcN int2) and a 32 x 33 chunk of values
  const cudaError_t e = tc_launch<kTcScreen, 128>(A8, B8, p, N, TcRoles<kTcScreen>::kEpi * (kTcN * 8 + 32 * 33 * 4), 0, s);
  splits = p.splits;
  seg_cols = p.per * kTcN;   // list segment sp starts at column sp * seg_cols
  return e;
}

cudaError_t launch_tc_estimate(const uint8_t* A8, uint64_t na, const uint8_t* B8, uint64_t nb, uint32_t N,
                               uint32_t measure, const int32_t* pa, const int32_t* pb, const double* L, float* out,
                               unsigned long long* ctr, cudaStream_t s, bool bcs, double dcap, double ham_scale) {
  if (na == 0 || nb == 0) return cudaSuccess;
  TcParams p = {};
  p.na = na; p.nb = nb; p.N = N; p.measure = measure; p.pa = pa; p.pb = pb; p.L = L; p.out_f32 = out;
  p.bcs = bcs ? 1u : 0u; p.dcap = dcap; p.ham_scale = ham_scale;
  p.item_ctr = ctr;
  const uint32_t lb = ((N + 1) * 8 + 15) / 16 * 16;
  p.l_smem = (lb <= 64 * 1024) ? lb : 0;
  return tc_launch<kTcEstimate, 64>(A8, B8, p, N,
                                    p.l_smem + TcRoles<kTcEstimate>::kEpi * 4 * 4 * 32 * (TcRoles<kTcEstimate>::kCW + 1), 0, s);   // table + 4-plane transposes
}

// The fused top-k keeps the query tile in TMEM (kTcTopkT) when its widened rows fit 256 columns;
// BINSKETCH_TC_ATM=0 forces the shared-memory A operand (dev A/B).
static bool tc_topk_atm(uint32_t N) {
  if (const char* e = std::getenv("BINSKETCH_TC_ATM")) if (!std::strcmp(e, "0")) return false;
  return tc_kpad(N) <= 1024u;
}
static uint32_t tc_topk_tn(uint32_t N) { return tc_topk_atm(N) ? 128u : (uint32_t)kTcN; }

// Shared memory of the fused top-k besides the operand stages: per-row heaps (k x 128 x 12 B),
// per-group scratch, metadata ring, per-warp queues / candidates / owner masks, row state; and
// the staged cardinality table.
static uint32_t topk_heap_smem(uint32_t N, uint32_t k) {
  const uint32_t ne = tc_topk_atm(N) ? TcRoles<kTcTopkT>::kEpi : TcRoles<kTcTopk>::kEpi;
  return k * kTcM * 12 + (ne / 4) * 32 * kTcM * 4 + 4 * kTcN * 8 + ne * BSK_TOPK_QCAP * 8 + ne * 32 * 16 + ne * 32 * 4 + kTcM * 20;
}
static uint32_t topk_table_smem(uint32_t N) { return (uint32_t)((((uint64_t)N + 1) * 8 + 15) / 16 * 16); }

bool tc_topk_fits(uint32_t N, uint32_t k) {
  if (k > tc_topk_max_k() || N > tc_topk_max_n()) return false;
  const uint64_t stage = tc_topk_atm(N) ? 128ull * 128 : (uint64_t)TcGeom<64, 1>::kStageBytes;
  return 2048ull + topk_heap_smem(N, k) + topk_table_smem(N) + 2 * stage <= kTcSmemMax;
}

uint32_t tc_topk_max_k() { return 64; }

uint32_t tc_topk_max_n() { return 6143; }   // cardinality table (N+1 doubles) staged in shared memory

bool tc_sortable(uint32_t N) { return N <= 65536; }

cudaError_t launch_sort_by_popcount(const int32_t* pb, uint64_t n, uint32_t N, uint32_t* bins, int32_t* perm,
                                    int32_t* spb, cudaStream_t s, bool descending) {
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(bins, 0, (size_t)(N + 1) * 4, s);
  if (e != cudaSuccess) return e;
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms() * 8);
  pb_hist_kernel<<<(unsigned)blocks, 256, 0, s>>>(pb, n, N, descending ? 1u : 0u, bins);
  pb_scan_kernel<<<1, 1024, 0, s>>>(bins, N + 1);
  pb_scatter_kernel<<<(unsigned)blocks, 256, 0, s>>>(pb, n, N, descending ? 1u : 0u, bins, perm, spb);
  count_launch(3);
  return cudaGetLastError();
}


uint32_t tc_topk_splits(uint64_t nq, uint64_t ndb, uint32_t N, uint32_t k) {
  // partial lists per query in the workspace: 1 when the heaps are chained, else one per chunk
  if (nq == 0 || ndb == 0 || k == 0) return 1;
  const TcSplit r = tc_split_rule(nq, ndb, N, true, k, tc_topk_tn(N));
  return r.chain ? 1u : r.splits;
}

bool tc_topk_packed_queries(uint32_t N) { return tc_topk_atm(N); }

cudaError_t launch_tc_topk(const uint8_t* Q8, const uint32_t* Qsk, uint64_t nq, const uint8_t* D8, uint64_t ndb, uint32_t N,
                           uint32_t measure, uint32_t k, uint32_t flags, const int32_t* pq, const int32_t* qperm,
                           const int32_t* pd, const int32_t* perm, const double* L, bool prefilter, double* part_key,
                           int32_t* part_idx, int32_t* out_idx, float* out_score, unsigned long long* ctr,
                           unsigned int* done, int2* meta, cudaStream_t s) {
  if (nq == 0 || k == 0) return cudaSuccess;
  if (k > tc_topk_max_k()) return cudaErrorInvalidValue;
  TcParams p = {};
  p.na = nq; p.nb = ndb; p.N = N; p.measure = measure; p.k = k; p.flags = flags; p.pa = pq; p.pb = pd; p.L = L;
  p.perm = perm; p.qperm = qperm; p.item_ctr = ctr;
  p.lc = std::log1p(-1.0 / (double)N);
  p.prefilter = (prefilter && perm) ? 1u : 0u;   // the per-tile bound needs the popcount-sorted db
  p.part_key = part_key; p.part_idx = part_idx;
  const bool atm = tc_topk_atm(N);
  p.heap_smem = topk_heap_smem(N, k);
  const uint32_t lb = topk_table_smem(N);
  if (!tc_topk_fits(N, k)) return cudaErrorInvalidValue;   // the caller routes by tc_topk_fits
  p.l_topk_smem = lb;
  // splits computed with the device-independent rule (148) so the workspace matches
  const TcSplit sc = tc_split_rule(nq, ndb, N, true, k, tc_topk_tn(N));
  p.qsk = Qsk;
  p.qw = (N + 31) / 32;
  p.kp = tc_kpad(N);
  if (atm && !Qsk) return cudaErrorInvalidValue;
  p.chain = sc.chain;
  p.done = done;
  {
    const uint64_t npad = ((ndb + kTcN - 1) / kTcN) * kTcN;
    const uint64_t blocks = std::min<uint64_t>((npad + 255) / 256, (uint64_t)num_sms() * 8);
    tile_meta_kernel<<<(unsigned)blocks, 256, 0, s>>>(pd, perm, ndb, npad, meta);
    count_launch();
    p.meta = meta;
#if BSK_TOPK_STRICT
    if (measure == 1u) {   // (the strict bound is IP-only)
    int32_t* tmin = reinterpret_cast<int32_t*>(meta + npad);
    const uint32_t tn = tc_topk_tn(N);
    tile_min_kernel<<<(unsigned)(npad / tn), tn, 0, s>>>(meta, tmin);
    count_launch();
    p.tmin = tmin;
    }
#endif
  }
  cudaError_t e = atm ? tc_launch<kTcTopkT, 128>(Q8, D8, p, N, p.heap_smem + p.l_topk_smem, sc.splits, s)
                      : tc_launch<kTcTopk, 64>(Q8, D8, p, N, p.heap_smem + p.l_topk_smem, sc.splits, s);
  if (e != cudaSuccess) return e;
  const uint32_t lists = p.chain ? 1u : p.splits;
  if (lists != tc_topk_splits(nq, ndb, N, k)) return cudaErrorInvalidConfiguration;
  return launch_topk_merge(nq, lists, k, measure, part_key, part_idx, out_idx, out_score, s);
}

uint32_t tc_join_max_thresholds() { return kTcMaxThr; }

cudaError_t launch_tc_join(const uint8_t* Q8, uint64_t nq, const uint8_t* D8, uint64_t ndb, uint32_t N,
                           uint32_t measure, const double* tkey, const uint32_t* tslot, uint32_t nthr, uint32_t flags,
                           bool exact, const int32_t* pq, const int32_t* pd, const double* L, uint32_t* bits,
                           unsigned long long* ctr, cudaStream_t s) {
  if (nq == 0 || ndb == 0 || nthr == 0) return cudaSuccess;
  if (nthr > kTcMaxThr || (!exact && !L)) return cudaErrorInvalidValue;
  TcParams p = {};
  p.na = nq; p.nb = ndb; p.N = N; p.measure = measure; p.flags = flags; p.pa = pq; p.pb = pd; p.L = exact ? nullptr : L;
  p.item_ctr = ctr; p.bits = bits; p.wpr = (ndb + 31) / 32; p.nthr = nthr; p.exact = exact ? 1u : 0u;
  for (uint32_t t = 0; t < nthr; ++t) { p.tkey[t] = tkey[t]; p.tslot[t] = tslot[t]; }
  p.lc = std::log1p(-1.0 / (double)N);
  p.heap_smem = 0;
  const uint32_t lb = ((N + 1) * 8 + 15) / 16 * 16;
  p.l_topk_smem = (!exact && lb <= 64 * 1024) ? lb : 0u;   // else the table is read from global (L1)
  const uint32_t kJoinScratch = TcRoles<kTcJoin>::kEpi * (32 * nthr * 2 * 4 + 32 * (TcRoles<kTcJoin>::kCW + 1) * 4 + 64);
  // long K (the exact rows): 128-byte K stages (SWIZZLE_128B) — fewer, larger TMA transactions and
  // barrier round trips per MMA (exact join 67.7 -> 60.2 ms, K11); the scratch still leaves >= 4 stages
  if (exact && tc_kpad(N) >= 16384u && TcGeom<128, 2>::kStageBytes * 4 + p.l_topk_smem + kJoinScratch + 2048 <= kTcSmemMax)
    return tc_launch<kTcJoin, 128>(Q8, D8, p, N, p.heap_smem + p.l_topk_smem + kJoinScratch, 0, s);
  return tc_launch<kTcJoin, 64>(Q8, D8, p, N, p.heap_smem + p.l_topk_smem + kJoinScratch, 0, s);
}

}  // namespace bsk
