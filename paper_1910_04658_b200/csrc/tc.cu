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
//                   the MMAs of tile t+1.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

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
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t x, int32_t y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
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
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
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

}  // namespace tc

// ------------------------------------------------------------- expansion ---
// out[r][b] = bit b of row r (LSB-first words), b < 32W; zero for 32W <= b < Kp.
__global__ void expand_kernel(const uint32_t* __restrict__ sk, uint64_t n, uint32_t W, uint32_t Kp,
                              uint8_t* __restrict__ out) {
  const uint32_t chunks = Kp / 32;   // one 32-byte chunk per sketch word
  const uint64_t total = n * chunks;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / chunks;
    const uint32_t c = (uint32_t)(i - r * chunks);
    const uint32_t w = c < W ? __ldg(sk + r * W + c) : 0u;
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

// --------------------------------------------------------- pairs kernel ---
constexpr int kTcM = 128, kTcN = 256, kTcK = 128, kTcStages = 4;
constexpr uint32_t kTcABytes = kTcM * kTcK, kTcBBytes = kTcN * kTcK, kTcStageBytes = kTcABytes + kTcBBytes;
constexpr uint32_t kTcThreads = 192;                       // producer, MMA, 4 epilogue warps
constexpr uint32_t kTcSmem = kTcStages * kTcStageBytes + 1024 /* barriers */ + 1024 /* align slack */;
// instruction descriptor: D s32, A/B u8, K-major, N = 256, M = 128
constexpr uint32_t kTcIdesc = (2u << 4) | ((uint32_t)(kTcN >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);

struct TcParams {
  uint64_t na, nb;
  uint32_t nk;          // K stages per tile = Kp / 128
  uint32_t tiles_n;     // ceil(nb / 256)
  uint64_t ntiles;
  int32_t* out;         // kAndPopc: int32 [na][nb]
};

template <int MODE>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_pairs_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const uint32_t base = tc::saddr(smem);
  const uint32_t bars = base + kTcStages * kTcStageBytes;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (kTcStages + s); };
  auto tfull = [&](int a) { return bars + 8u * (2 * kTcStages + a); };
  auto tempty = [&](int a) { return bars + 8u * (2 * kTcStages + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * kTcStages + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kTcStages; ++s) { tc::mbar_init(full(s), 1); tc::mbar_init(empty(s), 1); }
    for (int a = 0; a < 2; ++a) { tc::mbar_init(tfull(a), 1); tc::mbar_init(tempty(a), 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tmem_slot));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tmem_slot));

  if (warp == 0) {
    if (lane == 0) {   // ---- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const int32_t m0 = (int32_t)((t / p.tiles_n) * kTcM), n0 = (int32_t)((t % p.tiles_n) * kTcN);
        for (uint32_t kc = 0; kc < p.nk; ++kc) {
          tc::mbar_wait(empty(stage), phase ^ 1u);
          const uint32_t sa = base + stage * kTcStageBytes;
          tc::mbar_expect_tx(full(stage), kTcStageBytes);
          tc::tma_load_2d(sa, &tmA, (int32_t)(kc * kTcK), m0, full(stage));
          tc::tma_load_2d(sa + kTcABytes, &tmB, (int32_t)(kc * kTcK), n0, full(stage));
          if (++stage == kTcStages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---- MMA issuer
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        tc::mbar_wait(tempty(acc), aphase ^ 1u);
        tc::fence_after();
        const uint32_t d = tmem + (uint32_t)acc * kTcN;
        for (uint32_t kc = 0; kc < p.nk; ++kc) {
          tc::mbar_wait(full(stage), phase);
          tc::fence_after();
          const uint32_t sa = base + stage * kTcStageBytes;
          const uint64_t da = tc::desc_sw128(sa), db = tc::desc_sw128(sa + kTcABytes);
#pragma unroll
          for (int kk = 0; kk < kTcK / 32; ++kk)   // K = 32 bytes per MMA: +2 in 16-B units
            tc::mma_u8(d, da + 2u * kk, db + 2u * kk, kTcIdesc, (kc | (uint32_t)kk) != 0u);
          tc::commit(empty(stage));                // frees the smem stage when these MMAs finish
          if (++stage == kTcStages) { stage = 0; phase ^= 1u; }
        }
        tc::commit(tfull(acc));                    // accumulator ready for the epilogue
        if (++acc == 2) { acc = 0; aphase ^= 1u; }
      }
    }
  } else {             // ---- epilogue: warp w reads TMEM lanes 32*(w%4) .. +31
    const uint32_t lb = 32u * (uint32_t)(warp & 3);
    const uint32_t row_in_tile = lb + (uint32_t)lane;
    int acc = 0;
    uint32_t aphase = 0;
    for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      const uint64_t m0 = (t / p.tiles_n) * kTcM, n0 = (t % p.tiles_n) * kTcN;
      tc::mbar_wait(tfull(acc), aphase);
      tc::fence_after();
      const uint64_t r = m0 + row_in_tile;
#pragma unroll 1
      for (int c = 0; c < kTcN; c += 32) {
        uint32_t v[32];
        tc::tmem_ld32(tmem + (lb << 16) + (uint32_t)acc * kTcN + (uint32_t)c, v);
        if (MODE == kAndPopc && r < p.na && n0 + c < p.nb) {
          int32_t* o = p.out + r * p.nb + n0 + c;
          const uint64_t left = p.nb - (n0 + c);   // > 0 here
          if (left >= 32 && ((reinterpret_cast<uintptr_t>(o) & 15u) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              __stcs(reinterpret_cast<int4*>(o + j), make_int4((int)v[j], (int)v[j + 1], (int)v[j + 2], (int)v[j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if ((uint64_t)j < left) __stcs(o + j, (int32_t)v[j]);
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(tempty(acc));
      if (++acc == 2) { acc = 0; aphase ^= 1u; }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
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

bool make_map(CUtensorMap* m, const uint8_t* ptr, uint64_t rows, uint32_t Kp, uint32_t box_rows) {
  EncodeTiled enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {Kp, rows};
  const cuuint64_t strides[1] = {Kp};
  const cuuint32_t box[2] = {(cuuint32_t)kTcK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

uint32_t tc_kpad(uint32_t N) { return ((N + 127) / 128) * 128; }

cudaError_t launch_expand(const uint32_t* sk, uint64_t n, uint32_t N, uint8_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint32_t W = (N + 31) / 32, Kp = tc_kpad(N);
  const uint64_t total = n * (Kp / 32);
  const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, (uint64_t)num_sms() * 16);
  expand_kernel<<<(unsigned)blocks, 256, 0, s>>>(sk, n, W, Kp, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_tc_andpopc(const uint8_t* A8, uint64_t na, const uint8_t* B8, uint64_t nb, uint32_t N,
                              int32_t* out, cudaStream_t s) {
  if (na == 0 || nb == 0) return cudaSuccess;
  const uint32_t Kp = tc_kpad(N);
  if (na > 0x7fffffffull || nb > 0x7fffffffull) return cudaErrorInvalidValue;
  alignas(64) CUtensorMap ma, mb;
  if (!make_map(&ma, A8, na, Kp, kTcM) || !make_map(&mb, B8, nb, Kp, kTcN)) return cudaErrorNotSupported;
  TcParams p;
  p.na = na; p.nb = nb; p.nk = Kp / kTcK;
  p.tiles_n = (uint32_t)((nb + kTcN - 1) / kTcN);
  p.ntiles = ((na + kTcM - 1) / kTcM) * (uint64_t)p.tiles_n;
  p.out = out;
  cudaError_t e = cudaFuncSetAttribute(tc_pairs_kernel<kAndPopc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
  if (e != cudaSuccess) return e;
  uint64_t grid = std::min<uint64_t>(p.ntiles, (uint64_t)num_sms());
  if (const char* g = std::getenv("BINSKETCH_TC_GRID")) grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, std::strtoull(g, nullptr, 10)));
  tc_pairs_kernel<kAndPopc><<<(unsigned)grid, kTcThreads, kTcSmem, s>>>(ma, mb, p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsk
