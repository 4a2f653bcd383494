// bsk_device.cuh — small device helpers shared by the product kernels.
#pragma once
#include <cstdint>

#include "bsk_internal.cuh"

namespace bsk {

// mbarrier + 1-D bulk copy (TMA engine): build.cu's per-warp index stream, the pab-table
// top-k's row ring (pairs.cu).
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
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// generic-proxy accesses to a ring slot before the async proxy (bulk copy) overwrites it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// splitmix64 finalizer ("random mapping", reading R-G8).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

__device__ __forceinline__ uint32_t mod_n(uint64_t x, const ModN& m) {
  if (m.mask) return (uint32_t)x & m.mask;
  uint64_t q = __umul64hi(x, m.M);
  uint64_t r = x - q * (uint64_t)m.N;
  if (r >= m.N) r -= m.N;
  if (r >= m.N) r -= m.N;
  return (uint32_t)r;
}

// pi(i) = mix64(seed + (i+1)*gamma) mod N
__device__ __forceinline__ uint32_t pi_seeded(uint64_t seed, uint64_t i, const ModN& m) {
  return mod_n(mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ULL), m);
}

__device__ __forceinline__ void latch(unsigned int* status, unsigned int bits) {
  atomicOr(status, bits);
}

}  // namespace bsk
