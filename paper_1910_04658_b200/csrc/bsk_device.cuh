// bsk_device.cuh — small device helpers shared by the product kernels.
#pragma once
#include <cstdint>

#include "bsk_internal.cuh"

namespace bsk {

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
