// microbench.cu — K9: calibrate the per-SM issue rates the rooflines use (sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
// Prints one JSON line per measurement: ops per SM clock (clock64 in-kernel, so
// independent of the SM frequency) and the wall-clock rate.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

// Per block: (SM id, clock64 at start, clock64 at end). clock64 is a per-SM counter, so the
// host measures each SM's busy span as max(end) - min(start) over the blocks it ran: the
// per-clock rate then does not assume that all blocks of an SM started together.
__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
#define RECORD(cyc, t0, t1) do { if (threadIdx.x == 0) { cyc[3 * blockIdx.x] = smid(); cyc[3 * blockIdx.x + 1] = (t0); cyc[3 * blockIdx.x + 2] = (t1); } } while (0)

// ~0.5 s of dependent FMAs on every SM before the measurements, so the clock is at its boost value.
__global__ void k_warm(float* out, int iters) {
  float x = threadIdx.x * 1e-3f;
  for (int i = 0; i < iters; ++i) x = fmaf(x, 0.999f, 1e-4f);
  if (x == 12345.f) out[0] = x;
}

// AND + POPC + add into 16 independent accumulators (the estimate mainloop pattern, 4x4 tile).
__global__ void k_andpopc(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  uint32_t a[4], b[4], acc[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) { a[i] = seed * (threadIdx.x + 3 * i + 1); b[i] = seed ^ (threadIdx.x * 7 + i); }
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i * 4 + j] += __popc(a[i] & b[j]);
#pragma unroll
    for (int i = 0; i < 4; ++i) { a[i] = __funnelshift_l(a[i], a[i], 1); b[i] = __funnelshift_l(b[i], b[i], 3); }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  RECORD(cyc, t0, t1);
}

// POPC only (operands rotate): 16 POPC + 16 IADD per iteration per thread.
__global__ void k_popc(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  uint32_t a[16], acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { a[i] = seed * (threadIdx.x + i + 1); acc[i] = 0; }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] += __popc(a[i] ^ it);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  RECORD(cyc, t0, t1);
}

// LOP3 only: 16 independent xor/and chains.
__global__ void k_lop3(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  uint32_t a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed * (threadIdx.x + i + 1);
  uint32_t c = seed * 3u + threadIdx.x;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = (a[i] ^ c) & (a[(i + 1) & 15] | 0x5555u);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  RECORD(cyc, t0, t1);
}

// Shared atomicOr at random addresses inside a 4 KB tile (the build kernel's scatter).
__global__ void k_atoms(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  __shared__ uint32_t tile[8][1024];
  for (int i = threadIdx.x; i < 8 * 1024; i += blockDim.x) (&tile[0][0])[i] = 0;
  uint32_t x = seed ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS / 4; ++it) {
    x = x * 1664525u + 1013904223u;
    atomicOr(&tile[w][x >> 22], 1u << (x & 31));
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = tile[w][threadIdx.x & 1023];
  RECORD(cyc, t0, t1);
}

// Random 4-byte gathers from a global table of `mask+1` words through L1 (__ldg).
__global__ void k_gather(const uint32_t* __restrict__ tab, uint32_t mask, uint32_t seed, uint32_t* out,
                         unsigned long long* cyc) {
  uint32_t x = seed ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu);
  uint32_t s = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS / 16; ++it) {
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { x = x * 1664525u + 1013904223u; v[u] = __ldg(tab + ((x >> 4) & mask)); }
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  RECORD(cyc, t0, t1);
}

// Random 2-byte gathers from a shared-memory table (the smem-pi variant).
__global__ void k_lds16(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  __shared__ uint16_t tab[16384];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) tab[i] = (uint16_t)(i * 7);
  uint32_t x = seed ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu);
  uint32_t s = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS / 16; ++it) {
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { x = x * 1664525u + 1013904223u; v[u] = tab[x >> 18]; }
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  RECORD(cyc, t0, t1);
}

// In-kernel splitmix64 pi evaluation (the build_seeded variant): mix64 + mod N.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL; z ^= z >> 27; z *= 0x94D049BB133111EBULL; z ^= z >> 31; return z;
}
__global__ void k_hash(uint64_t seed, uint64_t M, uint32_t N, uint32_t* out, unsigned long long* cyc) {
  uint32_t s = 0;
  uint32_t i = threadIdx.x + blockIdx.x * 977u;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS / 16; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint64_t x = mix64(seed + (uint64_t)(i + u + 1) * 0x9E3779B97F4A7C15ULL);
      uint64_t q = __umul64hi(x, M);
      uint64_t r = x - q * N;
      if (r >= N) r -= N;
      if (r >= N) r -= N;
      s += (uint32_t)r;
    }
    i += 4 * 1315423911u;
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  RECORD(cyc, t0, t1);
}


// Legacy warp-level binary MMA (mma.sync m16n8k256 b1, AND + POPC): 4 independent accumulator
// sets per warp. One instruction = 16 x 8 x 256 = 32768 AND-popcount bit pairs per warp (1024
// per thread). ptxas lowers it on sm_100a to an emulation subroutine (MOVM.U4TO8 + 8 x
// IMMA.16832.U8.U8), so this measures what the toolchain actually offers for binary MMA.
__global__ void k_b1mma(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  uint32_t a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + i + 1);
  b[0] = seed ^ threadIdx.x; b[1] = seed + 7u * threadIdx.x;
  int c[4][4] = {};
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS / 16; ++it) {
#pragma unroll
    for (int s = 0; s < 4; ++s)
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[s][0]), "+r"(c[s][1]), "+r"(c[s][2]), "+r"(c[s][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  int sum = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) sum += c[s][0] + c[s][1] + c[s][2] + c[s][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)sum;
  RECORD(cyc, t0, t1);
}

// Legacy warp-level int8 MMA (mma.sync m16n8k32 u8): 16 x 8 x 32 = 4096 MACs per warp instruction
// (128 per thread), 4 independent accumulator sets — the baseline the b1 emulation is built on.
__global__ void k_i8mma(uint32_t seed, uint32_t* out, unsigned long long* cyc) {
  uint32_t a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + i + 1);
  b[0] = seed ^ threadIdx.x; b[1] = seed + 7u * threadIdx.x;
  int c[4][4] = {};
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int s = 0; s < 4; ++s)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[s][0]), "+r"(c[s][1]), "+r"(c[s][2]), "+r"(c[s][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  int sum = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) sum += c[s][0] + c[s][1] + c[s][2] + c[s][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)sum;
  RECORD(cyc, t0, t1);
}

template <typename F>
static int run(const char* name, double ops_per_thread, int blocks, int threads, F launch, int sms) {
  uint32_t* out;
  unsigned long long* cyc;
  CK(cudaMalloc(&out, (size_t)blocks * threads * 4));
  CK(cudaMalloc(&cyc, (size_t)blocks * 24));
  launch(out, cyc);
  CK(cudaDeviceSynchronize());
  double best_rate[3], best_ms[3], best_span[3];
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    launch(out, cyc);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long* h = new unsigned long long[3 * (size_t)blocks];
    CK(cudaMemcpy(h, cyc, (size_t)blocks * 24, cudaMemcpyDeviceToHost));
    // per SM: ops of its blocks over its busy span
    const int MAXSM = 512;
    unsigned long long lo[MAXSM], hi[MAXSM];
    int nb[MAXSM];
    for (int i = 0; i < MAXSM; ++i) { lo[i] = ~0ull; hi[i] = 0; nb[i] = 0; }
    for (int i = 0; i < blocks; ++i) {
      const int sm = (int)h[3 * i] % MAXSM;
      lo[sm] = h[3 * i + 1] < lo[sm] ? h[3 * i + 1] : lo[sm];
      hi[sm] = h[3 * i + 2] > hi[sm] ? h[3 * i + 2] : hi[sm];
      nb[sm]++;
    }
    double rates[MAXSM];
    double span_sum = 0;
    int m = 0;
    for (int i = 0; i < MAXSM; ++i)
      if (nb[i]) { rates[m++] = ops_per_thread * threads * nb[i] / (double)(hi[i] - lo[i]); span_sum += (double)(hi[i] - lo[i]); }
    // median over SMs
    for (int i = 1; i < m; ++i) for (int j = i; j > 0 && rates[j] < rates[j - 1]; --j) { double t = rates[j]; rates[j] = rates[j - 1]; rates[j - 1] = t; }
    best_rate[rep] = m ? rates[m / 2] : 0;
    best_ms[rep] = ms;
    best_span[rep] = m ? span_sum / m : 0;
    delete[] h;
  }
  // median of the 3 repetitions
  int idx[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i) for (int j = i; j > 0 && best_rate[idx[j]] < best_rate[idx[j - 1]]; --j) { int t = idx[j]; idx[j] = idx[j - 1]; idx[j - 1] = t; }
  const int r = idx[1];
  const double total = ops_per_thread * blocks * threads;
  printf("{\"bench\": \"%s\", \"ops_per_clk_per_sm\": %.2f, \"ops_per_s\": %.4e, \"ms\": %.4f, \"mean_sm_span_cycles\": %.0f, "
         "\"implied_mhz\": %.0f, \"reps\": 3, \"method\": \"median over SMs of ops / (max end - min start) by clock64; median of 3\"}\n",
         name, best_rate[r], total / (best_ms[r] * 1e-3), best_ms[r], best_span[r], best_span[r] / (best_ms[r] * 1e-3) / 1e6);
  cudaFree(out);
  cudaFree(cyc);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int T = 256;
  const int B = sms * 4;   // 4 x 256 threads per SM, all resident
  {
    float* w;
    CK(cudaMalloc(&w, 4));
    for (int i = 0; i < 4; ++i) k_warm<<<sms * 4, 256>>>(w, 1 << 20);
    CK(cudaDeviceSynchronize());
    cudaFree(w);
  }
  run("andpopc_word (LOP3+POPC+IADD per word)", 16.0 * ITERS, B, T,
      [&](uint32_t* o, unsigned long long* c) { k_andpopc<<<B, T>>>(12345u, o, c); }, sms);
  run("popc", 16.0 * ITERS, B, T, [&](uint32_t* o, unsigned long long* c) { k_popc<<<B, T>>>(777u, o, c); }, sms);
  run("lop3", 16.0 * ITERS, B, T, [&](uint32_t* o, unsigned long long* c) { k_lop3<<<B, T>>>(99u, o, c); }, sms);
  run("atoms_or_random_4KB", ITERS / 4.0, B, T, [&](uint32_t* o, unsigned long long* c) { k_atoms<<<B, T>>>(5u, o, c); }, sms);
  const uint32_t sizes[] = {1u << 14, 1u << 18, 1u << 20, 1u << 22};  // words: 64 KB, 1 MB, 4 MB, 16 MB
  uint32_t* tab;
  CK(cudaMalloc(&tab, (1u << 22) * 4));
  CK(cudaMemset(tab, 1, (1u << 22) * 4));
  for (uint32_t s : sizes) {
    char name[64];
    snprintf(name, sizeof(name), "ldg_gather_random_%uKB", s * 4 / 1024);
    run(name, ITERS / 16.0 * 8, B, T,
        [&](uint32_t* o, unsigned long long* c) { k_gather<<<B, T>>>(tab, s - 1, 3u, o, c); }, sms);
  }
  run("lds16_gather_random", ITERS / 16.0 * 8, sms, T * 4,
      [&](uint32_t* o, unsigned long long* c) { k_lds16<<<sms, T * 4>>>(3u, o, c); }, sms);
  const uint32_t N = 1224;
  run("splitmix64_pi_eval", ITERS / 16.0 * 4, B, T,
      [&](uint32_t* o, unsigned long long* c) { k_hash<<<B, T>>>(1ull, ~0ull / N, N, o, c); }, sms);
  cudaFree(tab);
  // binary / int8 warp MMA (legacy mma.sync): "ops" = AND-popcount bit pairs resp. u8 MACs
  run("mma_sync_b1_andpopc_bitpairs (emulated on sm_100a)", (ITERS / 16) * 4 * 1024.0, B, T,
      [&](uint32_t* o, unsigned long long* c) { k_b1mma<<<B, T>>>(0x9e3779b9u, o, c); }, sms);
  run("mma_sync_u8_macs", ITERS * 4 * 128.0, B, T,
      [&](uint32_t* o, unsigned long long* c) { k_i8mma<<<B, T>>>(0x9e3779b9u, o, c); }, sms);
  return 0;
}
