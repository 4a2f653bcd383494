// tmem_pack_probe.cu — dev probe: the column -> register mapping of
// tcgen05.ld.32x32b.x16.pack::16b on sm_100a (which TMEM columns land in which register half).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_pack_probe tools/tmem_pack_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(uint32_t* out) {
  __shared__ uint32_t taddr_s;
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  const uint32_t t = taddr_s;
  if (threadIdx.x < 32) {
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = 1000u * lane + (uint32_t)j;   // column j of lane: 1000*lane + j
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n\ttcgen05.wait::st.sync.aligned;"
                 ::"r"(t), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                 "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
                 "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
                 "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
    uint32_t p[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
                 "tcgen05.wait::ld.sync.aligned;"
                 : "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3]), "=r"(p[4]), "=r"(p[5]), "=r"(p[6]), "=r"(p[7]), "=r"(p[8]),
                   "=r"(p[9]), "=r"(p[10]), "=r"(p[11]), "=r"(p[12]), "=r"(p[13]), "=r"(p[14]), "=r"(p[15]) : "r"(t) : "memory");
    for (int j = 0; j < 16; ++j) out[lane * 16 + j] = p[j];
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
}
int main() {
  uint32_t* d; cudaMalloc(&d, 32 * 16 * 4);
  probe<<<1, 128>>>(d);
  uint32_t h[512];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"err\": \"%s\", \"lane0\": [", cudaGetErrorString(e));
  for (int j = 0; j < 16; ++j) printf("%s\"%u|%u\"", j ? ", " : "", h[j] & 0xffffu, h[j] >> 16);
  printf("], \"lane5\": [");
  for (int j = 0; j < 16; ++j) printf("%s\"%u|%u\"", j ? ", " : "", h[80 + j] & 0xffffu, h[80 + j] >> 16);
  printf("]}\n");
  return 0;
}
