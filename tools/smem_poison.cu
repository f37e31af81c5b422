// Debug aid: fill the shared memory of every SM with a NaN pattern (detects reads of
// uninitialised SMEM that silently reuse a previous kernel's leftovers).
#include <cuda_runtime.h>
#include <cstdint>
__global__ void poison(uint32_t pat) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < (int)(227 * 1024 / 4); i += blockDim.x) s[i] = pat;
  __syncthreads();
  if (s[threadIdx.x] == 0x12345678u) s[0] = 1;   // keep the stores
}
extern "C" int smem_poison(unsigned pat) {
  cudaFuncSetAttribute(poison, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  poison<<<148 * 4, 1024, 227 * 1024>>>(pat);
  return (int)cudaDeviceSynchronize();
}
