// Micro-benchmark (layout decision): HBM bandwidth of the azimuth-sweep and
// range-sweep access patterns on an 8192 x 8192 complex64 array in a TILED layout
//   [row / TR][col / TC][row % TR][col % TC]      (tiles of TR x TC samples, contiguous)
// az : one CTA owns TC whole columns (no cluster): TMA 2-D boxes of 256 tiles, the full
//      N x TC column group in SMEM, written back with 16-byte stores;
// rg : one CTA per row, 32 samples per thread (the range sweep's register layout).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_tiled.cu -o tools/mb_tiled
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int N = 8192;
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int TR, int TC>
__device__ __forceinline__ size_t tidx(int r, int c) {
  return (((size_t)(r / TR) * (N / TC) + (c / TC)) * TR + (r % TR)) * TC + (c % TC);
}

template <int TR, int TC>
__global__ void __launch_bounds__(512) az_copy(const __grid_constant__ CUtensorMap tm, float2* __restrict__ out) {
  constexpr int BOX = 256;                              // tiles per TMA box
  constexpr uint32_t BYTES = N * TC * 8;
  extern __shared__ __align__(1024) unsigned char sm[];
  float2* stage = reinterpret_cast<float2*>(sm);
  __shared__ __align__(8) uint64_t full;
  const int t = threadIdx.x;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int it = 0;
  for (int cg = blockIdx.x; cg < N / TC; cg += gridDim.x, ++it) {
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full)), "r"(BYTES) : "memory");
      for (int b = 0; b < (N / TR) / BOX; ++b)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(sa(stage + (size_t)b * BOX * TR * TC)), "l"(&tm), "r"(0), "r"(cg), "r"(b * BOX), "r"(sa(&full))
            : "memory");
    }
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(&full)),
                 "r"((uint32_t)(it & 1)) : "memory");
    const float4* s4 = reinterpret_cast<const float4*>(stage);
    for (int g = t; g < N * TC / 2; g += blockDim.x) {
      const int tile = g / (TR * TC / 2), within = g % (TR * TC / 2);
      const size_t o = ((size_t)tile * (N / TC) + cg) * (TR * TC) + 2 * within;
      *reinterpret_cast<float4*>(out + o) = s4[g];
    }
    __syncthreads();
  }
}

template <int TR, int TC>
__global__ void __launch_bounds__(256) rg_copy(const float2* __restrict__ in, float2* __restrict__ out) {
  constexpr int E = 32;
  const int t = threadIdx.x, row = blockIdx.x;
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = in[tidx<TR, TC>(row, e * 256 + t)];
#pragma unroll
  for (int e = 0; e < E; ++e) out[tidx<TR, TC>(row, e * 256 + t)] = v[e];
}

template <class F>
float timeit(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

static PFN_cuTensorMapEncodeTiled enc;

template <int TR, int TC>
void run(float2* in, float2* out, int per_sm, int promo) {
  // 3-D map over the tiled array: {TR*TC samples, column group, tile row}
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)TR * TC, (cuuint64_t)N / TC, (cuuint64_t)N / TR};
  cuuint64_t strides[2] = {(cuuint64_t)TR * TC * 8, (cuuint64_t)N * TR * 8};
  cuuint32_t box[3] = {(cuuint32_t)TR * TC, 1, 256};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return; }
  const size_t smem = (size_t)N * TC * 8;
  CK(cudaFuncSetAttribute(az_copy<TR, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  float ms = timeit([&] { az_copy<TR, TC><<<148 * per_sm, 512, smem>>>(tm, out); });
  CK(cudaGetLastError());
  float ms2 = timeit([&] { rg_copy<TR, TC><<<N, 256>>>(in, out); });
  CK(cudaGetLastError());
  const double gb = 2.0 * N * N * 8 / 1e6;
  printf("tile %dx%d (%3d B) az %d/SM promo %d: %.3f ms %5.0f GB/s | rg: %.3f ms %5.0f GB/s\n", TR, TC, TR * TC * 8,
         per_sm, promo, ms, gb / ms, ms2, gb / ms2);
}

int main() {
  float2 *in, *out;
  const size_t bytes = (size_t)N * N * 8;
  CK(cudaMalloc(&in, bytes));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMemset(in, 1, bytes));
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  run<8, 1>(in, out, 3, 3);
  run<8, 1>(in, out, 2, 3);
  run<4, 1>(in, out, 3, 3);
  run<16, 1>(in, out, 3, 3);
  run<4, 2>(in, out, 1, 3);
  run<8, 2>(in, out, 1, 3);
  run<2, 2>(in, out, 1, 3);
  run<8, 1>(in, out, 3, 0);
  run<8, 1>(in, out, 3, 1);
  return 0;
}
