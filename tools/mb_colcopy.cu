// Micro-benchmark: achievable HBM bandwidth of the azimuth-sweep access pattern
// (column panels of W complex64 columns, rows r = c + C m of a cluster rank c), copied
// in place of an FFT.  Variants: per-thread LDG (the v0-v3 az kernels' pattern) and a
// persistent TMA (3-D tensor map) pipeline with NS SMEM stages.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_colcopy.cu -o /tmp/mb -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int NAZ = 8192, NRG = 8192, C = 8;

template <int W, int E>
__global__ void ldg_copy(const float2* __restrict__ in, float2* __restrict__ out) {
  constexpr int M = NAZ / C;
  const int tile = blockIdx.x;
  const int rank = tile % C, col0 = (tile / C) * W;
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int g = e * blockDim.x + threadIdx.x;
    const int w = g % W, m = g / W;
    v[e] = in[(size_t)(rank + C * m) * NRG + col0 + w];
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int g = e * blockDim.x + threadIdx.x;
    const int w = g % W, m = g / W;
    out[(size_t)(rank + C * m) * NRG + col0 + w] = v[e];
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int W, int NS, int M>
__global__ void __launch_bounds__(512, 1) tma_copy(const __grid_constant__ CUtensorMap tm, float2* __restrict__ out, int ntiles, int C, int contig) {
  constexpr int BM = M < 256 ? M : 256;
  constexpr uint32_t STAGE_BYTES = M * W * 8;
  extern __shared__ __align__(1024) unsigned char sm[];
  float2* stage = reinterpret_cast<float2*>(sm);
  __shared__ __align__(8) uint64_t full[NS];
  const int t = threadIdx.x;
  auto issue = [&](int tile, int s) {
    const int rank = tile % C, col0 = (tile / C) * W;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(STAGE_BYTES) : "memory");
#pragma unroll
    for (int b = 0; b < M / BM; ++b) {
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(sa(stage + (size_t)s * M * W + b * BM * W)), "l"(&tm), "r"(col0), "r"(contig ? b * BM : rank), "r"(contig ? rank : b * BM), "r"(sa(&full[s]))
          : "memory");
    }
  };
  if (t == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int it = 0;
  if (t == 0)
    for (int s = 0; s < NS; ++s) {
      const int tile = blockIdx.x + s * gridDim.x;
      if (tile < ntiles) issue(tile, s);
    }
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % NS;
    const uint32_t par = (it / NS) & 1;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(&full[s])), "r"(par) : "memory");
    const int rank = tile % C, col0 = (tile / C) * W;
    const float4* st4 = reinterpret_cast<const float4*>(stage + (size_t)s * M * W);
    for (int g = t; g < M * W / 2; g += blockDim.x) {
      const int wp = g % (W / 2), m = g / (W / 2);
      float4 v = st4[g];
      const int row = contig ? rank * M + m : rank + C * m;
      *reinterpret_cast<float4*>(out + (size_t)row * NRG + col0 + 2 * wp) = v;
    }
    __syncthreads();
    if (t == 0) {
      const int nt = tile + NS * gridDim.x;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (nt < ntiles) issue(nt, s);
    }
  }
}

__global__ void row_copy(const float4* __restrict__ in, float4* __restrict__ out, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
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

template <int W, int NS, int C>
void run_tma(PFN_cuTensorMapEncodeTiled enc, float2* in, float2* out, int ctas_per_sm, int contig = 0, int promo = 3) {
  constexpr int M = NAZ / C, BM = M < 256 ? M : 256;
  CUtensorMap tm;
  cuuint64_t dims[3] = {NRG, C, NAZ / C};
  cuuint64_t strides[2] = {(cuuint64_t)NRG * 8, (cuuint64_t)C * NRG * 8};
  cuuint32_t box[3] = {W, 1, BM};
  if (contig) {
    dims[1] = M; dims[2] = C;
    strides[0] = (cuuint64_t)NRG * 8; strides[1] = (cuuint64_t)M * NRG * 8;
    box[1] = BM; box[2] = 1;
  }
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return; }
  const size_t smem = (size_t)NS * M * W * 8;
  auto k = tma_copy<W, NS, M>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int ntiles = (NRG / W) * C;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * ctas_per_sm;
  float ms = timeit([&] { k<<<grid, 256, smem>>>(tm, out, ntiles, C, contig); });
  CK(cudaGetLastError());
  printf("tma  promo=%d W=%2d C=%2d %s NS=%d stage=%3zu KB grid=%d : %.3f ms  %.0f GB/s\n", promo, W, C, contig ? "contig" : "strided", NS, smem / NS / 1024, grid, ms,
         2.0 * NAZ * NRG * 8 / ms / 1e6);
}

template <int W, int E, int T>
void run_ldg(float2* in, float2* out) {
  const int ntiles = (NRG / W) * C;
  float ms = timeit([&] { ldg_copy<W, E><<<ntiles, T>>>(in, out); });
  CK(cudaGetLastError());
  printf("ldg  W=%2d E=%d T=%d : %.3f ms  %.0f GB/s\n", W, E, T, ms, 2.0 * NAZ * NRG * 8 / ms / 1e6);
}

int main() {
  float2 *in, *out;
  const size_t bytes = (size_t)NAZ * NRG * 8;
  CK(cudaMalloc(&in, bytes));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMemset(in, 1, bytes));
  PFN_cuTensorMapEncodeTiled enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  float ms = timeit([&] { row_copy<<<148 * 8, 512>>>((const float4*)in, (float4*)out, bytes / 16); });
  printf("row copy: %.3f ms  %.0f GB/s\n", ms, 2.0 * bytes / ms / 1e6);
  run_tma<8, 2, 16>(enc, in, out, 1);
  run_tma<2, 2, 2>(enc, in, out, 1);
  run_tma<2, 3, 2>(enc, in, out, 1);
  run_tma<2, 2, 2>(enc, in, out, 1, 0, 0);
  run_tma<2, 2, 2>(enc, in, out, 1, 0, 2);
  run_tma<2, 3, 4>(enc, in, out, 1);
  run_tma<2, 3, 4>(enc, in, out, 2);
  run_tma<2, 2, 4>(enc, in, out, 1, 1);
  run_tma<4, 1, 2>(enc, in, out, 1);
  run_tma<4, 2, 4>(enc, in, out, 1);
  run_tma<4, 3, 4>(enc, in, out, 1);
  run_tma<4, 2, 4>(enc, in, out, 1, 0, 0);
  run_tma<2, 1, 1>(enc, in, out, 1);
  run_tma<8, 2, 8>(enc, in, out, 1, 0, 0);
  run_tma<8, 2, 8>(enc, in, out, 1, 0, 2);
  return 0;
}
