// Micro-benchmark (layout decision): HBM bandwidth of the two sweep access
// patterns on an 8192 x 8192 complex64 array stored
//   row-major      [row][col]                      (round-1 layout)
//   panel-major    [col / W][row][col % W]         (column panels of W contiguous)
// Each test copies the whole array (read + write = 2 x 512 MiB) with the sweep's pattern:
//   az   : a TMA box per CTA-rank of a cluster-style panel (rows rank + C m, W columns)
//   rg   : one CTA per row, thread loads of W-wide segments (range sweep), B rows per CTA
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_layout.cu -o /tmp/mbl
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int NAZ = 8192, NRG = 8192;
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// az pattern: tile = (panel, rank); stage = M x W rows rank + C m; stores the same elements
template <int W, int C, int NS, bool PM>
__global__ void __launch_bounds__(256, 2) az_copy(const __grid_constant__ CUtensorMap tm, float2* __restrict__ out,
                                                  int ntiles) {
  constexpr int M = NAZ / C, BM = M < 256 ? M : 256;
  constexpr uint32_t STAGE_BYTES = M * W * 8;
  extern __shared__ __align__(1024) unsigned char sm[];
  float2* stage = reinterpret_cast<float2*>(sm);
  __shared__ __align__(8) uint64_t full[NS];
  const int t = threadIdx.x;
  auto issue = [&](int tile, int s) {
    const int rank = tile % C, panel = tile / C;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(STAGE_BYTES) : "memory");
#pragma unroll
    for (int b = 0; b < M / BM; ++b) {
      // row-major map {col, rank, m}; panel-major map {w, rank, m, panel}
      if (PM)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
            ::"r"(sa(stage + (size_t)s * M * W + b * BM * W)), "l"(&tm), "r"(0), "r"(rank), "r"(b * BM), "r"(panel),
              "r"(sa(&full[s])) : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(sa(stage + (size_t)s * M * W + b * BM * W)), "l"(&tm), "r"(panel * W), "r"(rank), "r"(b * BM),
              "r"(sa(&full[s])) : "memory");
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
    const int rank = tile % C, panel = tile / C;
    const float4* st4 = reinterpret_cast<const float4*>(stage + (size_t)s * M * W);
    for (int g = t; g < M * W / 2; g += blockDim.x) {
      const int wp = g % (W / 2), m = g / (W / 2);
      const float4 v = st4[g];
      // output rows k + M q style (contiguous blocks of M/C rows) like the sweeps' epilogues
      const int q = m / (M / C), kk = m % (M / C);
      const int row = kk + rank * (M / C) + M * q;
      float2* dst = PM ? out + ((size_t)panel * NAZ + row) * W + 2 * wp : out + (size_t)row * NRG + panel * W + 2 * wp;
      *reinterpret_cast<float4*>(dst) = v;
    }
    __syncthreads();
    if (t == 0) {
      const int nt = tile + NS * gridDim.x;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (nt < ntiles) issue(nt, s);
    }
  }
}

// rg pattern: CTA = B rows; thread e-loop over the row's elements j = e*T + t (32 per thread)
template <int W, int B, bool PM>
__global__ void __launch_bounds__(256) rg_copy(const float2* __restrict__ in, float2* __restrict__ out) {
  constexpr int E = 32;
  const int t = threadIdx.x;
  for (int b = 0; b < B; ++b) {
    const int row = blockIdx.x * B + b;
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int j = e * 256 + t;
      v[e] = PM ? in[((size_t)(j / W) * NAZ + row) * W + (j % W)] : in[(size_t)row * NRG + j];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int j = e * 256 + t;
      if (PM) out[((size_t)(j / W) * NAZ + row) * W + (j % W)] = v[e];
      else out[(size_t)row * NRG + j] = v[e];
    }
  }
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

template <int W, int C, int NS, bool PM>
void run_az(float2* in, float2* out, int per_sm, int promo) {
  constexpr int M = NAZ / C, BM = M < 256 ? M : 256;
  CUtensorMap tm;
  CUresult r;
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (PM) {
    cuuint64_t dims[4] = {W, C, NAZ / C, NRG / W};
    cuuint64_t strides[3] = {(cuuint64_t)W * 8, (cuuint64_t)C * W * 8, (cuuint64_t)NAZ * W * 8};
    cuuint32_t box[4] = {W, 1, BM, 1};
    r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[3] = {NRG, C, NAZ / C};
    cuuint64_t strides[2] = {(cuuint64_t)NRG * 8, (cuuint64_t)C * NRG * 8};
    cuuint32_t box[3] = {W, 1, BM};
    r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return; }
  const size_t smem = (size_t)NS * M * W * 8;
  auto k = az_copy<W, C, NS, PM>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int ntiles = (NRG / W) * C;
  const int grid = 148 * per_sm;
  float ms = timeit([&] { k<<<grid, 256, smem>>>(tm, out, ntiles); });
  CK(cudaGetLastError());
  printf("az  %s W=%2d C=%2d NS=%d stage=%3zu KB %d/SM promo=%d : %.3f ms  %5.0f GB/s\n", PM ? "panel-major" : "row-major  ",
         W, C, NS, smem / NS / 1024, per_sm, promo, ms, 2.0 * NAZ * NRG * 8 / ms / 1e6);
}

template <int W, int B, bool PM>
void run_rg(float2* in, float2* out) {
  float ms = timeit([&] { rg_copy<W, B, PM><<<NAZ / B, 256>>>(in, out); });
  CK(cudaGetLastError());
  printf("rg  %s W=%2d B=%d : %.3f ms  %5.0f GB/s\n", PM ? "panel-major" : "row-major  ", W, B, ms,
         2.0 * NAZ * NRG * 8 / ms / 1e6);
}

int main() {
  float2 *in, *out;
  const size_t bytes = (size_t)NAZ * NRG * 8;
  CK(cudaMalloc(&in, bytes));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMemset(in, 1, bytes));
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  run_rg<4, 1, false>(in, out);
  run_rg<4, 1, true>(in, out);
  run_rg<8, 1, true>(in, out);
  run_rg<16, 1, true>(in, out);
  run_rg<4, 2, true>(in, out);
  run_az<4, 8, 1, false>(in, out, 2, 3);
  run_az<4, 8, 2, false>(in, out, 1, 3);
  run_az<8, 16, 1, false>(in, out, 2, 3);
  run_az<4, 8, 1, true>(in, out, 2, 3);
  run_az<4, 8, 2, true>(in, out, 1, 3);
  run_az<4, 8, 1, true>(in, out, 2, 0);
  run_az<8, 16, 1, true>(in, out, 2, 3);
  run_az<8, 8, 1, true>(in, out, 1, 3);
  run_az<2, 4, 1, true>(in, out, 2, 3);
  run_az<2, 2, 1, true>(in, out, 1, 3);
  return 0;
}
