// Prototype / micro-benchmark (az-sweep design decision): an azimuth sweep
// WITHOUT thread-block clusters on a tiled layout [row / TR][col / 2][TR][2]: one CTA per SM
// holds a whole 2-column panel (8192 x 2 complex64 = 128 KB) in SMEM, loaded by TMA, and runs
// the library's in-SMEM FFT engine (radices 16 / 32 / 16) over it.
//   fwd : threshold prologue + forward FFT + tiled store            (S1 shape)
//   res : inverse FFT -> r = Y - g -> forward FFT + tiled store     (S3 shape, no mask)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_1302_3120_b200/csrc tools/mb_aztile.cu -o tools/mb_aztile
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "fft_engine.cuh"

using namespace cssar;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int LOGN = 13, N = 1 << LOGN, NRG = 8192, W = 2, E = 32, T = N * W / E, TR = 4;
using En = Engine<LOGN, W, T, true, E>;

__device__ __forceinline__ size_t tid_(int r, int c) {
  return (((size_t)(r / TR) * (NRG / W) + (c / W)) * TR + (r % TR)) * W + (c % W);
}

// transform(+1) -> mid -> transform(-1) keeping the result in registers (Engine::conv without the store)
template <class Load, class Mid>
__device__ __forceinline__ void for_groups_conv(float2* s, float2 (&v)[E], Load&& ld, Mid&& mid, const float2* tw) {
  const int t = threadIdx.x;
  En::template for_groups<En::template lr<false>(0)>(v, t, ld);
  En::template passes_from<+1, false, 0>(s, v, t, tw);
  En::template for_groups<En::template lr<false>(En::P - 1)>(v, t, mid);
  En::template passes_from<-1, true, 0>(s, v, t, tw);
}

template <int MODE>
__global__ void __launch_bounds__(T, 1) azt(const __grid_constant__ CUtensorMap tm, const float2* __restrict__ Y,
                                            float2* __restrict__ out, const float2* __restrict__ twg, float sig2) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  float2* s = reinterpret_cast<float2*>(smraw);
  float2* tw = s + N * W;
  __shared__ __align__(8) uint64_t full;
  const int t = threadIdx.x;
  copy_table_async(tw, twg, En::TW_TOTAL + (En::TW_TOTAL & 1), t, T);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int cg) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full)), "r"(N * W * 8) : "memory");
    for (int b = 0; b < (N / TR) / 256; ++b)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(smem_u32(s + (size_t)b * 256 * TR * W)), "l"(&tm), "r"(0), "r"(cg), "r"(b * 256), "r"(smem_u32(&full))
          : "memory");
  };
  if (t == 0 && (int)blockIdx.x < NRG / W) issue(blockIdx.x);
  int it = 0;
  for (int cg = blockIdx.x; cg < NRG / W; cg += gridDim.x, ++it) {
    asm volatile("{ .reg .pred p; WT: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra WT; }"
                 ::"r"(smem_u32(&full)), "r"((uint32_t)(it & 1)) : "memory");
    constexpr int R0 = 1 << En::template lr<false>(0);
    auto ld = [&](int w, int j, float2* x) {
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        float2 v = s[(j + r * (N / R0)) * W + w];
        if (MODE == 0) {
          const float m2 = v.x * v.x + v.y * v.y;
          v = m2 > sig2 ? v : make_float2(0.f, 0.f);
        }
        x[r] = v;
      }
    };
    float2 v[E];
    if constexpr (MODE == 0) {
      En::template run_keep<-1>(s, v, ld, tw);
    } else {
      constexpr int RL = 1 << En::template lr<false>(En::P - 1);
      auto mid = [&](int w, int j, float2* x) {
        float2 y[RL];
#pragma unroll
        for (int r = 0; r < RL; ++r) y[r] = __ldg(Y + tid_(j + r * (N / RL), cg * W + w));
#pragma unroll
        for (int r = 0; r < RL; ++r) x[r] = y[r] - x[r] * 0.011f;
      };
      for_groups_conv(s, v, ld, mid, tw);
    }
    __syncthreads();                               // the stage is free: prefetch the next panel
    if (t == 0 && cg + (int)gridDim.x < NRG / W) issue(cg + gridDim.x);
    constexpr int RLa = 1 << En::template lr<(MODE != 0)>(En::P - 1);
    En::template for_groups<En::template lr<(MODE != 0)>(En::P - 1)>(v, t, [&](int w, int j, float2* x) {
#pragma unroll
      for (int r = 0; r < RLa; ++r) out[tid_(j + r * (N / RLa), cg * W + w)] = x[r] * 0.011f;
    });
  }
}

__global__ void tw_kernel(float2* dst) { En::build_tw(dst, threadIdx.x, blockDim.x); }

int main() {
  const size_t n = (size_t)N * NRG;
  float2 *in, *out, *Y, *tw;
  CK(cudaMalloc(&in, n * 8));
  CK(cudaMalloc(&out, n * 8));
  CK(cudaMalloc(&Y, n * 8));
  CK(cudaMalloc(&tw, (En::TW_TOTAL + 2) * 8));
  CK(cudaMemset(in, 0, n * 8));
  CK(cudaMemset(Y, 0, n * 8));
  tw_kernel<<<1, 256>>>(tw);
  PFN_cuTensorMapEncodeTiled enc;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)TR * W, (cuuint64_t)NRG / W, (cuuint64_t)N / TR};
  cuuint64_t strides[2] = {(cuuint64_t)TR * W * 8, (cuuint64_t)NRG * TR * 8};
  cuuint32_t box[3] = {(cuuint32_t)TR * W, 1, 256};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const size_t smem = (size_t)N * W * 8 + (En::TW_TOTAL + 2) * 8;
  CK(cudaFuncSetAttribute(azt<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(azt<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  printf("T=%d smem=%zu TW=%d\n", T, smem, En::TW_TOTAL);
  for (int mode = 0; mode < 2; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&] {
      if (mode == 0) azt<0><<<148, T, smem>>>(tm, Y, out, tw, 1.0f);
      else azt<1><<<148, T, smem>>>(tm, Y, out, tw, 1.0f);
    };
    run(); run();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) run();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    ms /= 20;
    const double bytes = (mode == 0 ? 16.0 : 24.0) * n;
    printf("%s: %.3f ms  (%.0f GB/s algorithmic)\n", mode == 0 ? "fwd (S1 shape)" : "res (S3 shape)", ms, bytes / ms / 1e6);
  }
  return 0;
}
