// Micro-benchmark (azimuth-sweep exchange design): DSMEM all-to-all throughput
// of st.async with 8-byte (v2.f32) vs 16-byte (v4.f32) stores.  Persistent clusters of C CTAs
// (2 per SM); each "panel" every CTA pushes BYTES to the C owners (1/C of its data each) and
// waits on its mbarrier for BYTES from all peers -- the exchange of the azimuth sweeps alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_dsmem.cu -o tools/mb_dsmem
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ uint32_t crank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int C, int VEC, int T>
__global__ void __launch_bounds__(T) xchg(int panels, float* sink) {
  constexpr int BYTES = 32768;
  extern __shared__ __align__(1024) float4 sm[];
  float2* buf = reinterpret_cast<float2*>(sm);                 // receive buffer [BYTES]
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  const uint32_t rank = crank();
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(BYTES) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  float acc = 0.f;
  const uint32_t base = sa(buf), bb = sa(&bar);
  constexpr int ELEMS = BYTES / 8;                             // float2 elements pushed per CTA
  for (int p = 0; p < panels; ++p) {
    // element e goes to owner e / (ELEMS / C), slot rank * (ELEMS / C) + e % (ELEMS / C)
    if (VEC == 0) {
    } else if (VEC == 2) {
      for (int e = t; e < ELEMS; e += T) {
        const uint32_t own = (uint32_t)(e / (ELEMS / C));
        const uint32_t off = (uint32_t)((rank * (ELEMS / C) + e % (ELEMS / C)) * 8);
        const float2 v = make_float2((float)e, (float)p);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
                     ::"r"(mapa(base + off, own)), "f"(v.x), "f"(v.y), "r"(mapa(bb, own)) : "memory");
      }
    } else {
      for (int e = 2 * t; e < ELEMS; e += 2 * T) {
        const uint32_t own = (uint32_t)(e / (ELEMS / C));
        const uint32_t off = (uint32_t)((rank * (ELEMS / C) + e % (ELEMS / C)) * 8);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                     ::"r"(mapa(base + off, own)), "f"((float)e), "f"((float)p), "f"((float)e + 1), "f"((float)p),
                       "r"(mapa(bb, own)) : "memory");
      }
    }
    if (VEC == 0) {
      // bulk DSMEM copies: the CTA's 32 KB source (in SMEM after the receive buffer), one
      // cp.async.bulk of BYTES/C per owner, issued by one thread (the TMA engine moves it)
      const uint32_t src = base + BYTES;
      if (t == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int q = 0; q < C; ++q)
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(mapa(base + rank * (BYTES / C), (uint32_t)q)), "r"(src + q * (BYTES / C)), "r"(BYTES / C),
                "r"(mapa(bb, (uint32_t)q)) : "memory");
      }
    }
    asm volatile("{ .reg .pred q; WT: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra WT; }"
                 ::"r"(bb), "r"((uint32_t)(p & 1)) : "memory");
    acc += buf[(t * 7) % ELEMS].x;
    __syncthreads();
    if (t == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(BYTES) : "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
  }
  if (acc == 1.2345f) *sink = acc;
}

template <int C, int VEC, int T>
void run(int per_sm) {
  auto k = xchg<C, VEC, T>;
  const int smem = 100 * 1024;                 // 2 CTAs per SM, as the sweeps
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (C > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  int ncl = 0;
  cfg.gridDim = dim3(C * 64);
  CK(cudaOccupancyMaxActiveClusters(&ncl, (const void*)k, &cfg));
  cfg.gridDim = dim3(C * ncl);
  float* sink;
  CK(cudaMalloc(&sink, 4));
  const int panels = 200;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaLaunchKernelEx(&cfg, k, panels, sink));
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  CK(cudaLaunchKernelEx(&cfg, k, panels, sink));
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)ncl * C * panels * 32768.0 * (C - 1) / C;    // remote bytes
  printf("C=%2d %s T=%d clusters=%d: %.3f ms, remote %.0f GB/s (%.1f B/cyc/SM at 1.965 GHz over %d CTAs)\n", C,
         VEC == 0 ? "bulk" : VEC == 2 ? "v2  " : "v4  ",
         T, ncl, ms, bytes / ms / 1e6, bytes / (ms * 1e-3) / 1.965e9 / (ncl * C / 2.0), ncl * C);
  (void)per_sm;
}

int main() {
  run<16, 0, 256>(2);
  run<8, 0, 256>(2);
  run<4, 0, 256>(2);
  run<2, 0, 256>(2);
  run<16, 2, 256>(2);
  run<16, 4, 256>(2);
  run<8, 2, 256>(2);
  run<8, 4, 256>(2);
  run<4, 2, 256>(2);
  run<4, 4, 256>(2);
  run<2, 2, 256>(2);
  run<2, 4, 256>(2);
  run<16, 2, 512>(2);
  run<16, 4, 512>(2);
  return 0;
}
