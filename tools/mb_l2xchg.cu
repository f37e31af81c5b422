// Micro-benchmark (azimuth-sweep exchange design): the cluster all-to-all of a
// sweep panel through DSMEM (st.async, as the sweeps do) against the same exchange through an
// L2-resident global scratch (coalesced 16-byte stores, cluster barrier release/acquire,
// 16-byte loads), and a half/half mix -- "DSMEM and L2 bandwidth are additive".  Persistent
// clusters of C CTAs at 2 CTAs/SM, 32 KB per CTA per panel; optionally every panel also streams
// 32 KB in from and 32 KB out to HBM (the sweep's own traffic) to see the contention.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_l2xchg.cu -o /tmp/mb_l2xchg
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

constexpr int BYTES = 32768;
constexpr int V4 = BYTES / 16;          // float4 per CTA per panel

// MODE 0: DSMEM, 1: L2 scratch, 2: half DSMEM / half L2, 3: no exchange (the HBM stream alone).
// HBM: stream 32 KB in and out per panel.
template <int C, int MODE, bool HBM, int T>
__global__ void __launch_bounds__(T) xchg(int panels, float4* scratch, const float4* hin, float4* hout,
                                         size_t hbm_v4, float* sink) {
  extern __shared__ __align__(1024) float4 sm[];
  float4* buf = sm;                                            // DSMEM receive buffer
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  const uint32_t rank = crank();
  const int cid = blockIdx.x / C, ncl = gridDim.x / C;
  constexpr int DS = MODE == 0 ? V4 : MODE == 2 ? V4 / 2 : 0;   // float4 through DSMEM
  constexpr int L2N = MODE == 3 ? 0 : V4 - DS;                 // float4 through L2
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    if (DS) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(DS * 16) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  float acc = 0.f;
  const uint32_t base = sa(buf), bb = sa(&bar);
  // scratch layout per cluster: [parity][owner][src][L2N / C] float4
  float4* scl = scratch + (size_t)cid * 2 * C * L2N;
  for (int p = 0; p < panels; ++p) {
    const size_t hoff = ((size_t)(p * ncl + cid) * C + rank) * V4 % (hbm_v4 - V4);
    float4 hv[V4 / T];
    if (HBM) {
#pragma unroll
      for (int j = 0; j < V4 / T; ++j) hv[j] = hin[hoff + j * T + t];
    }
    if (DS) {
      for (int e = t; e < DS; e += T) {
        const uint32_t own = (uint32_t)(e / (DS / C));
        const uint32_t off = (uint32_t)((rank * (DS / C) + e % (DS / C)) * 16);
        const float4 v = make_float4((float)e, (float)p, 1.f, 2.f);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                     ::"r"(mapa(base + off, own)), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(mapa(bb, own))
                     : "memory");
      }
    }
    float4* sp = scl + (size_t)(p & 1) * C * L2N;
    if (L2N) {
      for (int e = t; e < L2N; e += T) {
        const int own = e / (L2N / C);
        sp[((size_t)own * C + rank) * (L2N / C) + e % (L2N / C)] = make_float4((float)e, (float)p, 1.f, 2.f);
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      for (int e = t; e < L2N; e += T) {
        const float4 v = sp[(size_t)rank * L2N + e];          // [owner = rank][src][...] block
        acc += v.x;
      }
    }
    if (DS) {
      asm volatile("{ .reg .pred q; WT: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra WT; }"
                   ::"r"(bb), "r"((uint32_t)(p & 1)) : "memory");
      for (int e = t; e < DS; e += T) acc += buf[e].x;
    }
    if (HBM) {
#pragma unroll
      for (int j = 0; j < V4 / T; ++j) {
        float4 v = hv[j];
        v.x += acc;
        hout[hoff + j * T + t] = v;
      }
    }
    __syncthreads();
    if (DS && t == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(DS * 16) : "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
  }
  if (acc == 1.2345f) *sink = acc;
}

template <int C, int MODE, bool HBM, int T>
void run(float4* scratch, const float4* hin, float4* hout, size_t hbm_v4) {
  auto k = xchg<C, MODE, HBM, T>;
  const int smem = 100 * 1024;                 // 2 CTAs per SM, as the sweeps
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (C > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
  attr[1].val.clusterSchedulingPolicyPreference = cudaClusterSchedulingPolicyLoadBalancing;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  int ncl = 0;
  cfg.gridDim = dim3(C);
  CK(cudaOccupancyMaxActiveClusters(&ncl, (const void*)k, &cfg));
  cfg.gridDim = dim3(C * ncl);
  float* sink;
  CK(cudaMalloc(&sink, 4));
  // the same total data as one c3 exchange: 512 MiB over all CTAs
  const int panels = (int)((512.0 * 1024 * 1024) / ((double)ncl * C * BYTES));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaLaunchKernelEx(&cfg, k, panels, scratch, hin, hout, hbm_v4, sink));
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  CK(cudaLaunchKernelEx(&cfg, k, panels, scratch, hin, hout, hbm_v4, sink));
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)ncl * C * panels * BYTES;
  printf("C=%2d %-6s %-8s T=%d clusters=%d panels=%d: %.3f ms for %.0f MB exchanged (%.0f GB/s)\n", C,
         MODE == 0 ? "DSMEM" : MODE == 1 ? "L2" : MODE == 2 ? "mix" : "none", HBM ? "+hbm" : "", T, ncl, panels, ms, bytes / 1e6,
         bytes / ms / 1e6);
  CK(cudaFree(sink));
}

int main() {
  float4 *scratch, *hin, *hout;
  const size_t hbm_v4 = (size_t)512 * 1024 * 1024 / 16;
  CK(cudaMalloc(&scratch, (size_t)64 * 1024 * 1024));
  CK(cudaMalloc(&hin, hbm_v4 * 16));
  CK(cudaMalloc(&hout, hbm_v4 * 16));
  CK(cudaMemset(hin, 0, hbm_v4 * 16));
  run<8, 0, false, 256>(scratch, hin, hout, hbm_v4);
  run<8, 1, false, 256>(scratch, hin, hout, hbm_v4);
  run<8, 2, false, 256>(scratch, hin, hout, hbm_v4);
  run<16, 0, false, 256>(scratch, hin, hout, hbm_v4);
  run<16, 1, false, 256>(scratch, hin, hout, hbm_v4);
  run<16, 2, false, 256>(scratch, hin, hout, hbm_v4);
  run<8, 0, true, 256>(scratch, hin, hout, hbm_v4);
  run<8, 1, true, 256>(scratch, hin, hout, hbm_v4);
  run<8, 2, true, 256>(scratch, hin, hout, hbm_v4);
  run<16, 0, true, 256>(scratch, hin, hout, hbm_v4);
  run<16, 1, true, 256>(scratch, hin, hout, hbm_v4);
  run<16, 2, true, 256>(scratch, hin, hout, hbm_v4);
  run<8, 3, true, 256>(scratch, hin, hout, hbm_v4);
  run<16, 3, true, 256>(scratch, hin, hout, hbm_v4);
  run<4, 3, true, 256>(scratch, hin, hout, hbm_v4);
  run<4, 0, true, 256>(scratch, hin, hout, hbm_v4);
  run<4, 1, true, 256>(scratch, hin, hout, hbm_v4);
  run<2, 1, true, 256>(scratch, hin, hout, hbm_v4);
  return 0;
}
