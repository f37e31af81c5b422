// Micro-benchmark (azimuth-sweep design, DESIGN.md §9 "what would move it next"): how much of
// the cluster all-to-all can a panel pipeline hide behind the HBM stream?  The data movement
// of a head sweep (32 KB per CTA per panel: HBM in -> DSMEM all-to-all -> HBM out, 2 CTAs/SM,
// persistent clusters of C CTAs) in two structures:
//   sync : every thread loads its part of the panel (LDG), pushes (st.async), waits, stores (STG)
//          -- the structure of tools/mb_l2xchg.cu "+hbm" and of the sweeps' per-panel loop;
//   pipe : the HBM side moved to the TMA engine -- bulk loads two panels ahead into a 2-stage
//          ring, the received panel written back by one bulk store straight from the receive
//          buffer -- so the threads only push and wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_pipe.cu -o /tmp/mb_pipe
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
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  asm volatile("{ .reg .pred q; WT: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra WT; }"
               ::"r"(sa(b)), "r"(par) : "memory");
}

constexpr int BYTES = 32768;
constexpr int V4 = BYTES / 16;

template <int C, bool PIPE, int T>
__global__ void __launch_bounds__(T) xchg(int panels, const float4* hin, float4* hout, size_t hbm_v4, float* sink) {
  extern __shared__ __align__(1024) float4 sm[];
  float4* recv = sm;                        // [V4]
  float4* stage = sm + V4;                  // [2][V4] (PIPE)
  __shared__ __align__(8) uint64_t rbar, lbar[2];
  const int t = threadIdx.x;
  const uint32_t rank = crank();
  const int cid = blockIdx.x / C, ncl = gridDim.x / C;
  auto hoff = [&](int p) -> size_t { return ((size_t)(p * ncl + cid) * C + rank) * V4 % (hbm_v4 - V4); };
  if (t == 0) {
    mb_init(&rbar, 1);
    mb_init(&lbar[0], 1);
    mb_init(&lbar[1], 1);
    mb_expect(&rbar, BYTES);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (PIPE) {
      for (int s = 0; s < 2 && s < panels; ++s) {
        mb_expect(&lbar[s], BYTES);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(stage + s * V4)), "l"(hin + hoff(s)), "r"(BYTES), "r"(sa(&lbar[s])) : "memory");
      }
    }
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  float acc = 0.f;
  const uint32_t rb = sa(recv), bb = sa(&rbar);
  for (int p = 0; p < panels; ++p) {
    float4 hv[V4 / T];
    const float4* src = nullptr;
    if (PIPE) {
      mb_wait(&lbar[p & 1], (uint32_t)((p >> 1) & 1));
      src = stage + (p & 1) * V4;
    } else {
#pragma unroll
      for (int j = 0; j < V4 / T; ++j) hv[j] = hin[hoff(p) + j * T + t];
    }
    if (p > 0) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");   // peers' receive buffers free
    for (int e = t; e < V4; e += T) {
      const uint32_t own = (uint32_t)(e / (V4 / C));
      const uint32_t off = (uint32_t)((rank * (V4 / C) + e % (V4 / C)) * 16);
      const float4 v = PIPE ? src[e] : make_float4((float)e, (float)p, 1.f, 2.f);
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                   ::"r"(mapa(rb + off, own)), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(mapa(bb, own)) : "memory");
    }
    if (PIPE) {
      __syncthreads();                                  // stage read: refill it two panels ahead
      if (t == 0 && p + 2 < panels) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mb_expect(&lbar[p & 1], BYTES);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(stage + (p & 1) * V4)), "l"(hin + hoff(p + 2)), "r"(BYTES), "r"(sa(&lbar[p & 1]))
                     : "memory");
      }
    }
    mb_wait(&rbar, (uint32_t)(p & 1));                 // all C parts of this panel landed
    if (PIPE) {
      if (t == 0) {                                     // write the received panel back by one bulk store
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(hout + hoff(p)), "r"(rb), "r"(BYTES) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // receive buffer read
        mb_expect(&rbar, BYTES);
      }
      acc += recv[t].x;
      __syncthreads();
    } else {
#pragma unroll
      for (int j = 0; j < V4 / T; ++j) {
        float4 v = hv[j];
        v.x += recv[j * T + t].x;
        hout[hoff(p) + j * T + t] = v;
      }
      __syncthreads();
      if (t == 0) mb_expect(&rbar, BYTES);
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");    // my receive buffer is free
  }
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (PIPE && t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (acc == 1.2345f) *sink = acc;
}

template <int C, bool PIPE, int T>
void run(const float4* hin, float4* hout, size_t hbm_v4) {
  auto k = xchg<C, PIPE, T>;
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
  const int panels = (int)((512.0 * 1024 * 1024) / ((double)ncl * C * BYTES));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaLaunchKernelEx(&cfg, k, panels, hin, hout, hbm_v4, sink));
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  CK(cudaLaunchKernelEx(&cfg, k, panels, hin, hout, hbm_v4, sink));
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("C=%2d %-4s T=%d clusters=%d panels=%d: %.3f ms (512 MiB in + out through HBM, exchanged over DSMEM)\n", C,
         PIPE ? "pipe" : "sync", T, ncl, panels, ms);
  CK(cudaFree(sink));
}

int main() {
  float4 *hin, *hout;
  const size_t hbm_v4 = (size_t)512 * 1024 * 1024 / 16;
  CK(cudaMalloc(&hin, hbm_v4 * 16));
  CK(cudaMalloc(&hout, hbm_v4 * 16));
  CK(cudaMemset(hin, 0, hbm_v4 * 16));
  for (int r = 0; r < 2; ++r) {
    run<8, false, 256>(hin, hout, hbm_v4);
    run<8, true, 256>(hin, hout, hbm_v4);
    run<16, false, 256>(hin, hout, hbm_v4);
    run<16, true, 256>(hin, hout, hbm_v4);
  }
  return 0;
}
