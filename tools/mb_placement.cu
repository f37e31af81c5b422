// Micro-benchmark (azimuth-sweep design): where does the block scheduler put the
// CTAs of co-resident thread-block clusters?  For the production shapes (C CTAs per cluster,
// T threads, S bytes of dynamic SMEM, load-balancing cluster policy as in az_cluster_launch)
// every CTA of a grid of max-active-clusters records (%smid, cluster id, rank); the host reports
// how many SMs are busy and whether the CTAs sharing an SM belong to the same cluster (then
// their per-panel phases -- HBM load, DSMEM push, peer wait -- are locked together).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_placement.cu -o /tmp/mb_placement
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <map>
#include <set>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void where(uint32_t* out, int spin) {
  extern __shared__ float4 sm[];
  uint32_t smid, rank, cl;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cl));
  if (threadIdx.x == 0) {
    sm[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    out[3 * blockIdx.x + 0] = smid;
    out[3 * blockIdx.x + 1] = cl;
    out[3 * blockIdx.x + 2] = rank;
  }
  // hold the SM long enough that every cluster of the grid is co-resident
  const long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

static void run(int C, int T, int smem) {
  CK(cudaFuncSetAttribute(where, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(where, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
  at[1].val.clusterSchedulingPolicyPreference = cudaClusterSchedulingPolicyLoadBalancing;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.gridDim = dim3(C);
  int ncl = 0;
  CK(cudaOccupancyMaxActiveClusters(&ncl, where, &cfg));
  cfg.gridDim = dim3(ncl * C);
  uint32_t* d;
  CK(cudaMalloc(&d, 3 * sizeof(uint32_t) * ncl * C));
  CK(cudaLaunchKernelEx(&cfg, where, d, 2000000));
  CK(cudaDeviceSynchronize());
  std::vector<uint32_t> h(3 * ncl * C);
  CK(cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost));
  std::map<uint32_t, std::vector<std::pair<uint32_t, uint32_t>>> by_sm;
  for (int b = 0; b < ncl * C; ++b) by_sm[h[3 * b]].push_back({h[3 * b + 1], h[3 * b + 2]});
  int same = 0, mixed = 0, single = 0;
  std::map<int, int> hist;
  for (auto& kv : by_sm) {
    hist[(int)kv.second.size()]++;
    if (kv.second.size() == 1) { ++single; continue; }
    std::set<uint32_t> cls;
    for (auto& p : kv.second) cls.insert(p.first);
    if (cls.size() == 1) ++same; else ++mixed;
  }
  printf("C=%2d T=%4d smem=%6d: %3d clusters, %3zu SMs busy; SMs with 1 CTA %d, >1 CTA of one cluster %d, "
         ">1 CTA of different clusters %d; CTAs/SM histogram:", C, T, smem, ncl, by_sm.size(), single, same, mixed);
  for (auto& kv : hist) printf(" %d:%d", kv.first, kv.second);
  printf("\n");
  // rank pairs sharing an SM in cluster 0
  printf("   cluster 0 SM-mates:");
  for (auto& kv : by_sm) {
    std::vector<uint32_t> r;
    for (auto& p : kv.second) if (p.first == h[1]) r.push_back(p.second);
    if (r.size() > 1) { printf(" {"); for (auto x : r) printf("%u ", x); printf("}"); }
  }
  printf("\n");
  CK(cudaFree(d));
}

int main() {
  // production shapes at c3 (profiles/experiments_r02.md): head/tail C=8 T=256 ~110/90 KB,
  // residual C=16 T=256 ~106 KB; c4 C=16 T=512 ~210 KB; and 64 KB variants
  run(8, 256, 110376);
  run(8, 256, 89912);
  run(16, 256, 105768);
  run(16, 512, 210480);
  run(16, 256, 60000);
  run(8, 256, 60000);
  run(4, 256, 110000);
  run(2, 256, 110000);
  return 0;
}
