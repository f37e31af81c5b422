// Host helpers of the persistent azimuth cluster kernel: TMA tensor-map encoding (driver
// entry point via the runtime, no -lcuda) and the co-resident cluster count.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>

namespace cssar {

bool pdl_enabled() {
  static const bool on = [] { const char* v = std::getenv("CSSAR_PDL"); return v && std::atoi(v) != 0; }();
  return on;
}

std::mutex& az_setup_mutex() {
  static std::mutex m;
  return m;
}

// promo: L2 promotion of the loads (CUtensorMapL2promotion; < 0 = the default, 256 B)
cudaError_t make_az_tensor_map(CUtensorMap* tm, const void* base, int n_rg, int N, int C, int W, int BM, int promo) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc),
                                            cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !enc) {
      enc = nullptr;
      return e != cudaSuccess ? e : cudaErrorNotSupported;
    }
  }
  const cuuint64_t dims[3] = {(cuuint64_t)n_rg, (cuuint64_t)C, (cuuint64_t)(N / C)};
  const cuuint64_t strides[2] = {(cuuint64_t)n_rg * 8u, (cuuint64_t)C * (cuuint64_t)n_rg * 8u};
  const cuuint32_t box[3] = {(cuuint32_t)W, 1u, (cuuint32_t)BM};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   promo >= 0 ? (CUtensorMapL2promotion)promo : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int az_max_clusters(const void* kernel, int C, int T, size_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * 64));
  cfg.blockDim = dim3((unsigned)T);
  cfg.dynamicSmemBytes = smem;
  // cluster scheduling: load balancing (measured: 15 instead of 14 co-resident 16-CTA clusters
  // for the c3 residual sweep, 0.84 -> 0.78 ms); CSSAR_AZ_POLICY overrides (0 = driver default)
  static const int policy = [] { const char* e = std::getenv("CSSAR_AZ_POLICY"); return e ? std::atoi(e) : 2; }();
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
  attr[1].val.clusterSchedulingPolicyPreference = (cudaClusterSchedulingPolicy)policy;
  cfg.attrs = attr;
  cfg.numAttrs = policy ? 2 : 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess) return 0;
  return n;
}

void az_log_config(int logn, int mode, int C, int W, int NS, int T, size_t smem, int clusters) {
  if (std::getenv("CSSAR_VERBOSE"))
    std::fprintf(stderr, "libcssar: az_cluster_kernel<%d,%d> C=%d W=%d NS=%d T=%d smem=%zu -> %d clusters\n", logn,
                 mode, C, W, NS, T, smem, clusters);
}

}  // namespace cssar
