// Sparse-state schedule (NEXT-3, SURVEY.md 8(a) "Lower bound", 8(f) rank 3; world 1, k-rule):
// the ITA state between iterations is not the dense b = X + mu dX but, per column panel of the
// head/tail azimuth sweeps, the list of the b entries that can lie above the next threshold
// (Algorithm 1's X_i = E(b_(i-1); sigma_(i-1)) is k-sparse).  S5 (AZ_TAIL_SS)
// writes the list instead of a dense b, S1 (AZ_FWD_SS) and the next S5 scatter it into SMEM.
//   * the select's usual window path finds sigma_i inside the candidate window, and the list
//     holds every entry with |b|^2 in a bin >= the window's lowest: it contains supp(X_(i+1));
//   * when the select falls back to the full histogram, AZ_TAIL_SSD re-runs S5 writing the
//     dense b_i, the fallback kernels select on it, and ss_rebuild rebuilds the list from it;
//   * the last list becomes the dense X_I in ss_finalize.
// Every panel's list has room for the whole panel (capp = n_az W entries), so it cannot overflow.
#include "az.cuh"

namespace cssar {

int az_panel_width(int log_naz) {
  switch (log_naz) {
#define PW(L) case L: return AzShape<L, false>::C > 1 ? AzShape<L, false>::W : 0;
    PW(7) PW(8) PW(9) PW(10) PW(11) PW(12) PW(13) PW(14) PW(15)
#undef PW
    default: return 0;
  }
}

__global__ void ss_set_kernel(SelState* st, uint32_t* c0, uint32_t* c1, int npan) {
  st->ss_cnt[0] = c0;
  st->ss_cnt[1] = c1;
  st->ss_npan = npan;
  st->ss_fell = 0;
}

cudaError_t launch_ss_set(SelState* st, uint32_t* cnt0, uint32_t* cnt1, int npan, cudaStream_t s) {
  ss_set_kernel<<<1, 1, 0, s>>>(st, cnt0, cnt1, npan);
  return cudaGetLastError();
}

// One block per panel: the entries |b|^2 > sigma^2 of the panel's W columns (dense b) become
// the list S1 / S5 read next (the select has already advanced st->iter).
__global__ void __launch_bounds__(512) ss_rebuild_kernel(const float2* __restrict__ b, int n_az, int n_rg,
                                                         const SsLists L, const SelState* st, int force) {
  if (!force && !st->ss_fell) return;
  __shared__ uint32_t cnt;
  const int panel = blockIdx.x, W = L.W;
  const int li = (st->iter + 1) & 1;
  SsEntry* dst = L.ent[li] + (size_t)panel * L.capp;
  const uint32_t s2 = st->sigma2_bits;
  if (threadIdx.x == 0) cnt = 0u;
  __syncthreads();
  const long long nel = (long long)n_az * W;
  for (long long g = threadIdx.x; g < nel; g += blockDim.x) {
    const int row = (int)(g / W), w = (int)(g % W);
    const float2 v = b[(size_t)row * n_rg + (size_t)panel * W + w];
    if (mag2_bits(v) > s2) {
      const uint32_t pos = atomicAdd(&cnt, 1u);
      SsEntry e;
      e.row = (uint32_t)row;
      e.w = (uint32_t)w;
      e.v = v;
      dst[pos] = e;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) L.cnt[li][panel] = cnt;
}

cudaError_t launch_ss_rebuild(const float2* b, int n_az, int n_rg, const SsLists& L, const SelState* st, int force,
                              cudaStream_t s) {
  ss_rebuild_kernel<<<L.npan, 512, 0, s>>>(b, n_az, n_rg, L, st, force);
  return cudaGetLastError();
}

// X_I = E(b_(I-1); sigma_(I-1)) from the last list into the zeroed dense X
__global__ void __launch_bounds__(256) ss_finalize_kernel(float2* X, int n_rg, const SsLists L, int thr,
                                                          const SelState* st) {
  const int li = (st->iter + 1) & 1;
  const uint32_t s2 = st->sigma2_bits;
  const float sig = st->sigma;
  for (int panel = blockIdx.x; panel < L.npan; panel += gridDim.x) {
    const SsEntry* e = L.ent[li] + (size_t)panel * L.capp;
    const uint32_t n = L.cnt[li][panel];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const SsEntry x = e[i];
      X[(size_t)x.row * n_rg + (size_t)panel * L.W + x.w] = threshold(x.v, s2, sig, thr);
    }
  }
}

cudaError_t launch_ss_finalize(float2* X, int n_az, int n_rg, const SsLists& L, int thr, const SelState* st,
                               cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(X, 0, sizeof(float2) * (size_t)n_az * n_rg, s);
  if (e != cudaSuccess) return e;
  ss_finalize_kernel<<<L.npan < 4 * 148 ? L.npan : 4 * 148, 256, 0, s>>>(X, n_rg, L, thr, st);
  return cudaGetLastError();
}

}  // namespace cssar
