// Sparse-X' schedule of the multi-GPU path: replaces S1 (threshold +
// azimuth FFT on column slabs + transpose #1) by
//   compact : X = E(b; sigma) of this rank's column slab -> (row, col, value) list (k-rule:
//             at most k nonzeros over all ranks)
//   fold    : every rank pulls all ranks' lists (peer memory) and folds them into a length
//             m = n_az / world array F[n2][col] = sum_{n = n2 mod m} w_N^{p n} X[n][col]
//   az FFT  : the m-point azimuth DFT of F gives Doppler bins p + world k2 of F_eta X for all
//             n_rg gates, i.e. rank p's row slab in a cyclic bin distribution
// because X^[p + P k2] = sum_{n2} w_m^{n2 k2} (w_N^{n2 p} sum_{n1} w_P^{n1 p} x[m n1 + n2])
// and w_N^{n2 p} w_P^{n1 p} = w_N^{p n} for n = m n1 + n2.  The range sweep then reads the
// cyclic slab (RgArgs::row_step = world) and stores into the column slabs as usual.
#include "device_ops.cuh"

namespace cssar {

__global__ void __launch_bounds__(256) sx_compact_kernel(const float2* __restrict__ b, long long n, int log_ncol,
                                                         int col0, const SelState* st, int thr, SxEntry* list,
                                                         uint32_t* count, uint32_t cap) {
  const uint32_t s2 = st->sigma2_bits;
  const float sig = st->sigma;
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // whole warps iterate together (the ballot needs every lane)
  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
    const long long i = base + lane;
    float2 x = make_float2(0.f, 0.f);
    if (i < n) x = threshold(b[i], s2, sig, thr);
    const bool keep = i < n && (x.x != 0.f || x.y != 0.f);
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    if (!m) continue;
    uint32_t w0 = 0;
    if (lane == 0) w0 = atomicAdd(count, (uint32_t)__popc(m));
    w0 = __shfl_sync(0xffffffffu, w0, 0);
    if (keep) {
      const uint32_t slot = w0 + (uint32_t)__popc(m & ((1u << lane) - 1u));
      if (slot < cap) {
        SxEntry e;
        e.row = (int)(i >> log_ncol);
        e.col = col0 + (int)(i & ((1 << log_ncol) - 1));
        e.v = x;
        list[slot] = e;
      }
    }
  }
  __threadfence_system();     // the list is read by the peers over NVLink after the barrier
}

// Fold pass n1: the entries of rows n1 m .. n1 m + m - 1 (each (n2 = row mod m, col) at most
// once per pass), F[n2][col] += w_N^{p row} X[row][col].  Passes run n1 = 0 .. world-1 in
// stream order, so every F element sums its <= world terms in a fixed order: run-to-run
// deterministic, without floating-point atomics.
__global__ void __launch_bounds__(256) sx_fold_kernel(const SxLists L, int p, int log_n, int m, int n_rg, int n1,
                                                      float2* __restrict__ F) {
  const uint32_t nmask = (1u << log_n) - 1u;
  const float inv_n = 1.0f / (float)(1u << log_n);
  for (int q = 0; q < L.world; ++q) {
    const uint32_t cnt = min(*L.count[q], L.cap);
    const SxEntry* __restrict__ e = L.list[q];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
      const SxEntry x = e[i];
      if (x.row / m != n1) continue;
      // w_N^{p n} = exp(-2 pi i (p n mod N) / N), the fraction exact in fp32 (N <= 2^15)
      const uint32_t ph = ((uint32_t)p * (uint32_t)x.row) & nmask;
      float sn, cs;
      sincospif(-2.0f * (float)ph * inv_n, &sn, &cs);
      const float2 v = cmul(x.v, make_float2(cs, sn));
      float2* dst = F + (size_t)(x.row & (m - 1)) * n_rg + x.col;
      *dst = *dst + v;
    }
  }
}

cudaError_t launch_sx_compact(const float2* b, long long n, int log_ncol, int col0, const SelState* st, int thr,
                              SxEntry* list, uint32_t* count, uint32_t cap, int sm_count, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  sx_compact_kernel<<<4 * sm_count, 256, 0, s>>>(b, n, log_ncol, col0, st, thr, list, count, cap);
  return cudaGetLastError();
}

cudaError_t launch_sx_fold(const SxLists& L, int p, int log_n, int m, int n_rg, float2* F, int sm_count,
                           cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(F, 0, sizeof(float2) * (size_t)m * n_rg, s);
  if (e != cudaSuccess) return e;
  for (int n1 = 0; n1 < L.world; ++n1) {
    sx_fold_kernel<<<4 * sm_count, 256, 0, s>>>(L, p, log_n, m, n_rg, n1, F);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace cssar
