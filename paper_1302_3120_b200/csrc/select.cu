// Exact k-rule select (S6), fixed-lambda step, state init, finalize, mask packing.
#include "device_ops.cuh"

namespace cssar {

template <int LOGN>
cudaError_t az_dispatch_mode(int mode, int n_rg, const AzArgs& a, cudaStream_t s);
template <int LOGN>
size_t az_table_count_t(bool resid);
template <int LOGN>
cudaError_t az_table_fill_t(bool resid, float2* dst, cudaStream_t s);
extern template cudaError_t az_dispatch_mode<7>(int, int, const AzArgs&, cudaStream_t);
extern template cudaError_t az_dispatch_mode<8>(int, int, const AzArgs&, cudaStream_t);
extern template cudaError_t az_dispatch_mode<9>(int, int, const AzArgs&, cudaStream_t);
extern template cudaError_t az_dispatch_mode<10>(int, int, const AzArgs&, cudaStream_t);
extern template cudaError_t az_dispatch_mode<11>(int, int, const AzArgs&, cudaStream_t);
extern template cudaError_t az_dispatch_mode<12>(int, int, const AzArgs&, cudaStream_t);
extern template cudaError_t az_dispatch_mode<13>(int, int, const AzArgs&, cudaStream_t);
extern template cudaError_t az_dispatch_mode<14>(int, int, const AzArgs&, cudaStream_t);
extern template cudaError_t az_dispatch_mode<15>(int, int, const AzArgs&, cudaStream_t);

size_t az_table_count(int log_naz, bool resid) {
  switch (log_naz) {
#define AZT(L) case L: return az_table_count_t<L>(resid);
    AZT(7) AZT(8) AZT(9) AZT(10) AZT(11) AZT(12) AZT(13) AZT(14) AZT(15)
#undef AZT
    default: return 0;
  }
}

cudaError_t az_table_fill(int log_naz, bool resid, float2* dst, cudaStream_t s) {
  switch (log_naz) {
#define AZT(L) case L: return az_table_fill_t<L>(resid, dst, s);
    AZT(7) AZT(8) AZT(9) AZT(10) AZT(11) AZT(12) AZT(13) AZT(14) AZT(15)
#undef AZT
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_az(int log_naz, int mode, int n_rg, const AzArgs& a, cudaStream_t s) {
  switch (log_naz) {
    case 7: return az_dispatch_mode<7>(mode, n_rg, a, s);
    case 8: return az_dispatch_mode<8>(mode, n_rg, a, s);
    case 9: return az_dispatch_mode<9>(mode, n_rg, a, s);
    case 10: return az_dispatch_mode<10>(mode, n_rg, a, s);
    case 11: return az_dispatch_mode<11>(mode, n_rg, a, s);
    case 12: return az_dispatch_mode<12>(mode, n_rg, a, s);
    case 13: return az_dispatch_mode<13>(mode, n_rg, a, s);
    case 14: return az_dispatch_mode<14>(mode, n_rg, a, s);
    case 15: return az_dispatch_mode<15>(mode, n_rg, a, s);
    default: return cudaErrorInvalidValue;
  }
}


// ------------------------------------------------------------------ select (S6)
// suffix sums over a SMEM histogram of NB bins with 1024 threads: above[b] = sum_{b' > b} cnt[b']
template <int NB>
CSSAR_DEV void block_suffix(const uint32_t* cnt, uint32_t* above, uint32_t* warp_tot) {
  constexpr int PER = NB / 1024;
  const int t = threadIdx.x;
  // thread t owns bins (from the top) t*PER .. t*PER+PER-1, i.e. bins NB-1-t*PER-e
  uint32_t loc[PER];
  uint32_t sum = 0;
#pragma unroll
  for (int e = 0; e < PER; ++e) { loc[e] = cnt[NB - 1 - (t * PER + e)]; sum += loc[e]; }
  // inclusive warp scan
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if ((t & 31) >= o) inc += y;
  }
  if ((t & 31) == 31) warp_tot[t >> 5] = inc;
  __syncthreads();
  if (t < 32) {
    uint32_t w = warp_tot[t], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (t >= o) wi += y;
    }
    warp_tot[t] = wi - w;           // exclusive prefix of warp totals
  }
  __syncthreads();
  uint32_t run = warp_tot[t >> 5] + inc - sum;   // exclusive prefix for this thread
#pragma unroll
  for (int e = 0; e < PER; ++e) { above[NB - 1 - (t * PER + e)] = run; run += loc[e]; }
  __syncthreads();
}

// find bin B with above[B] <= rank < above[B] + cnt[B]; returns via out (bin, rank-in-bin, above)
template <int NB>
CSSAR_DEV void find_rank_bin(const uint32_t* cnt, const uint32_t* above, unsigned long long rank,
                             int* out_bin, uint32_t* out_r, uint32_t* out_above) {
  for (int b = threadIdx.x; b < NB; b += blockDim.x) {
    const unsigned long long ab = above[b], c = cnt[b];
    if (c && ab <= rank && rank < ab + c) {
      *out_bin = b;
      *out_r = (uint32_t)(rank - ab);
      *out_above = (uint32_t)ab;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024) sel_coarse_kernel(long long k, SelState* st, const uint32_t* hist) {
  pdl_wait();
  __shared__ uint32_t cnt[HIST_BINS], above[HIST_BINS], wt[32];
  __shared__ int sb;
  __shared__ uint32_t sr, sa;
  const int t = threadIdx.x;
  for (int i = t; i < HIST_BINS; i += 1024) cnt[i] = hist[i];
  if (t == 0) { sb = -1; sr = 0; sa = 0; }
  __syncthreads();
  block_suffix<HIST_BINS>(cnt, above, wt);
  find_rank_bin<HIST_BINS>(cnt, above, (unsigned long long)k, &sb, &sr, &sa);
  if (t == 0) {
    if (above[(0x7F800000u >> HIST_SHIFT)] + cnt[(0x7F800000u >> HIST_SHIFT)] > 0 ||
        cnt[HIST_BINS - 1] > 0)
      st->nonfinite = 1u;
    if (hist[HIST_BINS + 1]) st->nonfinite = 1u;          // any rank saw NaN/Inf (multi-GPU sum)
#if defined(CSSAR_FORCE_FALLBACK)
    const bool ok = false;
#else
    const bool ok = sb >= 0 && sb >= st->cand_lo && sb <= st->cand_hi && hist[HIST_BINS] == 0u;
#endif
    if (ok) {
      st->need_full = 0;
      st->target_bin = sb;
      st->target_rank = sr;
      st->above_count = sa;
    } else {
      st->need_full = 1;
      st->fallbacks += 1;
    }
  }
}

__global__ void __launch_bounds__(512) fb_hist_kernel(const float2* __restrict__ b, long long n, const SelState* st,
                                                      uint32_t* hist_full) {
  pdl_wait();
  if (!st->need_full) return;
  __shared__ uint32_t sh[HIST_BINS];
  for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x) sh[i] = 0u;
  __syncthreads();
  const float4* b4 = reinterpret_cast<const float4*>(b);
  const long long n2 = n / 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    const float4 q = b4[i];
    atomicAdd(&sh[mag2_bits(make_float2(q.x, q.y)) >> HIST_SHIFT], 1u);
    atomicAdd(&sh[mag2_bits(make_float2(q.z, q.w)) >> HIST_SHIFT], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist_full[i], sh[i]);
}

__global__ void __launch_bounds__(1024) fb_find_kernel(long long k, SelState* st, const uint32_t* hist_full) {
  pdl_wait();
  if (!st->need_full) return;
  __shared__ uint32_t cnt[HIST_BINS], above[HIST_BINS], wt[32];
  __shared__ int sb;
  __shared__ uint32_t sr, sa;
  const int t = threadIdx.x;
  for (int i = t; i < HIST_BINS; i += 1024) cnt[i] = hist_full[i];
  if (t == 0) { sb = -1; sr = 0; sa = 0; }
  __syncthreads();
  block_suffix<HIST_BINS>(cnt, above, wt);
  find_rank_bin<HIST_BINS>(cnt, above, (unsigned long long)k, &sb, &sr, &sa);
  if (t == 0) {
    st->target_bin = sb;
    st->target_rank = sr;
    st->above_count = sa;
    st->cand_lo = sb;
    st->cand_hi = sb;
    st->cand_count = 0u;
    st->cand_overflow = 0u;
  }
}

__global__ void __launch_bounds__(512) fb_collect_kernel(const float2* __restrict__ b, long long n, SelState* st,
                                                         uint32_t* cand, uint32_t cap) {
  pdl_wait();
  if (!st->need_full) return;
  const int B = st->target_bin;
  __shared__ uint32_t buf[2048];
  __shared__ uint32_t cntb, base;
  const long long n2 = n / 2;
  const float4* b4 = reinterpret_cast<const float4*>(b);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x; i0 < n2; i0 += stride) {
    if (threadIdx.x == 0) cntb = 0u;
    __syncthreads();
    const long long i = i0 + threadIdx.x;
    if (i < n2) {
      const float4 q = b4[i];
      const uint32_t u0 = mag2_bits(make_float2(q.x, q.y)), u1 = mag2_bits(make_float2(q.z, q.w));
      if ((int)(u0 >> HIST_SHIFT) == B) buf[atomicAdd(&cntb, 1u)] = u0;
      if ((int)(u1 >> HIST_SHIFT) == B) buf[atomicAdd(&cntb, 1u)] = u1;
    }
    __syncthreads();
    if (threadIdx.x == 0) base = cntb ? atomicAdd(&st->cand_count, cntb) : 0u;
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < cntb; e += blockDim.x) {
      const uint32_t g = base + e;
      if (g < cap) cand[g] = buf[e]; else st->cand_overflow = 1u;   // -> exact count over b (fine_count)
    }
    __syncthreads();
  }
}

// lambda_i of a threshold sigma: the penalty weight whose jump point is sigma, / mu
CSSAR_DEV float lambda_of_sigma(float sig, float mu, int thr) {
  if (thr == THR_SOFT) return sig / mu;
  if (thr == THR_HALF) return (float)(1.0886621079036347 * pow((double)sig, 1.5) / mu);
  if (thr == THR_HARD) return sig * sig / mu;
  return (float)(cbrt(pow(1.5 * (double)sig, 4.0) / 3.0) / mu);
}

// sigma^2 found: state for the next iteration (new sigma, histogram floor, candidate window,
// log entry, counter resets).  Runs in thread 0 (bookkeeping) and all threads (resets).
CSSAR_DEV void finish_select(uint32_t s2, unsigned long long abv, int thr, float mu, SelState* st, uint32_t* hist,
                             uint32_t* hist_full, IterLogDev* log, int log_cap, float gap = 0.0f, int gap_exact = 0) {
  const int t = threadIdx.x;
  if (t == 0) {
    const float sig = sqrtf(__uint_as_float(s2));
    st->sigma2_bits = s2;
    st->sigma = sig;
    const int it = st->iter;
    if (it < log_cap) {
      IterLogDev e;
      e.sigma = sig;
      const float m = st->mu > 0.f ? st->mu : mu;          // adaptive step of this iteration
      e.mu = m;
      e.lam = lambda_of_sigma(sig, m, thr);
      e.support = (long long)abv;
      e.resid2 = st->resid2;
      e.gap = gap;
      e.gap_exact = gap_exact;
      log[it] = e;
    }
    const int B = (int)(s2 >> HIST_SHIFT);
    st->iter = it + 1;
    st->floor_bin = max(0, B - FLOOR_MARGIN);
    st->cand_lo = B - CAND_MARGIN;
    st->cand_hi = B + CAND_MARGIN;
    st->cand_count = 0u;
    st->cand_overflow = 0u;
    st->resid2 = 0.0;
    st->mu_num = 0.0;
    st->mu_den = 0.0;
  }
  const int nf = st->need_full;
  __syncthreads();
  for (int i = t; i < HIST_WORDS; i += blockDim.x) {
    hist[i] = 0u;
    if (nf && i < HIST_BINS) hist_full[i] = 0u;
  }
  // sparse-state schedule: the list the next S5 writes starts empty (it was last read by this
  // iteration's S1 / S5)
  if (st->ss_cnt[0]) {
    uint32_t* c = st->ss_cnt[st->iter & 1];
    for (int i = t; i < st->ss_npan; i += blockDim.x) c[i] = 0u;
  }
  __syncthreads();
  if (t == 0) {
    st->ss_fell = nf;          // a fallback iteration: ss_rebuild re-derives the list from dense b
    st->need_full = 0;
  }
}

// one 10-bit radix level: counts of (u >> sh) & 1023 among the |b|^2 patterns u with
// (u >> (sh + 10)) == prefix -- over the candidate list, or, when the list overflowed (more
// than cand_cap patterns in the target bin, e.g. a flat or all-zero b), over all of b (one
// block scanning the array: the degenerate case stays exact, just slower)
CSSAR_DEV void fine_count(uint32_t* cnt, const uint32_t* cand, uint32_t nc, uint32_t prefix, int sh,
                          const float2* b = nullptr, long long n = 0) {
  const int t = threadIdx.x;
  cnt[t] = 0u;
  __syncthreads();
  if (b) {
    const float4* b4 = reinterpret_cast<const float4*>(b);
    for (long long i = t; i < n / 2; i += 1024) {
      const float4 q = b4[i];
      const uint32_t u0 = mag2_bits(make_float2(q.x, q.y)), u1 = mag2_bits(make_float2(q.z, q.w));
      if ((u0 >> (sh + 10)) == prefix) atomicAdd(&cnt[(u0 >> sh) & 1023u], 1u);
      if ((u1 >> (sh + 10)) == prefix) atomicAdd(&cnt[(u1 >> sh) & 1023u], 1u);
    }
  } else {
    for (uint32_t i = t; i < nc; i += 1024) {
      const uint32_t u = cand[i];
      if ((u >> (sh + 10)) == prefix) atomicAdd(&cnt[(u >> sh) & 1023u], 1u);
    }
  }
  __syncthreads();
}

// near-tie gap g = (|b|_(k) - |b|_(k+1)) / |b|_(k+1) (SURVEY.md 8(c).3 log, 8(c).6 diagnostic):
// 0 when ties leave fewer than k values above sigma; else the smallest candidate pattern above
// sigma^2 is |b|_(k)^2 if the candidate window holds it (exact), otherwise the window's upper
// bin edge bounds it from below.  Returns the gap; *exact = 0 for a bound.
CSSAR_DEV float near_tie_gap(uint32_t s2, unsigned long long abv, long long k, const uint32_t* cand, uint32_t nc,
                             bool have_list, int hi_bin, uint32_t* smin, int* exact) {
  const int t = threadIdx.x;
  if (t == 0) *smin = 0xFFFFFFFFu;
  __syncthreads();
  if (have_list && (long long)abv >= k) {
    uint32_t m = 0xFFFFFFFFu;
    for (uint32_t i = t; i < nc; i += blockDim.x) {
      const uint32_t u = cand[i];
      if (u > s2 && u < m) m = u;
    }
    atomicMin(smin, m);
  }
  __syncthreads();
  if ((long long)abv < k) { *exact = 1; return 0.0f; }
  if (s2 == 0u) { *exact = 0; return INFINITY; }
  const uint32_t um = *smin;
  const bool ex = have_list && um != 0xFFFFFFFFu;
  const uint32_t ub = ex ? um : (uint32_t)(hi_bin + 1) << HIST_SHIFT;
  *exact = ex ? 1 : 0;
  return (float)(sqrt((double)__uint_as_float(ub) / (double)__uint_as_float(s2)) - 1.0);
}

// radix refinement inside target_bin over the candidate list (two 10-bit levels: bits
// [19:10] then [9:0]), then finish_select
__global__ void __launch_bounds__(1024) sel_fine_kernel(long long k, int thr, float mu, SelState* st,
                                                        uint32_t* hist, uint32_t* hist_full, const uint32_t* cand,
                                                        uint32_t cap, IterLogDev* log, int log_cap, const float2* b,
                                                        long long n) {
  pdl_wait();
  __shared__ uint32_t cnt[1024], above[1024], wt[32];
  __shared__ int sd;
  __shared__ uint32_t sr, sa, smin;
  const int t = threadIdx.x;
  const bool ovf = st->cand_overflow != 0u;     // list truncated: count over b instead (exact)
  const uint32_t nc = min(st->cand_count, cap);
  uint32_t prefix = (uint32_t)st->target_bin;   // matched high bits so far
  uint32_t rank = st->target_rank;
  unsigned long long abv = st->above_count;
#pragma unroll 1
  for (int lvl = 0; lvl < 2; ++lvl) {
    fine_count(cnt, cand, nc, prefix, lvl == 0 ? 10 : 0, ovf ? b : nullptr, n);
    if (t == 0) { sd = -1; sr = 0; sa = 0; }
    __syncthreads();
    block_suffix<1024>(cnt, above, wt);
    find_rank_bin<1024>(cnt, above, (unsigned long long)rank, &sd, &sr, &sa);
    const int d = sd < 0 ? 0 : sd;
    prefix = (prefix << 10) | (uint32_t)d;
    rank = sr;
    abv += sa;
    __syncthreads();
  }
  int gx = 0;
  const float gap = near_tie_gap(prefix, abv, k, cand, nc, !ovf, st->cand_hi, &smin, &gx);
  finish_select(prefix, abv, thr, mu, st, hist, hist_full, log, log_cap, gap, gx);
}

// ---- split fine select (multi-GPU): local level histograms, global counts after the all-reduce
__global__ void __launch_bounds__(1024) fine_hist_kernel(int lvl, SelState* st, const uint32_t* cand, uint32_t cap,
                                                         uint32_t* out, const float2* b, long long n) {
  __shared__ uint32_t cnt[1024];
  if (lvl == 0 && threadIdx.x == 0) {
    st->fine_prefix = (uint32_t)st->target_bin;
    st->fine_rank = st->target_rank;
    st->fine_abv = st->above_count;
  }
  __syncthreads();
  const uint32_t prefix = lvl == 0 ? (uint32_t)st->target_bin : st->fine_prefix;
  fine_count(cnt, cand, min(st->cand_count, cap), prefix, lvl == 0 ? 10 : 0, st->cand_overflow ? b : nullptr, n);
  out[threadIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(1024) fine_find_kernel(int lvl, int thr, float mu, SelState* st, uint32_t* hist,
                                                         uint32_t* hist_full, const uint32_t* cand, uint32_t cap,
                                                         uint32_t* lvl_cnt, IterLogDev* log, int log_cap,
                                                         const float2* b, long long n) {
  __shared__ uint32_t cnt[1024], above[1024], wt[32];
  __shared__ int sd;
  __shared__ uint32_t sr, sa;
  const int t = threadIdx.x;
  cnt[t] = lvl_cnt[t];
  if (t == 0) { sd = -1; sr = 0; sa = 0; }
  __syncthreads();
  block_suffix<1024>(cnt, above, wt);
  find_rank_bin<1024>(cnt, above, (unsigned long long)st->fine_rank, &sd, &sr, &sa);
  const uint32_t prefix = (st->fine_prefix << 10) | (uint32_t)(sd < 0 ? 0 : sd);
  const unsigned long long abv = st->fine_abv + sa;
  __syncthreads();
  if (lvl == 0) {
    if (t == 0) {
      st->fine_prefix = prefix;
      st->fine_rank = sr;
      st->fine_abv = abv;
    }
    // level-1 local counts for the next all-reduce
    fine_count(cnt, cand, min(st->cand_count, cap), prefix, 0, st->cand_overflow ? b : nullptr, n);
    lvl_cnt[t] = cnt[t];
  } else {
    finish_select(prefix, abv, thr, mu, st, hist, hist_full, log, log_cap);
  }
}

__global__ void lambda_step_kernel(SelState* st, int thr, float mu, IterLogDev* log, int log_cap) {
  const int it = st->iter;
  const float m = st->mu > 0.f ? st->mu : mu;      // adaptive runs: sigma_fixed already = f(lambda mu_i)
  if (it < log_cap) {
    IterLogDev e;
    e.sigma = st->sigma_fixed;
    e.mu = m;
    e.lam = lambda_of_sigma(st->sigma_fixed, m, thr);
    e.support = (long long)st->support_fixed;
    e.resid2 = st->resid2;
    e.gap = 0.0f;                                  // no order statistic under a fixed lambda
    e.gap_exact = 0;
    log[it] = e;
  }
  st->iter = it + 1;
  st->sigma2_bits = st->sigma2_fixed_bits;
  st->sigma = st->sigma_fixed;
  st->support_fixed = 0ull;
  st->resid2 = 0.0;
  st->mu_num = 0.0;
  st->mu_den = 0.0;
}

__global__ void init_state_kernel(SelState* st, uint32_t* hist, uint32_t* hist_full, float sigma_fixed) {
  const int t = threadIdx.x;
  for (int i = t; i < HIST_WORDS; i += blockDim.x) { hist[i] = 0u; if (i < HIST_BINS) hist_full[i] = 0u; }
  if (t == 0) {
    SelState z{};
    z.sigma2_bits = 0u;          // X_0 = E(X_in; 0) = X_in (identity threshold)
    z.sigma = 0.f;
    z.sigma_fixed = sigma_fixed;
    z.sigma2_fixed_bits = __float_as_uint(__fmul_rn(sigma_fixed, sigma_fixed));
    z.floor_bin = HIST_BINS;     // first select has no history -> fallback path
    z.cand_lo = 1;
    z.cand_hi = 0;
    *st = z;
  }
}

__global__ void finalize_kernel(float2* b, long long n, int thr, const SelState* st) {
  const uint32_t s2 = st->sigma2_bits;
  const float sig = st->sigma;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = threshold(b[i], s2, sig, thr);
}

__global__ void pack_mask_kernel(const uint8_t* __restrict__ m, uint32_t* __restrict__ bits, long long words) {
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < words; w += (long long)gridDim.x * blockDim.x) {
    const uint4* src = reinterpret_cast<const uint4*>(m + w * 32);
    uint32_t acc = 0u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint4 q = src[h];
      const uint32_t qs[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int byte = 0; byte < 4; ++byte)
          acc |= (((qs[e] >> (8 * byte)) & 0xFFu) ? 1u : 0u) << (h * 16 + e * 4 + byte);
    }
    bits[w] = acc;
  }
}

cudaError_t launch_select(int sm_count, float2* b, long long n, long long k, int rule, int thr, float mu,
                          SelState* st, uint32_t* hist, uint32_t* hist_full, uint32_t* cand, uint32_t cand_cap,
                          IterLogDev* log, int log_cap, cudaStream_t s) {
  if (rule == RULE_LAMBDA) {
    lambda_step_kernel<<<1, 1, 0, s>>>(st, thr, mu, log, log_cap);
    return cudaGetLastError();
  }
  cudaError_t e = launch_pdl(sel_coarse_kernel, dim3(1), dim3(1024), 0, s, k, st, (const uint32_t*)hist);
  if (e != cudaSuccess) return e;
  return launch_select_rest(sm_count, b, n, k, thr, mu, st, hist, hist_full, cand, cand_cap, log, log_cap, s);
}

cudaError_t launch_select_rest(int sm_count, float2* b, long long n, long long k, int thr, float mu, SelState* st,
                               uint32_t* hist, uint32_t* hist_full, uint32_t* cand, uint32_t cand_cap, IterLogDev* log,
                               int log_cap, cudaStream_t s) {
  const int grid = sm_count * 4;
  cudaError_t e;
  if ((e = launch_pdl(fb_hist_kernel, dim3(grid), dim3(512), 0, s, (const float2*)b, n, (const SelState*)st,
                      hist_full)) != cudaSuccess)
    return e;
  if ((e = launch_pdl(fb_find_kernel, dim3(1), dim3(1024), 0, s, k, st, (const uint32_t*)hist_full)) != cudaSuccess)
    return e;
  if ((e = launch_pdl(fb_collect_kernel, dim3(grid), dim3(512), 0, s, (const float2*)b, n, st, cand, cand_cap)) !=
      cudaSuccess)
    return e;
  if ((e = launch_pdl(sel_fine_kernel, dim3(1), dim3(1024), 0, s, k, thr, mu, st, hist, hist_full,
                      (const uint32_t*)cand, cand_cap, log, log_cap, (const float2*)b, n)) != cudaSuccess)
    return e;
  return cudaGetLastError();
}

cudaError_t launch_select_part(int part, int sm_count, float2* b, long long n, long long k, int thr, float mu,
                               SelState* st, uint32_t* hist, uint32_t* hist_full, uint32_t* cand,
                               uint32_t cand_cap, uint32_t* lvl, IterLogDev* log, int log_cap, cudaStream_t s) {
  const int grid = sm_count * 4;
  switch (part) {
    case SEL_COARSE: sel_coarse_kernel<<<1, 1024, 0, s>>>(k, st, hist); break;
    case SEL_FB_HIST: fb_hist_kernel<<<grid, 512, 0, s>>>(b, n, st, hist_full); break;
    case SEL_FB_PICK:
      fb_find_kernel<<<1, 1024, 0, s>>>(k, st, hist_full);
      fb_collect_kernel<<<grid, 512, 0, s>>>(b, n, st, cand, cand_cap);
      break;
    case SEL_FINE0_HIST: fine_hist_kernel<<<1, 1024, 0, s>>>(0, st, cand, cand_cap, lvl, b, n); break;
    case SEL_FINE0_FIND:
      fine_find_kernel<<<1, 1024, 0, s>>>(0, thr, mu, st, hist, hist_full, cand, cand_cap, lvl, log, log_cap, b, n);
      break;
    case SEL_FINE1_FIND:
      fine_find_kernel<<<1, 1024, 0, s>>>(1, thr, mu, st, hist, hist_full, cand, cand_cap, lvl, log, log_cap, b, n);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_lambda_step(SelState* st, int thr, float mu, IterLogDev* log, int log_cap, cudaStream_t s) {
  lambda_step_kernel<<<1, 1, 0, s>>>(st, thr, mu, log, log_cap);
  return cudaGetLastError();
}

struct GroupPtrs { void* p[16]; };

template <class T>
__global__ void group_sum_kernel(GroupPtrs g, int world, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int r = 0; r < world; ++r) acc += static_cast<T*>(g.p[r])[i];
    for (int r = 0; r < world; ++r) static_cast<T*>(g.p[r])[i] = acc;
  }
}

// dtype: 0 = u32, 1 = u64, 2 = f64 (rank order of the sum is fixed: deterministic)
cudaError_t launch_group_sum(int dtype, void* const* bufs, int world, long long count, cudaStream_t s) {
  if (world < 1 || world > 16) return cudaErrorInvalidValue;
  GroupPtrs g{};
  for (int r = 0; r < world; ++r) g.p[r] = bufs[r];
  long long blocks = (count + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  if (blocks < 1) blocks = 1;
  if (dtype == 0) group_sum_kernel<uint32_t><<<(unsigned)blocks, 256, 0, s>>>(g, world, count);
  else if (dtype == 1) group_sum_kernel<unsigned long long><<<(unsigned)blocks, 256, 0, s>>>(g, world, count);
  else group_sum_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(g, world, count);
  return cudaGetLastError();
}

cudaError_t launch_init_state(SelState* st, uint32_t* hist, uint32_t* hist_full, int thr, float sigma_fixed,
                              cudaStream_t s) {
  (void)thr;
  init_state_kernel<<<1, 1024, 0, s>>>(st, hist, hist_full, sigma_fixed);
  return cudaGetLastError();
}

cudaError_t launch_finalize(float2* b, long long n, int thr, const SelState* st, cudaStream_t s) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  finalize_kernel<<<(unsigned)blocks, 256, 0, s>>>(b, n, thr, st);
  return cudaGetLastError();
}

cudaError_t launch_pack_mask(const uint8_t* m, uint32_t* bits, long long rows, long long cols, cudaStream_t s) {
  const long long words = rows * (cols / 32);
  long long blocks = (words + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  pack_mask_kernel<<<(unsigned)blocks, 256, 0, s>>>(m, bits, words);
  return cudaGetLastError();
}

}  // namespace cssar
