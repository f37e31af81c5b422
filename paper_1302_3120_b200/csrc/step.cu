// Adaptive-step ITA (NEXT-1; eq. 27, normalised-IHT form, R11/R20): the
// elementwise step that follows the gradient kernels.  mu_i = ||dX_k||^2 / ||Theta G(dX_k)||^2
// (reduced by AZ_GRAD / AZ_NORM into the solver state; 1 when either is 0), then
//   b_i = E(b_{i-1}; sigma_{i-1}) + mu_i D,   D = dX = M(Theta(Y - G X_i)) kept by AZ_GRAD,
// with the same |b|^2 histogram / candidate / fixed-lambda support bookkeeping as the tail
// kernel.  Fixed-lambda runs get sigma_i = lambda mu_i (soft) or the half-threshold jump point.
#include "az.cuh"

namespace cssar {

__global__ void __launch_bounds__(512) adaptive_step_kernel(const AzArgs a, long long n2) {
  __shared__ uint32_t shist[HIST_BINS], scand[1024], scount[4];
  __shared__ uint32_t sbase;
  const int t = threadIdx.x;
  const double num = a.st->mu_num, den = a.st->mu_den;
  const float mu = (num > 0.0 && den > 0.0) ? (float)(num / den) : 1.0f;
  TailCtx tc{};
  tc.shist = shist;
  tc.scand = scand;
  tc.scount = scount;
  tc.floor_bin = a.st->floor_bin;
  tc.cand_lo = a.st->cand_lo;
  tc.cand_hi = a.st->cand_hi;
  tc.s2bits = a.st->sigma2_bits;
  tc.sigma = a.st->sigma;
  float sf = 0.f;
  if (a.rule == RULE_LAMBDA) {
    const float lm = a.lambda * mu;
    sf = a.thr == THR_SOFT   ? lm
       : a.thr == THR_HALF   ? 0.94494078742115480f * powf(lm, 2.0f / 3.0f)   // (54^(1/3)/4)(lambda mu)^(2/3)
       : a.thr == THR_HARD   ? sqrtf(lm)
                             : (2.0f / 3.0f) * sqrtf(sqrtf(3.0f * lm * lm * lm));   // (2/3)(3 (lambda mu)^3)^(1/4)
    tc.s2fixed = __float_as_uint(__fmul_rn(sf, sf));
  }
  if (blockIdx.x == 0 && t == 0) {
    a.st->mu = mu;
    if (a.rule == RULE_LAMBDA) {
      a.st->sigma_fixed = sf;
      a.st->sigma2_fixed_bits = tc.s2fixed;
    }
  }
  for (int i = t; i < HIST_BINS; i += blockDim.x) shist[i] = 0u;
  if (t < 4) scount[t] = 0u;
  __syncthreads();
  float4* b4 = reinterpret_cast<float4*>(a.b);
  const float4* d4 = reinterpret_cast<const float4*>(a.D);
  for (long long i = blockIdx.x * (long long)blockDim.x + t; i < n2; i += (long long)gridDim.x * blockDim.x) {
    const float4 bq = b4[i], dq = d4[i];
    const float2 k0 = threshold(make_float2(bq.x, bq.y), tc.s2bits, tc.sigma, a.thr);
    const float2 k1 = threshold(make_float2(bq.z, bq.w), tc.s2bits, tc.sigma, a.thr);
    const float2 v0 = make_float2(fmaf(mu, dq.x, k0.x), fmaf(mu, dq.y, k0.y));
    const float2 v1 = make_float2(fmaf(mu, dq.z, k1.x), fmaf(mu, dq.w, k1.y));
    b4[i] = make_float4(v0.x, v0.y, v1.x, v1.y);
    AzOps<AZ_TAIL>::tail_stats(a, v0, tc);
    AzOps<AZ_TAIL>::tail_stats(a, v1, tc);
  }
  __syncthreads();
  if (a.rule == RULE_K) {
    for (int i = t; i < HIST_BINS; i += blockDim.x)
      if (shist[i]) atomicAdd(&a.hist[i], shist[i]);
    const uint32_t nc = min(scount[0], 1024u);
    if (t == 0) sbase = nc ? atomicAdd(&a.st->cand_count, nc) : 0u;
    __syncthreads();
    for (uint32_t i = t; i < nc; i += blockDim.x) {
      const uint32_t g = sbase + i;
      if (g < a.cand_cap) a.cand[g] = scand[i]; else { a.st->cand_overflow = 1u; a.hist[HIST_BINS] = 1u; }
    }
  } else if (t == 0 && scount[1]) {
    atomicAdd(&a.st->support_fixed, (unsigned long long)scount[1]);
  }
}

cudaError_t launch_adaptive_step(const AzArgs& a, long long n, int sm_count, cudaStream_t s) {
  adaptive_step_kernel<<<sm_count * 4, 512, 0, s>>>(a, n / 2);
  return cudaGetLastError();
}

// Tolerance stop (NEXT-4): after the select of iteration i, X_(i+1) = E(b_i; sigma_i)
// (the X the next S1 or the final pass forms) against the kept X_i.  Fixed grid, fp64 per-thread
// sums reduced in a fixed order per block: the per-block partials are summed in block order by
// the host, so the decision is deterministic.
__global__ void __launch_bounds__(256) conv_check_kernel(const float4* b, float4* xk, long long n2,
                                                         const SelState* st, int thr, double2* part) {
  __shared__ double2 red[8];
  const uint32_t s2 = st->sigma2_bits;
  const float sig = st->sigma;
  double d2 = 0.0, x2 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    const float4 bq = b[i], xq = xk[i];
    const float2 k0 = threshold(make_float2(bq.x, bq.y), s2, sig, thr);
    const float2 k1 = threshold(make_float2(bq.z, bq.w), s2, sig, thr);
    const double e0 = (double)k0.x - xq.x, e1 = (double)k0.y - xq.y, e2 = (double)k1.x - xq.z, e3 = (double)k1.y - xq.w;
    d2 += e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3;
    x2 += (double)xq.x * xq.x + (double)xq.y * xq.y + (double)xq.z * xq.z + (double)xq.w * xq.w;
    xk[i] = make_float4(k0.x, k0.y, k1.x, k1.y);
  }
  for (int o = 16; o > 0; o >>= 1) {
    d2 += __shfl_down_sync(0xffffffffu, d2, o);
    x2 += __shfl_down_sync(0xffffffffu, x2, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = make_double2(d2, x2);
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 r = red[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) { r.x += red[q].x; r.y += red[q].y; }
    part[blockIdx.x] = r;
  }
}

cudaError_t launch_conv_check(const float2* b, float2* Xk, long long n, const SelState* st, int thr, double2* part,
                              int blocks, cudaStream_t s) {
  conv_check_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(b), reinterpret_cast<float4*>(Xk), n / 2,
                                           st, thr, part);
  return cudaGetLastError();
}

}  // namespace cssar
