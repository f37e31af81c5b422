// libcssar device kernels (sm_100a): range sweeps, azimuth sweeps (thread-block clusters +
// DSMEM for long columns), fused residual / step / threshold epilogues, exact k-rule select.
//
// Hot path per ITA iteration (eq. 25, Algorithm 1):
//   S1 az FWD_THR : X = E(b; sigma) ; F_eta                                  (G head)
//   S2 rg <G>     : Phi3* -> F_tau -> Phi2* -> F_tau^-1 -> Phi1*              (G body)
//   S3 az RESID   : F_eta^-1 ; r = Theta o (Y - G X) ; F_eta                  (residual)
//   S4 rg <M>     : Phi1 -> F_tau -> Phi2 -> F_tau^-1 -> Phi3                 (M body)
//   S5 az TAIL    : F_eta^-1 ; b = E(b; sigma) + mu dX ; |b|^2 histogram      (step)
//   S6 select     : sigma^2 = (k+1)-th largest |b|^2 (exact radix select)     (lambda rule)
#pragma once
#include <cooperative_groups.h>
#include "fft_engine.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace cssar {

// ------------------------------------------------------------------ elementwise pieces
CSSAR_DEV uint32_t mag2_bits(float2 v) {
  // |v|^2 with explicit roundings (no FMA contraction): reproducible on the host
  return __float_as_uint(__fadd_rn(__fmul_rn(v.x, v.x), __fmul_rn(v.y, v.y)));
}

// MUFU reciprocal square root without the denormal rescaling rsqrtf() carries (a denormal
// |b|^2 is below any sigma^2 the select can produce except 0, which the callers guard)
CSSAR_DEV float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// shrink factor of the q = 2/3 and q = 1/2 thresholds (closed forms with transcendental
// functions).  Out of line by default: inlined at every element of the unrolled sweep
// epilogues they made the azimuth kernels' code several times larger than the soft / hard
// path that runs (instruction-cache stalls); CSSAR_THR_INLINE=1 restores inlining.
#if defined(CSSAR_THR_INLINE) && CSSAR_THR_INLINE
#define CSSAR_THR_HEAVY CSSAR_DEV
#else
#define CSSAR_THR_HEAVY static __device__ __noinline__
#endif
CSSAR_THR_HEAVY float thr_factor_heavy(float a2, float sigma, int thr) {
  float f;
  if (thr == THR_TWOTHIRDS) {
    // closed-form L2/3 minimiser in k-rule form (oracle/ita.py twothirds): q = 27 t^2 /
    // (16 lm^(3/2)) = (3 sqrt(3)/4)(t/sigma)^2, phi = c sigma^(1/3) sqrt(cosh(acosh(q)/3))
    const float t = a2 * rsqrt_ftz(a2);
    const float q = 1.2990381056766580f * a2 / (sigma * sigma);
    const float phi = 1.2061639667263164f * cbrtf(sigma) * sqrtf(coshf(acoshf(q) * (1.0f / 3.0f)));
    const float x = 0.5f * (phi + sqrtf(2.0f * t / phi - phi * phi));
    f = x * x * x / t;
    f = sigma == 0.f ? 1.0f : f;
  } else {
    const float ratio = sigma * rsqrt_ftz(a2);
    const float phi = acosf(0.70710678118654752f * ratio * sqrtf(ratio));
    f = (2.0f / 3.0f) * (1.0f + cosf(2.09439510239319549f - (2.0f / 3.0f) * phi));
    f = sigma == 0.f ? 1.0f : f;
  }
  return f;
}

// E(b; sigma): strict survival on the fp32 |b|^2 pattern,
// soft (eq. 9), half (q = 1/2), hard (q = 0) or q = 2/3 shrink of the magnitude, phase kept.
CSSAR_DEV float2 threshold(float2 b, uint32_t s2bits, float sigma, int thr) {
  const uint32_t u = mag2_bits(b);
  const float a2 = __uint_as_float(u);
  float f;
  if (thr == THR_SOFT) {
    f = sigma == 0.f ? 1.0f : fmaf(-sigma, rsqrt_ftz(a2), 1.0f);   // 1 - sigma/|b|
  } else if (thr == THR_HARD) {
    f = 1.0f;
  } else {
    f = thr_factor_heavy(a2, sigma, thr);
  }
  // strict survival on the |b|^2 pattern; a removed entry is +0 (not b * 0, whose sign would
  // follow b: the sparse-state schedule's zero-filled X must equal the dense one bitwise).
  // Explicitly rounded products: an FMA contraction with the consumer (e.g. the first FFT
  // butterfly) would make E(b) inside a kernel round differently from the X it returns
  return (u > s2bits) ? make_float2(__fmul_rn(b.x, f), __fmul_rn(b.y, f)) : make_float2(0.0f, 0.0f);
}

CSSAR_DEV uint32_t mask_bit(const uint32_t* mask, int words, int row, int col) {
  if (!mask) return 1u;
  return (__ldg(mask + (size_t)row * words + (col >> 5)) >> (col & 31)) & 1u;
}

// the mask word holding (row, col) (all ones without a mask): loaded early, the bit is taken
// at its use (mask_at) so the load latency overlaps the transform in between
CSSAR_DEV uint32_t mask_word(const uint32_t* mask, int words, int row, int col) {
  return mask ? __ldg(mask + (size_t)row * words + (col >> 5)) : 0xFFFFFFFFu;
}
CSSAR_DEV bool mask_at(uint32_t word, int col) { return (word >> (col & 31)) & 1u; }

// x[r] *= exp(+-2 pi i P(u0 + r S)), r < R, by u64 second differences: the first difference
// d1 is carried exactly in 64 bits, the phase itself only in its top 32 bits (the SFU path
// uses no more); dropping the low-word carries costs < R * 2^-32 cycle (< 5e-8 rad at R = 32).
template <int R, int S, bool CONJ>
CSSAR_DEV void phase_apply(const float2* tab, const Quad& q, int u0, float2* x) {
#if defined(CSSAR_PHASE_TABLE)
  uint64_t P = quad_eval(q, u0);
  uint64_t d1 = q.c2 * (uint64_t)((int64_t)2 * u0 * S + (int64_t)S * S) + q.c1 * (uint64_t)S;
  const uint64_t d2 = q.c2 * (uint64_t)(2ll * S * S);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    x[r] = cmul(x[r], phase_from_fixed<CONJ>(tab, P));
    P += d1;
    d1 += d2;
  }
#else
  // top 32 bits only: the phase and its first difference are advanced with 32-bit adds; the
  // dropped low-word carries cost < (R + R(R-1)/2) 2^-32 cycle (< 3.2e-8 cycle = 2e-7 rad at
  // R = 16), below the SFU's own 5e-7 rad
  (void)tab;
  uint32_t Ph = (uint32_t)(quad_eval(q, u0) >> 32);
  uint32_t d1 = (uint32_t)((q.c2 * (uint64_t)((int64_t)2 * u0 * S + (int64_t)S * S) + q.c1 * (uint64_t)S) >> 32);
  const uint32_t d2 = (uint32_t)((q.c2 * (uint64_t)(2ll * S * S)) >> 32);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    x[r] = cmul(x[r], phase_from_hi32<CONJ>(Ph));
    Ph += d1;
    d1 += d2;
  }
#endif
}


}  // namespace cssar
