// Device helpers: complex arithmetic, in-register radix-R DFTs, exact twiddles,
// fixed-point CSA phase evaluation.  sm_100a only; no code shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define CSSAR_DEV __device__ __forceinline__

namespace cssar {

CSSAR_DEV float2 operator+(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
CSSAR_DEV float2 operator-(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
CSSAR_DEV float2 operator*(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
CSSAR_DEV float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
CSSAR_DEV float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}

// cos(2 pi o / 32), o = 0..8 (first octant plus the octant edge), correctly rounded.
CSSAR_DEV constexpr float cos32(int o) {
  return o == 0 ? 1.0f : o == 1 ? 0.98078528040323043f : o == 2 ? 0.92387953251128674f
       : o == 3 ? 0.83146961230254524f : o == 4 ? 0.70710678118654752f : o == 5 ? 0.55557023301960218f
       : o == 6 ? 0.38268343236508977f : o == 7 ? 0.19509032201612827f : 0.0f;
}

// v * exp(DIR * 2 pi i * idx / 32); idx is a compile-time constant after unrolling.
template <int DIR>
CSSAR_DEV float2 tw32(float2 v, int idx) {
  idx &= 31;
  if (idx == 0) return v;
  if (idx == 16) return make_float2(-v.x, -v.y);
  if (idx == 8) return DIR > 0 ? make_float2(-v.y, v.x) : make_float2(v.y, -v.x);
  if (idx == 24) return DIR > 0 ? make_float2(v.y, -v.x) : make_float2(-v.y, v.x);
  const int q = idx >> 3, o = idx & 7;   // quadrant, offset within the quadrant
  const float c0 = cos32(o), s0 = cos32(8 - o);
  float c = q == 0 ? c0 : q == 1 ? -s0 : q == 2 ? -c0 : s0;
  float s = q == 0 ? s0 : q == 1 ? c0 : q == 2 ? -s0 : -c0;
  if (DIR < 0) s = -s;
  return make_float2(fmaf(v.x, c, -v.y * s), fmaf(v.x, s, v.y * c));
}

CSSAR_DEV constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x >> 1); }

template <int R>
struct Log2 { static constexpr int v = (R <= 1) ? 0 : 1 + Log2<R / 2>::v; };
template <>
struct Log2<1> { static constexpr int v = 0; };

template <int R>
CSSAR_DEV constexpr int bitrev(int i) {
  int r = 0;
  for (int b = 0; b < Log2<R>::v; ++b) r |= ((i >> b) & 1) << (Log2<R>::v - 1 - b);
  return r;
}

// In-register DFT of length R (power of two, R <= 32):
//   v[k] <- sum_n v[n] exp(DIR * 2 pi i n k / R), unscaled, natural order in and out.
template <int R, int DIR>
CSSAR_DEV void dft(float2 (&v)[R]) {
  if constexpr (R == 1) return;
  else {
#pragma unroll
    for (int span = R / 2; span >= 1; span >>= 1) {
#pragma unroll
      for (int blk = 0; blk < R; blk += 2 * span) {
#pragma unroll
        for (int m = 0; m < span; ++m) {
          float2 a = v[blk + m], b = v[blk + m + span];
          v[blk + m] = a + b;
          v[blk + m + span] = tw32<DIR>(a - b, m * (32 / (2 * span)));
        }
      }
    }
    float2 t[R];
#pragma unroll
    for (int i = 0; i < R; ++i) t[i] = v[i];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = t[bitrev<R>(i)];
  }
}

// v * w_N^k with w_N = exp(DIR 2 pi i / N), N | 32 (compile-time k after unrolling)
template <int N, int DIR>
CSSAR_DEV float2 twN(float2 v, int k) { return tw32<DIR>(v, (k * (32 / N)) & 31); }

// Split-radix DFT of length R (power of two, R <= 32), natural order in and out, unscaled:
//   X[k] = sum_n v[n] exp(DIR 2 pi i n k / R).  DIT split: U = DFT_{R/2}(v[2n]),
//   Z = DFT_{R/4}(v[4n+1]), Z' = DFT_{R/4}(v[4n+3]); for k < R/4, a = w^k Z[k],
//   b = w^{3k} Z'[k]:  X[k] = U[k] + (a + b),  X[k+R/2] = U[k] - (a + b),
//   X[k+R/4] = U[k+R/4] + DIR i (a - b),  X[k+3R/4] = U[k+R/4] - DIR i (a - b).
// Fewer twiddle multiplies than the radix-2 stages of dft<> (same additions).
template <int R, int DIR>
CSSAR_DEV void dft_sr(float2 (&v)[R]) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    const float2 a = v[0], b = v[1];
    v[0] = a + b;
    v[1] = a - b;
  } else {
    float2 u[R / 2], z[R / 4], zp[R / 4];
#pragma unroll
    for (int n = 0; n < R / 2; ++n) u[n] = v[2 * n];
#pragma unroll
    for (int n = 0; n < R / 4; ++n) {
      z[n] = v[4 * n + 1];
      zp[n] = v[4 * n + 3];
    }
    dft_sr<R / 2, DIR>(u);
    dft_sr<R / 4, DIR>(z);
    dft_sr<R / 4, DIR>(zp);
#pragma unroll
    for (int k = 0; k < R / 4; ++k) {
      const float2 a = twN<R, DIR>(z[k], k), b = twN<R, DIR>(zp[k], 3 * k);
      const float2 s = a + b, d = a - b;
      const float2 id = DIR > 0 ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);   // DIR i (a - b)
      v[k] = u[k] + s;
      v[k + R / 2] = u[k] - s;
      v[k + R / 4] = u[k + R / 4] + id;
      v[k + 3 * R / 4] = u[k + R / 4] - id;
    }
  }
}

// exp(DIR * 2 pi i * num / den) for integers 0 <= num < den, den a power of two <= 2^24:
// the argument 2*num/den is exact in fp32 and sincospif is accurate to ~1 ulp.
template <int DIR>
CSSAR_DEV float2 expi_frac(uint32_t num, uint32_t den) {
  float s, c;
  sincospif(2.0f * (float)num / (float)den, &s, &c);
  return make_float2(c, DIR > 0 ? s : -s);
}

// x[r] *= w^r, r = 1..R-1, w = exp(DIR 2 pi i k / L): exact anchors w^(2^a) from sincospif
// on the reduced integer argument; w^r = w^(r - lowbit(r)) * anchor(lowbit(r)), i.e. at
// most log2(R) - 1 roundings per power.
template <int R, int DIR>
CSSAR_DEV void apply_twiddles(float2* x, uint32_t k, uint32_t L) {
  constexpr int LR = Log2<R>::v;
  float2 anc[LR > 0 ? LR : 1];
#pragma unroll
  for (int a = 0; a < LR; ++a) anc[a] = expi_frac<DIR>((k << a) & (L - 1), L);
  float2 w[R];
  w[0] = make_float2(1.f, 0.f);
#pragma unroll
  for (int r = 1; r < R; ++r) {
    const int low = r & (-r);
    const int a = ilog2c(low);
    w[r] = (r == low) ? anc[a] : cmul(w[r - low], anc[a]);
  }
#pragma unroll
  for (int r = 1; r < R; ++r) x[r] = cmul(x[r], w[r]);
}

// exp(2 pi i t / 2^24) for a 24-bit integer t from a 256-entry SMEM table of exp(2 pi i h/256)
// (top 8 bits) times a short polynomial for the low 16 bits (|theta| < 2 pi/256:
// cos error theta^4/24 < 1.6e-8, sin error theta^5/120 < 1e-10).
CSSAR_DEV float2 expi24(const float2* tab256, uint32_t t) {
  const float2 h = tab256[t >> 16];
  const float th = (float)(t & 0xFFFFu) * 3.7450702829239464e-07f;   // 2 pi / 2^24
  const float t2 = th * th;
  const float c = fmaf(-0.5f, t2, 1.0f);
  const float s = th * fmaf(-0.16666667f, t2, 1.0f);
  return make_float2(fmaf(h.x, c, -h.y * s), fmaf(h.x, s, h.y * c));
}

// cooperative copy of n (even) float2 from global to SMEM with 16-byte accesses
CSSAR_DEV void copy_table(float2* dst, const float2* src, int n, int t, int nthreads) {
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int i = t; i < n / 2; i += nthreads) d4[i] = __ldg(s4 + i);
}

CSSAR_DEV void init_expi_table(float2* tab256, int t, int nthreads) {
  for (int i = t; i < 256; i += nthreads) {
    float s, c;
    sincospif((float)i * (1.0f / 128.0f), &s, &c);
    tab256[i] = make_float2(c, s);
  }
}

// ---------------------------------------------------------------------------------
// Fixed-point CSA phases: each phase screen row is a
// quadratic P(u) = C2 u^2 + C1 u + C0 in *cycles*, coefficients stored as u64 fractions
// of a cycle (2^64 = 1 cycle).  Wrap-around u64 arithmetic is exact mod 1 cycle.
// The phase is the top 24 bits rounded to nearest, converted exactly to fp32.
struct Quad { uint64_t c2, c1, c0; };

CSSAR_DEV uint64_t quad_eval(const Quad& q, int32_t u) {
  uint64_t uu = (uint64_t)(int64_t)u;
  uint64_t u2 = (uint64_t)((int64_t)u * (int64_t)u);
  return q.c2 * u2 + q.c1 * uu + q.c0;
}

// exp(+-2 pi i P / 2^64).  Default: the top 32 bits of P as a signed fraction of a cycle
// (|f| <= 1/2, i.e. |angle| <= pi, the SFU's most accurate range) through the SFU sin/cos
// (sin.approx / cos.approx: absolute error ~5e-7; 5 issue slots).  CSSAR_PHASE_TABLE: the
// earlier exact path, top 24 bits rounded -> 256-entry SMEM table x 2-term polynomial
// (error < 2e-8, ~13 issue slots + a table load).
// exp(+-2 pi i h / 2^32) for the top 32 bits h of a fixed-point phase (SFU path)
template <bool CONJ>
CSSAR_DEV float2 phase_from_hi32(uint32_t h) {
  const float ang = (float)(int32_t)h * 1.4629180792671596e-09f;   // 2 pi / 2^32
  float sn, cs;
  asm("sin.approx.f32 %0, %1;" : "=f"(sn) : "f"(ang));
  asm("cos.approx.f32 %0, %1;" : "=f"(cs) : "f"(ang));
  return make_float2(cs, CONJ ? -sn : sn);
}

template <bool CONJ>
CSSAR_DEV float2 phase_from_fixed(const float2* tab256, uint64_t P) {
#if defined(CSSAR_PHASE_TABLE)
  const uint32_t t = (uint32_t)((P + (1ull << 39)) >> 40) & 0xFFFFFFu;
  const float2 e = expi24(tab256, t);
#else
  (void)tab256;
  const int32_t hi = (int32_t)(uint32_t)(P >> 32);
  const float ang = (float)hi * 1.4629180792671596e-09f;          // 2 pi / 2^32
  float sn, cs;
  asm("sin.approx.f32 %0, %1;" : "=f"(sn) : "f"(ang));
  asm("cos.approx.f32 %0, %1;" : "=f"(cs) : "f"(ang));
  const float2 e = make_float2(cs, sn);
#endif
  return make_float2(e.x, CONJ ? -e.y : e.y);
}

}  // namespace cssar
