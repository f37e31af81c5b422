// CTA-level batched FFT engine (Stockham autosort, register butterflies, SMEM exchanges).
//
// A CTA holds B independent transforms of length N = 2^LOGN (B*N complex64 in SMEM).
// Each of the T threads owns E = N*B/T elements in registers.  A pass of radix R
// processes N*B/R butterflies; thread t handles butterflies g = m*T + t, m < E/R.
// Butterfly g -> (batch b, index j):  BMINOR (SMEM [i][b], azimuth panels): b = g % B,
// j = g / B;  otherwise (SMEM [b][i], range rows): b = g / (N/R), j = g % (N/R).
//
// Stockham pass (radix R, NS = product of earlier radices), butterfly j, k = j % NS:
//   v[r] = in[j + r N/R] * w_{NS R}^{r k};  v = DFT_R(v);  out[(j/NS) NS R + k + r NS] = v[r].
// The first pass reads through a caller Load functor (global memory + prologue), the last
// pass hands natural-order elements j + r N/R to a Store functor (epilogue + global
// memory).  fft_conv() runs transform -> Mid -> inverse transform with the Mid functor
// applied in registers between the last forward pass and the first inverse pass (they act
// on the same element groups j + r N/R), saving two SMEM exchanges.
//
// SMEM bank conflicts: the writer of an exchange with NS < G (G = transform indices per
// 128-byte wavefront) XOR-swizzles index bits [log2 NS, log2 G) with the bits above
// log2(NS R); reader and writer agree on the swizzle of each exchange.
#pragma once
#include "common.cuh"
#include "cluster.cuh"

namespace cssar {

// ----- radix plans: log2 of the radix of each pass for a length 2^logn with E elements per
// thread (every radix <= E).  E = 32: 7:[16,8] 8:[16,16] 9:[16,32] 10:[32,32] 11:[16,8,16]
// 12:[16,16,16] 13:[16,32,16] 14:[32,16,32] 15:[32,32,32].  E = 16: 7:[16,8] 8:[16,16]
// 9:[8,8,8] 10:[16,8,8] 11:[16,8,16] 12:[16,16,16].
CSSAR_DEV constexpr int plan_passes(int logn, int E) {
  return E == 16 ? (logn <= 8 ? 2 : 3) : (logn <= 10 ? 2 : 3);
}
CSSAR_DEV constexpr int plan_lr(int logn, int E, int p) {
  if (E == 16) {
    return logn == 7 ? (p == 0 ? 4 : 3)
         : logn == 8 ? 4
         : logn == 9 ? 3
         : logn == 10 ? (p == 0 ? 4 : 3)
         : logn == 11 ? (p == 1 ? 3 : 4)
         : 4;
  }
  return logn == 7 ? (p == 0 ? 4 : 3)
       : logn == 8 ? 4
       : logn == 9 ? (p == 0 ? 4 : 5)
       : logn == 10 ? 5
       : logn == 11 ? (p == 1 ? 3 : 4)
       : logn == 12 ? 4
       : logn == 13 ? (p == 1 ? 5 : 4)
       : logn == 14 ? (p == 1 ? 4 : 5)
       : 5;
}
CSSAR_DEV constexpr bool plan_ok(int logn, int E) {
  return (E == 32 && logn >= 7 && logn <= 15) || (E == 16 && logn >= 7 && logn <= 12);
}

// PIO_ (paired I/O, row engines): the first forward pass and the last reverse pass give each
// thread two ADJACENT butterfly groups j, j + 1 (g = 2t + m) instead of g = m T + t, so the
// caller's global loads / stores of those passes are 16-byte accesses of (j, j + 1) pairs; the
// exchange written by the first pass XOR-swizzles with the index bits one position higher
// (pairs of groups share a row of banks), which keeps its writes conflict-free.
template <int LOGN, int B, int T, bool BMINOR, int E_ = 32, bool PIO_ = false>
struct Engine {
  static constexpr int N = 1 << LOGN;
  static constexpr int E = E_;
  static_assert(plan_ok(LOGN, E), "no radix plan for this (N, E)");
  static constexpr int P = plan_passes(LOGN, E);
  static_assert(N * B == T * E, "CTA shape must give E elements per thread");
  static constexpr int G = BMINOR ? (B >= 16 ? 1 : 16 / B) : 16;

  // radix / NS of pass p; REV = passes in reverse order (the inverse half of fft_conv)
  template <bool REV>
  static CSSAR_DEV constexpr int lr(int p) { return plan_lr(LOGN, E, REV ? P - 1 - p : p); }
  template <bool REV>
  static CSSAR_DEV constexpr int lns(int p) {
    int s = 0;
    for (int q = 0; q < p; ++q) s += lr<REV>(q);
    return s;
  }

  // ---- inter-pass twiddle tables (SMEM, forward sign; conjugated on use for DIR = +1).
  // Pass (NS, R), L = NS R: single level T[r NS + k] = w_L^{r k} when L <= 1024, else two
  // levels with k = 64 kh + kl: lo[r 64 + kl] = w_L^{r kl}, hi[r (NS/64) + kh] = w_L^{64 r kh}.
  static CSSAR_DEV constexpr int tw_size_of(int lns, int lr) {
    return lns == 0 ? 0 : (lns + lr <= 10) ? (1 << (lns + lr)) : ((1 << lr) * 64 + (1 << lr) * (1 << (lns - 6)));
  }
  // forward pass with the same (NS, R) as reverse pass p, or 0 if none
  static CSSAR_DEV constexpr int tw_same_fwd(int p) {
    for (int q = 1; q < P; ++q)
      if (lns<false>(q) == lns<true>(p) && lr<false>(q) == lr<true>(p)) return q;
    return 0;
  }
  template <bool REV>
  static CSSAR_DEV constexpr int tw_off(int p) {
    if (REV && tw_same_fwd(p)) return tw_off<false>(tw_same_fwd(p));
    int o = 0;
    if (REV) {
      for (int q = 1; q < P; ++q) o += tw_size_of(lns<false>(q), lr<false>(q));
      for (int q = 1; q < p; ++q)
        if (!tw_same_fwd(q)) o += tw_size_of(lns<true>(q), lr<true>(q));
    } else {
      for (int q = 1; q < p; ++q) o += tw_size_of(lns<false>(q), lr<false>(q));
    }
    return o;
  }
  static CSSAR_DEV constexpr int tw_total() {
    int o = 0;
    for (int q = 1; q < P; ++q) o += tw_size_of(lns<false>(q), lr<false>(q));
    for (int q = 1; q < P; ++q)
      if (!tw_same_fwd(q)) o += tw_size_of(lns<true>(q), lr<true>(q));
    return o;
  }
  static constexpr int TW_TOTAL = tw_total();
  // forward-order tables come first: kernels that only run forward-order passes (run_keep,
  // run, run_from_smem) need just the first TW_FWD entries
  static CSSAR_DEV constexpr int tw_fwd() {
    int o = 0;
    for (int q = 1; q < P; ++q) o += tw_size_of(lns<false>(q), lr<false>(q));
    return o;
  }
  static constexpr int TW_FWD = tw_fwd();

  // fill the twiddle tables (one entry per thread-iteration; exact sincospif arguments)
  static CSSAR_DEV void build_tw(float2* tw, int t, int nthreads) {
    build_tw_rev<false, 1>(tw, t, nthreads);
    build_tw_rev<true, 1>(tw, t, nthreads);
  }
  template <bool REV, int p>
  static CSSAR_DEV void build_tw_rev(float2* tw, int t, int nthreads) {
    if constexpr (p < P) {
      if constexpr (REV && tw_same_fwd(p) != 0) {
        build_tw_rev<REV, p + 1>(tw, t, nthreads);
        return;
      }
      constexpr int LR = lr<REV>(p), LNS = lns<REV>(p);
      constexpr int R = 1 << LR, NS = 1 << LNS, L = NS * R;
      float2* base = tw + tw_off<REV>(p);
      if constexpr (L <= 1024) {
        for (int e = t; e < L; e += nthreads) {
          const int r = e / NS, k = e % NS;
          base[e] = expi_frac<-1>((uint32_t)(r * k) & (L - 1), L);
        }
      } else {
        for (int e = t; e < R * 64; e += nthreads) {
          const int r = e / 64, kl = e % 64;
          base[e] = expi_frac<-1>((uint32_t)(r * kl) & (L - 1), L);
        }
        for (int e = t; e < R * (NS / 64); e += nthreads) {
          const int r = e / (NS / 64), kh = e % (NS / 64);
          base[R * 64 + e] = expi_frac<-1>((uint32_t)(r * kh * 64) & (L - 1), L);
        }
      }
      build_tw_rev<REV, p + 1>(tw, t, nthreads);
    }
  }

  // (the first forward pass and the last reverse pass both have radix plan_lr(LOGN, E, 0))
  static constexpr bool PIO = PIO_ && !BMINOR && P >= 2;
  static_assert(!PIO || (E / (1 << plan_lr(LOGN, E, 0))) % 2 == 0,
                "paired I/O needs an even number of groups per thread in the first / last passes");

  template <int LNS, int LR, int SH = 0>
  static CSSAR_DEV int swz(int i) {
    constexpr int NS = 1 << LNS;
    if constexpr (NS >= G || LNS + LR + SH >= LOGN) {
      return i;
    } else {
      constexpr int mask = G / NS - 1;
      return i ^ (((i >> (LNS + LR + SH)) & mask) << LNS);
    }
  }
  // butterfly group of thread t's m-th group: m T + t, or (paired) 2 ((m / 2) T + t) + m % 2
  template <bool PM>
  static CSSAR_DEV int gmap(int m, int t) { return PM ? 2 * ((m >> 1) * T + t) + (m & 1) : m * T + t; }
  static CSSAR_DEV int addr(int b, int i) { return BMINOR ? i * B + b : b * N + i; }

  template <int R>
  static CSSAR_DEV void bj(int g, int& b, int& j) {
    if constexpr (BMINOR) { b = g % B; j = g / B; }
    else { b = g / (N / R); j = g % (N / R); }
  }

  // butterflies of one pass on registers v (E elements: group m at v[m*R .. m*R+R));
  // tw = this pass's SMEM twiddle table (required for passes with NS > 1)
  template <int LR, int LNS, int DIR, bool PM = false>
  static CSSAR_DEV void butterflies(float2 (&v)[E], int t, const float2* tw) {
    constexpr int R = 1 << LR, NS = 1 << LNS, L = NS * R;
#if defined(CSSAR_EXP_NOFFT_AZ)
    if constexpr (BMINOR) return;       // experiment: azimuth data movement without the arithmetic
#endif
#pragma unroll
    for (int m = 0; m < E / R; ++m) {
      int b, j;
      bj<R>(gmap<PM>(m, t), b, j);
      float2 x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = v[m * R + r];
      if constexpr (NS > 1) {
        const int k = j & (NS - 1);
        if constexpr (L <= 1024) {
#pragma unroll
          for (int r = 1; r < R; ++r) x[r] = DIR < 0 ? cmul(x[r], tw[r * NS + k]) : cmulc(x[r], tw[r * NS + k]);
        } else {
          const float2* lo = tw + (k & 63);
          const float2* hi = tw + R * 64 + (k >> 6);
#pragma unroll
          for (int r = 1; r < R; ++r) {
            const float2 w = cmul(lo[r * 64], hi[r * (NS / 64)]);
            x[r] = DIR < 0 ? cmul(x[r], w) : cmulc(x[r], w);
          }
        }
      }
#if defined(CSSAR_DFT_RADIX2)
      dft<R, DIR>(x);
#else
      dft_sr<R, DIR>(x);
#endif
#pragma unroll
      for (int r = 0; r < R; ++r) v[m * R + r] = x[r];
    }
  }

  // write pass output (writer LR, LNS) to SMEM, swizzled for this exchange
  template <int LR, int LNS, bool PM = false, int SH = 0>
  static CSSAR_DEV void write(float2* s, const float2 (&v)[E], int t) {
    constexpr int R = 1 << LR, NS = 1 << LNS;
#pragma unroll
    for (int m = 0; m < E / R; ++m) {
      int b, j;
      bj<R>(gmap<PM>(m, t), b, j);
      const int base = (j >> LNS) * (NS * R) + (j & (NS - 1));
#pragma unroll
      for (int r = 0; r < R; ++r) s[addr(b, swz<LNS, LR, SH>(base + r * NS))] = v[m * R + r];
    }
  }

  // read the input of a pass with radix 2^LR from SMEM written by exchange (WLR, WLNS, WSH);
  // PM (paired groups j, j + 1 of one row) with an unswizzled exchange: one 16-byte load per pair
  template <int LR, int WLR, int WLNS, int WSH = 0, bool PM = false>
  static CSSAR_DEV void read(const float2* s, float2 (&v)[E], int t) {
    constexpr int R = 1 << LR;
    constexpr bool VEC = PM && ((1 << WLNS) >= G || WLNS + WLR + WSH >= LOGN);   // identity swizzle
    if constexpr (VEC) {
#pragma unroll
      for (int m = 0; m < E / R; m += 2) {
        int b, j;
        bj<R>(gmap<PM>(m, t), b, j);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float4 q = *reinterpret_cast<const float4*>(&s[addr(b, j + r * (N / R))]);
          v[m * R + r] = make_float2(q.x, q.y);
          v[(m + 1) * R + r] = make_float2(q.z, q.w);
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < E / R; ++m) {
        int b, j;
        bj<R>(gmap<PM>(m, t), b, j);
#pragma unroll
        for (int r = 0; r < R; ++r) v[m * R + r] = s[addr(b, swz<WLNS, WLR, WSH>(j + r * (N / R)))];
      }
    }
  }

  template <int LR, class F, bool PM = false>
  static CSSAR_DEV void for_groups(float2 (&v)[E], int t, F&& f) {
    constexpr int R = 1 << LR;
#pragma unroll
    for (int m = 0; m < E / R; ++m) {
      int b, j;
      bj<R>(gmap<PM>(m, t), b, j);
      f(b, j, &v[m * R]);
    }
  }
  // the groups of the first forward / last reverse pass (paired when PIO)
  template <int LR, class F>
  static CSSAR_DEV void for_io(float2 (&v)[E], int t, F&& f) {
    for_groups<LR, F, PIO>(v, t, static_cast<F&&>(f));
  }

  // Passes p = P0 .. P-1 of a transform whose first pass input is already in registers.
  // On return the last pass output (natural order, groups j + r N/R_last) is in v.
  template <int DIR, bool REV, int p>
  static CSSAR_DEV void passes_from(float2* s, float2 (&v)[E], int t, const float2* tw) {
    constexpr int LR = lr<REV>(p), LNS = lns<REV>(p);
    // paired groups: the first forward pass (input from the caller) and the last reverse pass
    constexpr bool PM = PIO && ((p == 0 && !REV) || (p == P - 1 && REV));
    constexpr bool PMN = PIO && (p + 1 == P - 1 && REV);          // the next pass
    constexpr int SH = (PIO && p == 0 && !REV) ? 1 : 0;            // swizzle shift of this exchange
    if constexpr (p == 0 && !REV) cp_async_wait_all();   // async table staging (no-op if none)
    butterflies<LR, LNS, DIR, PM>(v, t, tw + tw_off<REV>(p));
    if constexpr (p + 1 < P) {
      __syncthreads();                 // everyone finished reading the previous exchange
#if defined(CSSAR_EXP_NOXCH_AZ)
      if constexpr (!BMINOR) {         // experiment: azimuth passes without the SMEM exchange
#endif
      write<LR, LNS, PM, SH>(s, v, t);
#if defined(CSSAR_EXP_NOXCH_AZ)
      }
#endif
      __syncthreads();
#if defined(CSSAR_EXP_NOXCH_AZ)
      if constexpr (!BMINOR)
#endif
      read<lr<REV>(p + 1), LR, LNS, SH, PMN>(s, v, t);
      passes_from<DIR, REV, p + 1>(s, v, t, tw);
    }
  }

  // Load functor: ld(b, j, x) fills x[r] = input element (b, j + r N/R0), R0 = first radix.
  // Store functor: st(b, j, x) consumes output elements (b, j + r N/R_last).
  template <int DIR, class Load, class Store>
  static CSSAR_DEV void run(float2* s, Load&& ld, Store&& st, const float2* tw) {
    const int t = threadIdx.x;
    float2 v[E];
    for_io<lr<false>(0)>(v, t, ld);
    passes_from<DIR, false, 0>(s, v, t, tw);
    for_groups<lr<false>(P - 1)>(v, t, st);
  }

  // transform(DIR) -> mid -> transform(-DIR), mid acting on natural-order groups in registers
  template <int DIR, class Load, class Mid, class Store>
  static CSSAR_DEV void conv(float2* s, Load&& ld, Mid&& mid, Store&& st, const float2* tw) {
    const int t = threadIdx.x;
    float2 v[E];
    for_io<lr<false>(0)>(v, t, ld);
    passes_from<DIR, false, 0>(s, v, t, tw);
    for_groups<lr<false>(P - 1)>(v, t, mid);
    passes_from<-DIR, true, 0>(s, v, t, tw);
    for_io<lr<true>(P - 1)>(v, t, st);
  }

  // run() without the Store: the natural-order output groups stay in v (for cluster kernels)
  template <int DIR, class Load>
  static CSSAR_DEV void run_keep(float2* s, float2 (&v)[E], Load&& ld, const float2* tw) {
    const int t = threadIdx.x;
    for_io<lr<false>(0)>(v, t, ld);
    passes_from<DIR, false, 0>(s, v, t, tw);
  }

  // write the natural-order output groups of the last pass (radix of pass P-1) unswizzled
  // to s[addr(b, i)]; brackets the write with barriers (other threads may still be reading
  // the last exchange, and readers of the result must wait for every writer)
  static CSSAR_DEV void store_natural(float2* s, const float2 (&v)[E]) {
    const int t = threadIdx.x;
    constexpr int LR = lr<false>(P - 1), R = 1 << LR;
    __syncthreads();
#pragma unroll
    for (int m = 0; m < E / R; ++m) {
      int b, j;
      bj<R>(m * T + t, b, j);
#pragma unroll
      for (int r = 0; r < R; ++r) s[addr(b, j + r * (N / R))] = v[m * R + r];
    }
    __syncthreads();
  }

  // Same as run(), but the first pass reads its input from SMEM in natural order
  // (s[addr(b, i)], unswizzled) — used after a cluster scatter.
  template <int DIR, class Store>
  static CSSAR_DEV void run_from_smem(float2* s, Store&& st, const float2* tw) {
    const int t = threadIdx.x;
    float2 v[E];
    constexpr int LR0 = lr<false>(0), R0 = 1 << LR0;
    for_io<LR0>(v, t, [&](int b, int j, float2* x) {
#pragma unroll
      for (int r = 0; r < R0; ++r) x[r] = s[addr(b, j + r * (N / R0))];
    });
    passes_from<DIR, false, 0>(s, v, t, tw);
    for_groups<lr<false>(P - 1)>(v, t, st);
  }
};

}  // namespace cssar
