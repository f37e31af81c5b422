// Range sweeps (S2 G body, S4 M body): one or more range lines per CTA.
#include <cstdlib>
#include <type_traits>
#include "device_ops.cuh"
#include "cluster.cuh"

namespace cssar {

// ------------------------------------------------------------------ range sweep
template <int LOGN>
struct RgCfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int E = 32;
  static constexpr int T = LOGN >= 14 ? 512 : 256;
  static constexpr int B = (T * E) / N > 0 ? (T * E) / N : 1;
#ifndef CSSAR_RG_MINB
#define CSSAR_RG_MINB 2
#endif
  static constexpr int MINB = LOGN >= 14 ? 1 : CSSAR_RG_MINB;   // resident CTAs per SM (register cap)
  // paired I/O (16-byte row loads / stores) where the first radix leaves two groups per thread
  static constexpr bool PIO = (E / (1 << plan_lr(LOGN, E, 0))) % 2 == 0;
  using En = Engine<LOGN, B, T, false, E, PIO>;
  static constexpr int TAB = 256 + En::TW_TOTAL;                // phase table + twiddle tables
  static constexpr size_t SMEM = sizeof(float2) * (N * B + TAB);
};

// ------------------------------------------------------------------ RDA RCMC (NEXT-2)
// eq. 16 with the truncated kernel of 8 taps on the torus (oracle/rda.py):
// output gate j of Doppler row i sits at j + d(j), d(j) = s0_i + alpha_i (j - N/2) range cells
// (alpha = 1/D - 1 >= 0, s0 = alpha 2 R_ref F_r / c), taps m = floor(d) - 3 .. floor(d) + 4:
//   C   : U[j] = sum_m sinc(m - d(j)) V[(j + m) mod N]
//   D=C^T (eq. 17, 23): W[k] = sum_{j, m : j + m = k mod N} sinc(m - d(j)) V[j]
// sinc(m - d) = (-1)^(m+1) sin(pi d) / (pi (m - d)) (= 1 at m = d).
//
// Evaluation: the row is staged in SMEM and every thread
// produces 32 consecutive outputs from a sliding register window of 9 inputs.  d varies by
// alpha <= 6e-6 cell per gate (alpha n_rg < 1/2, validated), so over a chunk's 64-gate bracket
// each tap weight sinc(m - d(i)) is linear in the gate index i to < 6e-8: it is evaluated
// exactly at the bracket ends and interpolated (one FMA per tap and output).  The union
// window m = F - 3 .. F + 5 (F = floor d at the bracket start) covers the one possible integer
// crossing of d inside the bracket; its end taps are switched by the crossing gate.  D outputs
// whose sources wrap around the torus (d jumps by alpha n_rg there) are recomputed exactly.
CSSAR_DEV float rcmc_shift(float2 rc, int j, int n) { return fmaf(rc.x, (float)(j - n / 2), rc.y); }
CSSAR_DEV int rsw(int i) { return i ^ ((i >> 5) & 31); }        // staged-row swizzle
constexpr float kInvPi = 0.318309886183790672f;
constexpr int kRcmcWrapLo = 12, kRcmcWrapHi = 3;                  // D outputs recomputed exactly

CSSAR_DEV float sinc_md(int m, float d, float sd) {                // sd = sin(pi d) / pi
  const float den = (float)m - d;
  return den == 0.f ? 1.0f : __fdividef((m & 1) ? sd : -sd, den);
}

// 32 consecutive outputs k0 .. k0+31 of C (TR = false) or D (TR = true) of one staged row
template <int N, bool TR>
CSSAR_DEV void rcmc_chunk(const float2* row, float2 rc, int k0, float2 (&out)[32]) {
  const int ia = k0 - 16, ib = ia + 64;
  const float da = rcmc_shift(rc, ia, N), db = rcmc_shift(rc, ib, N);
  const int F = (int)floorf(da);
  int brk = ib + 1;                                   // first gate with floor(d) = F + 1
  if ((int)floorf(db) > F) {
    int lo = ia, hi = ib;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if ((int)floorf(rcmc_shift(rc, mid, N)) > F) hi = mid; else lo = mid;
    }
    brk = hi;
  }
  const float sa = sinpif(da) * kInvPi, sb = sinpif(db) * kInvPi;
  float A[9], S[9];
#pragma unroll
  for (int u = 0; u < 9; ++u) {
    const int m = F - 3 + u;
    const float ga = sinc_md(m, da, sa);
    S[u] = (sinc_md(m, db, sb) - ga) * (1.0f / 64.0f);
    // weight of tap u at output n: ga + (i - ia) S, i = the gate whose d it uses
    A[u] = fmaf((float)(TR ? 19 - F - u : 16), S[u], ga);
  }
  const int n0 = TR ? brk - k0 + F - 3 : brk - k0;    // tap 0 only while n < n0
  const int n8 = TR ? brk - k0 + F + 5 : brk - k0;    // tap 8 only once n >= n8
  const int base = TR ? k0 - F - 5 : k0 + F - 3;
  float2 win[9];
#pragma unroll
  for (int q = 0; q < 8; ++q) win[q] = row[rsw((base + q) & (N - 1))];
#pragma unroll
  for (int n = 0; n < 32; ++n) {
    win[8] = row[rsw((base + n + 8) & (N - 1))];
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 9; ++u) {
      float w = fmaf(S[u], (float)n, A[u]);
      if (u == 0) w = n < n0 ? w : 0.0f;
      if (u == 8) w = n >= n8 ? w : 0.0f;
      const float2 x = win[TR ? 8 - u : u];
      acc.x = fmaf(w, x.x, acc.x);
      acc.y = fmaf(w, x.y, acc.y);
    }
    out[n] = acc;
#pragma unroll
    for (int q = 0; q < 8; ++q) win[q] = win[q + 1];
  }
}

// D at output k, exact: the sources j' = k - m whose 8 taps cover k; |d(j) - d(k)| < 1 for
// every gate of the row, so they lie in j' = k - floor(d(k)) - 5 .. + 4 (unwrapped)
template <int N>
CSSAR_DEV float2 rcmc_T_exact(const float2* row, float2 rc, int k) {
  const int jc = k - (int)floorf(rcmc_shift(rc, k, N));
  float2 acc = make_float2(0.f, 0.f);
  for (int c = -5; c < 5; ++c) {
    const int jp = jc + c;
    const int j = jp & (N - 1);
    const float d = rcmc_shift(rc, j, N);
    const int m = k - jp;
    const int mm = m - (int)floorf(d);
    if (mm >= -3 && mm <= 4) {
      const float w = sinc_md(m, d, sinpif(d) * kInvPi);
      const float2 x = row[rsw(j)];
      acc.x = fmaf(w, x.x, acc.x);
      acc.y = fmaf(w, x.y, acc.y);
    }
  }
  return acc;
}

// GBODY: Phi3* -> F -> Phi2* -> F^-1 -> Phi1*  (inverse of the focusing steps)
// else : Phi1  -> F -> Phi2  -> F^-1 -> Phi3   (CSA focusing body)
// RDA  : GBODY P_eta* -> D -> F -> P_tau* -> F^-1 ; else F -> P_tau -> F^-1 -> C -> P_eta
//        (eq. 14 / eq. 18 between the azimuth DFTs; q[1] = P_tau, q[2] = P_eta)
template <int LOGN, bool GBODY, bool BLK, bool RDA>
__global__ void __launch_bounds__(RgCfg<LOGN>::T, RgCfg<LOGN>::MINB) rg_sweep_kernel(const RgArgs a) {
  using C = RgCfg<LOGN>;
  using En = typename C::En;
  constexpr int N = C::N;
  constexpr int R0 = 1 << En::template lr<false>(0);
  constexpr int RL = 1 << En::template lr<false>(En::P - 1);
  extern __shared__ float4 smem4[];
  float2* s = reinterpret_cast<float2*>(smem4);
  int row0 = blockIdx.x * C::B;               // persistent: rows row0, row0 + gridDim B, ...
  const int nrows = a.nrows ? a.nrows : (int)gridDim.x * C::B;
  float2* tab = s + N * C::B;                 // exp(2 pi i h / 256) for the phase generator
  const float2* tw = tab + 256;               // inter-pass twiddles
  const int t = threadIdx.x;
#if defined(CSSAR_PHASE_TABLE)
  copy_table_async(tab, a.tab, C::TAB, t, C::T);
#else
  copy_table_async(tab + 256, a.tab + 256, C::TAB - 256, t, C::T);   // the exp table serves CSSAR_PHASE_TABLE only
#endif
  // fused-transpose destinations in SMEM: a dynamically indexed kernel-parameter array would
  // be copied to local memory (the multi-GPU variants spilled 300+ bytes per thread)
  __shared__ float2* sdst[16];
  if constexpr (BLK) {
    if (t < 16) sdst[t] = a.dst[t];
  }
  float2* __restrict__ data = a.data;
  constexpr int LR0 = En::template lr<false>(0), LRL = En::template lr<false>(En::P - 1);

  // global Doppler bin of local row rr: row_base + rr * row_step (contiguous slabs: step 1;
  // the sparse-X' schedule's cyclic slabs: base = rank, step = world)
  auto grow = [&](int rr) -> int {
    if constexpr (BLK) return a.row_base + rr * (a.row_step ? a.row_step : 1);
    else return a.row_base + rr;                                  // single GPU: contiguous rows
  };
  float2 v[En::E];
  static_assert(En::E == 32 && C::T * 32 == N * C::B, "RCMC chunking: 32 consecutive gates per thread");
  // RDA: RCMC of the staged rows (s[b N + rsw(i)]) -> v in the first-pass group layout
  auto rcmc_apply = [&](auto tr_tag, float2* sm, float2 (&vv)[En::E], int tt) {
    constexpr bool TR = decltype(tr_tag)::value;
    const int g = tt * 32, bb = g >> LOGN, k0 = g & (N - 1);
    rcmc_chunk<N, TR>(sm + bb * N, a.rcmc[grow(row0 + bb)], k0, vv);
    constexpr int NF = kRcmcWrapLo + kRcmcWrapHi, SL = C::B * NF, PER = (SL + C::T - 1) / C::T;
    float2 fx[TR ? PER : 1];
    if constexpr (TR) {
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int f = tt + q * C::T;
        if (f < SL) {
          const int fb = f / NF, sl = f % NF;
          const int k = sl < kRcmcWrapLo ? sl : N - NF + sl;
          fx[q] = rcmc_T_exact<N>(sm + fb * N, a.rcmc[grow(row0 + fb)], k);
        }
      }
    }
    __syncthreads();                    // all reads of the staged rows done
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const int k = k0 + n;
      if (!TR || (k >= kRcmcWrapLo && k < N - kRcmcWrapHi)) sm[bb * N + rsw(k)] = vv[n];
    }
    if constexpr (TR) {
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int f = tt + q * C::T;
        if (f < SL) {
          const int fb = f / NF, sl = f % NF;
          sm[fb * N + rsw(sl < kRcmcWrapLo ? sl : N - NF + sl)] = fx[q];
        }
      }
    }
    __syncthreads();
    En::template for_io<LR0>(vv, tt, [&](int b, int j, float2* x) {
#pragma unroll
      for (int r = 0; r < R0; ++r) x[r] = sm[b * N + rsw(j + r * (N / R0))];
    });
  };
  // element j of local row rr: plain row-major, or [peer][row][w] blocks (multi-GPU)
  auto at = [&](int rr, int j) -> size_t {
    if constexpr (BLK) {
      const int wm = (1 << a.log_w) - 1;
      return (size_t)(j >> a.log_w) * (size_t)a.blk + ((size_t)rr << a.log_w) + (size_t)(j & wm);
    } else {
      return (size_t)rr * N + j;
    }
  };
  pdl_wait();                                 // the previous sweep's output is complete
  for (; row0 < nrows; row0 += (int)gridDim.x * C::B) {
  // one CTA per SM (n_rg = 16384, persistent grid): nothing else on the SM hides the next row's
  // load latency, so its rows are brought into L2 while this one is transformed (c4: 4.15 ->
  // 3.65 ms per range sweep; with two CTAs per SM, n_rg <= 8192, the other CTA covers it and
  // the prefetch measured slower)
  if constexpr (!BLK && C::MINB == 1) {
    const int pr = row0 + (int)gridDim.x * C::B;
    if (t == 0 && pr < nrows)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(data + (size_t)pr * N),
                   "r"((uint32_t)(sizeof(float2) * N * C::B)) : "memory");
  }
  if constexpr (En::PIO && !BLK) {            // raw row loads, 16 bytes (groups j, j + 1) each
#pragma unroll
    for (int m = 0; m < En::E / R0; m += 2) {
      int b, j;
      En::template bj<R0>(En::template gmap<true>(m, t), b, j);
      const float2* src = data + (size_t)(row0 + b) * N + j;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const float4 q = *reinterpret_cast<const float4*>(src + r * (N / R0));
        v[m * R0 + r] = make_float2(q.x, q.y);
        v[(m + 1) * R0 + r] = make_float2(q.z, q.w);
      }
    }
  } else {
    En::template for_io<LR0>(v, t, [&](int b, int j, float2* x) {    // raw row loads
#pragma unroll
      for (int r = 0; r < R0; ++r) x[r] = data[at(row0 + b, j + r * (N / R0))];
    });
  }
  cp_async_wait_all();
  __syncthreads();                            // tables visible; the previous rows' SMEM reads done
  if constexpr (!RDA) {
    En::template for_io<LR0>(v, t, [&](int b, int j, float2* x) {    // prologue phase
      const Quad q = a.coef[grow(row0 + b)].q[GBODY ? 2 : 0];
      phase_apply<R0, N / R0, GBODY>(tab, q, j - N / 2, x);
    });
  } else if constexpr (GBODY) {
    En::template for_io<LR0>(v, t, [&](int b, int j, float2* x) {    // P_eta*, stage the row
      phase_apply<R0, N / R0, true>(tab, a.coef[grow(row0 + b)].q[2], j - N / 2, x);
#pragma unroll
      for (int r = 0; r < R0; ++r) s[b * N + rsw(j + r * (N / R0))] = x[r];
    });
    __syncthreads();
    rcmc_apply(std::true_type{}, s, v, t);          // D = C^T; the FFT's first exchange syncs before reusing s
  }
  En::template passes_from<-1, false, 0>(s, v, t, tw);                   // range FFT
  auto mid_quad = [&]() {
    En::template for_groups<LRL>(v, t, [&](int b, int j, float2* x) {
      const Quad q = a.coef[grow(row0 + b)].q[1];
      // bins j + r N/RL: r < RL/2 -> l' = i ; r >= RL/2 -> l' = i - N (fftfreq order, R9)
      phase_apply<RL / 2, N / RL, GBODY>(tab, q, j, x);
      phase_apply<RL / 2, N / RL, GBODY>(tab, q, j - N / 2, x + RL / 2);
    });
  };
  if constexpr (RDA) {
    if (a.hrange) {                     // recorded-pulse filter: H (G body) / conj H (M body)
      En::template for_groups<LRL>(v, t, [&](int b, int j, float2* x) {
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const float2 h = __ldg(a.hrange + j + r * (N / RL));
          x[r] = GBODY ? cmul(x[r], h) : cmulc(x[r], h);
        }
      });
    } else {
      mid_quad();
    }
  } else {
    mid_quad();
  }
  En::template passes_from<+1, true, 0>(s, v, t, tw);                    // range IFFT
  if constexpr (RDA && !GBODY) {                                          // C on the whole row
    __syncthreads();                    // every thread finished reading the last exchange
    En::template for_io<LR0>(v, t, [&](int b, int j, float2* x) {
#pragma unroll
      for (int r = 0; r < R0; ++r) s[b * N + rsw(j + r * (N / R0))] = x[r];
    });
    __syncthreads();
    rcmc_apply(std::false_type{}, s, v, t);
  }
  En::template for_io<LR0>(v, t, [&](int b, int j, float2* x) {
    if constexpr (!RDA) {
      const Quad q = a.coef[grow(row0 + b)].q[GBODY ? 0 : 2];
      phase_apply<R0, N / R0, GBODY>(tab, q, j - N / 2, x);
    } else if constexpr (!GBODY) {
      phase_apply<R0, N / R0, false>(tab, a.coef[grow(row0 + b)].q[2], j - N / 2, x);   // P_eta
    }
    if constexpr (BLK) {
      if (a.dst[0]) {                      // fused transpose: straight into the ranks' column slabs
        const int dlw = a.dlog_w ? a.dlog_w : a.log_w;         // column-slab width of the destinations
        const int wm = (1 << dlw) - 1;
        const size_t rowoff = (size_t)grow(row0 + b) << dlw;
#pragma unroll
        for (int r = 0; r < R0; ++r) {
          const int jj = j + r * (N / R0);
          sdst[jj >> dlw][rowoff + (size_t)(jj & wm)] = x[r];
        }
        return;
      }
    }
    if constexpr (!(En::PIO && !BLK)) {
#pragma unroll
      for (int r = 0; r < R0; ++r) data[at(row0 + b, j + r * (N / R0))] = x[r];   // 1/n_rg folded into AzArgs::oscale
    }
  });
  if constexpr (En::PIO && !BLK) {            // row stores, 16 bytes (groups j, j + 1) each
#pragma unroll
    for (int m = 0; m < En::E / R0; m += 2) {
      int b, j;
      En::template bj<R0>(En::template gmap<true>(m, t), b, j);
      float2* dst = data + (size_t)(row0 + b) * N + j;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const float2 lo = v[m * R0 + r], hi = v[(m + 1) * R0 + r];
        *reinterpret_cast<float4*>(dst + r * (N / R0)) = make_float4(lo.x, lo.y, hi.x, hi.y);
      }
    }
  }
  }
  pdl_launch_dependents();                   // (at the end: dependents may not run ahead)
  if constexpr (BLK) {
    if (a.dst[0]) __threadfence_system();   // peer stores performed before the flag barrier
  }
}

template <int LOGN>
__global__ void rg_table_kernel(float2* dst) {
  using C = RgCfg<LOGN>;
  init_expi_table(dst, threadIdx.x, blockDim.x);
  C::En::build_tw(dst + 256, threadIdx.x, blockDim.x);
}

int rg_rows_per_cta(int log_nrg) {
  switch (log_nrg) {
#define RGB(L) case L: return RgCfg<L>::B;
    RGB(7) RGB(8) RGB(9) RGB(10) RGB(11) RGB(12) RGB(13) RGB(14)
#undef RGB
    default: return 0;
  }
}

size_t rg_table_count(int log_nrg) {
  switch (log_nrg) {
#define RGT(L) case L: return RgCfg<L>::TAB;
    RGT(7) RGT(8) RGT(9) RGT(10) RGT(11) RGT(12) RGT(13) RGT(14)
#undef RGT
    default: return 0;
  }
}

cudaError_t rg_table_fill(int log_nrg, float2* dst, cudaStream_t s) {
  switch (log_nrg) {
#define RGT(L) case L: rg_table_kernel<L><<<1, 256, 0, s>>>(dst); return cudaGetLastError();
    RGT(7) RGT(8) RGT(9) RGT(10) RGT(11) RGT(12) RGT(13) RGT(14)
#undef RGT
    default: return cudaErrorInvalidValue;
  }
}

template <int LOGN, bool GB, bool BLK>
static cudaError_t rg_launch(int n_rows, const RgArgs& a, cudaStream_t s) {
  using C = RgCfg<LOGN>;
  auto k = a.rcmc ? rg_sweep_kernel<LOGN, GB, BLK, true> : rg_sweep_kernel<LOGN, GB, BLK, false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (e != cudaSuccess) return e;
  // one row block per CTA (measured faster than a persistent grid of co-resident CTAs looping
  // over the rows: 0.396 vs 0.436 ms at c3); CSSAR_RG_PERSIST=1 selects the persistent grid.
  // One CTA per SM (n_rg = 16384): always persistent, with the next row prefetched into L2
  static const bool persist_env = [] { const char* v = std::getenv("CSSAR_RG_PERSIST"); return v && std::atoi(v); }();
  const bool persist = persist_env || (C::MINB == 1 && !BLK);
  int grid = n_rows / C::B;
  RgArgs b = a;
  if (persist) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, C::T, C::SMEM) == cudaSuccess && per_sm > 0 &&
        per_sm * sms < grid) {
      grid = per_sm * sms;
      b.nrows = n_rows;
    }
  }
  e = launch_pdl(k, dim3(grid), dim3(C::T), C::SMEM, s, b);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_rg_sweep(int log_nrg, bool gbody, int n_rows, const RgArgs& a, cudaStream_t s) {
#define RG_CASE(L)                                                                        \
  case L:                                                                                 \
    if (a.blk) return gbody ? rg_launch<L, true, true>(n_rows, a, s) : rg_launch<L, false, true>(n_rows, a, s); \
    return gbody ? rg_launch<L, true, false>(n_rows, a, s) : rg_launch<L, false, false>(n_rows, a, s);
  switch (log_nrg) {
    RG_CASE(7) RG_CASE(8) RG_CASE(9) RG_CASE(10) RG_CASE(11) RG_CASE(12) RG_CASE(13) RG_CASE(14)
    default: return cudaErrorInvalidValue;
  }
#undef RG_CASE
}

}  // namespace cssar
