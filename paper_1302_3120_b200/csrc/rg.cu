// Range sweeps (S2 G body, S4 M body): one or more range lines per CTA.
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
  using En = Engine<LOGN, B, T, false, E>;
  static constexpr int TAB = 256 + En::TW_TOTAL;                // phase table + twiddle tables
  static constexpr size_t SMEM = sizeof(float2) * (N * B + TAB);
};

// ------------------------------------------------------------------ RDA RCMC (NEXT-2)
// eq. 16 with the truncated kernel of 8 taps on the torus (oracle/rda.py):
// output gate j of Doppler row i sits at j + d(j), d(j) = s0_i + alpha_i (j - N/2) range cells
// (alpha = 1/D - 1, s0 = alpha 2 R_ref F_r / c), taps m = floor(d) - 3 .. floor(d) + 4:
//   C   : U[j] = sum_m sinc(m - d(j)) V[(j + m) mod N]
//   D=C^T (eq. 17, 23): W[k] = sum_{j, m : j + m = k mod N} sinc(m - d(j)) V[j]
// with sinc(m - d) = (-1)^(m+1) sin(pi d) / (pi (m - d)) (= 1 at m = d, d an integer).
CSSAR_DEV float rcmc_shift(float2 rc, int j, int n) { return fmaf(rc.x, (float)(j - n / 2), rc.y); }

// C at output gate j of one row staged (unswizzled) in SMEM row v
template <int N>
CSSAR_DEV float2 rcmc_gather(const float2* v, float2 rc, int j) {
  const float d = rcmc_shift(rc, j, N);
  const float fl = floorf(d);
  const float S = sinpif(d) * 0.318309886183790672f;       // sin(pi d) / pi
  const int m0 = (int)fl - 3;
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int m = m0 + t;
    const float den = (float)m - d;
    const float w = den == 0.f ? 1.0f : __fdividef((m & 1) ? S : -S, den);
    const float2 x = v[(j + m) & (N - 1)];
    acc.x = fmaf(w, x.x, acc.x);
    acc.y = fmaf(w, x.y, acc.y);
  }
  return acc;
}

// S(d) V for the transpose: V premultiplied by sin(pi d(j)) / pi, or V itself where d(j) is an
// integer (the kernel is then the unit impulse at m = d)
template <int N>
CSSAR_DEV float2 rcmc_stage_T(float2 x, float2 rc, int j) {
  const float d = rcmc_shift(rc, j, N);
  const float S = d == floorf(d) ? 1.0f : sinpif(d) * 0.318309886183790672f;
  return make_float2(S * x.x, S * x.y);
}

// D = C^T at output gate k: the sources j' = k - m whose 8 taps cover k; |d(j) - d(k)| < 1
// for every j of the row (validated at plan creation: alpha n_rg < 1/2), so they lie in
// j' = k - floor(d(k)) - 5 .. k - floor(d(k)) + 4 (unwrapped; j = j' mod N)
template <int N>
CSSAR_DEV float2 rcmc_scatter_T(const float2* p, float2 rc, int k) {
  const int jc = k - (int)floorf(rcmc_shift(rc, k, N));
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = -5; c < 5; ++c) {
    const int jp = jc + c;
    const int j = jp & (N - 1);
    const float d = rcmc_shift(rc, j, N);
    const float fl = floorf(d);
    const int m = k - jp;
    const int mm = m - (int)fl;
    if (mm >= -3 && mm <= 4) {
      float w;
      if (d == fl) {
        w = mm == 0 ? 1.0f : 0.0f;
      } else {
        w = __fdividef((m & 1) ? 1.0f : -1.0f, (float)m - d);
      }
      const float2 x = p[j];
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
  const int row0 = blockIdx.x * C::B;
  float2* tab = s + N * C::B;                 // exp(2 pi i h / 256) for the phase generator
  const float2* tw = tab + 256;               // inter-pass twiddles
  const int t = threadIdx.x;
  copy_table_async(tab, a.tab, C::TAB, t, C::T);
  float2* __restrict__ data = a.data;
  constexpr int LR0 = En::template lr<false>(0), LRL = En::template lr<false>(En::P - 1);

  float2 v[En::E];
  // element j of local row rr: plain row-major, or [peer][row][w] blocks (multi-GPU)
  auto at = [&](int rr, int j) -> size_t {
    if constexpr (BLK) {
      const int wm = (1 << a.log_w) - 1;
      return (size_t)(j >> a.log_w) * (size_t)a.blk + ((size_t)rr << a.log_w) + (size_t)(j & wm);
    } else {
      return (size_t)rr * N + j;
    }
  };
  En::template for_groups<LR0>(v, t, [&](int b, int j, float2* x) {      // raw row loads
#pragma unroll
    for (int r = 0; r < R0; ++r) x[r] = data[at(row0 + b, j + r * (N / R0))];
  });
  cp_async_wait_all();
  __syncthreads();                                                        // tables visible
  if constexpr (!RDA) {
    En::template for_groups<LR0>(v, t, [&](int b, int j, float2* x) {    // prologue phase
      const Quad q = a.coef[a.row_base + row0 + b].q[GBODY ? 2 : 0];
      phase_apply<R0, N / R0, GBODY>(tab, q, j - N / 2, x);
    });
  } else if constexpr (GBODY) {
    En::template for_groups<LR0>(v, t, [&](int b, int j, float2* x) {    // P_eta*, stage S V
      const int row = a.row_base + row0 + b;
      phase_apply<R0, N / R0, true>(tab, a.coef[row].q[2], j - N / 2, x);
      const float2 rc = a.rcmc[row];
#pragma unroll
      for (int r = 0; r < R0; ++r) s[b * N + j + r * (N / R0)] = rcmc_stage_T<N>(x[r], rc, j + r * (N / R0));
    });
    __syncthreads();
    En::template for_groups<LR0>(v, t, [&](int b, int k, float2* x) {    // D = C^T
      const float2 rc = a.rcmc[a.row_base + row0 + b];
#pragma unroll
      for (int r = 0; r < R0; ++r) x[r] = rcmc_scatter_T<N>(s + b * N, rc, k + r * (N / R0));
    });                                 // the FFT's first exchange syncs before overwriting s
  }
  En::template passes_from<-1, false, 0>(s, v, t, tw);                   // range FFT
  En::template for_groups<LRL>(v, t, [&](int b, int j, float2* x) {
    const Quad q = a.coef[a.row_base + row0 + b].q[1];
    // bins j + r N/RL: r < RL/2 -> l' = i ; r >= RL/2 -> l' = i - N (fftfreq order, R9)
    phase_apply<RL / 2, N / RL, GBODY>(tab, q, j, x);
    phase_apply<RL / 2, N / RL, GBODY>(tab, q, j - N / 2, x + RL / 2);
  });
  En::template passes_from<+1, true, 0>(s, v, t, tw);                    // range IFFT
  if constexpr (RDA && !GBODY) {                                          // C on the whole row
    __syncthreads();                    // every thread finished reading the last exchange
    En::template for_groups<LR0>(v, t, [&](int b, int j, float2* x) {
#pragma unroll
      for (int r = 0; r < R0; ++r) s[b * N + j + r * (N / R0)] = x[r];
    });
    __syncthreads();
    En::template for_groups<LR0>(v, t, [&](int b, int j, float2* x) {
      const float2 rc = a.rcmc[a.row_base + row0 + b];
#pragma unroll
      for (int r = 0; r < R0; ++r) x[r] = rcmc_gather<N>(s + b * N, rc, j + r * (N / R0));
    });
  }
  En::template for_groups<LR0>(v, t, [&](int b, int j, float2* x) {
    if constexpr (!RDA) {
      const Quad q = a.coef[a.row_base + row0 + b].q[GBODY ? 0 : 2];
      phase_apply<R0, N / R0, GBODY>(tab, q, j - N / 2, x);
    } else if constexpr (!GBODY) {
      phase_apply<R0, N / R0, false>(tab, a.coef[a.row_base + row0 + b].q[2], j - N / 2, x);   // P_eta
    }
    if constexpr (BLK) {
      if (a.dst[0]) {                      // fused transpose: straight into the ranks' column slabs
        const int wm = (1 << a.log_w) - 1;
        const size_t rowoff = (size_t)((a.drank << a.dlog_nrow) + row0 + b) << a.log_w;
#pragma unroll
        for (int r = 0; r < R0; ++r) {
          const int jj = j + r * (N / R0);
          a.dst[jj >> a.log_w][rowoff + (size_t)(jj & wm)] = x[r];
        }
        return;
      }
    }
#pragma unroll
    for (int r = 0; r < R0; ++r) data[at(row0 + b, j + r * (N / R0))] = x[r];   // 1/n_rg folded into AzArgs::oscale
  });
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
  k<<<n_rows / C::B, C::T, C::SMEM, s>>>(a);
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
