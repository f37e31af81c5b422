// Azimuth sweeps (S1 head, S3 residual, S5 tail, operator heads/tails): column panels,
// thread-block clusters + DSMEM for long columns.  Instantiated per log2(n_az) in az_*.cu.
#pragma once
#include "device_ops.cuh"
#include "cluster.cuh"

namespace cssar {

// ------------------------------------------------------------------ azimuth sweeps
// R = configuration for the residual kernel (two transforms; more registers)
template <int LOGN, bool R>
struct AzCfg {
  // column panel of W range bins, split over a cluster of C CTAs (M = N/C rows each);
  // 4096-8192 complex64 per CTA (32-64 KB SMEM), E elements per thread
  static constexpr int C = LOGN <= 10 ? 1 : LOGN == 11 ? 2 : LOGN == 12 ? 4 : LOGN == 13 ? (R ? 16 : 8) : 16;
  static constexpr int W = LOGN <= 8 ? 16 : LOGN == 9 ? 8 : LOGN == 13 ? 8 : 4;
  static constexpr int E = 16;
};
#if defined(CSSAR_AZ13_C)
template <>
struct AzCfg<13, false> {
  static constexpr int C = CSSAR_AZ13_C, W = CSSAR_AZ13_W, E = CSSAR_AZ13_E;
};
#endif
#if defined(CSSAR_AZ13R_C)
template <>
struct AzCfg<13, true> {
  static constexpr int C = CSSAR_AZ13R_C, W = CSSAR_AZ13R_W, E = CSSAR_AZ13R_E;
};
#endif

template <int LOGN, bool R = false>
struct AzShape {
  using P = AzCfg<LOGN, R>;
  static constexpr int C = P::C, W = P::W, E = P::E;
  static constexpr int LOGM = LOGN - ilog2c(C);
  static constexpr int M = 1 << LOGM;
  static constexpr int T = M * W / E;
  static constexpr int MINB = T <= 128 ? 4 : T <= 256 ? (E == 32 ? 2 : 3) : (E == 32 ? 1 : 2);
  static constexpr int NBUF = C > 1 ? 2 : 1;               // RESID double-buffers the scatter
  using En = Engine<LOGM, W, T, true, E>;
  static constexpr int TW = En::TW_TOTAL;
  static constexpr size_t SMEM_FFT = sizeof(float2) * (M * W + TW);
  static constexpr int CAND_SMEM = 1024;
  static constexpr size_t SMEM_TAIL = SMEM_FFT + sizeof(uint32_t) * (HIST_BINS + CAND_SMEM + 4);
  static constexpr size_t SMEM_RESID = SMEM_FFT + sizeof(float2) * M * W * (NBUF - 1);
};

struct TailCtx {
  uint32_t* shist;
  uint32_t* scand;
  uint32_t* scount;      // [0] = candidates in SMEM, [1] = fixed-lambda survivors
  int floor_bin, cand_lo, cand_hi;
  uint32_t s2bits, s2fixed;
  float sigma;
};

// auxiliary per-element inputs, fetched for a whole group before any arithmetic so the
// loads are in flight together (long-scoreboard latency overlaps)
struct Aux {
  float2 v;        // Y (RESID) or b_{i-1} (TAIL)
  uint32_t m;      // mask bit
};

template <int MODE>
struct AzOps {
  static constexpr int DIR = (MODE <= AZ_FWD_THR) ? -1 : +1;   // first transform direction

  // prologue on a loaded input value (loads are issued for a whole group first)
  CSSAR_DEV static float2 pro(const AzArgs& a, int row, int col, float2 v, uint32_t s2, float sig) {
    if constexpr (MODE == AZ_FWD_MASK) {
      if (!mask_bit(a.mask, a.mask_words, row, col)) v = make_float2(0.f, 0.f);
    }
    if constexpr (MODE == AZ_FWD_THR) v = threshold(v, s2, sig, a.thr);
    return v;
  }

  CSSAR_DEV static Aux fetch(const AzArgs& a, int row, int col, size_t idx) {
    Aux x{make_float2(0.f, 0.f), 1u};
    if constexpr (MODE == AZ_RESID) {
      x.m = mask_bit(a.mask, a.mask_words, row, col);
      x.v = __ldg(a.Y + idx);
    } else if constexpr (MODE == AZ_INV_MASK) {
      x.m = mask_bit(a.mask, a.mask_words, row, col);
    } else if constexpr (MODE == AZ_TAIL) {
      x.v = a.b[idx];
    }
    return x;
  }

  // RESID mid: g = G(X) sample; r = Theta o (Y - g)
  CSSAR_DEV static float2 mid(const AzArgs& a, float2 x, const Aux& ax, float& acc) {
    const float2 g = x * a.scale;
    const float2 r = ax.m ? (ax.v - g) : make_float2(0.f, 0.f);
    acc = fmaf(r.x, r.x, fmaf(r.y, r.y, acc));
    return r;
  }

  CSSAR_DEV static void epi(const AzArgs& a, size_t idx, float2 x, const Aux& ax, TailCtx& tc) {
    float2 v = x * a.scale;
    if constexpr (MODE == AZ_INV_MASK) {
      if (!ax.m) v = make_float2(0.f, 0.f);
    }
    if constexpr (MODE == AZ_TAIL) {
      const float2 xk = threshold(ax.v, tc.s2bits, tc.sigma, a.thr);     // X_i recomputed
      const float2 bn = make_float2(fmaf(a.mu, v.x, xk.x), fmaf(a.mu, v.y, xk.y));
      a.b[idx] = bn;
      const uint32_t u = mag2_bits(bn);
      const int bin = (int)(u >> HIST_SHIFT);
      if (a.rule == RULE_K) {
        if (bin >= tc.floor_bin) atomicAdd(&tc.shist[bin], 1u);
        if (bin >= tc.cand_lo && bin <= tc.cand_hi) {
          const uint32_t pos = atomicAdd(&tc.scount[0], 1u);
          if (pos < 1024u) {
            tc.scand[pos] = u;
          } else {
            const uint32_t g = atomicAdd(&a.st->cand_count, 1u);
            if (g < a.cand_cap) a.cand[g] = u; else a.st->cand_overflow = 1u;
          }
        }
        if (bin >= (0x7F800000u >> HIST_SHIFT)) a.st->nonfinite = 1u;
      } else {
        if (u > tc.s2fixed) atomicAdd(&tc.scount[1], 1u);
        if (u >= 0x7F800000u) a.st->nonfinite = 1u;
      }
    } else {
      a.out[idx] = v;
    }
  }
};

template <int LOGN, int MODE>
__global__ void __launch_bounds__(AzShape<LOGN, MODE == AZ_RESID>::T,
                                  (MODE == AZ_RESID && AzShape<LOGN, true>::MINB > 2) ? 2 : AzShape<LOGN, MODE == AZ_RESID>::MINB)
    az_kernel(const AzArgs a) {
  using Cf = AzShape<LOGN, MODE == AZ_RESID>;
  constexpr int C = Cf::C, W = Cf::W, M = Cf::M, T = Cf::T, E = Cf::E;
  constexpr int N = M * C;
  using En = typename Cf::En;
  using Ops = AzOps<MODE>;
  constexpr int R0 = 1 << En::template lr<false>(0);
  constexpr int RL = 1 << En::template lr<false>(En::P - 1);

  extern __shared__ float4 smem4[];
  float2* tw = reinterpret_cast<float2*>(smem4);      // inter-pass twiddle tables
  float2* s = tw + Cf::TW;                             // panel data
  copy_table_async(tw, a.tw, Cf::TW, threadIdx.x, Cf::T);   // waited for before the first exchange
  int rank = 0;
  if constexpr (C > 1) rank = (int)cg::this_cluster().block_rank();
  const int col0 = (blockIdx.x / C) * W;
  const int n_rg = a.n_rg;
  const int t = threadIdx.x;

  TailCtx tc{};
  if constexpr (MODE == AZ_TAIL) {
    tc.shist = reinterpret_cast<uint32_t*>(s + M * W);
    tc.scand = tc.shist + HIST_BINS;
    tc.scount = tc.scand + Cf::CAND_SMEM;
    for (int i = t; i < HIST_BINS; i += T) tc.shist[i] = 0u;
    if (t < 4) tc.scount[t] = 0u;
    tc.floor_bin = a.st->floor_bin;
    tc.cand_lo = a.st->cand_lo;
    tc.cand_hi = a.st->cand_hi;
    tc.s2bits = a.st->sigma2_bits;
    tc.s2fixed = a.st->sigma2_fixed_bits;
    tc.sigma = a.st->sigma;
    // (the first FFT exchange's __syncthreads orders these writes before any use)
  }
  float racc = 0.f;

  uint32_t s2 = 0u;
  float sig = 0.f;
  if constexpr (MODE == AZ_FWD_THR) {
    s2 = a.st->sigma2_bits;
    sig = a.st->sigma;
  }
  // DIT-first input rows: local index m -> global row rank + C m; all loads of a group are
  // issued before the prologue arithmetic
  auto ld = [&](int w, int j, float2* x) {
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int row = rank + C * (j + r * (M / R0));
      x[r] = a.in[(size_t)row * n_rg + col0 + w];
    }
#pragma unroll
    for (int r = 0; r < R0; ++r) x[r] = Ops::pro(a, rank + C * (j + r * (M / R0)), col0 + w, x[r], s2, sig);
  };

  if constexpr (C == 1) {
    if constexpr (MODE == AZ_RESID) {
      auto mid = [&](int w, int j, float2* x) {
        Aux ax[RL];
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int row = j + r * (M / RL);
          ax[r] = Ops::fetch(a, row, col0 + w, (size_t)row * n_rg + col0 + w);
        }
#pragma unroll
        for (int r = 0; r < RL; ++r) x[r] = Ops::mid(a, x[r], ax[r], racc);
      };
      auto st = [&](int w, int j, float2* x) {
#pragma unroll
        for (int r = 0; r < R0; ++r) {
          const int row = j + r * (M / R0);
          a.out[(size_t)row * n_rg + col0 + w] = x[r] * a.scale;
        }
      };
      En::template conv<+1>(s, ld, mid, st, tw);
    } else {
      auto st = [&](int w, int j, float2* x) {
        Aux ax[RL];
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int row = j + r * (M / RL);
          ax[r] = Ops::fetch(a, row, col0 + w, (size_t)row * n_rg + col0 + w);
        }
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int row = j + r * (M / RL);
          Ops::epi(a, (size_t)row * n_rg + col0 + w, x[r], ax[r], tc);
        }
      };
      En::template run<Ops::DIR>(s, ld, st, tw);
    }
  } else {
    auto cluster = cg::this_cluster();
    float2 v[E];
    En::template run_keep<Ops::DIR>(s, v, ld, tw);
    En::store_natural(s, v);
    cluster.sync();
    // gather: this rank owns local output indices k in [rank M/C, (rank+1) M/C)
    constexpr int PT = E / C > 0 ? E / C : 1;       // (k, w) pairs per thread
    static_assert((M / C) * W == PT * T, "cluster gather shape");
    float2 z[PT][C];
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      const int pr = p * T + t;
      const int w = pr % W, k = rank * (M / C) + pr / W;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float2* rs = cluster.map_shared_rank(s, c);
        z[p][c] = rs[k * W + w];
      }
    }
    if constexpr (MODE != AZ_RESID) cluster.barrier_arrive();    // done reading remote SMEM
    // auxiliary inputs of the elements this thread finalises (rows k + M q)
    Aux ax[PT][C];
    if constexpr (MODE == AZ_RESID || MODE == AZ_TAIL || MODE == AZ_INV_MASK) {
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int pr = p * T + t;
        const int w = pr % W, k = rank * (M / C) + pr / W;
#pragma unroll
        for (int q = 0; q < C; ++q) {
          const int row = k + M * q;
          ax[p][q] = Ops::fetch(a, row, col0 + w, (size_t)row * n_rg + col0 + w);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      const int pr = p * T + t;
      const int k = rank * (M / C) + pr / W;
      apply_twiddles<C, Ops::DIR>(z[p], (uint32_t)k, (uint32_t)N);   // w_N^{c k}
      dft<C, Ops::DIR>(z[p]);                         // z[q] = X[k + M q]
    }
    if constexpr (MODE == AZ_RESID) {
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int pr = p * T + t;
        const int k = rank * (M / C) + pr / W;
#pragma unroll
        for (int q = 0; q < C; ++q) z[p][q] = Ops::mid(a, z[p][q], ax[p][q], racc);
        // forward DIF first stage: y_q = (sum_q' x_q' w_C^{q q'}) w_N^{q k}
        dft<C, -1>(z[p]);
        apply_twiddles<C, -1>(z[p], (uint32_t)k, (uint32_t)N);       // w_N^{-q k}
      }
      // scatter into the second SMEM buffer of CTA q (no barrier needed against the gathers,
      // which read the first buffer)
      float2* s2 = s + M * W;
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int pr = p * T + t;
        const int w = pr % W, k = rank * (M / C) + pr / W;
#pragma unroll
        for (int q = 0; q < C; ++q) {
          float2* rs = cluster.map_shared_rank(s2, q);
          rs[k * W + w] = z[p][q];
        }
      }
      cluster.sync();
      s = s2;
      // local forward FFT of y_rank: X[C m + rank] -> row rank + C m
      auto st = [&](int w, int j, float2* x) {
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int row = rank + C * (j + r * (M / RL));
          a.out[(size_t)row * n_rg + col0 + w] = x[r] * a.scale;
        }
      };
      En::template run_from_smem<-1>(s, st, tw);
    } else {
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int pr = p * T + t;
        const int w = pr % W, k = rank * (M / C) + pr / W;
#pragma unroll
        for (int q = 0; q < C; ++q) {
          const int row = k + M * q;
          Ops::epi(a, (size_t)row * n_rg + col0 + w, z[p][q], ax[p][q], tc);
        }
      }
      cluster.barrier_wait();                          // keep SMEM alive for remote readers
    }
  }

  if constexpr (MODE == AZ_RESID) {
    // block reduce ||r||^2 -> one double atomic per CTA
    __shared__ float red[32];
    float v = racc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((t & 31) == 0) red[t >> 5] = v;
    __syncthreads();
    if (t < 32) {
      float u = (t < T / 32) ? red[t] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
      if (t == 0) atomicAdd(&a.st->resid2, (double)u);
    }
  }
  if constexpr (MODE == AZ_TAIL) {
    __syncthreads();
    if (a.rule == RULE_K) {
      for (int i = t; i < HIST_BINS; i += T) {
        const uint32_t c = tc.shist[i];
        if (c) atomicAdd(&a.hist[i], c);
      }
      const uint32_t nc = min(tc.scount[0], (uint32_t)Cf::CAND_SMEM);
      __shared__ uint32_t base;
      if (t == 0) base = nc ? atomicAdd(&a.st->cand_count, nc) : 0u;
      __syncthreads();
      for (uint32_t i = t; i < nc; i += T) {
        const uint32_t g = base + i;
        if (g < a.cand_cap) a.cand[g] = tc.scand[i]; else a.st->cand_overflow = 1u;
      }
    } else if (t == 0 && tc.scount[1]) {
      atomicAdd(&a.st->support_fixed, (unsigned long long)tc.scount[1]);
    }
  }
}

template <int LOGN, int MODE>
static cudaError_t az_launch(int n_rg, const AzArgs& a, cudaStream_t s) {
  using Cf = AzShape<LOGN, MODE == AZ_RESID>;
  auto k = az_kernel<LOGN, MODE>;
  const size_t smem = (MODE == AZ_TAIL) ? Cf::SMEM_TAIL : (MODE == AZ_RESID) ? Cf::SMEM_RESID : Cf::SMEM_FFT;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (Cf::C > 8) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((n_rg / Cf::W) * Cf::C));
  cfg.blockDim = dim3(Cf::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Cf::C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, k, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int LOGN, bool R>
__global__ void az_table_kernel(float2* dst) {
  AzShape<LOGN, R>::En::build_tw(dst, threadIdx.x, blockDim.x);
}

template <int LOGN>
size_t az_table_count_t(bool resid) { return resid ? (size_t)AzShape<LOGN, true>::TW : (size_t)AzShape<LOGN, false>::TW; }

template <int LOGN>
cudaError_t az_table_fill_t(bool resid, float2* dst, cudaStream_t s) {
  if (resid) az_table_kernel<LOGN, true><<<1, 256, 0, s>>>(dst);
  else az_table_kernel<LOGN, false><<<1, 256, 0, s>>>(dst);
  return cudaGetLastError();
}

template <int LOGN>
cudaError_t az_dispatch_mode(int mode, int n_rg, const AzArgs& a, cudaStream_t s) {
  switch (mode) {
    case AZ_FWD_PLAIN: return az_launch<LOGN, AZ_FWD_PLAIN>(n_rg, a, s);
    case AZ_FWD_MASK: return az_launch<LOGN, AZ_FWD_MASK>(n_rg, a, s);
    case AZ_FWD_THR: return az_launch<LOGN, AZ_FWD_THR>(n_rg, a, s);
    case AZ_INV_PLAIN: return az_launch<LOGN, AZ_INV_PLAIN>(n_rg, a, s);
    case AZ_INV_MASK: return az_launch<LOGN, AZ_INV_MASK>(n_rg, a, s);
    case AZ_RESID: return az_launch<LOGN, AZ_RESID>(n_rg, a, s);
    case AZ_TAIL: return az_launch<LOGN, AZ_TAIL>(n_rg, a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cssar
