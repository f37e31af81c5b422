// Azimuth sweeps (S1 head, S3 residual, S5 tail, operator heads/tails): column panels,
// thread-block clusters + DSMEM for long columns.  Instantiated per log2(n_az) in az_*.cu.
#pragma once
#include <cuda.h>
#include <cstdlib>
#include <mutex>
#include "device_ops.cuh"
#include "cluster.cuh"

namespace cssar {

// ------------------------------------------------------------------ azimuth sweeps
// R = configuration for the residual kernel (two transforms; more registers)
template <int LOGN, bool R>
struct AzCfg {
  // column panel of W range bins, split over a cluster of C CTAs (M = N/C rows each);
  // C > 1: persistent cluster kernel with NS TMA stages of M*W complex64 per CTA
  // (measured on c3: head/tail C = 8, W = 4, one stage -> 64 KB SMEM, 2 CTAs/SM, 33 clusters;
  // residual C = 16, W = 8, one stage that also takes the scatter (XS) + receive buffer,
  // 73 KB, 14 clusters)
  static constexpr int C = LOGN <= 10 ? 1 : LOGN == 11 ? 2 : LOGN == 12 ? 4 : LOGN == 13 ? (R ? 16 : 8) : 16;
  static constexpr int W = LOGN <= 8 ? 16 : LOGN == 9 ? 8 : LOGN == 10 ? 4 : LOGN == 13 ? (R ? 8 : 4)
                         : LOGN <= 14 ? 8 : 4;
  static constexpr int E = 16;
  static constexpr int NS = 1;
  static constexpr bool XS = true;           // RESID: scatter into the (one) stage buffer
};
#if defined(CSSAR_AZ13_C)
template <>
struct AzCfg<13, false> {
  static constexpr int C = CSSAR_AZ13_C, W = CSSAR_AZ13_W, E = CSSAR_AZ13_E, NS = CSSAR_AZ13_NS;
  static constexpr bool XS = false;
};
#endif
#if defined(CSSAR_AZ12_C)
template <>
struct AzCfg<12, false> {
  static constexpr int C = CSSAR_AZ12_C, W = CSSAR_AZ12_W, E = CSSAR_AZ12_E, NS = 1;
  static constexpr bool XS = false;
};
template <>
struct AzCfg<12, true> {
  static constexpr int C = CSSAR_AZ12_C, W = CSSAR_AZ12_W, E = CSSAR_AZ12_E, NS = 1;
  static constexpr bool XS = true;
};
#endif
#if defined(CSSAR_AZ15_C)
template <>
struct AzCfg<15, false> {
  static constexpr int C = CSSAR_AZ15_C, W = CSSAR_AZ15_W, E = CSSAR_AZ15_E, NS = 1;
  static constexpr bool XS = false;
};
#endif
#if defined(CSSAR_AZ15R_C)
template <>
struct AzCfg<15, true> {
  static constexpr int C = CSSAR_AZ15R_C, W = CSSAR_AZ15R_W, E = CSSAR_AZ15R_E, NS = 1;
  static constexpr bool XS = true;
};
#endif
#if defined(CSSAR_AZ13R_C)
template <>
struct AzCfg<13, true> {
  static constexpr int C = CSSAR_AZ13R_C, W = CSSAR_AZ13R_W, E = CSSAR_AZ13R_E, NS = CSSAR_AZ13R_NS;
  static constexpr bool XS = CSSAR_AZ13R_XS;
};
#endif

constexpr int kSlCap = 512;      // sparse-state tail: list entries staged in SMEM per panel

template <int LOGN, bool R = false, int NSO = 0, bool TAILM = true, bool DEF = false, bool SSB = false>
struct AzShape {
  using P = AzCfg<LOGN, R>;
  static constexpr int C = P::C, W = P::W, E = P::E, NS = NSO > 0 ? NSO : P::NS;
  // RESID with XS: the scatter lands in the stage buffer itself (one stage, refilled after
  // the panel's last transform) -> no separate scatter buffer, 2 CTAs/SM fit
  static constexpr bool XS = R && P::XS && NS == 1;
  static constexpr int LOGM = LOGN - ilog2c(C);
  static constexpr int M = 1 << LOGM;
  static constexpr int T = M * W / E;
  static constexpr int MINB = T <= 128 ? 4 : T <= 256 ? (E == 32 ? 2 : 3) : (E == 32 ? 1 : 2);
  using En = Engine<LOGM, W, T, true, E>;
  static constexpr int TW = En::TW_TOTAL;
  static constexpr int TWK = R ? En::TW_TOTAL : En::TW_FWD;      // SMEM tables of the cluster kernel
  static constexpr int CAND_SMEM = 1024;
  // C == 1 (az_kernel): [twiddles | panel | (TAIL) hist, candidates, counters]
  static constexpr size_t SMEM_FFT = sizeof(float2) * (M * W + TW);
  static constexpr size_t SMEM_TAIL = SMEM_FFT + sizeof(uint32_t) * (HIST_BINS + CAND_SMEM + 4);
  static constexpr size_t SMEM_RESID = SMEM_FFT;
  // C > 1 (az_cluster_kernel): [NS stages | receive buffer | (RESID) scatter buffer | twiddles | mbarriers |
  // (TAIL) hist, candidates, counters], 1024-byte aligned stages
  static constexpr int BM = M < 256 ? M : 256;             // TMA box rows (box dims <= 256)
  static constexpr uint32_t STAGE_BYTES = (uint32_t)(sizeof(float2) * M * W);
  // RESID: + a TMA-loaded buffer of Y at the output rows k + M q ([q][k][w])
  // DEF (deferred epilogue): a second receive buffer, the panels' pushes alternate between them
  static constexpr size_t CL_Y_OFF = sizeof(float2) * (size_t)M * W * (NS + 1 + (R && !XS ? 1 : 0) + (DEF ? 1 : 0));
  static constexpr size_t CL_TW_OFF = CL_Y_OFF + (R ? sizeof(float2) * (size_t)M * W : 0);
  static constexpr int LO = (LOGN + 1) / 2;                      // cluster twiddle table split
  static constexpr int CTW = (1 << LO) + (1 << (LOGN - LO));      // lo[2^LO] | hi[N / 2^LO]
  static constexpr size_t CL_CTW_OFF = CL_TW_OFF + ((sizeof(float2) * TWK + 15) / 16) * 16;
  static constexpr size_t CL_BAR_OFF = CL_CTW_OFF + sizeof(float2) * CTW;
  static constexpr size_t CL_MISC_OFF = CL_BAR_OFF + 8 * NS + 24 + 8;
  // sparse-state tail: SMEM staging of the new list entries of a panel (flushed per panel)
  static constexpr int SL_CAP = kSlCap;
  static constexpr size_t CL_SL_OFF =
      ((CL_MISC_OFF + sizeof(uint32_t) * (64 + (TAILM ? HIST_BINS + CAND_SMEM + 4 : 0)) + 15) / 16) * 16;
  static constexpr size_t CL_SMEM = 1024 + CL_SL_OFF + (SSB ? sizeof(SsEntry) * SL_CAP : 0);
  static constexpr int CL_MINB = T <= 128 ? 3 : T <= 256 ? 2 : 1;
};

struct TailCtx {
  uint32_t* shist;
  uint32_t* scand;
  uint32_t* scount;      // [0] = candidates in SMEM, [1] = fixed-lambda survivors, [2] = list entries in SMEM
  int floor_bin, cand_lo, cand_hi;
  uint32_t s2bits, s2fixed;
  float sigma;
  // sparse-state tail: new list entries (|b|^2 >= list_floor) of the current panel
  SsEntry* sl_buf;
  SsEntry* went;         // write list entries (panel-major) and counters
  uint32_t* wcnt;
  uint32_t list_floor;
  uint32_t capp;
  int panel, col0;
};

// one new list entry of the sparse-state tail: staged in SMEM, overflow straight to the list
template <int SL_CAP>
CSSAR_DEV void ss_push(TailCtx& tc, int row, int col, float2 v) {
  SsEntry e;
  e.row = (uint32_t)row;
  e.w = (uint32_t)(col - tc.col0);
  e.v = v;
  const uint32_t pos = atomicAdd(&tc.scount[2], 1u);
  if (pos < (uint32_t)SL_CAP) {
    tc.sl_buf[pos] = e;
  } else {
    const uint32_t g = atomicAdd(&tc.wcnt[tc.panel], 1u);
    tc.went[(size_t)tc.panel * tc.capp + g] = e;
  }
}

// auxiliary per-element inputs, fetched for a whole group before any arithmetic so the
// loads are in flight together (long-scoreboard latency overlaps)
struct Aux {
  float2 v;        // Y (RESID) or b_{i-1} (TAIL)
  uint32_t m;      // mask word of the element (mask_at(m, col) is its bit)
};

// destination of output line `row`, column `col` (plain array or a rank's blocked row slab)
// FAST: a uniform single-destination shortcut (world 1).  Not in the residual sweep, which is
// at the 128-register bound: the second path spilled there (S3 0.757 -> 0.785 ms measured).
template <bool FAST = true>
CSSAR_DEV float2* out_at(const AzArgs& a, int row, int col) {
  if (FAST && a.dsingle) return a.dst[0] + (size_t)row * (size_t)a.n_rg + col;
  const int m = (1 << a.dlog_nrow) - 1;
  return a.dst[row >> a.dlog_nrow] + ((size_t)((a.drank << a.dlog_nrow) + (row & m))) * (size_t)a.n_rg + col;
}

// Deterministic squared-norm commit (called by every thread of the CTA after the block
// reduction; `u` valid in thread 0): the CTA's partial goes to slot blockIdx.x, the last CTA to
// arrive (ticket) sums the slots in block order -- lane l adds slots l, l+32, ... in order, then
// a fixed xor-shuffle tree -- and adds the sum to *target (zeroed by the previous select).
// Run-to-run bitwise reproducible, unlike one floating-point atomicAdd per CTA.
CSSAR_DEV void red_commit(double* part, uint32_t* ticket, double* target, float u, uint32_t* sflag) {
  if (threadIdx.x == 0) {
    part[blockIdx.x] = (double)u;
    __threadfence();
    *sflag = atomicAdd(ticket, 1u) == gridDim.x - 1 ? 1u : 0u;
  }
  __syncthreads();
  if (*sflag && threadIdx.x < 32) {
    __threadfence();
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += 32) s += reinterpret_cast<volatile double*>(part)[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) {
      *target += s;
      *ticket = 0u;
    }
  }
}

// candidate straight to the global list (the tail's SMEM buffer is full)
static __device__ __noinline__ void cand_spill(SelState* st, uint32_t* cand, uint32_t cap, uint32_t* hist, uint32_t u) {
  const uint32_t g = atomicAdd(&st->cand_count, 1u);
  if (g < cap) cand[g] = u; else { st->cand_overflow = 1u; hist[HIST_BINS] = 1u; }
}
static __device__ __noinline__ void flag_nonfinite(SelState* st, uint32_t* hist) {
  st->nonfinite = 1u;
  hist[HIST_BINS + 1] = 1u;
}

template <int MODE>
struct AzOps {
  static constexpr int DIR = (MODE <= AZ_FWD_THR || MODE == AZ_FWD_SS) ? -1 : +1;   // first transform direction
  // kernels that reduce a squared norm into the solver state
  static constexpr bool RED = az_is_res(MODE) || MODE == AZ_NORM;
  CSSAR_DEV static double* red_target(const AzArgs& a) {
    return MODE == AZ_RESID ? &a.st->resid2 : MODE == AZ_GRAD ? &a.st->mu_num : &a.st->mu_den;
  }
  static constexpr int RED_SLOT = MODE == AZ_RESID ? 0 : MODE == AZ_GRAD ? 1 : 2;
  CSSAR_DEV static void red_commit_mode(const AzArgs& a, float u, uint32_t* sflag) {
    red_commit(a.red_part + RED_SLOT * kRedSlots, a.red_ticket + RED_SLOT, red_target(a), u, sflag);
  }

  // prologue on a loaded input value (loads are issued for a whole group first)
  CSSAR_DEV static float2 pro(const AzArgs& a, int row, int col, float2 v, uint32_t s2, float sig) {
    if constexpr (MODE == AZ_FWD_MASK) {
      if (!mask_bit(a.mask, a.mask_words, row, col)) v = make_float2(0.f, 0.f);
    }
    if constexpr (az_is_thr(MODE)) v = threshold(v, s2, sig, a.thr);
    return v;
  }

  CSSAR_DEV static Aux fetch(const AzArgs& a, int row, int col, size_t idx) {
    Aux x{make_float2(0.f, 0.f), 0xFFFFFFFFu};
    if constexpr (MODE == AZ_RESID) {
      x.m = mask_word(a.mask, a.mask_words, row, col);
      x.v = __ldg(a.Y + idx);
    } else if constexpr (MODE == AZ_INV_MASK || MODE == AZ_NORM) {
      x.m = mask_word(a.mask, a.mask_words, row, col);
    } else if constexpr (MODE == AZ_TAIL || MODE == AZ_GRAD || MODE == AZ_FUSE) {
      x.v = a.b[idx];
    }
    return x;
  }

  // two adjacent columns (col even): one 16-byte load of b, one mask word
  CSSAR_DEV static void fetch2(const AzArgs& a, int row, int col, size_t idx, Aux& x0, Aux& x1) {
    x0 = Aux{make_float2(0.f, 0.f), 0xFFFFFFFFu};
    x1 = x0;
    if constexpr (MODE == AZ_TAIL) {
      const float4 q = *reinterpret_cast<const float4*>(a.b + idx);
      x0.v = make_float2(q.x, q.y);
      x1.v = make_float2(q.z, q.w);
    } else if constexpr (MODE == AZ_INV_MASK || MODE == AZ_RESID || MODE == AZ_NORM) {
      const uint32_t wd = mask_word(a.mask, a.mask_words, row, col);
      x0.m = wd;
      x1.m = wd;
      if constexpr (MODE == AZ_RESID) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(a.Y + idx));
        x0.v = make_float2(q.x, q.y);
        x1.v = make_float2(q.z, q.w);
      }
    }
  }

  // RESID mid: g = G(X) sample; r = Theta o (Y - g).  GRAD mid (ax.v = b_{i-1}): dX = the
  // sample, kept in D; returns dX on supp(X_i) = {|b_{i-1}|^2 > sigma_{i-1}^2} (R20).
  // FUSE mid (ax.v = b_{i-1}): b_i = E(b_{i-1}; sigma_{i-1}) + mu dX stored; returns
  // X_{i+1} = E(b_i; sigma_fixed) (eq. 7: sigma = lambda mu is known before the select) and
  // counts its support in acc
  CSSAR_DEV static float2 mid(const AzArgs& a, float2 x, const Aux& ax, float& acc, int row, int col, uint32_t s2,
                              float sig = 0.f, uint32_t s2f = 0u, float sigf = 0.f) {
    if constexpr (MODE == AZ_FUSE) {
      const float2 dx = x * a.scale;
      const float2 xk = threshold(ax.v, s2, sig, a.thr);
      const float2 bn = make_float2(fmaf(a.mu, dx.x, xk.x), fmaf(a.mu, dx.y, xk.y));
      a.b[(size_t)row * a.n_rg + col] = bn;
      const uint32_t u = mag2_bits(bn);
      if (u > s2f) acc += 1.0f;
      if (u >= 0x7F800000u) a.st->nonfinite = 1u;
      return threshold(bn, s2f, sigf, a.thr);
    } else if constexpr (MODE == AZ_GRAD) {
      const float2 d = x * a.scale;
      a.D[(size_t)row * a.n_rg + col] = d;
      const float2 z = mag2_bits(ax.v) > s2 ? d : make_float2(0.f, 0.f);
      acc = fmaf(z.x, z.x, fmaf(z.y, z.y, acc));
      return z;
    } else {
      (void)row; (void)s2;
      const float2 g = x * a.scale;
      const float2 r = mask_at(ax.m, col) ? (ax.v - g) : make_float2(0.f, 0.f);
      acc = fmaf(r.x, r.x, fmaf(r.y, r.y, acc));
      return r;
    }
  }

  // two adjacent columns: per-element epilogue, one 16-byte store
  CSSAR_DEV static void epi2(const AzArgs& a, int row, int col, float2 x0, float2 x1, const Aux& a0, const Aux& a1,
                             TailCtx& tc, float& acc) {
    const size_t idx = (size_t)row * a.n_rg + col;
    const float sc = DIR < 0 ? a.oscale : a.scale;
    float2 v0 = x0 * sc, v1 = x1 * sc;
    if constexpr (MODE == AZ_INV_MASK || MODE == AZ_NORM) {
      if (!mask_at(a0.m, col)) v0 = make_float2(0.f, 0.f);
      if (!mask_at(a1.m, col + 1)) v1 = make_float2(0.f, 0.f);
    }
    if constexpr (MODE == AZ_NORM) {
      acc = fmaf(v0.x, v0.x, fmaf(v0.y, v0.y, acc));
      acc = fmaf(v1.x, v1.x, fmaf(v1.y, v1.y, acc));
    } else if constexpr (az_is_tail(MODE)) {
      const float2 k0 = threshold(a0.v, tc.s2bits, tc.sigma, a.thr), k1 = threshold(a1.v, tc.s2bits, tc.sigma, a.thr);
      v0 = make_float2(fmaf(a.mu, v0.x, k0.x), fmaf(a.mu, v0.y, k0.y));
      v1 = make_float2(fmaf(a.mu, v1.x, k1.x), fmaf(a.mu, v1.y, k1.y));
      if constexpr (MODE != AZ_TAIL_SS) *reinterpret_cast<float4*>(a.b + idx) = make_float4(v0.x, v0.y, v1.x, v1.y);
      if constexpr (MODE != AZ_TAIL_SSD) {
        tail_stats(a, v0, tc);
        tail_stats(a, v1, tc);
      }
      if constexpr (MODE == AZ_TAIL_SS) {
        if (mag2_bits(v0) >= tc.list_floor) ss_push<kSlCap>(tc, row, col, v0);
        if (mag2_bits(v1) >= tc.list_floor) ss_push<kSlCap>(tc, row, col + 1, v1);
      }
    } else {
      *reinterpret_cast<float4*>(out_at(a, row, col)) = make_float4(v0.x, v0.y, v1.x, v1.y);
    }
  }

  // histogram / candidates / support of one new b (TAIL); the rare paths (SMEM candidate
  // buffer full, non-finite value) are out of line to keep the unrolled epilogue small
  CSSAR_DEV static void tail_stats(const AzArgs& a, float2 bn, TailCtx& tc) {
    const uint32_t u = mag2_bits(bn);
    const int bin = (int)(u >> HIST_SHIFT);
    if (a.rule == RULE_K) {
      if (bin >= tc.floor_bin) atomicAdd(&tc.shist[bin], 1u);
      if (bin >= tc.cand_lo && bin <= tc.cand_hi) {
        const uint32_t pos = atomicAdd(&tc.scount[0], 1u);
        if (pos < 1024u) tc.scand[pos] = u;
        else cand_spill(a.st, a.cand, a.cand_cap, a.hist, u);
      }
      if (bin >= (0x7F800000u >> HIST_SHIFT)) flag_nonfinite(a.st, a.hist);
    } else {
      if (u > tc.s2fixed) atomicAdd(&tc.scount[1], 1u);
      if (u >= 0x7F800000u) flag_nonfinite(a.st, a.hist);
    }
  }

  CSSAR_DEV static void epi(const AzArgs& a, int row, int col, float2 x, const Aux& ax, TailCtx& tc, float& acc) {
    const size_t idx = (size_t)row * a.n_rg + col;
    float2 v = x * (DIR < 0 ? a.oscale : a.scale);        // forward outputs feed a range sweep
    if constexpr (MODE == AZ_INV_MASK || MODE == AZ_NORM) {
      if (!mask_at(ax.m, col)) v = make_float2(0.f, 0.f);
    }
    if constexpr (MODE == AZ_NORM) {
      acc = fmaf(v.x, v.x, fmaf(v.y, v.y, acc));
    } else if constexpr (az_is_tail(MODE)) {
      const float2 xk = threshold(ax.v, tc.s2bits, tc.sigma, a.thr);     // X_i recomputed
      const float2 bn = make_float2(fmaf(a.mu, v.x, xk.x), fmaf(a.mu, v.y, xk.y));
      if constexpr (MODE != AZ_TAIL_SS) a.b[idx] = bn;
      if constexpr (MODE != AZ_TAIL_SSD) tail_stats(a, bn, tc);
      if constexpr (MODE == AZ_TAIL_SS) {
        if (mag2_bits(bn) >= tc.list_floor) ss_push<kSlCap>(tc, row, col, bn);
      }
    } else {
      *out_at(a, row, col) = v;
    }
  }
};

template <int LOGN, int MODE>
__global__ void __launch_bounds__(AzShape<LOGN, az_is_res(MODE)>::T,
                                  ((az_is_res(MODE)) && AzShape<LOGN, true>::MINB > 2) ? 2 : AzShape<LOGN, az_is_res(MODE)>::MINB)
    az_kernel(const AzArgs a) {
  using Cf = AzShape<LOGN, az_is_res(MODE)>;
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
  uint32_t s2f = 0u;
  float sigf = 0.f;
  if constexpr (MODE == AZ_FWD_THR || MODE == AZ_GRAD || MODE == AZ_FUSE) {
    s2 = a.st->sigma2_bits;
    sig = a.st->sigma;
  }
  if constexpr (MODE == AZ_FUSE) {
    s2f = a.st->sigma2_fixed_bits;
    sigf = a.st->sigma_fixed;
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

  static_assert(C == 1, "cluster shapes use az_cluster_kernel");
  {
    if constexpr (az_is_res(MODE)) {
      auto mid = [&](int w, int j, float2* x) {
        Aux ax[RL];
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int row = j + r * (M / RL);
          ax[r] = Ops::fetch(a, row, col0 + w, (size_t)row * n_rg + col0 + w);
        }
#pragma unroll
        for (int r = 0; r < RL; ++r) x[r] = Ops::mid(a, x[r], ax[r], racc, j + r * (M / RL), col0 + w, s2, sig, s2f, sigf);
      };
      auto st = [&](int w, int j, float2* x) {
#pragma unroll
        for (int r = 0; r < R0; ++r) {
          const int row = j + r * (M / R0);
          *out_at(a, row, col0 + w) = x[r] * a.oscale;
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
          Ops::epi(a, row, col0 + w, x[r], ax[r], tc, racc);
        }
      };
      En::template run<Ops::DIR>(s, ld, st, tw);
    }
  }

  if constexpr (MODE == AZ_FUSE) {                 // support of X_{i+1} (integer-valued float counts)
    unsigned long long cnt = (unsigned long long)racc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&a.st->support_fixed, cnt);
  }
  if constexpr (Ops::RED) {
    // block reduce the squared norm -> one double atomic per CTA
    __shared__ float red[32];
    __shared__ uint32_t rflag;
    float v = racc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((t & 31) == 0) red[t >> 5] = v;
    __syncthreads();
    float u = 0.f;
    if (t < 32) {
      u = (t < T / 32) ? red[t] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
    }
    Ops::red_commit_mode(a, u, &rflag);
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
        if (g < a.cand_cap) a.cand[g] = tc.scand[i]; else { a.st->cand_overflow = 1u; a.hist[HIST_BINS] = 1u; }
      }
    } else if (t == 0 && tc.scount[1]) {
      atomicAdd(&a.st->support_fixed, (unsigned long long)tc.scount[1]);
    }
  }
  if (a.dst[1]) __threadfence_system();      // multi-GPU fused transpose: peer stores performed
}


// ------------------------------------------------------------------ persistent cluster kernel
// C > 1: a cluster of C CTAs owns whole columns.  CTA `rank` holds the M rows rank + C m of a
// panel of W adjacent range bins; TMA (3-D tensor map {col, rank, m}) streams each panel into
// one of NS SMEM stages while the previous panel is transformed.  Per panel:
//   local M-point FFT (DIT-first: rows rank + C m) in the stage buffer -> cluster barrier ->
//   DSMEM gather of the C partial transforms of output rows k + M q (k in this rank's M/C
//   block) -> twiddle w_N^{c k} + radix-C DFT -> epilogue -> (RESID: DIF radix-C + DSMEM
//   scatter into the peers' scatter buffers -> cluster barrier -> local FFT -> rows rank + C m).
// The stage is refilled (TMA, panel + NS clusters ahead) once every peer has finished reading
// it (split cluster barrier after the gather).  Epilogue inputs (Y, mask words, b) of a panel
// are loaded into registers before its FFT so their latency hides behind the transform.
// Cluster barriers without the release fence: a release arrive compiles to MEMBAR.ALL.GPU,
// which would wait for every outstanding epilogue store.  Ordering is provided instead by
// (a) __syncthreads() before the arrive (drains this CTA's STS into SMEM) for data the peers
// read after the barrier, and (b) consuming every DSMEM-loaded value before arriving "done
// reading"; DSMEM scatters complete on an mbarrier (st.async ... complete_tx).
CSSAR_DEV void cl_arrive() { asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory"); }
CSSAR_DEV void cl_wait() { asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory"); }
CSSAR_DEV void cl_arrive_rel() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
CSSAR_DEV void cl_sync() { cl_arrive(); cl_wait(); }

// Force every DSMEM-loaded value to have arrived before the next memory operation (an empty
// asm does not: no instruction would read the registers).  The values feed a compare that
// predicates a (never taken) SMEM store, which cannot move across the following asm volatile.
template <int PT, int C>
CSSAR_DEV void consume(const float2 (&z)[PT][C], uint32_t* sink) {
  float acc = 0.f;
#pragma unroll
  for (int p = 0; p < PT; ++p)
#pragma unroll
    for (int c = 0; c < C; ++c) acc += z[p][c].x + z[p][c].y;
  if (acc == 1.2345e-38f) *reinterpret_cast<volatile uint32_t*>(sink) = 0u;
}

CSSAR_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// x[c] *= w_N^{DIR c k}, c = 1..C-1, each power read directly from the two-level SMEM table
// lo[l] = w_N^l, hi[h] = w_N^{h 2^LO} (one product: at most ~1.5 ulp, no recurrences)
template <int C, int DIR, int LOGN, int LO>
CSSAR_DEV void cluster_twiddles(float2* x, uint32_t k, const float2* ctw) {
#if defined(CSSAR_EXP_NOFFT_AZ)
  return;
#endif
  constexpr uint32_t NM = (1u << LOGN) - 1u, LM = (1u << LO) - 1u;
#pragma unroll
  for (int c = 1; c < C; ++c) {
    const uint32_t m = ((uint32_t)c * k) & NM;
    const float2 w = cmul(ctw[m & LM], ctw[(1u << LO) + (m >> LO)]);
    x[c] = DIR < 0 ? cmul(x[c], w) : cmulc(x[c], w);
  }
}

template <int C, int DIR, int LOGN, int LO>
CSSAR_DEV void cluster_twiddles2(float2* x, float2* y, uint32_t k, const float2* ctw) {
#if defined(CSSAR_EXP_NOFFT_AZ)
  return;
#endif
  constexpr uint32_t NM = (1u << LOGN) - 1u, LM = (1u << LO) - 1u;
#pragma unroll
  for (int c = 1; c < C; ++c) {
    const uint32_t m = ((uint32_t)c * k) & NM;
    const float2 w = cmul(ctw[m & LM], ctw[(1u << LO) + (m >> LO)]);
    x[c] = DIR < 0 ? cmul(x[c], w) : cmulc(x[c], w);
    y[c] = DIR < 0 ? cmul(y[c], w) : cmulc(y[c], w);
  }
}

// the radix-C DFT across the cluster's partial transforms
template <int C, int DIR>
CSSAR_DEV void cl_dft(float2 (&z)[C]) {
#if !defined(CSSAR_EXP_NOFFT_AZ)
  dft_sr<C, DIR>(z);
#endif
}

// async DSMEM store that signals the destination CTA's mbarrier (same SMEM offset mapped)
#if defined(CSSAR_EXP_NOPUSH_AZ)
constexpr bool kNoPush = true;      // experiment: no DSMEM exchange (values dropped, no peer waits)
#else
constexpr bool kNoPush = false;
#endif
CSSAR_DEV void st_async_cluster(uint32_t raddr, float2 v, uint32_t rbar) {
  if (kNoPush) return;
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "f"(v.x), "f"(v.y), "r"(rbar)
               : "memory");
}

CSSAR_DEV void mbar_wait_cta(const uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// deferred epilogue (HEAD): panel p's cross-CTA step and stores run after panel p+1's push,
// so the wait for the slowest peer's push overlaps a whole local transform
#if defined(CSSAR_AZ_NO_DEFER)
template <int MODE>
constexpr bool kAzDefer = false;
#else
template <int MODE>
constexpr bool kAzDefer = az_is_thr(MODE);
#endif
template <int LOGN, int MODE>
using AzClShape = AzShape<LOGN, az_is_res(MODE), 0, az_is_tail(MODE), kAzDefer<MODE>,
                          MODE == AZ_TAIL_SS>;

template <int LOGN, int MODE>
__global__ void __launch_bounds__(AzClShape<LOGN, MODE>::T, AzClShape<LOGN, MODE>::CL_MINB)
    az_cluster_kernel(const AzArgs a, const __grid_constant__ CUtensorMap tm,
                      const __grid_constant__ CUtensorMap tmy) {
  using Cf = AzClShape<LOGN, MODE>;
  constexpr int C = Cf::C, W = Cf::W, M = Cf::M, T = Cf::T, E = Cf::E, NS = Cf::NS, BM = Cf::BM;
  constexpr int N = M * C;
  constexpr bool RES = az_is_res(MODE);   // two transforms, scatter
  // BS (TAIL, one stage): b_{i-1} of the output rows arrives by TMA into the stage buffer once the
  // local transform has read it; the next panel's stage load is issued after the epilogue
  constexpr bool BS = az_is_tail(MODE) && NS == 1;
  constexpr bool SSR = az_is_ss(MODE);      // input state from the list (no dense b)
  // PP (RESID/GRAD with XS, TAIL with BS): the stage and the receive buffer swap roles every
  // panel, so the next panel's TMA load goes into the receive buffer as soon as it is consumed
  // (mid-panel) instead of into the stage after the panel's last use of it; the cluster arrive
  // that lets peers push into a CTA's receive buffer moves to the end of the panel
#if defined(CSSAR_AZ_NO_PP)
  constexpr bool PP = false;
#else
  constexpr bool PP = (RES && Cf::XS) || BS;
#endif
  constexpr bool AUX = az_is_res(MODE) || (az_is_tail(MODE) && !BS) || MODE == AZ_INV_MASK ||
                      MODE == AZ_NORM;
  static_assert(C > 1, "cluster kernel");
  constexpr bool DEFER = kAzDefer<MODE> && !RES && !AUX && !BS && NS == 1;
  using En = typename Cf::En;
  using Ops = AzOps<MODE>;
  constexpr int R0 = 1 << En::template lr<false>(0);
  constexpr int RL = 1 << En::template lr<false>(En::P - 1);
  constexpr int PT = E / C > 0 ? E / C : 1;       // (k, w) pairs per thread in the gather
  static_assert((M / C) * W == PT * T, "cluster gather shape");

  extern __shared__ float4 smem4[];
  // 1024-byte aligned base by offsetting the __shared__ pointer itself (an integer round trip
  // would lose the shared address space and turn every SMEM access into a generic one)
  char* base = reinterpret_cast<char*>(smem4) + ((1024u - (smem_u32(smem4) & 1023u)) & 1023u);
  float2* stages = reinterpret_cast<float2*>(base);
  float2* const rbuf0 = stages + (size_t)NS * M * W;               // pushed partial transforms [c][k][w]
  float2* const xbuf0 = rbuf0 + (size_t)M * W;                      // RESID scatter target (!XS)
  float2* tw = reinterpret_cast<float2*>(base + Cf::CL_TW_OFF);
  float2* ctw = reinterpret_cast<float2*>(base + Cf::CL_CTW_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + Cf::CL_BAR_OFF);
  uint64_t* rfull = full + NS;                                     // pushes landed in rbuf
  uint64_t* xfull = full + NS + 1;                                 // RESID scatter landed in xbuf
  uint64_t* yfull = full + NS + 2;                                 // RESID Y buffer landed
  float2* ybuf = reinterpret_cast<float2*>(base + Cf::CL_Y_OFF);
  uint32_t* misc = reinterpret_cast<uint32_t*>(base + Cf::CL_MISC_OFF);   // [0..31] reduce, [32] base
  const int t = threadIdx.x;
  const int rank = (int)cluster_rank();
  // VEC: a thread's gather slots come in adjacent-column pairs (16-byte loads and stores,
  // one cluster twiddle set per pair); slot p -> (w, k)
  constexpr bool VEC = !RES && PT % 2 == 0 && W % 2 == 0;
  auto slot_w = [&](int p) -> int {
    if constexpr (VEC) return ((p / 2) * T + threadIdx.x) % (W / 2) * 2 + (p & 1);
    else return (p * T + threadIdx.x) % W;
  };
  auto slot_k = [&](int p) -> int {
    if constexpr (VEC) return rank * (M / C) + ((p / 2) * T + threadIdx.x) / (W / 2);
    else return rank * (M / C) + (p * T + threadIdx.x) / W;
  };
  const int cid = blockIdx.x / C, ncl = gridDim.x / C;
  const int n_rg = a.n_rg;
  const int npan = n_rg / W;

  copy_table_async(tw, a.tw, Cf::TWK + (Cf::TWK & 1), t, T);   // waited for in the first FFT pass
  for (int i = t; i < Cf::CTW; i += T) {         // exact (sincospif) cluster twiddle tables
    const uint32_t m = i < (1 << Cf::LO) ? (uint32_t)i : (uint32_t)(i - (1 << Cf::LO)) << Cf::LO;
    ctw[i] = expi_frac<-1>(m, (uint32_t)N);
  }
  pdl_wait();                                     // the previous kernel's output and state are complete
  if constexpr (MODE == AZ_TAIL_SSD) {
    if (!a.st->need_full) return;               // fallback re-run only (uniform over the grid)
  }
  // sparse-state lists: read the one the previous S5 (or the rebuild) wrote, write the other
  const int ss_rd = SSR ? ((a.st->iter + 1) & 1) : 0;
  const int ss_wr = SSR ? (a.st->iter & 1) : 0;
  TailCtx tc{};
  if constexpr (az_is_tail(MODE)) {
    tc.shist = misc + 64;
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
    if constexpr (MODE == AZ_TAIL_SS) {
      // entries that can exceed any sigma_i the window select can return (bins >= cand_lo)
      tc.sl_buf = reinterpret_cast<SsEntry*>(base + Cf::CL_SL_OFF);
      tc.went = a.ss.ent[ss_wr];
      tc.wcnt = a.ss.cnt[ss_wr];
      tc.capp = a.ss.capp;
      tc.list_floor = tc.cand_lo > 0 ? (uint32_t)tc.cand_lo << HIST_SHIFT : 0u;
    }
  }
  // sparse-state input: zero the SMEM block and scatter the panel's list entries into it.
  //   FWD_SS : the stage rows rank + C m   -> s[m W + w]
  //   TAIL_SS: the output rows k + M q (k in this rank's M/C block) -> s[(q M/C + k mod M/C) W + w]
  // Split so the list loads overlap other work: ss_zero_prefetch (block free: zero it, load the
  // first kSsPf entries per thread into registers) ... __syncthreads ... ss_scatter.
  constexpr int kSsPf = 4;
  SsEntry pf[kSsPf];
  uint32_t pf_n = 0;
  int pf_panel = 0;
  auto ss_place = [&](float2* dst, const SsEntry& x) {
    if constexpr (MODE == AZ_FWD_SS) {
      if ((int)(x.row % C) == rank) dst[(x.row / C) * W + x.w] = x.v;
    } else {
      const uint32_t q = x.row / M, k = x.row % M;
      if ((int)(k / (M / C)) == rank) dst[(q * (M / C) + k % (M / C)) * W + x.w] = x.v;
    }
  };
  auto ss_zero_prefetch = [&](int panel, float2* dst) {
    pf_panel = panel;
    pf_n = a.ss.cnt[ss_rd][panel];
    const SsEntry* e = a.ss.ent[ss_rd] + (size_t)panel * a.ss.capp;
#pragma unroll
    for (int j = 0; j < kSsPf; ++j)
      if ((uint32_t)(t + j * T) < pf_n) pf[j] = e[t + j * T];
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int i = t; i < M * W / 2; i += T) d4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto ss_scatter = [&](float2* dst) {          // after a __syncthreads that follows the zeroing
#pragma unroll
    for (int j = 0; j < kSsPf; ++j)
      if ((uint32_t)(t + j * T) < pf_n) ss_place(dst, pf[j]);
    const SsEntry* e = a.ss.ent[ss_rd] + (size_t)pf_panel * a.ss.capp;
    for (uint32_t i = t + kSsPf * T; i < pf_n; i += T) ss_place(dst, e[i]);
  };
  uint32_t s2 = 0u;
  float sig = 0.f;
  uint32_t s2f = 0u;
  float sigf = 0.f;
  if constexpr (az_is_thr(MODE) || MODE == AZ_GRAD || MODE == AZ_FUSE) {
    s2 = a.st->sigma2_bits;
    sig = a.st->sigma;
  }
  if constexpr (MODE == AZ_FUSE) {
    s2f = a.st->sigma2_fixed_bits;
    sigf = a.st->sigma_fixed;
  }
  float racc = 0.f;

  auto issue = [&](int panel, int sidx, float2* dst) {   // one thread: arm the stage barrier, M/BM boxes
    const uint32_t bar = smem_u32(&full[sidx]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(Cf::STAGE_BYTES)
                 : "memory");
#pragma unroll
    for (int bx = 0; bx < M / BM; ++bx) {
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
          ::"r"(smem_u32(dst + bx * BM * W)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(panel * W), "r"(rank),
          "r"(bx * BM), "r"(bar)
          : "memory");
    }
  };
  if (t == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1u);
    mbar_init(rfull, 1u);
    mbar_init(xfull, 1u);
    mbar_init(yfull, 1u);
    if (!kNoPush) mbar_expect_tx(rfull, Cf::STAGE_BYTES);        // armed for the first panel
    if ((RES || DEFER) && !kNoPush) mbar_expect_tx(xfull, Cf::STAGE_BYTES);   // DEFER: xfull = second receive buffer
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    if constexpr (MODE != AZ_FWD_SS) {
      for (int i = 0; i < NS; ++i)
        if (cid + i * ncl < npan) issue(cid + i * ncl, i, stages + (size_t)i * M * W);
    }
  }
  __syncthreads();
  // barrier initialisation visible cluster-wide before any remote st.async (once per kernel)
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");

  // DEFER: cross-CTA step, consume, arrive and stores of panel `pp` (its it index `pit`)
  auto defer_finish = [&](int pp, int pit) {
    if constexpr (DEFER) {
      float2* rb = rbuf0 + ((pit & 1) ? (size_t)M * W : 0);
      uint64_t* rbar = (pit & 1) ? xfull : rfull;
      if (!kNoPush) mbar_wait_cta(rbar, (uint32_t)((pit >> 1) & 1));
      if (t == 0 && !kNoPush) mbar_expect_tx(rbar, Cf::STAGE_BYTES);
      float2 z[PT][C];
#pragma unroll
      for (int p = 0; p < PT; p += 2) {
        const int off = (slot_k(p) - rank * (M / C)) * W + slot_w(p);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const float4 q = *reinterpret_cast<const float4*>(rb + c * (M / C) * W + off);
          z[p][c] = make_float2(q.x, q.y);
          z[p + 1][c] = make_float2(q.z, q.w);
        }
        cluster_twiddles2<C, Ops::DIR, LOGN, Cf::LO>(z[p], z[p + 1], (uint32_t)slot_k(p), ctw);
        cl_dft<C, Ops::DIR>(z[p]);
        cl_dft<C, Ops::DIR>(z[p + 1]);
      }
      consume(z, misc + 40);
      cl_arrive();                                 // this receive buffer consumed
      Aux ax0[C];
      const int c0 = pp * W;
#pragma unroll
      for (int p = 0; p < PT; p += 2) {
        const int w = slot_w(p), k = slot_k(p);
#pragma unroll
        for (int q = 0; q < C; ++q) Ops::epi2(a, k + M * q, c0 + w, z[p][q], z[p + 1][q], ax0[q], ax0[q], tc, racc);
      }
    }
  };
  int it = 0;
  if constexpr (MODE == AZ_FWD_SS) {
    if (cid < npan) ss_zero_prefetch(cid, stages);
  }
  for (int panel = cid; panel < npan; panel += ncl, ++it) {
    const int sidx = it % NS;
    float2* s = stages + (size_t)sidx * M * W;
    float2* rbuf = rbuf0;
    if constexpr (PP) {
      if (it & 1) { s = rbuf0; rbuf = stages; }
    }
    if constexpr (DEFER) {
      if (it & 1) rbuf = rbuf0 + (size_t)M * W;
    }
    const int col0 = panel * W;
    const int next = panel + NS * ncl;
    if constexpr (MODE == AZ_TAIL_SS) {
      tc.panel = panel;
      tc.col0 = col0;
    }
    // epilogue / residual inputs of output rows k + M q (in flight during the FFT)
    Aux ax[PT][C];
    if constexpr (AUX) {
      if constexpr (VEC) {
#pragma unroll
        for (int p = 0; p < PT; p += 2) {
          const int w = slot_w(p), k = slot_k(p);
#pragma unroll
          for (int q = 0; q < C; ++q) {
            const int row = k + M * q;
            Ops::fetch2(a, row, col0 + w, (size_t)row * n_rg + col0 + w, ax[p][q], ax[p + 1][q]);
          }
        }
      } else if constexpr (RES) {
        if (t == 0) {                              // Y of the output rows: C boxes {W, M/C} by TMA
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          mbar_expect_tx(yfull, Cf::STAGE_BYTES);
          constexpr int BY = (M / C) < 256 ? (M / C) : 256;   // TMA box rows (<= 256)
#pragma unroll 1
          for (int q = 0; q < C; ++q)
#pragma unroll 1
            for (int by = 0; by < (M / C) / BY; ++by)
              asm volatile(
                  "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, 0, %3}], [%4];\n"
                  ::"r"(smem_u32(ybuf + (q * (M / C) + by * BY) * W)), "l"(reinterpret_cast<uint64_t>(&tmy)),
                  "r"(col0), "r"(rank * (M / C) + M * q + by * BY), "r"(smem_u32(yfull))
                  : "memory");
        }
        if constexpr (MODE == AZ_RESID) {
#pragma unroll
          for (int p = 0; p < PT; ++p) {
            const int w = slot_w(p), k = slot_k(p);
#pragma unroll
            for (int q = 0; q < C; ++q) ax[p][q].m = mask_word(a.mask, a.mask_words, k + M * q, col0 + w);
          }
        }
      } else {
#pragma unroll
        for (int p = 0; p < PT; ++p) {
          const int w = slot_w(p), k = slot_k(p);
#pragma unroll
          for (int q = 0; q < C; ++q) {
            const int row = k + M * q;
            ax[p][q] = Ops::fetch(a, row, col0 + w, (size_t)row * n_rg + col0 + w);
          }
        }
      }
    }
    if constexpr (MODE == AZ_FWD_SS) {
      __syncthreads();                             // the stage zeroed (previous refill point)
      ss_scatter(s);                               // the stage from the state list (no TMA)
      __syncthreads();
    } else {
      mbar_wait_cta(&full[sidx], (uint32_t)((it / NS) & 1));
    }
    // local transform of rows rank + C m (stage layout [m][w] = engine BMINOR layout)
    auto ld = [&](int w, int j, float2* x) {
#pragma unroll
      for (int r = 0; r < R0; ++r) x[r] = s[(j + r * (M / R0)) * W + w];
#pragma unroll
      for (int r = 0; r < R0; ++r) x[r] = Ops::pro(a, rank + C * (j + r * (M / R0)), col0 + w, x[r], s2, sig);
    };
    float2 v[E];
    En::template run_keep<Ops::DIR>(s, v, ld, tw);
    float2* const xbuf = Cf::XS ? s : xbuf0;
    if constexpr (BS && SSR) {
      __syncthreads();                             // stage read: b_{i-1} of the output rows from the list
      ss_zero_prefetch(panel, s);                  // (scattered after the cross-CTA step)
    } else if constexpr (BS) {
      __syncthreads();                             // stage read: bring in b_{i-1} of the output rows
      if (t == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(yfull, Cf::STAGE_BYTES);
        constexpr int BY = (M / C) < 256 ? (M / C) : 256;
#pragma unroll 1
        for (int q = 0; q < C; ++q)
#pragma unroll 1
          for (int by = 0; by < (M / C) / BY; ++by)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, 0, %3}], [%4];\n"
                ::"r"(smem_u32(s + (q * (M / C) + by * BY) * W)), "l"(reinterpret_cast<uint64_t>(&tmy)),
                "r"(col0), "r"(rank * (M / C) + M * q + by * BY), "r"(smem_u32(yfull))
                : "memory");
      }
    } else if constexpr (!Cf::XS) {
      __syncthreads();                             // stage fully read: refill it NS panels ahead
      if constexpr (MODE == AZ_FWD_SS) {
        if (next < npan) ss_zero_prefetch(next, s);
      } else if (t == 0 && next < npan) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(next, sidx, s);
      }
    }
    // push local output k of every column to its owner rank k / (M/C): rbuf[(rank M/C + k%(M/C)) W + w]
    if (it > 0) cl_wait();                         // owners are done reading their receive buffers
    {
      const uint32_t rb = smem_u32(rbuf), bar = smem_u32((DEFER && (it & 1)) ? xfull : rfull);
      En::template for_groups<En::template lr<false>(En::P - 1)>(v, t, [&](int w, int j, float2* x) {
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int kk = j + r * (M / RL);
          const uint32_t own = (uint32_t)(kk / (M / C));
          const uint32_t off = (uint32_t)(((rank * (M / C) + kk % (M / C)) * W + w) * sizeof(float2));
          st_async_cluster(mapa(rb + off, own), x[r], mapa(bar, own));
        }
      });
    }
    if constexpr (DEFER) {
      if (it > 0) defer_finish(panel - ncl, it - 1);   // previous panel: pushes landed long ago
      else cl_arrive();                            // (the second receive buffer is free)
      continue;
    }
    if (!kNoPush) mbar_wait_cta(rfull, (uint32_t)(it & 1));      // all C partial transforms of our block landed
    if (t == 0 && !kNoPush) mbar_expect_tx(rfull, Cf::STAGE_BYTES);   // re-arm for the next panel
    float2 z[PT][C];
    if constexpr (VEC) {
#pragma unroll
      for (int p = 0; p < PT; p += 2) {
        const int off = (slot_k(p) - rank * (M / C)) * W + slot_w(p);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const float4 q = *reinterpret_cast<const float4*>(rbuf + c * (M / C) * W + off);
          z[p][c] = make_float2(q.x, q.y);
          z[p + 1][c] = make_float2(q.z, q.w);
        }
        cluster_twiddles2<C, Ops::DIR, LOGN, Cf::LO>(z[p], z[p + 1], (uint32_t)slot_k(p), ctw);
        cl_dft<C, Ops::DIR>(z[p]);
        cl_dft<C, Ops::DIR>(z[p + 1]);
      }
    } else {
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int pr = p * T + t;
#pragma unroll
        for (int c = 0; c < C; ++c) z[p][c] = rbuf[c * (M / C) * W + pr];
      }
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int k = slot_k(p);
        cluster_twiddles<C, Ops::DIR, LOGN, Cf::LO>(z[p], (uint32_t)k, ctw);   // w_N^{c k}
        cl_dft<C, Ops::DIR>(z[p]);                                       // z[q] = X[k + M q]
      }
    }
    consume(z, misc + 40);
    if constexpr (!(PP && BS)) cl_arrive();        // rbuf (and, RESID, last panel's xbuf) consumed
    if constexpr (PP) {
      __syncthreads();                             // every thread done with the receive buffer:
      if (t == 0 && next < npan) {                 // it becomes the next panel's stage
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(next, sidx, rbuf);
      }
    }
    if constexpr (BS && SSR) {                     // b_{i-1} of the output rows (zeroed at the
      if constexpr (!PP) __syncthreads();          //  local transform's end; synced above)
      ss_scatter(s);
      __syncthreads();
    }
    if constexpr (RES) {
#pragma unroll
      mbar_wait_cta(yfull, (uint32_t)(it & 1));
      for (int p = 0; p < PT; ++p) {
#pragma unroll
        for (int q = 0; q < C; ++q) {
          ax[p][q].v = ybuf[q * (M / C) * W + p * T + t];
          z[p][q] = Ops::mid(a, z[p][q], ax[p][q], racc, slot_k(p) + M * q, col0 + slot_w(p), s2, sig, s2f, sigf);
        }
        const int pr = p * T + t;
        const int k = rank * (M / C) + pr / W;
        cl_dft<C, -1>(z[p]);                                           // forward DIF first stage
        cluster_twiddles<C, -1, LOGN, Cf::LO>(z[p], (uint32_t)k, ctw);     // w_N^{-q k}
      }
      cl_wait();                                   // peers are done with their scatter buffers
      if constexpr (!PP) cl_arrive();              // (pairs with the next panel's push wait)
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int pr = p * T + t;
        const int w = pr % W, k = rank * (M / C) + pr / W;
        const uint32_t xo = smem_u32(xbuf + k * W + w), xb = smem_u32(xfull);
#pragma unroll
        for (int q = 0; q < C; ++q) st_async_cluster(mapa(xo, (uint32_t)q), z[p][q], mapa(xb, (uint32_t)q));
      }
      if (!kNoPush) mbar_wait_cta(xfull, (uint32_t)(it & 1));    // all C peers' scatters landed here
      if (t == 0 && !kNoPush) mbar_expect_tx(xfull, Cf::STAGE_BYTES);
      auto st = [&](int w, int j, float2* x) {
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int row = rank + C * (j + r * (M / RL));
          *out_at<false>(a, row, col0 + w) = x[r] * a.oscale;
        }
      };
      En::template run_from_smem<-1>(xbuf, st, tw);
      if constexpr (PP) {
        cl_arrive();                               // stage free: peers may push into it next panel
      } else if constexpr (Cf::XS) {
        __syncthreads();                           // last transform done with the stage
        if (t == 0 && next < npan) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          issue(next, sidx, s);
        }
      }
    } else if constexpr (VEC) {
      if constexpr (BS && !SSR) mbar_wait_cta(yfull, (uint32_t)(it & 1));
#pragma unroll
      for (int p = 0; p < PT; p += 2) {
        const int w = slot_w(p), k = slot_k(p);
#pragma unroll
        for (int q = 0; q < C; ++q) {
          const int row = k + M * q;
          if constexpr (BS) {
            const float4 bq = *reinterpret_cast<const float4*>(s + (q * (M / C) + k - rank * (M / C)) * W + w);
            ax[p][q].v = make_float2(bq.x, bq.y);
            ax[p + 1][q].v = make_float2(bq.z, bq.w);
          }
          Ops::epi2(a, row, col0 + w, z[p][q], z[p + 1][q], ax[p][q], ax[p + 1][q], tc, racc);
        }
      }
    } else {
      if constexpr (BS && !SSR) mbar_wait_cta(yfull, (uint32_t)(it & 1));
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int w = slot_w(p), k = slot_k(p);
#pragma unroll
        for (int q = 0; q < C; ++q) {
          const int row = k + M * q;
          if constexpr (BS) ax[p][q].v = s[(q * (M / C) + k - rank * (M / C)) * W + w];
          Ops::epi(a, row, col0 + w, z[p][q], ax[p][q], tc, racc);
        }
      }
    }
    if constexpr (MODE == AZ_TAIL || MODE == AZ_TAIL_SS) {
      // flush the SMEM candidates once the buffer is half full (and at the end of the kernel;
      // a burst beyond it spills straight to the global list) and, sparse state, the panel's
      // list entries (stored per panel)
      if (a.rule == RULE_K) {
        __syncthreads();
        const uint32_t c0 = tc.scount[0];
        const bool fc = c0 >= (uint32_t)Cf::CAND_SMEM / 2;       // uniform: read after the barrier
        if (fc || MODE == AZ_TAIL_SS) {
        const uint32_t nc = fc ? min(c0, (uint32_t)Cf::CAND_SMEM) : 0u;
        uint32_t nl = 0;
        if constexpr (MODE == AZ_TAIL_SS) nl = min(tc.scount[2], (uint32_t)kSlCap);
        if (t == 0) {
          misc[32] = nc ? atomicAdd(&a.st->cand_count, nc) : 0u;
          if constexpr (MODE == AZ_TAIL_SS) misc[34] = nl ? atomicAdd(&tc.wcnt[panel], nl) : 0u;
        }
        __syncthreads();
        const uint32_t b0 = misc[32];
        for (uint32_t i = t; i < nc; i += T) {
          const uint32_t g = b0 + i;
          if (g < a.cand_cap) a.cand[g] = tc.scand[i]; else { a.st->cand_overflow = 1u; a.hist[HIST_BINS] = 1u; }
        }
        if constexpr (MODE == AZ_TAIL_SS) {
          SsEntry* dst = tc.went + (size_t)panel * tc.capp + misc[34];
          for (uint32_t i = t; i < nl; i += T) dst[i] = tc.sl_buf[i];
        }
        __syncthreads();
        if (t == 0) {
          if (fc) tc.scount[0] = 0u;
          tc.scount[2] = 0u;
        }
        }
      }
    }
    if constexpr (PP && BS) {
      cl_arrive();                                 // stage (b) read: peers may push into it next panel
    } else if constexpr (BS) {
      __syncthreads();                             // every b of the panel read from the stage
      if (t == 0 && next < npan) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(next, sidx, s);
      }
    }
  }

  pdl_launch_dependents();                         // last panel done: the next kernel may start
  if (it > 0) cl_wait();                           // pairs with the last arrive
  if constexpr (DEFER) {
    if (it > 0) defer_finish(cid + (it - 1) * ncl, it - 1);   // the last panel (its arrive is unpaired:
    if (it > 0) cl_wait();                                     //  pair it before leaving)
  }
  if constexpr (MODE == AZ_FUSE) {                 // support of X_{i+1} (integer-valued float counts)
    unsigned long long cnt = (unsigned long long)racc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&a.st->support_fixed, cnt);
  }
  if constexpr (Ops::RED) {
    float v = racc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((t & 31) == 0) reinterpret_cast<float*>(misc)[t >> 5] = v;
    __syncthreads();
    float u = 0.f;
    if (t < 32) {
      u = (t < T / 32) ? reinterpret_cast<float*>(misc)[t] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
    }
    Ops::red_commit_mode(a, u, misc + 33);
  }
  if constexpr (MODE == AZ_TAIL || MODE == AZ_TAIL_SS) {
    __syncthreads();
    if (a.rule == RULE_K) {
      const uint32_t nc = min(tc.scount[0], (uint32_t)Cf::CAND_SMEM);   // candidates still in SMEM
      if (t == 0) misc[32] = nc ? atomicAdd(&a.st->cand_count, nc) : 0u;
      __syncthreads();
      for (uint32_t i = t; i < nc; i += T) {
        const uint32_t g = misc[32] + i;
        if (g < a.cand_cap) a.cand[g] = tc.scand[i]; else { a.st->cand_overflow = 1u; a.hist[HIST_BINS] = 1u; }
      }
      for (int i = t; i < HIST_BINS; i += T) {
        const uint32_t c = tc.shist[i];
        if (c) atomicAdd(&a.hist[i], c);
      }
    } else if (t == 0 && tc.scount[1]) {
      atomicAdd(&a.st->support_fixed, (unsigned long long)tc.scount[1]);
    }
  }
  if (a.dst[1]) __threadfence_system();      // multi-GPU fused transpose: peer stores performed
}

// 3-D tensor map {col, rank, m} over a row-major [N][n_rg] complex64 array: element
// (col, c, m) = row c + C m; box {W, 1, BM}
cudaError_t make_az_tensor_map(CUtensorMap* tm, const void* base, int n_rg, int N, int C, int W, int BM, int promo);
constexpr int kMaxDevices = 64;
std::mutex& az_setup_mutex();
int az_max_clusters(const void* kernel, int C, int T, size_t smem);
void az_log_config(int logn, int mode, int C, int W, int NS, int T, size_t smem, int clusters);

template <int LOGN, int MODE>
static cudaError_t az_cluster_launch(int n_rg, const AzArgs& a, cudaStream_t s) {
  using Cf = AzClShape<LOGN, MODE>;
  auto k = az_cluster_kernel<LOGN, MODE>;
  const size_t smem = Cf::CL_SMEM;
  // function attributes and the co-resident cluster count belong to a device context: cached
  // per device ordinal, set up under a lock (plans on several devices / threads)
  static int max_cl_dev[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  int max_cl = __atomic_load_n(&max_cl_dev[dev], __ATOMIC_ACQUIRE);
  if (max_cl == 0) {
    std::lock_guard<std::mutex> lock(az_setup_mutex());
    max_cl = max_cl_dev[dev];
    if (max_cl == 0) {
      e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      if (Cf::C > 8) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
      }
      max_cl = az_max_clusters((const void*)k, Cf::C, Cf::T, smem);
      if (max_cl <= 0) return cudaErrorInvalidConfiguration;
      az_log_config(LOGN, MODE, Cf::C, Cf::W, Cf::NS, Cf::T, smem, max_cl);
      __atomic_store_n(&max_cl_dev[dev], max_cl, __ATOMIC_RELEASE);
    }
  }
  CUtensorMap tm;
  // L2 promotion of the TMA panel loads (measured at c3, profiles/experiments_r02.md):
  //  * head sweep: 64 B (0.391 -> 0.381 ms);
  //  * residual sweep, U and Y: 64 B -- same time as 256 B, but DRAM reads 1.346 -> 1.086 GB per
  //    launch (the algorithmic 1.082 GB): with 256 B the 64-byte panel rows pulled in lines of
  //    neighbouring panels that were evicted before their cluster reached them;
  //  * tail sweep (U and b): the default 256 B (64 B on b: 0.566 -> 0.60 ms).
#if !defined(CSSAR_AZ_PROMO_HEAD)
#define CSSAR_AZ_PROMO_HEAD 1
#endif
#if !defined(CSSAR_AZ_PROMO_RESID)
#define CSSAR_AZ_PROMO_RESID 1
#endif
#if !defined(CSSAR_AZ_PROMO_TAIL)
#define CSSAR_AZ_PROMO_TAIL -1
#endif
#if !defined(CSSAR_AZ_PROMO_Y)
#define CSSAR_AZ_PROMO_Y 1
#endif
  e = make_az_tensor_map(&tm, a.in, n_rg, 1 << LOGN, Cf::C, Cf::W, Cf::BM,
                         MODE == AZ_FWD_THR ? CSSAR_AZ_PROMO_HEAD
                         : MODE == AZ_RESID ? CSSAR_AZ_PROMO_RESID
                         : az_is_tail(MODE) ? CSSAR_AZ_PROMO_TAIL : -1);
  if (e != cudaSuccess) return e;
  CUtensorMap tmy = tm;
  if constexpr (az_is_res(MODE) || (MODE == AZ_TAIL && Cf::NS == 1)) {   // Y (RESID) / b with
    // consecutive rows ({col, 0, row}), box {W, 1, min(M/C, 256)}
    e = make_az_tensor_map(&tmy, MODE == AZ_RESID ? (const void*)a.Y : (const void*)a.b, n_rg, 1 << LOGN, 1, Cf::W,
                           Cf::M / Cf::C < 256 ? Cf::M / Cf::C : 256,
                           MODE == AZ_RESID ? CSSAR_AZ_PROMO_Y : CSSAR_AZ_PROMO_TAIL);
    if (e != cudaSuccess) return e;
  }
  const int npan = n_rg / Cf::W;
  // cluster scheduling: load balancing (measured: 15 instead of 14 co-resident 16-CTA clusters
  // for the c3 residual sweep, 0.84 -> 0.78 ms); CSSAR_AZ_POLICY overrides (0 = driver default)
  static const int policy = [] { const char* e = std::getenv("CSSAR_AZ_POLICY"); return e ? std::atoi(e) : 2; }();
  const int ncl = npan < max_cl ? npan : max_cl;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncl * Cf::C));
  cfg.blockDim = dim3(Cf::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = Cf::C;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (policy) {
    attr[na].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[na].val.clusterSchedulingPolicyPreference = (cudaClusterSchedulingPolicy)policy;
    ++na;
  }
  if (pdl_enabled()) {                           // programmatic dependent launch (cluster.cuh)
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  e = cudaLaunchKernelEx(&cfg, k, a, tm, tmy);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int LOGN, int MODE>
static cudaError_t az_launch(int n_rg, const AzArgs& a_in, cudaStream_t s) {
  using Cf = AzShape<LOGN, az_is_res(MODE)>;
  AzArgs a = a_in;
  if (!a.dst[0]) {                       // plain output array (single rank / in-place paths)
    a.dst[0] = a.out;
    a.dlog_nrow = LOGN;
    a.drank = 0;
  }
  a.dsingle = (a.dlog_nrow == LOGN && a.drank == 0) ? 1 : 0;
  if constexpr (Cf::C > 1) {
    return az_cluster_launch<LOGN, MODE>(n_rg, a, s);
  } else {
  auto k = az_kernel<LOGN, MODE>;
  const size_t smem = (MODE == AZ_TAIL) ? Cf::SMEM_TAIL : (MODE == AZ_RESID) ? Cf::SMEM_RESID : Cf::SMEM_FFT;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (Cf::C > 8) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  if (AzOps<MODE>::RED && (n_rg / Cf::W) * Cf::C > kRedSlots) return cudaErrorInvalidConfiguration;
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
    case AZ_GRAD: return az_launch<LOGN, AZ_GRAD>(n_rg, a, s);
    case AZ_NORM: return az_launch<LOGN, AZ_NORM>(n_rg, a, s);
    case AZ_FUSE: return az_launch<LOGN, AZ_FUSE>(n_rg, a, s);
    case AZ_FWD_SS:
    case AZ_TAIL_SS:
    case AZ_TAIL_SSD:
      if constexpr (AzShape<LOGN, false>::C > 1) {
        return mode == AZ_FWD_SS ? az_launch<LOGN, AZ_FWD_SS>(n_rg, a, s)
             : mode == AZ_TAIL_SS ? az_launch<LOGN, AZ_TAIL_SS>(n_rg, a, s)
                                  : az_launch<LOGN, AZ_TAIL_SSD>(n_rg, a, s);
      } else {
        return cudaErrorInvalidValue;              // sparse state: cluster sweeps only (n_az >= 2048)
      }
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cssar
