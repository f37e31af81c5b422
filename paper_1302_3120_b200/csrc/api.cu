// libcssar C ABI (include/cssar.h): plan (S0 phase-coefficient table), operator calls and
// the graph-replayed ITA loop.  Host code only; device work lives in kernels.cu.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/cssar.h"
#include "kernels.cuh"

using namespace cssar;

namespace {

constexpr long double kC = 299792458.0L;
constexpr int kLogCap = 1 << 16;

struct GraphKey {
  const void* Y;
  const void* mask;
  void* X;
  int thr, rule;
  long long k;
  double lambda, mu;
  bool operator==(const GraphKey& o) const {
    return Y == o.Y && mask == o.mask && X == o.X && thr == o.thr && rule == o.rule && k == o.k &&
           lambda == o.lambda && mu == o.mu;
  }
};

}  // namespace

struct cssar_plan_s {
  cssar_sar_params p;
  int log_naz = 0, log_nrg = 0;
  long long n = 0;
  int sm_count = 148;
  RowCoef* d_coef = nullptr;
  float2* d_rg_tab = nullptr;     // phase exp table + range-engine twiddles
  float2* d_az_tab = nullptr;     // azimuth-engine twiddles (head / tail / operator kernels)
  float2* d_az_tab_r = nullptr;   // azimuth-engine twiddles (residual kernel)
  SelState* d_st = nullptr;
  uint32_t* d_hist = nullptr;
  uint32_t* d_hist_full = nullptr;
  IterLogDev* d_log = nullptr;
  // caller-bound workspace
  char* ws = nullptr;
  size_t ws_bytes = 0;
  float2* U = nullptr;
  uint32_t* cand = nullptr;
  uint32_t cand_cap = 0;
  // graph cache for the iteration body
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey{};
  bool ghave = false;
  // per-step profiling (CSSAR_FLAG_PROFILE_STAGES)
  cudaEvent_t ev[7] = {};
  double stage_ms[6] = {};
  int stage_iters = 0;
};

namespace {

int ilog2_exact(long long v) {
  if (v <= 0 || (v & (v - 1))) return -1;
  int l = 0;
  while ((1ll << l) < v) ++l;
  return l;
}

bool aligned16(const void* p) { return p && ((reinterpret_cast<uintptr_t>(p) & 15u) == 0); }

// round(frac(x) * 2^64) as a u64 fraction of a cycle (wraps 1.0 -> 0)
uint64_t frac_u64(long double x) {
  long double f = x - floorl(x);
  long double hi = floorl(ldexpl(f, 32));
  long double lo = ldexpl(ldexpl(f, 32) - hi, 32);
  unsigned long long h = (unsigned long long)hi;
  long double lr = roundl(lo);
  unsigned long long l;
  if (lr >= 4294967296.0L) { l = 0; h += 1; } else { l = (unsigned long long)lr; }
  return ((uint64_t)(h & 0xFFFFFFFFull) << 32) | (uint64_t)l;
}

// S0: per Doppler bin i the three CSA phase screens (oracle/csa.py reading,
// DESIGN.md R1/R3/R7/R9/R10) as quadratics in the column index, in cycles:
//   Phi1 = a (u/Fr + d)^2,               a = Km (1/D - 1)/2,  d = -(2 R_ref/c)(1/D - 1)
//   Phi2 = (D/(2 Km)) (Fr/N)^2 l'^2 + (2 R_ref/c)(1/D - 1)(Fr/N) l'
//   Phi3 = -(Km (1-D)/(2 Fr^2 D^2)) u^2 + (fc D/Fr) u + (2/c) fc D R_ref
// with u = j - N/2 (range gate), l' the signed range-frequency bin, evaluated in long
// double with 1 - D = x/(1 + D) and 1/D - 1 = (1 - D)/D to avoid cancellation.
std::vector<RowCoef> build_coefficients(const cssar_sar_params& p) {
  const long long na = p.n_az, nr = p.n_rg;
  std::vector<RowCoef> tab((size_t)na);
  const long double fc = p.fc, Kr = p.Kr, Fr = p.Fr, prf = p.prf, Vr = p.Vr, Rr = p.R_ref;
  for (long long i = 0; i < na; ++i) {
    const long long is = (i < (na + 1) / 2) ? i : i - na;   // fftfreq order (Nyquist negative)
    const long double f = (long double)is * prf / (long double)na;
    const long double xr = kC * f / (2.0L * Vr * fc);
    const long double x = xr * xr;
    const long double D = sqrtl(1.0L - x);
    const long double omD = x / (1.0L + D);
    const long double idm1 = omD / D;
    const long double Km = Kr / (1.0L - Kr * kC * Rr * f * f / (2.0L * Vr * Vr * fc * fc * fc * D * D * D));
    const long double a = Km * idm1 / 2.0L;
    const long double d = -(2.0L * Rr / kC) * idm1;
    const long double df = Fr / (long double)nr;
    RowCoef rc;
    rc.q[0] = {frac_u64(a / (Fr * Fr)), frac_u64(2.0L * a * d / Fr), frac_u64(a * d * d)};
    rc.q[1] = {frac_u64(D / (2.0L * Km) * df * df), frac_u64((2.0L * Rr / kC) * idm1 * df), 0ull};
    rc.q[2] = {frac_u64(-Km * omD / (2.0L * Fr * Fr * D * D)), frac_u64(fc * D / Fr),
               frac_u64((2.0L / kC) * fc * D * Rr)};
    tab[(size_t)i] = rc;
  }
  return tab;
}

int validate_params(const cssar_sar_params& p) {
  if (!(p.fc > 0 && p.Kr > 0 && p.Tr > 0 && p.Fr > 0 && p.prf > 0 && p.Vr > 0 && p.R_ref > 0))
    return CSSAR_ERR_INVALID_PARAMS;
  if (!std::isfinite(p.fc) || !std::isfinite(p.Kr) || !std::isfinite(p.Tr) || !std::isfinite(p.Fr) ||
      !std::isfinite(p.prf) || !std::isfinite(p.Vr) || !std::isfinite(p.R_ref))
    return CSSAR_ERR_INVALID_PARAMS;
  if (p.squint != 0.0) return CSSAR_ERR_INVALID_PARAMS;               // SPEC S:L77, R29
  if (p.Tr * p.Fr < 2.0) return CSSAR_ERR_INVALID_PARAMS;             // pulse shorter than 2 samples
  // Doppler band must stay inside the visible region (D real)
  const double fmax = p.prf / 2.0;
  if (299792458.0 * fmax / (2.0 * p.Vr * p.fc) >= 1.0) return CSSAR_ERR_INVALID_PARAMS;
  const int la = ilog2_exact(p.n_az), lr = ilog2_exact(p.n_rg);
  if (la < 7 || la > 15 || lr < 7 || lr > 14) return CSSAR_ERR_UNSUPPORTED_SIZE;
  return CSSAR_OK;
}

#define CUDA_TRY(x)                                   \
  do {                                                \
    cudaError_t _e = (x);                             \
    if (_e != cudaSuccess) {                          \
      std::fprintf(stderr, "libcssar: %s failed: %s\n", #x, cudaGetErrorString(_e)); \
      return CSSAR_ERR_CUDA;                          \
    }                                                 \
  } while (0)

int enqueue_forward(cssar_plan pl, const void* X, const uint32_t* mask, void* Yout, cudaStream_t s) {
  AzArgs a{};
  a.tw = pl->d_az_tab;
  a.n_rg = (int)pl->p.n_rg;
  a.mask_words = (int)(pl->p.n_rg / 32);
  a.scale = (float)(1.0 / std::sqrt((double)pl->p.n_az));
  a.oscale = (float)(1.0 / (std::sqrt((double)pl->p.n_az) * (double)pl->p.n_rg));
  a.in = (const float2*)X;
  a.out = (float2*)Yout;
  CUDA_TRY(launch_az(pl->log_naz, AZ_FWD_PLAIN, a.n_rg, a, s));
  RgArgs r{(float2*)Yout, pl->d_coef, 0, pl->d_rg_tab};
  CUDA_TRY(launch_rg_sweep(pl->log_nrg, true, (int)pl->p.n_az, r, s));
  a.in = (const float2*)Yout;
  a.mask = mask;
  CUDA_TRY(launch_az(pl->log_naz, AZ_INV_MASK, a.n_rg, a, s));
  return CSSAR_OK;
}

int enqueue_adjoint(cssar_plan pl, const void* R, const uint32_t* mask, void* Xout, cudaStream_t s) {
  AzArgs a{};
  a.tw = pl->d_az_tab;
  a.n_rg = (int)pl->p.n_rg;
  a.mask_words = (int)(pl->p.n_rg / 32);
  a.scale = (float)(1.0 / std::sqrt((double)pl->p.n_az));
  a.oscale = (float)(1.0 / (std::sqrt((double)pl->p.n_az) * (double)pl->p.n_rg));
  a.in = (const float2*)R;
  a.out = (float2*)Xout;
  a.mask = mask;
  CUDA_TRY(launch_az(pl->log_naz, AZ_FWD_MASK, a.n_rg, a, s));
  RgArgs r{(float2*)Xout, pl->d_coef, 0, pl->d_rg_tab};
  CUDA_TRY(launch_rg_sweep(pl->log_nrg, false, (int)pl->p.n_az, r, s));
  a.in = (const float2*)Xout;
  a.mask = nullptr;
  CUDA_TRY(launch_az(pl->log_naz, AZ_INV_PLAIN, a.n_rg, a, s));
  return CSSAR_OK;
}

// one ITA iteration (S1..S6) on stream s
int enqueue_iteration(cssar_plan pl, const void* Y, const uint32_t* mask, const cssar_ita_params& prm, void* X,
                      cudaStream_t s, bool prof = false) {
#define MARK(i) do { if (prof) CUDA_TRY(cudaEventRecord(pl->ev[i], s)); } while (0)
  AzArgs a{};
  a.tw = pl->d_az_tab;
  a.n_rg = (int)pl->p.n_rg;
  a.mask_words = (int)(pl->p.n_rg / 32);
  a.scale = (float)(1.0 / std::sqrt((double)pl->p.n_az));
  a.oscale = (float)(1.0 / (std::sqrt((double)pl->p.n_az) * (double)pl->p.n_rg));
  a.thr = prm.thr;
  a.rule = prm.rule;
  a.mu = (float)prm.mu;
  a.st = pl->d_st;
  a.hist = pl->d_hist;
  a.cand = pl->cand;
  a.cand_cap = pl->cand_cap;
  a.Y = (const float2*)Y;
  a.mask = mask;
  float2* b = (float2*)X;
  RgArgs r{pl->U, pl->d_coef, 0, pl->d_rg_tab};
  MARK(0);
  // S1: X_i = E(b_{i-1}; sigma_{i-1}); F_eta
  a.in = b;
  a.out = pl->U;
  CUDA_TRY(launch_az(pl->log_naz, AZ_FWD_THR, a.n_rg, a, s));
  MARK(1);
  // S2: G body
  CUDA_TRY(launch_rg_sweep(pl->log_nrg, true, (int)pl->p.n_az, r, s));
  MARK(2);
  // S3: F_eta^-1 ; r = Theta o (Y - G X_i) ; F_eta
  a.in = pl->U;
  a.out = pl->U;
  a.tw = pl->d_az_tab_r;
  CUDA_TRY(launch_az(pl->log_naz, AZ_RESID, a.n_rg, a, s));
  a.tw = pl->d_az_tab;
  MARK(3);
  // S4: M body
  CUDA_TRY(launch_rg_sweep(pl->log_nrg, false, (int)pl->p.n_az, r, s));
  MARK(4);
  // S5: F_eta^-1 ; b_i = X_i + mu dX ; |b|^2 histogram + candidates
  a.b = b;
  CUDA_TRY(launch_az(pl->log_naz, AZ_TAIL, a.n_rg, a, s));
  MARK(5);
  // S6: sigma_i (k-rule select or fixed lambda)
  CUDA_TRY(launch_select(pl->sm_count, b, pl->n, prm.k, prm.rule, prm.thr, (float)prm.mu, pl->d_st, pl->d_hist,
                         pl->d_hist_full, pl->cand, pl->cand_cap, pl->d_log, kLogCap, s));
  MARK(6);
#undef MARK
  return CSSAR_OK;
}

double fixed_sigma(const cssar_ita_params& prm) {
  const double lm = prm.lambda * prm.mu;
  if (prm.thr == CSSAR_THR_SOFT) return lm;
  return std::cbrt(54.0) / 4.0 * std::pow(lm, 2.0 / 3.0);
}

}  // namespace

extern "C" {

const char* cssar_error_string(int code) {
  switch (code) {
    case CSSAR_OK: return "ok";
    case CSSAR_ERR_INVALID_PARAMS: return "invalid SAR parameters";
    case CSSAR_ERR_UNSUPPORTED_SIZE: return "unsupported grid size";
    case CSSAR_ERR_BAD_K: return "k out of range (need 1 <= k < n)";
    case CSSAR_ERR_BAD_MU: return "mu must be > 0 and finite (lambda >= 0)";
    case CSSAR_ERR_ALIGNMENT: return "null or misaligned pointer (16-byte alignment required)";
    case CSSAR_ERR_NONFINITE: return "non-finite values in the iterate";
    case CSSAR_ERR_CUDA: return "CUDA runtime error";
    case CSSAR_ERR_WORKSPACE: return "workspace missing or too small";
    case CSSAR_ERR_NCCL: return "NCCL error";
    case CSSAR_ERR_BAD_PLAN: return "bad plan / world / rank";
    default: return "unknown error";
  }
}

int cssar_plan_create(cssar_plan* out, const cssar_sar_params* p, int world, int rank, const void* nccl_unique_id,
                      void* stream) {
  (void)nccl_unique_id;
  (void)stream;
  if (!out || !p) return CSSAR_ERR_BAD_PLAN;
  *out = nullptr;
  if (world != 1 || rank != 0) return CSSAR_ERR_BAD_PLAN;
  int v = validate_params(*p);
  if (v != CSSAR_OK) return v;
  cssar_plan pl = new cssar_plan_s();
  pl->p = *p;
  pl->log_naz = ilog2_exact(p->n_az);
  pl->log_nrg = ilog2_exact(p->n_rg);
  pl->n = p->n_az * p->n_rg;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&pl->sm_count, cudaDevAttrMultiProcessorCount, dev);
  std::vector<RowCoef> tab = build_coefficients(*p);
  if (cudaMalloc(&pl->d_coef, sizeof(RowCoef) * tab.size()) != cudaSuccess ||
      cudaMemcpy(pl->d_coef, tab.data(), sizeof(RowCoef) * tab.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMalloc(&pl->d_st, sizeof(SelState)) != cudaSuccess ||
      cudaMalloc(&pl->d_hist, sizeof(uint32_t) * HIST_BINS) != cudaSuccess ||
      cudaMalloc(&pl->d_hist_full, sizeof(uint32_t) * HIST_BINS) != cudaSuccess ||
      cudaMalloc(&pl->d_log, sizeof(IterLogDev) * kLogCap) != cudaSuccess ||
      cudaStreamCreateWithFlags(&pl->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&pl->d_rg_tab, sizeof(float2) * rg_table_count(pl->log_nrg)) != cudaSuccess ||
      cudaMalloc(&pl->d_az_tab, sizeof(float2) * (az_table_count(pl->log_naz, false) + 2)) != cudaSuccess ||
      cudaMalloc(&pl->d_az_tab_r, sizeof(float2) * (az_table_count(pl->log_naz, true) + 2)) != cudaSuccess ||
      rg_table_fill(pl->log_nrg, pl->d_rg_tab, pl->cap_stream) != cudaSuccess ||
      az_table_fill(pl->log_naz, false, pl->d_az_tab, pl->cap_stream) != cudaSuccess ||
      az_table_fill(pl->log_naz, true, pl->d_az_tab_r, pl->cap_stream) != cudaSuccess ||
      cudaStreamSynchronize(pl->cap_stream) != cudaSuccess) {
    cssar_plan_destroy(pl);
    return CSSAR_ERR_CUDA;
  }
  for (int i = 0; i < 7; ++i) {
    if (cudaEventCreate(&pl->ev[i]) == cudaSuccess) continue;
    cssar_plan_destroy(pl);
    return CSSAR_ERR_CUDA;
  }
  *out = pl;
  return CSSAR_OK;
}

int cssar_plan_destroy(cssar_plan pl) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
  if (pl->cap_stream) cudaStreamDestroy(pl->cap_stream);
  for (int i = 0; i < 7; ++i)
    if (pl->ev[i]) cudaEventDestroy(pl->ev[i]);
  cudaFree(pl->d_coef);
  cudaFree(pl->d_rg_tab);
  cudaFree(pl->d_az_tab);
  cudaFree(pl->d_az_tab_r);
  cudaFree(pl->d_st);
  cudaFree(pl->d_hist);
  cudaFree(pl->d_hist_full);
  cudaFree(pl->d_log);
  delete pl;
  return CSSAR_OK;
}

static size_t cand_capacity(long long n) { return (size_t)(n / 8 + 65536); }

int cssar_workspace_size(cssar_plan pl, size_t* bytes) {
  if (!pl || !bytes) return CSSAR_ERR_BAD_PLAN;
  const size_t u = sizeof(float2) * (size_t)pl->n;
  *bytes = u + sizeof(uint32_t) * cand_capacity(pl->n) + 256;
  return CSSAR_OK;
}

int cssar_bind_workspace(cssar_plan pl, void* ws, size_t bytes) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  size_t need = 0;
  cssar_workspace_size(pl, &need);
  if (!ws || bytes < need) return CSSAR_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return CSSAR_ERR_ALIGNMENT;
  pl->ws = (char*)ws;
  pl->ws_bytes = bytes;
  pl->U = (float2*)ws;
  pl->cand = (uint32_t*)((char*)ws + sizeof(float2) * (size_t)pl->n);
  pl->cand_cap = (uint32_t)cand_capacity(pl->n);
  if (pl->gexec) { cudaGraphExecDestroy(pl->gexec); pl->gexec = nullptr; }
  pl->ghave = false;
  return CSSAR_OK;
}

int cssar_forward(cssar_plan pl, const void* X, const uint32_t* mask_bits, void* Y_out, void* stream) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(X) || !aligned16(Y_out) || (mask_bits && !aligned16(mask_bits))) return CSSAR_ERR_ALIGNMENT;
  return enqueue_forward(pl, X, mask_bits, Y_out, (cudaStream_t)stream);
}

int cssar_adjoint(cssar_plan pl, const void* R, const uint32_t* mask_bits, void* X_out, void* stream) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(R) || !aligned16(X_out) || (mask_bits && !aligned16(mask_bits))) return CSSAR_ERR_ALIGNMENT;
  return enqueue_adjoint(pl, R, mask_bits, X_out, (cudaStream_t)stream);
}

int cssar_image(cssar_plan pl, const void* Y, const uint32_t* mask_bits, void* X_out, void* stream) {
  return cssar_adjoint(pl, Y, mask_bits, X_out, stream);
}

int cssar_ita_iterate(cssar_plan pl, const void* Y, const uint32_t* mask_bits, const cssar_ita_params* prm,
                      void* X_inout, cssar_iter_log* log_host, void* stream) {
  if (!pl || !prm) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(Y) || !aligned16(X_inout) || (mask_bits && !aligned16(mask_bits))) return CSSAR_ERR_ALIGNMENT;
  if (prm->thr != CSSAR_THR_SOFT && prm->thr != CSSAR_THR_HALF) return CSSAR_ERR_INVALID_PARAMS;
  if (prm->rule != CSSAR_RULE_KSPARSE && prm->rule != CSSAR_RULE_FIXED_LAMBDA) return CSSAR_ERR_INVALID_PARAMS;
  if (!(prm->mu > 0.0) || !std::isfinite(prm->mu)) return CSSAR_ERR_BAD_MU;
  if (prm->rule == CSSAR_RULE_KSPARSE && (prm->k < 1 || prm->k >= pl->n)) return CSSAR_ERR_BAD_K;
  if (prm->rule == CSSAR_RULE_FIXED_LAMBDA && (!(prm->lambda >= 0.0) || !std::isfinite(prm->lambda)))
    return CSSAR_ERR_BAD_MU;
  if (prm->iters < 0 || prm->iters > kLogCap) return CSSAR_ERR_INVALID_PARAMS;
  if (!pl->U) return CSSAR_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const float sigma_fixed = prm->rule == CSSAR_RULE_FIXED_LAMBDA ? (float)fixed_sigma(*prm) : 0.f;
  CUDA_TRY(launch_init_state(pl->d_st, pl->d_hist, pl->d_hist_full, prm->thr, sigma_fixed, s));
  const bool prof = (prm->flags & CSSAR_FLAG_PROFILE_STAGES) != 0;
  if (prof) {
    for (int i = 0; i < 6; ++i) pl->stage_ms[i] = 0.0;
    pl->stage_iters = 0;
    for (int it = 0; it < prm->iters; ++it) {
      int rc = enqueue_iteration(pl, Y, mask_bits, *prm, X_inout, s, true);
      if (rc != CSSAR_OK) return rc;
      CUDA_TRY(cudaEventSynchronize(pl->ev[6]));
      for (int i = 0; i < 6; ++i) {
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, pl->ev[i], pl->ev[i + 1]));
        pl->stage_ms[i] += ms;
      }
      pl->stage_iters += 1;
    }
  } else if (prm->iters > 0) {
    GraphKey key{Y, mask_bits, X_inout, prm->thr, prm->rule, prm->rule == CSSAR_RULE_KSPARSE ? prm->k : 0,
                 prm->lambda, prm->mu};
    if (!pl->ghave || !(pl->gkey == key)) {
      if (pl->gexec) { cudaGraphExecDestroy(pl->gexec); pl->gexec = nullptr; }
      pl->ghave = false;
      cudaGraph_t g = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(pl->cap_stream, cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_iteration(pl, Y, mask_bits, *prm, X_inout, pl->cap_stream);
      cudaError_t ec = cudaStreamEndCapture(pl->cap_stream, &g);
      if (rc != CSSAR_OK) { if (g) cudaGraphDestroy(g); return rc; }
      CUDA_TRY(ec);
      cudaError_t ei = cudaGraphInstantiate(&pl->gexec, g, 0);
      cudaGraphDestroy(g);
      CUDA_TRY(ei);
      pl->gkey = key;
      pl->ghave = true;
    }
    for (int it = 0; it < prm->iters; ++it) CUDA_TRY(cudaGraphLaunch(pl->gexec, s));
  }
  CUDA_TRY(launch_finalize((float2*)X_inout, pl->n, prm->thr, pl->d_st, s));
  if (log_host) {
    std::vector<IterLogDev> tmp((size_t)prm->iters);
    SelState st;
    if (prm->iters > 0)
      CUDA_TRY(cudaMemcpyAsync(tmp.data(), pl->d_log, sizeof(IterLogDev) * prm->iters, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&st, pl->d_st, sizeof(SelState), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int i = 0; i < prm->iters; ++i) {
      log_host[i].sigma = tmp[i].sigma;
      log_host[i].lambda = tmp[i].lam;
      log_host[i].support = tmp[i].support;
      log_host[i].resid2 = tmp[i].resid2;
    }
    if (st.nonfinite) return CSSAR_ERR_NONFINITE;
  }
  return CSSAR_OK;
}

int cssar_pack_mask(const uint8_t* mask_u8, uint32_t* mask_bits, int64_t rows, int64_t cols, void* stream) {
  if (!aligned16(mask_u8) || !aligned16(mask_bits)) return CSSAR_ERR_ALIGNMENT;
  if (rows < 1 || cols < 32 || (cols % 32) != 0) return CSSAR_ERR_UNSUPPORTED_SIZE;
  CUDA_TRY(launch_pack_mask(mask_u8, mask_bits, rows, cols, (cudaStream_t)stream));
  return CSSAR_OK;
}

int cssar_debug_range_sweep(cssar_plan pl, void* U, int gbody, void* stream) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(U)) return CSSAR_ERR_ALIGNMENT;
  RgArgs r{(float2*)U, pl->d_coef, 0, pl->d_rg_tab};
  CUDA_TRY(launch_rg_sweep(pl->log_nrg, gbody != 0, (int)pl->p.n_az, r, (cudaStream_t)stream));
  return CSSAR_OK;
}

int cssar_debug_az_fft(cssar_plan pl, const void* in, void* out, int dir, void* stream) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(in) || !aligned16(out)) return CSSAR_ERR_ALIGNMENT;
  AzArgs a{};
  a.tw = pl->d_az_tab;
  a.n_rg = (int)pl->p.n_rg;
  a.mask_words = (int)(pl->p.n_rg / 32);
  a.scale = (float)(1.0 / std::sqrt((double)pl->p.n_az));
  a.oscale = a.scale;   // plain unitary transform (no range sweep follows)
  a.in = (const float2*)in;
  a.out = (float2*)out;
  CUDA_TRY(launch_az(pl->log_naz, dir < 0 ? AZ_FWD_PLAIN : AZ_INV_PLAIN, a.n_rg, a, (cudaStream_t)stream));
  return CSSAR_OK;
}

int cssar_debug_select(cssar_plan pl, const void* b, int64_t k, uint32_t* sigma2_bits_out, int64_t* above_out,
                       void* stream) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(b)) return CSSAR_ERR_ALIGNMENT;
  if (k < 1 || k >= pl->n) return CSSAR_ERR_BAD_K;
  if (!pl->U) return CSSAR_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(launch_init_state(pl->d_st, pl->d_hist, pl->d_hist_full, CSSAR_THR_SOFT, 0.f, s));
  CUDA_TRY(launch_select(pl->sm_count, (float2*)b, pl->n, k, CSSAR_RULE_KSPARSE, CSSAR_THR_SOFT, 1.0f, pl->d_st,
                         pl->d_hist, pl->d_hist_full, pl->cand, pl->cand_cap, pl->d_log, kLogCap, s));
  SelState st;
  IterLogDev e;
  CUDA_TRY(cudaMemcpyAsync(&st, pl->d_st, sizeof(SelState), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(&e, pl->d_log, sizeof(IterLogDev), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (sigma2_bits_out) *sigma2_bits_out = st.sigma2_bits;
  if (above_out) *above_out = e.support;
  return CSSAR_OK;
}

int cssar_stage_times(cssar_plan pl, double* ms_out, int32_t* iters_out) {
  if (!pl || !ms_out) return CSSAR_ERR_BAD_PLAN;
  for (int i = 0; i < 6; ++i) ms_out[i] = pl->stage_ms[i];
  if (iters_out) *iters_out = pl->stage_iters;
  return CSSAR_OK;
}

int cssar_debug_fallbacks(cssar_plan pl, int32_t* out, void* stream) {
  if (!pl || !out) return CSSAR_ERR_BAD_PLAN;
  SelState st;
  CUDA_TRY(cudaMemcpyAsync(&st, pl->d_st, sizeof(SelState), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  *out = st.fallbacks;
  return CSSAR_OK;
}

}  // extern "C"
