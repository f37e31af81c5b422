// libcssar C ABI (include/cssar.h): plan (S0 phase-coefficient table), operator calls and
// the graph-replayed ITA loop.  Host code only; device work lives in kernels.cu.
#include <nvtx3/nvToolsExt.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
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
  int flags;                        // the iteration body differs with CSSAR_FLAG_ADAPTIVE_MU
  bool operator==(const GraphKey& o) const {
    return Y == o.Y && mask == o.mask && X == o.X && thr == o.thr && rule == o.rule && k == o.k &&
           lambda == o.lambda && mu == o.mu && flags == o.flags;
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
  float2* d_rcmc = nullptr;       // RDA plans: per-row RCMC migration (alpha, s0); CSA: nullptr
  float2* d_hrange = nullptr;     // RDA plans with a recorded pulse: G's range filter H (n_rg)
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
  float2* D = nullptr;              // adaptive step: the dense gradient dX (world 1)
  float2* Xk = nullptr;             // tolerance stop: the kept X_i (world 1)
  double2* d_conv = nullptr;        // tolerance stop: per-block (||X_(i+1) - X_i||^2, ||X_i||^2)
  double2* h_conv = nullptr;        //   pinned host copy
  int conv_blocks = 0;
  int iters_done = 0;
  uint32_t* cand = nullptr;
  uint32_t cand_cap = 0;
  // graph cache for the iteration body
  cudaStream_t cap_stream = nullptr;
  cudaStream_t cond_stream = nullptr;   // captures the body of the conditional fallback round (world > 1)
  bool cond_ok = true;                  // conditional graph nodes usable (cleared if a capture with one fails)
  bool cond_used = false;               // the cached iteration graph gates the fallback round
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey{};
  bool ghave = false;
  // per-step profiling (CSSAR_FLAG_PROFILE_STAGES)
  cudaEvent_t ev[7] = {};
  double stage_ms[6] = {};
  int stage_iters = 0;
  // ---- multi-GPU slab partition; world == 1 leaves these unset
  int world = 1, rank = 0;
  long long nrow = 0, ncol = 0;     // row slab: nrow = n_az/world lines; column slab: ncol = n_rg/world gates
  int transport = 0;                // kTransportNone / kTransportNccl / kTransportGroup
  // the slab path (row / column slabs, transposes, rank-reduced select) runs: world > 1, or a
  // one-rank NCCL plan (cssar_debug_plan_create_nccl, a test of the NCCL plumbing on one GPU)
  bool multi = false;
  ncclComm_t comm = nullptr;
  uint32_t* d_lvl = nullptr;        // 1024 level counts of the split fine select
  // workspace views (world > 1): column slabs [n_az][ncol], blocked row slab [world][nrow][ncol]
  float2* Ucol = nullptr;
  float2* Vrow = nullptr;
  float2* Ycol = nullptr;
  float2* bcol = nullptr;
  uint32_t* mcol = nullptr;         // mask bits of the column slab, ncol/32 words per line
  bool have_mask = false;
  // fused transposes: every rank's Ucol / Vrow mapped in this process (peer memory over
  // NVLink via CUDA IPC on a multi-GPU box; the other emulated ranks' buffers in a group)
  bool fused = false;
  float2* peerU[16] = {};
  float2* peerV[16] = {};
  // sparse-X' schedule: this rank's X list [count | pad | entries] in the workspace, every
  // rank's list (peer memory), forward twiddles of the m = n_az/world point azimuth DFT
  char* sxl = nullptr;
  uint32_t sx_cap = 0;
  char* peerL[16] = {};
  float2* d_az_tab_m = nullptr;
  bool sparse_used = false;         // the last cssar_ita_iterate ran the sparse-X' schedule
  void* ipc_base[16] = {};          // IPC mappings opened by this rank (closed on rebind/destroy)
  uint32_t* d_bar = nullptr;        // 1-word all-reduce used as the inter-sweep barrier (NCCL)
  double* d_red = nullptr;          // deterministic norm reductions: [3][kRedSlots] partials + tickets
  // non-finite report of the last solve without a log: the flag word copied to pinned host
  // memory at the end of the call, read by cssar_ita_status after its event
  uint32_t* h_nonfinite = nullptr;
  cudaEvent_t ev_solve = nullptr;
  bool solve_pending = false;
  // sparse-state schedule (world 1, cluster azimuth shapes): two per-panel lists in the workspace
  SsLists ss{};
  bool ss_ok = false;
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

// NEXT-2 RDA operator pair (oracle/rda.py; eq. 14-18, 23): per Doppler bin i
//   q[1] = P_tau = exp(+j pi f_tau^2 / K_r)      cycles (1/(2 K_r)) (F_r/N)^2 l'^2
//   q[2] = P_eta = exp(-j pi f^2 / K_a(R0) + j 4 pi fc R0 / c),  K_a = 2 V_r^2 fc / (c R0),
//          R0 = R_ref + u c / (2 F_r):  cycles -(f^2 c R_ref)/(4 V_r^2 fc) + 2 fc R_ref / c
//          + u (fc / F_r - f^2 c^2 / (8 V_r^2 fc F_r))
//   rcmc = (alpha, s0): migration d = R0 (1/D - 1) 2 F_r / c = s0 + alpha u range cells,
//          alpha = 1/D - 1, s0 = alpha 2 R_ref F_r / c   (u = j - N/2)
std::vector<RowCoef> build_coefficients_rda(const cssar_sar_params& p, std::vector<float2>& rcmc) {
  const long long na = p.n_az, nr = p.n_rg;
  std::vector<RowCoef> tab((size_t)na);
  rcmc.assign((size_t)na, float2{0.f, 0.f});
  const long double fc = p.fc, Kr = p.Kr, Fr = p.Fr, prf = p.prf, Vr = p.Vr, Rr = p.R_ref;
  const long double df = Fr / (long double)nr;
  for (long long i = 0; i < na; ++i) {
    const long long is = (i < (na + 1) / 2) ? i : i - na;
    const long double f = (long double)is * prf / (long double)na;
    const long double xr = kC * f / (2.0L * Vr * fc);
    const long double x = xr * xr;
    const long double D = sqrtl(1.0L - x);
    const long double idm1 = (x / (1.0L + D)) / D;
    RowCoef rc{};
    rc.q[1] = {frac_u64(df * df / (2.0L * Kr)), 0ull, 0ull};
    rc.q[2] = {0ull, frac_u64(fc / Fr - f * f * kC * kC / (8.0L * Vr * Vr * fc * Fr)),
               frac_u64(2.0L * fc * Rr / kC - f * f * kC * Rr / (4.0L * Vr * Vr * fc))};
    tab[(size_t)i] = rc;
    rcmc[(size_t)i] = float2{(float)idm1, (float)(idm1 * 2.0L * Rr * Fr / kC)};
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
  if (p.op != 0 && p.op != CSSAR_OP_CSA && p.op != CSSAR_OP_RDA) return CSSAR_ERR_INVALID_PARAMS;
  if (p.op == CSSAR_OP_RDA) {
    // the RCMC transpose gathers from a fixed window: the migration may vary by < 1/2 cell
    // across the row at the Doppler edge (alpha n_rg < 1/2)
    const double xr = 299792458.0 * fmax / (2.0 * p.Vr * p.fc);
    const double D = std::sqrt(1.0 - xr * xr);
    if ((1.0 / D - 1.0) * (double)p.n_rg >= 0.5) return CSSAR_ERR_INVALID_PARAMS;
    // the wrap-around outputs of D recomputed exactly are those within 12 gates of the row
    // start (rg.cu kRcmcWrapLo): the migration must stay below 6 cells
    if ((1.0 / D - 1.0) * (2.0 * p.R_ref * p.Fr / 299792458.0 + 0.5 * (double)p.n_rg) >= 6.0)
      return CSSAR_ERR_INVALID_PARAMS;
  }
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

constexpr int kTransportNone = 0, kTransportNccl = 1, kTransportGroup = 2;
constexpr size_t kSxHeader = 256;               // sparse-X' list header (entry count) in the workspace
constexpr size_t kBarSlotOff = 64;              // flag-barrier slots [16] u32 inside that header

// NCCL entry points resolved at run time from the process's libnccl.so.2 (the one torch
// loaded, or CSSAR_NCCL_LIB); the single-GPU path never touches NCCL.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*asyncError)(ncclComm_t, ncclResult_t*) = nullptr;   // optional
};

NcclApi load_nccl() {
  NcclApi a;
  const char* path = std::getenv("CSSAR_NCCL_LIB");
  void* h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    std::fprintf(stderr, "libcssar: cannot load NCCL (%s)\n", dlerror());
    return a;
  }
#define NCCL_SYM(f, name) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, name))
  NCCL_SYM(getUniqueId, "ncclGetUniqueId");
  NCCL_SYM(commInitRank, "ncclCommInitRank");
  NCCL_SYM(commDestroy, "ncclCommDestroy");
  NCCL_SYM(groupStart, "ncclGroupStart");
  NCCL_SYM(groupEnd, "ncclGroupEnd");
  NCCL_SYM(send, "ncclSend");
  NCCL_SYM(recv, "ncclRecv");
  NCCL_SYM(allReduce, "ncclAllReduce");
  NCCL_SYM(allGather, "ncclAllGather");
  NCCL_SYM(asyncError, "ncclCommGetAsyncError");
#undef NCCL_SYM
  a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.groupStart && a.groupEnd && a.send && a.recv &&
         a.allReduce && a.allGather;
  return a;
}

NcclApi& nccl() {
  static NcclApi a = load_nccl();
  return a;
}

#define NCCL_TRY(x)                                                                      \
  do {                                                                                   \
    ncclResult_t _r = (x);                                                               \
    if (_r != ncclSuccess) {                                                             \
      std::fprintf(stderr, "libcssar: %s failed: NCCL error %d\n", #x, (int)_r);         \
      return CSSAR_ERR_NCCL;                                                             \
    }                                                                                    \
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
  r.rcmc = pl->d_rcmc;
  r.hrange = pl->d_hrange;
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
  r.rcmc = pl->d_rcmc;
  r.hrange = pl->d_hrange;
  CUDA_TRY(launch_rg_sweep(pl->log_nrg, false, (int)pl->p.n_az, r, s));
  a.in = (const float2*)Xout;
  a.mask = nullptr;
  CUDA_TRY(launch_az(pl->log_naz, AZ_INV_PLAIN, a.n_rg, a, s));
  return CSSAR_OK;
}

// S6 of the sparse-state schedule: coarse select; on a fallback the dense S5 re-run into b, the
// full-histogram kernels and the fine select on it, then the list rebuild (each early-exits
// unless the coarse select asked for the fallback)
cudaError_t launch_select_ss(cssar_plan pl, AzArgs a, float2* b, const cssar_ita_params& prm, cudaStream_t s) {
  cudaError_t e = launch_select_part(SEL_COARSE, pl->sm_count, b, pl->n, prm.k, prm.thr, (float)prm.mu, pl->d_st,
                                     pl->d_hist, pl->d_hist_full, pl->cand, pl->cand_cap, pl->d_lvl, pl->d_log, kLogCap,
                                     s);
  if (e != cudaSuccess) return e;
  a.in = pl->U;
  a.b = b;
  e = launch_az(pl->log_naz, AZ_TAIL_SSD, a.n_rg, a, s);
  if (e != cudaSuccess) return e;
  e = launch_select_rest(pl->sm_count, b, pl->n, prm.k, prm.thr, (float)prm.mu, pl->d_st, pl->d_hist,
                         pl->d_hist_full, pl->cand, pl->cand_cap, pl->d_log, kLogCap, s);
  if (e != cudaSuccess) return e;
  return launch_ss_rebuild(b, (int)pl->p.n_az, (int)pl->p.n_rg, pl->ss, pl->d_st, 0, s);
}

// one ITA iteration (S1..S6) on stream s
// fuse: fixed-lambda schedule -- S5 fused with the next iteration's S1 (AZ_FUSE); the iteration
// runs S1 only when s1 is set (the first one)
int enqueue_iteration(cssar_plan pl, const void* Y, const uint32_t* mask, const cssar_ita_params& prm, void* X,
                      cudaStream_t s, bool prof = false, bool ss = false, bool fuse = false, bool s1 = true) {
  // PROFILE_STAGES: CUDA events between the steps, and NVTX ranges S1..S6 for nsys timelines
  static const char* const kStage[6] = {"S1 az head", "S2 range G", "S3 az residual", "S4 range M", "S5 az tail",
                                         "S6 select"};
#define MARK(i)                                               \
  do {                                                        \
    if (prof) {                                               \
      if ((i) > 0) nvtxRangePop();                            \
      if ((i) < 6) nvtxRangePushA(kStage[(i) < 6 ? (i) : 0]); \
      CUDA_TRY(cudaEventRecord(pl->ev[i], s));                \
    }                                                         \
  } while (0)
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
  a.red_part = pl->d_red;
  a.red_ticket = reinterpret_cast<uint32_t*>(pl->d_red + 3 * kRedSlots);
  a.ss = pl->ss;
  float2* b = (float2*)X;
  RgArgs r{pl->U, pl->d_coef, 0, pl->d_rg_tab};
  r.rcmc = pl->d_rcmc;
  r.hrange = pl->d_hrange;
  MARK(0);
  // S1: X_i = E(b_{i-1}; sigma_{i-1}); F_eta   (sparse state: b_{i-1} from the list)
  a.in = ss ? pl->U : b;                 // (FWD_SS reads no dense input; any mapped pointer)
  a.out = pl->U;
  if (s1) CUDA_TRY(launch_az(pl->log_naz, ss ? AZ_FWD_SS : AZ_FWD_THR, a.n_rg, a, s));
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
  a.b = b;
  if (prm.flags & CSSAR_FLAG_ADAPTIVE_MU) {
    // S5 (adaptive step, eq. 27): dX = F_eta^-1 u kept in D, F_eta(dX on supp X_i), ||dX_k||^2;
    // G body; ||Theta o F_eta^-1 .||^2; mu_i = ratio; b_i = X_i + mu_i dX (+ histogram)
    a.in = pl->U;
    a.out = pl->U;
    a.D = pl->D;
    a.lambda = (float)prm.lambda;
    a.tw = pl->d_az_tab_r;
    CUDA_TRY(launch_az(pl->log_naz, AZ_GRAD, a.n_rg, a, s));
    a.tw = pl->d_az_tab;
    CUDA_TRY(launch_rg_sweep(pl->log_nrg, true, (int)pl->p.n_az, r, s));
    CUDA_TRY(launch_az(pl->log_naz, AZ_NORM, a.n_rg, a, s));
    CUDA_TRY(launch_adaptive_step(a, pl->n, pl->sm_count, s));
  } else if (fuse) {
    // S5 + next S1 (fixed lambda): b_i stored, X_{i+1} = E(b_i; sigma) transformed into U
    a.in = pl->U;
    a.out = pl->U;
    a.tw = pl->d_az_tab_r;
    CUDA_TRY(launch_az(pl->log_naz, AZ_FUSE, a.n_rg, a, s));
    a.tw = pl->d_az_tab;
  } else if (ss) {
    // S5 (sparse state): X_i from the list; b_i -> histogram, candidates and the next list
    a.in = pl->U;
    CUDA_TRY(launch_az(pl->log_naz, AZ_TAIL_SS, a.n_rg, a, s));
  } else {
    // S5: F_eta^-1 ; b_i = X_i + mu dX ; |b|^2 histogram + candidates
    CUDA_TRY(launch_az(pl->log_naz, AZ_TAIL, a.n_rg, a, s));
  }
  MARK(5);
  // S6: sigma_i (k-rule select or fixed lambda)
  if (ss) {
    // select fallback (target bin outside the window): S5 again with a dense b_i in X's buffer
    // for the full-histogram kernels (early exit otherwise), then the list rebuilt from it
    CUDA_TRY(launch_select_ss(pl, a, b, prm, s));
  } else {
    CUDA_TRY(launch_select(pl->sm_count, b, pl->n, prm.k, prm.rule, prm.thr, (float)prm.mu, pl->d_st, pl->d_hist,
                           pl->d_hist_full, pl->cand, pl->cand_cap, pl->d_log, kLogCap, s));
  }
  MARK(6);
#undef MARK
  return CSSAR_OK;
}

// end of a solve: the device's non-finite flag -> pinned host word, event for cssar_ita_status
cudaError_t note_solve_end(cssar_plan pl, cudaStream_t s) {
  static_assert(offsetof(SelState, sync_error) == offsetof(SelState, nonfinite) + 4, "flag words adjacent");
  cudaError_t e = cudaMemcpyAsync(pl->h_nonfinite, reinterpret_cast<char*>(pl->d_st) + offsetof(SelState, nonfinite),
                                  2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  e = cudaEventRecord(pl->ev_solve, s);
  pl->solve_pending = e == cudaSuccess;
  return e;
}

double fixed_sigma(const cssar_ita_params& prm) {
  const double lm = prm.lambda * prm.mu;
  if (prm.thr == CSSAR_THR_SOFT) return lm;
  if (prm.thr == CSSAR_THR_HARD) return std::sqrt(lm);
  if (prm.thr == CSSAR_THR_TWOTHIRDS) return (2.0 / 3.0) * std::pow(3.0 * lm * lm * lm, 0.25);
  return std::cbrt(54.0) / 4.0 * std::pow(lm, 2.0 / 3.0);
}


// ---------------------------------------------------------------- multi-rank path (world > 1)
// each rank owns the row slab of n_az/world azimuth lines (the user's arrays).
// Range sweeps run on row slabs, azimuth sweeps on column slabs of n_rg/world gates; four
// all-to-all transposes per iteration move between them, and the k-rule select reduces its
// histograms across ranks.  Block algebra: a column slab [n_az][ncol] is, read as send
// buffer, the blocks [q][nrow][ncol] for destination q; what rank q receives is the blocked
// row slab [p][nrow][ncol] the range kernel reads with RgArgs::blk (and vice versa), so no
// pack/unpack pass is needed inside the loop.  The same schedule drives either one NCCL rank
// (np == 1) or all ranks of a single-device emulation group (np == world, exchanges done
// with device copies and a summing kernel) — the group runs the identical kernels.
struct Ranks {
  cssar_plan* pl;
  int np;
  bool group() const { return pl[0]->transport == kTransportGroup; }
};

int xchg_a2a(const Ranks& R, void* const* send, void* const* recv, size_t blk, cudaStream_t s) {
  const int P = R.pl[0]->world;
  if (R.group()) {
    for (int p = 0; p < P; ++p)
      for (int q = 0; q < P; ++q)
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv[q]) + (size_t)p * blk,
                                 static_cast<const char*>(send[p]) + (size_t)q * blk, blk, cudaMemcpyDeviceToDevice,
                                 s));
    return CSSAR_OK;
  }
  NcclApi& n = nccl();
  cssar_plan pl = R.pl[0];
  NCCL_TRY(n.groupStart());
  for (int q = 0; q < P; ++q) {
    NCCL_TRY(n.send(static_cast<const char*>(send[0]) + (size_t)q * blk, blk, ncclUint8, q, pl->comm, s));
    NCCL_TRY(n.recv(static_cast<char*>(recv[0]) + (size_t)q * blk, blk, ncclUint8, q, pl->comm, s));
  }
  NCCL_TRY(n.groupEnd());
  return CSSAR_OK;
}

// in-place sum over ranks; dtype 0 = u32, 1 = u64, 2 = f64
int xchg_allreduce(const Ranks& R, void* const* bufs, int dtype, size_t count, cudaStream_t s) {
  if (R.group()) {
    CUDA_TRY(launch_group_sum(dtype, bufs, R.pl[0]->world, (long long)count, s));
    return CSSAR_OK;
  }
  const ncclDataType_t t = dtype == 0 ? ncclUint32 : dtype == 1 ? ncclUint64 : ncclFloat64;
  NCCL_TRY(nccl().allReduce(bufs[0], bufs[0], count, t, ncclSum, R.pl[0]->comm, s));
  return CSSAR_OK;
}

// two in-place sums in one NCCL group (one fused collective launch)
int xchg_allreduce2(const Ranks& R, void* const* a, int ta, size_t na, void* const* b, int tb, size_t nb,
                    cudaStream_t s) {
  if (R.group()) {
    CUDA_TRY(launch_group_sum(ta, a, R.pl[0]->world, (long long)na, s));
    CUDA_TRY(launch_group_sum(tb, b, R.pl[0]->world, (long long)nb, s));
    return CSSAR_OK;
  }
  auto ty = [](int t) { return t == 0 ? ncclUint32 : t == 1 ? ncclUint64 : ncclFloat64; };
  NcclApi& n = nccl();
  NCCL_TRY(n.groupStart());
  NCCL_TRY(n.allReduce(a[0], a[0], na, ty(ta), ncclSum, R.pl[0]->comm, s));
  NCCL_TRY(n.allReduce(b[0], b[0], nb, ty(tb), ncclSum, R.pl[0]->comm, s));
  NCCL_TRY(n.groupEnd());
  return CSSAR_OK;
}

// every rank's barrier slot array (16 u32 in the sparse-list header of its workspace)
PeerSlots peer_slots(cssar_plan pl) {
  PeerSlots ps{};
  for (int q = 0; q < pl->world; ++q)
    ps.slots[q] = pl->peerL[q] ? reinterpret_cast<uint32_t*>(pl->peerL[q] + kBarSlotOff) : nullptr;
  return ps;
}

// peer-store transposes run when the peers are mapped and, on real NCCL ranks, only on request
// (CSSAR_FLAG_PEER_TRANSPOSE); the single-device emulation group uses them by default
bool fused_active(const Ranks& R, const cssar_ita_params& prm) {
  return R.pl[0]->fused && (R.group() || (prm.flags & CSSAR_FLAG_PEER_TRANSPOSE));
}

template <class F>
void gather_ptrs(const Ranks& R, void** out, F f) {
  for (int i = 0; i < R.np; ++i) out[i] = (void*)f(R.pl[i]);
}

AzArgs az_col_args(cssar_plan pl, const cssar_ita_params& prm) {
  AzArgs a{};
  a.tw = pl->d_az_tab;
  a.n_rg = (int)pl->ncol;
  a.mask_words = (int)(pl->ncol / 32);
  a.scale = (float)(1.0 / std::sqrt((double)pl->p.n_az));
  a.oscale = (float)(1.0 / (std::sqrt((double)pl->p.n_az) * (double)pl->p.n_rg));
  a.thr = prm.thr;
  a.rule = prm.rule;
  a.mu = (float)prm.mu;
  a.st = pl->d_st;
  a.hist = pl->d_hist;
  a.cand = pl->cand;
  a.cand_cap = pl->cand_cap;
  a.Y = pl->Ycol;
  a.mask = pl->have_mask ? pl->mcol : nullptr;
  a.b = pl->bcol;
  a.red_part = pl->d_red;
  a.red_ticket = reinterpret_cast<uint32_t*>(pl->d_red + 3 * kRedSlots);
  return a;
}

RgArgs rg_row_args(cssar_plan pl) {
  RgArgs r{pl->Vrow, pl->d_coef, (int)(pl->rank * pl->nrow), pl->d_rg_tab, 0, 0};
  r.rcmc = pl->d_rcmc;
  r.hrange = pl->d_hrange;
  r.log_w = ilog2_exact(pl->ncol);
  r.blk = pl->nrow * pl->ncol;
  return r;
}

// the select's fallback round runs when the coarse step set need_full (conditional graph node)
__global__ void set_fallback_cond_kernel(cudaGraphConditionalHandle h, const SelState* st) {
  cudaGraphSetConditional(h, st->need_full ? 1u : 0u);
}

// one ITA iteration (S1..S6) of every rank in R
int iteration_multi(const Ranks& R, const cssar_ita_params& prm, cudaStream_t s, bool sparse = false) {
  cssar_plan p0 = R.pl[0];
  const size_t blk = (size_t)p0->nrow * (size_t)p0->ncol * sizeof(float2);
  void *U[16], *V[16], *B[16];
  gather_ptrs(R, U, [](cssar_plan q) { return q->Ucol; });
  gather_ptrs(R, V, [](cssar_plan q) { return q->Vrow; });
  const bool fused = fused_active(R, prm);
  auto az = [&](int mode) -> int {
    for (int i = 0; i < R.np; ++i) {
      cssar_plan pl = R.pl[i];
      AzArgs a = az_col_args(pl, prm);
      a.in = mode == AZ_FWD_THR ? pl->bcol : pl->Ucol;
      a.out = pl->Ucol;
      if (mode == AZ_RESID) a.tw = pl->d_az_tab_r;
      if (fused && mode != AZ_TAIL) {        // epilogue stores into every rank's row slab block
        for (int q = 0; q < pl->world; ++q) a.dst[q] = pl->peerV[q];
        a.dlog_nrow = ilog2_exact(pl->nrow);
        a.drank = pl->rank;
      }
      CUDA_TRY(launch_az(pl->log_naz, mode, a.n_rg, a, s));
    }
    return CSSAR_OK;
  };
  auto rg = [&](bool gbody) -> int {
    for (int i = 0; i < R.np; ++i) {
      cssar_plan pl = R.pl[i];
      RgArgs r = rg_row_args(pl);
      if (fused) {                           // epilogue stores into every rank's column slab
        for (int q = 0; q < pl->world; ++q) r.dst[q] = pl->peerU[q];
        r.dlog_nrow = ilog2_exact(pl->nrow);
        r.drank = pl->rank;
      }
      CUDA_TRY(launch_rg_sweep(pl->log_nrg, gbody, (int)pl->nrow, r, s));
    }
    return CSSAR_OK;
  };
  // after a fused sweep: every rank's peer stores into us are complete (NCCL: a one-word
  // all-reduce orders the ranks' streams; the emulation group is serialised on one stream)
  auto barrier = [&]() -> int {
    if (R.group()) return CSSAR_OK;            // one stream: already ordered
    CUDA_TRY(launch_flag_barrier(p0->rank, p0->world, peer_slots(p0), p0->d_bar + 1,
                                 reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(p0->d_st) +
                                                             offsetof(SelState, sync_error)),
                                 s));
    return CSSAR_OK;
  };
  auto local_sel = [&](int part, cudaStream_t ss) -> int {
    for (int i = 0; i < R.np; ++i) {
      cssar_plan pl = R.pl[i];
      CUDA_TRY(launch_select_part(part, pl->sm_count, pl->bcol, pl->p.n_az * pl->ncol, prm.k, prm.thr,
                                  (float)prm.mu, pl->d_st, pl->d_hist, pl->d_hist_full, pl->cand, pl->cand_cap,
                                  pl->d_lvl, pl->d_log, kLogCap, ss));
    }
    return CSSAR_OK;
  };
  // sparse-X' S1 (sparse.cu): compact X = E(b) into a list, all ranks'
  // lists folded into a length n_az/world array, m-point azimuth DFT -> cyclic row slab
  auto sx_s1 = [&]() -> int {
    for (int i = 0; i < R.np; ++i) {
      cssar_plan pl = R.pl[i];
      CUDA_TRY(launch_sx_compact(pl->bcol, pl->p.n_az * pl->ncol, ilog2_exact(pl->ncol), (int)(pl->rank * pl->ncol),
                                 pl->d_st, prm.thr, reinterpret_cast<SxEntry*>(pl->sxl + kSxHeader),
                                 reinterpret_cast<uint32_t*>(pl->sxl), pl->sx_cap, pl->sm_count, s));
    }
    int rc = barrier();                       // every rank's list complete
    if (rc != CSSAR_OK) return rc;
    for (int i = 0; i < R.np; ++i) {
      cssar_plan pl = R.pl[i];
      SxLists L{};
      for (int q = 0; q < pl->world; ++q) {
        L.list[q] = reinterpret_cast<const SxEntry*>(pl->peerL[q] + kSxHeader);
        L.count[q] = reinterpret_cast<const uint32_t*>(pl->peerL[q]);
      }
      L.cap = pl->sx_cap;
      L.world = pl->world;
      const int n_rg = (int)pl->p.n_rg;
      CUDA_TRY(launch_sx_fold(L, pl->rank, pl->log_naz, (int)pl->nrow, n_rg, pl->Vrow, pl->sm_count, s));
      AzArgs a{};
      a.tw = pl->d_az_tab_m;
      a.n_rg = n_rg;
      a.mask_words = n_rg / 32;
      a.scale = (float)(1.0 / std::sqrt((double)pl->p.n_az));
      a.oscale = (float)(1.0 / (std::sqrt((double)pl->p.n_az) * (double)n_rg));
      a.in = pl->Vrow;
      a.out = pl->Vrow;
      CUDA_TRY(launch_az(ilog2_exact(pl->nrow), AZ_FWD_PLAIN, n_rg, a, s));
      RgArgs r = rg_row_args(pl);             // S2 on the cyclic slab, plain row-major
      r.row_base = pl->rank;
      r.row_step = pl->world;
      r.log_w = pl->log_nrg;
      r.blk = 1;                              // blocked path (fused stores); j >> log_w = 0
      r.dlog_w = ilog2_exact(pl->ncol);
      for (int q = 0; q < pl->world; ++q) r.dst[q] = pl->peerU[q];
      CUDA_TRY(launch_rg_sweep(pl->log_nrg, true, (int)pl->nrow, r, s));
    }
    return CSSAR_OK;
  };
#define STEP(x) do { int _rc = (x); if (_rc != CSSAR_OK) return _rc; } while (0)
  if (fused && sparse) {
    STEP(sx_s1());                            // S1' + S2: lists -> cyclic row slab -> column slabs
    STEP(barrier());
    STEP(az(AZ_RESID));
    STEP(barrier());
    STEP(rg(false));
    STEP(barrier());
  } else if (fused) {                         // compute + transpose in one kernel per sweep
    STEP(az(AZ_FWD_THR));                     // S1: column slabs -> every rank's row slab
    STEP(barrier());
    STEP(rg(true));                           // S2: row slab -> every rank's column slab
    STEP(barrier());
    STEP(az(AZ_RESID));                       // S3
    STEP(barrier());
    STEP(rg(false));                          // S4
    STEP(barrier());
  } else {
    STEP(az(AZ_FWD_THR));                     // S1 on column slabs
    STEP(xchg_a2a(R, U, V, blk, s));          //    -> blocked row slabs
    STEP(rg(true));                           // S2
    STEP(xchg_a2a(R, V, U, blk, s));          //    -> column slabs
    STEP(az(AZ_RESID));                       // S3
    STEP(xchg_a2a(R, U, V, blk, s));
    STEP(rg(false));                          // S4
    STEP(xchg_a2a(R, V, U, blk, s));
  }
  STEP(az(AZ_TAIL));                          // S5: local histogram / candidates / support
  void* H[16];
  gather_ptrs(R, B, [](cssar_plan q) { return reinterpret_cast<char*>(q->d_st) + offsetof(SelState, resid2); });
  gather_ptrs(R, H, [](cssar_plan q) { return q->d_hist; });
  if (prm.rule == CSSAR_RULE_KSPARSE) {       // S6: exact (k+1)-th largest over all ranks
    // ||r||^2 and the |b|^2 histogram (+ flags) in one NCCL group: one collective launch
    STEP(xchg_allreduce2(R, B, 2, 1, H, 0, HIST_WORDS, s));
    STEP(local_sel(SEL_COARSE, s));
    // full-histogram fallback round (the coarse bin missed the speculative window): a pass over
    // b, an all-reduce of 2048 words and the pick.  Every rank takes the same decision from the
    // same reduced counts, so inside a captured iteration it is a conditional graph node whose
    // body runs only when need_full is set -- 3 collectives per iteration instead of 4
    auto fb_round = [&](cudaStream_t ss) -> int {
      STEP(local_sel(SEL_FB_HIST, ss));
      gather_ptrs(R, B, [](cssar_plan q) { return q->d_hist_full; });
      STEP(xchg_allreduce(R, B, 0, HIST_BINS, ss));
      STEP(local_sel(SEL_FB_PICK, ss));
      return CSSAR_OK;
    };
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(s, &cs));
    if (cs == cudaStreamCaptureStatusActive && p0->cond_ok && p0->cond_stream && !getenv("CSSAR_NO_COND")) {
      cudaGraph_t g = nullptr;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      CUDA_TRY(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
      cudaGraphConditionalHandle h;
      CUDA_TRY(cudaGraphConditionalHandleCreate(&h, g, 0u, 0u));
      set_fallback_cond_kernel<<<1, 1, 0, s>>>(h, p0->d_st);
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeIf;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      CUDA_TRY(cudaGraphAddNode(&node, g, deps, nd, &cp));
      CUDA_TRY(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      CUDA_TRY(cudaStreamBeginCaptureToGraph(p0->cond_stream, body, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal));
      const int rb = fb_round(p0->cond_stream);
      cudaGraph_t gb = nullptr;
      const cudaError_t eb = cudaStreamEndCapture(p0->cond_stream, &gb);
      STEP(rb);
      CUDA_TRY(eb);
      p0->cond_used = true;
    } else {
      STEP(fb_round(s));
    }
    STEP(local_sel(SEL_FINE0_HIST, s));
    gather_ptrs(R, B, [](cssar_plan q) { return q->d_lvl; });
    STEP(xchg_allreduce(R, B, 0, 1024, s));
    STEP(local_sel(SEL_FINE0_FIND, s));
    STEP(xchg_allreduce(R, B, 0, 1024, s));
    STEP(local_sel(SEL_FINE1_FIND, s));
  } else {
    void* S[16];
    gather_ptrs(R, S, [](cssar_plan q) {
      return reinterpret_cast<char*>(q->d_st) + offsetof(SelState, support_fixed);
    });
    STEP(xchg_allreduce2(R, B, 2, 1, S, 1, 1, s));
    for (int i = 0; i < R.np; ++i)
      CUDA_TRY(launch_lambda_step(R.pl[i]->d_st, prm.thr, (float)prm.mu, R.pl[i]->d_log, kLogCap, s));
  }
#undef STEP
  return CSSAR_OK;
}

// row slab [nrow][row_elems] (elem bytes each) -> blocks [world][nrow][row_elems/world] in dst
int pack_rows(cssar_plan pl, const void* src, void* dst, size_t row_elems, size_t elem, cudaStream_t s) {
  const size_t w = row_elems / (size_t)pl->world;
  for (int q = 0; q < pl->world; ++q)
    CUDA_TRY(cudaMemcpy2DAsync(static_cast<char*>(dst) + (size_t)q * pl->nrow * w * elem, w * elem,
                               static_cast<const char*>(src) + (size_t)q * w * elem, row_elems * elem, w * elem,
                               (size_t)pl->nrow, cudaMemcpyDeviceToDevice, s));
  return CSSAR_OK;
}

int unpack_rows(cssar_plan pl, const void* src, void* dst, size_t row_elems, size_t elem, cudaStream_t s) {
  const size_t w = row_elems / (size_t)pl->world;
  for (int q = 0; q < pl->world; ++q)
    CUDA_TRY(cudaMemcpy2DAsync(static_cast<char*>(dst) + (size_t)q * w * elem, row_elems * elem,
                               static_cast<const char*>(src) + (size_t)q * pl->nrow * w * elem, w * elem, w * elem,
                               (size_t)pl->nrow, cudaMemcpyDeviceToDevice, s));
  return CSSAR_OK;
}

// user row slabs (Y, mask, X_0) -> column slabs Ycol, mcol, bcol
int setup_multi(const Ranks& R, const void* const* Y, const uint32_t* const* mask, void* const* X, cudaStream_t s) {
  cssar_plan p0 = R.pl[0];
  const size_t n_rg = (size_t)p0->p.n_rg;
  const size_t blk = (size_t)p0->nrow * (size_t)p0->ncol * sizeof(float2);
  void *V[16], *D[16];
  gather_ptrs(R, V, [](cssar_plan q) { return q->Vrow; });
  for (int i = 0; i < R.np; ++i) {
    const int rc = pack_rows(R.pl[i], Y[i], R.pl[i]->Vrow, n_rg, sizeof(float2), s);
    if (rc != CSSAR_OK) return rc;
  }
  gather_ptrs(R, D, [](cssar_plan q) { return q->Ycol; });
  int rc = xchg_a2a(R, V, D, blk, s);
  if (rc != CSSAR_OK) return rc;
  const bool have_mask = mask[0] != nullptr;
  for (int i = 0; i < R.np; ++i) R.pl[i]->have_mask = have_mask;
  if (have_mask) {
    for (int i = 0; i < R.np; ++i) {
      rc = pack_rows(R.pl[i], mask[i], R.pl[i]->Vrow, n_rg / 32, sizeof(uint32_t), s);
      if (rc != CSSAR_OK) return rc;
    }
    gather_ptrs(R, D, [](cssar_plan q) { return q->mcol; });
    rc = xchg_a2a(R, V, D, (size_t)p0->nrow * (size_t)(p0->ncol / 32) * sizeof(uint32_t), s);
    if (rc != CSSAR_OK) return rc;
  }
  for (int i = 0; i < R.np; ++i) {
    rc = pack_rows(R.pl[i], X[i], R.pl[i]->Vrow, n_rg, sizeof(float2), s);
    if (rc != CSSAR_OK) return rc;
  }
  gather_ptrs(R, D, [](cssar_plan q) { return q->bcol; });
  return xchg_a2a(R, V, D, blk, s);
}

// X_I = E(b; sigma) on the column slabs, then back to the user row slabs
int final_multi(const Ranks& R, const cssar_ita_params& prm, void* const* X, cudaStream_t s) {
  cssar_plan p0 = R.pl[0];
  const size_t blk = (size_t)p0->nrow * (size_t)p0->ncol * sizeof(float2);
  void *Bc[16], *V[16];
  for (int i = 0; i < R.np; ++i)
    CUDA_TRY(launch_finalize(R.pl[i]->bcol, R.pl[i]->p.n_az * R.pl[i]->ncol, prm.thr, R.pl[i]->d_st, s));
  gather_ptrs(R, Bc, [](cssar_plan q) { return q->bcol; });
  gather_ptrs(R, V, [](cssar_plan q) { return q->Vrow; });
  int rc = xchg_a2a(R, Bc, V, blk, s);
  if (rc != CSSAR_OK) return rc;
  for (int i = 0; i < R.np; ++i) {
    rc = unpack_rows(R.pl[i], R.pl[i]->Vrow, X[i], (size_t)p0->p.n_rg, sizeof(float2), s);
    if (rc != CSSAR_OK) return rc;
  }
  return CSSAR_OK;
}

int validate_ita(cssar_plan pl, const cssar_ita_params* prm) {
  if (prm->thr < CSSAR_THR_SOFT || prm->thr > CSSAR_THR_TWOTHIRDS) return CSSAR_ERR_INVALID_PARAMS;
  if (prm->rule != CSSAR_RULE_KSPARSE && prm->rule != CSSAR_RULE_FIXED_LAMBDA) return CSSAR_ERR_INVALID_PARAMS;
  if (!(prm->mu > 0.0) || !std::isfinite(prm->mu)) return CSSAR_ERR_BAD_MU;
  if (prm->rule == CSSAR_RULE_KSPARSE && (prm->k < 1 || prm->k >= pl->n)) return CSSAR_ERR_BAD_K;
  if (prm->rule == CSSAR_RULE_FIXED_LAMBDA && (!(prm->lambda >= 0.0) || !std::isfinite(prm->lambda)))
    return CSSAR_ERR_BAD_MU;
  if (prm->iters < 0 || prm->iters > kLogCap) return CSSAR_ERR_INVALID_PARAMS;
  if ((prm->flags & CSSAR_FLAG_ADAPTIVE_MU) && pl->multi) return CSSAR_ERR_INVALID_PARAMS;
  if (!(prm->tol >= 0.0) || !std::isfinite(prm->tol) || (prm->tol > 0.0 && pl->multi))
    return CSSAR_ERR_INVALID_PARAMS;
  if ((prm->flags & CSSAR_FLAG_SPARSE_X) && !pl->multi) return CSSAR_ERR_INVALID_PARAMS;
  return CSSAR_OK;
}

// the whole multi-rank solve for the ranks in R (NCCL rank or emulation group)
// forward / adjoint / image on world > 1 plans (the boundary's "local slab" contract, SURVEY
// 8(b)): input row slabs -> column slabs (pack + all-to-all), first azimuth sweep, all-to-all
// into blocked row slabs, range sweep, all-to-all back, second azimuth sweep, column slabs ->
// output row slabs.  Same kernels and global indices as world 1 (bitwise equal results).
int op_multi(const Ranks& R, bool forward, const void* const* in, const uint32_t* const* mask, void* const* out,
             cudaStream_t s) {
  cssar_plan p0 = R.pl[0];
  for (int i = 0; i < R.np; ++i)
    if (!R.pl[i]->Ucol) return CSSAR_ERR_WORKSPACE;
  const size_t n_rg = (size_t)p0->p.n_rg;
  const size_t blk = (size_t)p0->nrow * (size_t)p0->ncol * sizeof(float2);
  void *U[16], *V[16], *Bc[16], *Mc[16];
  gather_ptrs(R, U, [](cssar_plan q) { return q->Ucol; });
  gather_ptrs(R, V, [](cssar_plan q) { return q->Vrow; });
  gather_ptrs(R, Bc, [](cssar_plan q) { return q->bcol; });
  gather_ptrs(R, Mc, [](cssar_plan q) { return q->mcol; });
  int rc;
  const bool have_mask = mask[0] != nullptr;
  for (int i = 0; i < R.np; ++i) R.pl[i]->have_mask = have_mask;
  if (have_mask) {
    for (int i = 0; i < R.np; ++i)
      if ((rc = pack_rows(R.pl[i], mask[i], R.pl[i]->Vrow, n_rg / 32, sizeof(uint32_t), s)) != CSSAR_OK) return rc;
    if ((rc = xchg_a2a(R, V, Mc, (size_t)p0->nrow * (size_t)(p0->ncol / 32) * sizeof(uint32_t), s)) != CSSAR_OK)
      return rc;
  }
  for (int i = 0; i < R.np; ++i)
    if ((rc = pack_rows(R.pl[i], in[i], R.pl[i]->Vrow, n_rg, sizeof(float2), s)) != CSSAR_OK) return rc;
  if ((rc = xchg_a2a(R, V, Bc, blk, s)) != CSSAR_OK) return rc;
  cssar_ita_params prm{};
  prm.thr = CSSAR_THR_SOFT;
  prm.rule = CSSAR_RULE_KSPARSE;
  prm.mu = 1.0;
  for (int i = 0; i < R.np; ++i) {                        // F_eta (forward: plain; adjoint: Theta first)
    cssar_plan pl = R.pl[i];
    AzArgs a = az_col_args(pl, prm);
    a.in = pl->bcol;
    a.out = pl->Ucol;
    if (forward) a.mask = nullptr;
    CUDA_TRY(launch_az(pl->log_naz, forward ? AZ_FWD_PLAIN : AZ_FWD_MASK, a.n_rg, a, s));
  }
  if ((rc = xchg_a2a(R, U, V, blk, s)) != CSSAR_OK) return rc;
  for (int i = 0; i < R.np; ++i) {                        // range body (G or M) on blocked row slabs
    cssar_plan pl = R.pl[i];
    RgArgs r = rg_row_args(pl);
    CUDA_TRY(launch_rg_sweep(pl->log_nrg, forward, (int)pl->nrow, r, s));
  }
  if ((rc = xchg_a2a(R, V, U, blk, s)) != CSSAR_OK) return rc;
  for (int i = 0; i < R.np; ++i) {                        // F_eta^-1 (forward: then Theta)
    cssar_plan pl = R.pl[i];
    AzArgs a = az_col_args(pl, prm);
    a.in = pl->Ucol;
    a.out = pl->bcol;
    if (!forward) a.mask = nullptr;
    CUDA_TRY(launch_az(pl->log_naz, forward ? AZ_INV_MASK : AZ_INV_PLAIN, a.n_rg, a, s));
  }
  if ((rc = xchg_a2a(R, Bc, V, blk, s)) != CSSAR_OK) return rc;
  for (int i = 0; i < R.np; ++i)
    if ((rc = unpack_rows(R.pl[i], R.pl[i]->Vrow, out[i], n_rg, sizeof(float2), s)) != CSSAR_OK) return rc;
  return CSSAR_OK;
}

int ita_multi(const Ranks& R, const void* const* Y, const uint32_t* const* mask, const cssar_ita_params& prm,
              void* const* X, cssar_iter_log* log_host, cudaStream_t s, cudaGraphExec_t* gexec, GraphKey* gkey,
              bool* ghave) {
  cssar_plan p0 = R.pl[0];
  const float sigma_fixed = prm.rule == CSSAR_RULE_FIXED_LAMBDA ? (float)fixed_sigma(prm) : 0.f;
  for (int i = 0; i < R.np; ++i)
    CUDA_TRY(launch_init_state(R.pl[i]->d_st, R.pl[i]->d_hist, R.pl[i]->d_hist_full, prm.thr, sigma_fixed, s));
  int rc = setup_multi(R, Y, mask, X, s);
  if (rc != CSSAR_OK) return rc;
  // sparse-X' (CSSAR_FLAG_SPARSE_X): X_0 is arbitrary, so iteration 0 runs the dense schedule
  // outside the graph; X_i (i >= 1) has at most k nonzeros
  const bool sparse = (prm.flags & CSSAR_FLAG_SPARSE_X) && prm.rule == CSSAR_RULE_KSPARSE && fused_active(R, prm) &&
                      p0->d_az_tab_m && (uint64_t)prm.k <= (uint64_t)p0->sx_cap;
  p0->sparse_used = sparse;
  int first = 0;
  if (sparse && prm.iters > 0) {
    rc = iteration_multi(R, prm, s, false);
    if (rc != CSSAR_OK) return rc;
    first = 1;
  }
  if (prm.iters > first) {
    GraphKey key{nullptr, (const void*)(uintptr_t)p0->have_mask, nullptr, prm.thr, prm.rule,
                 prm.rule == CSSAR_RULE_KSPARSE ? prm.k : 0, prm.lambda, prm.mu,
                 (sparse ? CSSAR_FLAG_SPARSE_X : 0) | (fused_active(R, prm) ? CSSAR_FLAG_PEER_TRANSPOSE : 0)};
    if (!*ghave || !(*gkey == key)) {
      if (*gexec) { cudaGraphExecDestroy(*gexec); *gexec = nullptr; }
      *ghave = false;
      // with the conditional fallback round first; if the capture or instantiation of that
      // graph fails (e.g. collective work the conditional body cannot hold), once more without it.
      // On NCCL ranks the outcome is agreed collectively (every rank reaches the agreement), so
      // all ranks replay graphs with the same collective sequence.
      for (int attempt = 0;; ++attempt) {
        cudaGraph_t g = nullptr;
        p0->cond_used = false;
        CUDA_TRY(cudaStreamBeginCapture(p0->cap_stream, cudaStreamCaptureModeThreadLocal));
        rc = iteration_multi(R, prm, p0->cap_stream, sparse);
        cudaError_t ec = cudaStreamEndCapture(p0->cap_stream, &g);
        cudaError_t ei = cudaErrorUnknown;
        if (rc == CSSAR_OK && ec == cudaSuccess) ei = cudaGraphInstantiate(gexec, g, 0);
        if (g) cudaGraphDestroy(g);
        const bool ok = rc == CSSAR_OK && ec == cudaSuccess && ei == cudaSuccess;
        bool all_ok = ok, same = true;
        if (!R.group() && p0->transport == kTransportNccl) {
          uint32_t w[2] = {ok ? 0u : 1u, p0->cond_used ? 1u : 0u};     // [failed ranks, ranks with the node]
          if (cudaMemcpy(p0->d_bar, w, 8, cudaMemcpyHostToDevice) != cudaSuccess ||
              nccl().allReduce(p0->d_bar, p0->d_bar, 2, ncclUint32, ncclSum, p0->comm, p0->cap_stream) != ncclSuccess ||
              cudaStreamSynchronize(p0->cap_stream) != cudaSuccess ||
              cudaMemcpy(w, p0->d_bar, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
            return CSSAR_ERR_NCCL;
          all_ok = w[0] == 0u;
          same = w[1] == 0u || w[1] == (uint32_t)p0->world;
        }
        if (all_ok && same) break;
        if (ok && *gexec) { cudaGraphExecDestroy(*gexec); *gexec = nullptr; }
        if (attempt > 0) {
          if (rc != CSSAR_OK) return rc;
          CUDA_TRY(ec);
          CUDA_TRY(ei);
          return CSSAR_ERR_NCCL;                 // another rank could not capture the iteration
        }
        (void)cudaGetLastError();
        p0->cond_ok = false;                     // retry with the unconditional fallback round
      }
      *gkey = key;
      *ghave = true;
    }
    for (int it = first; it < prm.iters; ++it) CUDA_TRY(cudaGraphLaunch(*gexec, s));
  }
  rc = final_multi(R, prm, X, s);
  if (rc != CSSAR_OK) return rc;
  for (int i = 0; i < R.np; ++i) CUDA_TRY(note_solve_end(R.pl[i], s));
  if (log_host) {
    std::vector<IterLogDev> tmp((size_t)prm.iters);
    SelState st;
    if (prm.iters > 0)
      CUDA_TRY(cudaMemcpyAsync(tmp.data(), p0->d_log, sizeof(IterLogDev) * prm.iters, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&st, p0->d_st, sizeof(SelState), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int i = 0; i < prm.iters; ++i) {
      log_host[i].sigma = tmp[i].sigma;
      log_host[i].lambda = tmp[i].lam;
      log_host[i].support = tmp[i].support;
      log_host[i].resid2 = tmp[i].resid2;
      log_host[i].mu = tmp[i].mu;
      log_host[i].gap = tmp[i].gap;
      log_host[i].gap_exact = tmp[i].gap_exact;
    }
    if (st.sync_error) return CSSAR_ERR_NCCL;
    if (st.nonfinite) return CSSAR_ERR_NONFINITE;
  }
  return CSSAR_OK;
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

}  // extern "C"

namespace {

// ---- fused transposes on a multi-GPU box: map every rank's workspace through CUDA IPC
void close_peers(cssar_plan pl) {
  for (int q = 0; q < 16; ++q) {
    if (pl->ipc_base[q]) cudaIpcCloseMemHandle(pl->ipc_base[q]);
    pl->ipc_base[q] = nullptr;
    pl->peerU[q] = pl->peerV[q] = nullptr;
  }
  pl->fused = false;
}

// collective over the plan's communicator; on any failure the plan keeps the NCCL
// all-to-all transposes (fused = false) and says so on stderr
int map_peers_nccl(cssar_plan pl) {
  close_peers(pl);
  if (std::getenv("CSSAR_MULTI_A2A")) return CSSAR_OK;
  static_assert(sizeof(IpcRec) % 16 == 0, "record size");
  IpcRec mine{};
  ipc_export(pl->ws, &mine);                     // off = ~0 marks a failed export
  // every rank takes part in the all-gather even if its own export failed
  IpcRec* d = nullptr;
  std::vector<IpcRec> all((size_t)pl->world);
  CUDA_TRY(cudaMalloc(&d, sizeof(IpcRec) * (size_t)(pl->world + 1)));
  int rc = CSSAR_OK;
  if (cudaMemcpy(d + pl->world, &mine, sizeof(IpcRec), cudaMemcpyHostToDevice) != cudaSuccess ||
      nccl().allGather(d + pl->world, d, sizeof(IpcRec), ncclUint8, pl->comm, pl->cap_stream) != ncclSuccess ||
      cudaStreamSynchronize(pl->cap_stream) != cudaSuccess ||
      cudaMemcpy(all.data(), d, sizeof(IpcRec) * (size_t)pl->world, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = CSSAR_ERR_NCCL;
  cudaFree(d);
  if (rc != CSSAR_OK) return rc;
  bool every = true;
  for (const IpcRec& r : all) every = every && r.off != ~0ull;
  const size_t voff = (size_t)((char*)pl->Vrow - (char*)pl->Ucol);
  for (int q = 0; q < pl->world && every; ++q) {
    if (q == pl->rank) {
      pl->peerU[q] = pl->Ucol;
      pl->peerV[q] = pl->Vrow;
      pl->peerL[q] = pl->sxl;
      continue;
    }
    void *pb = nullptr, *pp = nullptr;
    if (ipc_open(all[(size_t)q], &pb, &pp) != 0) {
      every = false;
      break;
    }
    pl->ipc_base[q] = pb;
    pl->peerU[q] = reinterpret_cast<float2*>(pp);
    pl->peerV[q] = reinterpret_cast<float2*>(reinterpret_cast<char*>(pl->peerU[q]) + voff);
    pl->peerL[q] = reinterpret_cast<char*>(pl->peerU[q]) + (pl->sxl - reinterpret_cast<char*>(pl->Ucol));
  }
  // the flag-barrier slots of this rank and every epoch start at 0 before anyone's first barrier
  // (the all-reduce below orders the clears across ranks)
  if (cudaMemset(pl->sxl + kBarSlotOff, 0, 16 * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemset(pl->d_bar, 0, 16) != cudaSuccess)
    return CSSAR_ERR_CUDA;
  // all ranks must agree on the mode: all-reduce the failure flag
  uint32_t bad = every ? 0u : 1u;
  if (cudaMemcpy(pl->d_bar, &bad, 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      nccl().allReduce(pl->d_bar, pl->d_bar, 1, ncclUint32, ncclSum, pl->comm, pl->cap_stream) != ncclSuccess ||
      cudaStreamSynchronize(pl->cap_stream) != cudaSuccess ||
      cudaMemcpy(&bad, pl->d_bar, 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    return CSSAR_ERR_NCCL;
  if (bad) {
    close_peers(pl);
    std::fprintf(stderr, "libcssar: peer mapping unavailable; using NCCL all-to-all transposes\n");
    return CSSAR_OK;
  }
  pl->fused = true;
  return CSSAR_OK;
}

int validate_world(const cssar_sar_params& p, int world, int rank, bool multi) {
  if (world < 1 || world > 16 || rank < 0 || rank >= world) return CSSAR_ERR_BAD_PLAN;
  if (!multi) return CSSAR_OK;
  if (p.n_az % world || p.n_rg % world) return CSSAR_ERR_UNSUPPORTED_SIZE;
  const long long nrow = p.n_az / world, ncol = p.n_rg / world;
  const int rpc = rg_rows_per_cta(ilog2_exact(p.n_rg));
  if (ncol < 128 || rpc <= 0 || nrow % rpc) return CSSAR_ERR_UNSUPPORTED_SIZE;
  return CSSAR_OK;
}

// plan for one rank; transport kTransportNone (world 1), kTransportNccl or kTransportGroup
int plan_create_impl(cssar_plan* out, const cssar_sar_params* p, int world, int rank, int transport,
                     const void* nccl_unique_id) {
  if (!out || !p) return CSSAR_ERR_BAD_PLAN;
  *out = nullptr;
  int v = validate_params(*p);
  if (v != CSSAR_OK) return v;
  const bool multi = world > 1 || transport == kTransportNccl;
  v = validate_world(*p, world, rank, multi);
  if (v != CSSAR_OK) return v;
  cssar_plan pl = new cssar_plan_s();
  pl->p = *p;
  pl->log_naz = ilog2_exact(p->n_az);
  pl->log_nrg = ilog2_exact(p->n_rg);
  pl->n = p->n_az * p->n_rg;
  pl->world = world;
  pl->rank = rank;
  pl->nrow = p->n_az / world;
  pl->ncol = p->n_rg / world;
  pl->transport = transport;
  pl->multi = multi;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&pl->sm_count, cudaDevAttrMultiProcessorCount, dev);
  std::vector<float2> rcmc;
  std::vector<RowCoef> tab = p->op == CSSAR_OP_RDA ? build_coefficients_rda(*p, rcmc) : build_coefficients(*p);
  if (!rcmc.empty() &&
      (cudaMalloc(&pl->d_rcmc, sizeof(float2) * rcmc.size()) != cudaSuccess ||
       cudaMemcpy(pl->d_rcmc, rcmc.data(), sizeof(float2) * rcmc.size(), cudaMemcpyHostToDevice) != cudaSuccess)) {
    cssar_plan_destroy(pl);
    return CSSAR_ERR_CUDA;
  }
  if (cudaMalloc(&pl->d_coef, sizeof(RowCoef) * tab.size()) != cudaSuccess ||
      cudaMemcpy(pl->d_coef, tab.data(), sizeof(RowCoef) * tab.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMalloc(&pl->d_st, sizeof(SelState)) != cudaSuccess ||
      cudaMalloc(&pl->d_hist, sizeof(uint32_t) * HIST_WORDS) != cudaSuccess ||
      cudaMalloc(&pl->d_hist_full, sizeof(uint32_t) * HIST_BINS) != cudaSuccess ||
      cudaMalloc(&pl->d_lvl, sizeof(uint32_t) * 1024) != cudaSuccess ||
      cudaMalloc(&pl->d_red, sizeof(double) * (3 * kRedSlots + 8)) != cudaSuccess ||
      cudaMemset(pl->d_red, 0, sizeof(double) * (3 * kRedSlots + 8)) != cudaSuccess ||
      cudaMalloc(&pl->d_log, sizeof(IterLogDev) * kLogCap) != cudaSuccess ||
      cudaStreamCreateWithFlags(&pl->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&pl->cond_stream, cudaStreamNonBlocking) != cudaSuccess ||
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
  if (cudaEventCreateWithFlags(&pl->ev_solve, cudaEventDisableTiming) != cudaSuccess ||
      cudaMallocHost(&pl->h_nonfinite, 2 * sizeof(uint32_t)) != cudaSuccess) {
    cssar_plan_destroy(pl);
    return CSSAR_ERR_CUDA;
  }
  pl->h_nonfinite[0] = pl->h_nonfinite[1] = 0u;
  if (multi && pl->log_naz - ilog2_exact(world) >= 7 &&
      (cudaMalloc(&pl->d_az_tab_m, sizeof(float2) * (az_table_count(pl->log_naz - ilog2_exact(world), false) + 2)) !=
           cudaSuccess ||
       az_table_fill(pl->log_naz - ilog2_exact(world), false, pl->d_az_tab_m, pl->cap_stream) != cudaSuccess ||
       cudaStreamSynchronize(pl->cap_stream) != cudaSuccess)) {
    cssar_plan_destroy(pl);
    return CSSAR_ERR_CUDA;
  }
  if (multi && (cudaMalloc(&pl->d_bar, 16) != cudaSuccess || cudaMemset(pl->d_bar, 0, 16) != cudaSuccess)) {
    cssar_plan_destroy(pl);
    return CSSAR_ERR_CUDA;
  }
  if (transport == kTransportNccl) {
    NcclApi& n = nccl();
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    if (!n.ok || n.commInitRank(&pl->comm, world, id, rank) != ncclSuccess) {
      pl->comm = nullptr;
      cssar_plan_destroy(pl);
      return CSSAR_ERR_NCCL;
    }
  }
  *out = pl;
  return CSSAR_OK;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
size_t cand_capacity(long long n) { return (size_t)(n / 8 + 65536); }

// workspace layout: world 1: [U | cand]; world > 1: [Ucol | Vrow | Ycol | bcol | mcol | cand]
// sparse-X' list of a world > 1 rank: kSxHeader-byte header (count) + nl/8 entries of 16 bytes
size_t sx_bytes(size_t nl) { return align256(kSxHeader + sizeof(SxEntry) * (nl / 8)); }

// sparse-state lists of a world-1 plan with cluster azimuth shapes: 2 x (a full-panel entry
// array per panel + its counter)
size_t ss_bytes(cssar_plan pl) {
  const int W = az_panel_width(pl->log_naz);
  if (pl->multi || W <= 0) return 0;
  const size_t npan = (size_t)(pl->p.n_rg / W);
  return 2 * (align256(sizeof(SsEntry) * (size_t)pl->n) + align256(sizeof(uint32_t) * npan));
}

size_t workspace_bytes(cssar_plan pl) {
  if (!pl->multi)
    return align256(3 * sizeof(float2) * (size_t)pl->n + sizeof(uint32_t) * cand_capacity(pl->n)) + ss_bytes(pl) + 256;
  const size_t nl = (size_t)pl->p.n_az * (size_t)pl->ncol;
  return 4 * align256(sizeof(float2) * nl) + align256(nl / 8) + align256(sizeof(uint32_t) * cand_capacity((long long)nl)) +
         256 + sx_bytes(nl) + 256;
}

void bind_views(cssar_plan pl, char* ws) {
  if (!pl->multi) {
    pl->U = (float2*)ws;
    pl->D = (float2*)(ws + sizeof(float2) * (size_t)pl->n);
    pl->Xk = (float2*)(ws + 2 * sizeof(float2) * (size_t)pl->n);
    pl->cand = (uint32_t*)(ws + 3 * sizeof(float2) * (size_t)pl->n);
    pl->cand_cap = (uint32_t)cand_capacity(pl->n);
    pl->ss = SsLists{};
    pl->ss_ok = ss_bytes(pl) > 0;
    if (pl->ss_ok) {
      char* q = ws + align256(3 * sizeof(float2) * (size_t)pl->n + sizeof(uint32_t) * cand_capacity(pl->n));
      const int W = az_panel_width(pl->log_naz);
      pl->ss.W = W;
      pl->ss.npan = (int)(pl->p.n_rg / W);
      pl->ss.capp = (uint32_t)(pl->p.n_az * W);
      for (int l = 0; l < 2; ++l) {
        pl->ss.ent[l] = reinterpret_cast<SsEntry*>(q);
        q += align256(sizeof(SsEntry) * (size_t)pl->n);
        pl->ss.cnt[l] = reinterpret_cast<uint32_t*>(q);
        q += align256(sizeof(uint32_t) * (size_t)pl->ss.npan);
      }
    }
    return;
  }
  const size_t nl = (size_t)pl->p.n_az * (size_t)pl->ncol;
  const size_t a = align256(sizeof(float2) * nl);
  pl->Ucol = (float2*)ws;
  pl->Vrow = (float2*)(ws + a);
  pl->Ycol = (float2*)(ws + 2 * a);
  pl->bcol = (float2*)(ws + 3 * a);
  pl->mcol = (uint32_t*)(ws + 4 * a);
  pl->cand = (uint32_t*)(ws + 4 * a + align256(nl / 8));
  pl->cand_cap = (uint32_t)cand_capacity((long long)nl);
  pl->sxl = ws + 4 * a + align256(nl / 8) + align256(sizeof(uint32_t) * cand_capacity((long long)nl)) + 256;
  pl->sx_cap = (uint32_t)(nl / 8);
  pl->U = pl->Ucol;
}

}  // namespace

// single-device emulation of a `world`-rank plan group (tests of the multi-GPU schedule)
struct cssar_group_s {
  std::vector<cssar_plan> pl;
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey{};
  bool ghave = false;
};

extern "C" {

int cssar_plan_create(cssar_plan* out, const cssar_sar_params* p, int world, int rank, const void* nccl_unique_id,
                      void* stream) {
  (void)stream;
  if (!out || !p) return CSSAR_ERR_BAD_PLAN;
  if (world > 1 && !nccl_unique_id) return CSSAR_ERR_BAD_PLAN;
  return plan_create_impl(out, p, world, rank, world > 1 ? kTransportNccl : kTransportNone, nccl_unique_id);
}

int cssar_debug_plan_create_nccl(cssar_plan* out, const cssar_sar_params* p, const void* nccl_unique_id) {
  if (!out || !p || !nccl_unique_id) return CSSAR_ERR_BAD_PLAN;
  return plan_create_impl(out, p, 1, 0, kTransportNccl, nccl_unique_id);
}

int cssar_nccl_unique_id(void* id_out) {
  if (!id_out) return CSSAR_ERR_BAD_PLAN;
  NcclApi& n = nccl();
  if (!n.ok) return CSSAR_ERR_NCCL;
  ncclUniqueId id;
  NCCL_TRY(n.getUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return CSSAR_OK;
}

int cssar_plan_destroy(cssar_plan pl) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  close_peers(pl);
  cudaFree(pl->d_bar);
  // the cached graph first: NCCL work captured in it holds the communicator (ncclCommDestroy
  // waits for the graph's release of it -- measured: a hang when destroyed in the other order)
  if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
  pl->gexec = nullptr;
  if (pl->comm && nccl().ok) {
    cudaDeviceSynchronize();
    nccl().commDestroy(pl->comm);
  }
  if (pl->cap_stream) cudaStreamDestroy(pl->cap_stream);
  if (pl->cond_stream) cudaStreamDestroy(pl->cond_stream);
  for (int i = 0; i < 7; ++i)
    if (pl->ev[i]) cudaEventDestroy(pl->ev[i]);
  if (pl->ev_solve) cudaEventDestroy(pl->ev_solve);
  if (pl->h_nonfinite) cudaFreeHost(pl->h_nonfinite);
  cudaFree(pl->d_coef);
  cudaFree(pl->d_rg_tab);
  cudaFree(pl->d_rcmc);
  cudaFree(pl->d_hrange);
  cudaFree(pl->d_conv);
  if (pl->h_conv) cudaFreeHost(pl->h_conv);
  cudaFree(pl->d_az_tab);
  cudaFree(pl->d_az_tab_r);
  cudaFree(pl->d_az_tab_m);
  cudaFree(pl->d_st);
  cudaFree(pl->d_hist);
  cudaFree(pl->d_hist_full);
  cudaFree(pl->d_lvl);
  cudaFree(pl->d_red);
  cudaFree(pl->d_log);
  delete pl;
  return CSSAR_OK;
}

int cssar_workspace_size(cssar_plan pl, size_t* bytes) {
  if (!pl || !bytes) return CSSAR_ERR_BAD_PLAN;
  *bytes = workspace_bytes(pl);
  return CSSAR_OK;
}

int cssar_bind_workspace(cssar_plan pl, void* ws, size_t bytes) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (!ws || bytes < workspace_bytes(pl)) return CSSAR_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return CSSAR_ERR_ALIGNMENT;
  pl->ws = (char*)ws;
  pl->ws_bytes = bytes;
  bind_views(pl, (char*)ws);
  if (pl->gexec) { cudaGraphExecDestroy(pl->gexec); pl->gexec = nullptr; }
  pl->ghave = false;
  if (pl->transport == kTransportNccl) return map_peers_nccl(pl);   // collective
  return CSSAR_OK;
}

int cssar_group_create(cssar_group* out, const cssar_sar_params* p, int world, void* stream) {
  (void)stream;
  if (!out || !p || world < 2) return CSSAR_ERR_BAD_PLAN;
  *out = nullptr;
  cssar_group g = new cssar_group_s();
  for (int r = 0; r < world; ++r) {
    cssar_plan pl = nullptr;
    const int rc = plan_create_impl(&pl, p, world, r, kTransportGroup, nullptr);
    if (rc != CSSAR_OK) {
      cssar_group_destroy(g);
      return rc;
    }
    g->pl.push_back(pl);
  }
  *out = g;
  return CSSAR_OK;
}

int cssar_group_destroy(cssar_group g) {
  if (!g) return CSSAR_ERR_BAD_PLAN;
  if (g->gexec) cudaGraphExecDestroy(g->gexec);
  for (cssar_plan pl : g->pl) cssar_plan_destroy(pl);
  delete g;
  return CSSAR_OK;
}

int cssar_group_workspace_size(cssar_group g, size_t* bytes_per_rank) {
  if (!g || g->pl.empty() || !bytes_per_rank) return CSSAR_ERR_BAD_PLAN;
  *bytes_per_rank = workspace_bytes(g->pl[0]);
  return CSSAR_OK;
}

int cssar_group_bind_workspace(cssar_group g, int rank, void* ws, size_t bytes) {
  if (!g || rank < 0 || rank >= (int)g->pl.size()) return CSSAR_ERR_BAD_PLAN;
  if (g->gexec) { cudaGraphExecDestroy(g->gexec); g->gexec = nullptr; }
  g->ghave = false;
  return cssar_bind_workspace(g->pl[(size_t)rank], ws, bytes);
}

int cssar_group_ita_iterate(cssar_group g, const void* const* Y, const uint32_t* const* mask_bits,
                            const cssar_ita_params* prm, void* const* X_inout, cssar_iter_log* log_host,
                            void* stream) {
  if (!g || g->pl.empty() || !prm || !Y || !mask_bits || !X_inout) return CSSAR_ERR_BAD_PLAN;
  const int P = (int)g->pl.size();
  for (int r = 0; r < P; ++r) {
    if (!aligned16(Y[r]) || !aligned16(X_inout[r])) return CSSAR_ERR_ALIGNMENT;
    if ((mask_bits[r] != nullptr) != (mask_bits[0] != nullptr)) return CSSAR_ERR_INVALID_PARAMS;
    if (mask_bits[r] && !aligned16(mask_bits[r])) return CSSAR_ERR_ALIGNMENT;
    if (!g->pl[(size_t)r]->Ucol) return CSSAR_ERR_WORKSPACE;
  }
  const bool fused = std::getenv("CSSAR_MULTI_A2A") == nullptr;
  for (int r = 0; r < P; ++r) if (g->pl[(size_t)r]->fused != fused) g->ghave = false;
  for (int r = 0; r < P; ++r) g->pl[(size_t)r]->fused = fused;
  const int v = validate_ita(g->pl[0], prm);
  if (v != CSSAR_OK) return v;
  for (int r = 0; r < P; ++r) {
    cssar_plan pl = g->pl[(size_t)r];
    for (int q = 0; q < P; ++q) {
      pl->peerU[q] = g->pl[(size_t)q]->Ucol;
      pl->peerV[q] = g->pl[(size_t)q]->Vrow;
      pl->peerL[q] = g->pl[(size_t)q]->sxl;
    }
    if (pl->fused != fused) { g->ghave = false; }
    pl->fused = fused;
  }
  Ranks R{g->pl.data(), P};
  return ita_multi(R, Y, mask_bits, *prm, X_inout, log_host, (cudaStream_t)stream, &g->gexec, &g->gkey,
                   &g->ghave);
}

int cssar_forward(cssar_plan pl, const void* X, const uint32_t* mask_bits, void* Y_out, void* stream) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(X) || !aligned16(Y_out) || (mask_bits && !aligned16(mask_bits))) return CSSAR_ERR_ALIGNMENT;
  if (pl->multi) {
    Ranks R{&pl, 1};
    return op_multi(R, true, &X, &mask_bits, &Y_out, (cudaStream_t)stream);
  }
  return enqueue_forward(pl, X, mask_bits, Y_out, (cudaStream_t)stream);
}

int cssar_adjoint(cssar_plan pl, const void* R, const uint32_t* mask_bits, void* X_out, void* stream) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(R) || !aligned16(X_out) || (mask_bits && !aligned16(mask_bits))) return CSSAR_ERR_ALIGNMENT;
  if (pl->multi) {
    Ranks Rk{&pl, 1};
    return op_multi(Rk, false, &R, &mask_bits, &X_out, (cudaStream_t)stream);
  }
  return enqueue_adjoint(pl, R, mask_bits, X_out, (cudaStream_t)stream);
}

int cssar_group_operator(cssar_group g, int forward, const void* const* in, const uint32_t* const* mask_bits,
                         void* const* out, void* stream) {
  if (!g || g->pl.empty() || !in || !mask_bits || !out) return CSSAR_ERR_BAD_PLAN;
  const int P = (int)g->pl.size();
  for (int r = 0; r < P; ++r) {
    if (!aligned16(in[r]) || !aligned16(out[r])) return CSSAR_ERR_ALIGNMENT;
    if ((mask_bits[r] != nullptr) != (mask_bits[0] != nullptr)) return CSSAR_ERR_INVALID_PARAMS;
    if (mask_bits[r] && !aligned16(mask_bits[r])) return CSSAR_ERR_ALIGNMENT;
  }
  Ranks R{g->pl.data(), P};
  return op_multi(R, forward != 0, in, mask_bits, out, (cudaStream_t)stream);
}

int cssar_image(cssar_plan pl, const void* Y, const uint32_t* mask_bits, void* X_out, void* stream) {
  return cssar_adjoint(pl, Y, mask_bits, X_out, stream);
}

namespace {
struct NvtxRange {
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

int cssar_ita_iterate(cssar_plan pl, const void* Y, const uint32_t* mask_bits, const cssar_ita_params* prm,
                      void* X_inout, cssar_iter_log* log_host, void* stream) {
  NvtxRange nvtx_range("cssar_ita_iterate");
  if (!pl || !prm) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(Y) || !aligned16(X_inout) || (mask_bits && !aligned16(mask_bits))) return CSSAR_ERR_ALIGNMENT;
  const int v = validate_ita(pl, prm);
  if (v != CSSAR_OK) return v;
  if (!pl->U) return CSSAR_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  pl->iters_done = prm->iters;
  if (pl->multi) {                              // this rank's row slabs; NCCL transposes
    Ranks R{&pl, 1};
    const int rc = ita_multi(R, &Y, &mask_bits, *prm, &X_inout, log_host, s, &pl->gexec, &pl->gkey, &pl->ghave);
    if (rc == CSSAR_OK && pl->comm && nccl().asyncError) {     // failure detection
      ncclResult_t ae = ncclSuccess;
      if (nccl().asyncError(pl->comm, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress))
        return CSSAR_ERR_NCCL;
    }
    return rc;
  }
  const float sigma_fixed = prm->rule == CSSAR_RULE_FIXED_LAMBDA ? (float)fixed_sigma(*prm) : 0.f;
  CUDA_TRY(launch_init_state(pl->d_st, pl->d_hist, pl->d_hist_full, prm->thr, sigma_fixed, s));
  const bool prof = (prm->flags & CSSAR_FLAG_PROFILE_STAGES) != 0;
  const bool tol = prm->tol > 0.0;
  // sparse-state schedule (NEXT-3, CSSAR_FLAG_SPARSE_STATE): k-rule, fixed step, no tolerance
  // stop, cluster azimuth shapes; iteration 0 (arbitrary X_0) runs dense and its b_0 seeds the list
  const bool ss = pl->ss_ok && prm->rule == CSSAR_RULE_KSPARSE && !(prm->flags & CSSAR_FLAG_ADAPTIVE_MU) && !tol &&
                  (prm->flags & CSSAR_FLAG_SPARSE_STATE) && prm->iters >= 2;
  // fixed-lambda fused schedule (CSSAR_FLAG_FUSE_LAMBDA: S5 + next S1 in one sweep, 88.125
  // B/sample) for the fixed-lambda rule with a fixed step and no tolerance stop
  const bool fuse = prm->rule == CSSAR_RULE_FIXED_LAMBDA && !(prm->flags & CSSAR_FLAG_ADAPTIVE_MU) && !tol &&
                    (prm->flags & CSSAR_FLAG_FUSE_LAMBDA);
  if (ss) {
    for (int l = 0; l < 2; ++l)
      CUDA_TRY(cudaMemsetAsync(pl->ss.cnt[l], 0, sizeof(uint32_t) * (size_t)pl->ss.npan, s));
    CUDA_TRY(launch_ss_set(pl->d_st, pl->ss.cnt[0], pl->ss.cnt[1], pl->ss.npan, s));
  }
  // sparse state after the dense iteration 0: the list from b_0 (the select has set sigma_0)
  auto ss_seed = [&]() -> int {
    CUDA_TRY(launch_ss_rebuild((const float2*)X_inout, (int)pl->p.n_az, (int)pl->p.n_rg, pl->ss, pl->d_st, 1, s));
    return CSSAR_OK;
  };
  if (tol) {                                   // X_0 = E(b; sigma_init) = X_inout
    if (!pl->d_conv) {
      pl->conv_blocks = 4 * pl->sm_count;
      CUDA_TRY(cudaMalloc(&pl->d_conv, sizeof(double2) * pl->conv_blocks));
      CUDA_TRY(cudaMallocHost(&pl->h_conv, sizeof(double2) * pl->conv_blocks));
    }
    CUDA_TRY(cudaMemcpyAsync(pl->Xk, X_inout, sizeof(float2) * (size_t)pl->n, cudaMemcpyDeviceToDevice, s));
  }
  // tolerance stop after update `it`: X_(it+1) = E(b_it; sigma_it) against the kept X_it
  auto converged = [&](int it, bool& stop) -> int {
    stop = false;
    if (!tol) return CSSAR_OK;
    CUDA_TRY(launch_conv_check((const float2*)X_inout, pl->Xk, pl->n, pl->d_st, prm->thr, pl->d_conv,
                               pl->conv_blocks, s));
    CUDA_TRY(cudaMemcpyAsync(pl->h_conv, pl->d_conv, sizeof(double2) * pl->conv_blocks, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    double d2 = 0.0, x2 = 0.0;
    for (int i = 0; i < pl->conv_blocks; ++i) { d2 += pl->h_conv[i].x; x2 += pl->h_conv[i].y; }
    if (std::sqrt(d2) <= prm->tol * std::sqrt(x2)) { stop = true; pl->iters_done = it + 1; }
    return CSSAR_OK;
  };
  if (prof) {
    for (int i = 0; i < 6; ++i) pl->stage_ms[i] = 0.0;
    pl->stage_iters = 0;
    for (int it = 0; it < prm->iters; ++it) {
      int rc = enqueue_iteration(pl, Y, mask_bits, *prm, X_inout, s, true, ss && it > 0, fuse, !fuse || it == 0);
      if (rc != CSSAR_OK) return rc;
      if (ss && it == 0 && (rc = ss_seed()) != CSSAR_OK) return rc;
      CUDA_TRY(cudaEventSynchronize(pl->ev[6]));
      for (int i = 0; i < 6; ++i) {
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, pl->ev[i], pl->ev[i + 1]));
        pl->stage_ms[i] += ms;
      }
      pl->stage_iters += 1;
      bool stop = false;
      rc = converged(it, stop);
      if (rc != CSSAR_OK) return rc;
      if (stop) break;
    }
  } else if (prm->iters > 0) {
    int first = 0;
    if (ss) {                                  // iteration 0: dense, outside the graph
      int rc = enqueue_iteration(pl, Y, mask_bits, *prm, X_inout, s);
      if (rc != CSSAR_OK) return rc;
      if ((rc = ss_seed()) != CSSAR_OK) return rc;
      first = 1;
    } else if (fuse) {                         // iteration 0 with its S1, outside the graph
      int rc = enqueue_iteration(pl, Y, mask_bits, *prm, X_inout, s, false, false, true, true);
      if (rc != CSSAR_OK) return rc;
      bool stop = false;
      if ((rc = converged(0, stop)) != CSSAR_OK) return rc;
      first = 1;
    }
    GraphKey key{Y, mask_bits, X_inout, prm->thr, prm->rule, prm->rule == CSSAR_RULE_KSPARSE ? prm->k : 0,
                 prm->lambda, prm->mu,
                 (prm->flags & CSSAR_FLAG_ADAPTIVE_MU) | (ss ? CSSAR_FLAG_SPARSE_STATE << 8 : 0) | (fuse ? 1 << 20 : 0)};
    if (!pl->ghave || !(pl->gkey == key)) {
      if (pl->gexec) { cudaGraphExecDestroy(pl->gexec); pl->gexec = nullptr; }
      pl->ghave = false;
      cudaGraph_t g = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(pl->cap_stream, cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_iteration(pl, Y, mask_bits, *prm, X_inout, pl->cap_stream, false, ss, fuse, !fuse);
      cudaError_t ec = cudaStreamEndCapture(pl->cap_stream, &g);
      if (rc != CSSAR_OK) { if (g) cudaGraphDestroy(g); return rc; }
      CUDA_TRY(ec);
      cudaError_t ei = cudaGraphInstantiate(&pl->gexec, g, 0);
      cudaGraphDestroy(g);
      CUDA_TRY(ei);
      pl->gkey = key;
      pl->ghave = true;
    }
    for (int it = first; it < prm->iters; ++it) {
      CUDA_TRY(cudaGraphLaunch(pl->gexec, s));
      bool stop = false;
      const int rc = converged(it, stop);
      if (rc != CSSAR_OK) return rc;
      if (stop) break;
    }
  }
  if (ss)                                      // X_I from the last list
    CUDA_TRY(launch_ss_finalize((float2*)X_inout, (int)pl->p.n_az, (int)pl->p.n_rg, pl->ss, prm->thr, pl->d_st, s));
  else
    CUDA_TRY(launch_finalize((float2*)X_inout, pl->n, prm->thr, pl->d_st, s));
  CUDA_TRY(note_solve_end(pl, s));
  if (log_host) {
    const int nl = pl->iters_done;
    std::vector<IterLogDev> tmp((size_t)nl);
    SelState st;
    if (nl > 0)
      CUDA_TRY(cudaMemcpyAsync(tmp.data(), pl->d_log, sizeof(IterLogDev) * nl, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&st, pl->d_st, sizeof(SelState), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int i = 0; i < nl; ++i) {
      log_host[i].sigma = tmp[i].sigma;
      log_host[i].lambda = tmp[i].lam;
      log_host[i].support = tmp[i].support;
      log_host[i].resid2 = tmp[i].resid2;
      log_host[i].mu = tmp[i].mu;
      log_host[i].gap = tmp[i].gap;
      log_host[i].gap_exact = tmp[i].gap_exact;
    }
    if (st.nonfinite) return CSSAR_ERR_NONFINITE;
  }
  return CSSAR_OK;
}

int cssar_plan_set_pulse(cssar_plan pl, const void* pulse_host, int64_t len) {
  if (!pl || pl->p.op != CSSAR_OP_RDA) return CSSAR_ERR_BAD_PLAN;
  const long long N = pl->p.n_rg;
  if (len < 0 || len > N || (len > 0 && !pulse_host)) return CSSAR_ERR_INVALID_PARAMS;
  if (pl->gexec) { cudaGraphExecDestroy(pl->gexec); pl->gexec = nullptr; }
  pl->ghave = false;
  if (len == 0) {
    CUDA_TRY(cudaFree(pl->d_hrange));
    pl->d_hrange = nullptr;
    return CSSAR_OK;
  }
  // H(f_l) = sum_m s_m exp(-j 2 pi l' (m - (L-1)/2) / N) / sqrt(sum |s_m|^2), l' the signed bin:
  // the phase l' (2m - L + 1) / (2N) cycles is reduced exactly in integers before the sincos
  const float* sp = static_cast<const float*>(pulse_host);
  long double e = 0.0L;
  for (long long m = 0; m < len; ++m) e += (long double)sp[2 * m] * sp[2 * m] + (long double)sp[2 * m + 1] * sp[2 * m + 1];
  if (!(e > 0.0L) || !std::isfinite((double)e)) return CSSAR_ERR_INVALID_PARAMS;
  const long double nrm = 1.0L / sqrtl(e);
  const long long twoN = 2 * N;
  std::vector<float2> H((size_t)N);
  for (long long l = 0; l < N; ++l) {
    const long long ls = l < N / 2 ? l : l - N;
    long double re = 0.0L, im = 0.0L;
    for (long long m = 0; m < len; ++m) {
      long long k = (ls * (2 * m - len + 1)) % twoN;
      if (k < 0) k += twoN;
      const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)k / (long double)twoN;
      const long double c = cosl(ang), sn = sinl(ang);
      re += sp[2 * m] * c - sp[2 * m + 1] * sn;
      im += sp[2 * m] * sn + sp[2 * m + 1] * c;
    }
    H[(size_t)l] = float2{(float)(re * nrm), (float)(im * nrm)};
  }
  if (!pl->d_hrange) CUDA_TRY(cudaMalloc(&pl->d_hrange, sizeof(float2) * (size_t)N));
  CUDA_TRY(cudaMemcpy(pl->d_hrange, H.data(), sizeof(float2) * (size_t)N, cudaMemcpyHostToDevice));
  return CSSAR_OK;
}

int cssar_ita_status(cssar_plan pl) {
  if (!pl) return CSSAR_ERR_BAD_PLAN;
  if (!pl->solve_pending) return CSSAR_OK;
  CUDA_TRY(cudaEventSynchronize(pl->ev_solve));
  if (pl->h_nonfinite[1]) return CSSAR_ERR_NCCL;          // a peer never reached a flag barrier
  return pl->h_nonfinite[0] ? CSSAR_ERR_NONFINITE : CSSAR_OK;
}

int cssar_ita_iters_done(cssar_plan pl, int32_t* iters_out) {
  if (!pl || !iters_out) return CSSAR_ERR_BAD_PLAN;
  *iters_out = pl->iters_done;
  return CSSAR_OK;
}

int cssar_pack_mask(const uint8_t* mask_u8, uint32_t* mask_bits, int64_t rows, int64_t cols, void* stream) {
  if (!aligned16(mask_u8) || !aligned16(mask_bits)) return CSSAR_ERR_ALIGNMENT;
  if (rows < 1 || cols < 32 || (cols % 32) != 0) return CSSAR_ERR_UNSUPPORTED_SIZE;
  CUDA_TRY(launch_pack_mask(mask_u8, mask_bits, rows, cols, (cudaStream_t)stream));
  return CSSAR_OK;
}

int cssar_debug_range_sweep(cssar_plan pl, void* U, int gbody, void* stream) {
  if (!pl || pl->multi) return CSSAR_ERR_BAD_PLAN;
  if (!aligned16(U)) return CSSAR_ERR_ALIGNMENT;
  RgArgs r{(float2*)U, pl->d_coef, 0, pl->d_rg_tab};
  r.rcmc = pl->d_rcmc;
  r.hrange = pl->d_hrange;
  CUDA_TRY(launch_rg_sweep(pl->log_nrg, gbody != 0, (int)pl->p.n_az, r, (cudaStream_t)stream));
  return CSSAR_OK;
}

int cssar_debug_az_fft(cssar_plan pl, const void* in, void* out, int dir, void* stream) {
  if (!pl || pl->multi) return CSSAR_ERR_BAD_PLAN;
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
  if (!pl || pl->multi) return CSSAR_ERR_BAD_PLAN;
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

int cssar_debug_ipc_export(const void* dev_ptr, void* rec_out) {
  if (!dev_ptr || !rec_out) return CSSAR_ERR_BAD_PLAN;
  IpcRec r{};
  if (ipc_export(dev_ptr, &r) != 0) return CSSAR_ERR_CUDA;
  std::memcpy(rec_out, &r, sizeof(r));
  return CSSAR_OK;
}

int cssar_debug_ipc_open(const void* rec, void** base_out, void** ptr_out) {
  if (!rec || !base_out || !ptr_out) return CSSAR_ERR_BAD_PLAN;
  IpcRec r;
  std::memcpy(&r, rec, sizeof(r));
  return ipc_open(r, base_out, ptr_out) == 0 ? CSSAR_OK : CSSAR_ERR_CUDA;
}

int cssar_debug_ipc_close(void* base) {
  if (!base) return CSSAR_ERR_BAD_PLAN;
  CUDA_TRY(cudaIpcCloseMemHandle(base));
  return CSSAR_OK;
}

int cssar_debug_peer_store(void* dst, uint32_t pattern, int64_t n_words, void* stream) {
  if (!dst || n_words < 0) return CSSAR_ERR_BAD_PLAN;
  CUDA_TRY(launch_peer_store(static_cast<uint32_t*>(dst), pattern, (long long)n_words, (cudaStream_t)stream));
  return CSSAR_OK;
}

int cssar_group_debug_barrier(cssar_group g, int32_t rounds, void* stream) {
  if (!g || g->pl.empty() || rounds < 0) return CSSAR_ERR_BAD_PLAN;
  const int P = (int)g->pl.size();
  PeerSlots ps{};
  EpochPtrs ep{};
  for (int r = 0; r < P; ++r) {
    cssar_plan pl = g->pl[(size_t)r];
    if (!pl->sxl) return CSSAR_ERR_WORKSPACE;
    ps.slots[r] = reinterpret_cast<uint32_t*>(pl->sxl + kBarSlotOff);
    ep.p[r] = pl->d_bar + 1;
  }
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t* err = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(g->pl[0]->d_st) + offsetof(SelState, sync_error));
  for (int r = 0; r < P; ++r) {
    cssar_plan pl = g->pl[(size_t)r];
    CUDA_TRY(cudaMemsetAsync(pl->sxl + kBarSlotOff, 0, 16 * sizeof(uint32_t), s));
    CUDA_TRY(cudaMemsetAsync(pl->d_bar, 0, 16, s));
  }
  CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(uint32_t), s));
  CUDA_TRY(launch_flag_barrier_group(P, ps, ep, rounds, err, s));
  uint32_t e = 0, epoch0 = 0;
  CUDA_TRY(cudaMemcpyAsync(&e, err, sizeof(e), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(&epoch0, g->pl[0]->d_bar + 1, sizeof(epoch0), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (e || epoch0 != (uint32_t)rounds) return CSSAR_ERR_NCCL;
  return CSSAR_OK;
}

int cssar_debug_graph_info(cssar_plan pl, int32_t* out) {
  if (!pl || !out) return CSSAR_ERR_BAD_PLAN;
  *out = pl->cond_used ? 1 : 0;
  return CSSAR_OK;
}

int cssar_group_debug_graph_info(cssar_group g, int32_t* out) {
  if (!g || !out || g->pl.empty()) return CSSAR_ERR_BAD_PLAN;
  *out = g->pl[0]->cond_used ? 1 : 0;
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
