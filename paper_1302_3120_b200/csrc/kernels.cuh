// Kernel declarations and device-side shared structures for libcssar.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>
#include "common.cuh"

namespace cssar {

// Per-Doppler-row CSA phase coefficients (u64 fixed-point cycles), DESIGN.md "Phase generation".
//   q[0] = Phi1 (chirp scaling)            in u = j - n_rg/2
//   q[1] = Phi2 (range compr. + bulk RCMC) in signed range-frequency bin l'
//   q[2] = Phi3 (azimuth compr. + residual) in u = j - n_rg/2
struct RowCoef { Quad q[3]; };

enum Thr : int { THR_SOFT = 1, THR_HALF = 2, THR_HARD = 3, THR_TWOTHIRDS = 4 };
enum Rule : int { RULE_K = 1, RULE_LAMBDA = 2 };

constexpr int HIST_BITS = 11;                  // top bits of the 31-bit |b|^2 pattern
constexpr int HIST_BINS = 1 << HIST_BITS;      // 2048 bins, 8 per octave of |b|^2
constexpr int HIST_SHIFT = 31 - HIST_BITS;     // 20
// the |b|^2 histogram buffer carries two flag words after the bins (summed by the multi-GPU
// all-reduce together with the bins): [HIST_BINS] candidate overflow, [HIST_BINS+1] non-finite
constexpr int HIST_WORDS = HIST_BINS + 2;
constexpr int FLOOR_MARGIN = 8;                // bins below the last sigma^2 bin still counted
constexpr int CAND_MARGIN = 2;                 // candidate window half-width (bins)

// Device-resident solver state (one per plan); no host round trip inside the loop.
struct SelState {
  uint32_t sigma2_bits;     // threshold sigma^2 (fp32 bit pattern) used by E(.)
  float sigma;              // sqrt(sigma^2) (shrink amount)
  float sigma_fixed;        // fixed-lambda rule: sigma = lambda mu (soft) / half jump point
  uint32_t sigma2_fixed_bits;
  int32_t floor_bin;        // TAIL histograms only bins >= floor_bin
  int32_t cand_lo, cand_hi; // TAIL writes candidates with bin in [lo, hi]
  uint32_t cand_count;
  uint32_t cand_overflow;
  int32_t need_full;        // 1: coarse select failed -> full-histogram fallback
  int32_t target_bin;
  uint32_t target_rank;     // 0-based rank from the top inside target_bin
  uint64_t above_count;     // # elements in bins above target_bin
  int32_t iter;             // iteration counter (log index)
  uint32_t nonfinite;
  uint32_t sync_error;      // multi-GPU flag barrier timed out (a peer never arrived)
  double resid2;            // ||Theta(Y - G X)||^2 of the current iteration
  unsigned long long support_fixed;
  int32_t fallbacks;        // # iterations that needed the full-histogram fallback
  uint32_t fine_prefix;     // split fine select (multi-GPU): matched high bits so far
  uint32_t fine_rank;       //   rank inside the current prefix
  unsigned long long fine_abv;  //   elements strictly above the prefix
  // adaptive step (NEXT-1, eq. 27): mu_i = mu_num / mu_den, 0 = fixed mu (prm.mu)
  double mu_num;            // ||dX_k||^2 (AZ_GRAD)
  double mu_den;            // ||Theta G(dX_k)||^2 (AZ_NORM)
  float mu;                 // mu_i of the current iteration (adaptive runs), else 0
  float lambda;             // fixed-lambda rule: lambda (adaptive runs recompute sigma = f(lambda mu_i))
  // sparse-state schedule: counters of the list the next S5 writes are zeroed by the select;
  // ss_fell records that this iteration's select needed the dense fallback (list rebuild)
  uint32_t* ss_cnt[2];
  int32_t ss_npan;
  int32_t ss_fell;
};

struct IterLogDev { float sigma; float lam; long long support; double resid2; float mu; float gap; int gap_exact; };

// sparse-state schedule (NEXT-3): one list entry: b at (row, column col0 + w of the panel)
struct SsEntry { uint32_t row; uint32_t w; float2 v; };
// the two state lists (iteration parity): panel p's entries at ent[l][p * capp ...], count cnt[l][p]
struct SsLists {
  SsEntry* ent[2];
  uint32_t* cnt[2];
  uint32_t capp;            // entries per panel (= n_az * W: a panel never overflows)
  int npan;
  int W;
};

struct AzArgs {
  const float2* in;
  float2* out;
  const float2* Y;
  const uint32_t* mask;     // bit-packed, mask_words per row; nullptr = all ones
  float2* b;                // TAIL / THR: state array
  SelState* st;
  uint32_t* hist;           // HIST_BINS
  uint32_t* cand;           // candidate |b|^2 patterns
  uint32_t cand_cap;
  int n_rg;
  int mask_words;
  int thr;
  int rule;
  float mu;
  float scale;              // 1/sqrt(n_az)
  float oscale;             // factor on outputs that feed a range sweep: scale/n_rg (range IFFT norm folded in)
  const float2* tw;         // precomputed inter-pass twiddle tables of the az engine (global)
  // output destinations (multi-GPU fused transpose): output line `row` of the
  // column slab is stored at dst[row >> dlog_nrow] + ((drank << dlog_nrow) + (row & (nrow-1))) *
  // n_rg + col, i.e. straight into block `drank` of rank q's blocked row slab (peer memory).
  // dst[0] == nullptr: plain `out` (launch_az fills dst[0] = out, dlog_nrow = log2 n_az).
  float2* dst[16];
  int dlog_nrow;
  int drank;
  int dsingle;              // set by launch_az: one destination (dst[0] + row n_rg + col)
  float2* D;                // AZ_GRAD: dense gradient dX (for the elementwise step)
  float lambda;             // fixed-lambda rule with the adaptive step (sigma_i = f(lambda mu_i))
  // deterministic squared-norm reductions (RESID / GRAD / NORM): per-CTA partials in slot
  // arrays [3][kRedSlots] reduced in block order by the last CTA (ticket counter per mode)
  double* red_part;
  uint32_t* red_ticket;
  SsLists ss;               // sparse-state modes
};
constexpr int kRedSlots = 8192;   // >= the grid of every reducing azimuth launch

struct RgArgs {
  float2* data;
  const RowCoef* coef;
  int row_base;             // global Doppler row of data row 0
  const float2* tab;        // [exp(2 pi i h/256), h < 256 | inter-pass twiddle tables] (global)
  // blocked row-slab layout of the multi-GPU path: sample j of local row r lives
  // at (j >> log_w) * blk + r * 2^log_w + (j & (2^log_w - 1)), i.e. [peer][row][w] blocks as
  // received from the all-to-all; log_w = log2(n_rg), blk = 0 is the plain row-major layout
  int log_w;
  long long blk;
  // blocked layout only: if dst[0] != nullptr the output goes to the column slabs of the
  // ranks instead of in place: sample j of local row r -> dst[j >> log_w] +
  // ((drank << dlog_nrow) + r) * 2^log_w + (j & (2^log_w - 1))   (peer memory, fused transpose)
  float2* dst[16];
  int dlog_nrow;
  int drank;
  // RDA operator pair (NEXT-2; cssar_sar_params::op = CSSAR_OP_RDA): per global Doppler row
  // (alpha, s0) of the RCMC migration d(j) = s0 + alpha (j - n_rg/2) range cells; nullptr = CSA
  const float2* rcmc;
  // RDA with a recorded pulse (NEXT-4): G's range filter H(f_l) in fftfreq order (M uses
  // conj H) instead of the chirp P_tau quadratic q[1]; nullptr = chirp
  const float2* hrange;
  // sparse-X' schedule (multi-GPU): local row rr is global Doppler bin row_base + rr*row_step
  // (0 = 1), and the fused destination slabs are 2^dlog_w gates wide (0 = log_w)
  int row_step;
  int dlog_w;
  // persistent launch: total rows (the CTAs loop over row blocks); 0 = one block per CTA
  int nrows;
};

enum AzMode : int {
  AZ_FWD_PLAIN = 0,   // F_eta x
  AZ_FWD_MASK = 1,    // F_eta (Theta o r)
  AZ_FWD_THR = 2,     // F_eta E(b; sigma)                          (S1)
  AZ_INV_PLAIN = 3,   // F_eta^-1 u
  AZ_INV_MASK = 4,    // Theta o F_eta^-1 u
  AZ_RESID = 5,       // F_eta Theta o (Y - F_eta^-1 u)               (S3)
  AZ_TAIL = 6,        // b <- E(b; sigma) + mu F_eta^-1 u, histogram  (S5)
  AZ_GRAD = 7,        // adaptive step: dX = F_eta^-1 u -> D; F_eta (dX on supp X_i); ||dX_k||^2
  AZ_NORM = 8,        // adaptive step: ||Theta o F_eta^-1 u||^2 only
  // sparse-state schedule (NEXT-3; world 1, k-rule): the state is a per-panel list of the b
  // entries above the candidate window's floor instead of a dense b array
  AZ_FWD_SS = 9,      // S1: X = E(b; sigma) from the list, scattered into the stage; F_eta
  AZ_TAIL_SS = 10,    // S5: X_i from the list; b_i = X_i + mu dX -> histogram, candidates, new list
  AZ_TAIL_SSD = 11,   // S5 re-run after a select fallback: dense b_i into a.b (early exit otherwise)
  // fixed-lambda rule (sigma known in advance, eq. 7): S5 fused with the next iteration's S1
  AZ_FUSE = 12,       // F_eta^-1 u -> b_i = E(b_{i-1}) + mu dX (stored), X_{i+1} = E(b_i; sigma) -> F_eta
};
constexpr bool az_is_res(int m) { return m == AZ_RESID || m == AZ_GRAD || m == AZ_FUSE; }   // two transforms
constexpr bool az_is_thr(int m) { return m == AZ_FWD_THR || m == AZ_FWD_SS; }
constexpr bool az_is_tail(int m) { return m == AZ_TAIL || m == AZ_TAIL_SS || m == AZ_TAIL_SSD; }
constexpr bool az_is_ss(int m) { return m == AZ_FWD_SS || m == AZ_TAIL_SS || m == AZ_TAIL_SSD; }


// programmatic dependent launch of the ITA-loop kernels (opt-in: CSSAR_PDL=1; measured neutral
// in the replayed graph at c3)
bool pdl_enabled();
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// host-side launchers (kernels.cu)
cudaError_t launch_rg_sweep(int log_nrg, bool gbody, int n_rows, const RgArgs& a, cudaStream_t s);   // blocked iff a.blk != 0
cudaError_t launch_az(int log_naz, int mode, int n_rg_local, const AzArgs& a, cudaStream_t s);
cudaError_t launch_select(int n_threads_hint, float2* b, long long n, long long k, int rule, int thr, float mu,
                          SelState* st, uint32_t* hist, uint32_t* hist_full, uint32_t* cand, uint32_t cand_cap,
                          IterLogDev* log, int log_cap, cudaStream_t s);
// the k-rule select after sel_coarse (fallback kernels + fine select)
cudaError_t launch_select_rest(int sm_count, float2* b, long long n, long long k, int thr, float mu, SelState* st,
                               uint32_t* hist, uint32_t* hist_full, uint32_t* cand, uint32_t cand_cap, IterLogDev* log,
                               int log_cap, cudaStream_t s);
// multi-GPU k-rule select, split around the all-reduces; world == 1 uses launch_select
enum SelPart : int {
  SEL_COARSE = 0,     // global |b|^2 histogram (+ flags) -> target bin or fallback decision
  SEL_FB_HIST = 1,    // (fallback only) local full histogram -> hist_full
  SEL_FB_PICK = 2,    // (fallback only) target bin from the global hist_full, collect candidates
  SEL_FINE0_HIST = 3, // local 1024-bin histogram of the candidates, bits [19:10]
  SEL_FINE0_FIND = 4, // global level-0 counts -> prefix; then local level-1 histogram, bits [9:0]
  SEL_FINE1_FIND = 5, // global level-1 counts -> sigma^2, log entry, next window
};
cudaError_t launch_select_part(int part, int sm_count, float2* b, long long n, long long k, int thr, float mu,
                               SelState* st, uint32_t* hist, uint32_t* hist_full, uint32_t* cand,
                               uint32_t cand_cap, uint32_t* lvl, IterLogDev* log, int log_cap, cudaStream_t s);
cudaError_t launch_lambda_step(SelState* st, int thr, float mu, IterLogDev* log, int log_cap, cudaStream_t s);
// adaptive step: mu_i = mu_num/mu_den (1 if either is 0); b <- E(b; sigma_{i-1}) + mu_i D; histogram /
// candidates / fixed-lambda support exactly as the tail kernel
cudaError_t launch_adaptive_step(const AzArgs& a, long long n, int sm_count, cudaStream_t s);
// sparse-X' schedule (multi-GPU; sparse.cu)
struct SxEntry { int row, col; float2 v; };          // global row, global gate, X value
struct SxLists {
  const SxEntry* list[16];                            // every rank's list (peer memory)
  const uint32_t* count[16];                          // every rank's entry count
  uint32_t cap;
  int world;
};
cudaError_t launch_sx_compact(const float2* b, long long n, int log_ncol, int col0, const SelState* st, int thr,
                              SxEntry* list, uint32_t* count, uint32_t cap, int sm_count, cudaStream_t s);
cudaError_t launch_sx_fold(const SxLists& L, int p, int log_n, int m, int n_rg, float2* F, int sm_count,
                           cudaStream_t s);
// multi-GPU peer plumbing (peer.cu)
struct PeerSlots { uint32_t* slots[16]; };            // every rank's barrier slot array (peer memory)
struct EpochPtrs { uint32_t* p[16]; };
struct IpcRec { cudaIpcMemHandle_t h; unsigned long long off; unsigned long long pad; };
cudaError_t launch_flag_barrier(int rank, int world, const PeerSlots& ps, uint32_t* epoch, uint32_t* err,
                                cudaStream_t s);
cudaError_t launch_flag_barrier_group(int world, const PeerSlots& ps, const EpochPtrs& ep, int rounds, uint32_t* err,
                                      cudaStream_t s);
int ipc_export(const void* p, IpcRec* rec);
int ipc_open(const IpcRec& rec, void** base_out, void** ptr_out);
cudaError_t launch_peer_store(uint32_t* dst, uint32_t pattern, long long n, cudaStream_t s);
// tolerance stop (NEXT-4): per-block (||E(b; sigma) - Xk||^2, ||Xk||^2) into part[blocks], Xk <- E(b; sigma)
cudaError_t launch_conv_check(const float2* b, float2* Xk, long long n, const SelState* st, int thr, double2* part,
                              int blocks, cudaStream_t s);
// bufs[p][i] <- sum_p bufs[p][i] for every p (single-device emulation of an all-reduce)
cudaError_t launch_group_sum(int dtype, void* const* bufs, int world, long long count, cudaStream_t s);
cudaError_t launch_init_state(SelState* st, uint32_t* hist, uint32_t* hist_full, int thr, float sigma_fixed,
                              cudaStream_t s);
cudaError_t launch_finalize(float2* b, long long n, int thr, const SelState* st, cudaStream_t s);
// sparse-state schedule (ss.cu): rebuild the list S1 reads next from the dense b of a fallback
// iteration (force = always, e.g. after the dense iteration 0); X = E(b; sigma) from the last list
cudaError_t launch_ss_rebuild(const float2* b, int n_az, int n_rg, const SsLists& L, const SelState* st, int force,
                              cudaStream_t s);
cudaError_t launch_ss_finalize(float2* X, int n_az, int n_rg, const SsLists& L, int thr, const SelState* st,
                               cudaStream_t s);
int az_panel_width(int log_naz);       // W of the head/tail cluster sweeps (0: not a cluster shape)
cudaError_t launch_ss_set(SelState* st, uint32_t* cnt0, uint32_t* cnt1, int npan, cudaStream_t s);
// precomputed SMEM tables (filled once per plan, copied into SMEM by each CTA)
size_t rg_table_count(int log_nrg);
int rg_rows_per_cta(int log_nrg);
cudaError_t rg_table_fill(int log_nrg, float2* dst, cudaStream_t s);
size_t az_table_count(int log_naz, bool resid);
cudaError_t az_table_fill(int log_naz, bool resid, float2* dst, cudaStream_t s);
cudaError_t launch_pack_mask(const uint8_t* m, uint32_t* bits, long long rows, long long cols, cudaStream_t s);

}  // namespace cssar
