/* cssar.h — C ABI of libcssar: the data-parallel hot path of fast CS-SAR imaging based on
 * approximated observation (Fang, Xu, Zhang, Hong, Wu, arXiv 1302.3120), B200 (sm_100a).
 *
 * The method (PAPER.md = P:Lnnn):
 *   Algorithm 1 / eq. 25:
 *       X^(i+1) = E_sigma( X^(i) + mu * M( Theta o (Y_s - Theta o G(X^(i))) ) )
 *   M = CSA matched-filter focusing chain (eq. 10, with the chirp-scaling
 *       algorithm named at P:L243 in place of RDA), G = M^H = M^-1 the approximated
 *       observation (eq. 11; Theorem 1), Theta the sampling mask (eq. 4,
 *       P:L81; eq. 24), E_sigma the soft (eq. 9) or q=1/2 threshold,
 *       sigma = lambda*mu from the k-sparsity rule or a fixed lambda.
 *
 * Conventions for every call:
 *   - Arrays are complex64 (interleaved fp32 re, im; 8 bytes/sample), row-major
 *     [n_az][n_rg]: row = azimuth line (or Doppler bin), column = range gate (or range-
 *     frequency bin).  Frequency axes are in FFT bin order (no fftshift).
 *   - DFTs are unitary (1/sqrt(N) per transform, "keep the throwaway consistent").
 *   - Array pointers are DEVICE pointers, 16-byte aligned, owned by the caller (the
 *     library never frees or retains them).  `stream` is a cudaStream_t (may be 0); all
 *     calls are asynchronous on it unless stated otherwise.
 *   - The mask is 1 bit per sample, row-major, LSB-first in uint32 words, each row padded
 *     to a whole number of words (n_rg/32 words per row).  mask_bits == NULL means
 *     Theta = all ones.  Y may hold garbage at unsampled positions (Theta is applied).
 *   - Return value: 0 (CSSAR_OK) or a negative CSSAR_ERR_* code; no partial side effects
 *     on argument-validation errors.
 *   - A plan is not thread-safe: one call in flight per plan.
 */
#ifndef CSSAR_H_
#define CSSAR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CSSAR_OK = 0,
  CSSAR_ERR_INVALID_PARAMS = -1,   /* non-positive rate/velocity/range, squint != 0, pulse < 2 samples */
  CSSAR_ERR_UNSUPPORTED_SIZE = -2, /* n_az, n_rg not powers of two in [128, 32768] / [128, 16384] */
  CSSAR_ERR_BAD_K = -3,            /* k-rule with k < 1 or k >= n_az*n_rg */
  CSSAR_ERR_BAD_MU = -4,           /* mu <= 0 or not finite; lambda < 0 */
  CSSAR_ERR_ALIGNMENT = -5,        /* a pointer is NULL or not 16-byte aligned */
  CSSAR_ERR_NONFINITE = -6,        /* NaN/Inf reached the iterate (reported when the log is read) */
  CSSAR_ERR_CUDA = -7,             /* a CUDA runtime call failed */
  CSSAR_ERR_WORKSPACE = -8,        /* no / too small workspace bound for cssar_ita_iterate */
  CSSAR_ERR_NCCL = -9,             /* NCCL missing or a NCCL call failed (world > 1) */
  CSSAR_ERR_BAD_PLAN = -10         /* NULL plan or world/rank combination not supported */
};

/* SAR system parameters: the fields of Table 1 used by CSA, plus the grid.
 * fc carrier [Hz], Kr range FM rate [Hz/s], Tr pulse duration [s], Fr range sampling
 * rate [Hz], prf [Hz], Vr effective velocity [m/s], R_ref scene-centre slant range [m]
 * (gate n_rg/2 <-> R_ref), squint [rad] (must be 0). */
typedef struct {
  double fc, Kr, Tr, Fr, prf, Vr, R_ref, squint;
  int64_t n_az, n_rg;
  int32_t op;       /* cssar_op: the approximated observation pair (0 = CSSAR_OP_CSA) */
} cssar_sar_params;

/* The focusing method M whose inverse is the approximated observation G = M^H:
 *   CSSAR_OP_CSA (north star): chirp scaling, M = F_eta^-1 Phi3 F_tau^-1 Phi2 F_tau Phi1 F_eta.
 *   CSSAR_OP_RDA (NEXT-2, the paper's own CSRDA, eq. 14-18, 23): range-Doppler,
 *     M = F_eta^-1 P_eta C F_tau^-1 P_tau F_tau F_eta with the 8-tap truncated-sinc RCMC C
 *     (space-variant shift R0 (1/D - 1), torus indices) and G = M^H with D = C^T.
 *     Requires (1/D_max - 1) n_rg < 1/2 at the Doppler edge (else CSSAR_ERR_INVALID_PARAMS).
 * Every call (operators, ITA, world > 1) uses the plan's pair; the sweeps are the same except
 * the range sweep, which carries the RCMC. */
typedef enum { CSSAR_OP_CSA = 1, CSSAR_OP_RDA = 2 } cssar_op;

/* thresholds E_sigma (eq. 7-9; P:L102 names q = 0, 1/2, 2/3, 1 as the analytic
 * cases): soft q = 1 (eq. 9), half q = 1/2 (the north star's two), and (NEXT-4) hard q = 0
 * and q = 2/3; all phase preserving with strict survival |b| > sigma.  Fixed-lambda jump
 * points sigma(lambda mu): lm, (54^(1/3)/4) lm^(2/3), sqrt(lm), (2/3)(3 lm^3)^(1/4). */
typedef enum {
  CSSAR_THR_SOFT = 1,
  CSSAR_THR_HALF = 2,
  CSSAR_THR_HARD = 3,
  CSSAR_THR_TWOTHIRDS = 4
} cssar_thr;
typedef enum { CSSAR_RULE_KSPARSE = 1 /* P:L320 */, CSSAR_RULE_FIXED_LAMBDA = 2 /* eq. 7 */ } cssar_rule;

/* flags: CSSAR_FLAG_PROFILE_STAGES launches the iteration body directly (no graph) with CUDA
 * events between the six steps S1..S6 on `stream`, synchronising once per iteration, and
 * accumulates per-step device time (read with cssar_stage_times). */
enum { CSSAR_FLAG_PROFILE_STAGES = 1, CSSAR_FLAG_ADAPTIVE_MU = 2, CSSAR_FLAG_SPARSE_X = 4,
       CSSAR_FLAG_PEER_TRANSPOSE = 8, CSSAR_FLAG_SPARSE_STATE = 16, CSSAR_FLAG_FUSE_LAMBDA = 32 };

/* ITA settings (Algorithm 1 "Initial": lambda, mu, I_max).  iters = number of X updates
 * (R18).  k is used by the k-rule, lambda by the fixed-lambda rule.
 * CSSAR_FLAG_ADAPTIVE_MU (world 1 only; NEXT-1): mu is ignored and every iteration uses
 * mu_i = ||dX_k||^2 / ||Theta G(dX_k)||^2, dX_k = the MF update M(Theta(Y - G X_i)) on the
 * support of X_i (eq. 27, in the normalised-IHT form of its cited source;
 * DESIGN.md R11, R20), mu_i = 1 on an empty support; the fixed-lambda rule then thresholds at
 * lambda mu_i.  Costs three more sweeps and an elementwise pass per iteration.
 * tol > 0 (world 1 only; NEXT-4): stop after the first update with
 * ||X_(i+1) - X_i||_F <= tol ||X_i||_F (iters stays the cap).  Needs the third workspace
 * array (the kept X_i); per iteration one more elementwise pass (X_(i+1) vs X_i, 24 B/sample)
 * and a host synchronisation on `stream`.  The number of updates performed is read with
 * cssar_ita_iters_done; log entries exist only for those.
 * CSSAR_FLAG_SPARSE_STATE (a request; NEXT-3; applies to world 1, k-rule, fixed mu, tol = 0,
 * n_az >= 2048, iters >= 2): from iteration 1 on the state between iterations is, per column
 * panel of the azimuth sweeps, the list of b entries at or above the select's candidate
 * window (X_i = E(b_(i-1)) is k-sparse) kept in the workspace instead of a dense b
 * in X_inout: S5 writes no dense b and S1 reads no dense b (72 instead of 96 B/sample per
 * iteration).  A select fallback re-runs S5 densely into X_inout.  Same results as the dense
 * schedule (bitwise).  Not the default: the sweeps are latency-bound, and on B200 the list
 * fills cost more than the dense b traffic they save.
 * CSSAR_FLAG_FUSE_LAMBDA (a request; fixed-lambda rule -- eq. 7: sigma = lambda mu is known
 * before the iteration's select -- fixed mu, tol = 0, world 1): S5 is fused with the next
 * iteration's S1 -- one azimuth sweep computes b_i = E(b_(i-1)) + mu dX, stores it and
 * transforms X_(i+1) = E(b_i; sigma) for the next G body (88.125 instead of 96.125 B/sample,
 * one sweep fewer).  Equal to the unfused schedule up to floating-point order (another FFT
 * factorisation).  Not the default: the fused sweep has the residual sweep's two cluster
 * exchanges and measured slower at c3 (2.47 vs 2.39 ms per iteration).
 * CSSAR_FLAG_PEER_TRANSPOSE (world > 1; a request): the fused transposes -- sweep epilogues
 * store straight into the peers' slabs through the CUDA-IPC mappings made at bind time, a
 * device flag barrier (system-scope release/acquire on slots in every rank's workspace, 20 s
 * timeout -> CSSAR_ERR_NCCL) orders the sweeps.  Without it (the default until a multi-GPU
 * run has validated peer stores) the transposes are NCCL all-to-alls.  Ignored if the peers
 * could not be mapped.
 * CSSAR_FLAG_SPARSE_X (world > 1; a request): the sparse-X' schedule where
 * it applies — k-rule, peer-memory transposes (CSSAR_FLAG_PEER_TRANSPOSE), k <= n_az n_rg / (8 world),
 * n_az / world >= 128; otherwise the dense schedule runs.  From iteration 1 on, S1 and its
 * transpose are replaced by a compacted X = E(b) (<= k entries of 16 B) that every rank
 * pulls from every other rank's workspace, folds into n_az/world Doppler bins (cyclic
 * distribution) and transforms locally.  Same results up to floating-point order (not
 * bitwise equal to world 1: another FFT factorisation and atomically summed folds).
 * world == 1: CSSAR_ERR_INVALID_PARAMS. */
typedef struct {
  int32_t thr;      /* cssar_thr */
  int32_t rule;     /* cssar_rule */
  int64_t k;
  double lambda;
  double mu;
  int32_t iters;
  int32_t flags;    /* CSSAR_FLAG_* bits; 0 = graph-replayed loop */
  double tol;       /* relative-change stopping tolerance; 0 = run `iters` updates */
} cssar_ita_params;

/* Per-iteration log (SPEC "SolverReport"): sigma_i = lambda_i mu_i, lambda_i,
 * support = #{|b_i| > sigma_i} (= #nonzeros of X_(i+1)), resid2 = ||Theta(Y - G X_i)||^2, mu_i,
 * and the near-tie gap g_i = (|b_i|_(k) - |b_i|_(k+1)) / |b_i|_(k+1) of the k-rule (SURVEY.md
 * 8(c).3 / 8(c).6 diagnostic; lambda rule P:L314-320): gap_exact = 1 when g_i is exact, 0 when
 * it is a lower bound (|b_i|_(k) lies above the select's candidate window), the fixed-lambda
 * rule (no order statistic: gap 0) or world > 1. */
typedef struct {
  float sigma;
  float lambda;
  int64_t support;
  double resid2;
  float mu;         /* step of the iteration (the fixed mu, or mu_i of the adaptive rule) */
  float gap;        /* g_i (exact or lower bound, see gap_exact) */
  int32_t gap_exact;
} cssar_iter_log;

typedef struct cssar_plan_s* cssar_plan;

/* Validate p, build the per-Doppler-bin CSA phase coefficient table (u64 fixed-point
 * cycles) and upload it.  Allocates only small device tables
 * (< 4 MB).  Synchronous.
 *   world == 1 (rank 0, nccl_unique_id NULL): single GPU; every call takes whole arrays.
 *   world > 1 (<= 16): multi-GPU slab partition (north star "slab-
 *     partitioned by azimuth lines"): this process is `rank` and owns the row slab of
 *     n_az/world consecutive azimuth lines [rank*n_az/world, (rank+1)*n_az/world) of Y,
 *     the mask and X (row-major [n_az/world][n_rg], mask n_rg/32 words per line).
 *     nccl_unique_id: host pointer to the 128-byte ncclUniqueId from cssar_nccl_unique_id()
 *     on one rank, distributed by the caller; the plan creates its own NCCL communicator
 *     (collective call: every rank must call it; NCCL from the process's libnccl.so.2).
 *     world must divide n_az and n_rg with n_rg/world >= 128 and n_az/world a multiple of
 *     the range kernel's rows per CTA; else CSSAR_ERR_UNSUPPORTED_SIZE.  cssar_ita_iterate
 *     and the operators cssar_forward / cssar_adjoint / cssar_image take this rank's row
 *     slabs and are collective over the ranks (needs a bound workspace); the debug hooks
 *     return CSSAR_ERR_BAD_PLAN.  NCCL failures: CSSAR_ERR_NCCL. */
int cssar_plan_create(cssar_plan* out, const cssar_sar_params* p, int world, int rank,
                      const void* nccl_unique_id, void* stream);
int cssar_plan_destroy(cssar_plan plan);

/* Fill id_out (host, 128 bytes) with a fresh ncclUniqueId for cssar_plan_create(world > 1). */
int cssar_nccl_unique_id(void* id_out);

/* Bytes of device workspace cssar_ita_iterate needs: world 1: three complex64 arrays of the
 * scene size (transform buffer; adaptive-step gradient; X_i of the tolerance stop) plus a
 * candidate buffer for the exact top-k select (~24.5 B/sample), and for n_az >= 2048 the two
 * sparse-state lists (16-byte entries, room for every sample: +32 B/sample); world > 1:
 * four complex64 column-slab arrays (transposes, Y, state), the column-slab mask and the
 * candidate buffer (~32.6 B per local sample). */
int cssar_workspace_size(cssar_plan plan, size_t* bytes);
/* Bind caller-owned workspace (device, 256-byte aligned).  Kept until rebound or the
 * plan is destroyed; the caller keeps it alive.  world > 1: a collective call (every rank
 * binds): the ranks map each other's transpose buffers through CUDA IPC (peer memory over
 * NVLink) so the sweeps store their output straight into the destination ranks' slabs
 * (fused transposes); if any rank cannot map its peers, all ranks keep NCCL all-to-all
 * transposes (also forced by the environment variable CSSAR_MULTI_A2A). */
int cssar_bind_workspace(cssar_plan plan, void* ws, size_t bytes);

/* Y_out = Theta o G(X)   (A X, eq. 24).  X and Y_out may alias.  world > 1: row slabs in and
 * out, collective (column-slab azimuth sweeps, two all-to-all transposes around the range
 * sweep; the workspace must be bound), bitwise equal to world 1. */
int cssar_forward(cssar_plan plan, const void* X, const uint32_t* mask_bits, void* Y_out, void* stream);
/* X_out = M(Theta o R)   (A^H R).  R and X_out may alias. */
int cssar_adjoint(cssar_plan plan, const void* R, const uint32_t* mask_bits, void* X_out, void* stream);
/* X_out = M(Theta o Y): the conventional matched-filter (CSA) image of eq. 10. */
int cssar_image(cssar_plan plan, const void* Y, const uint32_t* mask_bits, void* X_out, void* stream);

/* Run `iters` ITA iterations (Algorithm 1 / eq. 25) starting from X_inout (zeros for
 * Algorithm 1's X^(0) = 0; any X for resume).  On return X_inout = X^(iters).  Needs a
 * bound workspace.  log_host (host array of >= iters entries) may be NULL; when given,
 * the call copies the log back and SYNCHRONISES the stream, and reports
 * CSSAR_ERR_NONFINITE if NaN/Inf were seen.  The iteration body is replayed as a CUDA
 * graph captured once per (pointers, params) and cached in the plan.
 * world > 1: Y, mask_bits, X_inout are this rank's row slabs; collective over the ranks
 * (all must call with the same prm).  Per iteration: 4 transposes between row slabs (range
 * sweeps) and column slabs (azimuth sweeps) — fused into the sweeps' epilogues as peer
 * stores plus a one-word all-reduce barrier, or NCCL all-to-alls — and all-reduces of the
 * residual norm and of the select histograms; the log is global.  PROFILE_STAGES is
 * ignored.  Results are bitwise identical to world 1 (same kernels, same global indices;
 * only the floating-point order of the logged residual norm differs). */
int cssar_ita_iterate(cssar_plan plan, const void* Y, const uint32_t* mask_bits,
                      const cssar_ita_params* prm, void* X_inout, cssar_iter_log* log_host,
                      void* stream);
/* RDA plans (CSSAR_OP_RDA) only — non-chirp pulses (NEXT-4: "replacing P_tau* with
 * the transmitted pulse, which is always recorded"): pulse_host = len complex64 samples
 * (interleaved re, im; host) of the recorded transmitted pulse at range times
 * (m - (len-1)/2)/F_r, 1 <= len <= n_rg.  G's range filter becomes its spectrum
 * H(f_l) = sum_m s_m exp(-j 2 pi f_l tau_m) / sqrt(sum_m |s_m|^2) (signed bins, unit mean |H|^2)
 * and M's the matched filter conj(H), in place of the chirp P_tau.  len = 0 restores the chirp.
 * Synchronous (host DFT in long double, O(n_rg len)); drops the cached iteration graph.
 * Errors: CSSAR_ERR_BAD_PLAN (NULL or a CSA plan), CSSAR_ERR_INVALID_PARAMS (len out of range,
 * zero-energy or non-finite pulse). */
int cssar_plan_set_pulse(cssar_plan plan, const void* pulse_host, int64_t len);

/* Number of X updates the last cssar_ita_iterate on this plan performed (prm->iters unless
 * the tolerance stop fired). */
int cssar_ita_iters_done(cssar_plan plan, int32_t* iters_out);

/* Outcome of the last cssar_ita_iterate on this plan: waits (host) for that call's work on its
 * stream and returns CSSAR_ERR_NONFINITE if a NaN/Inf entered the iterate, else
 * CSSAR_OK.  cssar_ita_iterate itself reports it only when it synchronises for log_host. */
int cssar_ita_status(cssar_plan plan);

/* mask_u8 (device, rows*cols bytes, nonzero = sampled) -> bit-packed mask (rows*cols/32
 * words); cols must be a multiple of 32. */
int cssar_pack_mask(const uint8_t* mask_u8, uint32_t* mask_bits, int64_t rows, int64_t cols, void* stream);

const char* cssar_error_string(int code);

/* ---- single-device emulation of a multi-GPU group (tests of the world > 1 path) ------
 * A group holds `world` rank plans on the current device and runs exactly the kernels and
 * schedule of cssar_ita_iterate(world > 1), with the all-to-alls done by device copies
 * and the all-reduces by a summing kernel, all ranks' work serialised on `stream`.
 * Y[r], mask_bits[r] (all NULL or none), X_inout[r] are rank r's row slabs. */
typedef struct cssar_group_s* cssar_group;
int cssar_group_create(cssar_group* out, const cssar_sar_params* p, int world, void* stream);
int cssar_group_destroy(cssar_group group);
int cssar_group_workspace_size(cssar_group group, size_t* bytes_per_rank);
int cssar_group_bind_workspace(cssar_group group, int rank, void* ws, size_t bytes);
int cssar_group_ita_iterate(cssar_group group, const void* const* Y, const uint32_t* const* mask_bits,
                            const cssar_ita_params* prm, void* const* X_inout, cssar_iter_log* log_host,
                            void* stream);
/* The single-device emulation of cssar_forward (forward = 1) / cssar_adjoint = cssar_image
 * (forward = 0) on world > 1 row slabs: in, mask_bits (entries NULL = all ones), out are
 * arrays of `world` device pointers. */
int cssar_group_operator(cssar_group g, int forward, const void* const* in, const uint32_t* const* mask_bits,
                         void* const* out, void* stream);

/* ---- test hooks (parity of single sweeps / the select; not needed by users) ---------- */
/* One range sweep in place on a (Doppler, range-time) array: gbody=1 -> Phi3* F Phi2* F^-1
 * Phi1* (G body), gbody=0 -> Phi1 F Phi2 F^-1 Phi3 (M body), with UNNORMALISED transforms:
 * the result is n_rg times the unitary chain (the operator chain folds the 1/n_rg into the
 * preceding azimuth sweep's output scale). */
int cssar_debug_range_sweep(cssar_plan plan, void* U, int gbody, void* stream);
/* Unitary azimuth DFT of every column: dir = -1 forward, +1 inverse.  in/out may alias. */
int cssar_debug_az_fft(cssar_plan plan, const void* in, void* out, int dir, void* stream);
/* k-rule select on an arbitrary complex64 array b (n = n_az*n_rg): writes the fp32 bit
 * pattern of the (k+1)-th largest |b|^2 (explicitly rounded re*re + im*im) and the number
 * of entries strictly above it.  Synchronous.  Needs a bound workspace. */
int cssar_debug_select(cssar_plan plan, const void* b, int64_t k, uint32_t* sigma2_bits_out,
                       int64_t* above_out, void* stream);
/* Per-step device time accumulated by the last CSSAR_FLAG_PROFILE_STAGES run: ms_out[6] =
 * total milliseconds of S1 (az head), S2 (G range body), S3 (az residual), S4 (M range
 * body), S5 (az tail), S6 (select); iters_out = iterations measured.  Host-only call. */
int cssar_stage_times(cssar_plan plan, double* ms_out, int32_t* iters_out);

/* Number of full-histogram fallbacks taken by the last cssar_ita_iterate (synchronous). */
int cssar_debug_fallbacks(cssar_plan plan, int32_t* out, void* stream);

/* Multi-GPU select: *info_out = 1 when the cached iteration graph of a world > 1
 * plan (or of an emulation group's ranks) runs the select's full-histogram fallback round -- a
 * pass over b, one 2048-word all-reduce and the pick -- as a conditional graph node that only
 * executes when the coarse step missed its window (3 collectives per iteration instead of 4),
 * 0 when the round is captured unconditionally (world 1, no graph yet, or the conditional capture
 * failed and the library fell back).  Host-only, no synchronisation. */
int cssar_debug_graph_info(cssar_plan plan, int32_t* info_out);
int cssar_group_debug_graph_info(cssar_group group, int32_t* info_out);

/* Multi-GPU plumbing hooks (tests).  cssar_debug_ipc_export writes an 80-byte
 * record {cudaIpcMemHandle_t of the allocation holding dev_ptr, byte offset of dev_ptr in it,
 * pad} -- the same record cssar_bind_workspace all-gathers; cssar_debug_ipc_open maps a peer
 * process's record (base_out = the mapping to pass to cssar_debug_ipc_close, ptr_out = the
 * peer's dev_ptr in this process).  cssar_debug_peer_store writes dst[i] = pattern ^ i for
 * i < n_words (then a system-scope fence), asynchronously on `stream`.
 * cssar_group_debug_barrier runs `rounds` flag-barrier rounds of every rank of an emulation
 * group in one cooperative launch (one block per rank: co-resident, so spinning is legal on
 * one GPU); CSSAR_ERR_NCCL on a timeout or a wrong final epoch.  Synchronous. */
int cssar_debug_ipc_export(const void* dev_ptr, void* rec_out);
int cssar_debug_ipc_open(const void* rec, void** base_out, void** ptr_out);
int cssar_debug_ipc_close(void* base);
int cssar_debug_peer_store(void* dst, uint32_t pattern, int64_t n_words, void* stream);
int cssar_group_debug_barrier(cssar_group group, int32_t rounds, void* stream);
/* A world-1 plan over a ONE-rank NCCL communicator (nccl_unique_id: 128 bytes from
 * cssar_nccl_unique_id) that runs the slab path of cssar_plan_create(world > 1) -- the
 * all-to-all transposes (ncclSend / ncclRecv to itself in a group), the grouped all-reduces
 * of the select, the IPC all-gather of cssar_bind_workspace -- with whole arrays as slabs, so
 * the real NCCL plumbing can be checked on one GPU against the world-1 path (bitwise equal
 * results).  Same contract as a world > 1 plan otherwise (debug hooks: CSSAR_ERR_BAD_PLAN). */
int cssar_debug_plan_create_nccl(cssar_plan* out, const cssar_sar_params* p, const void* nccl_unique_id);

#ifdef __cplusplus
}
#endif
#endif /* CSSAR_H_ */
