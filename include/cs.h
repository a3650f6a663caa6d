/*
 * cs.h — C ABI of the B200-native greedy compressive-sensing library (libcsgpu.so).
 *
 * Method: Hsieh, Lu, Pei, "Fast Greedy Approaches for Compressive Sensing of
 * Large-Scale Signals", arXiv:1509.03979.  Citation key: P:n = PAPER.md line n,
 * S:n = SPEC.md line n (both under the reference mount).
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - Every pointer named d_* is CALLER-OWNED DEVICE memory on the current
 *    CUDA device (torch allocates it).  The library never allocates device
 *    memory; the only library-owned object is the small host struct behind
 *    cs_operator*.
 *  - Every compute call is asynchronous on `stream` (0 = legacy default stream).
 *    Results are valid after the caller synchronises that stream.
 *  - Errors are status codes; nothing throws across the ABI.  Host-side
 *    argument validation is synchronous and happens before any launch.
 *    cs_last_error() returns a thread-local detail string for the last
 *    non-CS_OK status of the calling thread.
 *  - fp32 and fp64 variants exist for each compute call (suffix _f64); the
 *    element type of the buffers is the arithmetic type of the whole path.
 *  - Vectors are row-major; batched arrays are [B][len].
 *  - Supported N: power of two with 8 <= N <= 2^25.  Other N return
 *    CS_ERR_UNSUPPORTED (the paper's grid is 2^11..2^24).
 */
#ifndef CS_H_
#define CS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* cs_stream_t; /* == cudaStream_t */

typedef enum {
  CS_OK = 0,
  CS_ERR_INVALID_ARG = 1,   /* bad sizes, NULL pointers, bad rows (checked at create) */
  CS_ERR_UNSUPPORTED = 2,   /* N not a power of two / outside [8, 2^25]; device not sm_100 */
  CS_ERR_WORKSPACE = 3,     /* ws_bytes / meta_bytes smaller than required */
  CS_ERR_CUDA = 4,          /* a CUDA runtime call failed (detail in cs_last_error) */
  CS_ERR_NONFINITE = 5      /* reserved for host-detected non-finite input */
} cs_status;

typedef enum { CS_OMP = 0, CS_SP = 1, CS_OMPR = 2, CS_COSAMP = 3 } cs_alg;

/* cs_report.termination — why the OUTER pursuit loop stopped. */
typedef enum {
  CS_TERM_DONE = 0,          /* OMP ran its K iterations                 */
  CS_TERM_ITER_CAP = 1,      /* SP/OMPR/CoSaMP hit max_outer                            */
  CS_TERM_STAGNATION = 2,    /* a CG solve broke down (d^T H d <= 0)             */
  CS_TERM_SUPPORT_FIXED = 3, /* SP/OMPR/CoSaMP: new support == old support              */
  CS_TERM_RESID_ROSE = 4     /* SP/CoSaMP: ||r'|| >= ||r|| — previous (S, x) kept */
} cs_term;

/* cs_report.status bits — conditions found on the device. */
#define CS_DEV_NONFINITE_Y   1u  /* y contained NaN/Inf: outputs are undefined */
#define CS_DEV_CG_CAP        2u  /* some CG solve stopped at its iteration cap          */
#define CS_DEV_CG_BREAKDOWN  4u  /* some CG solve stopped on d^T H d <= 0               */
#define CS_DEV_REFINED_FP64  8u  /* cs_options.refine_fp64: recovered again in fp64       */
#define CS_DEV_NOT_REFINED  16u  /* flagged for refinement, beyond CS_REFINE_CAP: fp32 kept */

typedef struct {
  int32_t outer_iters;     /* pursuit outer iterations executed                       */
  int32_t cg_iters_total;  /* sum of CG iterations over all solves                    */
  int32_t cg_solves;       /* number of CG solves                                     */
  int32_t applies;         /* number of A / A^T pairs ("sandwiches") executed         */
  int32_t termination;     /* cs_term                                                 */
  uint32_t status;         /* CS_DEV_* bits                                           */
  double resid_norm;       /* ||y - A s_hat||_2 at exit                               */
  double cg_rel_resid;     /* largest ||r_j||/||b|| at the exit of any CG solve       */
} cs_report;               /* 40 bytes */

typedef struct {
  int32_t max_outer;    /* SP/OMPR/CoSaMP outer cap; 0 -> SP 30, OMPR 2K, CoSaMP 30 */
  int32_t cg_max_iters; /* 0 -> |S| + 50 (Thm 5 bound |S| plus slack, SURVEY #29)           */
  int32_t ompr_l;       /* OMPR(l): indices swapped in per outer iteration; 0 -> 1  */
  float ompr_eta;       /* OMPR step eta; 0 -> 1.0                                   */
  int32_t refine_fp64;  /* fp32 batched recovery on the CTA tier only (SURVEY §8c.9 mixed
                         * policy): 1 -> every problem whose fp32 result holds a coefficient
                         * below the fp32 resolution floor, min |x_i| < CS_REFINE_FLOOR ||x||,
                         * is recovered again from scratch in fp64 and its result replaces
                         * the fp32 one (status CS_DEV_REFINED_FP64); at most CS_REFINE_CAP
                         * problems per call (the rest keep fp32, CS_DEV_NOT_REFINED).  The
                         * workspace grows by cs_workspace_bytes's refine share.  The
                         * host-buffer entry point runs it once over the whole batch after
                         * its fp32 chunks and copies the results out after it (workspace:
                         * cs_workspace_bytes_host with the same options).  0 -> off.      */
  int32_t reserved[3];  /* must be zero                                                      */
} cs_options;
#define CS_REFINE_FLOOR 1e-6  /* ~16 fp32 ulps: the sandwich's relative rounding */
#define CS_REFINE_CAP   256

/* ---------------------------------------------------------------- operator ---
 * A = P . C_N . diag(sigma)   (Eq.(7) Phi = D F R, with BASELINE.json's
 * sign randomizer and Psi = I; C_N = orthonormal DCT-II; P = row selection,
 * P:485).  A x = (C_N (sigma . x))[rows], A^T w = sigma . C_N^T scatter_rows(w).
 *
 * An operator holds `batch` independent instances (each with its own sigma and
 * rows), used by the batched calls.  Instance b occupies row b of every batched
 * array.
 */
typedef struct cs_operator cs_operator;

/* Bytes of device metadata `cs_operator_create` needs per instance: sign words; for
 * N <= 16384 the row bitmask and row-rank prefix in natural order (CTA tier); for every N
 * the row bitmask and prefix in the four-step FFT's transposed order plus a row
 * permutation of M int32 (grid tier) — (3 or 5) * ceil(N/32) * 4 + 4M
 * bytes; 256-byte aligned, plus a 256-byte status tail. */
size_t cs_operator_meta_bytes(int64_t N, int64_t M, int64_t batch);

/* Build an operator.
 *   d_sign_bits [batch][ceil(N/32)] uint32: bit (j % 32) of word j/32 set <=> sigma_j = -1.
 *   d_rows      [batch][M] int32: strictly increasing, each in [0, N).  Checked HERE on
 *               the device; violations return CS_ERR_INVALID_ARG.
 *   d_meta      caller buffer of >= cs_operator_meta_bytes bytes; must outlive the operator.
 * Synchronises `stream` (the row check is read back).  Inputs may be freed afterwards. */
cs_status cs_operator_create(int64_t N, int64_t M, int64_t batch, const uint32_t* d_sign_bits,
                             const int32_t* d_rows, void* d_meta, size_t meta_bytes,
                             cs_stream_t stream, cs_operator** out);

/* The paper's literal Eq.(7) sensing operator Phi = D F R with the
 * randomizer R a permutation (R34), optionally
 * composed with the sign diagonal:  A x = (C_N R (sigma . x))[rows],  (R u)_i = u_{pi(i)}.
 *   d_sign_bits [batch][ceil(N/32)] as above, or NULL for sigma = +1 (the paper's D F R);
 *   d_perm      [batch][N] int32: pi, a permutation of [0, N) per instance.  Checked HERE
 *               on the device; a non-permutation returns CS_ERR_INVALID_ARG.
 *   d_meta      >= cs_operator_meta_bytes_perm bytes (the plain metadata, then pi and
 *               pi^-1 per instance: + 8N bytes per instance, 256-byte aligned).
 * Every call taking a cs_operator accepts it (apply, adjoint, all recover variants); the
 * pursuits select over the ORIGINAL indices j (ties -> lowest j) and return supports
 * in them.  Synchronises `stream`. */
size_t cs_operator_meta_bytes_perm(int64_t N, int64_t M, int64_t batch);
cs_status cs_operator_create_perm(int64_t N, int64_t M, int64_t batch, const uint32_t* d_sign_bits,
                                  const int32_t* d_perm, const int32_t* d_rows, void* d_meta,
                                  size_t meta_bytes, cs_stream_t stream, cs_operator** out);

/* Dictionary Psi of A = Phi Psi (x = Psi s).  The paper's experiments use a DCT
 * ("Psi is chosen to be a discrete cosine transform"; R35): Psi = C_N,
 * the orthonormal DCT-II, so A s = (C_N R (sigma . C_N s))[rows].  BASELINE.json fixes
 * Psi = I. */
typedef enum { CS_PSI_IDENTITY = 0, CS_PSI_DCT = 1 } cs_psi;

/* General constructor: Phi = P C_N R diag(sigma) (d_sign_bits and/or d_perm as in
 * cs_operator_create_perm; either may be NULL, not both) and the dictionary `psi`.
 * d_meta: cs_operator_meta_bytes_ex(N, M, batch, d_perm != NULL, psi) bytes (CS_PSI_DCT adds
 * one all-rows metadata instance, about 4.4 N bytes, shared by the batch).  With CS_PSI_DCT,
 * apply/adjoint need the workspace cs_operator_ws_bytes reports.  Supports and values are in
 * the s-domain. */
size_t cs_operator_meta_bytes_ex(int64_t N, int64_t M, int64_t batch, int has_perm, int psi);
cs_status cs_operator_create_ex(int64_t N, int64_t M, int64_t batch, const uint32_t* d_sign_bits,
                                const int32_t* d_perm, const int32_t* d_rows, int psi, void* d_meta,
                                size_t meta_bytes, cs_stream_t stream, cs_operator** out);

/* F = partial Fourier (the MRI case of D F R; R36): real x,
 * n_freq frequencies f in [1, N/2 - 1] per instance (d_freqs [batch][n_freq], strictly
 * increasing — checked here), M = 2 n_freq measurements y[2r] = sqrt(2/N) Re X_f,
 * y[2r+1] = sqrt(2/N) Im X_f, X = unnormalised DFT of R diag(sigma) x.  d_sign_bits and
 * d_perm may be NULL (sigma = +1, R = I).  d_meta: cs_operator_meta_bytes_dft bytes.
 * The operator then works with every apply / adjoint / recover call, with M = 2 n_freq. */
size_t cs_operator_meta_bytes_dft(int64_t N, int64_t n_freq, int64_t batch);
cs_status cs_operator_create_dft(int64_t N, int64_t n_freq, int64_t batch, const uint32_t* d_sign_bits,
                                 const int32_t* d_perm, const int32_t* d_freqs, void* d_meta,
                                 size_t meta_bytes, cs_stream_t stream, cs_operator** out);
cs_status cs_operator_destroy(cs_operator* op);
cs_status cs_operator_info(const cs_operator* op, int64_t* N, int64_t* M, int64_t* batch);

/* Workspace bytes for apply/adjoint (0 for N <= 16384 — batch * N elements with
 * CS_PSI_DCT — else the four-step scratch per group of a batch run side by side). */
size_t cs_operator_ws_bytes(const cs_operator* op, int precision /*0 fp32, 1 fp64*/);

/* y[b] = A_b x[b] for every instance b.  x [batch][N], y [batch][M]. */
cs_status cs_operator_apply(const cs_operator* op, const float* d_x, float* d_y, void* d_ws,
                            size_t ws_bytes, cs_stream_t stream);
cs_status cs_operator_apply_f64(const cs_operator* op, const double* d_x, double* d_y,
                                void* d_ws, size_t ws_bytes, cs_stream_t stream);
/* x[b] = A_b^T y[b] (zero-fill unselected rows, DCT-III, sign).  y [batch][M], x [batch][N]. */
cs_status cs_operator_adjoint(const cs_operator* op, const float* d_y, float* d_x, void* d_ws,
                              size_t ws_bytes, cs_stream_t stream);
cs_status cs_operator_adjoint_f64(const cs_operator* op, const double* d_y, double* d_x,
                                  void* d_ws, size_t ws_bytes, cs_stream_t stream);

/* ---------------------------------------------------------------- recovery ---
 * Greedy recovery with the CG-solved weighted least squares of Eq.(11) (P:376,
 * Algorithm 1) in place of the pseudo-inverse:
 *   CS_OMP  — Algorithm 1, exactly K outer iterations;
 *   CS_SP   — CG-SP (named P:574-576; body per S:286-294, R15);
 *   CS_OMPR — CG-OMPR(l, eta) (named P:574-576; body per S:296-304, R16);
 *   CS_COSAMP — CG-CoSaMP (named P:84 among the greedy methods; the published CoSaMP
 *             iteration with this CG as its LS step, halting rule DESIGN.md R33).
 * Each CG solve is warm-started from the previous iterate and stops when
 * ||r_j|| <= tol * ||b|| (relative; R6/R7), at cg_max_iters, or on breakdown.
 *
 * Outputs: d_support [K] int32 ascending, d_vals [K] the LS coefficients on it,
 * d_report one cs_report (DEVICE memory).  Requirements: 1 <= K; OMP: K <= M;
 * SP: 2K <= M; OMPR: K + l <= M; CoSaMP: 3K <= M; K <= N/2; 0 <= tol.
 *
 * cs_workspace_bytes: DEVICE workspace for cs_recover*: 2 * batch * N elements when the
 * pursuit fits one CTA (N <= 16384, small K: A^T y per problem plus the Psi scratch), else
 * the grid tier's per-group layout times the groups a batch can run side by side.  The
 * workspace may be reused across calls on one stream; it needs no initialisation.
 */
cs_status cs_workspace_bytes(int alg, int64_t N, int64_t M, int32_t K, int64_t batch,
                             int precision /*0 fp32, 1 fp64*/, const cs_options* opts,
                             size_t* bytes);

cs_status cs_recover(const cs_operator* op, int alg, const float* d_y, int64_t M, int64_t N,
                     int32_t K, double tol, const cs_options* opts, float* d_vals,
                     int32_t* d_support, cs_report* d_report, void* d_ws, size_t ws_bytes,
                     cs_stream_t stream);
cs_status cs_recover_f64(const cs_operator* op, int alg, const double* d_y, int64_t M, int64_t N,
                         int32_t K, double tol, const cs_options* opts, double* d_vals,
                         int32_t* d_support, cs_report* d_report, void* d_ws, size_t ws_bytes,
                         cs_stream_t stream);

/* B independent problems; problem b uses operator instance b (op batch == B).
 * d_Y [B][M], d_vals [B][K], d_support [B][K], d_reports [B]. */
cs_status cs_recover_batched(const cs_operator* op, int alg, const float* d_Y, int64_t B,
                             int64_t M, int64_t N, int32_t K, double tol,
                             const cs_options* opts, float* d_vals, int32_t* d_support,
                             cs_report* d_reports, void* d_ws, size_t ws_bytes,
                             cs_stream_t stream);
cs_status cs_recover_batched_f64(const cs_operator* op, int alg, const double* d_Y, int64_t B,
                                 int64_t M, int64_t N, int32_t K, double tol,
                                 const cs_options* opts, double* d_vals, int32_t* d_support,
                                 cs_report* d_reports, void* d_ws, size_t ws_bytes,
                                 cs_stream_t stream);

/* Dense output: d_dense [B][N] = 0 except d_dense[b][d_support[b][k]] = d_vals[b][k]
 * (support entries < 0, as written for a short support, are skipped).  Async on `stream`. */
cs_status cs_support_to_dense(int64_t B, int64_t N, int32_t K, const int32_t* d_support, const float* d_vals,
                              float* d_dense, cs_stream_t stream);
cs_status cs_support_to_dense_f64(int64_t B, int64_t N, int32_t K, const int32_t* d_support,
                                  const double* d_vals, double* d_dense, cs_stream_t stream);

/* ---------------------------------------------------------------- multi-GPU ---
 * Results gather for independent problems sharded over the GPUs of one process (SV §8e:
 * the only cross-GPU traffic of the batched path; no data-path collective).  NCCL is
 * loaded at run time (libnccl.so.2); without it cs_comm_init returns CS_ERR_UNSUPPORTED.
 *   cs_comm_init(ndev, devices, &comm): one communicator per device (ncclCommInitAll).
 *   cs_gather_batched: device i (in `devices` order) holds B_per_dev records in
 *     d_vals[i] [B][K] fp32, d_support[i] [B][K], d_reports[i] [B]; they land at block i of
 *     the root's d_vals_all / d_support_all / d_reports_all ([ndev][B]...).  Blocking: returns
 *     after the transfers (NCCL send/recv over NVLink; the root copies its own block).  It runs
 *     on the library's own per-device streams and is NOT ordered after the caller's work: the
 *     caller synchronises the producing streams first, or uses cs_gather_batched_after.
 *   cs_gather_batched_after: the same, ordered after everything enqueued so far on
 *     after[i] (device i's producer stream; NULL entries / a NULL array: no ordering), so the
 *     recovery kernels that write the records need no host synchronisation in between.
 * (Multi-process jobs use torch.distributed, paper_1509_03979_b200/dist.py.) */
cs_status cs_comm_init(int ndev, const int* devices, void** comm);
cs_status cs_gather_batched(void* comm, int root, int64_t B_per_dev, int32_t K, const float* const* d_vals,
                            const int32_t* const* d_support, const cs_report* const* d_reports,
                            float* d_vals_all, int32_t* d_support_all, cs_report* d_reports_all);
cs_status cs_gather_batched_after(void* comm, int root, int64_t B_per_dev, int32_t K, const float* const* d_vals,
                                  const int32_t* const* d_support, const cs_report* const* d_reports,
                                  float* d_vals_all, int32_t* d_support_all, cs_report* d_reports_all,
                                  const cs_stream_t* after);
cs_status cs_comm_destroy(void* comm);

/* ---------------------------------------------------------------- single signal, G GPUs ---
 * (SV §8f NEXT-4; the paper's "large-scale" signals) The four-step operator of one
 * large signal (N > 16384, fp32, the plain P.DCT.diag(sigma) of Eq.(7) with the sign
 * randomizer, instance 0 of `op`) split over `world` ranks with ONE all-to-all per
 * application and no other collective.  The complex [L1][L2] intermediate of the four-step
 * FFT (L1 L2 = N / 2, cs_dist_geometry) is owned by column tiles (CT columns each) in the column
 * passes and by row-pair items (item i = rows i and L1 - i, which the DCT split pairs; items
 * 0 .. L1 / 2) in the row pass.  Rank r owns tiles [t_lo, t_hi) and items [i_lo, i_hi).
 * Distributed layouts (no rank holds a whole vector):
 *   x: "xc", the 2 L1 nc reals (nc = CT (t_hi - t_lo) columns) at the Makhoul positions of
 *      this rank's columns, row by row: xc[q] <-> p = 2 (k1 L2 + c0) + q - 2 nc k1,
 *      k1 = q / (2 nc), c0 = CT t_lo; natural index j = p < N/2 ? 2 p : 2 (N - 1 - p) + 1;
 *   y: "yT", an [M] buffer in the transposed row order of which a rank reads / writes only the
 *      entries of its rows (cs_dist_row_offsets gives where each row's entries start).
 *   apply   y = A x:   DP_A  (xc -> its column FFTs), all-to-all columns -> row pairs,
 *                      DP_BF (its row FFTs + DCT split + row select -> its entries of yT);
 *   adjoint x = A^T y: DP_BA (its entries of yT -> its rows), all-to-all row pairs -> columns,
 *                      DP_C  (its inverse column FFTs -> xc).
 *   layout changes (no arithmetic): DP_XS natural x [N] -> xc; DP_XG the xc of all ranks
 *   gathered in rank order ([G][2 L1 nc], equal tile ranges: G = (L2 / CT) / (t_hi - t_lo))
 *   -> natural x [N]; DP_YT natural y [M] -> yT; DP_P complete yT -> natural y [M].
 * d_in / d_out: DEVICE fp32 (DP_A, DP_BA: d_in only; DP_BF, DP_C: d_out only).
 * cs_dist_copy moves segments (row rows[k], columns [col0[k], col0[k] + seg_len)) of the
 * intermediate between the workspace and a flat exchange buffer of nseg seg_len complex fp32
 * values (to_buf 1: pack, 0: unpack); d_rows / d_col0 are DEVICE int32 arrays the caller keeps
 * in range (0 <= rows[k] < L1, 0 <= col0[k] <= L2 - seg_len; not checked on the device).  d_ws: DEVICE workspace of cs_dist_ws_bytes(N, M) bytes,
 * one per rank, kept across the phases of one application.  cs_dist_row_offsets fills
 * h_off[0 .. L1] (HOST) with the yT offset where row k1's entries start (h_off[L1] = M); it
 * synchronizes the device (plan time).  Orchestration and the all-to-alls (torch.distributed /
 * NCCL): paper_1509_03979_b200/dist.py.  Errors: CS_ERR_UNSUPPORTED for N <= 16384 or another
 * operator kind, CS_ERR_INVALID_ARG for ranges out of bounds or missing buffers.  Phases and
 * copies are asynchronous on `stream`. */
#define CS_DP_A 0
#define CS_DP_BF 1
#define CS_DP_BA 2
#define CS_DP_C 3
#define CS_DP_P 4
#define CS_DP_YT 5
#define CS_DP_XS 6
#define CS_DP_XG 7
cs_status cs_dist_geometry(int64_t N, int64_t* L1, int64_t* L2, int32_t* CT);
size_t cs_dist_ws_bytes(int64_t N, int64_t M);
cs_status cs_dist_phase(const cs_operator* op, int phase, int64_t t_lo, int64_t t_hi, int64_t i_lo, int64_t i_hi,
                        const float* d_in, float* d_out, void* d_ws, size_t ws_bytes, cs_stream_t stream);
cs_status cs_dist_copy(const cs_operator* op, void* d_ws, const int32_t* d_rows, const int32_t* d_col0, int64_t nseg,
                       int64_t seg_len, float* d_buf, int to_buf, cs_stream_t stream);
cs_status cs_dist_row_offsets(const cs_operator* op, int64_t* h_off);

/* Host-buffer variants (the end-to-end entry points): h_Y [B][M] and the outputs
 * h_vals [B][K], h_support [B][K], h_reports [B] are HOST memory (pinned for overlap).
 * The batch is copied in, recovered and copied out in chunks of two recovery waves, on
 * internal streams so that the copies of one chunk overlap the recovery of its
 * neighbours; `stream` is ordered before the first copy and after the last one (results
 * are valid once `stream` is synchronised).  d_ws: DEVICE workspace of at least
 * cs_workspace_bytes_host bytes (the recovery workspace plus device staging of the
 * batch).  Errors as cs_recover_batched. */
cs_status cs_workspace_bytes_host(int alg, int64_t N, int64_t M, int32_t K, int64_t batch,
                                  int precision /*0 fp32, 1 fp64*/, const cs_options* opts,
                                  size_t* bytes);
cs_status cs_recover_batched_host(const cs_operator* op, int alg, const float* h_Y, int64_t B,
                                  int64_t M, int64_t N, int32_t K, double tol,
                                  const cs_options* opts, float* h_vals, int32_t* h_support,
                                  cs_report* h_reports, void* d_ws, size_t ws_bytes,
                                  cs_stream_t stream);
cs_status cs_recover_batched_host_f64(const cs_operator* op, int alg, const double* h_Y, int64_t B,
                                      int64_t M, int64_t N, int32_t K, double tol,
                                      const cs_options* opts, double* h_vals,
                                      int32_t* h_support, cs_report* h_reports, void* d_ws,
                                      size_t ws_bytes, cs_stream_t stream);

/* ---------------------------------------------------------------- misc ------ */
const char* cs_status_string(cs_status s);
const char* cs_last_error(void);
/* Number of kernels this library launched on the calling thread since the last reset. */
uint64_t cs_launch_count(int reset);
const char* cs_version(void);

/* Diagnostics: byte offset, in a Tier L (N > 16384) recovery workspace, of 8 uint64 phase
 * accumulators (nanoseconds of %globaltimer seen by block 0: [0] everything between
 * sandwiches, [1] pass A of H, [2] pass B of H, [3] pass C of H, [4] pass A of the residual,
 * [5] its pass B, [6] its pass C + reduction), valid after the stream syncs; -1 for Tier S. */
int64_t cs_diag_phase_offset(int alg, int64_t N, int64_t M, int32_t K, int32_t ompr_l, int precision);
/* (alg < 0: the byte offset of the Tier L apply's five %globaltimer phase stamps of instance 0 —
 * start, input reorder, pass A, pass B, output permute — in the apply / adjoint workspace.) */
/* Test hook: the CTA tier's top-K selection on d_vals [n] (fp32 or fp64 by `precision`):
 * bit i of d_out_bits [ceil(n/32)] (device) is set iff |vals[i]| is among the K largest,
 * ties to the lowest index.  mode 0: the two-pass path (radix fallback),
 * mode 1: the radix path.  One CTA; asynchronous on `stream`.  1 <= K <= n <= 2^24. */
cs_status cs_diag_topk(const void* d_vals, int64_t n, int64_t K, int precision, int mode,
                       uint32_t* d_out_bits, cs_stream_t stream);
/* Test hook: the GRID tier's top-K (the radix select of detection at N >= 2^15) on d_vals [n]
 * over a full cooperative grid; same output and tie rule as cs_diag_topk.  d_ws: DEVICE
 * workspace of cs_diag_topk_grid_ws_bytes() bytes (caller-owned).  1 <= K <= n <= 2^26. */
size_t cs_diag_topk_grid_ws_bytes(void);
cs_status cs_diag_topk_grid(const void* d_vals, int64_t n, int64_t K, int precision, uint32_t* d_out_bits,
                            void* d_ws, size_t ws_bytes, cs_stream_t stream);
/* Diagnostics: microseconds per grid-wide barrier (with_sum: plus a grid reduction) in a
 * cooperative launch shaped like the Tier L recovery; synchronous; -1 on error. */
double cs_diag_grid_barrier_us(int iters, int with_sum);

#ifdef __cplusplus
}
#endif
#endif /* CS_H_ */
