/*
 * spmesl.h — C ABI of the B200-native SPMESL hot path.
 *
 * SPMESL (sparse precision matrix estimation via the scaled lasso), as computed by the
 * column-parallel coordinate descent of arXiv 2203.15031 (PAPER.md lines cited as P:<n>):
 *
 *   for every column k (Eq. spmesl):
 *     (b_k, sigma_k) = argmin ||x_k - X b||^2/(2 n sigma) + sigma/2 + lambda0 ||b||_1,  b_kk = 0
 *   solved by Algorithm 1 per column (inner CD sweeps j = 1..p ascending with
 *   a_j = x_j^T e / n + b_j, b_j <- Soft_{sigma lambda0}(a_j), inner stop
 *   max_j |db_j| < tol, sigma refit ||e||_2/sqrt(n) and outer stop |dsigma| < tol
 *   ); all columns advance together row by row (Proposition 2);
 *   then Theta1_jk = -b_jk / sigma_k^2, Theta1_kk = 1/sigma_k^2 (Eq. relation P:268-272,
 *   Alg. 2), Proposition 1 rescaling to the data's scale, and the
 *   minimum-magnitude symmetrization of Eq. (symm) (Alg. 2).
 *
 * Conventions (all entry points):
 *   - X is n x p, COLUMN-MAJOR, fp64, leading dimension n (column x_k contiguous).
 *   - Theta is p x p, column-major, fp64, leading dimension p.  It is symmetric on return
 *     unless opt->symmetrize == 0 (then Theta holds Theta1, the assembled and rescaled
 *     but unsymmetrized estimate).
 *   - sigma[p] is on the scale of the input data (sigma_k^o = s_k sigma_k^C) when
 *     opt->standardize == 1 (default); iters[p] = outer iterations r per column;
 *     sweeps[p] = inner CD sweeps summed over all outer iterations; converged[p] = 1 iff
 *     the column met |dsigma| < tol before max_iter and no inner loop hit max_inner.
 *   - Every pointer is caller-owned and never retained after return.  The library
 *     allocates its device scratch per device and reuses it across calls
 *     (spmesl_release_workspace frees it).  Calls on one device are serialised.
 *   - Return codes below.  On a negative code the contents of output buffers are
 *     unspecified (the host entry points may have zero-filled Theta); the message is
 *     available from spmesl_last_error() (thread-local).
 *   - Paper-silent points follow the readings listed in DESIGN.md §3 (tolerances are
 *     absolute; the residual is recomputed at each outer boundary; sigma floor; the
 *     (j,k), j<k entry wins a symmetrization tie; constant columns are an error).
 */
#ifndef SPMESL_H
#define SPMESL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPMESL_OK                   0
#define SPMESL_WARN_NOT_CONVERGED   1   /* outputs valid; >= 1 column hit max_iter or max_inner */
#define SPMESL_ERR_ARG             -1   /* n < 2, p < 2, lambda0 < 0 or non-finite, tol <= 0,
                                           max_iter < 1, NULL pointer, bad column range */
#define SPMESL_ERR_CONSTANT_COLUMN -2   /* s_k <= 1e-13 max_i |x_ik|; index in stats->bad_column */
#define SPMESL_ERR_NONFINITE       -3   /* NaN/Inf in X; column index in stats->bad_column */
#define SPMESL_ERR_CUDA            -4   /* CUDA runtime error (message in spmesl_last_error) */
#define SPMESL_ERR_NCCL            -5   /* options.num_devices >= 1: NCCL could not be loaded or a
                                           collective failed (message in spmesl_last_error) */
#define SPMESL_ERR_OOM             -6   /* device allocation failed (or p*p*8 overflows) */
#define SPMESL_ERR_UNSUPPORTED     -7   /* n too large for the on-chip residual tile (n > 2688),
                                           or no sm_100 device */

typedef struct {
  int32_t struct_size;    /* sizeof(spmesl_options); set by spmesl_default_options */
  int32_t max_inner;      /* cap on inner sweeps per outer iteration (default 10000) */
  int32_t standardize;    /* 1: centre + scale columns inside and return Theta and
                             sigma on the input scale (Prop. 1); 0: X is used as given */
  int32_t symmetrize;     /* 1 (default): Eq. (symm); 0: return Theta1 */
  double  sigma_floor;    /* sigma_k >= sigma_floor (default 1e-8; reading g5) */
  int32_t mode;           /* 0 (default): per-column stop — each column runs Algorithm 1 with
                             its own inner stop and leaves when its sigma settles.
                             1: Algorithm 3 — all active columns sweep together
                             until max over them of ||B_next - B_cur||_inf < tol, then
                             sigma is refit for all and settled columns leave the
                             active set.  Mode 1 ignores tail_after and, in
                             spmesl_fit_columns_device, needs the whole range [0, p)
                             (else SPMESL_ERR_UNSUPPORTED). */
  int32_t tile_cols;      /* 0: auto; 8, 16 or 32 resident columns per SM (tests) */
  int32_t device;         /* host entry points: CUDA device ordinal (-1: current device) */
  int32_t tail_after;     /* columns still running after this many sweeps finish in the
                             covariance-update tail solver (default 1; 0: never).  Same
                             iterates up to rounding. */
  int32_t solver;         /* 0 (default): auto — solver 3 when mode = 0, the whole column range
                             is fitted on one device, p is at most ~26000 (the sweep kernel
                             keeps z[p] on chip) and 8 p^2 bytes fit in device memory; else
                             the residual solver; on the device path a repeat of a fit (same
                             arguments) whose certified screening left most columns candidates
                             runs solver 2's path directly (same iterates bit for bit; a
                             full-Gram fit with few hit columns hands back to solver 3).
                             1: residual solver (persistent CD kernel on
                             X~ streamed through shared memory).  2: Gram solver with the full
                             S = X~^T X~ / n (symmetric FP64 DMMA contraction, first-sweep
                             screening fused in), then covariance updates.  3: Gram solver with
                             certified f16 screening: the first-sweep test |S_jc| > lambda0 is
                             decided on the f16 tensor cores with a rigorous error bound; only
                             the columns it cannot certify get exact FP64 Gram columns (and
                             their exact test), the others are known to stop after one sweep.
                             2 and 3: SPMESL_ERR_UNSUPPORTED where they do not apply.  All
                             solvers: same iterates up to FP64 rounding. */
  int32_t eager;          /* spmesl_fit_device, Gram solvers: 0 (default) captures the whole
                             enqueued fit as a CUDA graph the second time the same arguments
                             (pointers included) arrive and replays it from then on (one launch
                             per fit); 1: enqueue every operation on each call.  Same results. */
  int32_t num_devices;    /* host entry points (spmesl_fit, spmesl_fit_ex) only: 0 (default)
                             fits on one device (`device`); G >= 1 fits on G devices of this
                             node with NCCL: each device fits a contiguous block
                             of columns (X replicated), the devices exchange the p first-sweep
                             screening flags and, after the fit, the coefficients (see
                             `exchange`).  Mode 0 only (else SPMESL_ERR_UNSUPPORTED); results
                             are those of the single-device fit bit for bit. */
  int32_t exchange;       /* num_devices >= 1: how the devices exchange.
                             0 (default): peer-to-peer when every pair of the devices has peer
                             access (NVLink / NVSwitch), else NCCL.  1: NCCL — one max
                             all-reduce of the p flags, one all-gather of the coefficients as
                             CSC; device 0 symmetrizes and assembles (NCCL is loaded at run
                             time: SPMESL_ERR_NCCL if it cannot be).  2: peer-to-peer — each
                             device reads the other devices' screening flags and, for the
                             symmetrization of its own columns (Eq. symm), each
                             partner b_kj straight from the memory of the device that fitted
                             column j; every device assembles its own columns (no collective,
                             no NCCL; SPMESL_ERR_UNSUPPORTED without peer access or for more
                             than 16 devices).  With exchange 2 (or 0 resolving to it) device
                             ids may repeat: blocks that share a device. */
  const int32_t* device_ids;  /* host array of num_devices CUDA ordinals (distinct unless the
                                 exchange is peer-to-peer), or NULL for 0 .. num_devices - 1 */
  int32_t reserved[2];
} spmesl_options;

typedef struct {
  int64_t coord_updates;  /* algorithmic coordinate updates V = sum_k sweeps_k (p - 1) */
  int64_t total_sweeps;   /* sum_k sweeps_k */
  int32_t max_sweeps;     /* max_k sweeps_k */
  int32_t max_outer;      /* max_k iters_k */
  int32_t n_unconverged;  /* columns with converged_k == 0 */
  int32_t tile_cols;      /* resident columns per CTA actually used */
  int32_t num_ctas;       /* persistent CTAs launched by the CD kernel */
  int32_t kernel_launches;/* kernels launched by this call (excluding memsets/copies) */
  int64_t bad_column;     /* column index for SPMESL_ERR_CONSTANT_COLUMN / _NONFINITE, else -1 */
  int64_t nnz;            /* nonzero off-diagonal coefficients b_jk over the fitted columns */
  double  ms_standardize; /* device time of standardization + Gram band (CUDA events) */
  double  ms_cd;          /* device time of the persistent CD kernel */
  double  ms_assemble;    /* device time of assembly + symmetrization (incl. CSC build) */
  double  ms_total;       /* device time of the whole call on the stream */
  double  ms_tail;        /* device time of the tail solver (0 if it did not run) */
  int64_t tail_columns;   /* columns finished by the tail solver */
  int64_t tail_gram_ondemand; /* Gram columns the tail solver computed on first use */
  int64_t tail_sweeps;    /* sweeps performed by the tail solver (the CD kernel did the rest) */
  int32_t solver;         /* solver used: 1 residual, 2 Gram (FP64 S), 3 Gram (certified f16
                             screening) */
  int32_t gram_fallback;  /* solver 3: 1 if most columns were candidates and the full FP64 Gram
                             kernel decided them instead */
  double  ms_gram;        /* Gram solver: device time of the screening pass (solver 2: the FP64
                             Gram kernel; solver 3: f16 screening + exact Gram columns of the
                             candidates) */
  int64_t screen_candidates; /* solver 3: columns the f16 screening could not certify hit-free */
  double  ms_screen;      /* device time of the screening kernel alone (solver 2: the FP64 Gram
                             kernel; solver 3: the f16 screening kernel incl. its share of
                             Theta's zero fill) */
  int64_t screen_fill_bytes; /* bytes of Theta the screening kernel zero-filled (the rest of the
                             fill, if any, ran on a side stream beside the later kernels) */
  int32_t graph_replay;   /* 1 if this call ran as one CUDA-graph launch (options.eager); then
                             only ms_total and ms_screen are measured, the other ms_* read -1 */
  int32_t pad1;
  int64_t tail_changes;   /* coordinate changes (b_jk moved) made by the covariance-update sweep
                             kernel; each reads one Gram column (8 p bytes: its algorithmic
                             traffic) */
  int64_t tail_passes;    /* segments (speculative chain + one pass over the rows) the sweep
                             kernel ran: one per sweep plus one per row that entered the support
                             within a sweep */
  double  ms_comm;        /* options.num_devices >= 1: device time of the exchange on device 0
                             (NCCL: flag all-reduce + CSC all-gather; peer-to-peer: the flag
                             max over the peers + the symmetrizing assembly that reads them) */
  int32_t num_devices;    /* devices the fit ran on (0: the single-device path) */
  int32_t exchange;       /* multi-device fits: 1 NCCL collectives, 2 peer-to-peer (0: one device) */
} spmesl_stats;

/* Fill *opt with the defaults listed above. */
void spmesl_default_options(spmesl_options* opt);

/*
 * Host-memory entry point (BASELINE.json: spmesl_fit(X, n, p, lambda0, tol, max_iter ->
 * Theta, sigma, iters)).  X: host n x p; Theta: host p x p; sigma: host [p]; iters: host [p].
 * Copies X to the current device and runs the whole path there.  Theta is zero-filled by host
 * threads while the device computes; only its nonzero entries (and the diagonal) are copied
 * back and scattered.  Host buffers may be pageable or pinned.  Blocking.
 */
int spmesl_fit(const double* X, int64_t n, int64_t p, double lambda0, double tol,
               int32_t max_iter, double* Theta, double* sigma, int32_t* iters);

/* As spmesl_fit with options, optional per-column sweeps[p] / converged[p] (nullable) and
 * optional statistics (nullable). */
int spmesl_fit_ex(const double* X, int64_t n, int64_t p, double lambda0, double tol,
                  int32_t max_iter, const spmesl_options* opt, double* Theta, double* sigma,
                  int32_t* iters, int32_t* sweeps, uint8_t* converged, spmesl_stats* st);

/*
 * Device-memory entry point: every array pointer is a device pointer on the current
 * device (e.g. a torch tensor's data_ptr()); work is enqueued on cuda_stream (a
 * cudaStream_t; NULL = legacy default stream).  dSweeps / dConverged nullable.
 * Blocking: returns after the work completes (it must read the error flags).
 */
int spmesl_fit_device(const double* dX, int64_t n, int64_t p, double lambda0, double tol,
                      int32_t max_iter, const spmesl_options* opt, double* dTheta,
                      double* dSigma, int32_t* dIters, int32_t* dSweeps, uint8_t* dConverged,
                      void* cuda_stream, spmesl_stats* st);

/*
 * Sparse-output device entry point: as spmesl_fit_device, but Theta —
 * symmetrized per options.symmetrize, rescaled per options.standardize, diagonal included —
 * is returned in compressed sparse column form instead of a dense p x p array (no 8 p^2-byte
 * fill): dColPtr[p + 1] (int64, device), dRows[cap] (int32, device; ascending within each
 * column), dVals[cap] (double, device).  Theta is symmetric, so this is also its CSR form.
 * Every entry equals the dense path's bit for bit; the absent ones are zeros there.
 * *nnz_out (host) receives the entry count; if it exceeds cap the call returns SPMESL_ERR_ARG
 * with dColPtr filled and dRows/dVals untouched.  dSigma / dIters [p] as spmesl_fit_device;
 * dSweeps / dConverged nullable.  Any mode / solver.  Blocking.
 */
int spmesl_fit_sparse_device(const double* dX, int64_t n, int64_t p, double lambda0, double tol,
                             int32_t max_iter, const spmesl_options* opt, int64_t* dColPtr,
                             int32_t* dRows, double* dVals, int64_t cap, int64_t* nnz_out,
                             double* dSigma, int32_t* dIters, int32_t* dSweeps,
                             uint8_t* dConverged, void* cuda_stream, spmesl_stats* st);

/*
 * Host sparse-output entry point: as spmesl_fit_ex (host X), with Theta returned in compressed
 * sparse column form in host buffers — col_ptr[p + 1] (int64), rows[cap] (int32, ascending
 * within a column), vals[cap] (double); symmetric, so also its CSR form; diagonal included;
 * every entry equals the dense output's bit for bit (spmesl_fit_sparse_device on the current
 * or options.device device).  Only the nonzeros cross PCIe and no p x p array is written.
 * *nnz_out receives the entry count; if it exceeds cap the call returns SPMESL_ERR_ARG with
 * col_ptr/rows/vals untouched (call again with cap >= *nnz_out).  sigma / iters [p];
 * sweeps / converged (nullable) [p].  Blocking.
 */
int spmesl_fit_sparse(const double* X, int64_t n, int64_t p, double lambda0, double tol,
                      int32_t max_iter, const spmesl_options* opt, int64_t* col_ptr,
                      int32_t* rows, double* vals, int64_t cap, int64_t* nnz_out, double* sigma,
                      int32_t* iters, int32_t* sweeps, uint8_t* converged, spmesl_stats* st);

/*
 * Multi-GPU building blocks (one process per GPU; columns [col_begin, col_end) on this rank,
 * X replicated; BASELINE.json north_star "column-block sharding ... one all-gather").
 *
 * spmesl_fit_columns_device: standardize X (all p columns, needed as predictors), solve the
 *   scaled lassos of columns [col_begin, col_end) and export them as CSC on the device:
 *   dColCount[m] (m = col_end - col_begin) = nonzeros of column k (off-diagonal b_jk != 0),
 *   dRows/dVals (capacity `cap` entries, caller-allocated) hold the entries of all m columns
 *   concatenated in column order, rows ascending within a column; dSigmaStd[m] = sigma_k on
 *   the standardized scale; dScale[p] = s_k (column scales, 1 when standardize == 0).
 *   *nnz_out = total entries; if it exceeds cap, returns SPMESL_ERR_ARG and *nnz_out holds the
 *   capacity needed.  Blocking.
 *
 * spmesl_assemble_device: from the GLOBAL CSC of all p columns (dColPtr[p+1], dRows, dVals),
 *   dSigmaStd[p] and dScale[p], write columns [col_begin, col_end) of Theta (symmetrized or
 *   Theta1 as opt->symmetrize says) into dTheta (p x (col_end-col_begin), ld p) and
 *   dSigmaOut[col_end-col_begin] = s_k sigma_k.  Enqueued on cuda_stream, non-blocking.
 */
int spmesl_fit_columns_device(const double* dX, int64_t n, int64_t p, int64_t col_begin,
                              int64_t col_end, double lambda0, double tol, int32_t max_iter,
                              const spmesl_options* opt, int32_t* dColCount, int32_t* dRows,
                              double* dVals, int64_t cap, int64_t* nnz_out, double* dSigmaStd,
                              double* dScale, int32_t* dIters, int32_t* dSweeps,
                              uint8_t* dConverged, void* cuda_stream, spmesl_stats* st);

/*
 * Several penalty levels in one call (a regularization path; SURVEY.md §8(f) f4's "batch the
 * three lambda0 in one launch"), e.g. lambda_pb, lambda_univ, lambda_ub (SPMESL-P, -2,
 * -4).  lambdas: HOST array of nlam (1..8) penalty levels.  Outputs are device arrays laid out
 * level by level: dTheta[nlam][p x p] (each column-major), dSigma[nlam][p], dIters[nlam][p],
 * dSweeps / dConverged (nullable) [nlam][p].  Level l's results are those of spmesl_fit_device
 * with lambda0 = lambdas[l] (same iterates; with the Gram solver bit-identical): X~, S and the
 * screening pass are computed once and shared by all levels.  Enqueued on cuda_stream; returns
 * after one synchronisation.  Errors as spmesl_fit_device; SPMESL_ERR_ARG for nlam outside
 * 1..8.
 */
int spmesl_fit_path_device(const double* dX, int64_t n, int64_t p, const double* lambdas,
                           int32_t nlam, double tol, int32_t max_iter, const spmesl_options* opt,
                           double* dTheta, double* dSigma, int32_t* dIters, int32_t* dSweeps,
                           uint8_t* dConverged, void* cuda_stream, spmesl_stats* st);

/*
 * Multi-GPU building blocks of the Gram solver (SURVEY.md §8(f) f2 + §8(e)).
 * The first sweep of column c with b_c = 0 changes coefficient j iff |x~_j^T x~_c / n| > lambda0
 * (sigma^(0) = 1); "screening" evaluates that test for all pairs (j, c) from the
 * tiles of the symmetric S = X~^T X~ / n.
 *
 * spmesl_gram_tile_count: number of 128 x 128 upper-triangle tiles of S (-1 if p is invalid);
 *   ranks split [0, count) into contiguous shares (solver 2 screening).
 * spmesl_screen_tile_count: the tile count of the screening pass opt selects: solver 2 as
 *   spmesl_gram_tile_count; solvers 0 / 3 the 128 x 256 tiles of the certified f16 screening.
 * spmesl_gram_screen_device: standardize dX (n x p, column-major, device) and evaluate tiles
 *   [tile_begin, tile_end) of the screening pass opt selects; dHit[c] = 1 (never cleared; the
 *   caller zero-fills dHit[p] once) for
 *     solver 2: every column c with some |S_jc| > lambda0, j != c, in those tiles (exact);
 *     solvers 0 / 3: every column c of a pair (j, c) in those tiles that the certified f16
 *       bound cannot clear (candidates: a superset of the columns with a hit).
 *   The OR (max) of dHit over all ranks is the global screening result.  Blocking; errors as
 *   spmesl_fit.
 * spmesl_fit_columns_gram_device: as spmesl_fit_columns_device, for the Gram solver, given the
 *   global dHit[p] of spmesl_gram_screen_device with the same solver (for solvers 0 / 3 the
 *   candidates of the block get their exact FP64 Gram columns, which decide): columns without
 *   a hit finish after one sweep; the others run covariance-update sweeps.  mode must be 0.
 *   Same outputs and iterates as the single-device Gram solver (bit for bit).  Blocking.
 */
int64_t spmesl_gram_tile_count(int64_t p);
int64_t spmesl_screen_tile_count(int64_t p, const spmesl_options* opt);
/* 1 if the Gram solver's sweep state fits on chip for (n, p) on the current device, else 0. */
int spmesl_gram_supported(int64_t n, int64_t p);
int spmesl_gram_screen_device(const double* dX, int64_t n, int64_t p, double lambda0,
                              int64_t tile_begin, int64_t tile_end, const spmesl_options* opt,
                              uint8_t* dHit, void* cuda_stream, spmesl_stats* st);
int spmesl_fit_columns_gram_device(const double* dX, int64_t n, int64_t p, int64_t col_begin,
                                   int64_t col_end, double lambda0, double tol, int32_t max_iter,
                                   const spmesl_options* opt, const uint8_t* dHit,
                                   int32_t* dColCount, int32_t* dRows, double* dVals, int64_t cap,
                                   int64_t* nnz_out, double* dSigmaStd, double* dScale,
                                   int32_t* dIters, int32_t* dSweeps, uint8_t* dConverged,
                                   void* cuda_stream, spmesl_stats* st);

/*
 * TEST-ONLY (not on the fit path): the certified f16 screening (solvers 0 / 3) over all of its
 * tiles, writing the raw f32 tensor-core accumulators acc_jc = n R_hat_jc = sum_i fp16(y_ij)
 * fp16(y_ic) (y_k = x~_k / sqrt(N_k), N_k = x~_k^T x~_k / n) of every pair (j, c)
 * the tiles cover into dAcc[c * acc_ld + j] (device float array, acc_ld >= p rounded up to 256,
 * at least acc_ld columns; the caller zero-fills it: pairs no tile covers stay untouched —
 * every j <= c is covered), and the candidate flags into dCand[p] (device, zero-filled by the
 * caller) at lambda0 = 0.  dY16 (nullable, device): receives the f16 operand tiles the
 * contraction read, 2 * ceil(p / 256) x ceil(n_pad / 64) tiles of 128 variables x 64 samples
 * (n_pad = n rounded up to 32), each 16 KB, [tile row][sample chunk][variable][sample] with the
 * 16-byte groups of each 128-byte row XOR-swizzled by (variable & 7) (screen16.cu header).
 * Lets tests measure |R_hat - R| of the real tcgen05 accumulation against the bound eps(n_pad)
 * the certification assumes.  Blocking; errors as spmesl_fit.
 */
int spmesl_screen_accumulators_device(const double* dX, int64_t n, int64_t p,
                                      const spmesl_options* opt, float* dAcc, int64_t acc_ld,
                                      uint8_t* dCand, void* dY16, void* cuda_stream);

int spmesl_assemble_device(int64_t p, int64_t col_begin, int64_t col_end, const int64_t* dColPtr,
                           const int32_t* dRows, const double* dVals, const double* dSigmaStd,
                           const double* dScale, const spmesl_options* opt, double* dTheta,
                           double* dSigmaOut, void* cuda_stream);

/* Penalty levels of §2.2 (host helpers, not on the device path):
 *   lambda_univ = sqrt(2 log(p-1) / n)
 *   lambda_ub   = A sqrt(4 log p / n)
 *   lambda_pb   = A Phi^{-1}(1 - k/p) / sqrt(n),  k = L_1^4(k/p) + 2 L_1^2(k/p)
 * Return NaN on invalid arguments. */
double spmesl_lambda_univ(int64_t n, int64_t p);
double spmesl_lambda_ub(int64_t n, int64_t p, double A);
double spmesl_lambda_pb(int64_t n, int64_t p, double A);
double spmesl_solve_k(int64_t p);

/* Thread-local message for the last non-OK return on this thread. */
const char* spmesl_last_error(void);
/* Free the cached device workspaces of all devices.  Returns SPMESL_OK. */
int spmesl_release_workspace(void);
/* Library version string. */
const char* spmesl_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPMESL_H */
