// Internal definitions shared by the SPMESL CUDA sources (product path only).
//
// HBM layout of the standardized predictors ("Xb", written by standardize_kernel):
//   X~ (n x p) is stored in tiles of J = 32 predictor columns x KC = 32 samples.  Tile
//   (blk, q) is one contiguous, unpadded 8192-byte block (so one cp.async.bulk moves it to
//   shared memory verbatim) holding x~_{blk*32 + jl}[q*32 + kl] at row jl, position
//   kl ^ (8 (jl & 1)): odd rows have their two 64-byte halves swapped.  That XOR swizzle makes
//   the paired-k 128-bit DMMA fragment loads (8 lanes = rows g, g+1 x 4 lanes, 16 B each) hit
//   8 distinct 16-byte bank groups per phase without any padding bytes in HBM, L2 or smem.
//   Samples i >= n and predictors j >= p are zero.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

namespace spmesl {

constexpr int J = 32;                    // predictor rows per row block (CD visits rows block-wise)
constexpr int KC = 32;                   // samples per staged X chunk
constexpr int XS = KC;                   // chunk row stride (doubles), swizzled not padded
constexpr int CHUNK_DOUBLES = J * XS;    // 1024
constexpr int CHUNK_BYTES = CHUNK_DOUBLES * 8;   // 8192
constexpr int NMW = 8;                   // CD kernel: MMA warps (2 chunk-parity groups x 4)
constexpr int NEW = 1;                   // CD kernel: epilogue warp (lane = column)
constexpr int NWORK = NMW + NEW;         // warps that take part in the per-step barrier
constexpr int WORK_THREADS = NWORK * 32;
constexpr int PRODUCER_WARP = NWORK;     // the X-tile producer warp
constexpr int KSPLIT = 2;                // k-split by chunk parity (fixed => deterministic)
constexpr int RPAD = 8;                  // residual row padding (n_pad + 8 = 8 mod 16)
constexpr int CD_THREADS = (NWORK + 1) * 32;     // + 1 producer warp
constexpr int MAX_T = 32;                // max resident columns (slots) per CTA

struct Layout {
  int64_t n, p;
  int n_pad;      // n rounded up to KC
  int nchunk;     // n_pad / KC
  int64_t nblk;   // ceil(p / J)
  size_t xb_doubles() const { return (size_t)nblk * nchunk * CHUNK_DOUBLES; }
};

// position of k within row jl of a tile (the XOR swizzle above)
__host__ __device__ inline int xswz(int jl, int kl) { return kl ^ ((jl & 1) << 3); }

__host__ __device__ inline size_t xb_index(int64_t i, int64_t j, int nchunk) {
  int64_t blk = j / J, jl = j % J, q = i / KC, kl = i % KC;
  return (size_t)(((blk * nchunk + q) * J + jl) * XS + xswz((int)jl, (int)kl));
}

// Error flags written by kernels (device int32[4]).
enum : int { FLAG_CODE = 0, FLAG_OVERFLOW = 1 };

// State of a column handed from the CD kernel to the tail solver at a sweep boundary
// (coefficients stay in the column's list `cur` with `cnt` entries).
constexpr int SPMESL_MAX_LAM = 8;

struct TailState {
  int col;        // local column index
  int outer;      // outer iterations completed
  int sweeps;     // sweeps completed
  int inner;      // sweeps completed in the current outer iteration
  int flags;      // bit1: an inner loop hit max_inner
  int cur, cnt;   // current coefficient list
  int lam;        // penalty index (multi-lambda fits; 0 otherwise)
  double sigma;   // current sigma (lambda = sigma lambda0)
};

struct CDParams {
  const double* Xb;
  const double* Gband;     // [nblk][J][2J]: x~_j^T x~_j' / n with j' in the previous block
                           //   (G^x, columns 0..31) and in the same block (G^w, 32..63)
  int n, n_pad, nchunk;
  int p;
  int nblk;
  int64_t col_begin;       // global index of local column 0
  int ncols;               // local columns (queue length)
  double lambda0, tol, sigma_floor, sqrt_n;
  int max_outer, max_inner;
  int T;                   // resident columns per CTA (8, 16, 32)
  int nst;                 // X chunk pipeline stages
  int nzcap;               // per-column capacity of each coefficient list
  int evict_after;         // hand columns that continue after this many sweeps to the tail
                           //   solver (0: never)
  int* tail_count;         // number of columns handed over
  TailState* tail;         // [ncols]
  int* queue;              // atomic head (queue index)
  int* flags;              // FLAG_*
  const int* err_in;       // standardization error code (CD exits early when nonzero)
  int* nz_rows;            // [ncols][2][nzcap]
  double* nz_vals;         // [ncols][2][nzcap]
  int* nz_count;           // [ncols] entries of the final list
  int* nz_cur;             // [ncols] which of the 2 lists is final
  double* sigma_std;       // [ncols]
  int* iters;              // [ncols]
  int* sweeps;             // [ncols]
  uint8_t* converged;      // [ncols]
  // Algorithm 3 joint mode (mode 1): every queued column does exactly one sweep at its current
  // sigma and lambda, starting from its carried residual, then hands its state back
  int joint;
  const int* act;          // [ncols] local column index of each queue entry (active set I)
  double* Ej;              // [m][n_pad] residual e_c carried between launches
  unsigned long long* joint_maxd;   // max over columns of max_j |db_jc| (bits of a double >= 0)
};

struct TailParams {
  const double* Xb;
  int n, n_pad, nchunk, p, nblk;
  int64_t col_begin;
  double lambda0, tol, sigma_floor, sqrt_n;
  int max_outer, max_inner;
  int nzcap;
  const double* lambdas;   // multi-lambda fits: lambda0 of TailState::lam (nullptr: lambda0)
  int slot_stride;         // multi-lambda fits: outputs of (lam, col) at lam * slot_stride + col
  int M;                   // tail columns (or, if M_dev != nullptr, *M_dev at kernel start)
  const int* M_dev;
  const TailState* tail;   // [M]
  const double* Zz;        // [M][p]: z_k = X~^T r_k / n for tail column k
  double* Gtab;            // [p][p]: Gram column G[:, j] = X~^T x~_j / n of variable j
  int* gstate;             // [p]: 0 absent, 1 being computed, 2 ready
  int* next;               // atomic work counter
  int* ondemand_count;     // Gram columns computed on first use
  int* sweeps_count;       // sweeps performed here
  unsigned long long* changes_count;   // optional [2]: coordinate changes (d != 0), passes
  int z_from_gtab;         // 1: z starts as Gtab[:, col] (Gram solver: b = 0, r = x~_c)
  int gtab_full;           // 1: every Gram column is present (no on-demand path)
  int occ;                 // column CTAs per SM the launch provides for (grid multiplier)
  int z2;                  // 1: a second z buffer (tail_z2_bytes more shared memory): a pass
                           //    that finds no new row swaps in z + all chain changes
  double* z2g;             // (z2 == 0) optional [grid][p] global scratch for the multi-sweep mode
  int gate;                // 0: run; 1: run only if the hit counts are skewed (tail_skewed),
                           //   2: only if they are not (two launch shapes, one of which exits)
  int* flags;
  int* nz_rows;            // column coefficient lists (as in CDParams)
  double* nz_vals;
  int* nz_count;
  int* nz_cur;
  double* sigma_std;
  int* iters;
  int* sweeps;
  uint8_t* converged;
  // Algorithm 3 (mode 1) on the Gram form: each launch performs ONE sweep of every listed work
  // item (TailState slots work[0 .. *M_dev)), at lambda = sigma_std[col] lambda0, keeps z in
  // Zj[slot] between launches, max-reduces |db| into joint_maxd and writes the state back; the
  // outer boundary (sigma refit, F_c, compaction) and the sweep counts are the host loop's.
  // optional: the work order by hit count, most first (bhist / tail_key: GramParams'; order:
  // *M_dev entries; order_bar: a zeroed grid-barrier counter)
  const int* bhist;
  const int* tail_key;
  int* order;
  int* order_bar;
  int joint;
  TailState* jtail;                  // [slots] state written back after each sweep
  const int* work;                   // slots to sweep in this launch
  double* Zj;                        // [slots][p]
  unsigned long long* joint_maxd;    // max |db| (double bits; non-negative, so integer max)
};
// Gram solver (gram_full.cu): symmetric S = X~^T X~ / n with fused first-sweep screening.
struct GramParams {
  const double* Xb;
  int n, n_pad, nchunk, p, nblk;
  int64_t col_begin;
  int ncols;
  double lambda0, tol, sigma_floor, sqrt_n;
  int max_outer;
  int nst;
  double* G;               // [p][p] column-major (nullptr: screening only)
  uint8_t* hit;            // [nlam][p] column has some |G_jc| > lambda0_l, j != c
  int* hitcnt;             // optional [p]: number of such j at the screening level (zeroed)
  int* bhist;              // optional [1024]: tail columns per hit-count bucket (zeroed), and
  int* tail_key;           //   per tail entry: bucket << 20 | rank in it (the sweep order)
  const double* ssq;       // optional [p]: x~_c^T x~_c as the standardization summed it
  int nlam;                // penalty levels screened / fitted together (1..SPMESL_MAX_LAM)
  double lams[8];          // their lambda0 values
  int tile_begin, tile_end;   // upper-triangle tiles to process (multi-GPU share)
  double* zero_ptr;        // optional: zero-filled by the producer's bulk stores (Theta)
  size_t zero_count;       // doubles (even; zero_ptr 16-byte aligned)
  double* zero_last;       // optional: one more double to zero (odd Theta sizes)
  const int* cond_nU;      // optional: run only if 2 * *cond_nU > p (solver 3 fallback)
  TailState* tail;         // columns for the sweep kernel
  int* tail_count;
  double* sigma_std;
  int* iters;
  int* sweeps;
  uint8_t* converged;
  int* nz_count;
  int* nz_cur;
};
size_t syrk_smem_bytes(int nst);

// Certified screening: the exact FP64 decision of its nU candidate columns costs 2 n p nU flops
// in gram_cols_kernel (~0.44 of the DMMA peak) against n p (p + 1) in the symmetric Gram kernel
// (~0.9 of it): above p / 4 candidates the full Gram kernel decides instead (measured crossover)
// Exact first-sweep decision of the certified screening's nU candidates (device count): the
// exact Gram columns of the candidates (2 n p nU flops, gram_cols_kernel) for up to p/4 and up
// to 1024 of them, else the full symmetric Gram kernel (n p (p+1) flops).  Only the
// candidates' columns are computed on the first path; a sweep that needs another one computes
// it on first use inside its CTA (about 1 ms each at p = 20000), which more candidates make
// likelier: at config 5 with 1126 candidates (lambda between univ and ub) one such column made
// the fit 12.5 ms against 8.3 with the full kernel.
__host__ __device__ inline bool gram_fallback_taken(int64_t nU, int64_t p) {
  return 4 * nU > p || nU > 1024;
}

// Certified f16 screening (screen16.cu)
struct Screen16Params {
  const __half* Y16;       // normalized f16 tiles
  const double* sq;        // [p] sqrt(N_k)
  const float* inv_sq;     // [ntb*128] 1 / sqrt(N_k) rounded down; +inf past p
  const float* lam_n;      // [ntb*128] n lambda0 / sqrt(N_k) rounded down; 0 past p
  int p, n, ntb, nchunk64;
  int tile_begin, tile_end;
  double lambda0, eps;
  float epsn;              // n eps rounded up (f32 epilogue)
  uint8_t* cand;           // [p] column may have a hit (must be checked exactly)
  double* zero_ptr;        // optional Theta zero fill (as GramParams)
  size_t zero_count;
  double* zero_last;       // optional: one more double to zero (odd Theta sizes)
  float* acc_out;          // optional (tests): raw accumulators n R_hat_jc at [c * acc_ld + j]
  int64_t acc_ld;
};
size_t screen16_y_halves(int64_t p, int n_pad);
int screen16_tile_count(int64_t p);
int64_t screen16_pad(int64_t p);   // p rounded up to the 128-column tiles
double screen16_eps(int n_pad);
cudaError_t launch_screen16(const Screen16Params& P, int grid, cudaStream_t s);
// candidates restricted to the columns [cb, ce) (ce < 0: all p); gstate[c] = 2 for those, else 0
cudaError_t launch_cand_compact(const uint8_t* cand, int p, int* U, int* nU, int* gstate,
                                cudaStream_t s, int cb = 0, int ce = -1);
cudaError_t launch_syrk_screen(const GramParams& P, int grid, cudaStream_t s);
cudaError_t launch_gram_init(const GramParams& P, cudaStream_t s);
cudaError_t launch_level_flags(const GramParams& P, cudaStream_t s);
int gram_tile_count(int64_t p);

constexpr int TAIL_THREADS = 256;   // (the sweep kernel also runs with 512: TAIL_MAXW warps)
constexpr int TAIL_MAXW = 16;
#ifndef SPMESL_TAIL_SCAN_R
#define SPMESL_TAIL_SCAN_R 4
#endif
constexpr int TAIL_SCAN = SPMESL_TAIL_SCAN_R * TAIL_THREADS;   // rows tested per search round
constexpr int TAIL_ODC = 8;          // on-demand Gram column cache entries per CTA
__host__ __device__ size_t tail_smem_bytes(int p, int n_pad, int nzcap);

__host__ __device__ size_t tail_z2_bytes(int p);
cudaError_t launch_tail_residuals(const double* Xb, const TailState* tail, int M, const int* nz_rows,
                                  const double* nz_vals, int nzcap, int64_t col_begin, int n,
                                  int n_pad, int nchunk, double* V, cudaStream_t s);
// Exact Gram columns of a candidate list U (count nU, or *nU_dev read on the device; with a
// device count and gram_fallback_taken(nU, p) the kernel only sets gstate[:] = 2 — the full Gram
// kernel decides)
cudaError_t launch_gram_cols(const double* Xb, int nblk, int nchunk, int n, int p, const int* U,
                             int nU, const int* nU_dev, int sms, double* Gtab, uint8_t* hit,
                             const double* lams, int nlam, int* gstate, cudaStream_t s,
                             bool fallback = true, double lam1 = 0.0);   // lams == nullptr: lam1

// hit (optional): hit[l p + c] = 1 for every candidate c = U[.] with some |G_jc| > lams[l], j != c
// (hit must be zeroed first; only ones are written)
cudaError_t launch_gram_pass(const double* Xb, int nblk, int nchunk, int n, int p, const double* V,
                             int M, const int* U, int nU, double* Zz, double* Gtab, cudaStream_t s,
                             uint8_t* hit = nullptr, const double* lams = nullptr, int nlam = 0);
cudaError_t launch_tail_mark(const TailState* tail, int M, const int* nz_rows, int nzcap, int* umark,
                             cudaStream_t s);
cudaError_t launch_tail_sweeps(const TailParams& P, int grid, cudaStream_t s);


// Algorithm 3 joint mode helpers (joint.cu)
cudaError_t launch_joint_live_init(const uint8_t* hit, int m, int* nslots, TailState* jtail,
                                   int* slotmap, cudaStream_t s);
cudaError_t launch_joint_work(const int* act, int nact, const int* slotmap, int* work, int* nwork,
                              cudaStream_t s);
cudaError_t launch_joint_live_add(const int* act, int nact, int* slotmap, TailState* jtail,
                                  int* nslots, const int* nz_cur, cudaStream_t s);
cudaError_t launch_joint_count_unslotted(const int* act, int nact, const int* slotmap, int* cnt,
                                         cudaStream_t s);
cudaError_t launch_joint_add_sweeps(const int* act, int nact, int inner, int* sweeps, cudaStream_t s);
cudaError_t launch_joint_init(const double* Xb, int64_t col_begin, int m, int n_pad, int nchunk,
                              int* act, double* sigma, double* Ej, cudaStream_t s);
cudaError_t launch_joint_sigma(const double* Xb, int64_t col_begin, const int* act, int nact,
                               const int* nz_rows, const double* nz_vals, const int* nz_count,
                               const int* nz_cur, int nzcap, int n, int n_pad, int nchunk,
                               double sqrt_n, double sigma_floor, double tol, int capped,
                               double* sigma, int* iters, uint8_t* jflags, uint8_t* converged,
                               double* Ej, uint8_t* keep, cudaStream_t s);
cudaError_t launch_joint_compact(const int* act, const uint8_t* keep, int nact, int* act_out,
                                 int* nact_out, cudaStream_t s);

size_t cd_smem_bytes(int T, int n_pad);          // with the minimum 2 stages
int cd_stages(int T, int n_pad, size_t smem_optin);  // stages that fit (0: does not fit)

// Launchers (stream-ordered, no host synchronisation).
// Optional outputs of the standardization for the certified f16 screening (screen16.cu):
// y_k = x~_k / sqrt(N_k) as f16 tiles, sq_k = sqrt(N_k), inv_sq / lam_n (directed roundings),
// including the zero / +inf padding up to p_pad.  Replaces to_f16 + sqrt kernels.
struct S16Prep {
  __half* Y16;
  int nchunk64;
  int64_t p_pad;
  double* sq;
  float* inv_sq;
  float* lam_n;
  double lambda0;
};
cudaError_t launch_standardize(const double* X, const Layout& L, int standardize, double* Xb,
                               double* mu, double* scale, int* err, unsigned long long* bad_key,
                               cudaStream_t s, double* nrm = nullptr, const S16Prep* y = nullptr,
                               double* ssq = nullptr);
cudaError_t launch_gram(const double* Xb, const Layout& L, double* Gband, cudaStream_t s);
cudaError_t launch_cd(const CDParams& P, int num_ctas, cudaStream_t s);
cudaError_t launch_csc_build(const int* nz_count, const int* nz_cur, const int* nz_rows,
                             const double* nz_vals, int ncols, int nzcap, int64_t* col_ptr,
                             int32_t* rows, double* vals, int64_t* total, cudaStream_t s);
cudaError_t launch_assemble_coo(int64_t p, const int64_t* col_ptr, const int32_t* rows,
                                const double* vals, const double* sigma_std, const double* scale,
                                int symmetrize, int32_t* coo_row, int32_t* coo_col, double* coo_val,
                                int* coo_count, double* diag, double* sigma_out, cudaStream_t s);
cudaError_t launch_column_stats(const int32_t* iters, const int32_t* sweeps, const uint8_t* conv,
                                int64_t m, unsigned long long* tot, int* mx_sweeps, int* mx_outer,
                                int* nunc, cudaStream_t s, unsigned long long* t_end = nullptr);
cudaError_t launch_zero_fill(double* a, size_t count, int sms, cudaStream_t s);
cudaError_t launch_zero_fill_bulk(double* a, size_t count, int grid, cudaStream_t s);
// (z0 / z1: optional extra byte ranges to zero in the same launch)
cudaError_t launch_reset(void* counters, int counters_bytes, int key_off, int t_off, int* queue,
                         int* nz_count, int* nz_cur, int64_t m, cudaStream_t s,
                         void* z0 = nullptr, size_t z0_bytes = 0, void* z1 = nullptr,
                         size_t z1_bytes = 0);
cudaError_t launch_csc_counts(const int* nz_count, int ncols, int32_t* out, cudaStream_t s);
cudaError_t launch_sparse_count(int64_t p, const int* cnt, const int* cur, const int* nz_rows,
                                const double* nz_vals, int nzcap, int symmetrize, int* ccount,
                                cudaStream_t s);
cudaError_t launch_sparse_write(int64_t p, const int* cnt, const int* cur, const int* nz_rows,
                                const double* nz_vals, int nzcap, const double* sigma_std,
                                const double* scale, int symmetrize, const int64_t* col_ptr,
                                int32_t* rows, double* vals, double* sigma_out, cudaStream_t s,
                                int64_t cap = -1);   // cap >= 0: write only if nnz <= cap
cudaError_t launch_csc_scan(const int* cnt, int ncols, int64_t* col_ptr, int64_t* total,
                            cudaStream_t s);
// Peer-to-peer exchange of the multi-device fit (assemble.cu; multi.cu): the column blocks of
// all G devices as pointers valid on the launching device (its own, or peers' through
// cudaDeviceEnablePeerAccess).  Block e holds columns column_range(p, e, G).
constexpr int kP2PMax = 16;
struct P2PBlocks {
  int64_t p;
  int G;
  const uint8_t* flags[kP2PMax];       // screening flags of the device's tile share [p]
  const int64_t* col_ptr[kP2PMax];     // block-local CSC column pointers [m_e + 1]
  const int32_t* rows[kP2PMax];        // rows ascending per column
  const double* vals[kP2PMax];         // b_jk
  const double* sigma_std[kP2PMax];    // sigma_k of the block's columns [m_e]
};
cudaError_t launch_p2p_flag_max(const P2PBlocks& B, uint8_t* out, cudaStream_t s);
cudaError_t launch_assemble_coo_p2p(const P2PBlocks& B, int self, const double* scale,
                                    int symmetrize, int32_t* coo_row, int32_t* coo_col,
                                    double* coo_val, int* coo_count, double* diag,
                                    double* sigma_out, cudaStream_t s);
// fit statistics gathered by the assembly (fused column_stats_kernel; sweeps == NULL: none)
struct ColStats {
  const int32_t* iters;
  const int32_t* sweeps;
  const uint8_t* conv;
  unsigned long long* tot;
  int* mx_sweeps;
  int* mx_outer;
  int* nunc;
  unsigned long long* t_end;
};
cudaError_t launch_assemble_lists(int64_t p, const int* nz_count, const int* nz_cur,
                                  const int* nz_rows, const double* nz_vals, int nzcap,
                                  const double* sigma_std, const double* scale, int symmetrize,
                                  double* Theta, double* sigma_out, int64_t* nnz_total,
                                  cudaStream_t s, const ColStats* cs = nullptr);
cudaError_t launch_assemble(int64_t p, int64_t col_begin, int64_t col_end, const int64_t* col_ptr,
                            const int32_t* rows, const double* vals, const double* sigma_std,
                            const double* scale, int symmetrize, double* Theta, double* sigma_out,
                            cudaStream_t s, bool zero_fill = true);

}  // namespace spmesl
