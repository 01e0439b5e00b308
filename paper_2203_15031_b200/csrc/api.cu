// Host orchestration and C ABI (include/spmesl.h).  Validation, per-device cached
// workspace, kernel sequencing on the caller's stream, error/stat readback.
//
// Device sequence of one fit:
//   memset scratch -> standardize_kernel (a2) -> gram_kernel -> cd_sweep_kernel (a3-a7)
//   -> csc_scan + csc_copy -> memset Theta + assemble_entries + assemble_diag (a8, a10)
//   -> one 64-byte readback of flags/counters.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "spmesl.h"
#include "spmesl_internal.cuh"

using namespace spmesl;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? SPMESL_ERR_OOM : SPMESL_ERR_CUDA,      \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                     \
  } while (0)

// Device counters written by the kernels and read back once per call.
struct DevCounters {
  int err;                      // standardization error seen
  int overflow;                 // a coefficient list exceeded nzcap
  int tail_count;               // columns handed to the tail solver
  int tail_next;                // tail solver work counter
  int gram_ondemand;            // Gram columns computed on first use by the tail solver
  int coo_count;                // host API: nonzero entries of Theta emitted as COO
  int tail_sweeps;              // sweeps performed by the tail solver
  int joint_nact;               // mode 1: active columns after the last compaction
  unsigned long long bad_key;   // 2*col + (0 nonfinite | 1 constant)
  int64_t csc_total;
  unsigned long long joint_maxd;   // mode 1: max |db| of the last sweep (double bits)
  unsigned long long st_sweeps;    // column statistics (column_stats_kernel)
  int st_max_sweeps, st_max_outer, st_unconv, pad4;
  int s16_nU, pad5;                // solver 3: candidate columns of the certified screening
  int joint_nslots, joint_nwork;   // mode 1 on the Gram form: sweep slots, slots this sweep
  unsigned long long t_start, t_end;   // device clock (ns) at the fit's first / last kernel
  unsigned long long tail_changes;     // coordinate changes made by the sweep kernel
  unsigned long long tail_passes;      // its chain + pass segments
  int tail_ordered, pad6;              // the sweep kernel's work-order grid barrier
};

struct Buffer {
  void* ptr = nullptr;
  size_t bytes = 0;
};

// bumped on every (re)allocation: a captured CUDA graph is only valid while no buffer moved
std::atomic<uint64_t> g_alloc_gen{0};

int ensure(Buffer& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return SPMESL_OK;
  g_alloc_gen.fetch_add(1);
  if (b.ptr) cudaFree(b.ptr);
  b.ptr = nullptr;
  b.bytes = 0;
  cudaError_t e = cudaMalloc(&b.ptr, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(SPMESL_ERR_OOM, "cudaMalloc(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  }
  b.bytes = bytes;
  return SPMESL_OK;
}

struct Workspace {
  std::mutex mu;
  int device = -1;
  int sms = 0;
  int smem_optin = 0;
  int smem_sm = 0;      // shared memory per SM (all resident CTAs)
  int cc_major = 0;
  Buffer xb, gband, mean, scale, counters, queue, sigma_std, iters, sweeps, conv, nz_count, nz_cur,
      nz_rows, nz_vals, col_ptr, csc_rows, csc_vals;
  Buffer tail, tail2, umark, umap, uvars, tailV, zall, ondemand;   // tail solver (tail2: order)
  Buffer z2g;                                                      // its global second z buffers
  Buffer ej, act0, act1, keep, jflags;                      // mode 1 (Algorithm 3)
  Buffer jtail, slotmap, jwork, zj;                         // mode 1 on the Gram form
  Buffer hit;                                               // Gram solver screening flags
  Buffer lam_dev;                                           // multi-lambda: penalty levels
  Buffer nrm, sq, y16, cand;                                // certified f16 screening
  Buffer ssq;                                               // x~_c^T x~_c (Gram solvers)
  Buffer ccount;                                            // sparse Theta: entries per column
  // host-API staging
  Buffer hx, htheta, hsigma, hiters, hsweeps, hconv, coo_r, coo_c, coo_v, hdiag, zeros;
  DevCounters* host_counters = nullptr;   // pinned
  cudaEvent_t ev[10] = {};   // [8], [9]: around the screening kernel
  cudaStream_t side = nullptr;            // Theta zero-fill overlapped with the CD kernel
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double* pending_zero = nullptr;         // Theta to zero-fill once standardization is done
  size_t pending_count = 0;
  double* take_zero = nullptr;            // Theta the Gram kernel may zero-fill itself
  size_t take_count = 0;
  double* lam_pinned = nullptr;           // staging of the penalty levels (pinned, H2D)
  // CUDA-graph replay of the device-path fit: the whole enqueue is captured
  // once per argument set and replayed with one launch
  cudaStream_t cap = nullptr;             // capture stream
  bool capturing = false;                 // timing events become external record nodes
  cudaGraphExec_t gexec = nullptr;
  std::vector<unsigned char> gkey;        // arguments of the captured graph
  std::vector<unsigned char> last_key;    // arguments of the previous eager device-path fit
  int graph_nzcap = 0;                    // coefficient-list capacity the graph was built for
  // sparse-output fit (spmesl_fit_sparse_device): Theta as CSC instead of the dense array
  struct SparseOut { int64_t* col_ptr; int32_t* rows; double* vals; int64_t cap; };
  const SparseOut* sparse = nullptr;
  int64_t graph_screen_fill = 0;          // host-side facts of the captured fit (for its stats)
  int graph_launches = 0;
  bool zero_join = false;     // part of Theta's zero fill runs on `side` (join ev_join)
  int64_t screen_fill = 0;    // doubles of Theta the screening kernel zero-filled (last fit)
  int gram_launches = 0;      // kernels fit_gram_enqueue launched (last fit)
  // auto solver: the arguments (X, n, p, lambda0, tol, max_iter, options, outputs) of the last
  // fit whose certified screening fell back to the full FP64 Gram kernel — a repeat runs the full
  // Gram path directly (fit_device_impl)
  std::vector<unsigned char> auto_full_key;
  // ... and of the last fit whose screening left few candidates: a repeat launches the exact
  // Gram columns without the full Gram kernel behind them (which would only exit)
  std::vector<unsigned char> auto_few_key;
  bool no_fallback = false;   // (fit_gram_enqueue, screening path: no fallback launch)
  bool init = false;
};

// Timing events: inside a graph capture they must be external record nodes (recorded at every
// replay), not the intra-graph dependency a plain record becomes.
// Each external record node costs a few microseconds of idle GPU between its neighbours, so
// a captured fit keeps only the events of ms_total (ev[0], ev[4]) and of the screening kernel
// (ev[8], ev[9], the roofline's denominator); the other phase times read -1 after a replay.
cudaError_t ev_record(const Workspace& W, cudaEvent_t e, cudaStream_t s) {
  if (!W.capturing) return cudaEventRecord(e, s);
  if (e != W.ev[8] && e != W.ev[9]) return cudaSuccess;   // (ms_total: the device clock)
  return cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
}

std::mutex g_ws_mu;
std::vector<Workspace*> g_ws;

Workspace* workspace_for(int dev) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if ((int)g_ws.size() <= dev) g_ws.resize(dev + 1, nullptr);
  if (!g_ws[dev]) g_ws[dev] = new Workspace();
  return g_ws[dev];
}

int ws_init(Workspace& W, int dev) {
  if (W.init) return SPMESL_OK;
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  W.device = dev;
  W.sms = prop.multiProcessorCount;
  W.smem_optin = (int)prop.sharedMemPerBlockOptin;
  W.smem_sm = (int)prop.sharedMemPerMultiprocessor;
  W.cc_major = prop.major;
  CUDA_TRY(cudaMallocHost((void**)&W.host_counters, sizeof(DevCounters)));
  CUDA_TRY(cudaMallocHost((void**)&W.lam_pinned, sizeof(double) * SPMESL_MAX_LAM));
  CUDA_TRY(cudaStreamCreateWithFlags(&W.cap, cudaStreamNonBlocking));
  for (auto& e : W.ev) CUDA_TRY(cudaEventCreate(&e));
  CUDA_TRY(cudaStreamCreateWithFlags(&W.side, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&W.ev_fork, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&W.ev_join, cudaEventDisableTiming));
  W.init = true;
  return SPMESL_OK;
}

int validate(const void* X, int64_t n, int64_t p, double lambda0, double tol, int32_t max_iter,
             const spmesl_options& o) {
  if (!X) return fail(SPMESL_ERR_ARG, "X is NULL");
  if (n < 2) return fail(SPMESL_ERR_ARG, "n must be >= 2");
  if (p < 2) return fail(SPMESL_ERR_ARG, "p must be >= 2");
  if (p > (int64_t)0x7fffffff) return fail(SPMESL_ERR_ARG, "p must be < 2^31");
  if (n > (int64_t)0x7fff0000) return fail(SPMESL_ERR_ARG, "n must be < 2^31 - 2^16");
  if (!(lambda0 >= 0.0) || !std::isfinite(lambda0)) return fail(SPMESL_ERR_ARG, "lambda0 must be finite and >= 0");
  if (!(tol > 0.0) || !std::isfinite(tol)) return fail(SPMESL_ERR_ARG, "tol must be finite and > 0");
  if (max_iter < 1) return fail(SPMESL_ERR_ARG, "max_iter must be >= 1");
  if (o.max_inner < 1) return fail(SPMESL_ERR_ARG, "max_inner must be >= 1");
  if (!(o.sigma_floor > 0.0)) return fail(SPMESL_ERR_ARG, "sigma_floor must be > 0");
  if (o.mode != 0 && o.mode != 1) return fail(SPMESL_ERR_ARG, "mode must be 0 (per-column stop) or 1 (Algorithm 3 joint stop)");
  if (o.solver < 0 || o.solver > 3) return fail(SPMESL_ERR_ARG, "solver must be 0, 1, 2 or 3");
  if (o.num_devices < 0 || o.num_devices > 64) return fail(SPMESL_ERR_ARG, "num_devices must be 0 .. 64");
  if (o.exchange < 0 || o.exchange > 2) return fail(SPMESL_ERR_ARG, "exchange must be 0 (auto), 1 (NCCL) or 2 (peer-to-peer)");
  if (o.tile_cols != 0 && o.tile_cols != 8 && o.tile_cols != 16 && o.tile_cols != 32)
    return fail(SPMESL_ERR_ARG, "tile_cols must be 0, 8, 16 or 32");
  const double pp = (double)p * (double)p * 8.0;
  if (pp > 9.0e18) return fail(SPMESL_ERR_OOM, "p*p*8 overflows");
  return SPMESL_OK;
}

spmesl_options resolve(const spmesl_options* opt) {
  spmesl_options o;
  spmesl_default_options(&o);
  if (opt) {
    if (opt->struct_size != (int32_t)sizeof(spmesl_options)) {
      // tolerate older/newer callers by copying the common prefix
      size_t m = opt->struct_size > 0 ? std::min((size_t)opt->struct_size, sizeof(o)) : sizeof(o);
      std::memcpy(&o, opt, m);
      o.struct_size = sizeof(o);
    } else {
      o = *opt;
    }
  }
  return o;
}

int choose_T(const Workspace& W, int64_t ncols, int n_pad, int requested) {
  const int cands[3] = {32, 16, 8};
  int fallback = 0;
  for (int T : cands) {
    if (requested && T != requested) continue;
    if (cd_stages(T, n_pad, W.smem_optin) < 4) continue;
    if (!fallback) fallback = T;
    if (requested || (ncols + T - 1) / T >= W.sms || T == 8) return T;
  }
  return fallback;
}

struct FitOut {
  int64_t col_begin, col_end;
  double* sigma_std;
  int32_t* iters;
  int32_t* sweeps;
  uint8_t* conv;
};

// Sweep-kernel launch shape: two column CTAs per SM whenever their state fits side
// by side (their latency-bound chains and passes interleave), preferably each with the second z
// buffer (a pass without a new row then commits by swapping buffers instead of re-reading the
// chain's Gram columns in the next pass); else one CTA of 512 threads per SM.
void set_tail_shape(const Workspace& W, TailParams& T) {
  const size_t base = tail_smem_bytes(T.p, T.n_pad, T.nzcap);
  const size_t z2b = tail_z2_bytes(T.p);
  const size_t sm = (size_t)W.smem_sm, optin = (size_t)W.smem_optin;
  if (2 * (base + z2b + 1024) <= sm && base + z2b <= optin) { T.occ = 2; T.z2 = 1; }
  else if (2 * (base + 1024) <= sm) { T.occ = 2; T.z2 = 0; }
  else { T.occ = 1; T.z2 = base + z2b <= optin ? 1 : 0; }
}

bool tail_enabled(const Workspace& W, const spmesl_options& o, const Layout& L, int nzcap) {
  // (the fit-wide Gram table is p x p doubles: keep it under 16 GB)
  return o.tail_after > 0 && tail_smem_bytes((int)L.p, L.n_pad, nzcap) <= (size_t)W.smem_optin &&
         (double)L.p * (double)L.p * 8.0 <= 16e9;
}

// Tail solver for the columns the CD kernel handed over: fresh residuals, one
// batched DMMA pass for z = X~^T r / n and the Gram columns of every active variable, then the
// covariance-update sweeps.  Host work: the union of active variables (a p-flag readback).
int run_tail(Workspace& W, const Layout& L, int64_t cb, double lambda0, double tol,
             int32_t max_iter, const spmesl_options& o, int nzcap, const FitOut& out, int M,
             cudaStream_t s, spmesl_stats* st) {
  const int p = (int)L.p;
  int rc;
  // active variables of the handed-over columns (device marks, one readback)
  if ((rc = ensure(W.umark, (size_t)p * 4))) return rc;
  CUDA_TRY(cudaMemsetAsync(W.umark.ptr, 0, (size_t)p * 4, s));
  CUDA_TRY(launch_tail_mark((const TailState*)W.tail.ptr, M, (const int*)W.nz_rows.ptr, nzcap,
                            (int*)W.umark.ptr, s));
  std::vector<int> mark(p);
  CUDA_TRY(cudaMemcpyAsync(mark.data(), W.umark.ptr, (size_t)p * 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  // Gram columns to precompute: the active variables, or all p when the tail is large (the
  // others are computed on first use by the tail kernel, once per fit)
  std::vector<int> U;
  const bool all = (int64_t)M * 16 > p;
  for (int j = 0; j < p; ++j)
    if (all || mark[j]) U.push_back(j);
  const int nU = (int)U.size();
  if ((rc = ensure(W.uvars, (size_t)std::max(nU, 1) * 4))) return rc;
  if ((rc = ensure(W.umap, (size_t)p * 4))) return rc;             // gstate
  if ((rc = ensure(W.tailV, (size_t)M * L.n_pad * 8))) return rc;
  if ((rc = ensure(W.zall, (size_t)M * p * 8))) return rc;
  if ((rc = ensure(W.ondemand, (size_t)p * p * 8))) return rc;     // Gtab
  int grid = std::min(M, W.sms);
  std::vector<int> gstate(p, 0);
  for (int j : U) gstate[j] = 2;
  CUDA_TRY(cudaMemcpyAsync(W.umap.ptr, gstate.data(), (size_t)p * 4, cudaMemcpyHostToDevice, s));
  if (nU) CUDA_TRY(cudaMemcpyAsync(W.uvars.ptr, U.data(), (size_t)nU * 4, cudaMemcpyHostToDevice, s));
  CUDA_TRY(ev_record(W, W.ev[5], s));
  CUDA_TRY(launch_tail_residuals((const double*)W.xb.ptr, (const TailState*)W.tail.ptr, M,
                                 (const int*)W.nz_rows.ptr, (const double*)W.nz_vals.ptr, nzcap, cb,
                                 (int)L.n, L.n_pad, L.nchunk, (double*)W.tailV.ptr, s));
  CUDA_TRY(launch_gram_pass((const double*)W.xb.ptr, (int)L.nblk, L.nchunk, (int)L.n, p,
                            (const double*)W.tailV.ptr, M, (const int*)W.uvars.ptr, nU,
                            (double*)W.zall.ptr, (double*)W.ondemand.ptr, s));
  DevCounters* dc = (DevCounters*)W.counters.ptr;
  TailParams T{};
  T.Xb = (const double*)W.xb.ptr;
  T.n = (int)L.n; T.n_pad = L.n_pad; T.nchunk = L.nchunk; T.p = p; T.nblk = (int)L.nblk;
  T.col_begin = cb;
  T.lambda0 = lambda0; T.tol = tol; T.sigma_floor = o.sigma_floor; T.sqrt_n = std::sqrt((double)L.n);
  T.max_outer = max_iter; T.max_inner = o.max_inner;
  T.nzcap = nzcap;
  T.M = M;
  T.tail = (const TailState*)W.tail.ptr;
  T.Zz = (const double*)W.zall.ptr;
  T.Gtab = (double*)W.ondemand.ptr;
  T.gstate = (int*)W.umap.ptr;
  T.next = &dc->tail_next;
  T.ondemand_count = &dc->gram_ondemand;
  T.sweeps_count = &dc->tail_sweeps;
  T.changes_count = &dc->tail_changes;
  T.flags = &dc->err;
  T.nz_rows = (int*)W.nz_rows.ptr; T.nz_vals = (double*)W.nz_vals.ptr;
  T.nz_count = (int*)W.nz_count.ptr; T.nz_cur = (int*)W.nz_cur.ptr;
  T.sigma_std = out.sigma_std; T.iters = out.iters; T.sweeps = out.sweeps; T.converged = out.conv;
  set_tail_shape(W, T);
  CUDA_TRY(launch_tail_sweeps(T, grid, s));
  CUDA_TRY(ev_record(W, W.ev[6], s));   // end of the tail solver
  if (st) { st->tail_columns = M; st->kernel_launches += 4; }
  return SPMESL_OK;
}

// Scratch reset + standardize (a2) + Gram band for columns [cb, cb + m) on stream s.
// (Xb's padding is written by the standardization itself; y16: the certified screening's
// operands, written by the same kernel)
int run_prep(Workspace& W, const double* dX, int64_t m, const spmesl_options& o, const Layout& L,
             cudaStream_t s, bool band = true, const S16Prep* y16 = nullptr,
             void* z0 = nullptr, size_t z0_bytes = 0, void* z1 = nullptr, size_t z1_bytes = 0) {
  CUDA_TRY(launch_reset(W.counters.ptr, (int)sizeof(DevCounters), (int)offsetof(DevCounters, bad_key),
                        (int)offsetof(DevCounters, t_start), (int*)W.queue.ptr,
                        (int*)W.nz_count.ptr, (int*)W.nz_cur.ptr, m, s, z0, z0_bytes, z1,
                        z1_bytes));
  CUDA_TRY(ev_record(W, W.ev[0], s));
  DevCounters* dc = (DevCounters*)W.counters.ptr;
  CUDA_TRY(launch_standardize(dX, L, o.standardize, (double*)W.xb.ptr, (double*)W.mean.ptr,
                              (double*)W.scale.ptr, &dc->err, &dc->bad_key, s,
                              W.nrm.bytes >= (size_t)L.p * 8 ? (double*)W.nrm.ptr : nullptr,
                              y16, W.ssq.bytes >= (size_t)L.p * 8 ? (double*)W.ssq.ptr : nullptr));
  if (band) CUDA_TRY(launch_gram((const double*)W.xb.ptr, L, (double*)W.gband.ptr, s));
  CUDA_TRY(ev_record(W, W.ev[1], s));
  if (W.pending_zero) {
    // Theta's zero fill (HBM-bound) overlaps the solver (compute-bound), not standardization
    CUDA_TRY(cudaStreamWaitEvent(W.side, W.ev[1], 0));
    CUDA_TRY(launch_zero_fill(W.pending_zero, W.pending_count, W.sms, W.side));
    CUDA_TRY(cudaEventRecord(W.ev_join, W.side));
    W.pending_zero = nullptr;
  }
  return SPMESL_OK;
}

CDParams cd_params(Workspace& W, const Layout& L, int64_t cb, int64_t m, double lambda0,
                   double tol, int32_t max_iter, const spmesl_options& o, int nzcap,
                   const FitOut& out, int T) {
  DevCounters* dc = (DevCounters*)W.counters.ptr;
  CDParams P{};
  P.Xb = (const double*)W.xb.ptr;
  P.Gband = (const double*)W.gband.ptr;
  P.n = (int)L.n;
  P.n_pad = L.n_pad;
  P.nchunk = L.nchunk;
  P.p = (int)L.p;
  P.nblk = (int)L.nblk;
  P.col_begin = cb;
  P.ncols = (int)m;
  P.lambda0 = lambda0;
  P.tol = tol;
  P.sigma_floor = o.sigma_floor;
  P.sqrt_n = std::sqrt((double)L.n);
  P.max_outer = max_iter;
  P.max_inner = o.max_inner;
  P.T = T;
  P.nst = cd_stages(T, L.n_pad, W.smem_optin);
  P.nzcap = nzcap;
  P.evict_after = tail_enabled(W, o, L, nzcap) ? o.tail_after : 0;
  P.tail_count = &dc->tail_count;
  P.tail = (TailState*)W.tail.ptr;
  P.queue = (int*)W.queue.ptr;
  P.flags = &dc->err;   // FLAG_CODE (unused by CD), FLAG_OVERFLOW at +1
  P.err_in = &dc->err;
  P.nz_rows = (int*)W.nz_rows.ptr;
  P.nz_vals = (double*)W.nz_vals.ptr;
  P.nz_count = (int*)W.nz_count.ptr;
  P.nz_cur = (int*)W.nz_cur.ptr;
  P.sigma_std = out.sigma_std;
  P.iters = out.iters;
  P.sweeps = out.sweeps;
  P.converged = out.conv;
  return P;
}

// Core: standardize + gram + CD for columns [cb, ce) on stream s.  Leaves the coefficient
// lists in the workspace (nz_*), per-column results in `out`.  Returns after enqueueing.
int run_cd(Workspace& W, const double* dX, int64_t n, int64_t p, int64_t cb, int64_t ce,
           double lambda0, double tol, int32_t max_iter, const spmesl_options& o, int nzcap,
           const FitOut& out, cudaStream_t s, int T, Layout& L, int* num_ctas) {
  const int64_t m = ce - cb;
  int rc;
  if ((rc = run_prep(W, dX, m, o, L, s))) return rc;
  CDParams P = cd_params(W, L, cb, m, lambda0, tol, max_iter, o, nzcap, out, T);
  const int ctas = (int)std::min<int64_t>(W.sms, (m + T - 1) / T);
  *num_ctas = ctas;
  CUDA_TRY(launch_cd(P, ctas, s));
  CUDA_TRY(ev_record(W, W.ev[2], s));
  return SPMESL_OK;
}

int alloc_core(Workspace& W, const Layout& L, int64_t m, int nzcap) {
  int rc;
  if ((rc = ensure(W.xb, L.xb_doubles() * 8))) return rc;
  if ((rc = ensure(W.gband, (size_t)L.nblk * J * 2 * J * 8))) return rc;
  if ((rc = ensure(W.mean, (size_t)L.p * 8))) return rc;
  if ((rc = ensure(W.scale, (size_t)L.p * 8))) return rc;
  if ((rc = ensure(W.counters, sizeof(DevCounters)))) return rc;
  if ((rc = ensure(W.queue, 16))) return rc;
  if ((rc = ensure(W.nz_count, (size_t)m * 4))) return rc;
  if ((rc = ensure(W.nz_cur, (size_t)m * 4))) return rc;
  if ((rc = ensure(W.nz_rows, (size_t)m * 2 * nzcap * 4))) return rc;
  if ((rc = ensure(W.nz_vals, (size_t)m * 2 * nzcap * 8))) return rc;
  if ((rc = ensure(W.col_ptr, (size_t)(m + 1) * 8))) return rc;
  if ((rc = ensure(W.tail, (size_t)m * sizeof(TailState)))) return rc;
  return SPMESL_OK;
}

int read_counters(Workspace& W, cudaStream_t s) {
  CUDA_TRY(cudaMemcpyAsync(W.host_counters, W.counters.ptr, sizeof(DevCounters),
                           cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return SPMESL_OK;
}

int std_error(Workspace& W, spmesl_stats* st) {
  const unsigned long long key = W.host_counters->bad_key;
  const int64_t col = (int64_t)(key >> 1);
  if (st) st->bad_column = col;
  if (key & 1ull)
    return fail(SPMESL_ERR_CONSTANT_COLUMN, "constant column " + std::to_string(col));
  return fail(SPMESL_ERR_NONFINITE, "non-finite value in column " + std::to_string(col));
}

int initial_nzcap(int64_t n, int64_t p) {
  int64_t c = ((n + 31) / 32) * 32 + 64;
  if (c > p) c = p;
  if (c < 8) c = 8;
  return (int)c;
}

// Per-column statistics computed on the device into the counters (read with them).
int device_stats(Workspace& W, const int32_t* dIters, const int32_t* dSweeps, const uint8_t* dConv,
                 int64_t m, cudaStream_t s) {
  DevCounters* dc = (DevCounters*)W.counters.ptr;
  // (st_* start at zero: every fit resets the whole counter block in run_prep)
  CUDA_TRY(launch_column_stats(dIters, dSweeps, dConv, m, &dc->st_sweeps, &dc->st_max_sweeps,
                               &dc->st_max_outer, &dc->st_unconv, s, &dc->t_end));
  return SPMESL_OK;
}

void stats_from_counters(const DevCounters& c, int64_t p, spmesl_stats* st, int* any_unconv) {
  *any_unconv = c.st_unconv > 0;
  if (st) {
    st->total_sweeps = (int64_t)c.st_sweeps;
    st->coord_updates = (int64_t)c.st_sweeps * (p - 1);
    st->max_sweeps = c.st_max_sweeps;
    st->max_outer = c.st_max_outer;
    st->n_unconverged = c.st_unconv;
  }
}

// n eps rounded upwards to f32 (the product of the two doubles is rounded first; the margin
// 2^-40 relative covers that rounding)
float screen16_epsn(int64_t n, double eps) {
  const double ne = (double)n * eps * (1.0 + 0x1p-40);
  float f = (float)ne;
  if ((double)f < ne) f = std::nextafter(f, INFINITY);
  return f;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) { cudaGetLastError(); return 0.f; }
  return ms;
}

int current_device(int requested, int* dev) {
  if (requested >= 0) CUDA_TRY(cudaSetDevice(requested));
  CUDA_TRY(cudaGetDevice(dev));
  return SPMESL_OK;
}

void set_layout(Layout& L, int64_t n, int64_t p) {
  L.n = n;
  L.p = p;
  L.n_pad = (int)(((n + KC - 1) / KC) * KC);
  L.nchunk = L.n_pad / KC;
  L.nblk = (p + J - 1) / J;
}

// Mode 1: Algorithm 3 for columns [cb, ce).  Host loop: one CD-kernel launch per
// joint sweep (every active column sweeps once at lambda_c = sigma_c lambda0, residuals carried
// in Ej), then the joint stop on max |db| (one 8-byte readback); at the outer boundary
// the sigma kernel (fresh residuals) and the order-preserving compaction of the
// active set.  Coefficient lists regrow on overflow like mode 0.
int fit_joint_core(Workspace& W, const double* dX, int64_t n, int64_t p, int64_t cb, int64_t ce,
                   double lambda0, double tol, int32_t max_iter, const spmesl_options& o,
                   const FitOut& out, cudaStream_t s, spmesl_stats* st, Layout& L,
                   int* nzcap_used) {
  const int64_t m = ce - cb;
  set_layout(L, n, p);
  if (!choose_T(W, m, L.n_pad, o.tile_cols))
    return fail(SPMESL_ERR_UNSUPPORTED, "n = " + std::to_string(n) +
                                            " does not fit the on-chip residual tile");
  DevCounters* dc = (DevCounters*)W.counters.ptr;
  int nzcap = initial_nzcap(n, p);
  for (int attempt = 0; attempt < 4; ++attempt) {
    int rc = alloc_core(W, L, m, nzcap);
    if (rc) return rc;
    if ((rc = ensure(W.ej, (size_t)m * L.n_pad * 8))) return rc;
    if ((rc = ensure(W.act0, (size_t)m * 4))) return rc;
    if ((rc = ensure(W.act1, (size_t)m * 4))) return rc;
    if ((rc = ensure(W.keep, (size_t)m))) return rc;
    if ((rc = ensure(W.jflags, (size_t)m))) return rc;
    dc = (DevCounters*)W.counters.ptr;
    if ((rc = run_prep(W, dX, m, o, L, s))) return rc;
    CUDA_TRY(cudaMemsetAsync(out.iters, 0, 4 * (size_t)m, s));
    CUDA_TRY(cudaMemsetAsync(out.sweeps, 0, 4 * (size_t)m, s));
    CUDA_TRY(cudaMemsetAsync(out.conv, 0, (size_t)m, s));
    CUDA_TRY(cudaMemsetAsync(W.jflags.ptr, 0, (size_t)m, s));
    CUDA_TRY(launch_joint_init((const double*)W.xb.ptr, cb, (int)m, L.n_pad, L.nchunk,
                               (int*)W.act0.ptr, out.sigma_std, (double*)W.ej.ptr, s));
    if ((rc = read_counters(W, s))) return rc;
    if (W.host_counters->err) return std_error(W, st);
    int* act = (int*)W.act0.ptr;
    int* act_next = (int*)W.act1.ptr;
    int nact = (int)m, launches = 3, T0 = 0, ctas0 = 0;
    bool overflow = false;
    for (int r = 0; r < max_iter && nact > 0 && !overflow; ++r) {
      int inner = 0;
      double jm = 0.0;
      do {
        CUDA_TRY(cudaMemsetAsync(&dc->joint_maxd, 0, 8, s));
        CUDA_TRY(cudaMemsetAsync(W.queue.ptr, 0, 16, s));
        const int T = choose_T(W, nact, L.n_pad, o.tile_cols);
        CDParams P = cd_params(W, L, cb, nact, lambda0, tol, max_iter, o, nzcap, out, T);
        P.evict_after = 0;
        P.joint = 1;
        P.act = act;
        P.Ej = (double*)W.ej.ptr;
        P.joint_maxd = &dc->joint_maxd;
        const int ctas = (int)std::min<int64_t>(W.sms, (nact + T - 1) / T);
        if (!T0) { T0 = T; ctas0 = ctas; }
        CUDA_TRY(launch_cd(P, ctas, s));
        ++launches;
        if ((rc = read_counters(W, s))) return rc;
        if (W.host_counters->overflow) { overflow = true; break; }
        std::memcpy(&jm, &W.host_counters->joint_maxd, 8);
        ++inner;
      } while (!(jm < tol) && inner < o.max_inner);
      if (overflow) break;
      CUDA_TRY(launch_joint_sigma((const double*)W.xb.ptr, cb, act, nact, (const int*)W.nz_rows.ptr,
                                  (const double*)W.nz_vals.ptr, (const int*)W.nz_count.ptr,
                                  (const int*)W.nz_cur.ptr, nzcap, (int)n, L.n_pad, L.nchunk,
                                  std::sqrt((double)n), o.sigma_floor, tol, !(jm < tol),
                                  out.sigma_std, out.iters, (uint8_t*)W.jflags.ptr, out.conv,
                                  (double*)W.ej.ptr, (uint8_t*)W.keep.ptr, s));
      CUDA_TRY(launch_joint_compact(act, (const uint8_t*)W.keep.ptr, nact, act_next,
                                    &dc->joint_nact, s));
      launches += 2;
      if ((rc = read_counters(W, s))) return rc;
      nact = W.host_counters->joint_nact;
      std::swap(act, act_next);
    }
    if (!overflow) {
      CUDA_TRY(ev_record(W, W.ev[2], s));
      if (st) { st->solver = 1; st->tile_cols = T0; st->num_ctas = ctas0; st->kernel_launches += launches; }
      *nzcap_used = nzcap;
      return SPMESL_OK;
    }
    if (nzcap >= p) break;
    nzcap = (int)std::min<int64_t>(p, (int64_t)nzcap * 4);
  }
  return fail(SPMESL_ERR_OOM, "coefficient list overflow");
}

// Whether the Gram solver applies (see spmesl_options.solver).
bool gram_applicable(const Workspace& W, const spmesl_options& o, int64_t n, int64_t p, int64_t cb,
                     int64_t ce, std::string* why) {
  if (o.mode != 0) { if (why) *why = "the Gram solver implements mode 0"; return false; }
  if (cb != 0 || ce != p) { if (why) *why = "the Gram solver fits the whole column range"; return false; }
  const int n_pad = (int)(((n + KC - 1) / KC) * KC);
  if (tail_smem_bytes((int)p, n_pad, initial_nzcap(n, p)) > (size_t)W.smem_optin) {
    if (why) *why = "p too large for the on-chip gradient vector";
    return false;
  }
  const double need = (double)p * (double)p * 8.0;
  if ((double)W.ondemand.bytes >= need) return true;   // (no driver query on repeat calls)
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) { cudaGetLastError(); free_b = 0; }
  const double have = (double)free_b + (double)W.ondemand.bytes;
  if (need > 0.6 * have) { if (why) *why = "8 p^2 bytes do not fit in device memory"; return false; }
  return true;
}

// Gram solver for [0, p): standardize, S = X~^T X~ / n with fused
// screening, retire the columns whose first sweep changes nothing, covariance-update sweeps for
// the rest (tail.cu with z = S[:, c]).  Enqueue only (no host synchronisation): the caller reads
// the counters afterwards and checks err / overflow.
int fit_gram_enqueue(Workspace& W, const double* dX, int64_t n, int64_t p, double lambda0,
                     double tol, int32_t max_iter, const spmesl_options& o, const FitOut& out,
                     cudaStream_t s, Layout& L, int nzcap, const double* lams = nullptr,
                     int nlam = 1, bool screen16 = false, bool screen_only = false) {
  // nlam > 1: several penalty levels share X~, S and its screening pass (regularization path);
  // the outputs of level l, column c sit at l p + c
  const int64_t m = p;
  set_layout(L, n, p);
  int rc = alloc_core(W, L, m * nlam, nzcap);
  if (rc) return rc;
  if (tail_smem_bytes((int)p, L.n_pad, nzcap) > (size_t)W.smem_optin)
    return fail(SPMESL_ERR_UNSUPPORTED, "Gram solver: sweep state does not fit on chip");
  if ((rc = ensure(W.ondemand, (size_t)p * p * 8))) return rc;
  // screening flags [nlam][p], then (16-byte aligned) the hit count per column (both zeroed
  // by the reset kernel)
  const size_t hit_off = ((size_t)p * nlam + 15) & ~(size_t)15;
  const size_t hit_bytes = hit_off + (size_t)p * 4 + 1024 * 4;   // + the sweep order's buckets
  if ((rc = ensure(W.hit, hit_bytes))) return rc;
  int* hitcnt = (int*)((char*)W.hit.ptr + hit_off);
  int* bhist = hitcnt + p;
  if ((rc = ensure(W.lam_dev, (size_t)SPMESL_MAX_LAM * 8))) return rc;
  if ((rc = ensure(W.ssq, (size_t)p * 8))) return rc;
  if (screen16) {
    if ((rc = ensure(W.nrm, (size_t)p * 8))) return rc;
    // inv_sq, lam_n (f32, padded to the 128-column tiles; 16-byte aligned) + sq (f64, p)
    if ((rc = ensure(W.sq, (size_t)screen16_pad(p) * 8 + (size_t)p * 8))) return rc;
    if ((rc = ensure(W.y16, screen16_y_halves(p, L.n_pad) * 2))) return rc;
    if ((rc = ensure(W.cand, (size_t)p))) return rc;
    if ((rc = ensure(W.umap, (size_t)p * 4))) return rc;
    if ((rc = ensure(W.uvars, (size_t)p * 4))) return rc;
  }
  DevCounters* dc = (DevCounters*)W.counters.ptr;
  // the screening level: the smallest penalty (a superset of every level's hits)
  double lam_screen = lambda0;
  if (nlam > 1) { lam_screen = lams[0]; for (int l = 1; l < nlam; ++l) lam_screen = std::min(lam_screen, lams[l]); }
  const int64_t p_pad16 = screen16 ? screen16_pad(p) : 0;
  float* inv_sq = screen16 ? (float*)W.sq.ptr : nullptr;
  float* lam_n = screen16 ? inv_sq + p_pad16 : nullptr;
  double* sqv = screen16 ? (double*)(lam_n + p_pad16) : nullptr;
  S16Prep yprep{};
  if (screen16) {
    yprep.Y16 = (__half*)W.y16.ptr;
    yprep.nchunk64 = (L.n_pad + 63) / 64;
    yprep.p_pad = p_pad16;
    yprep.sq = sqv; yprep.inv_sq = inv_sq; yprep.lam_n = lam_n;
    yprep.lambda0 = lam_screen;
  }
  // (the reset kernel also clears the screening flags and the candidate flags)
  if ((rc = run_prep(W, dX, m * nlam, o, L, s, /*band=*/false, screen16 ? &yprep : nullptr,
                     W.hit.ptr, hit_bytes, screen16 ? W.cand.ptr : nullptr,
                     screen16 ? (size_t)p : 0)))
    return rc;
  {
    double lv[SPMESL_MAX_LAM];
    for (int l = 0; l < nlam; ++l) lv[l] = nlam > 1 ? lams[l] : lambda0;
    std::memcpy(W.lam_pinned, lv, (size_t)nlam * 8);
    CUDA_TRY(cudaMemcpyAsync(W.lam_dev.ptr, W.lam_pinned, (size_t)nlam * 8,
                             cudaMemcpyHostToDevice, s));
  }
  GramParams G{};
  G.Xb = (const double*)W.xb.ptr;
  G.n = (int)n; G.n_pad = L.n_pad; G.nchunk = L.nchunk; G.p = (int)p; G.nblk = (int)L.nblk;
  G.col_begin = 0;
  G.ncols = (int)m;
  G.lambda0 = lambda0; G.tol = tol; G.sigma_floor = o.sigma_floor; G.sqrt_n = std::sqrt((double)n);
  G.nlam = nlam;
  for (int l = 0; l < nlam; ++l) G.lams[l] = nlam > 1 ? lams[l] : lambda0;
  if (nlam > 1) {   // the Gram kernel screens at the smallest level (a superset of all hits)
    G.lambda0 = G.lams[0];
    for (int l = 1; l < nlam; ++l) G.lambda0 = std::min(G.lambda0, G.lams[l]);
  }
  G.max_outer = max_iter;
  G.G = (double*)W.ondemand.ptr;
  G.hit = (uint8_t*)W.hit.ptr;
  G.hitcnt = hitcnt;
  if ((rc = ensure(W.tail2, (size_t)m * nlam * 8))) return rc;   // tail keys, then the order
  G.bhist = bhist;
  G.tail_key = (int*)W.tail2.ptr;
  G.ssq = (const double*)W.ssq.ptr;
  G.tile_begin = 0;
  G.tile_end = gram_tile_count(p);
  if (W.pending_zero == nullptr && W.take_zero && (((uintptr_t)W.take_zero & 15) == 0)) {
    // the Gram kernel's producer zero-fills Theta with bulk stores while it computes (16-byte
    // pieces: an odd element count leaves the last double to one plain store)
    G.zero_ptr = W.take_zero;
    G.zero_count = W.take_count & ~(size_t)1;
    G.zero_last = (W.take_count & 1) ? W.take_zero + (W.take_count - 1) : nullptr;
  }
  G.tail = (TailState*)W.tail.ptr;
  G.tail_count = &dc->tail_count;
  G.sigma_std = out.sigma_std; G.iters = out.iters; G.sweeps = out.sweeps;
  G.converged = out.conv;
  G.nz_count = (int*)W.nz_count.ptr; G.nz_cur = (int*)W.nz_cur.ptr;
  const bool full_gram = !screen16;
  W.screen_fill = screen16 ? 0 : (int64_t)G.zero_count;
  int launches = 0;
  if (screen16) {
    // certified f16 screening (screen16.cu): candidate columns, then their exact FP64 Gram
    // columns and the exact decision; one host round trip for the candidate list
    // (y16 operands and threshold factors were written by the standardization)

    Screen16Params Q{};
    Q.Y16 = (const __half*)W.y16.ptr;
    Q.sq = sqv;
    Q.inv_sq = inv_sq;
    Q.lam_n = lam_n;
    Q.p = (int)p; Q.n = (int)n;
    Q.ntb = (int)((p + 127) / 128);
    Q.nchunk64 = (L.n_pad + 63) / 64;
    Q.tile_begin = 0;
    Q.tile_end = screen16_tile_count(p);
    Q.lambda0 = G.lambda0;
    Q.eps = screen16_eps(L.n_pad);
    Q.epsn = screen16_epsn(n, Q.eps);
    Q.cand = (uint8_t*)W.cand.ptr;
    // Theta's zero fill rides along the screening kernel's contraction (bulk stores from its
    // producer): it is the kernel's HBM floor at large p (a side-stream fill of part of it, run
    // under the exact Gram columns and the sweeps instead, measured the same: DESIGN.md §10)
    Q.zero_ptr = G.zero_ptr;
    Q.zero_count = G.zero_ptr ? G.zero_count : 0;
    Q.zero_last = G.zero_last;
    W.screen_fill = (int64_t)Q.zero_count;
    CUDA_TRY(ev_record(W, W.ev[8], s));
    CUDA_TRY(launch_screen16(Q, std::min(W.sms, Q.tile_end), s));
    CUDA_TRY(ev_record(W, W.ev[9], s));
    launches += 1;   // screen16
    // candidate list on the device; then, by its count (read on the device), either the exact
    // Gram columns of the candidates (2 n p nU flops) or — when most columns are candidates
    // (multi-sweep workloads) — the symmetric FP64 Gram kernel (n p (p+1) flops) decides
    // exactly; the kernel not needed exits at once.  No host round trip.
    int* nU_dev = &dc->s16_nU;
    CUDA_TRY(launch_cand_compact((const uint8_t*)W.cand.ptr, (int)p, (int*)W.uvars.ptr, nU_dev,
                                 (int*)W.umap.ptr, s));
    G.zero_ptr = nullptr;              // (Theta's zero fill is already under way)
    G.cond_nU = nU_dev;
    // (W.no_fallback: the exact Gram columns of every candidate, however many — correct for
    // any count, and what the screening history of these arguments expects)
    const bool fb = !W.no_fallback || nlam > 1;
    if (fb) {
      const int nT = (int)((L.nblk + 3) / 4);
      const int ntiles = nT * (nT + 1) / 2;
      CUDA_TRY(launch_syrk_screen(G, std::min(W.sms, ntiles), s));
      if (nlam > 1) CUDA_TRY(launch_level_flags(G, s));
    }
    CUDA_TRY(launch_gram_cols((const double*)W.xb.ptr, (int)L.nblk, L.nchunk, (int)n, (int)p,
                              (const int*)W.uvars.ptr, 0, nU_dev, W.sms, (double*)W.ondemand.ptr,
                              (uint8_t*)W.hit.ptr,
                              nlam > 1 ? (const double*)W.lam_dev.ptr : nullptr, nlam,
                              (int*)W.umap.ptr, s, /*fallback=*/fb, lambda0));
    launches += (fb ? 3 : 2) + (nlam > 1);
    CUDA_TRY(ev_record(W, W.ev[7], s));
  } else {
    const int nT = (int)((L.nblk + 3) / 4);
    const int ntiles = nT * (nT + 1) / 2;
    CUDA_TRY(ev_record(W, W.ev[8], s));
    CUDA_TRY(launch_syrk_screen(G, std::min(W.sms, ntiles), s));
    CUDA_TRY(ev_record(W, W.ev[9], s));
    CUDA_TRY(ev_record(W, W.ev[7], s));
    if (nlam > 1) CUDA_TRY(launch_level_flags(G, s));
    launches += 1 + (nlam > 1);
  }
  // (mode 1 on the Gram form continues from here with its own sweep loop: W.hit holds the
  // exact first-sweep decisions, W.ondemand the Gram columns of the hit columns)
  if (screen_only) { W.gram_launches = launches; return SPMESL_OK; }
  CUDA_TRY(launch_gram_init(G, s));
  CUDA_TRY(ev_record(W, W.ev[5], s));
  // the sweep kernel reads the number of columns with hits from the device counter (no host
  // round trip); one CTA per SM, each takes columns from the shared work counter
  TailParams T{};
  T.Xb = (const double*)W.xb.ptr;
  T.n = (int)n; T.n_pad = L.n_pad; T.nchunk = L.nchunk; T.p = (int)p; T.nblk = (int)L.nblk;
  T.col_begin = 0;
  T.lambda0 = lambda0; T.tol = tol; T.sigma_floor = o.sigma_floor; T.sqrt_n = std::sqrt((double)n);
  T.max_outer = max_iter; T.max_inner = o.max_inner;
  T.nzcap = nzcap;
  T.M = 0;
  T.M_dev = &dc->tail_count;
  T.tail = (const TailState*)W.tail.ptr;
  T.Zz = nullptr;
  T.Gtab = (double*)W.ondemand.ptr;
  T.gstate = full_gram ? nullptr : (int*)W.umap.ptr;
  T.z_from_gtab = 1;
  T.gtab_full = full_gram ? 1 : 0;
  T.next = &dc->tail_next;
  T.ondemand_count = &dc->gram_ondemand;
  T.sweeps_count = &dc->tail_sweeps;
  T.changes_count = &dc->tail_changes;
  T.flags = &dc->err;
  T.nz_rows = (int*)W.nz_rows.ptr; T.nz_vals = (double*)W.nz_vals.ptr;
  T.nz_count = (int*)W.nz_count.ptr; T.nz_cur = (int*)W.nz_cur.ptr;
  T.sigma_std = out.sigma_std; T.iters = out.iters; T.sweeps = out.sweeps; T.converged = out.conv;
  if (nlam > 1) { T.lambdas = (const double*)W.lam_dev.ptr; T.slot_stride = (int)p; }
  // the columns with the most hits first (the sweep kernel orders its list; results do not
  // depend on the order)
  T.bhist = bhist;
  T.tail_key = (const int*)W.tail2.ptr;
  T.order = (int*)W.tail2.ptr + m * nlam;
  T.order_bar = &dc->tail_ordered;
  set_tail_shape(W, T);
  const int tgrid = (int)std::min<int64_t>(W.sms, p * nlam);
  // Without skewed hit counts (band-like workloads) three 160-thread column CTAs per SM with the
  // multi-sweep mode's second z buffer in global memory beat two with it on chip (more chains
  // interleave); with them (hub) the on-chip buffer wins by far (its per-segment passes).  The
  // counts are on the device: both shapes are launched, gated, and one exits at once.
  const bool dual = bhist && nlam == 1 && T.occ == 2 && T.z2 &&
                    3 * (tail_smem_bytes((int)p, T.n_pad, T.nzcap) + 1024) <= (size_t)W.smem_sm;
  if (!T.z2 || dual) {   // (the multi-sweep mode's second z buffer in global memory, one slice per CTA)
    if ((rc = ensure(W.z2g, (size_t)tgrid * (dual ? 3 : std::max(T.occ, 1)) * p * 8))) return rc;
  }
  if (!T.z2) T.z2g = (double*)W.z2g.ptr;
  if (dual) {
    TailParams T3 = T;
    T3.occ = 3; T3.z2 = 0; T3.z2g = (double*)W.z2g.ptr; T3.gate = 2;
    T.gate = 1;
    CUDA_TRY(launch_tail_sweeps(T, tgrid, s));
    CUDA_TRY(launch_tail_sweeps(T3, tgrid, s));
    launches += 1;
  } else {
    CUDA_TRY(launch_tail_sweeps(T, tgrid, s));
  }
  CUDA_TRY(ev_record(W, W.ev[6], s));
  CUDA_TRY(ev_record(W, W.ev[2], s));
  W.gram_launches = launches + 2;   // + gram_init, tail
  return SPMESL_OK;
}

void gram_stats(Workspace& W, int64_t p, int nzcap, spmesl_stats* st, bool screen16 = false,
                bool replay = false) {
  (void)nzcap;
  if (!st) return;
  const int nT = (int)((((p + J - 1) / J) + 3) / 4);
  st->solver = screen16 ? 3 : 2;
  if (screen16) {
    st->screen_candidates = W.host_counters->s16_nU;
    st->gram_fallback = gram_fallback_taken(W.host_counters->s16_nU, p);
  }
  st->tile_cols = 0;
  st->num_ctas = std::min(W.sms, nT * (nT + 1) / 2);
  st->kernel_launches += W.gram_launches;
  // (a replay records only the events of ms_total and ms_screen: see ev_record)
  st->ms_gram = replay ? -1.0 : ev_ms(W.ev[1], W.ev[7]);
  st->ms_screen = ev_ms(W.ev[8], W.ev[9]);
  st->screen_fill_bytes = W.screen_fill * 8;
  st->ms_tail = replay ? -1.0 : ev_ms(W.ev[5], W.ev[6]);
  st->tail_columns = W.host_counters->tail_count;
  st->tail_sweeps = W.host_counters->tail_sweeps;
  st->tail_gram_ondemand = W.host_counters->gram_ondemand;
  st->tail_changes = (int64_t)W.host_counters->tail_changes;
  st->tail_passes = (int64_t)W.host_counters->tail_passes;
}

// The Gram solver with its own synchronisation and coefficient-list regrowth (for callers that
// continue on the host).
int fit_gram_core(Workspace& W, const double* dX, int64_t n, int64_t p, double lambda0, double tol,
                  int32_t max_iter, const spmesl_options& o, const FitOut& out, cudaStream_t s,
                  spmesl_stats* st, Layout& L, int* nzcap_used) {
  int nzcap = initial_nzcap(n, p);
  for (int attempt = 0; attempt < 4; ++attempt) {
    int rc = fit_gram_enqueue(W, dX, n, p, lambda0, tol, max_iter, o, out, s, L, nzcap, nullptr, 1,
                              o.solver != 2);
    if (rc) return rc;
    if ((rc = read_counters(W, s))) return rc;
    if (W.host_counters->err) return std_error(W, st);
    if (!W.host_counters->overflow) {
      gram_stats(W, p, nzcap, st, o.solver != 2);
      *nzcap_used = nzcap;
      return SPMESL_OK;
    }
    if (nzcap >= p) break;
    nzcap = (int)std::min<int64_t>(p, (int64_t)nzcap * 4);
  }
  return fail(SPMESL_ERR_OOM, "coefficient list overflow");
}

// Algorithm 3 (mode 1) on the Gram form: the first joint sweep of every
// column is the screening pass (solver 3's certified f16 screening or solver 2's FP64 Gram
// kernel, with the exact decisions); only the columns with a hit get a sweep slot, whose z is
// carried between the joint sweeps, each joint sweep being one launch of the sweep kernel over
// the active slots with max |db| reduced on the device.  The others are exact no-ops
// (b = 0 and every |z_j| <= lambda) until their sigma refit; an active column without a slot
// after a refit (sigma moved: lambda changed) gets one.  The outer boundary is the residual
// path's: fresh residual, sigma, F_c, in-order compaction (joint.cu).  One host synchronisation
// per joint sweep, as in the residual path.
int fit_joint_gram_core(Workspace& W, const double* dX, int64_t n, int64_t p, double lambda0,
                        double tol, int32_t max_iter, const spmesl_options& o, const FitOut& out,
                        cudaStream_t s, spmesl_stats* st, Layout& L, int* nzcap_used) {
  const int64_t m = p;
  const bool s16 = o.solver != 2;
  int nzcap = initial_nzcap(n, p);
  for (int attempt = 0; attempt < 4; ++attempt) {
    int rc = fit_gram_enqueue(W, dX, n, p, lambda0, tol, max_iter, o, out, s, L, nzcap, nullptr, 1,
                              s16, /*screen_only=*/true);
    if (rc) return rc;
    int launches = W.gram_launches + 1;
    const int full = W.screen_fill ? 0 : 0;
    (void)full;
    if ((rc = ensure(W.ej, (size_t)m * L.n_pad * 8))) return rc;
    if ((rc = ensure(W.act0, (size_t)m * 4))) return rc;
    if ((rc = ensure(W.act1, (size_t)m * 4))) return rc;
    if ((rc = ensure(W.keep, (size_t)m))) return rc;
    if ((rc = ensure(W.jflags, (size_t)m))) return rc;
    if ((rc = ensure(W.jtail, (size_t)m * sizeof(TailState)))) return rc;
    if ((rc = ensure(W.slotmap, (size_t)m * 4))) return rc;
    if ((rc = ensure(W.jwork, (size_t)m * 4))) return rc;
    DevCounters* dc = (DevCounters*)W.counters.ptr;
    CUDA_TRY(launch_joint_live_init((const uint8_t*)W.hit.ptr, (int)m, &dc->joint_nslots,
                                    (TailState*)W.jtail.ptr, (int*)W.slotmap.ptr, s));
    CUDA_TRY(cudaMemsetAsync(out.iters, 0, 4 * (size_t)m, s));
    CUDA_TRY(cudaMemsetAsync(out.sweeps, 0, 4 * (size_t)m, s));
    CUDA_TRY(cudaMemsetAsync(out.conv, 0, (size_t)m, s));
    CUDA_TRY(cudaMemsetAsync(W.jflags.ptr, 0, (size_t)m, s));
    CUDA_TRY(launch_joint_init((const double*)W.xb.ptr, 0, (int)m, L.n_pad, L.nchunk,
                               (int*)W.act0.ptr, out.sigma_std, (double*)W.ej.ptr, s));
    launches += 2;
    if ((rc = read_counters(W, s))) return rc;
    if (W.host_counters->err) return std_error(W, st);
    int nslots = W.host_counters->joint_nslots;
    if ((rc = ensure(W.zj, (size_t)std::max(nslots, 1) * (size_t)p * 8))) return rc;
    size_t zcap = W.zj.bytes / ((size_t)p * 8);
    int* act = (int*)W.act0.ptr;
    int* act_next = (int*)W.act1.ptr;
    int nact = (int)m;
    bool overflow = false;
    int64_t joint_sweeps = 0;
    for (int r = 0; r < max_iter && nact > 0 && !overflow; ++r) {
      if (r > 0) {
        // active columns without a slot (their sigma moved, so lambda did): give them one
        CUDA_TRY(cudaMemsetAsync(&dc->joint_nwork, 0, 4, s));
        CUDA_TRY(launch_joint_count_unslotted(act, nact, (const int*)W.slotmap.ptr,
                                              &dc->joint_nwork, s));
        if ((rc = read_counters(W, s))) return rc;
        const int need = W.host_counters->joint_nwork;
        ++launches;
      if (need > 0) {
        const int before = nslots;
        if ((size_t)(nslots + need) > zcap) {   // grow z storage, keeping the slots' contents
          Buffer nb;
          const size_t ncap = std::max((size_t)nslots + (size_t)need, 2 * zcap);
          if ((rc = ensure(nb, ncap * (size_t)p * 8))) return rc;
          if (nslots) CUDA_TRY(cudaMemcpyAsync(nb.ptr, W.zj.ptr, (size_t)nslots * p * 8,
                                               cudaMemcpyDeviceToDevice, s));
          CUDA_TRY(cudaStreamSynchronize(s));
          cudaFree(W.zj.ptr);
          W.zj = nb;
          zcap = ncap;
        }
        CUDA_TRY(launch_joint_live_add(act, nact, (int*)W.slotmap.ptr, (TailState*)W.jtail.ptr,
                                       &dc->joint_nslots, (const int*)W.nz_cur.ptr, s));
        if ((rc = read_counters(W, s))) return rc;
        nslots = W.host_counters->joint_nslots;
        (void)before;
        ++launches;
      }
      }
      int inner = 0;
      double jm = 0.0;
      // the slots of this outer iteration's active set (fixed during its sweeps)
      CUDA_TRY(cudaMemsetAsync(&dc->joint_nwork, 0, 4, s));
      CUDA_TRY(launch_joint_work(act, nact, (const int*)W.slotmap.ptr, (int*)W.jwork.ptr,
                                 &dc->joint_nwork, s));
      ++launches;
      do {
        CUDA_TRY(cudaMemsetAsync(&dc->joint_maxd, 0, 8, s));
        CUDA_TRY(cudaMemsetAsync(&dc->tail_next, 0, 4, s));
        TailParams T{};
        T.Xb = (const double*)W.xb.ptr;
        T.n = (int)n; T.n_pad = L.n_pad; T.nchunk = L.nchunk; T.p = (int)p; T.nblk = (int)L.nblk;
        T.col_begin = 0;
        T.lambda0 = lambda0; T.tol = tol; T.sigma_floor = o.sigma_floor;
        T.sqrt_n = std::sqrt((double)n);
        T.max_outer = max_iter; T.max_inner = o.max_inner;
        T.nzcap = nzcap;
        T.M = 0;
        T.M_dev = &dc->joint_nwork;
        T.Gtab = (double*)W.ondemand.ptr;
        T.gstate = s16 ? (int*)W.umap.ptr : nullptr;
        T.z_from_gtab = 1;
        T.gtab_full = s16 ? 0 : 1;
        T.next = &dc->tail_next;
        T.ondemand_count = &dc->gram_ondemand;
        T.sweeps_count = &dc->tail_sweeps;
  T.changes_count = &dc->tail_changes;
        T.flags = &dc->err;
        T.nz_rows = (int*)W.nz_rows.ptr; T.nz_vals = (double*)W.nz_vals.ptr;
        T.nz_count = (int*)W.nz_count.ptr; T.nz_cur = (int*)W.nz_cur.ptr;
        T.sigma_std = out.sigma_std; T.iters = out.iters; T.sweeps = out.sweeps;
        T.converged = out.conv;
        T.joint = 1;
        T.jtail = (TailState*)W.jtail.ptr;
        T.work = (const int*)W.jwork.ptr;
        T.Zj = (double*)W.zj.ptr;
        T.joint_maxd = &dc->joint_maxd;
        set_tail_shape(W, T);
        CUDA_TRY(launch_tail_sweeps(T, (int)std::max(1, std::min(W.sms, nslots)), s));
        ++launches;
        ++joint_sweeps;
        if ((rc = read_counters(W, s))) return rc;
        if (W.host_counters->err) return std_error(W, st);
        if (W.host_counters->overflow) { overflow = true; break; }
        std::memcpy(&jm, &W.host_counters->joint_maxd, 8);
        ++inner;
      } while (!(jm < tol) && inner < o.max_inner);
      if (overflow) break;
      CUDA_TRY(launch_joint_add_sweeps(act, nact, inner, out.sweeps, s));
      CUDA_TRY(launch_joint_sigma((const double*)W.xb.ptr, 0, act, nact, (const int*)W.nz_rows.ptr,
                                  (const double*)W.nz_vals.ptr, (const int*)W.nz_count.ptr,
                                  (const int*)W.nz_cur.ptr, nzcap, (int)n, L.n_pad, L.nchunk,
                                  std::sqrt((double)n), o.sigma_floor, tol, !(jm < tol),
                                  out.sigma_std, out.iters, (uint8_t*)W.jflags.ptr, out.conv,
                                  (double*)W.ej.ptr, (uint8_t*)W.keep.ptr, s));
      CUDA_TRY(launch_joint_compact(act, (const uint8_t*)W.keep.ptr, nact, act_next,
                                    &dc->joint_nact, s));
      launches += 3;
      if ((rc = read_counters(W, s))) return rc;
      nact = W.host_counters->joint_nact;
      std::swap(act, act_next);
    }
    if (!overflow) {
      CUDA_TRY(ev_record(W, W.ev[2], s));
      if (st) {
        st->solver = s16 ? 3 : 2;
        st->tile_cols = 0;
        st->num_ctas = W.sms;
        st->kernel_launches += launches;
        st->tail_columns = nslots;
        st->tail_sweeps = W.host_counters->tail_sweeps;
        st->tail_gram_ondemand = W.host_counters->gram_ondemand;
        st->screen_candidates = s16 ? W.host_counters->s16_nU : 0;
        st->ms_gram = ev_ms(W.ev[1], W.ev[7]);
        st->ms_screen = ev_ms(W.ev[8], W.ev[9]);
      }
      *nzcap_used = nzcap;
      return SPMESL_OK;
    }
    if (nzcap >= p) break;
    nzcap = (int)std::min<int64_t>(p, (int64_t)nzcap * 4);
  }
  return fail(SPMESL_ERR_OOM, "coefficient list overflow");
}

// Runs CD for [cb, ce) with automatic coefficient-list regrowth on overflow.
int fit_columns_core(Workspace& W, const double* dX, int64_t n, int64_t p, int64_t cb, int64_t ce,
                     double lambda0, double tol, int32_t max_iter, const spmesl_options& o,
                     const FitOut& out, cudaStream_t s, spmesl_stats* st, Layout& L,
                     int* nzcap_used) {
  const int64_t m = ce - cb;
  if (o.mode == 1) {
    // Algorithm 3 on the Gram form when the whole column range is fitted here and the Gram
    // solver's state fits (solver 0/2/3); else (or solver 1) on the residual CD kernel
    spmesl_options o0 = o;
    o0.mode = 0;
    std::string why;
    if (o.solver != 1 && gram_applicable(W, o0, n, p, cb, ce, &why))
      return fit_joint_gram_core(W, dX, n, p, lambda0, tol, max_iter, o, out, s, st, L,
                                 nzcap_used);
    if (o.solver == 2 || o.solver == 3)
      return fail(SPMESL_ERR_UNSUPPORTED, "Gram solver: " + why);
    return fit_joint_core(W, dX, n, p, cb, ce, lambda0, tol, max_iter, o, out, s, st, L,
                          nzcap_used);
  }
  {
    std::string why;
    const bool ok = gram_applicable(W, o, n, p, cb, ce, &why);
    if ((o.solver == 2 || o.solver == 3) && !ok) return fail(SPMESL_ERR_UNSUPPORTED, "Gram solver: " + why);
    if (ok && o.solver != 1)
      return fit_gram_core(W, dX, n, p, lambda0, tol, max_iter, o, out, s, st, L, nzcap_used);
  }
  if (st) st->solver = 1;
  set_layout(L, n, p);
  const int T = choose_T(W, m, L.n_pad, o.tile_cols);
  if (!T || cd_stages(T, L.n_pad, W.smem_optin) < 2)
    return fail(SPMESL_ERR_UNSUPPORTED, "n = " + std::to_string(n) +
                                            " does not fit the on-chip residual tile");
  int nzcap = initial_nzcap(n, p);
  for (int attempt = 0; attempt < 4; ++attempt) {
    int rc = alloc_core(W, L, m, nzcap);
    if (rc) return rc;
    int ctas = 0;
    if ((rc = run_cd(W, dX, n, p, cb, ce, lambda0, tol, max_iter, o, nzcap, out, s, T, L, &ctas)))
      return rc;
    if ((rc = read_counters(W, s))) return rc;
    if (W.host_counters->err) return std_error(W, st);
    if (st) { st->tile_cols = T; st->num_ctas = ctas; }
    if (!W.host_counters->overflow && W.host_counters->tail_count > 0) {
      if ((rc = run_tail(W, L, cb, lambda0, tol, max_iter, o, nzcap, out,
                         W.host_counters->tail_count, s, st)))
        return rc;
      if ((rc = read_counters(W, s))) return rc;
      if (st) {
        st->ms_tail = ev_ms(W.ev[5], W.ev[6]);
        st->tail_gram_ondemand = W.host_counters->gram_ondemand;
        st->tail_sweeps = W.host_counters->tail_sweeps;
      }
    }
    if (!W.host_counters->overflow) { *nzcap_used = nzcap; return SPMESL_OK; }
    if (nzcap >= p) break;
    nzcap = (int)std::min<int64_t>(p, (int64_t)nzcap * 4);
  }
  return fail(SPMESL_ERR_OOM, "coefficient list overflow");
}

// One attempt of the device-path Gram fit, enqueued on `cs` up to and including the read of
// the counter block into pinned host memory (no synchronisation): the eager path runs it on
// the caller's stream; the graph path captures it once and replays it.
int gram_fit_enqueue_all(Workspace& W, const double* dX, int64_t n, int64_t p, double lambda0,
                         double tol, int32_t max_iter, const spmesl_options& o, double* dTheta,
                         double* dSigma, int32_t* dIters, int32_t* dSweeps, uint8_t* dConv,
                         const FitOut& out, cudaStream_t cs, Layout& L, int nzcap,
                         bool screen16) {
  int rc;
  const size_t pp = (size_t)p * (size_t)p;
  // the screening kernel zero-fills Theta itself (bulk stores from its producer warp) when the
  // buffer allows 16-byte pieces; otherwise a side-stream kernel does, after standardization
  const bool sparse = W.sparse != nullptr;   // (CSC output: no dense Theta, no fill)
  const bool take = !sparse && (((uintptr_t)dTheta & 15) == 0);
  if (take) { W.take_zero = dTheta; W.take_count = pp; }
  else if (!sparse) { W.pending_zero = dTheta; W.pending_count = pp; }
  rc = fit_gram_enqueue(W, dX, n, p, lambda0, tol, max_iter, o, out, cs, L, nzcap, nullptr, 1,
                        screen16);
  W.take_zero = nullptr;
  if (W.pending_zero) {    // (the solver failed before standardization)
    W.pending_zero = nullptr;
    if (!rc) rc = fail(SPMESL_ERR_CUDA, "internal: Theta zero fill was not launched");
  }
  const bool join = (!take && !sparse) || W.zero_join;
  W.zero_join = false;
  if (rc) { if (join) cudaStreamWaitEvent(cs, W.ev_join, 0); return rc; }
  if (join) CUDA_TRY(cudaStreamWaitEvent(cs, W.ev_join, 0));
  DevCounters* dc = (DevCounters*)W.counters.ptr;
  CUDA_TRY(ev_record(W, W.ev[3], cs));
  if (sparse) {
    // Theta as CSC: entries per column, scan, then the entries (skipped on the device when
    // they would exceed the caller's capacity; the host reports the count)
    if ((rc = ensure(W.ccount, (size_t)p * 4))) return rc;
    CUDA_TRY(launch_sparse_count(p, (const int*)W.nz_count.ptr, (const int*)W.nz_cur.ptr,
                                 (const int*)W.nz_rows.ptr, (const double*)W.nz_vals.ptr, nzcap,
                                 o.symmetrize, (int*)W.ccount.ptr, cs));
    CUDA_TRY(launch_csc_scan((const int*)W.ccount.ptr, (int)p, W.sparse->col_ptr, &dc->csc_total,
                             cs));
    CUDA_TRY(launch_sparse_write(p, (const int*)W.nz_count.ptr, (const int*)W.nz_cur.ptr,
                                 (const int*)W.nz_rows.ptr, (const double*)W.nz_vals.ptr, nzcap,
                                 (const double*)W.sigma_std.ptr,
                                 o.standardize ? (const double*)W.scale.ptr : nullptr,
                                 o.symmetrize, W.sparse->col_ptr, W.sparse->rows,
                                 W.sparse->vals, dSigma, cs, W.sparse->cap));
  } else {
    // assembly + symmetrization straight from the coefficient lists (no CSC packing), with
    // the fit statistics (column_stats_kernel's work) fused in
    const ColStats cst{dIters, dSweeps, dConv, &dc->st_sweeps, &dc->st_max_sweeps,
                       &dc->st_max_outer, &dc->st_unconv, &dc->t_end};
    CUDA_TRY(launch_assemble_lists(p, (const int*)W.nz_count.ptr, (const int*)W.nz_cur.ptr,
                                   (const int*)W.nz_rows.ptr, (const double*)W.nz_vals.ptr, nzcap,
                                   (const double*)W.sigma_std.ptr,
                                   o.standardize ? (const double*)W.scale.ptr : nullptr,
                                   o.symmetrize, dTheta, dSigma, &dc->csc_total, cs, &cst));
  }
  CUDA_TRY(ev_record(W, W.ev[4], cs));
  if (sparse && (rc = device_stats(W, dIters, dSweeps, dConv, p, cs))) return rc;
  CUDA_TRY(cudaMemcpyAsync(W.host_counters, W.counters.ptr, sizeof(DevCounters),
                           cudaMemcpyDeviceToHost, cs));
  return SPMESL_OK;
}

void finish_stats(Workspace& W, int64_t p, spmesl_stats* st, int* any_unconv, int launches,
                  bool replay = false) {
  stats_from_counters(*W.host_counters, p, st, any_unconv);
  if (st) {
    st->nnz = W.host_counters->csc_total;
    st->ms_standardize = replay ? -1.0 : ev_ms(W.ev[0], W.ev[1]);
    st->ms_cd = replay ? -1.0 : ev_ms(W.ev[1], W.ev[2]);
    st->ms_assemble = replay ? -1.0 : ev_ms(W.ev[3], W.ev[4]);
    // (the device clock from the fit's first kernel to its statistics kernel: no timing-event
    // nodes needed in a captured fit)
    const DevCounters& hc = *W.host_counters;
    st->ms_total = hc.t_end > hc.t_start ? (double)(hc.t_end - hc.t_start) * 1e-6
                                         : ev_ms(W.ev[0], W.ev[4]);
    st->kernel_launches += launches;   // (+ the solver kernels, counted by the solver)
    st->bad_column = -1;
  }
}

// The arguments a captured fit depends on (pointers included: the graph bakes them in) plus the
// allocation generation (no workspace buffer may have moved since the capture).
std::vector<unsigned char> graph_key(const double* dX, int64_t n, int64_t p, double lambda0,
                                     double tol, int32_t max_iter, const spmesl_options& o,
                                     const void* dTheta, const void* dSigma, const void* dIters,
                                     const void* dSweeps, const void* dConv, int nzcap,
                                     cudaStream_t s, const Workspace::SparseOut* sp = nullptr) {
  struct K {
    const void* x; int64_t n, p; double lam, tol; int32_t mi, nzcap; spmesl_options o;
    const void *th, *sg, *it, *sw, *cv; uint64_t gen; int dev;
    const void *scp, *srows, *svals; int64_t scap;
  } k;
  std::memset(&k, 0, sizeof(k));
  k.x = dX; k.n = n; k.p = p; k.lam = lambda0; k.tol = tol; k.mi = max_iter; k.nzcap = nzcap;
  k.o = o; k.th = dTheta; k.sg = dSigma; k.it = dIters; k.sw = dSweeps; k.cv = dConv;
  k.gen = g_alloc_gen.load();
  if (sp) { k.scp = sp->col_ptr; k.srows = sp->rows; k.svals = sp->vals; k.scap = sp->cap; }
  cudaGetDevice(&k.dev);
  (void)s;
  const unsigned char* b = (const unsigned char*)&k;
  return std::vector<unsigned char>(b, b + sizeof(k));
}

void drop_graph(Workspace& W) {
  if (W.gexec) { cudaGraphExecDestroy(W.gexec); W.gexec = nullptr; }
  W.gkey.clear();
}

int fit_device_impl(const double* dX, int64_t n, int64_t p, double lambda0, double tol,
                    int32_t max_iter, const spmesl_options& o, double* dTheta, double* dSigma,
                    int32_t* dIters, int32_t* dSweeps, uint8_t* dConv, cudaStream_t s,
                    spmesl_stats* st, Workspace& W) {
  int rc;
  if ((rc = ensure(W.sigma_std, (size_t)p * 8))) return rc;
  if (!dSweeps) { if ((rc = ensure(W.sweeps, (size_t)p * 4))) return rc; dSweeps = (int32_t*)W.sweeps.ptr; }
  if (!dConv) { if ((rc = ensure(W.conv, (size_t)p))) return rc; dConv = (uint8_t*)W.conv.ptr; }
  FitOut out{0, p, (double*)W.sigma_std.ptr, dIters, dSweeps, dConv};
  Layout L;
  int nzcap = 0;
  std::string why;
  const bool gram_ok = gram_applicable(W, o, n, p, 0, p, &why);
  if ((o.solver == 2 || o.solver == 3) && !gram_ok)
    return fail(SPMESL_ERR_UNSUPPORTED, "Gram solver: " + why);
  const bool gram = gram_ok && o.solver != 1 && o.mode == 0;
  if (gram) {
    // (no side-stream work may be captured: the fill must be the screening kernel's own)
    const bool use_graph = !o.eager && o.solver != 2 && (((uintptr_t)dTheta & 15) == 0);
    // Auto solver: the certified screening pays off only when it leaves few candidates; when
    // the last fit on these very arguments fell back to the full FP64 Gram kernel (most columns
    // candidates: band, hub, lambda_univ), this one runs the full-Gram path (solver 2) directly
    // — no f16 screening pass, and Theta's zero fill rides inside the DMMA-bound Gram kernel.
    // Solvers 2 and 3 give the same iterates bit for bit, so the history only decides speed; a
    // full-Gram fit with few hit columns hands the choice back to the screening.
    spmesl_options ko = o;   // (the choice is part of the captured graph's key)
    std::vector<unsigned char> akey;
    bool full = o.solver == 2, few = false;
    if (o.solver == 0) {
      spmesl_options ao = o;
      ao.eager = 0;          // (eager and replayed fits share the history)
      akey = graph_key(dX, n, p, lambda0, tol, max_iter, ao, dTheta, dSigma, dIters, dSweeps, dConv,
                       0, s, W.sparse);
      full = !W.auto_full_key.empty() && W.auto_full_key == akey;
      few = !full && !W.auto_few_key.empty() && W.auto_few_key == akey;
      if (full) ko.solver = 2;
      else if (few) ko.solver = 5;   // (a key value of its own: no fallback launch)
    }
    // the captured fit's list capacity if these are its arguments, else the initial one
    nzcap = initial_nzcap(n, p);
    if (W.gexec && W.graph_nzcap > 0 &&
        graph_key(dX, n, p, lambda0, tol, max_iter, ko, dTheta, dSigma, dIters, dSweeps, dConv,
                  W.graph_nzcap, s, W.sparse) == W.gkey)
      nzcap = W.graph_nzcap;
    for (int attempt = 0; attempt < 4; ++attempt) {
      std::vector<unsigned char> key = graph_key(dX, n, p, lambda0, tol, max_iter, ko, dTheta,
                                                 dSigma, dIters, dSweeps, dConv, nzcap, s, W.sparse);
      bool launched = false;
      if (use_graph && W.gexec && key == W.gkey) {
        // replay: one launch for the whole fit (the penalty level is re-staged first)
        W.lam_pinned[0] = lambda0;
        W.screen_fill = W.graph_screen_fill;
        W.gram_launches = W.graph_launches;
        CUDA_TRY(cudaGraphLaunch(W.gexec, s));
        launched = true;
      } else if (use_graph && key == W.last_key) {
        // the same arguments twice in a row and nothing reallocated since: capture them
        drop_graph(W);
        const uint64_t gen0 = g_alloc_gen.load();
        W.capturing = true;
        cudaError_t e = cudaStreamBeginCapture(W.cap, cudaStreamCaptureModeRelaxed);
        if (e == cudaSuccess) {
          W.no_fallback = few;
          rc = gram_fit_enqueue_all(W, dX, n, p, lambda0, tol, max_iter, o, dTheta, dSigma,
                                    dIters, dSweeps, dConv, out, W.cap, L, nzcap, !full);
          W.no_fallback = false;
          cudaGraph_t g = nullptr;
          e = cudaStreamEndCapture(W.cap, &g);
          W.capturing = false;
          if (rc == SPMESL_OK && e == cudaSuccess && g &&
              g_alloc_gen.load() == gen0 &&
              cudaGraphInstantiate(&W.gexec, g, 0) == cudaSuccess) {
            W.gkey = key;
            W.graph_nzcap = nzcap;
            W.graph_screen_fill = W.screen_fill;
            W.graph_launches = W.gram_launches;
          } else {
            W.gexec = nullptr;
          }
          if (g) cudaGraphDestroy(g);
          cudaGetLastError();
          if (rc) return rc;
        }
        W.capturing = false;
        if (W.gexec) {
          W.lam_pinned[0] = lambda0;
          CUDA_TRY(cudaGraphLaunch(W.gexec, s));
          launched = true;
        }
      }
      if (!launched) {
        W.no_fallback = few;
        rc = gram_fit_enqueue_all(W, dX, n, p, lambda0, tol, max_iter, o, dTheta, dSigma,
                                  dIters, dSweeps, dConv, out, s, L, nzcap, !full);
        W.no_fallback = false;
        if (rc) return rc;
        W.last_key = key;
      }
      CUDA_TRY(cudaStreamSynchronize(s));
      if (W.host_counters->err) return std_error(W, st);
      if (!W.host_counters->overflow) {
        gram_stats(W, p, nzcap, st, !full, launched);
        if (st) st->graph_replay = launched ? 1 : 0;
        if (o.solver == 0) {   // (the screening history of these arguments)
          if (!full) {
            if (gram_fallback_taken(W.host_counters->s16_nU, p)) {
              W.auto_full_key = akey;
              W.auto_few_key.clear();
            } else {
              W.auto_few_key = akey;
            }
          } else if (!gram_fallback_taken(W.host_counters->tail_count, p)) {
            W.auto_full_key.clear();
          }
          if (st) st->gram_fallback = full ? 1 : few ? 0 : st->gram_fallback;
        }
        break;
      }
      if (nzcap >= p) return fail(SPMESL_ERR_OOM, "coefficient list overflow");
      nzcap = (int)std::min<int64_t>(p, (int64_t)nzcap * 4);
      drop_graph(W);
      // (Theta's zero fill is redone by the next attempt: the assembly above wrote into it)
    }
    int any_unconv = 0;
    // (standardize, assemble_lists, column_stats)
    // (reset + standardize + assemble_lists with the statistics fused; the sparse output: reset,
    // standardize, sparse_count, csc_scan, sparse_write, column_stats)
    finish_stats(W, p, st, &any_unconv, W.sparse ? 6 : 3, st && st->graph_replay);
    return any_unconv ? SPMESL_WARN_NOT_CONVERGED : SPMESL_OK;
  }
  // residual solver / joint mode: enqueue per call
  for (int attempt = 0; attempt < 4; ++attempt) {
    W.pending_zero = dTheta; W.pending_count = (size_t)p * (size_t)p;
    rc = fit_columns_core(W, dX, n, p, 0, p, lambda0, tol, max_iter, o, out, s, st, L, &nzcap);
    if (W.pending_zero) {    // (the solver failed before standardization)
      W.pending_zero = nullptr;
      if (!rc) rc = fail(SPMESL_ERR_CUDA, "internal: Theta zero fill was not launched");
    }
    if (rc) { cudaStreamWaitEvent(s, W.ev_join, 0); return rc; }
    CUDA_TRY(cudaStreamWaitEvent(s, W.ev_join, 0));
    const size_t cap = (size_t)p * (size_t)nzcap;
    if ((rc = ensure(W.csc_rows, cap * 4))) return rc;
    if ((rc = ensure(W.csc_vals, cap * 8))) return rc;
    DevCounters* dc = (DevCounters*)W.counters.ptr;
    CUDA_TRY(ev_record(W, W.ev[3], s));
    CUDA_TRY(launch_csc_build((const int*)W.nz_count.ptr, (const int*)W.nz_cur.ptr,
                              (const int*)W.nz_rows.ptr, (const double*)W.nz_vals.ptr, (int)p,
                              nzcap, (int64_t*)W.col_ptr.ptr, (int32_t*)W.csc_rows.ptr,
                              (double*)W.csc_vals.ptr, &dc->csc_total, s));
    CUDA_TRY(launch_assemble(p, 0, p, (const int64_t*)W.col_ptr.ptr,
                             (const int32_t*)W.csc_rows.ptr, (const double*)W.csc_vals.ptr,
                             (const double*)W.sigma_std.ptr,
                             o.standardize ? (const double*)W.scale.ptr : nullptr, o.symmetrize,
                             dTheta, dSigma, s, /*zero_fill=*/false));
    CUDA_TRY(ev_record(W, W.ev[4], s));
    if ((rc = device_stats(W, dIters, dSweeps, dConv, p, s))) return rc;
    if ((rc = read_counters(W, s))) return rc;
    break;
  }
  int any_unconv = 0;
  finish_stats(W, p, st, &any_unconv, 5);   // standardize, csc_scan, csc_copy, assemble x2
  return any_unconv ? SPMESL_WARN_NOT_CONVERGED : SPMESL_OK;
}

// CSC export of the fitted columns into the caller's device arrays (columns API).
int export_columns(Workspace& W, int64_t m, int64_t p, int nzcap, int32_t* dColCount,
                   int32_t* dRows, double* dVals, int64_t cap, int64_t* nnz_out, double* dScale,
                   const int32_t* dIters, const int32_t* dSweeps, const uint8_t* dConverged,
                   cudaStream_t s, spmesl_stats* st) {
  int rc;
  DevCounters* dc = (DevCounters*)W.counters.ptr;
  // scan only to learn the total, then copy straight into the caller's arrays
  const size_t need_cap = (size_t)m * (size_t)nzcap;
  if ((rc = ensure(W.csc_rows, need_cap * 4))) return rc;
  if ((rc = ensure(W.csc_vals, need_cap * 8))) return rc;
  dc = (DevCounters*)W.counters.ptr;
  CUDA_TRY(launch_csc_build((const int*)W.nz_count.ptr, (const int*)W.nz_cur.ptr,
                            (const int*)W.nz_rows.ptr, (const double*)W.nz_vals.ptr, (int)m, nzcap,
                            (int64_t*)W.col_ptr.ptr, (int32_t*)W.csc_rows.ptr,
                            (double*)W.csc_vals.ptr, &dc->csc_total, s));
  CUDA_TRY(launch_csc_counts((const int*)W.nz_count.ptr, (int)m, dColCount, s));
  CUDA_TRY(cudaMemcpyAsync(dScale, W.scale.ptr, (size_t)p * 8, cudaMemcpyDeviceToDevice, s));
  if ((rc = device_stats(W, dIters, dSweeps, dConverged, m, s))) return rc;
  if ((rc = read_counters(W, s))) return rc;
  const int64_t total = W.host_counters->csc_total;
  *nnz_out = total;
  if (total > cap) return fail(SPMESL_ERR_ARG, "CSC capacity too small: need " + std::to_string(total));
  if (total > 0) {
    CUDA_TRY(cudaMemcpyAsync(dRows, W.csc_rows.ptr, (size_t)total * 4, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(dVals, W.csc_vals.ptr, (size_t)total * 8, cudaMemcpyDeviceToDevice, s));
  }
  int any_unconv = 0;
  stats_from_counters(*W.host_counters, p, st, &any_unconv);
  if (st) {
    st->nnz = total;
    st->ms_standardize = ev_ms(W.ev[0], W.ev[1]);
    st->ms_cd = ev_ms(W.ev[1], W.ev[2]);
    st->kernel_launches += 6;
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  return any_unconv ? SPMESL_WARN_NOT_CONVERGED : SPMESL_OK;
}

// Multi-GPU Gram solver, part 2: columns [cb, ce) given the global screening flags.  Gram
// columns of the hit columns of the range come from one batched DMMA pass; any other column a
// sweep needs is computed on first use.
int fit_gram_columns_core(Workspace& W, const double* dX, int64_t n, int64_t p, int64_t cb,
                          int64_t ce, double lambda0, double tol, int32_t max_iter,
                          const spmesl_options& o, const uint8_t* dHit, const FitOut& out,
                          cudaStream_t s, spmesl_stats* st, Layout& L, int* nzcap_used) {
  const int64_t m = ce - cb;
  const bool cand = o.solver != 2;   // dHit: candidates of the certified screening (solver 0/3)
  set_layout(L, n, p);
  int nzcap = initial_nzcap(n, p);
  for (int attempt = 0; attempt < 4; ++attempt) {
    int rc = alloc_core(W, L, m, nzcap);
    if (rc) return rc;
    if (tail_smem_bytes((int)p, L.n_pad, nzcap) > (size_t)W.smem_optin)
      return fail(SPMESL_ERR_UNSUPPORTED, "Gram solver: sweep state does not fit on chip");
    if ((rc = ensure(W.ondemand, (size_t)p * p * 8))) return rc;
    if ((rc = ensure(W.umap, (size_t)p * 4))) return rc;             // gstate
    if ((rc = ensure(W.uvars, (size_t)std::max<int64_t>(m, 1) * 4))) return rc;
    if ((rc = ensure(W.ssq, (size_t)p * 8))) return rc;
    DevCounters* dc = (DevCounters*)W.counters.ptr;
    if ((rc = run_prep(W, dX, m, o, L, s, /*band=*/false))) return rc;
    // the flagged columns of this block: their Gram columns are computed up front (device-side
    // list, no host round trip); any other column a sweep needs is computed on first use
    DevCounters* dcs = (DevCounters*)W.counters.ptr;
    CUDA_TRY(launch_cand_compact(dHit, (int)p, (int*)W.uvars.ptr, &dcs->s16_nU, (int*)W.umap.ptr,
                                 s, (int)cb, (int)ce));
    const uint8_t* hit = dHit;
    if (cand) {
      // dHit holds candidates (certified screening): their exact Gram columns decide
      if ((rc = ensure(W.hit, (size_t)p))) return rc;
      if ((rc = ensure(W.lam_dev, (size_t)SPMESL_MAX_LAM * 8))) return rc;
      W.lam_pinned[0] = lambda0;
      CUDA_TRY(cudaMemcpyAsync(W.lam_dev.ptr, W.lam_pinned, 8, cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemsetAsync(W.hit.ptr, 0, (size_t)p, s));
      CUDA_TRY(launch_gram_cols((const double*)W.xb.ptr, (int)L.nblk, L.nchunk, (int)n, (int)p,
                                (const int*)W.uvars.ptr, 0, &dcs->s16_nU, W.sms,
                                (double*)W.ondemand.ptr, (uint8_t*)W.hit.ptr,
                                (const double*)W.lam_dev.ptr, 1, nullptr, s, /*fallback=*/false));
      hit = (const uint8_t*)W.hit.ptr;
    } else {
      CUDA_TRY(launch_gram_cols((const double*)W.xb.ptr, (int)L.nblk, L.nchunk, (int)n, (int)p,
                                (const int*)W.uvars.ptr, 0, &dcs->s16_nU, W.sms,
                                (double*)W.ondemand.ptr, nullptr, nullptr, 0, nullptr, s,
                                /*fallback=*/false));
    }
    CUDA_TRY(ev_record(W, W.ev[7], s));
    GramParams G{};
    G.Xb = (const double*)W.xb.ptr;
    G.n = (int)n; G.n_pad = L.n_pad; G.nchunk = L.nchunk; G.p = (int)p; G.nblk = (int)L.nblk;
    G.col_begin = cb;
    G.ncols = (int)m;
    G.lambda0 = lambda0; G.tol = tol; G.sigma_floor = o.sigma_floor; G.sqrt_n = std::sqrt((double)n);
    G.nlam = 1;
    G.lams[0] = lambda0;
    G.max_outer = max_iter;
    G.G = nullptr;
    G.hit = const_cast<uint8_t*>(hit);
    G.ssq = (const double*)W.ssq.ptr;
    G.tail = (TailState*)W.tail.ptr;
    G.tail_count = &dc->tail_count;
    G.sigma_std = out.sigma_std; G.iters = out.iters; G.sweeps = out.sweeps;
    G.converged = out.conv;
    G.nz_count = (int*)W.nz_count.ptr; G.nz_cur = (int*)W.nz_cur.ptr;
    CUDA_TRY(launch_gram_init(G, s));
    CUDA_TRY(ev_record(W, W.ev[5], s));
    TailParams T{};
    T.Xb = (const double*)W.xb.ptr;
    T.n = (int)n; T.n_pad = L.n_pad; T.nchunk = L.nchunk; T.p = (int)p; T.nblk = (int)L.nblk;
    T.col_begin = cb;
    T.lambda0 = lambda0; T.tol = tol; T.sigma_floor = o.sigma_floor; T.sqrt_n = std::sqrt((double)n);
    T.max_outer = max_iter; T.max_inner = o.max_inner;
    T.nzcap = nzcap;
    T.M = 0;
    T.M_dev = &dc->tail_count;
    T.tail = (const TailState*)W.tail.ptr;
    T.Zz = nullptr;
    T.Gtab = (double*)W.ondemand.ptr;
    T.gstate = (int*)W.umap.ptr;
    T.z_from_gtab = 1;
    T.gtab_full = 0;
    T.next = &dc->tail_next;
    T.ondemand_count = &dc->gram_ondemand;
    T.sweeps_count = &dc->tail_sweeps;
  T.changes_count = &dc->tail_changes;
    T.flags = &dc->err;
    T.nz_rows = (int*)W.nz_rows.ptr; T.nz_vals = (double*)W.nz_vals.ptr;
    T.nz_count = (int*)W.nz_count.ptr; T.nz_cur = (int*)W.nz_cur.ptr;
    T.sigma_std = out.sigma_std; T.iters = out.iters; T.sweeps = out.sweeps; T.converged = out.conv;
    set_tail_shape(W, T);
    CUDA_TRY(launch_tail_sweeps(T, (int)std::min<int64_t>(W.sms, m), s));
    CUDA_TRY(ev_record(W, W.ev[6], s));
    CUDA_TRY(ev_record(W, W.ev[2], s));
    if ((rc = read_counters(W, s))) return rc;
    if (W.host_counters->err) return std_error(W, st);
    if (!W.host_counters->overflow) {
      if (st) {
        st->solver = cand ? 3 : 2;
        st->kernel_launches += 4;
        if (cand) st->screen_candidates = W.host_counters->s16_nU;
        st->ms_gram = ev_ms(W.ev[1], W.ev[7]);
        st->ms_tail = ev_ms(W.ev[5], W.ev[6]);
        st->tail_columns = W.host_counters->tail_count;
        st->tail_sweeps = W.host_counters->tail_sweeps;
        st->tail_gram_ondemand = W.host_counters->gram_ondemand;
      }
      *nzcap_used = nzcap;
      return SPMESL_OK;
    }
    if (nzcap >= p) break;
    nzcap = (int)std::min<int64_t>(p, (int64_t)nzcap * 4);
  }
  return fail(SPMESL_ERR_OOM, "coefficient list overflow");
}

void init_stats(spmesl_stats* st) {
  if (st) { std::memset(st, 0, sizeof(*st)); st->bad_column = -1; }
}

}  // namespace

// staging buffers of the host sparse-output entry, per device
namespace {
struct SparseStage {
  std::mutex mu;
  Buffer x, colptr, rows, vals, sigma, iters, sweeps, conv;
};
std::mutex g_stage_mu;
std::vector<SparseStage*> g_stage;
SparseStage* stage_for(int dev) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  if ((int)g_stage.size() <= dev) g_stage.resize(dev + 1, nullptr);
  if (!g_stage[dev]) g_stage[dev] = new SparseStage();
  return g_stage[dev];
}
}  // namespace


namespace spmesl {
int multi_fail(int code, const std::string& msg) { return fail(code, msg); }
int fit_multi_device(const double* X, int64_t n, int64_t p, double lambda0, double tol,
                     int32_t max_iter, const spmesl_options& o, double* Theta, double* sigma,
                     int32_t* iters, int32_t* sweeps, uint8_t* converged, spmesl_stats* st);
}  // namespace spmesl

extern "C" {

void spmesl_default_options(spmesl_options* opt) {
  if (!opt) return;
  std::memset(opt, 0, sizeof(*opt));
  opt->struct_size = sizeof(spmesl_options);
  opt->max_inner = 10000;
  opt->standardize = 1;
  opt->symmetrize = 1;
  opt->sigma_floor = 1e-8;
  opt->mode = 0;
  opt->tile_cols = 0;
  opt->device = -1;
  opt->tail_after = 1;
}

const char* spmesl_last_error(void) { return g_last_error.c_str(); }

const char* spmesl_version(void) { return "spmesl-b200 0.1 (sm_100a)"; }

int spmesl_release_workspace(void) {
  {
    std::lock_guard<std::mutex> ls(g_stage_mu);
    int prev0 = -1;
    cudaGetDevice(&prev0);
    for (size_t d = 0; d < g_stage.size(); ++d) {
      SparseStage* S = g_stage[d];
      if (!S) continue;
      std::lock_guard<std::mutex> l2(S->mu);
      cudaSetDevice((int)d);
      for (Buffer* b : {&S->x, &S->colptr, &S->rows, &S->vals, &S->sigma, &S->iters, &S->sweeps,
                        &S->conv}) {
        if (b->ptr) cudaFree(b->ptr);
        b->ptr = nullptr;
        b->bytes = 0;
      }
    }
    if (prev0 >= 0) cudaSetDevice(prev0);
  }
  std::lock_guard<std::mutex> lk(g_ws_mu);
  int prev = -1;
  cudaGetDevice(&prev);
  for (auto*& w : g_ws) {
    if (!w) continue;
    std::lock_guard<std::mutex> lw(w->mu);
    if (w->init) cudaSetDevice(w->device);
    Buffer* bufs[] = {&w->tail, &w->tail2, &w->z2g, &w->umark, &w->umap, &w->uvars, &w->tailV, &w->zall, &w->ondemand,
                      &w->xb, &w->gband, &w->mean, &w->scale, &w->counters, &w->queue,
                      &w->sigma_std, &w->iters, &w->sweeps, &w->conv, &w->nz_count, &w->nz_cur,
                      &w->nz_rows, &w->nz_vals, &w->col_ptr, &w->csc_rows, &w->csc_vals,
                      &w->hx, &w->htheta, &w->hsigma, &w->hiters, &w->hsweeps, &w->hconv,
                      &w->coo_r, &w->coo_c, &w->coo_v, &w->hdiag, &w->zeros, &w->ej, &w->act0,
                      &w->act1, &w->keep, &w->jflags, &w->hit, &w->lam_dev, &w->nrm, &w->sq,
                      &w->y16, &w->cand, &w->ssq, &w->jtail, &w->slotmap, &w->jwork, &w->zj, &w->ccount};
    drop_graph(*w);
    w->last_key.clear();
    g_alloc_gen.fetch_add(1);
    for (Buffer* b : bufs) { if (b->ptr) cudaFree(b->ptr); b->ptr = nullptr; b->bytes = 0; }
    if (w->host_counters) cudaFreeHost(w->host_counters);
    if (w->lam_pinned) cudaFreeHost(w->lam_pinned);
    w->host_counters = nullptr;
    w->lam_pinned = nullptr;
    for (auto& e : w->ev) if (e) cudaEventDestroy(e);
    if (w->side) cudaStreamDestroy(w->side);
    if (w->cap) cudaStreamDestroy(w->cap);
    w->cap = nullptr;
    if (w->ev_fork) cudaEventDestroy(w->ev_fork);
    if (w->ev_join) cudaEventDestroy(w->ev_join);
    w->side = nullptr; w->ev_fork = w->ev_join = nullptr;
    w->init = false;
  }
  if (prev >= 0) cudaSetDevice(prev);
  return SPMESL_OK;
}

int spmesl_fit_device(const double* dX, int64_t n, int64_t p, double lambda0, double tol,
                      int32_t max_iter, const spmesl_options* opt, double* dTheta,
                      double* dSigma, int32_t* dIters, int32_t* dSweeps, uint8_t* dConverged,
                      void* cuda_stream, spmesl_stats* st) {
  init_stats(st);
  spmesl_options o = resolve(opt);
  int rc = validate(dX, n, p, lambda0, tol, max_iter, o);
  if (rc) return rc;
  if (!dTheta || !dSigma || !dIters) return fail(SPMESL_ERR_ARG, "output pointer is NULL");
  int dev;
  if ((rc = current_device(-1, &dev))) return rc;
  Workspace* W = workspace_for(dev);
  std::lock_guard<std::mutex> lk(W->mu);
  if ((rc = ws_init(*W, dev))) return rc;
  if (W->cc_major < 10) return fail(SPMESL_ERR_UNSUPPORTED, "needs an sm_100 device");
  return fit_device_impl(dX, n, p, lambda0, tol, max_iter, o, dTheta, dSigma, dIters, dSweeps,
                         dConverged, (cudaStream_t)cuda_stream, st, *W);
}

int spmesl_fit_sparse_device(const double* dX, int64_t n, int64_t p, double lambda0, double tol,
                             int32_t max_iter, const spmesl_options* opt, int64_t* dColPtr,
                             int32_t* dRows, double* dVals, int64_t cap, int64_t* nnz_out,
                             double* dSigma, int32_t* dIters, int32_t* dSweeps,
                             uint8_t* dConverged, void* cuda_stream, spmesl_stats* st) {
  init_stats(st);
  spmesl_options o = resolve(opt);
  int rc = validate(dX, n, p, lambda0, tol, max_iter, o);
  if (rc) return rc;
  if (!dColPtr || !dRows || !dVals || !nnz_out || !dSigma || !dIters)
    return fail(SPMESL_ERR_ARG, "output pointer is NULL");
  int dev;
  if ((rc = current_device(-1, &dev))) return rc;
  Workspace* W = workspace_for(dev);
  std::lock_guard<std::mutex> lk(W->mu);
  if ((rc = ws_init(*W, dev))) return rc;
  if (W->cc_major < 10) return fail(SPMESL_ERR_UNSUPPORTED, "needs an sm_100 device");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if ((rc = ensure(W->sigma_std, (size_t)p * 8))) return rc;
  if (!dSweeps) { if ((rc = ensure(W->sweeps, (size_t)p * 4))) return rc; dSweeps = (int32_t*)W->sweeps.ptr; }
  if (!dConverged) { if ((rc = ensure(W->conv, (size_t)p))) return rc; dConverged = (uint8_t*)W->conv.ptr; }
  {
    // mode 0 on a Gram solver: the device-path fit with the CSC written in place of the dense
    // assembly (one synchronisation; CUDA-graph replay of repeated calls)
    std::string why;
    if (o.mode == 0 && o.solver != 1 && gram_applicable(*W, o, n, p, 0, p, &why)) {
      const Workspace::SparseOut so{dColPtr, dRows, dVals, cap};
      W->sparse = &so;
      rc = fit_device_impl(dX, n, p, lambda0, tol, max_iter, o, nullptr, dSigma, dIters, dSweeps,
                           dConverged, s, st, *W);
      W->sparse = nullptr;
      if (rc < 0) return rc;
      const int64_t total = W->host_counters->csc_total;
      *nnz_out = total;
      if (st) st->nnz = total - p;   // off-diagonal entries of Theta
      if (total > cap)
        return fail(SPMESL_ERR_ARG, "sparse Theta capacity too small: need " + std::to_string(total));
      return rc;
    }
  }
  FitOut out{0, p, (double*)W->sigma_std.ptr, dIters, dSweeps, dConverged};
  Layout L;
  int nzcap = 0;
  // the fit itself (residual solver / mode 1; no dense Theta, so no fill)
  if ((rc = fit_columns_core(*W, dX, n, p, 0, p, lambda0, tol, max_iter, o, out, s, st, L, &nzcap)))
    return rc;
  if ((rc = ensure(W->ccount, (size_t)p * 4))) return rc;
  DevCounters* dc = (DevCounters*)W->counters.ptr;
  CUDA_TRY(ev_record(*W, W->ev[3], s));
  CUDA_TRY(launch_sparse_count(p, (const int*)W->nz_count.ptr, (const int*)W->nz_cur.ptr,
                               (const int*)W->nz_rows.ptr, (const double*)W->nz_vals.ptr, nzcap,
                               o.symmetrize, (int*)W->ccount.ptr, s));
  CUDA_TRY(launch_csc_scan((const int*)W->ccount.ptr, (int)p, dColPtr, &dc->csc_total, s));
  if ((rc = device_stats(*W, dIters, dSweeps, dConverged, p, s))) return rc;
  if ((rc = read_counters(*W, s))) return rc;
  const int64_t total = W->host_counters->csc_total;
  *nnz_out = total;
  if (total > cap)
    return fail(SPMESL_ERR_ARG, "sparse Theta capacity too small: need " + std::to_string(total));
  CUDA_TRY(launch_sparse_write(p, (const int*)W->nz_count.ptr, (const int*)W->nz_cur.ptr,
                               (const int*)W->nz_rows.ptr, (const double*)W->nz_vals.ptr, nzcap,
                               (const double*)W->sigma_std.ptr,
                               o.standardize ? (const double*)W->scale.ptr : nullptr, o.symmetrize,
                               dColPtr, dRows, dVals, dSigma, s));
  CUDA_TRY(ev_record(*W, W->ev[4], s));
  CUDA_TRY(cudaStreamSynchronize(s));
  int any_unconv = 0;
  stats_from_counters(*W->host_counters, p, st, &any_unconv);
  if (st) {
    st->nnz = total - p;   // off-diagonal entries of Theta
    st->ms_standardize = ev_ms(W->ev[0], W->ev[1]);
    st->ms_cd = ev_ms(W->ev[1], W->ev[2]);
    st->ms_assemble = ev_ms(W->ev[3], W->ev[4]);
    st->ms_total = ev_ms(W->ev[0], W->ev[4]);
    st->kernel_launches += 5;   // standardize, sparse count, scan, write, column stats
    st->bad_column = -1;
  }
  return any_unconv ? SPMESL_WARN_NOT_CONVERGED : SPMESL_OK;
}

int spmesl_fit_path_device(const double* dX, int64_t n, int64_t p, const double* lambdas,
                           int32_t nlam, double tol, int32_t max_iter, const spmesl_options* opt,
                           double* dTheta, double* dSigma, int32_t* dIters, int32_t* dSweeps,
                           uint8_t* dConverged, void* cuda_stream, spmesl_stats* st) {
  init_stats(st);
  spmesl_options o = resolve(opt);
  if (!lambdas || nlam < 1 || nlam > SPMESL_MAX_LAM)
    return fail(SPMESL_ERR_ARG, "nlam must be 1..8 and lambdas non-NULL");
  int rc;
  for (int l = 0; l < nlam; ++l)
    if ((rc = validate(dX, n, p, lambdas[l], tol, max_iter, o))) return rc;
  if (!dTheta || !dSigma || !dIters) return fail(SPMESL_ERR_ARG, "output pointer is NULL");
  int dev;
  if ((rc = current_device(-1, &dev))) return rc;
  Workspace* W = workspace_for(dev);
  std::lock_guard<std::mutex> lk(W->mu);
  if ((rc = ws_init(*W, dev))) return rc;
  if (W->cc_major < 10) return fail(SPMESL_ERR_UNSUPPORTED, "needs an sm_100 device");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const size_t pp = (size_t)p * (size_t)p;
  std::string why;
  const bool gram = o.mode == 0 && o.solver != 1 && gram_applicable(*W, o, n, p, 0, p, &why);
  if (!gram) {
    // (no shared pass to exploit: one fit per level)
    int worst = SPMESL_OK;
    for (int l = 0; l < nlam; ++l) {
      spmesl_stats sl;
      init_stats(&sl);
      rc = fit_device_impl(dX, n, p, lambdas[l], tol, max_iter, o, dTheta + l * pp, dSigma + l * p,
                           dIters + l * p, dSweeps ? dSweeps + l * p : nullptr,
                           dConverged ? dConverged + l * p : nullptr, s, &sl, *W);
      if (rc < 0) return rc;
      worst = std::max(worst, rc);
      if (st) { st->coord_updates += sl.coord_updates; st->total_sweeps += sl.total_sweeps;
                st->ms_total += sl.ms_total; st->solver = sl.solver; }
    }
    return worst;
  }
  const int64_t m = p * nlam;
  if ((rc = ensure(W->sigma_std, (size_t)m * 8))) return rc;
  if (!dSweeps) { if ((rc = ensure(W->sweeps, (size_t)m * 4))) return rc; dSweeps = (int32_t*)W->sweeps.ptr; }
  if (!dConverged) { if ((rc = ensure(W->conv, (size_t)m))) return rc; dConverged = (uint8_t*)W->conv.ptr; }
  FitOut out{0, p, (double*)W->sigma_std.ptr, dIters, dSweeps, dConverged};
  Layout L;
  int nzcap = initial_nzcap(n, p);
  DevCounters* dc = nullptr;
  for (int attempt = 0; attempt < 4; ++attempt) {
    const bool take = (((uintptr_t)dTheta & 15) == 0) && ((pp * nlam) & 1) == 0;
    if (take) { W->take_zero = dTheta; W->take_count = pp * nlam; }
    else { W->pending_zero = dTheta; W->pending_count = pp * nlam; }
    rc = fit_gram_enqueue(*W, dX, n, p, lambdas[0], tol, max_iter, o, out, s, L, nzcap, lambdas,
                          nlam, o.solver != 2);
    W->take_zero = nullptr;
    if (W->pending_zero) { W->pending_zero = nullptr; if (!rc) rc = fail(SPMESL_ERR_CUDA, "internal"); }
    const bool join = !take || W->zero_join;
    W->zero_join = false;
    if (rc) { if (join) cudaStreamWaitEvent(s, W->ev_join, 0); return rc; }
    if (join) CUDA_TRY(cudaStreamWaitEvent(s, W->ev_join, 0));
    const size_t cap = (size_t)p * (size_t)nzcap;
    if ((rc = ensure(W->csc_rows, cap * 4))) return rc;
    if ((rc = ensure(W->csc_vals, cap * 8))) return rc;
    dc = (DevCounters*)W->counters.ptr;
    CUDA_TRY(ev_record(*W, W->ev[3], s));
    for (int l = 0; l < nlam; ++l) {   // CSC + assembly of each level (stream-ordered reuse)
      const size_t lo = (size_t)l * p;
      CUDA_TRY(launch_csc_build((const int*)W->nz_count.ptr + lo, (const int*)W->nz_cur.ptr + lo,
                                (const int*)W->nz_rows.ptr + lo * 2 * nzcap,
                                (const double*)W->nz_vals.ptr + lo * 2 * nzcap, (int)p, nzcap,
                                (int64_t*)W->col_ptr.ptr, (int32_t*)W->csc_rows.ptr,
                                (double*)W->csc_vals.ptr, &dc->csc_total, s));
      CUDA_TRY(launch_assemble(p, 0, p, (const int64_t*)W->col_ptr.ptr,
                               (const int32_t*)W->csc_rows.ptr, (const double*)W->csc_vals.ptr,
                               (const double*)W->sigma_std.ptr + lo,
                               o.standardize ? (const double*)W->scale.ptr : nullptr, o.symmetrize,
                               dTheta + l * pp, dSigma + lo, s, /*zero_fill=*/false));
    }
    CUDA_TRY(ev_record(*W, W->ev[4], s));
    if ((rc = device_stats(*W, dIters, dSweeps, dConverged, m, s))) return rc;
    if ((rc = read_counters(*W, s))) return rc;
    if (W->host_counters->err) return std_error(*W, st);
    if (!W->host_counters->overflow) break;
    if (nzcap >= p) return fail(SPMESL_ERR_OOM, "coefficient list overflow");
    nzcap = (int)std::min<int64_t>(p, (int64_t)nzcap * 4);
  }
  int any_unconv = 0;
  stats_from_counters(*W->host_counters, p, st, &any_unconv);
  if (st) {
    gram_stats(*W, p, nzcap, st, o.solver != 2);
    st->ms_standardize = ev_ms(W->ev[0], W->ev[1]);
    st->ms_cd = ev_ms(W->ev[1], W->ev[2]);
    st->ms_assemble = ev_ms(W->ev[3], W->ev[4]);
    st->ms_total = ev_ms(W->ev[0], W->ev[4]);
    st->kernel_launches += 2 + 3 * nlam;
    st->bad_column = -1;
  }
  return any_unconv ? SPMESL_WARN_NOT_CONVERGED : SPMESL_OK;
}

int spmesl_fit_ex(const double* X, int64_t n, int64_t p, double lambda0, double tol,
                  int32_t max_iter, const spmesl_options* opt, double* Theta, double* sigma,
                  int32_t* iters, int32_t* sweeps, uint8_t* converged, spmesl_stats* st) {
  init_stats(st);
  spmesl_options o = resolve(opt);
  int rc = validate(X, n, p, lambda0, tol, max_iter, o);
  if (rc) return rc;
  if (!Theta || !sigma || !iters) return fail(SPMESL_ERR_ARG, "output pointer is NULL");
  if (o.num_devices > 0)   // several devices with NCCL (multi.cu)
    return fit_multi_device(X, n, p, lambda0, tol, max_iter, o, Theta, sigma, iters, sweeps,
                            converged, st);
  int dev;
  if ((rc = current_device(o.device, &dev))) return rc;
  Workspace* W = workspace_for(dev);
  std::lock_guard<std::mutex> lk(W->mu);
  if ((rc = ws_init(*W, dev))) return rc;
  if (W->cc_major < 10) return fail(SPMESL_ERR_UNSUPPORTED, "needs an sm_100 device");
  const size_t np = (size_t)n * p, pp = (size_t)p * p;
  // Theta is dense on the host but sparse in content: it is zero-filled while the device
  // computes — by the copy engine (D2H of a device zero buffer, when Theta is pinned) and by host
  // threads, in parallel; only the nonzero entries (COO) and the diagonal cross PCIe afterwards.
  size_t dma_elems = 0;
  // (share of Theta's zero fill given to the copy engine: the host threads do the rest)
  const double dma_frac = 0.3;
  {
    cudaPointerAttributes pa;
    const bool pinned = cudaPointerGetAttributes(&pa, Theta) == cudaSuccess &&
                        pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const size_t zbytes = (size_t)64 << 20;
    if (pinned && pp * 8 >= ((size_t)256 << 20) && ensure(W->zeros, zbytes) == SPMESL_OK) {
      if (cudaMemsetAsync(W->zeros.ptr, 0, zbytes, W->side) == cudaSuccess) {
        dma_elems = (size_t)(dma_frac * (double)pp);
        for (size_t off = 0; off < dma_elems; off += zbytes / 8) {
          const size_t cnt = std::min(zbytes / 8, dma_elems - off);
          if (cudaMemcpyAsync(Theta + off, W->zeros.ptr, cnt * 8, cudaMemcpyDeviceToHost, W->side) !=
              cudaSuccess) {
            dma_elems = off;
            break;
          }
        }
      }
      cudaGetLastError();
    }
  }
  std::vector<std::thread> zero;
  {
    const size_t rest = pp - dma_elems;
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    const unsigned cap_th = 16u;
    const size_t nth = std::min<size_t>(std::min(cap_th, hc), std::max<size_t>(1, rest >> 20));
    const size_t per = (rest + nth - 1) / nth;
    for (size_t t = 0; t < nth; ++t) {
      const size_t lo = dma_elems + t * per, hi = std::min(pp, lo + per);
      if (lo < hi) zero.emplace_back([=] { std::memset(Theta + lo, 0, (hi - lo) * sizeof(double)); });
    }
  }
  auto join = [&] {
    for (auto& th : zero) if (th.joinable()) th.join();
    if (dma_elems) cudaStreamSynchronize(W->side);
  };
  auto bail = [&](int code) { join(); return code; };
  if ((rc = ensure(W->hx, np * 8))) return bail(rc);
  if ((rc = ensure(W->sigma_std, (size_t)p * 8))) return bail(rc);
  if ((rc = ensure(W->hsigma, (size_t)p * 8))) return bail(rc);
  if ((rc = ensure(W->hiters, (size_t)p * 4))) return bail(rc);
  if ((rc = ensure(W->hsweeps, (size_t)p * 4))) return bail(rc);
  if ((rc = ensure(W->hconv, (size_t)p))) return bail(rc);
  if ((rc = ensure(W->hdiag, (size_t)p * 8))) return bail(rc);
  cudaStream_t s = 0;
  {
    cudaError_t e = cudaMemcpyAsync(W->hx.ptr, X, np * 8, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return bail(fail(SPMESL_ERR_CUDA, cudaGetErrorString(e)));
  }
  FitOut out{0, p, (double*)W->sigma_std.ptr, (int32_t*)W->hiters.ptr, (int32_t*)W->hsweeps.ptr,
             (uint8_t*)W->hconv.ptr};
  Layout L;
  int nzcap = 0;
  rc = fit_columns_core(*W, (const double*)W->hx.ptr, n, p, 0, p, lambda0, tol, max_iter, o, out, s,
                        st, L, &nzcap);
  if (rc) return bail(rc);
  const size_t cap = (size_t)p * (size_t)nzcap;
  if ((rc = ensure(W->csc_rows, cap * 4))) return bail(rc);
  if ((rc = ensure(W->csc_vals, cap * 8))) return bail(rc);
  DevCounters* dc = (DevCounters*)W->counters.ptr;
  std::vector<int32_t> cr, cc;
  std::vector<double> cv;
  int ncoo = 0;
  {
    auto step = [&]() -> int {
      CUDA_TRY(ev_record(*W, W->ev[3], s));
      CUDA_TRY(launch_csc_build((const int*)W->nz_count.ptr, (const int*)W->nz_cur.ptr,
                                (const int*)W->nz_rows.ptr, (const double*)W->nz_vals.ptr, (int)p,
                                nzcap, (int64_t*)W->col_ptr.ptr, (int32_t*)W->csc_rows.ptr,
                                (double*)W->csc_vals.ptr, &dc->csc_total, s));
      if ((rc = read_counters(*W, s))) return rc;
      const int64_t nnz = W->host_counters->csc_total;
      if ((rc = ensure(W->coo_r, (size_t)std::max<int64_t>(nnz, 1) * 4))) return rc;
      if ((rc = ensure(W->coo_c, (size_t)std::max<int64_t>(nnz, 1) * 4))) return rc;
      if ((rc = ensure(W->coo_v, (size_t)std::max<int64_t>(nnz, 1) * 8))) return rc;
      CUDA_TRY(launch_assemble_coo(p, (const int64_t*)W->col_ptr.ptr, (const int32_t*)W->csc_rows.ptr,
                                   (const double*)W->csc_vals.ptr, (const double*)W->sigma_std.ptr,
                                   o.standardize ? (const double*)W->scale.ptr : nullptr,
                                   o.symmetrize, (int32_t*)W->coo_r.ptr, (int32_t*)W->coo_c.ptr,
                                   (double*)W->coo_v.ptr, &dc->coo_count, (double*)W->hdiag.ptr,
                                   (double*)W->hsigma.ptr, s));
      CUDA_TRY(ev_record(*W, W->ev[4], s));
      if ((rc = read_counters(*W, s))) return rc;
      ncoo = W->host_counters->coo_count;
      cr.resize(ncoo); cc.resize(ncoo); cv.resize(ncoo);
      if (ncoo) {
        CUDA_TRY(cudaMemcpyAsync(cr.data(), W->coo_r.ptr, (size_t)ncoo * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(cc.data(), W->coo_c.ptr, (size_t)ncoo * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(cv.data(), W->coo_v.ptr, (size_t)ncoo * 8, cudaMemcpyDeviceToHost, s));
      }
      CUDA_TRY(cudaMemcpyAsync(sigma, W->hsigma.ptr, (size_t)p * 8, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaMemcpyAsync(iters, W->hiters.ptr, (size_t)p * 4, cudaMemcpyDeviceToHost, s));
      if (sweeps) CUDA_TRY(cudaMemcpyAsync(sweeps, W->hsweeps.ptr, (size_t)p * 4, cudaMemcpyDeviceToHost, s));
      if (converged) CUDA_TRY(cudaMemcpyAsync(converged, W->hconv.ptr, (size_t)p, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      return SPMESL_OK;
    };
    if ((rc = step())) return bail(rc);
  }
  std::vector<double> diag(p);
  {
    cudaError_t e = cudaMemcpy(diag.data(), W->hdiag.ptr, (size_t)p * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return bail(fail(SPMESL_ERR_CUDA, cudaGetErrorString(e)));
  }
  int any_unconv = 0;
  if ((rc = device_stats(*W, (const int32_t*)W->hiters.ptr, (const int32_t*)W->hsweeps.ptr,
                         (const uint8_t*)W->hconv.ptr, p, s)))
    return bail(rc);
  if ((rc = read_counters(*W, s))) return bail(rc);
  stats_from_counters(*W->host_counters, p, st, &any_unconv);
  join();
  for (int e = 0; e < ncoo; ++e) Theta[(size_t)cc[e] * p + cr[e]] = cv[e];
  for (int64_t k = 0; k < p; ++k) Theta[(size_t)k * p + k] = diag[k];
  if (st) {
    st->nnz = W->host_counters->csc_total;
    st->ms_standardize = ev_ms(W->ev[0], W->ev[1]);
    st->ms_cd = ev_ms(W->ev[1], W->ev[2]);
    st->ms_assemble = ev_ms(W->ev[3], W->ev[4]);
    st->ms_total = ev_ms(W->ev[0], W->ev[4]);
    st->kernel_launches += 7;
    st->bad_column = -1;
  }
  return any_unconv ? SPMESL_WARN_NOT_CONVERGED : SPMESL_OK;
}

// Host sparse-output entry (spmesl.h): the device sparse fit on this device's staging buffers
// (SparseStage, kept per device behind their own lock; the fit serialises on the workspace lock).
int spmesl_fit_sparse(const double* X, int64_t n, int64_t p, double lambda0, double tol,
                      int32_t max_iter, const spmesl_options* opt, int64_t* col_ptr,
                      int32_t* rows, double* vals, int64_t cap, int64_t* nnz_out, double* sigma,
                      int32_t* iters, int32_t* sweeps, uint8_t* converged, spmesl_stats* st) {
  init_stats(st);
  spmesl_options o = resolve(opt);
  int rc = validate(X, n, p, lambda0, tol, max_iter, o);
  if (rc) return rc;
  if (!col_ptr || !rows || !vals || !nnz_out || !sigma || !iters || cap < 0)
    return fail(SPMESL_ERR_ARG, "output pointer is NULL");
  int dev;
  if ((rc = current_device(o.device, &dev))) return rc;
  SparseStage* S = stage_for(dev);
  std::lock_guard<std::mutex> lk(S->mu);
  const size_t np = (size_t)n * (size_t)p;
  const int64_t dcap = std::max<int64_t>(cap, p + 16 * p);   // (device side: room to report)
  if ((rc = ensure(S->x, np * 8))) return rc;
  if ((rc = ensure(S->colptr, (size_t)(p + 1) * 8))) return rc;
  if ((rc = ensure(S->rows, (size_t)dcap * 4))) return rc;
  if ((rc = ensure(S->vals, (size_t)dcap * 8))) return rc;
  if ((rc = ensure(S->sigma, (size_t)p * 8))) return rc;
  if ((rc = ensure(S->iters, (size_t)p * 4))) return rc;
  if ((rc = ensure(S->sweeps, (size_t)p * 4))) return rc;
  if ((rc = ensure(S->conv, (size_t)p))) return rc;
  cudaStream_t s = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamDestroy(s); } } sg{s};
  CUDA_TRY(cudaMemcpyAsync(S->x.ptr, X, np * 8, cudaMemcpyHostToDevice, s));
  int64_t nnz = 0;
  rc = spmesl_fit_sparse_device((const double*)S->x.ptr, n, p, lambda0, tol, max_iter, &o,
                                (int64_t*)S->colptr.ptr, (int32_t*)S->rows.ptr,
                                (double*)S->vals.ptr, dcap, &nnz, (double*)S->sigma.ptr,
                                (int32_t*)S->iters.ptr, (int32_t*)S->sweeps.ptr,
                                (uint8_t*)S->conv.ptr, s, st);
  *nnz_out = nnz;
  if (rc < 0) return rc;
  if (nnz > cap) return fail(SPMESL_ERR_ARG, "sparse Theta capacity too small: need " + std::to_string(nnz));
  CUDA_TRY(cudaMemcpyAsync(col_ptr, S->colptr.ptr, (size_t)(p + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (nnz) {
    CUDA_TRY(cudaMemcpyAsync(rows, S->rows.ptr, (size_t)nnz * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(vals, S->vals.ptr, (size_t)nnz * 8, cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(cudaMemcpyAsync(sigma, S->sigma.ptr, (size_t)p * 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(iters, S->iters.ptr, (size_t)p * 4, cudaMemcpyDeviceToHost, s));
  if (sweeps) CUDA_TRY(cudaMemcpyAsync(sweeps, S->sweeps.ptr, (size_t)p * 4, cudaMemcpyDeviceToHost, s));
  if (converged) CUDA_TRY(cudaMemcpyAsync(converged, S->conv.ptr, (size_t)p, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return rc;
}

int spmesl_fit(const double* X, int64_t n, int64_t p, double lambda0, double tol,
               int32_t max_iter, double* Theta, double* sigma, int32_t* iters) {
  return spmesl_fit_ex(X, n, p, lambda0, tol, max_iter, nullptr, Theta, sigma, iters, nullptr,
                       nullptr, nullptr);
}

int spmesl_fit_columns_device(const double* dX, int64_t n, int64_t p, int64_t col_begin,
                              int64_t col_end, double lambda0, double tol, int32_t max_iter,
                              const spmesl_options* opt, int32_t* dColCount, int32_t* dRows,
                              double* dVals, int64_t cap, int64_t* nnz_out, double* dSigmaStd,
                              double* dScale, int32_t* dIters, int32_t* dSweeps,
                              uint8_t* dConverged, void* cuda_stream, spmesl_stats* st) {
  init_stats(st);
  spmesl_options o = resolve(opt);
  int rc = validate(dX, n, p, lambda0, tol, max_iter, o);
  if (rc) return rc;
  if (col_begin < 0 || col_end > p || col_begin >= col_end)
    return fail(SPMESL_ERR_ARG, "bad column range");
  if (o.mode == 1 && (col_begin != 0 || col_end != p))
    return fail(SPMESL_ERR_UNSUPPORTED, "mode 1 (joint stop over all columns) needs the whole "
                                        "column range on one device");
  if (!dColCount || !dRows || !dVals || !nnz_out || !dSigmaStd || !dScale || !dIters)
    return fail(SPMESL_ERR_ARG, "output pointer is NULL");
  int dev;
  if ((rc = current_device(-1, &dev))) return rc;
  Workspace* W = workspace_for(dev);
  std::lock_guard<std::mutex> lk(W->mu);
  if ((rc = ws_init(*W, dev))) return rc;
  if (W->cc_major < 10) return fail(SPMESL_ERR_UNSUPPORTED, "needs an sm_100 device");
  const int64_t m = col_end - col_begin;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (!dSweeps) { if ((rc = ensure(W->sweeps, (size_t)m * 4))) return rc; dSweeps = (int32_t*)W->sweeps.ptr; }
  if (!dConverged) { if ((rc = ensure(W->conv, (size_t)m))) return rc; dConverged = (uint8_t*)W->conv.ptr; }
  FitOut out{col_begin, col_end, dSigmaStd, dIters, dSweeps, dConverged};
  Layout L;
  int nzcap = 0;
  rc = fit_columns_core(*W, dX, n, p, col_begin, col_end, lambda0, tol, max_iter, o, out, s, st, L,
                        &nzcap);
  if (rc) return rc;
  return export_columns(*W, m, p, nzcap, dColCount, dRows, dVals, cap, nnz_out, dScale, dIters,
                        dSweeps, dConverged, s, st);
}

int spmesl_gram_supported(int64_t n, int64_t p) {
  if (n < 2 || p < 2 || p > (int64_t)0x7fffffff) return 0;
  int dev;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 0; }
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const int n_pad = (int)(((n + KC - 1) / KC) * KC);
  return tail_smem_bytes((int)p, n_pad, initial_nzcap(n, p)) <= (size_t)optin ? 1 : 0;
}

int64_t spmesl_gram_tile_count(int64_t p) {
  if (p < 1 || p > (int64_t)0x7fffffff) return -1;
  return gram_tile_count(p);
}

int64_t spmesl_screen_tile_count(int64_t p, const spmesl_options* opt) {
  if (p < 1 || p > (int64_t)0x7fffffff) return -1;
  const spmesl_options o = resolve(opt);
  return o.solver == 2 ? gram_tile_count(p) : screen16_tile_count(p);
}

}  // extern "C"

namespace {
// The screening pass over tiles [tile_begin, tile_end) (spmesl_gram_screen_device); acc (tests
// only, solver 3): the raw f32 accumulators n R_hat_jc of every tile into acc[c * acc_ld + j].
int gram_screen_impl(const double* dX, int64_t n, int64_t p, double lambda0, int64_t tile_begin,
                     int64_t tile_end, const spmesl_options* opt, uint8_t* dHit,
                     void* cuda_stream, spmesl_stats* st, float* acc, int64_t acc_ld) {
  init_stats(st);
  spmesl_options o = resolve(opt);
  int rc = validate(dX, n, p, lambda0, 1.0, 1, o);
  if (rc) return rc;
  if (!dHit) return fail(SPMESL_ERR_ARG, "dHit is NULL");
  const bool s16 = o.solver != 2;     // certified f16 screening (solvers 0 / 3)
  const int64_t nt = s16 ? screen16_tile_count(p) : gram_tile_count(p);
  if (tile_begin < 0 || tile_end > nt || tile_begin > tile_end)
    return fail(SPMESL_ERR_ARG, "bad tile range");
  int dev;
  if ((rc = current_device(-1, &dev))) return rc;
  Workspace* W = workspace_for(dev);
  std::lock_guard<std::mutex> lk(W->mu);
  if ((rc = ws_init(*W, dev))) return rc;
  if (W->cc_major < 10) return fail(SPMESL_ERR_UNSUPPORTED, "needs an sm_100 device");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  Layout L;
  set_layout(L, n, p);
  if ((rc = alloc_core(*W, L, 1, 8))) return rc;
  S16Prep yprep{};
  const int64_t p_pad = screen16_pad(p);
  float* inv_sq = nullptr;
  float* lam_n = nullptr;
  double* sqv = nullptr;
  if (s16) {
    if ((rc = ensure(W->nrm, (size_t)p * 8))) return rc;
    if ((rc = ensure(W->sq, (size_t)p_pad * 8 + (size_t)p * 8))) return rc;
    if ((rc = ensure(W->y16, screen16_y_halves(p, L.n_pad) * 2))) return rc;
    inv_sq = (float*)W->sq.ptr;
    lam_n = inv_sq + p_pad;
    sqv = (double*)(lam_n + p_pad);
    // the certified operands y = x~ / sqrt(N) and the threshold factors come from the
    // standardization's fused writer, exactly as in the single-device fit
    yprep.Y16 = (__half*)W->y16.ptr;
    yprep.nchunk64 = (L.n_pad + 63) / 64;
    yprep.p_pad = p_pad;
    yprep.sq = sqv; yprep.inv_sq = inv_sq; yprep.lam_n = lam_n;
    yprep.lambda0 = lambda0;
  }
  if ((rc = run_prep(*W, dX, 1, o, L, s, /*band=*/false, s16 ? &yprep : nullptr))) return rc;
  if (s16) {
    // dHit[c] = 1 for the columns the certified f16 screening of these tiles cannot clear
    // (candidates: a superset of the columns with a hit there)
    Screen16Params Q{};
    Q.Y16 = (const __half*)W->y16.ptr;
    Q.sq = sqv;
    Q.inv_sq = inv_sq;
    Q.lam_n = lam_n;
    Q.p = (int)p; Q.n = (int)n;
    Q.ntb = (int)((p + 127) / 128);
    Q.nchunk64 = (L.n_pad + 63) / 64;
    Q.tile_begin = (int)tile_begin;
    Q.tile_end = (int)tile_end;
    Q.lambda0 = lambda0;
    Q.eps = screen16_eps(L.n_pad);
    Q.epsn = screen16_epsn(n, Q.eps);
    Q.cand = dHit;
    Q.acc_out = acc;
    Q.acc_ld = acc_ld;
    CUDA_TRY(ev_record(*W, W->ev[8], s));
    CUDA_TRY(launch_screen16(Q, (int)std::min<int64_t>(W->sms, std::max<int64_t>(1, tile_end - tile_begin)), s));
    CUDA_TRY(ev_record(*W, W->ev[9], s));
    CUDA_TRY(ev_record(*W, W->ev[7], s));
    if ((rc = read_counters(*W, s))) return rc;
    if (W->host_counters->err) return std_error(*W, st);
    if (st) {
      st->solver = 3;
      st->ms_standardize = ev_ms(W->ev[0], W->ev[1]);
      st->ms_gram = ev_ms(W->ev[1], W->ev[7]);
      st->ms_screen = ev_ms(W->ev[8], W->ev[9]);
      st->kernel_launches = 3;   // reset, standardize (+ f16 operands), screening
      st->bad_column = -1;
    }
    return SPMESL_OK;
  }
  GramParams G{};
  G.Xb = (const double*)W->xb.ptr;
  G.n = (int)n; G.n_pad = L.n_pad; G.nchunk = L.nchunk; G.p = (int)p; G.nblk = (int)L.nblk;
  G.lambda0 = lambda0;
  G.nlam = 1;
  G.lams[0] = lambda0;
  G.G = nullptr;
  G.hit = dHit;
  G.tile_begin = (int)tile_begin;
  G.tile_end = (int)tile_end;
  CUDA_TRY(launch_syrk_screen(G, (int)std::min<int64_t>(W->sms, std::max<int64_t>(1, tile_end - tile_begin)), s));
  CUDA_TRY(ev_record(*W, W->ev[7], s));
  if ((rc = read_counters(*W, s))) return rc;
  if (W->host_counters->err) return std_error(*W, st);
  if (st) {
    st->solver = 2;
    st->ms_standardize = ev_ms(W->ev[0], W->ev[1]);
    st->ms_gram = ev_ms(W->ev[1], W->ev[7]);
    st->kernel_launches = 2;
    st->bad_column = -1;
  }
  return SPMESL_OK;
}

}  // namespace

extern "C" {

int spmesl_gram_screen_device(const double* dX, int64_t n, int64_t p, double lambda0,
                              int64_t tile_begin, int64_t tile_end, const spmesl_options* opt,
                              uint8_t* dHit, void* cuda_stream, spmesl_stats* st) {
  return gram_screen_impl(dX, n, p, lambda0, tile_begin, tile_end, opt, dHit, cuda_stream, st,
                          nullptr, 0);
}

int spmesl_screen_accumulators_device(const double* dX, int64_t n, int64_t p,
                                      const spmesl_options* opt, float* dAcc, int64_t acc_ld,
                                      uint8_t* dCand, void* dY16, void* cuda_stream) {
  spmesl_options o = resolve(opt);
  if (o.solver == 1 || o.solver == 2)
    return fail(SPMESL_ERR_ARG, "the accumulators exist for the certified screening (solver 0/3)");
  if (!dAcc || !dCand || acc_ld < screen16_pad(p)) return fail(SPMESL_ERR_ARG, "bad accumulator buffer");
  if (p < 1 || p > (int64_t)0x7fffffff) return fail(SPMESL_ERR_ARG, "bad p");
  int rc = gram_screen_impl(dX, n, p, 0.0, 0, screen16_tile_count(p), opt, dCand, cuda_stream,
                            nullptr, dAcc, acc_ld);
  if (rc || !dY16) return rc;
  int dev;
  if ((rc = current_device(-1, &dev))) return rc;
  Workspace* W = workspace_for(dev);
  std::lock_guard<std::mutex> lk(W->mu);
  const int n_pad = (int)(((n + KC - 1) / KC) * KC);
  CUDA_TRY(cudaMemcpyAsync(dY16, W->y16.ptr, screen16_y_halves(p, n_pad) * 2,
                           cudaMemcpyDeviceToDevice, (cudaStream_t)cuda_stream));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)cuda_stream));
  return SPMESL_OK;
}

int spmesl_fit_columns_gram_device(const double* dX, int64_t n, int64_t p, int64_t col_begin,
                                   int64_t col_end, double lambda0, double tol, int32_t max_iter,
                                   const spmesl_options* opt, const uint8_t* dHit,
                                   int32_t* dColCount, int32_t* dRows, double* dVals, int64_t cap,
                                   int64_t* nnz_out, double* dSigmaStd, double* dScale,
                                   int32_t* dIters, int32_t* dSweeps, uint8_t* dConverged,
                                   void* cuda_stream, spmesl_stats* st) {
  init_stats(st);
  spmesl_options o = resolve(opt);
  int rc = validate(dX, n, p, lambda0, tol, max_iter, o);
  if (rc) return rc;
  if (col_begin < 0 || col_end > p || col_begin >= col_end)
    return fail(SPMESL_ERR_ARG, "bad column range");
  if (o.mode != 0) return fail(SPMESL_ERR_UNSUPPORTED, "the Gram solver implements mode 0");
  if (!dHit || !dColCount || !dRows || !dVals || !nnz_out || !dSigmaStd || !dScale || !dIters)
    return fail(SPMESL_ERR_ARG, "pointer argument is NULL");
  int dev;
  if ((rc = current_device(-1, &dev))) return rc;
  Workspace* W = workspace_for(dev);
  std::lock_guard<std::mutex> lk(W->mu);
  if ((rc = ws_init(*W, dev))) return rc;
  if (W->cc_major < 10) return fail(SPMESL_ERR_UNSUPPORTED, "needs an sm_100 device");
  const int64_t m = col_end - col_begin;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (!dSweeps) { if ((rc = ensure(W->sweeps, (size_t)m * 4))) return rc; dSweeps = (int32_t*)W->sweeps.ptr; }
  if (!dConverged) { if ((rc = ensure(W->conv, (size_t)m))) return rc; dConverged = (uint8_t*)W->conv.ptr; }
  FitOut out{col_begin, col_end, dSigmaStd, dIters, dSweeps, dConverged};
  Layout L;
  int nzcap = 0;
  rc = fit_gram_columns_core(*W, dX, n, p, col_begin, col_end, lambda0, tol, max_iter, o, dHit, out,
                             s, st, L, &nzcap);
  if (rc) return rc;
  return export_columns(*W, m, p, nzcap, dColCount, dRows, dVals, cap, nnz_out, dScale, dIters,
                        dSweeps, dConverged, s, st);
}

int spmesl_assemble_device(int64_t p, int64_t col_begin, int64_t col_end, const int64_t* dColPtr,
                           const int32_t* dRows, const double* dVals, const double* dSigmaStd,
                           const double* dScale, const spmesl_options* opt, double* dTheta,
                           double* dSigmaOut, void* cuda_stream) {
  spmesl_options o = resolve(opt);
  if (p < 2 || col_begin < 0 || col_end > p || col_begin >= col_end)
    return fail(SPMESL_ERR_ARG, "bad column range");
  if (!dColPtr || !dSigmaStd || !dTheta || (o.standardize && !dScale))
    return fail(SPMESL_ERR_ARG, "NULL pointer");
  CUDA_TRY(launch_assemble(p, col_begin, col_end, dColPtr, dRows, dVals, dSigmaStd,
                           o.standardize ? dScale : nullptr, o.symmetrize, dTheta, dSigmaOut,
                           (cudaStream_t)cuda_stream));
  return SPMESL_OK;
}

}  // extern "C"
