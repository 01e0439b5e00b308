// Covariance-update tail solver (SURVEY.md §8(f) f2 applied to the columns that need more than
// one sweep).
//
// The CD kernel performs every column's first sweep — the dense screening pass, z = X~^T x~_c / n
// for all rows, on the tensor cores.  A column that does not retire after it is handed over
// here.  For such a column Algorithm 1 continues in the SAME cyclic row order, but
// instead of forming x_j^T e / n by a length-n dot product at every visit, it keeps
//     z_j = x~_j^T e / n   for all rows j  (shared memory)
// and, whenever b_j changes by -d (e += x~_j d, Prop. 2), updates z += d G[:, j] with the
// Gram column G[:, j] = X~^T x~_j / n.  A visit to a row with b_j = 0 and |z_j| <= lambda cannot
// change anything (Soft returns 0, d = 0), so a sweep only visits the rows with b_j != 0 or
// |z_j| > lambda, found in row order by a block-wide search: O(p (1 + changes)) work per sweep
// instead of O(p n).  The iterates are Algorithm 1's up to rounding; every operation is a fixed
// function of the column (the Gram columns come from one DMMA routine, whether precomputed in
// the batched pass or computed on demand), so results do not depend on scheduling.
//
// One sweep is processed as a speculative chain over the column's current nonzeros plus one
// block-wide pass over the rows per segment (see "per-column sweeps" below), so the dependent
// latency per sweep is a few passes, not one block-wide update and search per change.  When the
// whole support fits one chain, the multi-sweep mode (run_mpass) lets the chain run up to 32
// sweeps ahead — refitting sigma where inner loops end — and one pass applies them all; the
// columns are taken most-hits-first.  Every mode keeps the row-at-a-time loop's FMAs in its
// order: the iterates are bit-identical whatever mode, order or launch shape processed them.
//
// Development build only: -DSPMESL_TAIL_PROF adds per-phase cycle counters (scripts/
// tail_prof_build.sh); the shipped library has no run-time switches.
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include "spmesl_internal.cuh"

namespace spmesl {


__device__ __forceinline__ void dmma_t(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Block barrier after reconverging the warp: __syncthreads() is the aligned bar.sync, which
// needs all lanes of a warp to arrive together, and several call sites follow a block executed
// by thread 0 alone (lanes 1-31 could otherwise reach the barrier first and release it early).
__device__ __forceinline__ void bsync() {
  __syncwarp();
  __syncthreads();
}

__device__ __forceinline__ uint32_t smem_u32t(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init_t(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32t(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32t(bar)),
      "r"(parity)
      : "memory");
}
// (issued by one thread) Gram column j -> shared buffer, completion on bar
__device__ __forceinline__ void prefetch_col(double* dst, const double* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32t(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32t(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32t(bar))
      : "memory");
}

__device__ __forceinline__ double soft_t(double a, double lam) {
  double m = fabs(a) - lam;
  return m > 0.0 ? copysign(m, a) : 0.0;
}

// ------------------------------------------------------------------ fresh residuals
// V[k] = x~_c - sum_{b_j != 0, ascending} x~_j b_j for tail column k (one warp per column;
// the same per-element order as the CD kernel's refresh).
__global__ void tail_residuals_kernel(const double* __restrict__ Xb, const TailState* __restrict__ tail,
                                      int M, const int* __restrict__ nz_rows,
                                      const double* __restrict__ nz_vals, int nzcap,
                                      int64_t col_begin, int n_pad, int nchunk, double* __restrict__ V) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= M) return;
  const TailState ts = tail[k];
  const int64_t gc = col_begin + ts.col;
  const size_t lo = (size_t)ts.col * 2 * nzcap + (size_t)ts.cur * nzcap;
  double* r = V + (size_t)k * n_pad;
  for (int i = lane; i < n_pad; i += 32) r[i] = Xb[xb_index(i, gc, nchunk)];
  const int m_end = min(ts.cnt, nzcap);
  for (int m = 0; m < m_end; ++m) {
    const int j = nz_rows[lo + m];
    const double bj = nz_vals[lo + m];
    for (int i = lane; i < n_pad; i += 32) r[i] = fma(-Xb[xb_index(i, j, nchunk)], bj, r[i]);
  }
}

// ------------------------------------------------------------------ Gram / z columns (DMMA)
// Loads chunk q of vector `vid` (row `vr` of a 32 x 32 smem tile, stored swizzled like Xb).
// vid < M: residual V[vid]; vid - M < nU: variable U[vid - M] (a row of Xb); else zero.
__device__ __forceinline__ void load_vec_chunk(double* tile, int vr, int vid, int q, int lane,
                                               const double* Xb, int nchunk, const double* V,
                                               int M, const int* U, int nU, int n_pad) {
  double v = 0.0;
  if (vid < M) {
    v = V[(size_t)vid * n_pad + q * KC + lane];
  } else if (vid - M < nU) {
    v = Xb[xb_index((int64_t)q * KC + lane, U[vid - M], nchunk)];
  }
  tile[vr * XS + xswz(vr, lane)] = v;
}

// One 32-row block x one 32-vector tile of Z = X~_b^T W / n on 8 warps (warp w: m-tile w & 3,
// n-tiles 2 (w >> 2), +1).  Per output the chain is: chunks q ascending, k-pairs 0..3, even
// then odd sample — identical for every caller.
__device__ __forceinline__ void gram_tile(const double* Xb, int b, int nchunk, int n, int p,
                                          const double* V, int M, const int* U, int nU, int n_pad,
                                          int vt, int nvec_valid, double* tx, double* tv,
                                          double* Zz, double* Gtab, uint8_t* hit = nullptr,
                                          const double* lams = nullptr, int nlam = 0) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3, sw = g & 1;
  const int mt = warp & 3, nt0 = (warp >> 2) * 2;
  const bool mma_warp = warp < 8;   // (8 warps own the 32 x 32 output tile; more only load)
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int q = 0; q < nchunk; ++q) {
    const double2* src = (const double2*)(Xb + ((size_t)b * nchunk + q) * CHUNK_DOUBLES);
    for (int e = tid; e < CHUNK_DOUBLES / 2; e += blockDim.x) ((double2*)tx)[e] = src[e];
    for (int vr = warp; vr < 32; vr += blockDim.x >> 5)
      load_vec_chunk(tv, vr, vt * 32 + vr, q, lane, Xb, nchunk, V, M, U, nU, n_pad);
    bsync();
    const double* xa = tx + (mt * 8 + g) * XS + 2 * t4;
    if (mma_warp) {
#pragma unroll
      for (int kp = 0; kp < KC / 8; ++kp) {
        const double2 a = *(const double2*)(xa + (kp ^ sw) * 8);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const double2 bb = *(const double2*)(tv + ((nt0 + u) * 8 + g) * XS + 2 * t4 + (kp ^ sw) * 8);
          dmma_t(acc[u][0], acc[u][1], a.x, bb.x);
          dmma_t(acc[u][0], acc[u][1], a.y, bb.y);
        }
      }
    }
    bsync();
  }
  if (!mma_warp) return;
  const double inv_n = 1.0 / (double)n;
  const int row = b * J + mt * 8 + g;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int v = (nt0 + u) * 8 + 2 * t4 + e;
      if (row < p && v < nvec_valid) {
        const int vid = vt * 32 + v;
        double* col = vid < M ? Zz + (size_t)vid * p : Gtab + (size_t)U[vid - M] * p;
        const double g_rc = acc[u][e] * inv_n;
        col[row] = g_rc;
        if (hit && vid >= M) {   // exact screening decision: some |S_jc| > lambda, j != c
          const int c = U[vid - M];
          if (row != c)
            for (int l = 0; l < nlam; ++l)
              if (fabs(g_rc) > lams[l]) hit[(size_t)l * p + c] = 1;
        }
      }
    }
}

__global__ void __launch_bounds__(256) gram_pass_kernel(const double* __restrict__ Xb, int nchunk,
                                                        int n, int p, const double* __restrict__ V,
                                                        int M, const int* __restrict__ U, int nU,
                                                        int n_pad, double* __restrict__ Zz,
                                                        double* __restrict__ Gtab,
                                                        uint8_t* __restrict__ hit,
                                                        const double* __restrict__ lams, int nlam) {
  __shared__ __align__(128) double tx[J * XS];
  __shared__ __align__(128) double tv[J * XS];
  const int b = blockIdx.x, vt = blockIdx.y;
  const int total = M + nU;
  gram_tile(Xb, b, nchunk, n, p, V, M, U, nU, n_pad, vt, total - vt * 32, tx, tv, Zz, Gtab, hit,
            lams, nlam);
}

// Exact Gram columns G[:, U[v]] = X~^T x~_U[v] / n of a candidate list (no residual vectors):
// 8 rows per warp x up to 96 columns per vector group, a 3-stage cp.async ring of 32-sample chunks (the two
// 8 KB row blocks of Xb + the candidates' rows, re-swizzled by destination row parity), and
// per output the same DMMA chain as gram_tile (chunks ascending, k-pairs 0..3, even then odd
// sample), so every caller sees bit-identical columns.  Optional exact screening decision as
// in gram_tile.
// n-tiles of 8 vectors per vector group (96 columns; measured at config 5, 65 candidates:
// 16 -> 85 us, 12 -> 73 us, 9 -> 72 us — fewer accumulators and a smaller ring stage), and
// the ring's stages
constexpr int GC_NTMAX = 12;
constexpr int GC_STAGES = 3;
#ifndef SPMESL_GC_GROUP
#define SPMESL_GC_GROUP 3
#endif
constexpr int GC_GROUP = SPMESL_GC_GROUP;   // n-tiles per group of independent DMMAs

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}

// nU_dev (optional): the candidate count is read on the device; when gram_fallback_taken the full Gram
// kernel decides instead (solver 3 fallback): this kernel then only marks every column of its
// rows present (gstate = 2) and exits.
// Work split: one CTA per SM with T <= 17 warps, one 8-row m-tile per warp; CTA i owns a
// balanced contiguous range of m-tiles and walks it in rounds of T (one round when
// p <= 8 T #SMs: 17 warps x 148 SMs cover p = 20000 in one round, so no SM runs a second wave).
constexpr int GC_MAXW = 17;
__global__ void __launch_bounds__(GC_MAXW * 32, 1) gram_cols_kernel(const double* __restrict__ Xb,
                                                                 int nchunk, int n, int p,
                                                                 const int* __restrict__ U, int nU_host,
                                                                 const int* __restrict__ nU_dev,
                                                                 double* __restrict__ Gtab,
                                                                 uint8_t* __restrict__ hit,
                                                                 const double* __restrict__ lams,
                                                                 int nlam, int* __restrict__ gstate,
                                                                 int fallback, double lam1) {
  extern __shared__ __align__(128) double gsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nthr = blockDim.x;
  const int T = nthr >> 5;
  const int g = lane >> 2, t4 = lane & 3, sw = g & 1;
  const int nmt = (p + 7) / 8;
  const int m0 = (int)((int64_t)blockIdx.x * nmt / gridDim.x);
  const int m1 = (int)((int64_t)(blockIdx.x + 1) * nmt / gridDim.x);
  const int nU = nU_dev ? *(volatile const int*)nU_dev : nU_host;
  if (nU_dev && fallback && gram_fallback_taken(nU, p)) {
    if (gstate)
      for (int r = m0 * 8 + tid; r < min(p, m1 * 8); r += nthr) gstate[r] = 2;
    return;
  }
  const int xrows = T * 8;
  const int stage_d = xrows * XS + GC_NTMAX * 8 * XS;
  const double inv_n = 1.0 / (double)n;
  for (int v0 = 0; v0 < nU; v0 += GC_NTMAX * 8) {
    const int nvec = min(nU - v0, GC_NTMAX * 8);
    const int ntc = (nvec + 7) >> 3;
    for (int r0 = m0; r0 < m1; r0 += T) {
      const int mcnt = min(T, m1 - r0);
      const bool active = warp < mcnt;
      auto load = [&](int q, int st) {
        double* sx = gsm + (size_t)st * stage_d;
        double* sv = sx + xrows * XS;
        for (int e = tid; e < mcnt * 128; e += nthr) {     // m-tile rows: 2 KB contiguous each
          const int lm = e >> 7, r = e & 127;
          const int mt = r0 + lm;
          const double* src = Xb + (((size_t)(mt >> 2) * nchunk + q) * J + (mt & 3) * 8) * XS;
          cp_async16(sx + lm * 8 * XS + 2 * r, src + 2 * r);
        }
        for (int e = tid; e < nvec * 16; e += nthr) {      // candidate rows, 16 pieces each
          const int v = e >> 4, pos = 2 * (e & 15);
          const int u = U[v0 + v];
          const double* src = Xb + (((size_t)(u / J) * nchunk + q) * J + (u % J)) * XS;
          cp_async16(sv + v * XS + (pos ^ (((u ^ v) & 1) << 3)), src + pos);
        }
      };
      double acc[GC_NTMAX][2];
#pragma unroll
      for (int t = 0; t < GC_NTMAX; ++t) acc[t][0] = acc[t][1] = 0.0;
      __syncthreads();   // the previous round's stages have been read
#pragma unroll
      for (int q = 0; q < GC_STAGES - 1; ++q) {
        if (q < nchunk) load(q, q);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      }
      for (int q = 0; q < nchunk; ++q) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(GC_STAGES - 2) : "memory");
        __syncthreads();
        if (q + GC_STAGES - 1 < nchunk) load(q + GC_STAGES - 1, (q + GC_STAGES - 1) % GC_STAGES);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        if (active) {
          const double* sx = gsm + (size_t)(q % GC_STAGES) * stage_d;
          const double* sv = sx + xrows * XS;
          const double* xa = sx + (warp * 8 + g) * XS + 2 * t4;
#pragma unroll
          for (int kp = 0; kp < KC / 8; ++kp) {
            const double2 a = *(const double2*)(xa + (kp ^ sw) * 8);
            // groups of 4 n-tiles: the even samples of the group, then the odd ones — per
            // output the chain is unchanged (even then odd), consecutive DMMAs are independent
#pragma unroll
            for (int t0 = 0; t0 < GC_NTMAX; t0 += GC_GROUP) {
              if (t0 < ntc) {
                double2 b2[GC_GROUP];
#pragma unroll
                for (int u = 0; u < GC_GROUP; ++u)
                  if (t0 + u < ntc && t0 + u < GC_NTMAX)
                    b2[u] = *(const double2*)(sv + ((t0 + u) * 8 + g) * XS + 2 * t4 + (kp ^ sw) * 8);
#pragma unroll
                for (int u = 0; u < GC_GROUP; ++u)
                  if (t0 + u < ntc && t0 + u < GC_NTMAX) dmma_t(acc[t0 + u][0], acc[t0 + u][1], a.x, b2[u].x);
#pragma unroll
                for (int u = 0; u < GC_GROUP; ++u)
                  if (t0 + u < ntc && t0 + u < GC_NTMAX) dmma_t(acc[t0 + u][0], acc[t0 + u][1], a.y, b2[u].y);
              }
            }
          }
        }
      }
      const int row = (r0 + warp) * 8 + g;
      if (active && row < p) {
#pragma unroll
        for (int t = 0; t < GC_NTMAX; ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int v = t * 8 + 2 * t4 + e;
            if (t < ntc && v < nvec) {
              const int c = U[v0 + v];
              const double g_rc = acc[t][e] * inv_n;
              Gtab[(size_t)c * p + row] = g_rc;
              if (hit && row != c)   // exact screening decision: some |S_jc| > lambda, j != c
                for (int l = 0; l < nlam; ++l)
                  if (fabs(g_rc) > (lams ? lams[l] : lam1)) hit[(size_t)l * p + c] = 1;
            }
          }
      }
    }
  }
}

// mark the active variables of the handed-over columns (umark[j] = 1)
__global__ void tail_mark_kernel(const TailState* __restrict__ tail, int M, const int* __restrict__ nz_rows,
                                 int nzcap, int* __restrict__ umark) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= M) return;
  const TailState ts = tail[k];
  const size_t lo = (size_t)ts.col * 2 * nzcap + (size_t)ts.cur * nzcap;
  for (int m = lane; m < min(ts.cnt, nzcap); m += 32) umark[nz_rows[lo + m]] = 1;
}

// ------------------------------------------------------------------ per-column sweeps
// Chain + pass formulation of one sweep.  Algorithm 1 visits the rows in cyclic
// order; a visit can only change b_j if b_j != 0 (an "old" row: the column's current nonzeros,
// known at sweep start) or |z_j| > lambda (a "new" row).  The sweep is processed in segments:
//   chain  (warp 0): assume no new row appears before the next K <= KMAX old rows O_0 < O_1 <
//          ...; their visits form a dependent chain that needs only z at those rows and the
//          K x K Gram block G[O, O]:  a_k = z_{O_k} + sum_{l < k} d_l G[O_k, O_l] (+ pending
//          changes first), b' = Soft(a_k + b_k), d_k = b_k - b' — one lane per row, d_k
//          broadcast by shuffle, serial latency ~K shuffles instead of K block-wide passes;
//   pass   (all threads, one sweep over the rows): apply the pending changes to every z_i
//          (committed), form each row's value at its visit w_i = z_i + sum_{l: O_l < i} d_l
//          G[i, O_l] and find the first row in [pos, next unprocessed old row) with b_i = 0 and
//          |w_i| > lambda (a new row), by one block-wide min reduction;
//   commit: chain entries before that row are valid (their changes become pending; with a
//          second z buffer, when no new row appeared, z2 = z + all chain changes is swapped in
//          instead); the new row is visited with a = w_i, its change becomes pending too, and
//          the next segment starts right after it.
// Every z_i receives exactly the FMAs z_i <- fma(d, G[i, j], z_i) of the one-row-at-a-time
// covariance-update loop, in the same order (changes in row order), and every visit sees the
// same value — the iterates are bit-identical to it.  Per sweep the dependent chain is one
// pass (plus one per new row) instead of one block-wide update + search per change.
#ifdef SPMESL_TAIL_PROF   // (development build only: per-phase cycle counters of the sweep kernel)
__device__ unsigned long long g_tail_prof[32];
#define TPROF_T(v) const long long v = clock64()
#define TPROF_C(stmt) stmt
#define TPROF_ADD(i, val) do { if (threadIdx.x == 0) atomicAdd(&g_tail_prof[i], (unsigned long long)(val)); } while (0)
#else
#define TPROF_T(v)
#define TPROF_ADD(i, val)
#define TPROF_C(stmt)
#endif
constexpr int KMAX = 31;    // old rows per speculative chain (lanes of warp 0)
constexpr int PMAX = 32;    // pending changes (valid chain entries + one new row)
constexpr int PASS_U = 4;   // row pairs per thread per chunk of the pass (one LDG.128 each)
constexpr int PASS_PD = 2;  // columns whose loads are in flight (deeper spills: slower)
constexpr int KMS = 31;     // multi-sweep mode: at most KMS nonzeros (the whole support in one chain)
constexpr int MMAX = 32;    //   and at most MMAX sweeps speculated at once (16 when K > 16: the
constexpr int MDCAP = 512;  //   changes and new values are MDCAP doubles each, stride 16 or 32)

struct TailShared {
  uint64_t z_bar;        // z <- G[:, c] bulk copy
  double red[TAIL_MAXW];
  int wmin[TAIL_MAXW];   // per-warp first new row of a pass
  double wval[TAIL_MAXW];
  int oc_var[TAIL_ODC];
  int oc_next;
  int k;
  int k2;
  int ncol;

  int sg_n;              // the chain rows SG (in the tiles) was gathered for: sg_rows[0..sg_n)
  int sg_rows[KMAX];     //   (-1: invalid — the tiles were used for an on-demand Gram column)
  int so[KMAX];          // chain rows (old rows O_cursor ...)
  double sd[KMAX];       // chain changes d_l
  double sbn[KMAX];      // chain new values b'_l
  int prow[PMAX];        // pending changes (rows ascending, not yet applied to z)
  double pd[PMAX];
  union {   // (per-segment pass / multi-sweep: never live at the same time)
    struct {
      int crow[PMAX + KMAX]; // the pass's Gram columns: pending changes, then nonzero chain changes
      double cd[PMAX + KMAX];
      int cO[PMAX + KMAX];   // (chain columns: their row O_l; pending: -1)
    };
    struct {
      double mlam[MMAX];     // multi-sweep: lambda, sigma, outer / inner counts and flags in
      double msig[MMAX];     //   effect in sweep s (the chain refits sigma where an inner loop
      int mout[MMAX];        //   ends, and continues into the next outer iteration)
      int minr[MMAX];
      int mflg[MMAX];
    };
  };
  int sg_full;           // SG holds the whole K x K block (multi-sweep), not only k < m
  int mkey;              // multi-sweep pass: smallest (sweep, row) key of a new row found so far
  int mi[4];             // multi-sweep commit: old count, cursor, new count, changes
  double mmaxd;          //   and max |d| of the sweep in progress
  double mds[MMAX];      // multi-sweep: sum_l |d_sl| per sweep
  double msig_e;         //   the state after the last sweep of the chain
  int mout_e, minr_e, mflg_e, mret_e;
  int ordered;           // the work order by hit count is in use
};
constexpr size_t TS_BYTES = (sizeof(TailShared) + 127) & ~(size_t)127;

// Shared-memory layout (byte offsets; TailShared first so its address is a constant):
//   TailShared | tiles [2][J*XS] doubles (on-demand Gram columns; the chain's Gram blocks alias
//   them) | z [p] | r [n_pad] | old/new list values [2][nzcap] | old/new list rows [2][nzcap]
//   | old-row bitmap [ceil(p/32)] | (z2 [p], optional, after the base)
__host__ __device__ inline size_t tail_off_z() { return TS_BYTES + (size_t)2 * J * XS * 8; }
__host__ __device__ inline size_t tail_off_r(int pz) { return tail_off_z() + (((size_t)pz * 8 + 15) & ~(size_t)15); }
// (pz: rows of z this CTA holds — p, or its share of the rows in a cluster)
__host__ __device__ size_t tail_smem_bytes_rows(int pz, int p, int n_pad, int nzcap) {
  size_t b = tail_off_r(pz) + (size_t)n_pad * 8 + (size_t)2 * nzcap * 8 + (size_t)2 * nzcap * 4 +
             (size_t)((p + 31) / 32) * 4;
  return (b + 127) & ~(size_t)127;
}
__host__ __device__ size_t tail_smem_bytes(int p, int n_pad, int nzcap) {
  return tail_smem_bytes_rows(p, p, n_pad, nzcap);
}

// the optional second z buffer (z2, after the base layout)
__host__ __device__ size_t tail_z2_bytes(int p) { return (((size_t)p * 8) + 127) & ~(size_t)127; }

// Gram column G[:, j] of the fit-wide table: precomputed, or computed here once (claim 0 -> 1,
// write, publish 2) by the same DMMA routine as the batched pass; every CTA is resident, so
// waiting for another CTA's claim is safe.  Called by all threads of the block.
__device__ void ensure_gram_column(const TailParams& P, int j, TailShared& TS, double* tx,
                                   double* tvv) {
  if (P.gtab_full || *(volatile int*)&P.gstate[j] == 2) return;
  const int tid = threadIdx.x;
  bsync();
  if (tid == 0) { TS.oc_var[0] = j; TS.k2 = atomicCAS(&P.gstate[j], 0, 1); }
  bsync();
  if (TS.k2 == 0) {
    for (int b = 0; b < P.nblk; ++b)     // vector j alone in a tile: same DMMA chain
      gram_tile(P.Xb, b, P.nchunk, P.n, P.p, nullptr, 0, &TS.oc_var[0], 1, P.n_pad, 0, 1, tx,
                tvv, nullptr, P.Gtab);
    __threadfence();
    bsync();
    if (tid == 0) {
      atomicExch(&P.gstate[j], 2);
      atomicAdd(P.ondemand_count, 1);
      TS.sg_n = -1;   // (the tiles held the chain's cached Gram block)
    }
  } else if (tid == 0) {
    while (*(volatile int*)&P.gstate[j] != 2) __nanosleep(200);
  }
  __threadfence();
  bsync();
}

// rows of pair u of a thread in a pass chunk: base + 2 (u NT + tid) + {0, 1}
template <bool EVEN>
__device__ __forceinline__ double2 ld_pair_s(const double* z, int i, int p) {
  if (EVEN) return *(const double2*)(z + i);
  double2 v = make_double2(0.0, 0.0);
  v.x = z[i];
  if (i + 1 < p) v.y = z[i + 1];
  return v;
}
template <bool EVEN>
__device__ __forceinline__ void st_pair_s(double* z, int i, int p, double2 v) {
  if (EVEN) { *(double2*)(z + i) = v; return; }
  z[i] = v.x;
  if (i + 1 < p) z[i + 1] = v.y;
}

// One pass over the rows: chunks of RN = 2 U NT rows (each thread U pairs of
// adjacent rows, one LDG.128 per pair and column); per chunk the Gram columns it needs, in
// order, the next column's loads in flight while one is applied.  A chunk with no chain row
// inside it sees every row's visit value at one point — after the pending columns and the chain
// columns of rows before the chunk (split) — and tests it there; a chunk with a chain row inside
// tests each row just before the first chain column at or after it.
struct PassArgs {
  double* z;
  double* z2;
  const uint32_t* oldmask;
  const double* Gtab;
  int p, npend, C, pos, range_end, gc;
  bool spec_all;
  double lam;
  int r0, r1;            // the rows of this pass (z and z2 are indexed by the global row)
};

template <int NT, bool EVEN, int U, int PD>
__device__ __forceinline__ void run_pass(const PassArgs& A, const TailShared& TS, int& best,
                                         double& bestw) {
  constexpr int RN = 2 * U * NT;
  const int tid = threadIdx.x;
  const int p = A.p, npend = A.npend, C = A.C, pos = A.pos, range_end = A.range_end;
  const double lam = A.lam;
  const int r0 = A.r0, r1 = A.r1;
  const int nch = (r1 - r0 + RN - 1) / RN;
  // a new row: |w_i| > lambda (Soft != 0), i in [pos, range_end), b_i = 0 (not an old row),
  // i != c; the first one wins
  auto test = [&](int i, double w) {   // (callers have checked |w| > lambda)
    if (i >= pos && i < range_end && i < best && i != A.gc &&
        !((A.oldmask[i >> 5] >> (i & 31)) & 1u)) { best = i; bestw = w; }
  };
  for (int c = 0; c < nch; ++c) {
    const int base = r0 + c * RN;
    const bool det = base < range_end && base + RN > pos;
    if (npend == 0 && !A.spec_all && !det) continue;
    // chain columns of rows before the chunk (split), a chain row inside it (complex chunk)
    int split = npend;
    while (split < C && TS.cO[split] < base) ++split;
    const bool cx = det && split < C && TS.cO[split] < base + RN - 1;
    // columns this chunk needs: all for z2; else the pending ones and, when it holds detection
    // rows, the chain columns before its rows
    const int lend = A.spec_all ? C : (det ? (cx ? C : split) : npend);
    const int ptr0 = base + 2 * tid;
    double2 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = ptr0 + 2 * u * NT;
      acc[u] = i < r1 ? ld_pair_s<EVEN>(A.z, i, r1) : make_double2(0.0, 0.0);
    }
    // rows tested so far: for each parity v, the pairs u < done[v] (a thread's rows of the
    // chunk ascend with u, so the rows up to any chain row are a prefix)
    int done0 = det ? 0 : U, done1 = det ? 0 : U;
    auto test_upto = [&](int c0, int c1) {   // rows of pairs [done, c) of each parity
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = ptr0 + 2 * u * NT;
        if (u >= done0 && u < c0 && fabs(acc[u].x) > lam) test(i, acc[u].x);
        if (u >= done1 && u < c1 && fabs(acc[u].y) > lam) test(i + 1, acc[u].y);
      }
      done0 = max(done0, c0);
      done1 = max(done1, c1);
    };
    auto apply = [&](int l, const double2 (&g)[U]) {
      if (done0 + done1 < 2 * U && l >= split) {
        if (!cx) test_upto(U, U);
        else {
          // chain column l (row O_l): rows i <= O_l are visited before it
          const int O = TS.cO[l];
          const int n0 = O - ptr0, n1 = n0 - 1;   // row base + 2 (u NT + tid) + v <= O
          const int c0 = n0 < 0 ? 0 : min(U, n0 / (2 * NT) + 1);
          const int c1 = n1 < 0 ? 0 : min(U, n1 / (2 * NT) + 1);
          test_upto(c0, c1);
        }
      }
      const double d = TS.cd[l];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u].x = fma(d, g[u].x, acc[u].x);
        acc[u].y = fma(d, g[u].y, acc[u].y);
      }
      if (l == npend - 1) {         // committed: every pending change applied
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = ptr0 + 2 * u * NT;
          if (i < r1) st_pair_s<EVEN>(A.z, i, r1, acc[u]);
        }
      }
    };
    if (lend > 0) {
      auto load = [&](int l, double2 (&g)[U]) {
        const double* gcol = A.Gtab + (size_t)TS.crow[l] * p + ptr0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = ptr0 + 2 * u * NT;
          double2 v = make_double2(0.0, 0.0);
          if (i < r1) {
            if (EVEN) v = __ldcg((const double2*)(gcol + 2 * u * NT));
            else {
              v.x = __ldcg(gcol + 2 * u * NT);
              if (i + 1 < r1) v.y = __ldcg(gcol + 2 * u * NT + 1);
            }
          }
          g[u] = v;
        }
      };
      // a rolling window of PD columns in flight: column l + PD - 1 is requested into the
      // slot column l - 1 just freed, then column l is applied
      double2 g[PD][U];
#pragma unroll
      for (int q = 0; q < PD - 1; ++q)
        if (q < lend) load(q, g[q]);
      for (int l0 = 0; l0 < lend; l0 += PD) {
#pragma unroll
        for (int q = 0; q < PD; ++q) {
          const int l = l0 + q;
          if (l < lend) {
            if (l + PD - 1 < lend) load(l + PD - 1, g[(q + PD - 1) % PD]);
            apply(l, g[q]);
          }
        }
      }
    }
    if (done0 + done1 < 2 * U) test_upto(U, U);   // rows after every chain column
    if (A.spec_all) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = ptr0 + 2 * u * NT;
        if (i < r1) st_pair_s<EVEN>(A.z2, i, r1, acc[u]);
      }
    }
  }
}

// Multi-sweep pass.  When the column's whole support fits one chain (K <= KMS
// rows O_0 < ... < O_{K-1}) and no change is pending, warp 0 runs the chain for up to 32 whole
// sweeps ahead (16 when K > 16; assuming no other row enters; it stops at the sweep that ends
// the inner loop), recording every change d[s][l]; one pass then loads each row's K Gram
// entries G[i, O_l] once and applies all M K changes in their order (sweep s, then l), testing
// every row i outside the chain at its visit in each sweep (after the changes of sweep s at rows
// O_l < i).  SPEC: write the result to zd, record the first (sweep, row) with |w| > lambda as
// key s p + i.  !SPEC (after a new row at (sstar, istar)): apply only the changes before it —
// sweeps < sstar, and in sweep sstar the qstar chain rows before istar — to z in place.  The
// FMAs are the one-row-at-a-time loop's, in its order, plus FMAs with d = 0 (a zero change, the
// padding beyond K): those leave every z_i unchanged up to the sign of a zero, on which no
// decision or coefficient depends (|w| > lambda; Soft(+-0 + b) = Soft(b)).  So the iterates are
// bit-identical to the per-sweep chain + pass and to the one-row-at-a-time loop.
template <int NT, int KR, int R, bool SPEC>
__device__ __forceinline__ void run_mpass(const double* zs, double* zd, const uint32_t* oldmask,
                                          const double* Gtab, const TailShared& TS, const double* MD,
                                          int KS, const double* MDS, int p, int K, int Msw, int gc,
                                          const double* mlam, int sstar, int qstar, int* mkey,
                                          int& best, double& bestw) {
  // chunks of R NT rows: R rows per thread (rows base + r NT + tid), R K loads in flight per
  // thread.  Every thread walks every chunk (rows >= p masked), so warp votes see all lanes.
  constexpr int RN = R * NT;
  const int tid = threadIdx.x;
  // a row can only enter in sweep s if |w| > lambda_s at its visit; |w| <= |a| + max_l
  // |G[i, O_l]| sum_l |d_sl| (a: its value at the start of the sweep), so a sweep whose bound
  // stays below lambda_s (1 - 2^-40) for every row of a warp (the margin covers the rounding of
  // w and of the bound) needs no test site: its K changes are applied straight
  const int best_in = best;
  for (int base = 0; base < p; base += RN) {
    double g[R][KR];
#pragma unroll
    for (int l = 0; l < KR; ++l) {
      const double* gcol = Gtab + (size_t)(l < K ? TS.so[l] : 0) * p;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = base + r * NT + tid;
        g[r][l] = (l < K && i < p) ? __ldcg(gcol + i) : 0.0;
      }
    }
    double acc[R];
    float gm[R];              // max_l |G[i, O_l]| rounded up
    int q[R];
    bool t[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = base + r * NT + tid;
      acc[r] = i < p ? zs[i] : 0.0;
      q[r] = 0;
      gm[r] = 0.0f;
      t[r] = SPEC && i < p && i != gc && !((oldmask[i >> 5] >> (i & 31)) & 1u);
    }
    int smax = sstar + 1;
    if (SPEC) {
#pragma unroll
      for (int l = 0; l < KR; ++l)
#pragma unroll
        for (int r = 0; r < R; ++r) gm[r] = fmaxf(gm[r], __double2float_ru(fabs(g[r][l])));
      for (int l = 0; l < K; ++l) {
        const int o = TS.so[l];
#pragma unroll
        for (int r = 0; r < R; ++r) q[r] += o < base + r * NT + tid;
      }
      // a new row already found: later sweeps are moot (warp-uniform: the vote below)
      const int cut = __reduce_min_sync(0xffffffffu, min(*(volatile const int*)mkey, best));
      smax = cut == 0x7fffffff ? Msw : min(Msw, cut / p + 1);
    }
    auto rec = [&](bool f, int s, int i, double w) {   // (predicated, no branch per site)
      const int key = s * p + i;
      const bool take = f && key < best;
      best = take ? key : best;
      bestw = take ? w : bestw;
    };
    for (int s = 0; s < smax; ++s) {
      const double* md = MD + s * KS;
      bool exact = false;
      const double lam = SPEC ? mlam[s] : 0.0;
      if (SPEC) {
        const double Ds = MDS[s];
        const double lamm = lam - lam * 0x1p-40;
        bool f = false;
#pragma unroll
        for (int r = 0; r < R; ++r) f |= t[r] && fma((double)gm[r], Ds, fabs(acc[r])) >= lamm;
        exact = __any_sync(0xffffffffu, f);
      }
      if (!exact && (SPEC || s < sstar)) {
        // no row of the warp can enter in this sweep: the K changes (MD is zero-padded to KR)
#pragma unroll
        for (int l = 0; l < KR; ++l) {
          const double d = md[l];
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = fma(d, g[r][l], acc[r]);
        }
      } else if (!SPEC) {
        // (the rollback's last sweep: only the chain rows before the new row)
#pragma unroll
        for (int l = 0; l < KR; ++l) {
          const double d = l < qstar ? md[l] : 0.0;
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = fma(d, g[r][l], acc[r]);
        }
      } else {
        // test every row at its visit: after the changes of the chain rows before it
#pragma unroll
        for (int l = 0; l < KR; ++l) {
          const double d = md[l];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            rec(l == q[r] && t[r] && fabs(acc[r]) > lam, s, base + r * NT + tid, acc[r]);
            acc[r] = fma(d, g[r][l], acc[r]);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
          rec(q[r] >= K && t[r] && fabs(acc[r]) > lam, s, base + r * NT + tid, acc[r]);
      }
    }
#pragma unroll
    if (zd)   // (NULL: the chain ends the column; z after the pass is not needed)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = base + r * NT + tid;
        if (i < p) zd[i] = acc[r];
      }
    if (SPEC && best < best_in) atomicMin(mkey, best);
  }
}

template <int NT, bool SPEC>
__device__ __forceinline__ void mpass(const double* zs, double* zd, const uint32_t* oldmask,
                                      const double* Gtab, const TailShared& TS, const double* MD,
                                      int KS, const double* MDS, int p, int K, int Msw, int gc,
                                      const double* mlam, int sstar, int qstar, int* mkey,
                                      int& best, double& bestw) {
  if (K <= 4)
    run_mpass<NT, 4, 4, SPEC>(zs, zd, oldmask, Gtab, TS, MD, KS, MDS, p, K, Msw, gc, mlam, sstar,
                              qstar, mkey, best, bestw);
  else if (K <= 8)
    run_mpass<NT, 8, 4, SPEC>(zs, zd, oldmask, Gtab, TS, MD, KS, MDS, p, K, Msw, gc, mlam, sstar,
                              qstar, mkey, best, bestw);
  else if (K <= 16)
    run_mpass<NT, 16, 2, SPEC>(zs, zd, oldmask, Gtab, TS, MD, KS, MDS, p, K, Msw, gc, mlam, sstar,
                               qstar, mkey, best, bestw);
  else if (K <= 24)
    run_mpass<NT, 24, 1, SPEC>(zs, zd, oldmask, Gtab, TS, MD, KS, MDS, p, K, Msw, gc, mlam, sstar,
                               qstar, mkey, best, bestw);
  else
    run_mpass<NT, 32, 1, SPEC>(zs, zd, oldmask, Gtab, TS, MD, KS, MDS, p, K, Msw, gc, mlam, sstar,
                               qstar, mkey, best, bestw);
}

// Work order by hit count, most first: those columns tend to need the most sweeps, and at
// config 4 hub the slowest ones would otherwise start late and set the kernel's end.  The
// exact-decision kernel gave every tail entry its hit-count bucket and a rank in it; here each
// CTA scans the 1024 bucket sizes, writes the positions of its share of the entries, and all
// CTAs meet at a grid barrier (all are resident).  The order inside a bucket is arbitrary: it
// only decides which CTA takes a column when; results do not depend on it.  Returns whether
// the order is used (not when the counts are too even to matter: the most hits below twice
// the median + 4, e.g. band(3): 6 vs 3; hub: 70 vs 12).
// Are the per-column hit counts skewed (the most hits >= 2 x the median + 4)?  Every CTA reads
// the same histogram, so every CTA reaches the same answer.  Leaves in off[0..1023] the
// exclusive scan of the bucket sizes (bucket 0: the most hits), which order_tail places by.
template <int NT>
__device__ bool tail_skewed(const TailParams& P, int M, int* off) {
  const int tid = threadIdx.x;
  for (int b = tid; b < 1024; b += NT) off[b] = P.bhist[b];   // (one round of loads)
  __syncthreads();
  if (tid < 32) {   // exclusive scan of the bucket sizes (bucket 0: the most hits), one warp
    int carry = 0, top = -1, med = -1;
    for (int b0 = 0; b0 < 1024; b0 += 32) {
      const int v = off[b0 + tid];
      int incl = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, d);
        if (tid >= d) incl += t;
      }
      off[b0 + tid] = carry + incl - v;
      const unsigned nz = __ballot_sync(0xffffffffu, v > 0);
      if (top < 0 && nz) top = b0 + __ffs(nz) - 1;
      const unsigned hm = __ballot_sync(0xffffffffu, carry + incl >= (M + 1) / 2);
      if (med < 0 && hm) med = b0 + __ffs(hm) - 1;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 0) off[1024] = (1023 - top) >= 2 * (1023 - med) + 4;   // hits: top vs median
  }
  __syncthreads();
  return off[1024] != 0;
}

template <int NT>
__device__ bool order_tail(const TailParams& P, int M, int* off) {
  const int tid = threadIdx.x;
  if (!tail_skewed<NT>(P, M, off)) return false;   // (the same decision in every CTA)
  const int per = (M + gridDim.x - 1) / gridDim.x;
  for (int k = blockIdx.x * per + tid; k < min(M, (int)(blockIdx.x + 1) * per); k += NT) {
    const int key = P.tail_key[k];
    P.order[off[key >> 20] + (key & 0xFFFFF)] = k;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    atomicAdd(P.order_bar, 1);
    while (*(volatile const int*)P.order_bar < (int)gridDim.x) __nanosleep(64);
  }
  __syncthreads();
  __threadfence();
  return true;
}

template <int NT, bool EVEN, int MINB, bool MULTI>
__global__ void __launch_bounds__(NT, MINB) tail_sweep_kernel(const TailParams P) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int p = P.p, n = P.n, n_pad = P.n_pad, nchunk = P.nchunk, nzcap = P.nzcap;
  const int r0 = 0, r1 = p;
  TailShared& TS = *(TailShared*)sm;
  double* tx = (double*)(sm + TS_BYTES);                     // [J*XS]
  double* tvv = tx + J * XS;                                 // [J*XS]
  double* zA = (double*)(sm + tail_off_z());                 // [p]
  double* r = (double*)(sm + tail_off_r(p));                 // [n_pad]
  double* ov = r + n_pad;                                    // [nzcap] old list values
  double* nv = ov + nzcap;                                   // [nzcap] new list values
  int* orow = (int*)(nv + nzcap);                            // [nzcap]
  int* nrow = orow + nzcap;                                  // [nzcap]
  uint32_t* oldmask = (uint32_t*)(nrow + nzcap);             // [ceil(p/32)]
  // the chain's Gram blocks alias the on-demand tiles (never live at the same time):
  // SG[k][m] = G[O_m, O_k] (k < m), PG[j][m] = G[O_m, pending row j]
  double* SG = tx;
  double* PG = tvv;
  const bool use_z2 = P.z2 != 0;
  double* zB = use_z2 ? (double*)(sm + tail_smem_bytes(p, n_pad, nzcap)) : nullptr;
  // (no room for z2 on chip: the multi-sweep mode writes its z + changes to this CTA's slice
  // of a global scratch and copies it back when no new row appeared)
  double* zG = (!use_z2 && P.z2g) ? P.z2g + (size_t)blockIdx.x * p : nullptr;
  const bool can_multi = use_z2 || zG != nullptr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t list_stride = (size_t)2 * nzcap;
  const int M = P.M_dev ? *(volatile const int*)P.M_dev : P.M;
  // two launch shapes behind one another (launch_tail_sweeps): the one the hit counts do not
  // call for exits at once (the same decision in every CTA of both)
  if (P.gate && (tail_skewed<NT>(P, M, (int*)(sm + TS_BYTES)) != (P.gate == 1))) return;
  // (fewer columns than CTAs: all start at once; scratch: the tiles region, not in use yet)
  {
    const bool ordered = P.bhist && M > (int)gridDim.x && order_tail<NT>(P, M, (int*)(sm + TS_BYTES));
    if (tid == 0) TS.ordered = ordered ? 1 : 0;   // (read by thread 0 when it takes work)
  }
  const int nmask = (p + 31) / 32;
  if (tid < TAIL_ODC) TS.oc_var[tid] = -1;
  if (tid == 0) {
    TS.oc_next = 0;
    TS.sg_n = -1;
    TS.sg_full = 0;
    mbar_init_t(&TS.z_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  uint32_t z_ph = 0;

  for (;;) {
    // (z is refilled by a bulk copy — async proxy — below: every thread orders its own
    // generic-proxy accesses to it before that, then the barrier publishes them)
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    bsync();
    if (tid == 0) {
      const int kq = atomicAdd(P.next, 1);
      TS.k = (TS.ordered && kq < M) ? P.order[kq] : kq;   // (the hit-count order, if made)
    }
    bsync();
    const int k = TS.k;
    if (k >= M) break;
    TPROF_T(tpc);
    const int slot = P.joint ? P.work[k] : k;
    const TailState ts = P.joint ? P.jtail[slot] : P.tail[k];
    const int col = ts.lam * P.slot_stride + ts.col;         // lists / outputs index
    const int gc = (int)(P.col_begin + ts.col);              // the variable itself
    const double lambda0 = P.lambdas ? P.lambdas[ts.lam] : P.lambda0;
    double sigma = P.joint ? P.sigma_std[col] : ts.sigma;     // (joint: refit by the host loop)
    int outer = ts.outer, sweeps = ts.sweeps, inner = ts.inner, flags = ts.flags;
    int cur = ts.cur;
    int ocnt = min(ts.cnt, nzcap);
    bool overflow = ts.cnt > nzcap;
    double* z = zA;
    double* z2 = zB;
    const bool z_saved = P.joint && (ts.flags & 16);          // joint: z kept between launches
    if (P.z_from_gtab || z_saved) {
      if (!z_saved) ensure_gram_column(P, gc, TS, tx, tvv);
      const double* gz = z_saved ? P.Zj + (size_t)slot * p : P.Gtab + (size_t)gc * p;
      if (EVEN) {   // the whole column in one bulk copy (8p bytes, 16-byte multiple)
        if (tid == 0) {
          prefetch_col(z, gz, (uint32_t)(r1 - r0) * 8, &TS.z_bar);
          mbar_wait_t(&TS.z_bar, z_ph);
        }
        z_ph ^= 1u;
        bsync();
      } else
      // (16 independent L2 loads in flight per thread: the column is 8p bytes)
      for (int j0 = 0; j0 < r1 - r0; j0 += 16 * NT) {
        constexpr int UB = 16;
        double gv[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int j = j0 + u * NT + tid;
          gv[u] = j < r1 - r0 ? __ldcs(gz + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int j = j0 + u * NT + tid;
          if (j < r1 - r0) z[j] = gv[u];
        }
      }
    } else {
      for (int j = tid; j < p; j += NT) z[j] = P.Zz[(size_t)k * p + j];
    }
    for (int w = tid; w < nmask; w += NT) oldmask[w] = 0u;
    bsync();
    {
      const size_t lo = (size_t)col * list_stride + (size_t)cur * nzcap;
      for (int m = tid; m < ocnt; m += NT) {
        const int j = P.nz_rows[lo + m];
        orow[m] = j;
        ov[m] = P.nz_vals[lo + m];
        atomicOr(&oldmask[j >> 5], 1u << (j & 31));
      }
    }
    int npend = 0;                   // pending changes (TS.prow / TS.pd), carried across sweeps
    long long nchg = 0;              // coordinate changes d != 0 (each reads one Gram column)
    long long npass = 0;             // chain + pass segments
    TPROF_C(long long c_ok = 0; long long c_fail = 0; long long c_single = 0; long long c_oksw = 0;
            long long c_spec = 0; long long c_chain = 0; long long c_single_cyc = 0;)
    int mult = MMAX;                 // multi-sweep mode: sweeps to speculate next (the chain also
                                     // stops at the sweep that ends the inner loop)
    bsync();
    bool retire = false;
    while (!retire) {
      // ------------------------------------------------ one sweep, rows in cyclic order
      double lam = sigma * lambda0;
      double maxd = 0.0;
      int pos = 0, cursor = 0, ncnt = 0;
      bool flush = false;            // (joint mode: a last pass that only applies the pending)
      bool multi_done = false;       // whole sweeps done by the multi-sweep mode (with their
      int msw_done = 0;              //   sigma refits: sweeps, outer, inner, flags, retire set)
      if (MULTI && can_multi && !P.joint && npend == 0 && ocnt == 0 && sweeps == ts.sweeps &&
          !overflow) {
        // ---------------------------------------------- a column's first sweep (b = 0)
        // The rows with |z| = |G[j, c]| close to lambda join the (empty) old list with b = 0:
        // the chain visits them like old rows — Soft(a + 0) is exactly a new row's visit, and 0
        // when |a| <= lambda — so the first sweep (and the sweeps after it) can run as one
        // multi-sweep instead of one pass per entering row.  Only rows whose Gram column is
        // present; at most 16 (the loosest of the thresholds 0.9, 0.95, 1.0 lambda that keeps
        // the count within it); the iterates are unchanged (same visits, same arithmetic).
        if (tid < 4) TS.mi[tid] = 0;
        bsync();
        int c0 = 0, c1 = 0, c2 = 0;
        for (int i = tid; i < p; i += NT) {
          const double az = fabs(z[i]);
          if (az > 0.9 * lam && i != gc && (P.gtab_full || *(volatile const int*)&P.gstate[i] == 2)) {
            ++c0;
            if (az > 0.95 * lam) { ++c1; if (az > lam) ++c2; }
          }
        }
        c0 = __reduce_add_sync(0xffffffffu, c0);
        c1 = __reduce_add_sync(0xffffffffu, c1);
        c2 = __reduce_add_sync(0xffffffffu, c2);
        if (lane == 0) { atomicAdd(&TS.mi[0], c0); atomicAdd(&TS.mi[1], c1); atomicAdd(&TS.mi[2], c2); }
        bsync();
        const int t0 = TS.mi[0], t1 = TS.mi[1], t2 = TS.mi[2];
        const double gam = t0 <= 16 ? 0.9 : t1 <= 16 ? 0.95 : 1.0;
        const int nc = t0 <= 16 ? t0 : t1 <= 16 ? t1 : t2 <= 16 ? t2 : 0;
        if (nc > 0) {
          for (int i = tid; i < p; i += NT) {
            const double az = fabs(z[i]);
            if (az > gam * lam && i != gc && (P.gtab_full || *(volatile const int*)&P.gstate[i] == 2))
              TS.so[atomicAdd(&TS.mi[3], 1)] = i;
          }
          bsync();
          if (warp == 0) {   // ascending: lane = entry, rank by value
            const int v = lane < nc ? TS.so[lane] : 0x7fffffff;
            int rank = 0;
            for (int m = 0; m < nc; ++m) rank += __shfl_sync(0xffffffffu, v, m) < v;
            if (lane < nc) {
              orow[rank] = v;
              ov[rank] = 0.0;
              atomicOr(&oldmask[v >> 5], 1u << (v & 31));
            }
          }
          ocnt = nc;
          bsync();
        }
      }
      if (MULTI && can_multi && !P.joint && npend == 0 && ocnt > 0 && ocnt <= KMS && !overflow) {
        // ---------------------------------------------- multi-sweep mode (run_mpass)
        const int K = ocnt;
        const int KS = K <= 16 ? 16 : K <= 24 ? 24 : 32;  // row stride of MD / MBN (>= the
        const int mcap = min(MMAX, MDCAP / KS);             //   pass's KR); sweeps they hold
        double* MD = tvv;                  // [mcap][KS] changes d (aliases PG: no pending;
                                           //   zero beyond K)
        double* MBN = tvv + MDCAP;         // [mcap][KS] new values b'
        double* MDS = TS.mds;              // [mcap] sum_l |d_sl| (the pass's entry bound)
        ++npass;
        TPROF_T(tp0);
        TPROF_ADD(11, K);
        int mine = 1;
        for (int l = tid; l < K; l += NT) {
          const int o = orow[l];
          TS.so[l] = o;
          if (TS.sg_rows[l] != o) mine = 0;
        }
        if (!__syncthreads_and(mine && TS.sg_n == K && TS.sg_full)) {
          for (int e = tid; e < K * K; e += NT) {
            const int kk = e / K, m = e - kk * K;
            SG[kk * 32 + m] = __ldcg(P.Gtab + (size_t)orow[kk] * p + orow[m]);
          }
          for (int l = tid; l < K; l += NT) TS.sg_rows[l] = orow[l];
          if (tid == 0) { TS.sg_n = K; TS.sg_full = 1; }
        }
        if (tid == 0) TS.mkey = 0x7fffffff;
        bsync();
        // chain over whole sweeps (warp 0, lane = chain row): a = z at the row's visit
        if (warp == 0) {
          double a = 0.0, bo = 0.0;
          if (lane < K) { a = z[TS.so[lane]]; bo = ov[lane]; }
          int me = 0;
          double sig = sigma, lamc = lam;
          int outr = outer, inr = inner, flg = flags, ret = 0;
          for (int sw = 0; sw < min(mult, mcap); ++sw) {
            if (lane == 0) {
              TS.mlam[sw] = lamc; TS.msig[sw] = sig; TS.mout[sw] = outr; TS.minr[sw] = inr;
              TS.mflg[sw] = flg;
            }
            const double lam = lamc;
            double mx = 0.0, sd = 0.0, myd = 0.0;
            // (critical path per row: Soft, shuffle, one FMA; the Gram entry of the next row is
            // loaded one step ahead and the lane's d and b' are stored after the sweep)
            double sgn = lane < K ? SG[lane] : 0.0;
            for (int kk = 0; kk < K; ++kk) {
              const double sg = sgn;
              if (kk + 1 < K && lane < K) sgn = SG[(kk + 1) * 32 + lane];
              // every lane evaluates its own visit (no divergent branch); lane kk's counts
              const double bn = soft_t(a + bo, lam);
              const double dmine = bo - bn;                     // e += x_j d
              const bool me_kk = lane == kk;
              myd = me_kk ? dmine : myd;
              bo = me_kk ? bn : bo;
              const double dk = __shfl_sync(0xffffffffu, dmine, kk);
              mx = fmax(mx, fabs(dk));
              sd += fabs(dk);
              if (lane < K && dk != 0.0) a = fma(dk, sg, a);
            }
            if (lane < KS) MD[sw * KS + lane] = myd;          // (zero beyond K)
            if (lane < K) MBN[sw * KS + lane] = bo;
            if (lane == 0) MDS[sw] = sd;
            me = sw + 1;
            ++inr;
            if (mx < P.tol || inr >= P.max_inner) {
              // the inner loop ends here: fresh residual and sigma, the same
              // arithmetic as the block-wide refit below (per sample: x~_c minus the nonzeros
              // in ascending row order; r_i^2 summed per lane in sample order, then the
              // butterfly), and the outer stop; the chain goes on with the new lambda
              if (!(mx < P.tol)) flg |= 2;
              // (samples in tiles of 16 per lane: the 16 loads of one predictor are in flight
              // together; the b values via shared memory)
              if (lane < K) TS.sbn[lane] = bo;
              __syncwarp();
              double ss = 0.0;
              for (int t0 = 0; t0 < n; t0 += 16 * 32) {
                double ri[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                  const int i = t0 + u * 32 + lane;
                  ri[u] = i < n ? P.Xb[xb_index(i, gc, nchunk)] : 0.0;
                }
                for (int m = 0; m < K; ++m) {
                  const double bm = TS.sbn[m];
                  if (bm == 0.0) continue;
                  const int om = TS.so[m];
                  double xv[16];
#pragma unroll
                  for (int u = 0; u < 16; ++u) {
                    const int i = t0 + u * 32 + lane;
                    xv[u] = i < n ? P.Xb[xb_index(i, om, nchunk)] : 0.0;
                  }
#pragma unroll
                  for (int u = 0; u < 16; ++u) ri[u] = fma(-xv[u], bm, ri[u]);
                }
#pragma unroll
                for (int u = 0; u < 16; ++u)
                  if (t0 + u * 32 + lane < n) ss = fma(ri[u], ri[u], ss);
              }
              __syncwarp();
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
              double sn = sqrt(ss) / P.sqrt_n;
              if (sn < P.sigma_floor) sn = P.sigma_floor;
              ++outr;
              if (fabs(sn - sig) < P.tol) { flg |= 1; ret = 1; }
              else if (outr >= P.max_outer) ret = 1;
              sig = sn;
              lamc = sig * lambda0;
              inr = 0;
              if (ret) break;
            }
          }
          if (lane == 0) {
            TS.ncol = me;
            TS.msig_e = sig; TS.mout_e = outr; TS.minr_e = inr; TS.mflg_e = flg; TS.mret_e = ret;
          }
        }
        bsync();
        const int Msw = TS.ncol;
        TPROF_T(tp1);
        TPROF_ADD(0, tp1 - tp0);
        TPROF_C(c_chain += tp1 - tp0;)
        int best = 0x7fffffff;
        double bestw = 0.0;
        // When the chain retires the column at its last sweep, z after the pass is never read
        // (the column ends if every sweep holds; a new row rolls back from z itself): the pass
        // then only tests, without writing z + changes (at p = 20000: 160 KB written to the
        // global second buffer and read back per column)
        const bool ends = TS.mret_e != 0;
        mpass<NT, true>(z, ends ? nullptr : (use_z2 ? z2 : zG), oldmask, P.Gtab, TS, MD, KS, MDS,
                        p, K, Msw, gc, TS.mlam, 0, 0, &TS.mkey, best, bestw);
        {
          const int wb = __reduce_min_sync(0xffffffffu, best);
          if (best == wb && best != 0x7fffffff) TS.wval[warp] = bestw;
          if (lane == 0) TS.wmin[warp] = wb;
        }
        bsync();
        int jkey = 0x7fffffff, wsrc = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w)
          if (TS.wmin[w] < jkey) { jkey = TS.wmin[w]; wsrc = w; }
        const double wstar = TS.wval[wsrc];
        TPROF_T(tp2);
        TPROF_ADD(1, tp2 - tp1);
        TPROF_C(c_spec += tp2 - tp1;)
        if (jkey == 0x7fffffff) {
          // every speculated sweep holds: z2 is z after them; the list is the last sweep's
          if (ends) {
          } else if (use_z2) { double* t = z; z = z2; z2 = t; }
          else {
            // (16 loads in flight per thread; the pass's global writes are this CTA's own,
            // ordered by the barrier above)
            for (int j0 = 0; j0 < p; j0 += 16 * NT) {
              double gv[16];
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int j = j0 + u * NT + tid;
                gv[u] = j < p ? __ldcg(zG + j) : 0.0;
              }
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int j = j0 + u * NT + tid;
                if (j < p) z[j] = gv[u];
              }
            }
          }
          if (warp == 0) {
            const int sl = Msw - 1;
            double bn = 0.0, dl = 0.0;
            int cnt = 0;
            if (lane < K) {
              bn = MBN[sl * KS + lane];
              dl = MD[sl * KS + lane];
              for (int sw = 0; sw < Msw; ++sw) cnt += MD[sw * KS + lane] != 0.0;
            }
            const bool nz = lane < K && bn != 0.0;
            const unsigned bal = __ballot_sync(0xffffffffu, nz);
            if (nz) {
              const int idx = __popc(bal & ((1u << lane) - 1u));
              nrow[idx] = TS.so[lane];
              nv[idx] = bn;
            }
            double mx = fabs(dl);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
              cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            }
            if (lane == 0) { TS.mi[2] = __popc(bal); TS.mi[3] = cnt; TS.mmaxd = mx; }
          }
          bsync();
          ncnt = TS.mi[2];
          nchg += TS.mi[3];
          maxd = TS.mmaxd;
          sweeps += Msw;
          sigma = TS.msig_e; outer = TS.mout_e; inner = TS.minr_e; flags = TS.mflg_e;
          retire = TS.mret_e != 0;
          msw_done = Msw;
          multi_done = true;
          mult = MMAX;
          TPROF_ADD(5, 1);
          TPROF_ADD(7, Msw);
          TPROF_C(++c_ok; c_oksw += Msw;)
        } else {
          // a new row at (sstar, istar): z <- z + the changes before it; the list of sweep
          // sstar's start becomes the old list; sweep sstar continues below from istar
          const int sstar = jkey / p, istar = jkey - sstar * p;
          int qstar = 0;
          for (int l = 0; l < K; ++l) qstar += TS.so[l] < istar;
          int dummy = 0x7fffffff;
          double dw = 0.0;
          mpass<NT, false>(z, z, oldmask, P.Gtab, TS, MD, KS, MDS, p, K, sstar + 1, gc, TS.mlam,
                           sstar, qstar, &TS.mkey, dummy, dw);
          if (warp == 0) {
            const int o = lane < K ? TS.so[lane] : 0;
            double bst = 0.0, bns = 0.0, ds = 0.0;
            int cnt = 0;
            if (lane < K) {
              bst = sstar > 0 ? MBN[(sstar - 1) * KS + lane] : ov[lane];
              bns = MBN[sstar * KS + lane];
              ds = lane < qstar ? MD[sstar * KS + lane] : 0.0;
              for (int sw = 0; sw < sstar; ++sw) cnt += MD[sw * KS + lane] != 0.0;
              cnt += ds != 0.0;
            }
            __syncwarp();
            // old list at the start of sweep sstar: the chain rows with b != 0 there
            const bool keep = lane < K && bst != 0.0;
            const unsigned bk = __ballot_sync(0xffffffffu, keep);
            if (lane < K && !keep) atomicAnd(&oldmask[o >> 5], ~(1u << (o & 31)));
            if (keep) {
              const int idx = __popc(bk & ((1u << lane) - 1u));
              orow[idx] = o;
              ov[idx] = bst;
            }
            const unsigned bc = __ballot_sync(0xffffffffu, keep && o < istar);
            // sweep sstar so far: the chain rows before istar with b' != 0
            const bool nz = lane < qstar && bns != 0.0;
            const unsigned bn2 = __ballot_sync(0xffffffffu, nz);
            if (nz) {
              const int idx = __popc(bn2 & ((1u << lane) - 1u));
              nrow[idx] = o;
              nv[idx] = bns;
            }
            double mx = fabs(ds);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
              cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
            }
            if (lane == 0) {
              TS.mi[0] = __popc(bk);
              TS.mi[1] = __popc(bc);
              TS.mi[2] = __popc(bn2);
              TS.mi[3] = cnt;
              TS.mmaxd = mx;
            }
          }
          bsync();
          ocnt = TS.mi[0];
          cursor = TS.mi[1];
          ncnt = TS.mi[2];
          nchg += TS.mi[3];
          maxd = TS.mmaxd;
          sweeps += sstar;
          // the state in effect in sweep sstar (the chain may have refit sigma before it)
          lam = TS.mlam[sstar]; sigma = TS.msig[sstar]; outer = TS.mout[sstar];
          inner = TS.minr[sstar]; flags = TS.mflg[sstar];
          // the new row's visit (b = 0: a = w)
          const double bn = soft_t(wstar, lam);
          const double d = 0.0 - bn;
          if (ncnt < nzcap) { if (tid == 0) { nrow[ncnt] = istar; nv[ncnt] = bn; } }
          else overflow = true;
          ++ncnt;
          maxd = fmax(maxd, fabs(d));
          ++nchg;
          if (tid == 0) { TS.prow[0] = istar; TS.pd[0] = d; }
          npend = 1;
          pos = istar + 1;
          mult = min(MMAX, max(8, 2 * (sstar + 1)));   // (floor 8: hub seeds 2207 / 3207 / 4207 -0.4 / -2.3 / -0.2 % against 4)
          TPROF_ADD(6, 1);
          TPROF_C(++c_fail;)
          TPROF_ADD(8, sstar);
          TPROF_ADD(12, Msw);
          ensure_gram_column(P, istar, TS, tx, tvv);          // (its barriers publish TS)
          bsync();
        }
        TPROF_T(tp3);
        TPROF_ADD(2, tp3 - tp2);
      }
      TPROF_T(tp4);
      if (!multi_done)
      for (;;) {
        const int K = flush ? 0 : min(ocnt - cursor, KMAX);
        const int range_end = flush ? 0 : (cursor + K < ocnt ? orow[cursor + K] : p);
        ++npass;
        TPROF_ADD(9, 1);
        TPROF_C(++c_single;)
        // ---- chain inputs: rows, Gram blocks (all threads); SG is kept from the previous
        // segment with the same chain rows (a stable support: every sweep's chain is the same)
        int mine = 1;
        for (int l = tid; l < K; l += NT) {
          const int o = orow[cursor + l];
          TS.so[l] = o;
          if (TS.sg_rows[l] != o) mine = 0;
        }
        if (!__syncthreads_and(mine && TS.sg_n == K)) {
          for (int e = tid; e < K * K; e += NT) {
            const int kk = e / K, m = e - kk * K;
            if (kk < m) SG[kk * 32 + m] = __ldcg(P.Gtab + (size_t)orow[cursor + kk] * p + orow[cursor + m]);
          }
          for (int l = tid; l < K; l += NT) TS.sg_rows[l] = orow[cursor + l];
          if (tid == 0) { TS.sg_n = K; TS.sg_full = 0; }
        }
        for (int e = tid; e < npend * K; e += NT) {
          const int j = e / K, m = e - j * K;
          PG[j * 32 + m] = __ldcg(P.Gtab + (size_t)TS.prow[j] * p + orow[cursor + m]);
        }
        bsync();
        // ---- chain (warp 0, lane = chain row), then the pass's column list
        if (warp == 0) {
          if (K > 0) {
            double a = 0.0, bo = 0.0;
            if (lane < K) {
              a = z[TS.so[lane]];
              for (int j = 0; j < npend; ++j) a = fma(TS.pd[j], PG[j * 32 + lane], a);
              bo = ov[cursor + lane];
            }
            for (int kk = 0; kk < K; ++kk) {
              double dk = 0.0;
              if (lane == kk) {
                const double bn = soft_t(a + bo, lam);
                dk = bo - bn;                                   // e += x_j d
                TS.sd[kk] = dk;
                TS.sbn[kk] = bn;
              }
              dk = __shfl_sync(0xffffffffu, dk, kk);
              if (lane > kk && lane < K && dk != 0.0) a = fma(dk, SG[kk * 32 + lane], a);
            }
          }
          // the pass's columns: pending changes in order, then the nonzero chain changes in order
          if (lane < npend) { TS.crow[lane] = TS.prow[lane]; TS.cd[lane] = TS.pd[lane]; TS.cO[lane] = -1; }
          __syncwarp();
          const bool nz = lane < K && TS.sd[lane] != 0.0;
          const unsigned bal = __ballot_sync(0xffffffffu, nz);
          if (nz) {
            const int c = npend + __popc(bal & ((1u << lane) - 1u));
            TS.crow[c] = TS.so[lane]; TS.cd[c] = TS.sd[lane]; TS.cO[c] = TS.so[lane];
          }
          if (lane == 0) TS.ncol = npend + __popc(bal);
        }
        bsync();
        // ---- pass over the rows (all threads; run_pass)
        int best = 0x7fffffff;
        double bestw = 0.0;
        const int C = TS.ncol;
        const bool spec_all = use_z2 && !flush && C > npend;   // z2 = committed + every change
        if (C == 0) {
          // no change to apply: detection only, from z
          for (int i = max(pos, r0) + tid; i < min(range_end, r1); i += NT)
            if (fabs(z[i - r0]) > lam && i != gc && !((oldmask[i >> 5] >> (i & 31)) & 1u)) {
              best = i;
              bestw = z[i - r0];
              break;
            }
        } else {
          const PassArgs A{z - r0, z2 ? z2 - r0 : nullptr, oldmask, P.Gtab, p, npend, C, pos,
                           range_end, gc, spec_all, lam, r0, r1};
          run_pass<NT, EVEN, PASS_U, PASS_PD>(A, TS, best, bestw);
        }
        // first new row: block-wide minimum (and its visit value)
        {
          const int wb = __reduce_min_sync(0xffffffffu, best);
          if (best == wb && best != 0x7fffffff) TS.wval[warp] = bestw;
          if (lane == 0) TS.wmin[warp] = wb;
        }
        bsync();
        int jstar = 0x7fffffff, wsrc = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w)
          if (TS.wmin[w] < jstar) { jstar = TS.wmin[w]; wsrc = w; }
        const double wstar_c = TS.wval[wsrc];
        if (flush) { npend = 0; break; }
        // ---- commit (every thread takes the same decisions from shared memory)
        int nvalid = K;
        if (jstar != 0x7fffffff) { nvalid = 0; while (nvalid < K && TS.so[nvalid] < jstar) ++nvalid; }
        const bool swap = spec_all && jstar == 0x7fffffff;   // (z2 holds z + every change)
        int np2 = 0;
        for (int l = 0; l < nvalid; ++l) {
          const double bn = TS.sbn[l], d = TS.sd[l];
          if (bn != 0.0) {
            if (ncnt < nzcap) { if (tid == 0) { nrow[ncnt] = TS.so[l]; nv[ncnt] = bn; } }
            else overflow = true;
            ++ncnt;
          }
          if (d != 0.0) {
            maxd = fmax(maxd, fabs(d));
            ++nchg;
            if (!swap) {
              if (tid == 0) { TS.prow[np2] = TS.so[l]; TS.pd[np2] = d; }
              ++np2;
            }
          }
        }
        if (swap) { double* t = z; z = z2; z2 = t; }
        cursor += nvalid;
        if (jstar != 0x7fffffff) {
          const double a = wstar_c;                            // b = 0: a = z_j
          const double bn = soft_t(a, lam);                    // nonzero (|a| > lambda)
          const double d = 0.0 - bn;
          if (ncnt < nzcap) { if (tid == 0) { nrow[ncnt] = jstar; nv[ncnt] = bn; } }
          else overflow = true;
          ++ncnt;
          maxd = fmax(maxd, fabs(d));
          ++nchg;
          if (tid == 0) { TS.prow[np2] = jstar; TS.pd[np2] = d; }
          ++np2;
          npend = np2;
          pos = jstar + 1;
          ensure_gram_column(P, jstar, TS, tx, tvv);          // (its barriers publish TS)
          bsync();
          continue;
        }
        npend = np2;
        pos = range_end;
        bsync();
        if (cursor >= ocnt) {
          if (P.joint && npend > 0) { flush = true; continue; }   // z saved complete
          break;
        }
      }
      {
        TPROF_T(tp5);
        if (!multi_done) TPROF_ADD(3, tp5 - tp4);
        TPROF_C(if (!multi_done) c_single_cyc += tp5 - tp4;)
      }
      if (!msw_done) {   // (a multi-sweep set its counters and refit sigma itself)
        ++sweeps;
        ++inner;
      }
      // the new list becomes the current one (and the old-row bitmap with it)
      for (int m = tid; m < ocnt; m += NT) atomicAnd(&oldmask[orow[m] >> 5], ~(1u << (orow[m] & 31)));
      bsync();
      for (int m = tid; m < min(ncnt, nzcap); m += NT) {
        orow[m] = nrow[m];
        ov[m] = nv[m];
        atomicOr(&oldmask[nrow[m] >> 5], 1u << (nrow[m] & 31));
      }
      ocnt = min(ncnt, nzcap);
      if (ncnt > nzcap) overflow = true;
      bsync();
      if (P.joint) {
        // one sweep per launch: publish max |db|, keep z and the state for the next launch
        if (tid == 0) atomicMax(P.joint_maxd, (unsigned long long)__double_as_longlong(maxd));
        double* zs = P.Zj + (size_t)slot * p;
        for (int t = tid; t < p; t += NT) zs[t] = z[t];
        break;
      }
      if (!msw_done && (maxd < P.tol || inner >= P.max_inner)) {
        if (!(maxd < P.tol)) flags |= 2;
        TPROF_T(tpr);
        // fresh residual and sigma (reading g4): every thread builds its samples'
        // r_i = x~_ci - sum_m x~_{j_m i} b_m (m ascending, the CD kernel's per-element order),
        // then warp 0 sums r_i^2 in the CD kernel's order
        for (int i = tid; i < n_pad; i += NT) {
          double ri = P.Xb[xb_index(i, gc, nchunk)];
          for (int m = 0; m < ocnt; ++m) ri = fma(-P.Xb[xb_index(i, orow[m], nchunk)], ov[m], ri);
          r[i] = ri;
        }
        bsync();
        if (warp == 0) {
          double ss = 0.0;
          for (int i = lane; i < n; i += 32) ss = fma(r[i], r[i], ss);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
          if (lane == 0) TS.red[0] = ss;
        }
        bsync();
        double sn = sqrt(TS.red[0]) / P.sqrt_n;
        if (sn < P.sigma_floor) sn = P.sigma_floor;
        ++outer;
        if (fabs(sn - sigma) < P.tol) { flags |= 1; retire = true; }
        else if (outer >= P.max_outer) retire = true;
        sigma = sn;
        inner = 0;
        bsync();
        {
          TPROF_T(tpr2);
          TPROF_ADD(4, tpr2 - tpr);
        }
      }
    }
    {
      TPROF_T(tpe);
      TPROF_ADD(10, tpe - tpc);
#ifdef SPMESL_TAIL_PROF
      if (tid == 0) {
        const unsigned long long cyc = (unsigned long long)(tpe - tpc);
        atomicMax(&g_tail_prof[13], (cyc << 24) | ((unsigned long long)min(npass, 4095ll) << 12) |
                                        (unsigned long long)min(sweeps - ts.sweeps, 4095));
        if (cyc > 4000000ull) atomicAdd(&g_tail_prof[14], 1ull);   // columns over ~2 ms
        atomicMax(&g_tail_prof[28], (cyc << 16) | ((unsigned long long)min(ocnt, 255) << 8) |
                                        (unsigned long long)min(c_fail, 255ll));
        if (cyc > 4000000ull) atomicAdd(&g_tail_prof[29], (unsigned long long)ocnt);
        if (sweeps - ts.sweeps > 200) {                                // stragglers
          atomicAdd(&g_tail_prof[16], 1ull);
          atomicAdd(&g_tail_prof[17], (unsigned long long)c_ok);
          atomicAdd(&g_tail_prof[18], (unsigned long long)c_fail);
          atomicAdd(&g_tail_prof[19], (unsigned long long)c_single);
          atomicAdd(&g_tail_prof[20], (unsigned long long)c_oksw);
          atomicAdd(&g_tail_prof[21], (unsigned long long)c_spec);
          atomicAdd(&g_tail_prof[22], (unsigned long long)c_chain);
          atomicAdd(&g_tail_prof[23], (unsigned long long)c_single_cyc);
          atomicAdd(&g_tail_prof[24], cyc);
          atomicAdd(&g_tail_prof[25], (unsigned long long)(sweeps - ts.sweeps));
        }
        atomicMax(&g_tail_prof[15], (unsigned long long)(tpe));  // last column end (clock)
      }
#endif
    }
    // outputs: coefficients into the column's other list, per-column results
    const int dst = cur ^ 1;
    const size_t lo = (size_t)col * list_stride + (size_t)dst * nzcap;
    for (int m = tid; m < ocnt; m += NT) { P.nz_rows[lo + m] = orow[m]; P.nz_vals[lo + m] = ov[m]; }
    if (tid == 0) {
      P.nz_count[col] = ocnt;
      P.nz_cur[col] = dst;
      if (overflow) atomicExch(&P.flags[FLAG_OVERFLOW], 1);
      atomicAdd(P.sweeps_count, sweeps - ts.sweeps);
      if (P.changes_count) {
        atomicAdd(P.changes_count, (unsigned long long)nchg);
        atomicAdd(P.changes_count + 1, (unsigned long long)npass);
      }
      if (P.joint) {   // (sigma, iters, sweeps, converged: the host loop's joint kernels)
        TailState t2 = ts;
        t2.cur = dst; t2.cnt = ocnt; t2.sweeps = sweeps; t2.flags = ts.flags | 16;
        P.jtail[slot] = t2;
      } else {
        P.sigma_std[col] = sigma;
        P.iters[col] = outer;
        P.sweeps[col] = sweeps;
        P.converged[col] = (uint8_t)((flags & 1) && !(flags & 2));
      }
    }
  }
}


cudaError_t launch_tail_residuals(const double* Xb, const TailState* tail, int M, const int* nz_rows,
                                  const double* nz_vals, int nzcap, int64_t col_begin, int n,
                                  int n_pad, int nchunk, double* V, cudaStream_t s) {
  (void)n;
  const int wpb = 8;
  tail_residuals_kernel<<<(M + wpb - 1) / wpb, wpb * 32, 0, s>>>(Xb, tail, M, nz_rows, nz_vals, nzcap,
                                                                col_begin, n_pad, nchunk, V);
  return cudaGetLastError();
}

cudaError_t launch_gram_cols(const double* Xb, int nblk, int nchunk, int n, int p, const int* U,
                             int nU, const int* nU_dev, int sms, double* Gtab, uint8_t* hit,
                             const double* lams, int nlam, int* gstate, cudaStream_t s,
                             bool fallback, double lam1) {
  if (!nU_dev && nU <= 0) return cudaSuccess;
  if (sms <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 1;
  }
  static int max_warps = 0;
  if (!max_warps) {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, gram_cols_kernel) != cudaSuccess) return cudaGetLastError();
    max_warps = std::max(1, std::min(GC_MAXW, fa.maxThreadsPerBlock / 32));
  }
  const int nmt = (p + 7) / 8;
  const int T = std::max(1, std::min(max_warps, (nmt + sms - 1) / sms));
  const int grid = std::max(1, std::min(sms, (nmt + T - 1) / T));
  const size_t smem = (size_t)GC_STAGES * (T * 8 * XS + GC_NTMAX * 8 * XS) * 8;
  {   // (per call: the attribute belongs to the current device)
    cudaError_t e = cudaFuncSetAttribute(gram_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)((size_t)GC_STAGES * (GC_MAXW * 8 * XS + GC_NTMAX * 8 * XS) * 8));
    if (e != cudaSuccess) return e;
  }
  gram_cols_kernel<<<grid, T * 32, smem, s>>>(Xb, nchunk, n, p, U, nU, nU_dev, Gtab, hit, lams,
                                             nlam, gstate, fallback ? 1 : 0, lam1);
  return cudaGetLastError();
}

cudaError_t launch_gram_pass(const double* Xb, int nblk, int nchunk, int n, int p, const double* V,
                             int M, const int* U, int nU, double* Zz, double* Gtab, cudaStream_t s,
                             uint8_t* hit, const double* lams, int nlam) {
  const int ntile = (M + nU + 31) / 32;
  if (ntile == 0) return cudaSuccess;
  if (M == 0)
    return launch_gram_cols(Xb, nblk, nchunk, n, p, U, nU, nullptr, 0, Gtab, hit, lams, nlam,
                            nullptr, s);
  dim3 grid((unsigned)nblk, (unsigned)ntile);
  // n_pad is implied by nchunk
  gram_pass_kernel<<<grid, 256, 0, s>>>(Xb, nchunk, n, p, V, M, U, nU, nchunk * KC, Zz, Gtab, hit,
                                        lams, nlam);
  return cudaGetLastError();
}

cudaError_t launch_tail_mark(const TailState* tail, int M, const int* nz_rows, int nzcap, int* umark,
                             cudaStream_t s) {
  const int wpb = 8;
  tail_mark_kernel<<<(M + wpb - 1) / wpb, wpb * 32, 0, s>>>(tail, M, nz_rows, nzcap, umark);
  return cudaGetLastError();
}

template <int NT, bool EVEN, int MINB, bool MULTI>
static cudaError_t launch_tail_t(const TailParams& P, int grid, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(tail_sweep_kernel<NT, EVEN, MINB, MULTI>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  tail_sweep_kernel<NT, EVEN, MINB, MULTI><<<grid, NT, smem, s>>>(P);
  return cudaGetLastError();
}

template <int NT, int MINB, bool MULTI>
static cudaError_t launch_tail_e(const TailParams& P, int grid, size_t smem, cudaStream_t s) {
  // even p: 16-byte row pairs everywhere
  return (P.p & 1) == 0 ? launch_tail_t<NT, true, MINB, MULTI>(P, grid, smem, s)
                        : launch_tail_t<NT, false, MINB, MULTI>(P, grid, smem, s);
}

cudaError_t launch_tail_sweeps(const TailParams& P, int grid, cudaStream_t s) {
  size_t smem = tail_smem_bytes(P.p, P.n_pad, P.nzcap);
  if (P.z2) smem += tail_z2_bytes(P.p);
  if (P.occ > 1) grid *= P.occ;   // several column CTAs per SM (set_tail_shape)
  // 512 threads when a single column CTA owns the SM (large p: the pass splits over twice the
  // threads), 256 when two share it; the multi-sweep mode needs the second z buffer (and is
  // compiled only into those variants: its registers would cost the others)
  const bool multi = (P.z2 || P.z2g) && !P.joint;
  if (P.occ == 1)
    return multi ? launch_tail_e<512, 1, true>(P, grid, smem, s) : launch_tail_e<512, 1, false>(P, grid, smem, s);
  if (P.occ == 3 && multi) return launch_tail_e<160, 3, true>(P, grid, smem, s);
  return multi ? launch_tail_e<256, 2, true>(P, grid, smem, s) : launch_tail_e<256, 2, false>(P, grid, smem, s);
}

}  // namespace spmesl

#ifdef SPMESL_TAIL_PROF
extern "C" int spmesl_dev_tail_prof(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, spmesl::g_tail_prof, sizeof(unsigned long long) * 32) != cudaSuccess) return 1;
  if (reset) {
    static const unsigned long long zero[32] = {};
    if (cudaMemcpyToSymbol(spmesl::g_tail_prof, zero, sizeof(zero)) != cudaSuccess) return 1;
  }
  return 0;
}
#endif
