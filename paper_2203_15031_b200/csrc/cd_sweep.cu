// Persistent column-parallel coordinate-descent kernel for SPMESL (steps a3-a7 of
// SURVEY.md §8(a)).  One CTA per SM; each CTA keeps T "slots" (resident columns c, i.e.
// independent scaled-lasso problems) and sweeps the predictor rows j = 0..p-1
// for all of them together (Proposition 2).
//
// Per column the arithmetic is exactly Algorithm 1 with per-column stopping
// (reading g1): a_j = x_j^T e / n + b_j, b_j <- Soft_{sigma lambda0}(a_j), e += x_j (b_old -
// b_new), inner stop max |db| < tol, then a fresh residual, sigma = max(||e||/sqrt(n), floor),
// outer stop |dsigma| < tol.  A column that retires frees its slot, which is refilled from a
// global queue at the next sweep boundary (the active-set shrink of Alg. 3, P:920-926,
// generalised to dynamic refill).  Columns only join at row 0, so each column sees the
// exact cyclic order j = 0..p-1 of Algorithm 1.
//
// Rows are processed in blocks of J = 32 with a lag-1 software pipeline:
//   step t:  MMA warps      Z_t = X_{B_t}^T R / n      (dense fp64 contraction over n,
//                           mma.sync m8n8k4 DMMA; X tiles stream L2 -> smem by
//                           cp.async.bulk into two mbarrier rings fed by a producer warp)
//            epilogue warps finish block t-1:
//              a_jc = Z_{t-1}[j,c] + sum_{j' in B_{t-2} changed} G^x_{jj'} d_j'c + b_jc
//              (R used by Z_{t-1} lacked block t-2's updates; G^x = x_j^T x_j'/n folds them
//              in exactly), Soft for all 32 rows at once; columns with a change are walked
//              row by row from the first changed row, adding G^w_{jj'} d_j'c for the changes
//              earlier in the same block.
//   between steps: R_c += x_j d_jc for block t-1's changes (rare; skipped when none).
// This is Proposition 2's row order j = 0..p-1 with the residual identity
// x_j^T (e + x_j' d) / n = x_j^T e / n + (x_j^T x_j' / n) d, i.e. the same iterates as
// Algorithm 1 up to rounding.  Every dot product is reduced in one fixed order (chunk-parity
// partials p0 + p1), so a column's result does not depend on its slot, its CTA, the tile
// occupancy or the GPU count.
//
// Coefficients never live in a dense p x p array: each column keeps its nonzeros as a list
// (rows ascending) rebuilt every sweep (double-buffered in HBM), read back with a cursor in
// the next sweep and used for the residual refresh and the final CSC export.
#include <algorithm>
#include <cstdio>
#include "spmesl_internal.cuh"

namespace spmesl {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Named barriers in their NON-aligned form (barrier.sync / barrier.arrive): several call
// sites follow lane-divergent code, and the .aligned form that bar.sync denotes requires the
// whole warp to arrive converged.  The __syncwarp() reconverges the warp first.
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  __syncwarp();
  asm volatile("barrier.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  __syncwarp();
  asm volatile("barrier.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
// barrier ids: 0 __syncthreads, 1 work warps (MMA + epilogue), 2 producer handshake,
// 3..6 MMA warp pairs (wg, wg + 4)
constexpr int BAR_WORK = 1, BAR_PROD = 2, BAR_PAIR0 = 3;
__device__ __forceinline__ void work_sync() { named_bar_sync(BAR_WORK, WORK_THREADS); }

// D(8x8) += A(8x4, row) * B(4x8, col), fp64 tensor-core MMA.
// Fragments (verified on B200, microbench/peaks.cu): lane = 4g + t;
//   a = A[g][t], b = B[t][g], d0 = D[g][2t], d1 = D[g][2t+1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Soft_lambda(a) = sign(a)(|a| - lambda)_+, +0.0 when |a| <= lambda (reading g18).
__device__ __forceinline__ double soft(double a, double lam) {
  double m = fabs(a) - lam;
  return m > 0.0 ? copysign(m, a) : 0.0;
}

constexpr int MAX_NST = 12;  // max X chunk pipeline depth (runtime: as many as smem allows)

constexpr int JP = J + 1;    // padded row-block stride of the per-column [c][row] tiles

struct SlotState {
  int col[MAX_T];       // local column index, -1 = free
  int outer[MAX_T];
  int sweeps[MAX_T];
  int inner[MAX_T];
  int flags[MAX_T];     // bit0 sigma converged, bit1 inner cap hit
  int cur[MAX_T];       // which list holds the previous sweep's coefficients
  int cnt_old[MAX_T];
  int cnt_new[MAX_T];
  int cursor[MAX_T];
  int first[MAX_T];     // first changed row in the block being finished (J = none)
  int nchg[2][MAX_T];   // changes per column in the block of parity x
  int retire[MAX_T];
  double sigma[MAX_T];
  double lam[MAX_T];
  double maxd[MAX_T];
  // control
  int A;
  int go;
  int taken;            // columns this CTA has taken from the queue
  int nmoves, nloads;
  int mv_dst[MAX_T], mv_src[MAX_T];
  int ld_dst[MAX_T];
};

// Shared-memory carve-up (bytes) for T slots and padded n (plus the X ring).
static __host__ __device__ size_t smem_fixed_bytes(int T, int n_pad) {
  size_t b = 0;
  b += (size_t)T * (n_pad + RPAD) * 8;  // Rs      [T][n_pad+RPAD]
  b += (size_t)2 * T * JP * 8;          // Zp      [2 (block parity)][T][JP]
  b += (size_t)2 * J * T * 8;           // chg_d   [2][J][T]
  b += (size_t)2 * J * T;               // chg_row [2][J][T]
  b = (b + 15) & ~(size_t)15;
  b += sizeof(SlotState);
  b = (b + 15) & ~(size_t)15;
  b += 2 * MAX_NST * 8;                 // mbarriers
  b = (b + 127) & ~(size_t)127;         // stage ring is 128-byte aligned
  return b;
}

int cd_stages(int T, int n_pad, size_t smem_optin) {
  const size_t fixed = smem_fixed_bytes(T, n_pad);
  if (fixed + 2 * (size_t)CHUNK_BYTES > smem_optin) return 0;
  // even: the stages are split between the two parity-group rings
  return (int)std::min<size_t>(MAX_NST, (smem_optin - fixed) / CHUNK_BYTES) & ~1;
}

size_t cd_smem_bytes(int T, int n_pad) {     // minimum (2 stages)
  return smem_fixed_bytes(T, n_pad) + 2 * (size_t)CHUNK_BYTES;
}

// One row block's contraction for the chunks q = grp (mod 2) of this warp's parity group,
// for the warp's MT x NT subtile of 8x8 tiles starting at (m0, n0); the two parity partials
// of a subtile (warps wg and wg+4) are combined as (p0 + p1) * (1/n) into Zb[col][row].
// Paired-k fragments: for k-pair kp of a chunk, lane (g, t) loads the 2 consecutive samples
// k = 8kp + 2t, 8kp + 2t + 1 of row g with one 128-bit LDS; the first DMMA takes the even
// sample, the second the odd one (the same k mapping for A and B).  Each output's
// accumulation order depends only on k, never on the subtile mapping, so results are
// independent of NTa and of the column's slot.
template <int MT, int NT, bool COMPUTE>
__device__ __forceinline__ void gemm_block(const double* __restrict__ Xs, const double* __restrict__ Rs,
                                           double* __restrict__ Zb, uint64_t* full, uint64_t* empty,
                                           int grp, int wg, int m0, int n0, int nchunk, int NSTG,
                                           int& s, uint32_t& ph, int SR, double inv_n, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  // two accumulators per 8x8 tile: even samples (h = 0) and odd samples (h = 1) of each pair,
  // so consecutive DMMAs never depend on each other; summed as (even + odd) at the end
  double acc[MT][NT][2][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) acc[mi][ni][h][0] = acc[mi][ni][h][1] = 0.0;
  const double* rbase = Rs + (size_t)(n0 * 8 + g) * SR + 2 * t4;
  for (int q = grp; q < nchunk; q += 2) {
    mbar_wait(&full[s], ph);
    const double* xs = Xs + (size_t)s * CHUNK_DOUBLES + (size_t)(m0 * 8 + g) * XS + 2 * t4;
    const double* rs = rbase + q * KC;
    const int sw = g & 1;                 // row parity of this lane's A rows (xswz)
#pragma unroll
    for (int kp = 0; kp < (COMPUTE ? KC / 8 : 0); ++kp) {
      double2 a[MT], bb[NT];
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) a[mi] = *(const double2*)(xs + mi * 8 * XS + (kp ^ sw) * 8);
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) bb[ni] = *(const double2*)(rs + (size_t)ni * 8 * SR + kp * 8);
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) dmma(acc[mi][ni][0][0], acc[mi][ni][0][1], a[mi].x, bb[ni].x);
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) dmma(acc[mi][ni][1][0], acc[mi][ni][1][1], a[mi].y, bb[ni].y);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == NSTG) { s = 0; ph ^= 1u; }
  }
  // parity-1 partial -> Zb, pair barrier, parity-0 warp adds its partial and scales by 1/n
  if (grp == 1) {
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        double* z = Zb + (size_t)((n0 + ni) * 8 + 2 * t4) * JP + (m0 + mi) * 8 + g;
        z[0] = acc[mi][ni][0][0] + acc[mi][ni][1][0];
        z[JP] = acc[mi][ni][0][1] + acc[mi][ni][1][1];
      }
  }
  named_bar_sync(BAR_PAIR0 + wg, 64);
  if (grp == 0) {
#pragma unroll
    for (int mi = 0; mi < MT; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        double* z = Zb + (size_t)((n0 + ni) * 8 + 2 * t4) * JP + (m0 + mi) * 8 + g;
        z[0] = ((acc[mi][ni][0][0] + acc[mi][ni][1][0]) + z[0]) * inv_n;
        z[JP] = ((acc[mi][ni][0][1] + acc[mi][ni][1][1]) + z[JP]) * inv_n;
      }
  }
}

// Subtile mapping of the 4 warps of a parity group for NTa active n-tiles.
template <bool COMPUTE>
__device__ __forceinline__ void run_gemm(int NTa, int grp, int wg, const double* Xs,
                                         const double* Rs, double* Zb, uint64_t* full,
                                         uint64_t* empty, int nchunk, int NSTG, int& s,
                                         uint32_t& ph, int SR, double inv_n, int lane) {
  switch (NTa) {
    case 4:
      gemm_block<2, 2, COMPUTE>(Xs, Rs, Zb, full, empty, grp, wg, 2 * (wg & 1), 2 * (wg >> 1),
                                nchunk, NSTG, s, ph, SR, inv_n, lane);
      break;
    case 3:
      if (wg < 2)
        gemm_block<2, 2, COMPUTE>(Xs, Rs, Zb, full, empty, grp, wg, 2 * (wg & 1), 0, nchunk, NSTG,
                                  s, ph, SR, inv_n, lane);
      else
        gemm_block<2, 1, COMPUTE>(Xs, Rs, Zb, full, empty, grp, wg, 2 * (wg & 1), 2, nchunk, NSTG,
                                  s, ph, SR, inv_n, lane);
      break;
    case 2:
      gemm_block<2, 1, COMPUTE>(Xs, Rs, Zb, full, empty, grp, wg, 2 * (wg & 1), wg >> 1, nchunk,
                                NSTG, s, ph, SR, inv_n, lane);
      break;
    default:
      gemm_block<1, 1, COMPUTE>(Xs, Rs, Zb, full, empty, grp, wg, wg, 0, nchunk, NSTG, s, ph, SR,
                                inv_n, lane);
      break;
  }
}

__global__ void __launch_bounds__(CD_THREADS, 1) cd_sweep_kernel(const CDParams P) {
  // (pointer arithmetic only from the __shared__ array, so every access compiles to LDS/STS)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int T = P.T;
  const int SR = P.n_pad + RPAD;
  const int NSTG = P.nst / KSPLIT;   // stages per parity-group ring
  double* Rs = (double*)smem_raw;                               // [T][SR]
  double* Zp = Rs + (size_t)T * SR;                             // [2][T][JP]
  double* chg_d = Zp + (size_t)2 * T * JP;                      // [2][J][T]
  unsigned char* chg_row = (unsigned char*)(chg_d + (size_t)2 * J * T);  // [2][J][T]
  size_t off = (size_t)T * SR * 8 + (size_t)2 * T * JP * 8 + (size_t)2 * J * T * 8 +
               (size_t)2 * J * T;
  off = (off + 15) & ~(size_t)15;
  SlotState& S = *(SlotState*)(smem_raw + off);
  off += sizeof(SlotState);
  off = (off + 15) & ~(size_t)15;
  uint64_t* full = (uint64_t*)(smem_raw + off);
  uint64_t* empty = full + MAX_NST;
  off += 2 * MAX_NST * 8;
  off = (off + 127) & ~(size_t)127;
  double* Xs = (double*)(smem_raw + off);                       // [2 rings][NSTG][J][XS]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = P.n, n_pad = P.n_pad, nchunk = P.nchunk, p = P.p, nblk = P.nblk;
  const int nzcap = P.nzcap;
  const double inv_n = 1.0 / (double)n;

  if (tid == 0) {
    // one ring per parity group: every phase of a stage is consumed by the same 4 warps, so a
    // parity wait can never alias a phase two rounds back
    for (int s = 0; s < KSPLIT * NSTG; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NMW / KSPLIT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  for (int c = tid; c < MAX_T; c += blockDim.x) {
    S.col[c] = -1;
    S.retire[c] = 0;
    S.nchg[0][c] = S.nchg[1][c] = 0;
  }
  for (size_t e = tid; e < (size_t)T * SR; e += blockDim.x) Rs[e] = 0.0;
  if (tid == 0) { S.A = 0; S.taken = 0; }
  __syncthreads();

  // ===================================================== producer warp: X tile stream
  if (warp == PRODUCER_WARP) {
    int sg[KSPLIT] = {0, 0};
    uint32_t phg[KSPLIT] = {0u, 0u};
    for (;;) {
      named_bar_sync(BAR_PROD, CD_THREADS);
      int go = *(volatile int*)&S.go;
      if (!go) break;
      if (lane == 0) {
        const double* src = P.Xb;
        for (int b = 0; b < nblk; ++b)
          for (int q = 0; q < nchunk; ++q, src += CHUNK_DOUBLES) {
            const int g = q & 1;
            const int st = g * NSTG + sg[g];
            mbar_wait(&empty[st], phg[g] ^ 1u);
            mbar_arrive_expect_tx(&full[st], CHUNK_BYTES);
            bulk_g2s(Xs + (size_t)st * CHUNK_DOUBLES, src, CHUNK_BYTES, &full[st]);
            if (++sg[g] == NSTG) { sg[g] = 0; phg[g] ^= 1u; }
          }
      }
      __syncwarp();
    }
    return;
  }

  // ===================================================== work warps (MMA 0..7, epilogue 8..9)
  const bool is_mma = warp < NMW;
  const int grp = (warp >> 2) & 1;       // MMA: chunk parity group (consumes chunks q = grp mod 2)
  const int wg = warp & 3;               // MMA: warp within the group (its subtile)
  const bool std_error = (*(volatile const int*)P.err_in) != 0;
  int ring_s = 0;                        // MMA: position in this group's ring
  uint32_t ring_ph = 0;
  const int ncols = P.ncols;
  const int64_t cb = P.col_begin;
  const size_t list_stride = (size_t)2 * nzcap;   // per column: 2 lists
  const double* Xr = Xs + (size_t)grp * NSTG * CHUNK_DOUBLES;
  uint64_t* fr = full + grp * NSTG;
  uint64_t* er = empty + grp * NSTG;

  for (bool first_round = true;; first_round = false) {
    // ---------------------------------------------------------------- sweep boundary
    if (!first_round) {
      // (a) per-slot end-of-sweep logic; work warp w owns slots c = w (mod NWORK)
      for (int c = warp; c < S.A; c += NWORK) {
        const int col = S.col[c];
        // the list built in this sweep becomes the current coefficients
        const int cur = S.cur[c] ^ 1;
        const int cnt = S.cnt_new[c];
        const double maxd = S.maxd[c];
        if (P.joint) {
          // Algorithm 3: one sweep per launch; the host applies the joint stop.  Carry
          // the residual (not recomputed inside the inner loop) and the list.
          const double* r = Rs + (size_t)c * SR;
          double* e = P.Ej + (size_t)col * n_pad;
          for (int i = lane; i < n_pad; i += 32) e[i] = r[i];
          __syncwarp();
          if (lane == 0) {
            P.nz_count[col] = cnt;
            P.nz_cur[col] = cur;
            P.sweeps[col] = S.sweeps[c] + 1;
            atomicMax(P.joint_maxd, (unsigned long long)__double_as_longlong(maxd));
            S.retire[c] = 1;
          }
          continue;
        }
        int inner = S.inner[c] + 1;
        int flags = S.flags[c];
        bool done_inner = (maxd < P.tol) || inner >= P.max_inner;
        int retire = 0;
        double sigma = S.sigma[c];
        int outer = S.outer[c];
        if (done_inner) {
          if (!(maxd < P.tol)) flags |= 2;
          // fresh residual r = x~_c - sum_{b_j != 0, ascending} x~_j b_j (reading g4), in Rs[c]
          double* r = Rs + (size_t)c * SR;
          const int64_t gcol = cb + col;
          for (int i = lane; i < n_pad; i += 32) r[i] = P.Xb[xb_index(i, gcol, nchunk)];
          const int* lr = P.nz_rows + (size_t)col * list_stride + (size_t)cur * nzcap;
          const double* lv = P.nz_vals + (size_t)col * list_stride + (size_t)cur * nzcap;
          const int m_end = min(cnt, nzcap);
          for (int m = 0; m < m_end; ++m) {
            const int j = lr[m];
            const double bj = lv[m];
            for (int i = lane; i < n_pad; i += 32)
              r[i] = fma(-P.Xb[xb_index(i, j, nchunk)], bj, r[i]);
          }
          double ss = 0.0;
          for (int i = lane; i < n; i += 32) ss = fma(r[i], r[i], ss);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
          double sn = sqrt(ss) / P.sqrt_n;
          if (sn < P.sigma_floor) sn = P.sigma_floor;           // reading g5
          ++outer;
          if (fabs(sn - sigma) < P.tol) { flags |= 1; retire = 1; }
          else if (outer >= P.max_outer) retire = 1;                  // reading g16
          sigma = sn;
          inner = 0;
        }
        __syncwarp();
        if (lane == 0) {
          S.cur[c] = cur;
          S.cnt_old[c] = cnt;
          S.cnt_new[c] = 0;
          S.cursor[c] = 0;
          S.sweeps[c] += 1;
          S.inner[c] = inner;
          S.flags[c] = flags;
          S.outer[c] = outer;
          S.sigma[c] = sigma;
          S.lam[c] = sigma * P.lambda0;
          S.maxd[c] = 0.0;
          if (!retire && P.evict_after > 0 && S.sweeps[c] >= P.evict_after) {
            // hand the column to the covariance-update tail solver (tail.cu): a decision that
            // depends only on the column, so results stay independent of scheduling
            const int k = atomicAdd(P.tail_count, 1);
            TailState ts;
            ts.col = col; ts.outer = outer; ts.sweeps = S.sweeps[c]; ts.inner = inner;
            ts.flags = flags; ts.cur = cur; ts.cnt = cnt; ts.lam = 0; ts.sigma = sigma;
            P.tail[k] = ts;
            retire = 1;
          } else if (retire) {
            P.sigma_std[col] = sigma;
            P.iters[col] = outer;
            P.sweeps[col] = S.sweeps[c];
            P.converged[col] = (uint8_t)((flags & 1) && !(flags & 2));
            P.nz_count[col] = cnt;
            P.nz_cur[col] = cur;
          }
          S.retire[c] = retire;
        }
      }
      work_sync();
    }
    // ---------------------------------------------------------------- refill / compaction plan
    if (tid == 0) {
      const int T_ = T;
      for (int c = 0; c < S.A; ++c)
        if (S.retire[c]) { S.col[c] = -1; S.retire[c] = 0; }
      int nfree = 0;
      for (int c = 0; c < T_; ++c) nfree += (S.col[c] < 0);
      int got = 0, start = 0;
      if (nfree > 0 && !std_error) {
        // each CTA first takes its quota (an equal split of the queue, so when every column
        // needs the same number of sweeps all CTAs finish together); past its quota it takes
        // at most a fair share of what is left (work stealing from slower CTAs)
        const int quota = ncols / (int)gridDim.x + ((int)blockIdx.x < ncols % (int)gridDim.x);
        int share;
        if (S.taken < quota) {
          share = quota - S.taken;
        } else {
          const int left = ncols - *(volatile int*)P.queue;
          share = max(1, (left + (int)gridDim.x - 1) / (int)gridDim.x);
        }
        const int want = min(nfree, share);
        start = atomicAdd(P.queue, want);
        got = max(0, min(want, ncols - start));
        S.taken += got;
      }
      int nl = 0;
      for (int c = 0; c < T_ && nl < got; ++c)
        if (S.col[c] < 0) {
          const int col = P.joint ? P.act[start + nl] : start + nl;
          S.col[c] = col;
          S.ld_dst[nl++] = c;
          S.outer[c] = 0; S.sweeps[c] = 0; S.inner[c] = 0; S.flags[c] = 0;
          S.cur[c] = 0; S.cnt_old[c] = 0; S.cnt_new[c] = 0; S.cursor[c] = 0;
          S.sigma[c] = 1.0;                                     // P:608 sigma^(0) = 1
          S.lam[c] = P.lambda0;
          S.maxd[c] = 0.0;
          if (P.joint) {                                        // resume the column (Alg. 3)
            S.sweeps[c] = P.sweeps[col];
            S.cur[c] = P.nz_cur[col];
            S.cnt_old[c] = P.nz_count[col];
            S.sigma[c] = P.sigma_std[col];
            S.lam[c] = S.sigma[c] * P.lambda0;
          }
        }
      S.nloads = nl;
      // compaction: move the highest active slots into the lowest holes (loads took the
      // lowest holes, so a loaded slot never moves)
      int nm = 0;
      int lo = 0, hi = T_ - 1;
      for (;;) {
        while (lo < T_ && S.col[lo] >= 0) ++lo;
        while (hi >= 0 && S.col[hi] < 0) --hi;
        if (lo >= hi || lo >= T_ || hi < 0) break;
        S.mv_dst[nm] = lo; S.mv_src[nm] = hi; ++nm;
        S.col[lo] = S.col[hi]; S.outer[lo] = S.outer[hi]; S.sweeps[lo] = S.sweeps[hi];
        S.inner[lo] = S.inner[hi]; S.flags[lo] = S.flags[hi]; S.cur[lo] = S.cur[hi];
        S.cnt_old[lo] = S.cnt_old[hi]; S.cnt_new[lo] = 0; S.cursor[lo] = 0;
        S.sigma[lo] = S.sigma[hi]; S.lam[lo] = S.lam[hi]; S.maxd[lo] = 0.0;
        S.col[hi] = -1;
      }
      S.nmoves = nm;
      int A = 0;
      for (int c = 0; c < T_; ++c) if (S.col[c] >= 0) A = c + 1;
      S.A = A;
      S.go = A > 0;
      for (int c = 0; c < MAX_T; ++c) S.nchg[0][c] = S.nchg[1][c] = 0;
    }
    work_sync();
    // execute moves (R columns) and loads (r = x~_c, e = x_c - X*0)
    {
      const int nm = S.nmoves, nl = S.nloads;
      for (int m = 0; m < nm; ++m) {
        const double* src = Rs + (size_t)S.mv_src[m] * SR;
        double* dst = Rs + (size_t)S.mv_dst[m] * SR;
        for (int i = tid; i < n_pad; i += WORK_THREADS) dst[i] = src[i];
      }
      for (int l = 0; l < nl; ++l) {
        const int c = S.ld_dst[l];
        const int64_t gcol = cb + S.col[c];
        double* dst = Rs + (size_t)c * SR;
        if (P.joint) {
          const double* e = P.Ej + (size_t)S.col[c] * n_pad;
          for (int i = tid; i < n_pad; i += WORK_THREADS) dst[i] = e[i];
        } else {
          for (int i = tid; i < n_pad; i += WORK_THREADS) dst[i] = P.Xb[xb_index(i, gcol, nchunk)];
        }
      }
    }
    const int A = S.A;
    __threadfence_block();
    work_sync();
    named_bar_arrive(BAR_PROD, CD_THREADS);   // release the producer for this sweep (or exit)
    if (A == 0) break;

    // ---------------------------------------------------------------- one sweep, lag-1 pipeline
    const int NTa = (A + 7) >> 3;          // active n-tiles of 8 columns
    // epilogue warp: lane = column; the column's state lives in registers for the sweep
    const bool c_act = !is_mma && lane < A;
    int gcol = 0, cnt_old = 0, cursor = 0, cnt_new = 0, nx_row = 0x7fffffff;
    double lam = 0.0, maxd = 0.0, nx_val = 0.0;
    const int* lst_old_r = nullptr;
    const double* lst_old_v = nullptr;
    int* lst_new_r = nullptr;
    double* lst_new_v = nullptr;
    if (c_act) {
      const int col = S.col[lane];
      gcol = (int)(cb + col);
      lam = S.lam[lane];
      cnt_old = S.cnt_old[lane];
      const size_t base = (size_t)col * list_stride;
      lst_old_r = P.nz_rows + base + (size_t)S.cur[lane] * nzcap;
      lst_old_v = P.nz_vals + base + (size_t)S.cur[lane] * nzcap;
      lst_new_r = P.nz_rows + base + (size_t)(S.cur[lane] ^ 1) * nzcap;
      lst_new_v = P.nz_vals + base + (size_t)(S.cur[lane] ^ 1) * nzcap;
      if (cnt_old > 0) { nx_row = lst_old_r[0]; nx_val = lst_old_v[0]; }
    }
    for (int t = 0; t <= nblk; ++t) {
      if (is_mma) {
        // ======== MMA warps: Z_t
        if (t < nblk) {
          double* Zb = Zp + (size_t)(t & 1) * T * JP;
          run_gemm<true>(NTa, grp, wg, Xr, Rs, Zb, fr, er, nchunk, NSTG, ring_s, ring_ph, SR,
                         inv_n, lane);
        }
      } else if (c_act) {
        // ======== epilogue warp, lane = column c: finish block b = t-1 row by row
        if (t >= 1) {
          const int b = t - 1;
          const int j0 = b * J;
          const int xb = b & 1, xp = xb ^ 1;   // chg buffers: this block / previous block
          const double* Zc = Zp + (size_t)xb * T * JP + (size_t)lane * JP;
          const double* Gb = P.Gband + (size_t)b * J * (2 * J);   // [r][Gx(32) | Gw(32)]
          const int np = (b >= 1) ? S.nchg[xp][lane] : 0;         // block b-1's changes
          // fast path (almost every visit): b_old = 0 on all 32 rows, no correction from block
          // b-1, and |z| <= lambda on every valid row => nothing changes, no nonzero to list.
          // Soft(z, lam) != 0  <=>  |z| - lam > 0  <=>  |z| > lam for finite doubles.
          // (branch-free: all 32 loads issue back to back, predicates combined bitwise)
          double zv[J];
#pragma unroll
          for (int r = 0; r < J; ++r) zv[r] = Zc[r];
          unsigned hit = 0u;
#pragma unroll
          for (int r = 0; r < J; ++r) hit |= (unsigned)(fabs(zv[r]) > lam) << r;
          // rows that are valid predictors: j < p and j != this column's own index
          unsigned valid = (j0 + J <= p) ? 0xffffffffu : ((1u << (p - j0)) - 1u);
          if (gcol >= j0 && gcol < j0 + J) valid &= ~(1u << (gcol - j0));
          hit &= valid;
          int nch = 0;
          if (hit != 0u || np != 0 || nx_row < j0 + J) {
            // general path: the rows of this block in order (Algorithm 1's cyclic order)
            for (int r = 0; r < J; ++r) {
              const int j = j0 + r;
              double z = Zc[r];
              // R lacked block b-1's updates when Z_b was formed: add G^x_{jj'} d_j'
              for (int m = 0; m < np; ++m)
                z = fma(Gb[r * 2 * J + chg_row[(xp * J + m) * T + lane]],
                        chg_d[(xp * J + m) * T + lane], z);
              // and this block's earlier changes: G^w_{jj'} d_j'
              for (int m = 0; m < nch; ++m)
                z = fma(Gb[r * 2 * J + J + chg_row[(xb * J + m) * T + lane]],
                        chg_d[(xb * J + m) * T + lane], z);
              // previous coefficient b_jc: merge with the column's sorted list of the last sweep
              double bo = 0.0;
              if (nx_row == j) {
                bo = nx_val;
                ++cursor;
                nx_row = 0x7fffffff;
                if (cursor < cnt_old && cursor < nzcap) { nx_row = lst_old_r[cursor]; nx_val = lst_old_v[cursor]; }
              }
              if (j < p && j != gcol) {
                const double bn = soft(z + bo, lam);
                const double d = bo - bn;                        // e += x_j d
                if (d != 0.0) {
                  chg_row[(xb * J + nch) * T + lane] = (unsigned char)r;
                  chg_d[(xb * J + nch) * T + lane] = d;
                  ++nch;
                  maxd = fmax(maxd, fabs(d));
                }
                if (bn != 0.0) {                                 // this sweep's list
                  if (cnt_new < nzcap) { lst_new_r[cnt_new] = j; lst_new_v[cnt_new] = bn; }
                  else atomicExch(&P.flags[FLAG_OVERFLOW], 1);
                  ++cnt_new;
                }
              }
            }
          }
          S.nchg[xb][lane] = nch;
        }
      }
      work_sync();   // ---- end of step t
      // -- residual updates e_c += x_j d for block t-1's changes (Prop. 2); rare
      if (t >= 1) {
        const int xb = (t - 1) & 1;
        const bool any = __any_sync(0xffffffffu, lane < A && S.nchg[xb][lane] > 0);
        if (any) {
          const int j0 = (t - 1) * J;
          for (int c = 0; c < A; ++c) {
            const int nch = S.nchg[xb][c];
            if (nch == 0) continue;
            double* r = Rs + (size_t)c * SR;
            for (int i = tid; i < n_pad; i += WORK_THREADS) {
              double v = r[i];
              for (int m = 0; m < nch; ++m)
                v = fma(P.Xb[xb_index(i, j0 + chg_row[(xb * J + m) * T + c], nchunk)],
                        chg_d[(xb * J + m) * T + c], v);
              r[i] = v;
            }
          }
          work_sync();
        }
      }
    }
    if (c_act) {
      S.maxd[lane] = maxd;
      S.cnt_new[lane] = cnt_new;
    }
    work_sync();
  }
}

cudaError_t launch_cd(const CDParams& P, int num_ctas, cudaStream_t s) {
  const size_t smem = smem_fixed_bytes(P.T, P.n_pad) + (size_t)P.nst * CHUNK_BYTES;
  cudaError_t e = cudaFuncSetAttribute(cd_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  cd_sweep_kernel<<<num_ctas, CD_THREADS, smem, s>>>(P);
  return cudaGetLastError();
}

}  // namespace spmesl
