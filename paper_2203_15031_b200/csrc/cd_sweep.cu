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
// How 32 rows are processed at once ("blocked walk"):
//   1. Z = X_J^T R_T for the 32 rows j0..j0+31 of the block and the T resident residuals R_T
//      (a dense fp64 contraction over n: mma.sync m8n8k4 DMMA, operands in shared memory;
//      X tiles stream HBM/L2 -> smem by cp.async.bulk on an mbarrier ring driven by a
//      producer warp).
//   2. Parallel epilogue: a_jc = Z_jc/n + b_jc and Soft for all 32 x T visits at once.  Until
//      the first row where b_jc changes, these are exactly Algorithm 1's values.
//   3. Only for columns with a change: a one-lane-per-column walk from that first row on,
//      correcting later rows with G_J (x_j^T x_j'/n): a_jc += sum_{j' changed} G_jj' d_j'c.
//   4. R_c += x_j d_jc for the (rare) changed visits.
// Every dot product is reduced in one fixed order (k-split of 4 warps, summed 0..3), so a
// column's result does not depend on its slot, its CTA, the tile occupancy or the GPU count.
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
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void consumer_sync() { named_bar_sync(1, NCW * 32); }

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

constexpr int MAX_NST = 12; // max X chunk pipeline depth (runtime: as many as smem allows)
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
  int first[MAX_T];     // first changed row in the current block (J = none)
  int nchg[MAX_T];
  int retire[MAX_T];
  double sigma[MAX_T];
  double lam[MAX_T];
  double maxd[MAX_T];
  // control
  int A;
  int go;
  int anychg[2];
  int nmoves, nloads;
  int mv_dst[MAX_T], mv_src[MAX_T];
  int ld_dst[MAX_T];
};

// Shared-memory carve-up (bytes), given T slots, padded n and the pipeline depth.
static __host__ __device__ size_t smem_fixed_bytes(int T, int n_pad) {
  size_t b = 0;
  b += (size_t)T * (n_pad + RPAD) * 8;  // Rs   [T][n_pad+RPAD]
  b += (size_t)KSPLIT * T * JP * 8;     // Zp   [KSPLIT][T][JP]
  b += (size_t)T * JP * 8;              // Bt   [T][JP]
  b += (size_t)J * T * 8;               // chg_d  [J][T]
  b += (size_t)J * T;                   // chg_row[J][T]
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
  return (int)std::min<size_t>(MAX_NST, (smem_optin - fixed) / CHUNK_BYTES);
}

size_t cd_smem_bytes(int T, int n_pad) {     // minimum (2 stages)
  return smem_fixed_bytes(T, n_pad) + 2 * (size_t)CHUNK_BYTES;
}

// One row block's contraction Z(32 x 8NTa) = X_J^T R for the chunks q = grp (mod 2) of this
// warp's parity group, for the warp's MT x NT subtile of 8x8 tiles starting at (m0, n0).
// Paired-k fragments: for k-pair kp of a chunk, lane (g, t) loads the 2 consecutive samples
// k = 8kp + 2t, 8kp + 2t + 1 of row g with one 128-bit LDS; the first DMMA takes the even
// sample, the second the odd one (the same k mapping for A and B, so the sum is exact up to
// its fixed association).  Each output's accumulation order depends only on k, never on the
// subtile mapping, so results are independent of NTa and of the column's slot.
template <int MT, int NT>
__device__ __forceinline__ void gemm_block(const double* __restrict__ Xs, const double* __restrict__ Rs,
                                           double* __restrict__ Zp, uint64_t* full, uint64_t* empty,
                                           int grp, int m0, int n0, int nchunk, int NST, int s_base,
                                           uint32_t ph_base, int SR, int T, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  double acc[MT][NT][2];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  int s = s_base + grp;
  uint32_t ph = ph_base;
  if (s >= NST) { s -= NST; ph ^= 1u; }
  const double* rbase = Rs + (size_t)(n0 * 8 + g) * SR + 2 * t4;
  for (int q = grp; q < nchunk; q += 2) {
    mbar_wait(&full[s], ph);
    const double* xs = Xs + (size_t)s * CHUNK_DOUBLES + (size_t)(m0 * 8 + g) * XS + 2 * t4;
    const double* rs = rbase + q * KC;
    const int sw = g & 1;                 // row parity of this lane's A rows (xswz)
#pragma unroll
    for (int kp = 0; kp < KC / 8; ++kp) {
      double2 a[MT], bb[NT];
#pragma unroll
      for (int mi = 0; mi < MT; ++mi) a[mi] = *(const double2*)(xs + mi * 8 * XS + (kp ^ sw) * 8);
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) bb[ni] = *(const double2*)(rs + (size_t)ni * 8 * SR + kp * 8);
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi].x, bb[ni].x);
#pragma unroll
      for (int mi = 0; mi < MT; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi].y, bb[ni].y);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    s += 2;
    if (s >= NST) { s -= NST; ph ^= 1u; }
  }
  // partial sums: Zp[grp][col][row]
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      double* z = Zp + ((size_t)grp * T + (n0 + ni) * 8 + 2 * t4) * JP + (m0 + mi) * 8 + g;
      z[0] = acc[mi][ni][0];
      z[JP] = acc[mi][ni][1];
    }
}

__global__ void __launch_bounds__(CD_THREADS, 1) cd_sweep_kernel(const CDParams P) {
  // (pointer arithmetic only from the __shared__ array, so every access compiles to LDS/STS)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int T = P.T;
  const int SR = P.n_pad + RPAD;
  const int NST = P.nst;
  double* Rs = (double*)smem_raw;                               // [T][SR]
  double* Zp = Rs + (size_t)T * SR;                             // [KSPLIT][T][JP]
  double* Bt = Zp + (size_t)KSPLIT * T * JP;                    // [T][JP]
  double* chg_d = Bt + (size_t)T * JP;                          // [J][T]
  unsigned char* chg_row = (unsigned char*)(chg_d + (size_t)J * T);  // [J][T]
  size_t off = (size_t)T * SR * 8 + (size_t)KSPLIT * T * JP * 8 + (size_t)T * JP * 8 +
               (size_t)J * T * 8 + (size_t)J * T;
  off = (off + 15) & ~(size_t)15;
  SlotState& S = *(SlotState*)(smem_raw + off);
  off += sizeof(SlotState);
  off = (off + 15) & ~(size_t)15;
  uint64_t* full = (uint64_t*)(smem_raw + off);
  uint64_t* empty = full + MAX_NST;
  off += 2 * MAX_NST * 8;
  off = (off + 127) & ~(size_t)127;
  double* Xs = (double*)(smem_raw + off);                       // [NST][J][XS]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = P.n, n_pad = P.n_pad, nchunk = P.nchunk, p = P.p, nblk = P.nblk;
  const int nzcap = P.nzcap;

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW / KSPLIT);   // the 4 warps of the chunk's parity group
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  for (int c = tid; c < MAX_T; c += blockDim.x) {
    S.col[c] = -1;
    S.retire[c] = 0;
  }
  for (size_t e = tid; e < (size_t)T * SR; e += blockDim.x) Rs[e] = 0.0;
  if (tid == 0) { S.A = 0; S.anychg[0] = S.anychg[1] = 0; }
  __syncthreads();

  // ===================================================== producer warp: X tile stream
  if (warp == NCW) {
    int s = 0;
    uint32_t ph = 0;
    for (;;) {
      named_bar_sync(2, CD_THREADS);
      int go = *(volatile int*)&S.go;
      if (!go) break;
      if (lane == 0) {
        const double* src = P.Xb;
        for (int b = 0; b < nblk; ++b)
          for (int q = 0; q < nchunk; ++q, src += CHUNK_DOUBLES) {
            mbar_wait(&empty[s], ph ^ 1u);
            mbar_arrive_expect_tx(&full[s], CHUNK_BYTES);
            bulk_g2s(Xs + (size_t)s * CHUNK_DOUBLES, src, CHUNK_BYTES, &full[s]);
            if (++s == NST) { s = 0; ph ^= 1u; }
          }
      }
      __syncwarp();
    }
    return;
  }

  // ===================================================== consumer warps
  const bool std_error = (*(volatile const int*)P.err_in) != 0;
  // ring position of the first chunk of the current block (identical sequence to the producer)
  int s_base = 0;
  uint32_t ph_base = 0;
  const int ncols = P.ncols;
  const int64_t cb = P.col_begin;
  const size_t list_stride = (size_t)2 * nzcap;   // per column: 2 lists

  for (bool first_round = true;; first_round = false) {
    // ---------------------------------------------------------------- sweep boundary
    if (!first_round) {
      // (a) per-slot end-of-sweep logic; warp w owns slots c = w (mod 8)
      for (int c = warp; c < S.A; c += NCW) {
        const int col = S.col[c];
        // the list built in this sweep becomes the current coefficients
        const int cur = S.cur[c] ^ 1;
        const int cnt = S.cnt_new[c];
        const double maxd = S.maxd[c];
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
          S.retire[c] = retire;
          if (retire) {
            P.sigma_std[col] = sigma;
            P.iters[col] = outer;
            P.sweeps[col] = S.sweeps[c];
            P.converged[col] = (uint8_t)((flags & 1) && !(flags & 2));
            P.nz_count[col] = cnt;
            P.nz_cur[col] = cur;
          }
        }
      }
      consumer_sync();
    }
    // ---------------------------------------------------------------- refill / compaction plan
    if (tid == 0) {
      int T_ = T;
      for (int c = 0; c < S.A; ++c)
        if (S.retire[c]) { S.col[c] = -1; S.retire[c] = 0; }
      int nfree = 0;
      for (int c = 0; c < T_; ++c) nfree += (S.col[c] < 0);
      int got = 0, start = 0;
      if (nfree > 0 && !std_error) {
        // take at most a fair share of what is left, so the last wave stays balanced
        const int left = ncols - *(volatile int*)P.queue;
        const int share = max(1, (left + (int)gridDim.x - 1) / (int)gridDim.x);
        const int want = min(nfree, share);
        start = atomicAdd(P.queue, want);
        got = max(0, min(want, ncols - start));
      }
      int nl = 0;
      for (int c = 0; c < T_ && nl < got; ++c)
        if (S.col[c] < 0) {
          const int col = start + nl;
          S.col[c] = col;
          S.ld_dst[nl++] = c;
          S.outer[c] = 0; S.sweeps[c] = 0; S.inner[c] = 0; S.flags[c] = 0;
          S.cur[c] = 0; S.cnt_old[c] = 0; S.cnt_new[c] = 0; S.cursor[c] = 0;
          S.sigma[c] = 1.0;                                     // P:608 sigma^(0) = 1
          S.lam[c] = P.lambda0;
          S.maxd[c] = 0.0;
        }
      S.nloads = nl;
      // compaction: move the highest active slots into the lowest holes
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
        // a slot loaded this round may move (only if holes remain below it, impossible since
        // loads fill the lowest holes first) — keep the load target map consistent anyway
        for (int l = 0; l < nl; ++l)
          if (S.ld_dst[l] == hi) S.ld_dst[l] = lo;
      }
      S.nmoves = nm;
      int A = 0;
      for (int c = 0; c < T_; ++c) if (S.col[c] >= 0) A = c + 1;
      S.A = A;
      S.go = A > 0;
      S.anychg[0] = S.anychg[1] = 0;
    }
    consumer_sync();
    // execute moves (R columns) and loads (r = x~_c, e = x_c - X*0)
    {
      const int nm = S.nmoves, nl = S.nloads;
      for (int m = 0; m < nm; ++m) {
        const double* src = Rs + (size_t)S.mv_src[m] * SR;
        double* dst = Rs + (size_t)S.mv_dst[m] * SR;
        for (int i = tid; i < n_pad; i += NCW * 32) dst[i] = src[i];
      }
      for (int l = 0; l < nl; ++l) {
        const int c = S.ld_dst[l];
        const int64_t gcol = cb + S.col[c];
        double* dst = Rs + (size_t)c * SR;
        for (int i = tid; i < n_pad; i += NCW * 32) dst[i] = P.Xb[xb_index(i, gcol, nchunk)];
      }
    }
    const int A = S.A;
    __threadfence_block();
    consumer_sync();
    named_bar_arrive(2, CD_THREADS);   // release the producer for this sweep (or exit)
    if (A == 0) break;

    // ---------------------------------------------------------------- one sweep over all rows
    const int NTa = (A + 7) >> 3;          // active n-tiles of 8 columns
    const int grp = warp >> 2;             // chunk parity group: consumes chunks q = grp (mod 2)
    const int wg = warp & 3;               // warp within the group (its 8x8-tile subtile)

    for (int b = 0; b < nblk; ++b) {
      const int j0 = b * J;
      // -- prefetch this block's previous coefficients from each column's sorted list
      int pf_row[4];
      double pf_val[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = warp + NCW * u;
        pf_row[u] = 0x7fffffff;
        pf_val[u] = 0.0;
        if (c < A) {
          const int col = S.col[c];
          const int idx = S.cursor[c] + lane;
          if (idx < S.cnt_old[c] && idx < nzcap) {
            const size_t o = (size_t)col * list_stride + (size_t)S.cur[c] * nzcap + idx;
            pf_row[u] = P.nz_rows[o];
            pf_val[u] = P.nz_vals[o];
          }
        }
      }
      // -- Z = X_J^T R over this group's chunks (DMMA), partial sums to Zp[grp]
      switch (NTa) {
        case 4: gemm_block<2, 2>(Xs, Rs, Zp, full, empty, grp, 2 * (wg & 1), 2 * (wg >> 1), nchunk,
                                 NST, s_base, ph_base, SR, T, lane); break;
        case 3:
          if (wg < 2) gemm_block<2, 2>(Xs, Rs, Zp, full, empty, grp, 2 * (wg & 1), 0, nchunk, NST,
                                       s_base, ph_base, SR, T, lane);
          else gemm_block<2, 1>(Xs, Rs, Zp, full, empty, grp, 2 * (wg & 1), 2, nchunk, NST,
                                s_base, ph_base, SR, T, lane);
          break;
        case 2: gemm_block<2, 1>(Xs, Rs, Zp, full, empty, grp, 2 * (wg & 1), wg >> 1, nchunk, NST,
                                 s_base, ph_base, SR, T, lane); break;
        default: gemm_block<1, 1>(Xs, Rs, Zp, full, empty, grp, wg, 0, nchunk, NST, s_base,
                                  ph_base, SR, T, lane); break;
      }
      s_base += nchunk;
      while (s_base >= NST) { s_base -= NST; ph_base ^= 1u; }
      // -- previous coefficients of this block into Bt (zero, then scatter list entries)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = warp + NCW * u;
        if (c < A) {
          Bt[c * JP + lane] = 0.0;
          __syncwarp();
          const bool in = pf_row[u] < j0 + J;
          const unsigned m = __ballot_sync(0xffffffffu, in);
          if (in) Bt[c * JP + (pf_row[u] - j0)] = pf_val[u];
          if (lane == 0) S.cursor[c] += __popc(m);
        }
      }
      consumer_sync();  // ---- #1: Z partials, Bt ready
      if (tid == 0) S.anychg[(b + 1) & 1] = 0;
      // -- parallel epilogue: warp w owns columns c = w (mod 8), lane = row jl
      {
        const int jl = lane;
        const int j = j0 + jl;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = warp + NCW * u;
          if (c < A) {
            const int gcol = (int)(cb + S.col[c]);
            const double zs = Zp[(size_t)c * JP + jl] + Zp[((size_t)T + c) * JP + jl];
            const double z = zs / (double)n;                   // x_j^T e / n
            Zp[(size_t)c * JP + jl] = z;
            const double bo = Bt[c * JP + jl];
            const bool valid = (j < p) && (j != gcol);
            const double a = z + bo;
            const double bn = soft(a, S.lam[c]);
            const bool chg = valid && (bn != bo);
            const unsigned mask = __ballot_sync(0xffffffffu, chg);
            if (mask == 0u) {
              // no change: the coefficients of this block are final; append nonzeros
              const bool nz = bo != 0.0;
              const unsigned nzm = __ballot_sync(0xffffffffu, nz);
              if (nzm) {
                const int basecnt = S.cnt_new[c];
                if (nz) {
                  const int pos = basecnt + __popc(nzm & ((1u << lane) - 1u));
                  if (pos < nzcap) {
                    const int col = S.col[c];
                    const size_t o = (size_t)col * list_stride + (size_t)(S.cur[c] ^ 1) * nzcap + pos;
                    P.nz_rows[o] = j;
                    P.nz_vals[o] = bo;
                  }
                }
                __syncwarp();
                if (lane == 0) {
                  S.cnt_new[c] = basecnt + __popc(nzm);
                  if (basecnt + __popc(nzm) > nzcap) atomicExch(&P.flags[FLAG_OVERFLOW], 1);
                }
              }
              if (lane == 0) S.first[c] = J;
            } else {
              if (lane == 0) {
                S.first[c] = __ffs(mask) - 1;
                S.anychg[b & 1] = 1;
              }
            }
          }
        }
      }
      consumer_sync();  // ---- #2
      if (S.anychg[b & 1]) {
        // -- sequential walk for columns with a change (one lane per column)
        if (warp == 0 && lane < A && S.first[lane] < J) {
          const int c = lane;
          const int gcol = (int)(cb + S.col[c]);
          const double lam = S.lam[c];
          const double* G = P.Gband + (size_t)b * J * J;
          double md = S.maxd[c];
          int nch = 0;
          for (int jl = S.first[c]; jl < J; ++jl) {
            const int j = j0 + jl;
            if (j >= p) break;
            if (j == gcol) continue;                             // b_cc = 0 (reading g6)
            double corr = 0.0;
            for (int m = 0; m < nch; ++m)
              corr = fma(G[jl * J + chg_row[m * T + c]], chg_d[m * T + c], corr);
            const double bo = Bt[c * JP + jl];
            const double a = (Zp[(size_t)c * JP + jl] + corr) + bo;
            const double bn = soft(a, lam);
            const double d = bo - bn;                            // e += x_j d
            if (d != 0.0) {
              chg_row[nch * T + c] = (unsigned char)jl;
              chg_d[nch * T + c] = d;
              ++nch;
              Bt[c * JP + jl] = bn;
              md = fmax(md, fabs(d));
            }
          }
          S.maxd[c] = md;
          S.nchg[c] = nch;
          // append the block's final nonzeros in row order
          const int col = S.col[c];
          int cnt = S.cnt_new[c];
          const size_t o = (size_t)col * list_stride + (size_t)(S.cur[c] ^ 1) * nzcap;
          for (int jl = 0; jl < J; ++jl) {
            const double v = Bt[c * JP + jl];
            if (v != 0.0) {
              if (cnt < nzcap) { P.nz_rows[o + cnt] = j0 + jl; P.nz_vals[o + cnt] = v; }
              else atomicExch(&P.flags[FLAG_OVERFLOW], 1);
              ++cnt;
            }
          }
          S.cnt_new[c] = cnt;
        } else if (warp == 0 && lane < A) {
          S.nchg[lane] = 0;
        }
        consumer_sync();  // ---- #3
        // -- residual updates e_c += x_j d for the changed visits (Prop. 2)
        for (int c = 0; c < A; ++c) {
          const int nch = S.nchg[c];
          if (nch == 0) continue;
          double* r = Rs + (size_t)c * SR;
          for (int i = tid; i < n_pad; i += NCW * 32) {
            double v = r[i];
            for (int m = 0; m < nch; ++m)
              v = fma(P.Xb[xb_index(i, j0 + chg_row[m * T + c], nchunk)], chg_d[m * T + c], v);
            r[i] = v;
          }
        }
        consumer_sync();  // ---- #4
      }
    }
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
