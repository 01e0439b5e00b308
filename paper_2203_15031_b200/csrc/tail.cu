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
// Gram-column prefetch (TailParams::prefetch, when two p-vectors fit in shared memory): the rows
// of the column's current nonzeros are visited in order every sweep and almost every visit
// changes b_j, so the Gram columns of the next two such rows are streamed L2 -> shared memory
// by cp.async.bulk while the sweep proceeds; the z update then reads shared memory instead of
// paying an L2 round trip per change (the straggler columns of hub graphs make hundreds of
// sweeps with ~10 changes each).
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
// 64 rows x up to 128 columns per CTA, a 3-stage cp.async ring of 32-sample chunks (the two
// 8 KB row blocks of Xb + the candidates' rows, re-swizzled by destination row parity), and
// per output the same DMMA chain as gram_tile (chunks ascending, k-pairs 0..3, even then odd
// sample), so every caller sees bit-identical columns.  Optional exact screening decision as
// in gram_tile.
constexpr int GC_NTMAX = 16;            // n-tiles of 8 vectors per vector group (128 columns)
constexpr int GC_STAGES = 3;
#ifndef SPMESL_GC_GROUP
#define SPMESL_GC_GROUP 3
#endif
constexpr int GC_GROUP = SPMESL_GC_GROUP;   // n-tiles per group of independent DMMAs            // 3 x (34 + 32) KB at 17 warps

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}

// nU_dev (optional): the candidate count is read on the device; when 2 nU > p the full Gram
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
  if (nU_dev && fallback && 2 * (int64_t)nU > p) {
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
struct TailShared {
  uint64_t pf_bar[2];    // prefetch buffers' mbarriers
  uint64_t z_bar;        // z <- G[:, c] bulk copy
  double red[TAIL_MAXW];
  int wmin[2][TAIL_MAXW];   // per-warp first hits, double-buffered across rounds
  int oc_var[TAIL_ODC];
  int oc_next;
  int k;
  int k2;
  int pf_row[2];         // variable whose Gram column is (being) loaded into each buffer, or -1
};

// doubles: tiles [2][J*XS], z [p], r [n_pad], old/new list values [2][nzcap];
// ints: old/new list rows [2][nzcap]; then TailShared (8-aligned)
__host__ __device__ size_t tail_smem_bytes(int p, int n_pad, int nzcap) {
  size_t b = ((size_t)2 * J * XS + p + n_pad + 2 * (size_t)nzcap) * 8;
  b += (size_t)2 * nzcap * 4;
  b = (b + 15) & ~(size_t)15;
  b += sizeof(TailShared);
  return (b + 127) & ~(size_t)127;
}

size_t tail_prefetch_bytes(int p) { return (((size_t)2 * p * 8) + 127) & ~(size_t)127; }

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
    if (tid == 0) { atomicExch(&P.gstate[j], 2); atomicAdd(P.ondemand_count, 1); }
  } else if (tid == 0) {
    while (*(volatile int*)&P.gstate[j] != 2) __nanosleep(200);
  }
  __threadfence();
  bsync();
}

template <int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 1) tail_sweep_kernel(const TailParams P) {
  constexpr int TSCAN = SPMESL_TAIL_SCAN_R * NT;   // rows tested per search round
  extern __shared__ __align__(128) unsigned char sm[];
  const int p = P.p, n = P.n, n_pad = P.n_pad, nchunk = P.nchunk, nzcap = P.nzcap;
  double* tx = (double*)sm;                                  // [J*XS]
  double* tvv = tx + J * XS;                                 // [J*XS]
  double* z = tvv + J * XS;                                  // [p]
  double* r = z + p;                                         // [n_pad]
  double* ov = r + n_pad;                                    // [nzcap] old list values
  double* nv = ov + nzcap;                                   // [nzcap] new list values
  int* orow = (int*)(nv + nzcap);                            // [nzcap]
  int* nrow = orow + nzcap;                                  // [nzcap]
  size_t ts_off = ((size_t)2 * J * XS + p + n_pad + 2 * (size_t)nzcap) * 8 + (size_t)2 * nzcap * 4;
  ts_off = (ts_off + 15) & ~(size_t)15;
  TailShared& TS = *(TailShared*)(sm + ts_off);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t list_stride = (size_t)2 * nzcap;
  const int M = P.M_dev ? *(volatile const int*)P.M_dev : P.M;
  // prefetch buffers [2][p] after the base layout (128-byte aligned)
  double* gbuf = (double*)(sm + tail_smem_bytes(p, n_pad, nzcap));
  const bool pf = P.prefetch != 0;
  uint32_t pf_ph[2] = {0u, 0u};
  if (tid < TAIL_ODC) TS.oc_var[tid] = -1;
  if (tid == 0) {
    TS.oc_next = 0;
    TS.pf_row[0] = TS.pf_row[1] = -1;
    if (pf) {
      mbar_init_t(&TS.pf_bar[0], 1);
      mbar_init_t(&TS.pf_bar[1], 1);
    }
    mbar_init_t(&TS.z_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  uint32_t z_ph = 0;
  // (one thread) start loading the Gram column of old-list entry c into buffer c & 1
  auto pf_issue = [&](int c, int cnt) {
    if (c < cnt) {
      const int jv = orow[c];
      if (P.gtab_full || *(volatile int*)&P.gstate[jv] == 2) {
        prefetch_col(gbuf + (size_t)(c & 1) * p, P.Gtab + (size_t)jv * p, (uint32_t)p * 8,
                     &TS.pf_bar[c & 1]);
        TS.pf_row[c & 1] = jv;
        return;
      }
    }
    TS.pf_row[c & 1] = -1;
  };

  for (;;) {
    bsync();
    if (tid == 0) TS.k = atomicAdd(P.next, 1);
    bsync();
    const int k = TS.k;
    if (k >= M) break;
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
    const bool z_saved = P.joint && (ts.flags & 16);          // joint: z kept between launches
    if (P.z_from_gtab || z_saved) {
      if (!z_saved) ensure_gram_column(P, gc, TS, tx, tvv);
      const double* gz = z_saved ? P.Zj + (size_t)slot * p : P.Gtab + (size_t)gc * p;
      if ((p & 1) == 0) {   // the whole column in one bulk copy (8p bytes, 16-byte multiple)
        if (tid == 0) {
          prefetch_col(z, gz, (uint32_t)p * 8, &TS.z_bar);
          mbar_wait_t(&TS.z_bar, z_ph);
        }
        z_ph ^= 1u;
        bsync();
      } else
      // (16 independent L2 loads in flight per thread: the column is 8p bytes)
      for (int j0 = 0; j0 < p; j0 += 16 * NT) {
        constexpr int UB = 16;
        double gv[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int j = j0 + u * NT + tid;
          gv[u] = j < p ? __ldcs(gz + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int j = j0 + u * NT + tid;
          if (j < p) z[j] = gv[u];
        }
      }
    } else {
      for (int j = tid; j < p; j += NT) z[j] = P.Zz[(size_t)k * p + j];
    }
    {
      const size_t lo = (size_t)col * list_stride + (size_t)cur * nzcap;
      for (int m = tid; m < ocnt; m += NT) { orow[m] = P.nz_rows[lo + m]; ov[m] = P.nz_vals[lo + m]; }
    }
    bsync();
    bool retire = false;
    while (!retire) {
      // ------------------------------------------------ one sweep, rows in cyclic order
      const double lam = sigma * lambda0;
      double maxd = 0.0;
      int pos = 0, cursor = 0, ncnt = 0;
      if (pf) {
        if (tid == 0) { pf_issue(0, ocnt); pf_issue(1, ocnt); }
        bsync();
      }
      for (;;) {
        const int na = cursor < ocnt ? orow[cursor] : p;     // next row with b_j != 0
        // first row in [pos, na) with |z_j| > lambda (j != this column)
        // (rounds of TSCAN rows: thread t tests rows base + t + NT r,
        // r < TSCAN / NT; the first hit is the block-wide minimum of the hit rows;
        // one barrier per round: the per-warp minima alternate between two buffers, and a
        // buffer is rewritten only after the next round's barrier, which every reader of it
        // has passed)
        int j = na;
        int rbuf = 0;
        for (int base = pos; base < na; base += TSCAN, rbuf ^= 1) {
          int my = 0x7fffffff;
#pragma unroll
          for (int r = TSCAN / NT - 1; r >= 0; --r) {
            const int jj = base + tid + r * NT;
            if (jj < na && jj != gc && fabs(z[jj]) > lam) my = jj;
          }
          my = __reduce_min_sync(0xffffffffu, my);
          if (lane == 0) TS.wmin[rbuf][warp] = my;
          bsync();
          int best = 0x7fffffff;
#pragma unroll
          for (int w = 0; w < NT / 32; ++w) best = min(best, TS.wmin[rbuf][w]);
          if (best != 0x7fffffff) { j = best; break; }
        }
        if (j >= p) break;
        double bo = 0.0;
        int pfb = -1;                 // prefetch buffer holding G[:, j], if any
        int pf_next = -1;             // old-list entry to prefetch after this visit
        if (j == na) {
          bo = ov[cursor];
          if (pf) {
            const int b = cursor & 1;
            if (TS.pf_row[b] == j) {   // consume the load (wait even if b_j does not change):
              if (tid == 0) {          // the issuing thread waits, the barrier publishes it
                mbar_wait_t(&TS.pf_bar[b], pf_ph[b]);
                pf_ph[b] ^= 1u;
              }
              bsync();
              pfb = b;
            }
            pf_next = cursor + 2;
          }
          ++cursor;
        }
        const double a = z[j] + bo;
        const double bn = soft_t(a, lam);
        const double d = bo - bn;                             // e += x_j d
        if (bn != 0.0) {
          if (ncnt < nzcap) { if (tid == 0) { nrow[ncnt] = j; nv[ncnt] = bn; } }
          else overflow = true;
          ++ncnt;
        }
        if (d != 0.0 && pfb >= 0) {
          maxd = fmax(maxd, fabs(d));
          const double* gs = gbuf + (size_t)pfb * p;          // G[:, j] in shared memory
          for (int t = tid; t < p; t += NT) z[t] = fma(d, gs[t], z[t]);
        } else if (d != 0.0) {
          maxd = fmax(maxd, fabs(d));
          const double* gcol = P.Gtab + (size_t)j * p;
          ensure_gram_column(P, j, TS, tx, tvv);
          // (up to 16 independent L2 loads in flight per thread: one round trip per 4096 rows)
          constexpr int UB = 16;
          for (int t0 = 0; t0 < p; t0 += UB * NT) {
            double gv[UB];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
              const int t = t0 + u * NT + tid;
              gv[u] = t < p ? __ldcg(gcol + t) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
              const int t = t0 + u * NT + tid;
              if (t < p) z[t] = fma(d, gv[u], z[t]);
            }
          }
        }
        bsync();
        if (pf_next >= 0 && tid == 0) pf_issue(pf_next, ocnt);   // (buffer just released)
        pos = j + 1;
      }
      ++sweeps;
      ++inner;
      // the new list becomes the current one
      for (int m = tid; m < min(ncnt, nzcap); m += NT) { orow[m] = nrow[m]; ov[m] = nv[m]; }
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
      if (maxd < P.tol || inner >= P.max_inner) {
        if (!(maxd < P.tol)) flags |= 2;
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
      }
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

cudaError_t launch_tail_sweeps(const TailParams& P, int grid, cudaStream_t s) {
  size_t smem = tail_smem_bytes(P.p, P.n_pad, P.nzcap);
  if (P.prefetch) smem += tail_prefetch_bytes(P.p);
  if (P.occ > 1) grid *= P.occ;   // several column CTAs per SM (set_prefetch)
  cudaError_t e = cudaFuncSetAttribute(tail_sweep_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  // 512 threads when a single column CTA owns the SM (large p: the search rounds and the z
  // updates split over twice the threads), 256 when two share it
  const bool wide = P.occ == 1;
  if (wide) {
    cudaError_t e2 = cudaFuncSetAttribute(tail_sweep_kernel<512>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e2 != cudaSuccess) return e2;
    tail_sweep_kernel<512><<<grid, 512, smem, s>>>(P);
  } else {
    tail_sweep_kernel<256><<<grid, 256, smem, s>>>(P);
  }
  return cudaGetLastError();
}

}  // namespace spmesl
