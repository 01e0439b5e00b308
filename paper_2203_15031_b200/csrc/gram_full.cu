// Gram solver: S = X~^T X~ / n once, by a symmetric DMMA
// contraction (only the upper triangle of 128 x 128 tiles is computed; each tile is written
// to both G[I, J] and G[J, I]), then covariance-update coordinate descent on it.
//
// Why: for b_c = 0 the residual of column c is x~_c, so the first sweep of every column of
// Algorithm 1 visits z_j = x~_j^T x~_c / n = G_jc — the first sweeps of all p
// columns together ARE the Gram matrix (2 n p^2 flops); computing it once with symmetry costs
// n p (p + 1).  The screening test of that first sweep (b_j = 0 stays 0 unless |G_jc| >
// lambda0, since sigma^(0) = 1) is fused into the tile epilogue: a column with no
// hit finishes its first sweep with no change, and its outer iteration ends right there
// (gram_init_kernel); the others continue in the covariance-update sweep kernel (tail.cu) from
// z = G[:, c].  Iterates are Algorithm 1's up to rounding (the residual identity of Prop. 2).
#include "spmesl_internal.cuh"

namespace spmesl {

namespace {

__device__ __forceinline__ uint32_t smem_u32g(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init_g(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32g(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_g(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32g(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_g(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32g(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_g(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32g(bar);
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
// (X~ is re-read by every tile row/column: keep it in L2 ahead of the streaming G stores)
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32g(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32g(bar)), "l"(pol)
      : "memory");
}
// bulk store shared -> global (async proxy), grouped for a final wait
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32g(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void dmma_g(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int GB = 4;                  // 32-row blocks per tile side (tile = 128 x 128)
#ifndef SPMESL_SYRK_WM
#define SPMESL_SYRK_WM 8
#endif
constexpr int WM = SPMESL_SYRK_WM;     // 8-row m-tiles per warp (warp tile WM*8 x 32)
constexpr int MR = 128 / (8 * WM);     // warp row groups per tile
constexpr int G_MMA_WARPS = MR * 4;
#ifndef SPMESL_SYRK_SMNR
#define SPMESL_SYRK_SMNR 1
#endif
// With SMNR the producer is a whole warpgroup (warps G_MMA_WARPS .. +3, one lane working) that
// gives registers back (setmaxnreg.dec) so the MMA warpgroups can hold their 64 accumulators,
// fragments and addresses without spilling (setmaxnreg.inc): 8 x 232 + 4 x 40 registers.
constexpr int G_PROD_WARPS = SPMESL_SYRK_SMNR ? 4 : 1;
constexpr int G_THREADS = (G_MMA_WARPS + G_PROD_WARPS) * 32;
constexpr int G_STAGE_DOUBLES = 2 * GB * CHUNK_DOUBLES;     // 8 Xb tiles = 64 KB
constexpr int G_MAX_NST = 3;
constexpr int G_ZPIECE = 2048;
#ifndef SPMESL_SYRK_MIG
#define SPMESL_SYRK_MIG 2
#endif
constexpr int MI_G = SPMESL_SYRK_MIG;     // A fragments per DMMA group         // doubles per zero-fill bulk store (16 KB)

// tile index t of the upper triangle (I <= J) of an nT x nT tile grid, row-major by I
__device__ __forceinline__ void tri_tile(int t, int nT, int& I, int& Jt) {
  int i = 0, rowlen = nT;
  while (t >= rowlen) { t -= rowlen; ++i; --rowlen; }
  I = i;
  Jt = i + t;
}

__global__ void __launch_bounds__(G_THREADS, 1) syrk_screen_kernel(const GramParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  if (P.cond_nU && !gram_fallback_taken(*(volatile const int*)P.cond_nU, P.p)) return;
  if (P.zero_last && blockIdx.x == 0 && threadIdx.x == 0) *P.zero_last = 0.0;
  uint64_t* full = (uint64_t*)smem_raw;
  uint64_t* empty = full + G_MAX_NST;
  double* Xs = (double*)(smem_raw + 128);
  double* zbuf = Xs + (size_t)P.nst * G_STAGE_DOUBLES;        // [G_ZPIECE] zeros
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nst = P.nst;
  const int nchunk = P.nchunk, nblk = P.nblk, p = P.p;
  const int nT = (nblk + GB - 1) / GB;
  const int t_begin = P.tile_begin, t_end = P.tile_end;
  if (P.zero_ptr) {
    for (int e = tid; e < G_ZPIECE; e += blockDim.x) zbuf[e] = 0.0;
    // the producer's bulk stores (async proxy) read zbuf: every writer fences its stores first
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init_g(&full[s], 1);
      mbar_init_g(&empty[s], G_MMA_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= G_MMA_WARPS) {
    // ---------------------------------------------------------------- producer
#if SPMESL_SYRK_SMNR
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
#endif
    if (warp == G_MMA_WARPS && lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint64_t pol = l2_evict_last_policy();
      // Theta's zero fill rides along: one 16 KB bulk store of zeros per X chunk issued
      // (pieces b, b + G, ... of the output), the rest after the last tile
      const size_t npieces = P.zero_ptr ? (P.zero_count + G_ZPIECE - 1) / G_ZPIECE : 0;
      size_t zp = blockIdx.x;
      auto zero_piece = [&]() {
        if (zp < npieces) {
          const size_t off = zp * G_ZPIECE;
          const size_t cnt = min((size_t)G_ZPIECE, P.zero_count - off);
          bulk_s2g(P.zero_ptr + off, zbuf, (uint32_t)(cnt * 8));
          zp += gridDim.x;
        }
      };
      for (int t = t_begin + blockIdx.x; t < t_end; t += gridDim.x) {
        int I, Jt;
        tri_tile(t, nT, I, Jt);
        for (int q = 0; q < nchunk; ++q) {
          mbar_wait_g(&empty[s], ph ^ 1u);
          double* st = Xs + (size_t)s * G_STAGE_DOUBLES;
          int cnt = 0;
          for (int u = 0; u < 2 * GB; ++u) {
            const int blk = (u < GB ? I * GB + u : Jt * GB + (u - GB));
            if (blk < nblk) ++cnt;
          }
          mbar_expect_g(&full[s], (uint32_t)cnt * CHUNK_BYTES);
          for (int u = 0; u < 2 * GB; ++u) {
            const int blk = (u < GB ? I * GB + u : Jt * GB + (u - GB));
            if (blk < nblk)
              bulk_g2s_hint(st + (size_t)u * CHUNK_DOUBLES,
                            P.Xb + ((size_t)blk * nchunk + q) * CHUNK_DOUBLES, CHUNK_BYTES, &full[s],
                            pol);
          }
          zero_piece();
          if (++s == nst) { s = 0; ph ^= 1u; }
        }
      }
      while (zp < npieces) zero_piece();
      bulk_wait_all();
    }
    return;
  }

  // ------------------------------------------------------------------ MMA warps
#if SPMESL_SYRK_SMNR
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
#endif
  const int g = lane >> 2, t4 = lane & 3, sw = g & 1;
  const int mq = warp % MR;         // rows [8 WM mq, 8 WM (mq + 1)) of the tile
  const int nq = warp / MR;         // cols [32 nq, 32 nq + 32)
  const double inv_n = 1.0 / (double)P.n;
  const double lam0 = P.lambda0;   // (multi-level fits: the smallest level; see level_flags)
  int s = 0;
  uint32_t ph = 0;
  double* const Gout = P.G;
  for (int t = t_begin + blockIdx.x; t < t_end; t += gridDim.x) {
    int I, Jt;
    tri_tile(t, nT, I, Jt);
    double acc[WM][4][2];
#pragma unroll
    for (int mi = 0; mi < WM; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    for (int q = 0; q < nchunk; ++q) {
      mbar_wait_g(&full[s], ph);
      const double* st = Xs + (size_t)s * G_STAGE_DOUBLES;
      const double* abase = st + (size_t)g * XS + 2 * t4;
      const double* bbase = st + (size_t)(GB + nq) * CHUNK_DOUBLES + (size_t)g * XS + 2 * t4;
#pragma unroll
      for (int kp = 0; kp < KC / 8; ++kp) {
        const int ko = (kp ^ sw) * 8;
        double2 b[4];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = *(const double2*)(bbase + ni * 8 * XS + ko);
#pragma unroll
        for (int m2 = 0; m2 < WM; m2 += MI_G) {
          // (MI_G A fragments live at a time — 9 warps leave 168 registers per thread — and
          // 4 MI_G DMMAs between two updates of the same accumulator)
          double2 a[MI_G];
#pragma unroll
          for (int u = 0; u < MI_G; ++u) {
            const int mt = mq * WM + m2 + u;          // m-tile within the 128-row tile
            a[u] = *(const double2*)(abase + (size_t)(mt >> 2) * CHUNK_DOUBLES + (mt & 3) * 8 * XS + ko);
          }
#pragma unroll
          for (int u = 0; u < MI_G; ++u)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
              dmma_g(acc[m2 + u][ni][0], acc[m2 + u][ni][1], a[u].x, b[ni].x);
#pragma unroll
          for (int u = 0; u < MI_G; ++u)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
              dmma_g(acc[m2 + u][ni][0], acc[m2 + u][ni][1], a[u].y, b[ni].y);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_g(&empty[s]);
      if (++s == nst) { s = 0; ph ^= 1u; }
    }
    // epilogue: G = acc / n to both triangles; screening hits |G_jc| > lambda0 (j != c)
    const bool diag_tile = (I == Jt);
    const int row0 = I * GB * J + 8 * WM * mq;
    const int col0 = Jt * GB * J + 32 * nq;
    // stores are whole 32-byte sectors when p % 4 == 0 (8 lanes x 8 B down a column of G, or
    // 4 lanes x 16 B along a row for the mirror), so L2 never reads back partial sectors
    const bool vec = (p & 3) == 0;
#pragma unroll
    for (int mi = 0; mi < WM; ++mi) {
      const int row = row0 + mi * 8 + g;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int colp = col0 + ni * 8 + 2 * t4;         // this lane's column pair
        const double v0 = acc[mi][ni][0] * inv_n, v1 = acc[mi][ni][1] * inv_n;
        if (Gout) {
          if (vec && row < p && colp + 1 < p) {
            __stcs(Gout + (size_t)colp * p + row, v0);
            __stcs(Gout + (size_t)(colp + 1) * p + row, v1);
            if (!diag_tile) __stcs((double2*)(Gout + (size_t)row * p + colp), make_double2(v0, v1));
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = colp + e;
              if (row < p && col < p) {
                const double v = e ? v1 : v0;
                __stcs(Gout + (size_t)col * p + row, v);
                if (!diag_tile) __stcs(Gout + (size_t)row * p + col, v);
              }
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = colp + e;
          const double v = e ? v1 : v0;
          if (row < p && col < p && row != col && fabs(v) > lam0) {
            P.hit[col] = 1;
            if (!diag_tile) P.hit[row] = 1;
            if (P.hitcnt) {
              atomicAdd(&P.hitcnt[col], 1);
              if (!diag_tile) atomicAdd(&P.hitcnt[row], 1);
            }
          }
        }
      }
    }
  }
}

// Multi-level fits: the screening flags of every level (hit[l][c] = max_{j != c} |S_jc| >
// lambda_l), from the stored S (one warp per column, coalesced); the Gram kernel's epilogue
// screens at the smallest level only.
__global__ void level_flags_kernel(const GramParams P) {
  if (P.cond_nU && !gram_fallback_taken(*(volatile const int*)P.cond_nU, P.p)) return;
  const int lane = threadIdx.x & 31;
  const int c = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  if (c >= P.p) return;
  const double* col = P.G + (size_t)c * P.p;
  double m = 0.0;
  for (int j = lane; j < P.p; j += 32)
    if (j != c) m = fmax(m, fabs(col[j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0)
    for (int l = 0; l < P.nlam; ++l) P.hit[(size_t)l * P.p + c] = (uint8_t)(m > P.lams[l]);
}

// Columns without a screening hit: the first sweep changes nothing (b stays 0, max|db| = 0),
// so outer iteration 1 ends with the fresh residual x~_c (reading g4).  Retire it or,
// if sigma moved by >= tol (possible only without standardization), hand it to the sweep
// kernel like every column with a hit.
// PT (P.ssq given: x~_c^T x~_c is known, nothing to sum): one thread per column instead of a warp
template <bool PT>
__global__ void gram_init_kernel(const GramParams P) {
  const int lane = PT ? 0 : (int)(threadIdx.x & 31);
  const int q = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> (PT ? 0 : 5));
  if (q >= P.ncols * P.nlam) return;
  const int l = q / P.ncols, c = q - l * P.ncols;                // penalty level, column
  const int slot = l * P.ncols + c;                              // output index
  const int64_t gc = P.col_begin + c;
  TailState ts;
  ts.col = c; ts.outer = 0; ts.sweeps = 0; ts.inner = 0; ts.flags = 0; ts.cur = 0; ts.cnt = 0;
  ts.lam = l; ts.sigma = 1.0;
  if (!P.hit[(size_t)l * P.p + gc]) {
    double ss = 0.0;
    if (PT || P.ssq) {
      ss = P.ssq[gc];   // (summed by the standardization in this very order)
    } else {
      for (int i = lane; i < P.n; i += 32) {
        const double r = P.Xb[xb_index(i, gc, P.nchunk)];
        ss = fma(r, r, ss);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    double sn = sqrt(ss) / P.sqrt_n;
    if (sn < P.sigma_floor) sn = P.sigma_floor;                  // reading g5
    if (lane == 0) {
      const bool conv = fabs(sn - 1.0) < P.tol;
      if (conv || P.max_outer <= 1) {
        P.sigma_std[slot] = sn;
        P.iters[slot] = 1;
        P.sweeps[slot] = 1;
        P.converged[slot] = (uint8_t)conv;
        P.nz_count[slot] = 0;
        P.nz_cur[slot] = 0;
        return;
      }
      ts.outer = 1; ts.sweeps = 1; ts.sigma = sn;
    } else {
      return;
    }
  }
  if (lane == 0) {
    const int idx = atomicAdd(P.tail_count, 1);
    P.tail[idx] = ts;
    if (P.bhist) {   // (the sweep kernel's work order: hit-count bucket and rank within it)
      const int b = 1023 - min(P.hitcnt[gc], 1023);
      P.tail_key[idx] = (b << 20) | atomicAdd(&P.bhist[b], 1);
    }
  }
}

}  // namespace

size_t syrk_smem_bytes(int nst) { return 128 + ((size_t)nst * G_STAGE_DOUBLES + G_ZPIECE) * 8; }

int gram_tile_count(int64_t p) {
  const int64_t nT = (((p + J - 1) / J) + GB - 1) / GB;
  return (int)(nT * (nT + 1) / 2);
}

cudaError_t launch_syrk_screen(const GramParams& P, int grid, cudaStream_t s) {
  GramParams Q = P;
  Q.nst = G_MAX_NST;
  if (Q.tile_end <= Q.tile_begin) return cudaSuccess;
  const size_t smem = syrk_smem_bytes(Q.nst);
  cudaError_t e = cudaFuncSetAttribute(syrk_screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  syrk_screen_kernel<<<grid, G_THREADS, smem, s>>>(Q);
  return cudaGetLastError();
}

cudaError_t launch_level_flags(const GramParams& P, cudaStream_t s) {
  const int wpb = 8;
  level_flags_kernel<<<(P.p + wpb - 1) / wpb, wpb * 32, 0, s>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_gram_init(const GramParams& P, cudaStream_t s) {
  if (P.ncols <= 0) return cudaSuccess;
  const int wpb = 8;
  const int w = P.ncols * P.nlam;
  if (P.ssq)
    gram_init_kernel<true><<<(w + 255) / 256, 256, 0, s>>>(P);
  else
    gram_init_kernel<false><<<(w + wpb - 1) / wpb, wpb * 32, 0, s>>>(P);
  return cudaGetLastError();
}

}  // namespace spmesl
