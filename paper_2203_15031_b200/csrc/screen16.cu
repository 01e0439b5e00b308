// Certified low-precision screening for the Gram solver.
//
// The first sweep of column c changes some b_jc iff |S_jc| > lambda0 for some j != c
// (sigma^(0) = 1), S = X~^T X~ / n.  Deciding that needs S only to the extent of a
// comparison, so it is done on the f16 tensor cores (mma.sync m16n8k16, f32 accumulate; ~15x
// the FP64 DMMA rate on B200) with a rigorous error bound, and only the columns that cannot be
// certified hit-free get their exact FP64 Gram column (DMMA, gram_pass in tail.cu), from which
// the exact decision is taken.  No low-precision value ever enters the iterates.
//
// Bound.  y_k = x~_k / sqrt(N_k) with N_k = x~_k^T x~_k / n, so y_k^T y_k = n and
// R = Y^T Y / n is the correlation-scaled S: S_jc = R_jc sqrt(N_j N_c), |R_jc| <= 1.
// y_hat = fp16(y) (|y| <= sqrt(n) < 65504): |y_hat - y| <= u |y| + 2^-25 (u = 2^-11; the
// absolute term covers subnormals).  Products of two f16 values are exact in f32; allow every
// f32 accumulation step a relative error 2^-23 (round or truncate).  With sum_i |y_ij y_ic| <= n
// (Cauchy-Schwarz):
//   |R_hat_jc - R_jc| <= 2.1 u + n_pad 2^-22 + 2^-23 + 2^-20 =: eps      (n_pad <= 2^16)
// The pair is certified hit-free when (|R_hat_jc| + eps)(1 + 2^-40) sqrt(N_j N_c) <= lambda0.
//
// Layout of Y16: tiles of 128 variables x 64 samples, one contiguous 16 KB block per tile
// ([nblk128][nchunk64][128][64] halves), each 128-byte row's 16-byte chunks XOR-swizzled by
// (row & 7) so the ldmatrix row fetches hit distinct bank groups.
#include <cuda_fp16.h>
#include "spmesl_internal.cuh"

namespace spmesl {

namespace {

constexpr int S16_TB = 128;                 // variables per tile side
constexpr int S16_KC = 64;                  // samples per chunk
constexpr int S16_TILE_HALVES = S16_TB * S16_KC;     // 8192 halves = 16 KB
constexpr int S16_MMA_WARPS = 8;
constexpr int S16_THREADS = (S16_MMA_WARPS + 1) * 32;
#ifndef SPMESL_S16_NST
#define SPMESL_S16_NST 4
#endif
constexpr int S16_NST = SPMESL_S16_NST;     // ring stages (2 tiles = 32 KB each)
constexpr int S16_ZPIECE = 2048;            // doubles per Theta zero-fill bulk store

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait_s(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(su32(bar)), "r"(parity) : "memory");
}

// Xb (FP64 tiles) -> Y16 (normalized f16 tiles).  One CTA per (128-block, 64-chunk) tile.
__global__ void to_f16_kernel(const double* __restrict__ Xb, const double* __restrict__ nrm,
                              int p, int nchunk32, int nchunk64, __half* __restrict__ Y16) {
  const int blk = blockIdx.x, q = blockIdx.y;
  __half* tile = Y16 + ((size_t)blk * nchunk64 + q) * S16_TILE_HALVES;
  for (int e = threadIdx.x; e < S16_TB * (S16_KC / 8); e += blockDim.x) {
    const int r = e >> 3, ch = e & 7;               // row (variable), 16-byte chunk
    const int j = blk * S16_TB + r;
    const int k0 = q * S16_KC + ch * 8;
    __align__(16) __half v[8];
    const double sc = (j < p) ? rsqrt(nrm[j]) : 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = k0 + t;
      double x = 0.0;
      if (j < p && i < nchunk32 * KC) x = Xb[xb_index(i, j, nchunk32)] * sc;
      v[t] = __double2half(x);
    }
    *(uint4*)(tile + r * S16_KC + ((ch ^ (r & 7)) << 3)) = *(const uint4*)v;
  }
}

// upper-triangle tile t -> (I, J), row-major by I
__device__ __forceinline__ void tri_tile16(int t, int nT, int& I, int& Jt) {
  int i = 0, rowlen = nT;
  while (t >= rowlen) { t -= rowlen; ++i; --rowlen; }
  I = i;
  Jt = i + t;
}

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                        const void* addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(su32(addr)));
}

__device__ __forceinline__ void hmma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(S16_THREADS, 1) screen16_kernel(const Screen16Params P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* full = (uint64_t*)smem_raw;
  uint64_t* empty = full + S16_NST;
  __half* ring = (__half*)(smem_raw + 128);                 // [NST][2 tiles]
  double* zbuf = (double*)(ring + (size_t)S16_NST * 2 * S16_TILE_HALVES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nT = P.ntb;                                     // 128-variable blocks
  const int nchunk = P.nchunk64;
  if (P.zero_ptr)
    for (int e = tid; e < S16_ZPIECE; e += blockDim.x) zbuf[e] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < S16_NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&empty[s])),
                   "r"(S16_MMA_WARPS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == S16_MMA_WARPS) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const size_t npieces = P.zero_ptr ? (P.zero_count + S16_ZPIECE - 1) / S16_ZPIECE : 0;
      size_t zp = blockIdx.x;
      for (int t = P.tile_begin + blockIdx.x; t < P.tile_end; t += gridDim.x) {
        int I, Jt;
        tri_tile16(t, nT, I, Jt);
        for (int q = 0; q < nchunk; ++q) {
          mbar_wait_s(&empty[s], ph ^ 1u);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&full[s])),
                       "r"(2u * S16_TILE_HALVES * 2u)
                       : "memory");
          const __half* srcA = P.Y16 + ((size_t)I * nchunk + q) * S16_TILE_HALVES;
          const __half* srcB = P.Y16 + ((size_t)Jt * nchunk + q) * S16_TILE_HALVES;
          __half* dst = ring + (size_t)s * 2 * S16_TILE_HALVES;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  su32(dst)),
              "l"(srcA), "r"((uint32_t)S16_TILE_HALVES * 2u), "r"(su32(&full[s]))
              : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  su32(dst + S16_TILE_HALVES)),
              "l"(srcB), "r"((uint32_t)S16_TILE_HALVES * 2u), "r"(su32(&full[s]))
              : "memory");
          if (zp < npieces) {   // Theta's zero fill rides along (16 KB per chunk issued)
            const size_t off = zp * S16_ZPIECE;
            const size_t cnt = min((size_t)S16_ZPIECE, P.zero_count - off);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                             P.zero_ptr + off),
                         "r"(su32(zbuf)), "r"((uint32_t)(cnt * 8))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            zp += gridDim.x;
          }
          if (++s == S16_NST) { s = 0; ph ^= 1u; }
        }
      }
      while (zp < npieces) {
        const size_t off = zp * S16_ZPIECE;
        const size_t cnt = min((size_t)S16_ZPIECE, P.zero_count - off);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(P.zero_ptr + off),
                     "r"(su32(zbuf)), "r"((uint32_t)(cnt * 8))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        zp += gridDim.x;
      }
      asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
    return;
  }

  // -------------------------------------------------------------------- MMA warps: 64 x 32 each
  const int mq = warp & 1, nq = warp >> 1;
  const int g = lane >> 2, t4 = lane & 3;
  const double inv_n = 1.0 / (double)P.n;
  int s = 0;
  uint32_t ph = 0;
  for (int t = P.tile_begin + blockIdx.x; t < P.tile_end; t += gridDim.x) {
    int I, Jt;
    tri_tile16(t, nT, I, Jt);
    float acc[4][4][4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = acc[mi][ni][2] = acc[mi][ni][3] = 0.f;
    for (int q = 0; q < nchunk; ++q) {
      mbar_wait_s(&full[s], ph);
      const __half* tA = ring + (size_t)s * 2 * S16_TILE_HALVES;
      const __half* tB = tA + S16_TILE_HALVES;
      // fragments of k-step kk + 1 are loaded while the MMAs of k-step kk issue
      uint32_t a[2][4][4], b[2][4][2];
      auto load_frags = [&](int kk, int buf) {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {   // A: rows mq*64 + mi*16 + (lane & 15), chunk 2kk + lane/16
          const int r = mq * 64 + mi * 16 + (lane & 15);
          const int ch = 2 * kk + (lane >> 4);
          ldsm_x4(a[buf][mi][0], a[buf][mi][1], a[buf][mi][2], a[buf][mi][3],
                  tA + r * S16_KC + ((ch ^ (r & 7)) << 3));
        }
#pragma unroll
        for (int np = 0; np < 2; ++np) {   // B: (cols 0-7, k lo/hi), (cols 8-15, k lo/hi)
          const int r = nq * 32 + np * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int ch = 2 * kk + ((lane >> 3) & 1);
          ldsm_x4(b[buf][2 * np][0], b[buf][2 * np][1], b[buf][2 * np + 1][0], b[buf][2 * np + 1][1],
                  tB + r * S16_KC + ((ch ^ (r & 7)) << 3));
        }
      };
      load_frags(0, 0);
#pragma unroll
      for (int kk = 0; kk < S16_KC / 16; ++kk) {
        if (kk + 1 < S16_KC / 16) load_frags(kk + 1, (kk + 1) & 1);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) hmma(acc[mi][ni], a[kk & 1][mi], b[kk & 1][ni][0], b[kk & 1][ni][1]);
      }
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&empty[s])) : "memory");
      if (++s == S16_NST) { s = 0; ph ^= 1u; }
    }
    // epilogue: certify or flag (both orientations of an off-diagonal tile).  The pair is
    // certified when |acc| <= n (lambda0 / (sq_j sq_c) - eps); that threshold is evaluated in
    // f32 with every rounding directed downwards (a smaller threshold only adds candidates).
    const bool diag_tile = (I == Jt);
    float cB[4][2];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = Jt * S16_TB + nq * 32 + ni * 8 + 2 * t4 + e;
        cB[ni][e] = c < P.p ? P.inv_sq[c] : 0.f;
      }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = I * S16_TB + mq * 64 + mi * 16 + g + 8 * h;
        if (j >= P.p) continue;
        const float rA = P.lam_sq[j];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = Jt * S16_TB + nq * 32 + ni * 8 + 2 * t4 + e;
            const float thr = __fmul_rd(__fsub_rd(__fmul_rd(rA, cB[ni][e]), P.eps_f), P.n_f);
            if (fabsf(acc[mi][ni][2 * h + e]) > thr && c < P.p && c != j) {
              P.cand[c] = 1;
              if (!diag_tile) P.cand[j] = 1;
            }
          }
      }
  }
}

// exact decision for the candidate columns from their FP64 Gram columns (one warp each)
__global__ void exact_hits_kernel(const double* __restrict__ Gtab, int p, const int* __restrict__ U,
                                  int nU, const double* __restrict__ lams, int nlam,
                                  uint8_t* __restrict__ hit) {
  const int lane = threadIdx.x & 31;
  const int w = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  if (w >= nU) return;
  const int c = U[w];
  const double* col = Gtab + (size_t)c * p;
  double m = 0.0;
  for (int j = lane; j < p; j += 32)
    if (j != c) m = fmax(m, fabs(col[j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0)
    for (int l = 0; l < nlam; ++l) hit[(size_t)l * p + c] = (uint8_t)(m > lams[l]);
}

__global__ void sqrt_kernel(const double* __restrict__ in, double* __restrict__ out,
                            float* __restrict__ inv_sq, float* __restrict__ lam_sq, double lambda0,
                            int p) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < p) {
    const double q = sqrt(in[k]);
    out[k] = q;
    // directed roundings: the epilogue's f32 threshold may only come out smaller
    inv_sq[k] = __double2float_rd(1.0 / q * (1.0 - 0x1p-40));
    lam_sq[k] = __double2float_rd(lambda0 / q * (1.0 - 0x1p-40));
  }
}

}  // namespace

cudaError_t launch_sqrt(const double* in, double* out, float* inv_sq, float* lam_sq,
                        double lambda0, int p, cudaStream_t s) {
  sqrt_kernel<<<(p + 255) / 256, 256, 0, s>>>(in, out, inv_sq, lam_sq, lambda0, p);
  return cudaGetLastError();
}

size_t screen16_y_halves(int64_t p, int n_pad) {
  const int64_t nb = (p + S16_TB - 1) / S16_TB;
  const int64_t nc = (n_pad + S16_KC - 1) / S16_KC;
  return (size_t)(nb * nc * S16_TILE_HALVES);
}

int screen16_tile_count(int64_t p) {
  const int64_t nT = (p + S16_TB - 1) / S16_TB;
  return (int)(nT * (nT + 1) / 2);
}

double screen16_eps(int n_pad) {
  return 2.1 * 0x1p-11 + (double)n_pad * 0x1p-22 + 0x1p-23 + 0x1p-20;
}

cudaError_t launch_to_f16(const double* Xb, const double* nrm, int p, int n_pad, int nchunk32,
                          __half* Y16, cudaStream_t s) {
  const int nb = (p + S16_TB - 1) / S16_TB;
  const int nc = (n_pad + S16_KC - 1) / S16_KC;
  dim3 grid((unsigned)nb, (unsigned)nc);
  to_f16_kernel<<<grid, 256, 0, s>>>(Xb, nrm, p, nchunk32, nc, Y16);
  return cudaGetLastError();
}

cudaError_t launch_screen16(const Screen16Params& P, int grid, cudaStream_t s) {
  if (P.tile_end <= P.tile_begin) return cudaSuccess;
  const size_t smem = 128 + (size_t)S16_NST * 2 * S16_TILE_HALVES * 2 + (size_t)S16_ZPIECE * 8;
  cudaError_t e = cudaFuncSetAttribute(screen16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  screen16_kernel<<<grid, S16_THREADS, smem, s>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_exact_hits(const double* Gtab, int p, const int* U, int nU, const double* lams,
                              int nlam, uint8_t* hit, cudaStream_t s) {
  if (nU <= 0) return cudaSuccess;
  const int wpb = 8;
  exact_hits_kernel<<<(nU + wpb - 1) / wpb, wpb * 32, 0, s>>>(Gtab, p, U, nU, lams, nlam, hit);
  return cudaGetLastError();
}

}  // namespace spmesl
