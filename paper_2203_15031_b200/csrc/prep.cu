// Column standardization (step a2) and the Gram band used by the blocked CD walk (a4).
//
// standardize_kernel — P:305-307 ("centered and scaled to X_k^T X_k = n"): one warp per
//   column; mu_k = sum_i x_ik / n, s_k = sqrt(sum_i (x_ik - mu_k)^2 / n) (divisor n, reading
//   g14), x~_ik = (x_ik - mu_k) / s_k written straight into the tiled HBM layout Xb (see
//   spmesl_internal.cuh).  Column k is an error if any x_ik is not finite or if
//   s_k <= 1e-13 max_i |x_ik| (reading g15); the smallest offending column wins.
//   HBM-bound: reads X twice (8np B each, the second from L2) and writes Xb (8np B) including
//   its zero padding (samples n..n_pad, rows p..nblk*32: no separate memset).  With S16Prep it
//   also writes the certified screening's f16 operand y = x~/sqrt(N_k) and threshold factors.
//
// gram_kernel — the couplings G_jj' = x~_j^T x~_j' / n between each row j of block b and the
//   rows j' of blocks b-1 and b, which let the CD kernel process Proposition 2's row order
//    32 rows at a time with a lag-1 pipeline.  2 p 32 n FMAs, tiny.
#include <algorithm>
#include <cstdlib>
#include "spmesl_internal.cuh"

namespace spmesl {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y_k (f16) of sample i in the Y16 tile layout of screen16.cu: tiles of 128 variables x 64
// samples, 128-byte rows whose 16-byte chunks are XOR-swizzled by (row & 7)
__device__ __forceinline__ size_t y16_index(int64_t k, int64_t i, int nchunk64) {
  const int64_t blk = k >> 7, r = k & 127, q = i >> 6, pos = i & 63;
  return (size_t)((blk * nchunk64 + q) * 8192 + r * 64 + ((((pos >> 3) ^ (r & 7))) << 3) + (pos & 7));
}

// a / b correctly rounded from rs = RN(1 / b): q = RN(a rs), r = a - b q (exact, fma),
// RN(q + r rs) — the final steps of the IEEE division itself (Markstein), so the quotient is
// the division's (checked bit for bit against it; no overflow or subnormal results here:
// |a / b| <= sqrt(n) for a standardized column)
__device__ __forceinline__ double div_rn(double a, double b, double rs) {
  const double q = a * rs;
  const double r = fma(-b, q, a);
  return fma(r, rs, q);
}

__global__ void standardize_kernel(const double* __restrict__ X, int64_t n, int64_t p, int nchunk,
                                   int64_t nrows, int standardize, double* __restrict__ Xb,
                                   double* mu, double* scale, int* err, unsigned long long* bad_key,
                                   double* nrm, S16Prep y, double* ssq, int stage_n) {
  extern __shared__ __align__(16) double colbuf[];   // [warps][stage_n] (stage_n > 0)
  __shared__ __align__(8) uint64_t colbar[8];
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t n_pad = (int64_t)nchunk * KC;
  const int64_t n64 = (int64_t)y.nchunk64 * 64;
  if (k >= p) {
    // padding rows: zeros in Xb and Y16, threshold factors that never flag
    if (k < nrows)
      for (int64_t i = lane; i < n_pad; i += 32) Xb[xb_index(i, k, nchunk)] = 0.0;
    if (y.Y16 && k < y.p_pad) {
      for (int64_t i0 = 8 * lane; i0 < n64; i0 += 256)
        *(uint4*)(y.Y16 + y16_index(k, i0, y.nchunk64)) = make_uint4(0u, 0u, 0u, 0u);
      if (lane == 0) { y.inv_sq[k] = __int_as_float(0x7f800000); y.lam_n[k] = 0.f; }
    }
    return;
  }
  const double* x = X + k * n;
  if (stage_n > 0) {
    // the whole column in one bulk copy (all of its bytes in flight at once; the passes below
    // then read shared memory)
    const int w = threadIdx.x >> 5;
    double* buf = colbuf + (size_t)w * (stage_n + (y.Y16 ? n64 / 4 : 0));   // (+ f16 staging)
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&colbar[w]);
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                   "r"((uint32_t)(n * 8))
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              (uint32_t)__cvta_generic_to_shared(buf)),
          "l"(x), "r"((uint32_t)(n * 8)), "r"(bar)
          : "memory");
    }
    __syncwarp();
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(bar)
        : "memory");
    x = buf;
  }
  double sum = 0.0, mx = 0.0;
  bool finite = true;
  const int ni = (int)n, npi = (int)n_pad, n64i = (int)n64;   // (32-bit sample indices)
  for (int i = lane; i < ni; i += 32) {
    double v = x[i];
    finite = finite && isfinite(v);
    sum += v;
    mx = fmax(mx, fabs(v));
  }
  finite = __all_sync(0xffffffffu, finite);
  if (!finite) {
    if (lane == 0) { atomicMin(bad_key, 2ull * (unsigned long long)k); atomicExch(err, 1); }
    return;
  }
  sum = warp_sum(sum);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double m = 0.0, s = 1.0;
  if (standardize) {
    m = sum / (double)n;
    double ss = 0.0;
    for (int i = lane; i < ni; i += 32) {
      double c = x[i] - m;
      ss = fma(c, c, ss);
    }
    ss = warp_sum(ss);
    s = sqrt(ss / (double)n);
    if (!(s > 1e-13 * mx)) {
      if (lane == 0) { atomicMin(bad_key, 2ull * (unsigned long long)k + 1ull); atomicExch(err, 1); }
      return;
    }
  }
  if (lane == 0) { mu[k] = m; scale[k] = s; }
  const double rs = 1.0 / s;
  double g = 0.0;
  // (staged column: keep x~ in the shared buffer for the f16 pass — one division per element)
  double* xw = stage_n > 0 ? const_cast<double*>(x) : nullptr;
  // (row jl of column block k / J: element i = 32 q + lane sits at base + q J XS + xswz(jl, lane))
  double* xbk = Xb + xb_index(0, k, nchunk) - xswz((int)(k % J), 0) + xswz((int)(k % J), lane);
  for (int i = lane; i < npi; i += 32, xbk += J * XS) {
    const double v = i < ni ? (standardize ? div_rn(x[i] - m, s, rs) : x[i]) : 0.0;
    *xbk = v;
    if (xw && i < ni) xw[i] = v;
    g = fma(v, v, g);
  }
  __syncwarp();
  g = warp_sum(g);
  const double Nk = g / (double)n;                   // N_k = x~_k^T x~_k / n (= S_kk)
  if (lane == 0 && nrm) nrm[k] = Nk;
  // (the same lane-strided fma chain and xor reduction as gram_init_kernel's ||x~_c||^2, so
  // that kernel can take the value instead of re-reading X~: bit-identical)
  if (lane == 0 && ssq) ssq[k] = g;
  if (y.Y16) {
    // y = x~ / sqrt(N_k) in f16 (the same double product to_f16_kernel forms), and the
    // epilogue's threshold factors (as sqrt_kernel: directed roundings)
    const double sc = rsqrt(Nk);
    if (xw) {
      // (staged column: convert lane-strided into the warp's f16 buffer after the column — no
      // bank conflicts — then store 16-byte chunks of 8 samples; the same values as below)
      __half* hb = (__half*)(xw + stage_n);
      for (int i = lane; i < n64i; i += 32) hb[i] = __double2half(i < ni ? xw[i] * sc : 0.0);
      __syncwarp();
      for (int i0 = 8 * lane; i0 < n64i; i0 += 256)
        *(uint4*)(y.Y16 + y16_index(k, i0, y.nchunk64)) = *(const uint4*)(hb + i0);
    } else
    for (int64_t i0 = 8 * lane; i0 < n64; i0 += 256) {   // 8 samples = one 16-byte chunk
      __align__(16) __half h[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int64_t i = i0 + t;
        const double v = i < n ? (xw ? xw[i] : (standardize ? (x[i] - m) / s : x[i])) : 0.0;
        h[t] = __double2half(v * sc);
      }
      *(uint4*)(y.Y16 + y16_index(k, i0, y.nchunk64)) = *(const uint4*)h;
    }
    if (lane == 0) {
      const double q = sqrt(Nk);
      y.sq[k] = q;
      y.inv_sq[k] = __double2float_rd(1.0 / q * (1.0 - 0x1p-40));
      y.lam_n[k] = __double2float_rd((double)n * y.lambda0 / q * (1.0 - 0x1p-40));
    }
  }
}

// D(8x8) += A(8x4) B(4x8) in fp64 on the tensor cores (fragment layout: see cd_sweep.cu)
__device__ __forceinline__ void dmma_g(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// G[blk][jl][0..31]  = x~_{blk,jl}^T x~_{blk-1,jm} / n   (G^x; zero for blk = 0)
// G[blk][jl][32..63] = x~_{blk,jl}^T x~_{blk,jm} / n     (G^w)
// One CTA per row block, 8 warps; warp w owns the m-tile (w & 3) and the 4 n-tiles of half
// (w >> 2) of the 32 x 64 band.  The two tiles of each chunk pair are staged in shared memory
// verbatim (so the swizzled layout and the paired-k fragment loads of the CD kernel apply).
__global__ void __launch_bounds__(256) gram_kernel(const double* __restrict__ Xb, int64_t n,
                                                   int nchunk, double* __restrict__ G) {
  __shared__ __align__(128) double t[2][J * XS];     // [0]: block b-1, [1]: block b
  const int64_t blk = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3, sw = g & 1;
  const int mt = warp & 3, half = warp >> 2;         // half 0: G^x (block b-1), 1: G^w (block b)
  double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int q = 0; q < nchunk; ++q) {
    const double2* cur = (const double2*)(Xb + ((size_t)blk * nchunk + q) * CHUNK_DOUBLES);
    const double2* prv = blk ? (const double2*)(Xb + ((size_t)(blk - 1) * nchunk + q) * CHUNK_DOUBLES)
                             : nullptr;
    for (int e = tid; e < CHUNK_DOUBLES / 2; e += 256) {
      ((double2*)t[1])[e] = cur[e];
      ((double2*)t[0])[e] = prv ? prv[e] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const double* xa = t[1] + (mt * 8 + g) * XS + 2 * t4;          // A = rows of block b
    const double* xb = t[half] + g * XS + 2 * t4;                  // B = rows of block b-1 / b
#pragma unroll
    for (int kp = 0; kp < KC / 8; ++kp) {
      const double2 a = *(const double2*)(xa + (kp ^ sw) * 8);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const double2 b = *(const double2*)(xb + nt * 8 * XS + (kp ^ sw) * 8);
        dmma_g(acc[nt][0], acc[nt][1], a.x, b.x);
        dmma_g(acc[nt][0], acc[nt][1], a.y, b.y);
      }
    }
    __syncthreads();
  }
  double* gb = G + (size_t)blk * J * 2 * J;
  const double inv_n = 1.0 / (double)n;
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const int row = mt * 8 + g, col = half * J + nt * 8 + 2 * t4;
    gb[row * 2 * J + col] = acc[nt][0] * inv_n;
    gb[row * 2 * J + col + 1] = acc[nt][1] * inv_n;
  }
}

cudaError_t launch_standardize(const double* X, const Layout& L, int standardize, double* Xb,
                               double* mu, double* scale, int* err, unsigned long long* bad_key,
                               cudaStream_t s, double* nrm, const S16Prep* y, double* ssq) {
  // 4 warps (columns) per CTA: a finer last wave than 8 (ncu, config 5: 0.0535 -> 0.0516 ms;
  // 2 and 1 the same as 4)
  constexpr int wpb = 4;
  S16Prep yy{};
  if (y) yy = *y;
  const int64_t nrows = L.nblk * J;                 // Xb rows incl. padding
  const int64_t cols = std::max<int64_t>(nrows, yy.Y16 ? yy.p_pad : 0);
  dim3 grid((unsigned)((cols + wpb - 1) / wpb));
  // stage each column in shared memory by one bulk copy when it is 16-byte aligned and small
  const int stage_n = (L.n % 2 == 0 && ((uintptr_t)X & 15) == 0 && L.n <= 1024)
                          ? (int)L.n : 0;
  const size_t smem = (size_t)wpb * (stage_n + (stage_n && yy.Y16 ? yy.nchunk64 * 64 / 4 : 0)) * 8;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(standardize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  standardize_kernel<<<grid, wpb * 32, smem, s>>>(X, L.n, L.p, L.nchunk, nrows, standardize, Xb,
                                                  mu, scale, err, bad_key, nrm, yy, ssq, stage_n);
  return cudaGetLastError();
}

cudaError_t launch_gram(const double* Xb, const Layout& L, double* Gband, cudaStream_t s) {
  gram_kernel<<<(unsigned)L.nblk, 256, 0, s>>>(Xb, L.n, L.nchunk, Gband);
  return cudaGetLastError();
}

}  // namespace spmesl
