#include <algorithm>
// Coefficient export (CSC) and Theta assembly + symmetrization (steps a8-a10).
//
// csc_*      — each fitted column's final coefficient list (rows ascending, nonzeros only)
//              is packed into one CSC array (col_ptr, rows, vals).  This is also the unit
//              exchanged between GPUs (one all-gather of nonzeros instead of p^2 doubles).
// assemble   — Alg. 2: omega_kk = 1/(sigma_k sigma_k), omega_jk = -b_jk omega_kk,
//              Proposition 1 rescale omega_jk / (s_j s_k), and the
//              minimum-magnitude symmetrization of Eq. (symm) (Alg. 2 P:709-719:
//              for r < c keep Theta1[r,c] unless |Theta1[r,c]| > |Theta1[c,r]|).  Theta is
//              zero-filled first (a cudaMemsetAsync, the only dense pass: 8 p^2 bytes
//              written); then one thread per nonzero b_jk looks up its partner b_kj by binary
//              search in column j and writes the chosen value into column k.  An entry whose
//              partner is zero symmetrizes to zero (already there), so only mutual pairs and
//              the diagonal are written.
#include "spmesl_internal.cuh"

namespace spmesl {

// Exclusive scan of counts -> col_ptr[0..ncols], single CTA: thread t sums its contiguous
// segment of ceil(ncols / 1024) counts, one block-wide scan of the 1024 partial sums, then each
// thread writes its segment (one barrier round instead of one per 1024 columns).
__global__ void __launch_bounds__(1024) csc_scan_kernel(const int* __restrict__ cnt_g, int ncols,
                                                        int64_t* __restrict__ col_ptr,
                                                        int64_t* total, int staged) {
  __shared__ int64_t warp_tot[32];
  extern __shared__ int cnt_s[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // counts staged in shared memory by coalesced loads when they fit (the segments below are
  // strided across threads)
  const int* cnt = cnt_g;
  if (staged) {
    for (int i0 = tid; i0 < ncols; i0 += 8 * 1024) {   // 8 loads in flight per thread
      int v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (i0 + u * 1024 < ncols) ? __ldg(cnt_g + i0 + u * 1024) : 0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + u * 1024 < ncols) cnt_s[i0 + u * 1024] = v[u];
    }
    __syncthreads();
    cnt = cnt_s;
  }
  const int seg = (ncols + 1023) / 1024;
  const int lo = min(ncols, tid * seg), hi = min(ncols, lo + seg);
  int64_t v = 0;
  for (int i = lo; i < hi; ++i) v += cnt[i];
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  int64_t run = (w ? warp_tot[w - 1] : 0) + x - v;   // exclusive prefix of this segment
  for (int i = lo; i < hi; ++i) {
    col_ptr[i] = run;
    run += cnt[i];
  }
  if (tid == 1023) {
    col_ptr[ncols] = warp_tot[31];
    *total = warp_tot[31];
  }
}

__global__ void csc_copy_kernel(const int* __restrict__ cnt, const int* __restrict__ cur,
                                const int* __restrict__ nz_rows, const double* __restrict__ nz_vals,
                                int ncols, int nzcap, const int64_t* __restrict__ col_ptr,
                                int32_t* __restrict__ rows, double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= ncols) return;
  const int m = min(cnt[c], nzcap);
  const size_t src = (size_t)c * 2 * nzcap + (size_t)cur[c] * nzcap;
  const int64_t dst = col_ptr[c];
  for (int e = lane; e < m; e += 32) {
    rows[dst + e] = nz_rows[src + e];
    vals[dst + e] = nz_vals[src + e];
  }
}

__global__ void csc_counts_kernel(const int* __restrict__ cnt, int ncols, int32_t* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ncols) out[c] = cnt[c];
}

__device__ __forceinline__ double theta1(double b, double sigma_k, double s_j, double s_k,
                                         bool rescale) {
  const double wkk = 1.0 / (sigma_k * sigma_k);     // Alg. 2: omega_kk = sigma_k^-2
  double w = -b * wkk;                              // omega_jk = -beta_jk omega_kk
  if (rescale) w = w / (s_j * s_k);                 // Prop. 1
  return w;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Binary search for row r in the sorted rows[lo, hi); returns the value or 0.
__device__ __forceinline__ double csc_lookup(const int32_t* __restrict__ rows,
                                             const double* __restrict__ vals, int64_t lo,
                                             int64_t hi, int32_t r) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int32_t v = rows[mid];
    if (v == r) return vals[mid];
    if (v < r) lo = mid + 1;
    else hi = mid;
  }
  return 0.0;
}

__global__ void assemble_entries_kernel(int64_t p, int64_t col_begin, int64_t col_end,
                                        const int64_t* __restrict__ col_ptr,
                                        const int32_t* __restrict__ rows,
                                        const double* __restrict__ vals,
                                        const double* __restrict__ sigma_std,
                                        const double* __restrict__ scale, int symmetrize,
                                        int rescale, double* __restrict__ Theta) {
  const int64_t e0 = col_ptr[col_begin], e1 = col_ptr[col_end];
  for (int64_t e = e0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * blockDim.x) {
    // column k of entry e: binary search in col_ptr[col_begin..col_end]
    int64_t lo = col_begin, hi = col_end;   // find k with col_ptr[k] <= e < col_ptr[k+1]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (col_ptr[mid] <= e) lo = mid;
      else hi = mid;
    }
    const int64_t k = lo;
    const int32_t j = rows[e];
    // (scale is NULL when the fit did not standardize: no rescaling then)
    const double sj = rescale ? scale[j] : 1.0, sk = rescale ? scale[k] : 1.0;
    const double t_jk = theta1(vals[e], sigma_std[k], sj, sk, rescale != 0);
    double out = t_jk;
    if (symmetrize) {
      const double b_kj = csc_lookup(rows, vals, col_ptr[j], col_ptr[j + 1], (int32_t)k);
      if (b_kj == 0.0) continue;            // partner zero -> symmetrized value is zero
      const double t_kj = theta1(b_kj, sigma_std[j], sk, sj, rescale != 0);
      // pair (r, c), r < c: keep Theta1[r,c] unless |Theta1[r,c]| > |Theta1[c,r]|
      const double u = (j < k) ? t_jk : t_kj;   // Theta1[min, max]
      const double l = (j < k) ? t_kj : t_jk;   // Theta1[max, min]
      out = (fabs(u) > fabs(l)) ? l : u;
    }
    Theta[(size_t)(k - col_begin) * (size_t)p + (size_t)j] = out;
  }
}

// Device-path assembly straight from the per-column coefficient lists (rows ascending; no CSC
// packing): each warp owns 32 consecutive columns.  Lane l writes the diagonal and sigma of
// column 32 w + l (coalesced) and, when `cs` is given, adds that column's
// sweeps / outer iterations / converged flag to the fit statistics (what column_stats_kernel
// does otherwise, fused here: the last kernel of the fit also stamps its end); then the warp
// walks the columns of its 32 that have entries (most have none) and writes their off-diagonal
// entries together (a8 + a10: the partner b_kj is found by binary search in column j's list,
// exactly as in the CSC variant).  Each column's entry count is added to *nnz_total.
// Bit-identical to csc_build + assemble_entries + assemble_diag.
__global__ void assemble_lists_kernel(int64_t p, const int* __restrict__ cnt,
                                      const int* __restrict__ cur,
                                      const int* __restrict__ nz_rows,
                                      const double* __restrict__ nz_vals, int nzcap,
                                      const double* __restrict__ sigma_std,
                                      const double* __restrict__ scale, int symmetrize,
                                      int rescale, double* __restrict__ Theta,
                                      double* __restrict__ sigma_out,
                                      unsigned long long* __restrict__ nnz_total, ColStats cs) {
  const int lane = threadIdx.x & 31;
  const int64_t k0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
  if (k0 >= p) return;
  const int64_t kl = k0 + lane;
  int mine = 0;
  unsigned long long tsw = 0;
  int msw = 0, mo = 0, nu = 0;
  if (kl < p) {
    mine = min(cnt[kl], nzcap);
    const double sk = rescale ? scale[kl] : 1.0;
    const double sg = sigma_std[kl];
    double w = 1.0 / (sg * sg);
    if (rescale) w = w / (sk * sk);
    Theta[(size_t)kl * (size_t)p + (size_t)kl] = w;
    if (sigma_out) sigma_out[kl] = rescale ? sk * sg : sg;
    if (cs.sweeps) {
      const int sw = cs.sweeps[kl];
      tsw = (unsigned long long)sw;
      msw = sw;
      mo = cs.iters[kl];
      nu = cs.conv[kl] ? 0 : 1;
    }
  }
  unsigned long long tot = (unsigned long long)mine;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if (lane == 0 && tot) atomicAdd(nnz_total, tot);
  if (cs.sweeps) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tsw += __shfl_xor_sync(0xffffffffu, tsw, o);
      msw = max(msw, __shfl_xor_sync(0xffffffffu, msw, o));
      mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, o));
      nu += __shfl_xor_sync(0xffffffffu, nu, o);
    }
  }
  unsigned todo = __ballot_sync(0xffffffffu, mine > 0);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int64_t k = k0 + src;
    const int m = __shfl_sync(0xffffffffu, mine, src);
    const double sk = rescale ? scale[k] : 1.0;
    const size_t base = (size_t)k * 2 * nzcap + (size_t)cur[k] * nzcap;
    for (int e = lane; e < m; e += 32) {
      const int j = nz_rows[base + e];
      const double sj = rescale ? scale[j] : 1.0;
      const double t_jk = theta1(nz_vals[base + e], sigma_std[k], sj, sk, rescale != 0);
      double out = t_jk;
      if (symmetrize) {
        const size_t bj = (size_t)j * 2 * nzcap + (size_t)cur[j] * nzcap;
        const int mj = min(cnt[j], nzcap);
        int lo = 0, hi = mj;
        double b_kj = 0.0;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const int v = nz_rows[bj + mid];
          if (v == (int)k) { b_kj = nz_vals[bj + mid]; break; }
          if (v < (int)k) lo = mid + 1;
          else hi = mid;
        }
        if (b_kj == 0.0) continue;            // partner zero -> symmetrized value is zero
        const double t_kj = theta1(b_kj, sigma_std[j], sk, sj, rescale != 0);
        const double u = (j < k) ? t_jk : t_kj;   // Theta1[min, max]
        const double l = (j < k) ? t_kj : t_jk;   // Theta1[max, min]
        out = (fabs(u) > fabs(l)) ? l : u;
      }
      Theta[(size_t)k * (size_t)p + (size_t)j] = out;
    }
  }
  if (cs.sweeps && lane == 0) {
    if (tsw) atomicAdd(cs.tot, tsw);
    atomicMax(cs.mx_sweeps, msw);
    atomicMax(cs.mx_outer, mo);
    if (nu) atomicAdd(cs.nunc, nu);
    if (cs.t_end) atomicMax(cs.t_end, global_ns());   // the fit's end (ms_total)
  }
}

__global__ void assemble_diag_kernel(int64_t p, int64_t col_begin, int64_t col_end,
                                     const double* __restrict__ sigma_std,
                                     const double* __restrict__ scale, int rescale,
                                     double* __restrict__ Theta, double* __restrict__ sigma_out) {
  const int64_t k = col_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= col_end) return;
  const double sg = sigma_std[k];
  double w = 1.0 / (sg * sg);
  if (rescale) w = w / (scale[k] * scale[k]);
  Theta[(size_t)(k - col_begin) * (size_t)p + (size_t)k] = w;
  if (sigma_out) sigma_out[k - col_begin] = rescale ? scale[k] * sg : sg;
}

// Host-API variant: the nonzero entries of Theta (symmetrized or Theta1) as COO triplets plus
// the diagonal and sigma, so that only these cross PCIe (the dense zero-fill happens on the
// host while the device computes).  Entry order is arbitrary; positions are distinct.
__global__ void assemble_coo_kernel(int64_t p, const int64_t* __restrict__ col_ptr,
                                    const int32_t* __restrict__ rows, const double* __restrict__ vals,
                                    const double* __restrict__ sigma_std,
                                    const double* __restrict__ scale, int symmetrize, int rescale,
                                    int32_t* __restrict__ coo_row, int32_t* __restrict__ coo_col,
                                    double* __restrict__ coo_val, int* __restrict__ coo_count) {
  const int64_t e1 = col_ptr[p];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = p;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (col_ptr[mid] <= e) lo = mid;
      else hi = mid;
    }
    const int64_t k = lo;
    const int32_t j = rows[e];
    const double sj = scale ? scale[j] : 1.0, sk = scale ? scale[k] : 1.0;
    const double t_jk = theta1(vals[e], sigma_std[k], sj, sk, rescale != 0);
    double out = t_jk;
    if (symmetrize) {
      const double b_kj = csc_lookup(rows, vals, col_ptr[j], col_ptr[j + 1], (int32_t)k);
      if (b_kj == 0.0) continue;
      const double t_kj = theta1(b_kj, sigma_std[j], sk, sj, rescale != 0);
      const double u = (j < k) ? t_jk : t_kj;
      const double l = (j < k) ? t_kj : t_jk;
      out = (fabs(u) > fabs(l)) ? l : u;
    }
    const int slot = atomicAdd(coo_count, 1);
    coo_row[slot] = j;
    coo_col[slot] = (int32_t)k;
    coo_val[slot] = out;
  }
}

cudaError_t launch_assemble_coo(int64_t p, const int64_t* col_ptr, const int32_t* rows,
                                const double* vals, const double* sigma_std, const double* scale,
                                int symmetrize, int32_t* coo_row, int32_t* coo_col, double* coo_val,
                                int* coo_count, double* diag, double* sigma_out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(coo_count, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  const int rescale = scale != nullptr;
  assemble_coo_kernel<<<148 * 4, 256, 0, s>>>(p, col_ptr, rows, vals, sigma_std, scale, symmetrize,
                                              rescale, coo_row, coo_col, coo_val, coo_count);
  // diagonal written as a 1-row "Theta" of stride 0: reuse the diag kernel on a p-vector
  assemble_diag_kernel<<<(unsigned)((p + 255) / 256), 256, 0, s>>>(0, 0, p, sigma_std, scale,
                                                                   rescale, diag, sigma_out);
  return cudaGetLastError();
}

cudaError_t launch_csc_build(const int* nz_count, const int* nz_cur, const int* nz_rows,
                             const double* nz_vals, int ncols, int nzcap, int64_t* col_ptr,
                             int32_t* rows, double* vals, int64_t* total, cudaStream_t s) {
  const bool staged = (size_t)ncols * 4 <= 160 * 1024;
  if (staged)   // (per call: the attribute belongs to the current device)
    cudaFuncSetAttribute(csc_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  csc_scan_kernel<<<1, 1024, staged ? (size_t)ncols * 4 : 0, s>>>(nz_count, ncols, col_ptr, total,
                                                                 staged ? 1 : 0);
  const int wpb = 8;
  csc_copy_kernel<<<(ncols + wpb - 1) / wpb, wpb * 32, 0, s>>>(nz_count, nz_cur, nz_rows, nz_vals,
                                                               ncols, nzcap, col_ptr, rows, vals);
  return cudaGetLastError();
}

cudaError_t launch_csc_counts(const int* nz_count, int ncols, int32_t* out, cudaStream_t s) {
  csc_counts_kernel<<<(ncols + 255) / 256, 256, 0, s>>>(nz_count, ncols, out);
  return cudaGetLastError();
}

cudaError_t launch_assemble(int64_t p, int64_t col_begin, int64_t col_end, const int64_t* col_ptr,
                            const int32_t* rows, const double* vals, const double* sigma_std,
                            const double* scale, int symmetrize, double* Theta, double* sigma_out,
                            cudaStream_t s, bool zero_fill) {
  const int64_t m = col_end - col_begin;
  if (zero_fill) {
    cudaError_t e = cudaMemsetAsync(Theta, 0, sizeof(double) * (size_t)p * (size_t)m, s);
    if (e != cudaSuccess) return e;
  }
  const int rescale = scale != nullptr;
  assemble_entries_kernel<<<148 * 4, 256, 0, s>>>(p, col_begin, col_end, col_ptr, rows, vals,
                                                  sigma_std, scale, symmetrize, rescale, Theta);
  assemble_diag_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(p, col_begin, col_end,
                                                                   sigma_std, scale, rescale,
                                                                   Theta, sigma_out);
  return cudaGetLastError();
}

// Sparse Θ (§8(f) f3): per column k the kept off-diagonal entries (symmetrize: the partner
// b_kj is nonzero — the dense path writes exactly these) plus the diagonal, rows ascending.
__device__ __forceinline__ bool theta_kept(int k, int j, const int* __restrict__ cnt,
                                           const int* __restrict__ cur,
                                           const int* __restrict__ nz_rows,
                                           const double* __restrict__ nz_vals, int nzcap,
                                           int symmetrize, double* b_kj_out) {
  if (!symmetrize) return true;
  const size_t bj = (size_t)j * 2 * nzcap + (size_t)cur[j] * nzcap;
  int lo = 0, hi = min(cnt[j], nzcap);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int v = nz_rows[bj + mid];
    if (v == k) { *b_kj_out = nz_vals[bj + mid]; return nz_vals[bj + mid] != 0.0; }
    if (v < k) lo = mid + 1;
    else hi = mid;
  }
  return false;
}

__global__ void sparse_count_kernel(int64_t p, const int* __restrict__ cnt, const int* __restrict__ cur,
                                    const int* __restrict__ nz_rows, const double* __restrict__ nz_vals,
                                    int nzcap, int symmetrize, int* __restrict__ ccount) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= p) return;
  const int m = min(cnt[k], nzcap);
  const size_t base = (size_t)k * 2 * nzcap + (size_t)cur[k] * nzcap;
  int kept = 0;
  for (int e = lane; e < m; e += 32) {
    double bkj = 0.0;
    kept += theta_kept((int)k, nz_rows[base + e], cnt, cur, nz_rows, nz_vals, nzcap, symmetrize, &bkj);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kept += __shfl_xor_sync(0xffffffffu, kept, o);
  if (lane == 0) ccount[k] = kept + 1;   // + the diagonal
}

__global__ void sparse_write_kernel(int64_t p, const int* __restrict__ cnt, const int* __restrict__ cur,
                                    const int* __restrict__ nz_rows, const double* __restrict__ nz_vals,
                                    int nzcap, const double* __restrict__ sigma_std,
                                    const double* __restrict__ scale, int symmetrize, int rescale,
                                    const int64_t* __restrict__ col_ptr, int32_t* __restrict__ rows,
                                    double* __restrict__ vals, double* __restrict__ sigma_out,
                                    int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= p) return;
  if (cap >= 0 && col_ptr[p] > cap) {   // too small: the arrays stay untouched (host reports)
    if (lane == 0 && sigma_out) sigma_out[k] = scale ? scale[k] * sigma_std[k] : sigma_std[k];
    return;
  }
  const int m = min(cnt[k], nzcap);
  const size_t base = (size_t)k * 2 * nzcap + (size_t)cur[k] * nzcap;
  const double sk = rescale ? scale[k] : 1.0;
  int64_t pos = col_ptr[k];
  bool diag_done = false;
  for (int e0 = 0; e0 < m; e0 += 32) {
    const int e = e0 + lane;
    int j = 0x7fffffff;
    double out = 0.0;
    bool kept = false;
    if (e < m) {
      j = nz_rows[base + e];
      const double sj = rescale ? scale[j] : 1.0;
      const double t_jk = theta1(nz_vals[base + e], sigma_std[k], sj, sk, rescale != 0);
      double b_kj = 0.0;
      kept = theta_kept((int)k, j, cnt, cur, nz_rows, nz_vals, nzcap, symmetrize, &b_kj);
      out = t_jk;
      if (kept && symmetrize) {   // as assemble_lists_kernel
        const double t_kj = theta1(b_kj, sigma_std[j], sk, sj, rescale != 0);
        const double u = (j < k) ? t_jk : t_kj;
        const double l = (j < k) ? t_kj : t_jk;
        out = (fabs(u) > fabs(l)) ? l : u;
      }
    }
    // the diagonal goes before the first kept row above k
    const unsigned kept_mask = __ballot_sync(0xffffffffu, kept);
    const unsigned above = __ballot_sync(0xffffffffu, kept && j > k);
    int dpos = -1;
    if (!diag_done && above) { dpos = __popc(kept_mask & ((above & -above) - 1u)); diag_done = true; }
    if (kept) {
      const int before = __popc(kept_mask & ((1u << lane) - 1u));
      const int shift = (dpos >= 0 && before >= dpos) ? 1 : 0;
      rows[pos + before + shift] = j;
      vals[pos + before + shift] = out;
    }
    if (dpos >= 0 && lane == 0) rows[pos + dpos] = (int32_t)k;
    if (dpos >= 0 && lane == 0) {
      const double sg = sigma_std[k];
      double w = 1.0 / (sg * sg);
      if (rescale) w = w / (sk * sk);
      vals[pos + dpos] = w;
    }
    pos += __popc(kept_mask) + (dpos >= 0 ? 1 : 0);
  }
  if (lane == 0) {
    if (!diag_done) {
      const double sg = sigma_std[k];
      double w = 1.0 / (sg * sg);
      if (rescale) w = w / (sk * sk);
      rows[pos] = (int32_t)k;
      vals[pos] = w;
    }
    if (sigma_out) sigma_out[k] = rescale ? sk * sigma_std[k] : sigma_std[k];
  }
}

cudaError_t launch_sparse_count(int64_t p, const int* cnt, const int* cur, const int* nz_rows,
                                const double* nz_vals, int nzcap, int symmetrize, int* ccount,
                                cudaStream_t s) {
  const int wpb = 8;
  sparse_count_kernel<<<(unsigned)((p + wpb - 1) / wpb), wpb * 32, 0, s>>>(p, cnt, cur, nz_rows,
                                                                          nz_vals, nzcap, symmetrize,
                                                                          ccount);
  return cudaGetLastError();
}

cudaError_t launch_sparse_write(int64_t p, const int* cnt, const int* cur, const int* nz_rows,
                                const double* nz_vals, int nzcap, const double* sigma_std,
                                const double* scale, int symmetrize, const int64_t* col_ptr,
                                int32_t* rows, double* vals, double* sigma_out, cudaStream_t s,
                                int64_t cap) {
  const int wpb = 8;
  sparse_write_kernel<<<(unsigned)((p + wpb - 1) / wpb), wpb * 32, 0, s>>>(
      p, cnt, cur, nz_rows, nz_vals, nzcap, sigma_std, scale, symmetrize, scale != nullptr,
      col_ptr, rows, vals, sigma_out, cap);
  return cudaGetLastError();
}

// ---- Peer-to-peer exchange of the multi-device fit (§8(f) f3) ----------------
// Every device fits a contiguous column block (blocks in device order, sizes p/G rounded as
// column_range does).  Instead of all-gathering the coefficients, each device reads what it
// needs straight from its peers' memory over NVLink (peer access enabled by the host):
//   p2p_flag_max — the global first-sweep screening flags, max over every device's share;
//   assemble_coo_p2p — a8 + a10 of the device's own columns: for each nonzero b_jk of its
//     block the partner b_kj is looked up by binary search in column j's list *on the device
//     that owns column j*, and sigma_j is read there too.  Same arithmetic as
//     assemble_coo_kernel (theta1, the P:391-393 tie rule), so the entries are bit-identical;
//     the symmetrization is spread over the G devices ("easily parallelizable")
//     instead of running on one after an all-gather.

// owner block of column j and its first column (column_range in multi.cu: the first p % G
// blocks have one column more)
__device__ __forceinline__ int p2p_owner(const P2PBlocks& B, int64_t j, int64_t* c0) {
  const int64_t base = B.p / B.G, rem = B.p % B.G;
  const int64_t big = rem * (base + 1);
  const int o = (j < big) ? (int)(j / (base + 1)) : (int)(rem + (j - big) / base);
  *c0 = (int64_t)o * base + min((int64_t)o, rem);
  return o;
}

__global__ void p2p_flag_max_kernel(P2PBlocks B, uint8_t* __restrict__ out) {
  const int64_t nw = B.p >> 2;   // whole 32-bit words (cudaMalloc'd buffers: aligned)
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw;
       w += (int64_t)gridDim.x * blockDim.x) {
    unsigned v = 0;
    for (int e = 0; e < B.G; ++e) v = __vmaxu4(v, ((const unsigned*)B.flags[e])[w]);
    ((unsigned*)out)[w] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x < (B.p & 3)) {
    const int64_t i = (nw << 2) + threadIdx.x;
    uint8_t v = 0;
    for (int e = 0; e < B.G; ++e) v = max(v, B.flags[e][i]);
    out[i] = v;
  }
}

__global__ void assemble_coo_p2p_kernel(P2PBlocks B, int self, const double* __restrict__ scale,
                                        int symmetrize, int rescale,
                                        int32_t* __restrict__ coo_row, int32_t* __restrict__ coo_col,
                                        double* __restrict__ coo_val, int* __restrict__ coo_count) {
  const int64_t* __restrict__ cp = B.col_ptr[self];
  const int32_t* __restrict__ rows = B.rows[self];
  const double* __restrict__ vals = B.vals[self];
  const int64_t base = B.p / B.G, rem = B.p % B.G;
  const int64_t c0s = (int64_t)self * base + min((int64_t)self, rem);
  const int64_t m = base + (self < rem ? 1 : 0);
  const int64_t e1 = cp[m];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = m;   // local column of entry e
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (cp[mid] <= e) lo = mid;
      else hi = mid;
    }
    const int64_t k = c0s + lo;
    const int32_t j = rows[e];
    const double sj = rescale ? scale[j] : 1.0, sk = rescale ? scale[k] : 1.0;
    const double t_jk = theta1(vals[e], B.sigma_std[self][lo], sj, sk, rescale != 0);
    double out = t_jk;
    if (symmetrize) {
      int64_t c0j;
      const int oj = p2p_owner(B, j, &c0j);
      const int64_t* __restrict__ cpj = B.col_ptr[oj];
      const int64_t jl = j - c0j;
      const double b_kj = csc_lookup(B.rows[oj], B.vals[oj], cpj[jl], cpj[jl + 1], (int32_t)k);
      if (b_kj == 0.0) continue;
      const double t_kj = theta1(b_kj, B.sigma_std[oj][jl], sk, sj, rescale != 0);
      const double u = (j < k) ? t_jk : t_kj;
      const double l = (j < k) ? t_kj : t_jk;
      out = (fabs(u) > fabs(l)) ? l : u;
    }
    const int slot = atomicAdd(coo_count, 1);
    coo_row[slot] = j;
    coo_col[slot] = (int32_t)k;
    coo_val[slot] = out;
  }
}

// diagonal and sigma of the device's own columns (as assemble_diag_kernel)
__global__ void assemble_diag_block_kernel(int64_t c0, int64_t m, const double* __restrict__ sig,
                                           const double* __restrict__ scale, int rescale,
                                           double* __restrict__ diag, double* __restrict__ sigma_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t k = c0 + i;
  const double sg = sig[i];
  double w = 1.0 / (sg * sg);
  if (rescale) w = w / (scale[k] * scale[k]);
  diag[i] = w;
  sigma_out[i] = rescale ? scale[k] * sg : sg;
}

cudaError_t launch_p2p_flag_max(const P2PBlocks& B, uint8_t* out, cudaStream_t s) {
  const int64_t nw = std::max<int64_t>(B.p >> 2, 1);
  const unsigned grid = (unsigned)std::min<int64_t>((nw + 255) / 256, 148 * 4);
  p2p_flag_max_kernel<<<grid, 256, 0, s>>>(B, out);
  return cudaGetLastError();
}

cudaError_t launch_assemble_coo_p2p(const P2PBlocks& B, int self, const double* scale,
                                    int symmetrize, int32_t* coo_row, int32_t* coo_col,
                                    double* coo_val, int* coo_count, double* diag,
                                    double* sigma_out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(coo_count, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  const int rescale = scale != nullptr;
  assemble_coo_p2p_kernel<<<148 * 4, 256, 0, s>>>(B, self, scale, symmetrize, rescale, coo_row,
                                                  coo_col, coo_val, coo_count);
  const int64_t base = B.p / B.G, rem = B.p % B.G;
  const int64_t c0 = (int64_t)self * base + std::min<int64_t>(self, rem);
  const int64_t m = base + (self < rem ? 1 : 0);
  assemble_diag_block_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(
      c0, m, B.sigma_std[self], scale, rescale, diag, sigma_out);
  return cudaGetLastError();
}

cudaError_t launch_csc_scan(const int* cnt, int ncols, int64_t* col_ptr, int64_t* total,
                            cudaStream_t s) {
  const bool staged = (size_t)ncols * 4 <= 160 * 1024;
  if (staged)
    cudaFuncSetAttribute(csc_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  csc_scan_kernel<<<1, 1024, staged ? (size_t)ncols * 4 : 0, s>>>(cnt, ncols, col_ptr, total,
                                                                 staged ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_assemble_lists(int64_t p, const int* nz_count, const int* nz_cur,
                                  const int* nz_rows, const double* nz_vals, int nzcap,
                                  const double* sigma_std, const double* scale, int symmetrize,
                                  double* Theta, double* sigma_out, int64_t* nnz_total,
                                  cudaStream_t s, const ColStats* cs) {
  const int wpb = 4;                     // (32 columns per warp)
  const int64_t warps = (p + 31) / 32;
  ColStats c{};
  if (cs) c = *cs;
  assemble_lists_kernel<<<(unsigned)((warps + wpb - 1) / wpb), wpb * 32, 0, s>>>(
      p, nz_count, nz_cur, nz_rows, nz_vals, nzcap, sigma_std, scale, symmetrize,
      scale != nullptr, Theta, sigma_out, (unsigned long long*)nnz_total, c);
  return cudaGetLastError();
}


// Per-column statistics on the device (no host copy of iters/sweeps/converged):
// out[0] += sum sweeps (64-bit), out[2] = max sweeps, out[3] = max iters, out[4] += unconverged.
__global__ void column_stats_kernel(const int32_t* __restrict__ iters, const int32_t* __restrict__ sweeps,
                                    const uint8_t* __restrict__ conv, int64_t m,
                                    unsigned long long* tot, int* mx_sweeps, int* mx_outer, int* nunc,
                                    unsigned long long* t_end) {
  unsigned long long t = 0;
  int ms = 0, mo = 0, nu = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    t += (unsigned long long)sweeps[k];
    ms = max(ms, sweeps[k]);
    mo = max(mo, iters[k]);
    nu += conv[k] ? 0 : 1;
  }
  for (int o = 16; o > 0; o >>= 1) {
    t += __shfl_xor_sync(0xffffffffu, t, o);
    ms = max(ms, __shfl_xor_sync(0xffffffffu, ms, o));
    mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, o));
    nu += __shfl_xor_sync(0xffffffffu, nu, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (t) atomicAdd(tot, t);
    atomicMax(mx_sweeps, ms);
    atomicMax(mx_outer, mo);
    if (nu) atomicAdd(nunc, nu);
    if (t_end) atomicMax(t_end, global_ns());   // the fit's end (ms_total)
  }
}

cudaError_t launch_column_stats(const int32_t* iters, const int32_t* sweeps, const uint8_t* conv,
                                int64_t m, unsigned long long* tot, int* mx_sweeps, int* mx_outer,
                                int* nunc, cudaStream_t s, unsigned long long* t_end) {
  if (m <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>(64, (m + 255) / 256);
  column_stats_kernel<<<blocks, 256, 0, s>>>(iters, sweeps, conv, m, tot, mx_sweeps, mx_outer, nunc,
                                             t_end);
  return cudaGetLastError();
}

// Zero-fill of Theta on a side stream with a grid of one 256-thread block per SM: small enough
// to stay co-resident with the solver kernel (one CTA per SM), so the 8 p^2-byte write really
// overlaps the solve instead of occupying every SM first as a library memset would.
__global__ void __launch_bounds__(256) zero_fill_kernel(double2* __restrict__ a, size_t n2) {
  const double2 z = make_double2(0.0, 0.0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2;
       i += (size_t)gridDim.x * blockDim.x)
    __stcs(a + i, z);
}

// The same fill with bulk (TMA) stores from one elected thread per 32-thread CTA: almost no SM
// footprint (it runs beside the exact Gram-column and sweep kernels), and the stores carry an
// L2 evict-first hint so the 8 p^2 bytes streaming through L2 do not push out X~.
constexpr int ZB_PIECE = 2048;   // doubles per bulk store (16 KB)
__global__ void __launch_bounds__(32) zero_fill_bulk_kernel(double* __restrict__ a, size_t count) {
  __shared__ __align__(128) double zb[ZB_PIECE];
  for (int e = threadIdx.x; e < ZB_PIECE; e += 32) zb[e] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncwarp();
  if (threadIdx.x != 0) return;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(zb);
  const size_t npieces = (count + ZB_PIECE - 1) / ZB_PIECE;
  for (size_t k = blockIdx.x; k < npieces; k += gridDim.x) {
    const size_t off = k * ZB_PIECE;
    const size_t cnt = min((size_t)ZB_PIECE, count - off);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(
                     a + off),
                 "r"(src), "r"((uint32_t)(cnt * 8)), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// Per-fit scratch reset in one launch (instead of five memsets): the counter block (zeros,
// with the 8-byte bad-column key at key_off set to all ones), the 16-byte work queue and the
// per-slot list counters nz_count / nz_cur.
// (also stamps the fit's start, t_off: the device-side clock of ms_total, so that a captured
// fit needs no timing-event nodes for it; the counter block is <= 256 bytes, so block 0 alone
// resets it and the stamp cannot be overwritten)
__global__ void reset_kernel(unsigned char* counters, int counters_bytes, int key_off, int t_off,
                             int* queue, int* nz_count, int* nz_cur, int64_t m, uint8_t* z0,
                             size_t z0_bytes, uint8_t* z1, size_t z1_bytes) {
  const unsigned long long t0 = global_ns();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t; i < counters_bytes; i += stride)
    counters[i] = (i >= key_off && i < key_off + 8) ? 0xff : 0;
  if (t < 4) queue[t] = 0;
  for (int64_t i = t; i < m; i += stride) { nz_count[i] = 0; nz_cur[i] = 0; }
  for (int64_t i = t; i < (int64_t)z0_bytes; i += stride) z0[i] = 0;
  for (int64_t i = t; i < (int64_t)z1_bytes; i += stride) z1[i] = 0;
  if (blockIdx.x == 0) {
    __syncthreads();
    if (threadIdx.x == 0) *(unsigned long long*)(counters + t_off) = t0;
  }
}

cudaError_t launch_reset(void* counters, int counters_bytes, int key_off, int t_off, int* queue,
                         int* nz_count, int* nz_cur, int64_t m, cudaStream_t s, void* z0,
                         size_t z0_bytes, void* z1, size_t z1_bytes) {
  if (counters_bytes > 256) return cudaErrorInvalidValue;   // (block 0 resets it alone)
  const int64_t work = std::max<int64_t>(std::max<int64_t>(m, counters_bytes),
                                         (int64_t)std::max(z0_bytes, z1_bytes));
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(296, (work + 255) / 256));
  reset_kernel<<<blocks, 256, 0, s>>>((unsigned char*)counters, counters_bytes, key_off, t_off,
                                      queue, nz_count, nz_cur, m, (uint8_t*)z0, z0_bytes,
                                      (uint8_t*)z1, z1_bytes);
  return cudaGetLastError();
}

cudaError_t launch_zero_fill_bulk(double* a, size_t count, int grid, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  if (((uintptr_t)a & 15) != 0 || (count & 1)) return cudaMemsetAsync(a, 0, count * 8, s);
  zero_fill_bulk_kernel<<<grid, 32, 0, s>>>(a, count);
  return cudaGetLastError();
}

cudaError_t launch_zero_fill(double* a, size_t count, int sms, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  if (((uintptr_t)a & 15) != 0 || (count & 1)) return cudaMemsetAsync(a, 0, count * 8, s);
  // same shared-memory carve-out as the solver kernels, so an SM running this kernel can take a
  // solver CTA without being reconfigured (which would serialize the two)
  cudaFuncSetAttribute(zero_fill_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       (int)cudaSharedmemCarveoutMaxShared);

  zero_fill_kernel<<<sms, 256, 0, s>>>((double2*)a, count / 2);
  return cudaGetLastError();
}

}  // namespace spmesl
