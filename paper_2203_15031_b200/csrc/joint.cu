// Algorithm 3, the paper's joint ("PCD") mode: every active column sweeps in
// lockstep until max over active columns of ||B_next - B_cur||_inf < delta; then sigma
// is refit for all of them at once and the columns whose sigma moved by less than
// delta leave the active set (F_j).  The sweeps themselves run in the persistent CD
// kernel (cd_sweep.cu, CDParams::joint: one sweep per launch, residuals carried in Ej); this
// file holds the outer-boundary kernels the host driver (api.cu, fit_joint_core) chains.
#include <algorithm>
#include "spmesl_internal.cuh"

namespace spmesl {

namespace {

// E = X_I - X B^(0) = x~_c for every column (P:949 at r = 0); sigma^(0) = 1.
__global__ void joint_init_kernel(const double* __restrict__ Xb, int64_t col_begin, int m,
                                  int n_pad, int nchunk, int* __restrict__ act,
                                  double* __restrict__ sigma, double* __restrict__ Ej) {
  const int c = blockIdx.x;
  if (c >= m) return;
  const int64_t gcol = col_begin + c;
  double* e = Ej + (size_t)c * n_pad;
  for (int i = threadIdx.x; i < n_pad; i += blockDim.x) e[i] = Xb[xb_index(i, gcol, nchunk)];
  if (threadIdx.x == 0) {
    act[c] = c;
    sigma[c] = 1.0;
  }
}

// Outer boundary for the active columns (one warp each): fresh residual
// e_c = x~_c - sum_{b_jc != 0, ascending j} x~_j b_jc (reading g4; it is also the E of the next
// outer iteration), sigma_c = max(||e_c|| / sqrt(n), floor) (reading g5),
// F_c = |sigma_new - sigma_old| >= delta.
__global__ void joint_sigma_kernel(const double* __restrict__ Xb, int64_t col_begin,
                                   const int* __restrict__ act, int nact,
                                   const int* __restrict__ nz_rows,
                                   const double* __restrict__ nz_vals,
                                   const int* __restrict__ nz_count, const int* __restrict__ nz_cur,
                                   int nzcap, int n, int n_pad, int nchunk, double sqrt_n,
                                   double sigma_floor, double tol, int capped,
                                   double* __restrict__ sigma, int* __restrict__ iters,
                                   uint8_t* __restrict__ jflags, uint8_t* __restrict__ converged,
                                   double* __restrict__ Ej, uint8_t* __restrict__ keep) {
  const int lane = threadIdx.x & 31;
  const int q = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  if (q >= nact) return;
  const int col = act[q];
  const int64_t gcol = col_begin + col;
  double* e = Ej + (size_t)col * n_pad;
  for (int i = lane; i < n_pad; i += 32) e[i] = Xb[xb_index(i, gcol, nchunk)];
  const size_t base = (size_t)col * 2 * nzcap + (size_t)nz_cur[col] * nzcap;
  const int cnt = min(nz_count[col], nzcap);
  for (int m = 0; m < cnt; ++m) {
    const int j = nz_rows[base + m];
    const double bj = nz_vals[base + m];
    for (int i = lane; i < n_pad; i += 32) e[i] = fma(-Xb[xb_index(i, j, nchunk)], bj, e[i]);
  }
  double ss = 0.0;
  for (int i = lane; i < n; i += 32) ss = fma(e[i], e[i], ss);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) {
    double sn = sqrt(ss) / sqrt_n;
    if (sn < sigma_floor) sn = sigma_floor;              // reading g5
    const double so = sigma[col];
    const int k = !(fabs(sn - so) < tol);                // F_c
    uint8_t fl = jflags[col];
    if (capped) fl |= 2;                                 // an inner loop hit max_inner (g16)
    jflags[col] = fl;
    sigma[col] = sn;
    iters[col] += 1;
    converged[col] = (uint8_t)(!k && !(fl & 2));
    keep[q] = (uint8_t)k;
  }
}

// Stable compaction I <- {I_j : F_j = 1} in order: one block, chunked scan.
__global__ void joint_compact_kernel(const int* __restrict__ act, const uint8_t* __restrict__ keep,
                                     int nact, int* __restrict__ act_out, int* __restrict__ nact_out) {
  __shared__ int wsum[32];
  __shared__ int base_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) base_s = 0;
  __syncwarp();
  __syncthreads();
  for (int off = 0; off < nact; off += blockDim.x) {
    const int q = off + tid;
    const int f = (q < nact) ? (int)keep[q] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    const int pre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += wsum[w];
    const int base = base_s;
    if (f) act_out[base + wbase + pre] = act[q];
    __syncwarp();
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < nw; ++w) t += wsum[w];
      base_s = base + t;
    }
    __syncwarp();
    __syncthreads();
  }
  if (tid == 0) *nact_out = base_s;
}

// Mode 1 on the Gram form: the columns with a first-sweep hit become sweep slots (their z is
// carried between joint sweeps); the others sweep as no-ops until their sigma converges.
__global__ void joint_live_init_kernel(const uint8_t* __restrict__ hit, int m, int* __restrict__ nslots,
                                       TailState* __restrict__ jtail, int* __restrict__ slotmap) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m; c += gridDim.x * blockDim.x) {
    if (hit[c]) {
      const int sl = atomicAdd(nslots, 1);
      TailState t;
      t.col = c; t.outer = 0; t.sweeps = 0; t.inner = 0; t.flags = 0; t.cur = 0; t.cnt = 0;
      t.lam = 0; t.sigma = 1.0;
      jtail[sl] = t;
      slotmap[c] = sl;
    } else {
      slotmap[c] = -1;
    }
  }
}

// active columns without a slot get one (z from their Gram column, b = 0 so far)
__global__ void joint_live_add_kernel(const int* __restrict__ act, int nact, int* __restrict__ slotmap,
                                      TailState* __restrict__ jtail, int* __restrict__ nslots,
                                      const int* __restrict__ nz_cur) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nact; q += gridDim.x * blockDim.x) {
    const int c = act[q];
    if (slotmap[c] >= 0) continue;
    const int sl = atomicAdd(nslots, 1);
    TailState t;
    t.col = c; t.outer = 0; t.sweeps = 0; t.inner = 0; t.flags = 0; t.cur = nz_cur[c]; t.cnt = 0;
    t.lam = 0; t.sigma = 1.0;
    jtail[sl] = t;
    slotmap[c] = sl;
  }
}

// how many active columns have no slot yet
__global__ void joint_count_unslotted_kernel(const int* __restrict__ act, int nact,
                                             const int* __restrict__ slotmap, int* __restrict__ cnt) {
  int c = 0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nact; q += gridDim.x * blockDim.x)
    c += slotmap[act[q]] < 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// the slots of the active columns (work list of one joint sweep, any order)
__global__ void joint_work_kernel(const int* __restrict__ act, int nact, const int* __restrict__ slotmap,
                                  int* __restrict__ work, int* __restrict__ nwork) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nact; q += gridDim.x * blockDim.x) {
    const int sl = slotmap[act[q]];
    if (sl >= 0) work[atomicAdd(nwork, 1)] = sl;
  }
}

// every active column swept `inner` times in this outer iteration
__global__ void joint_add_sweeps_kernel(const int* __restrict__ act, int nact, int inner,
                                        int* __restrict__ sweeps) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nact; q += gridDim.x * blockDim.x)
    sweeps[act[q]] += inner;
}

}  // namespace

cudaError_t launch_joint_live_init(const uint8_t* hit, int m, int* nslots, TailState* jtail,
                                   int* slotmap, cudaStream_t s) {
  joint_live_init_kernel<<<std::max(1, std::min(296, (m + 255) / 256)), 256, 0, s>>>(hit, m, nslots,
                                                                                  jtail, slotmap);
  return cudaGetLastError();
}

cudaError_t launch_joint_live_add(const int* act, int nact, int* slotmap, TailState* jtail,
                                  int* nslots, const int* nz_cur, cudaStream_t s) {
  if (nact <= 0) return cudaSuccess;
  joint_live_add_kernel<<<std::max(1, std::min(296, (nact + 255) / 256)), 256, 0, s>>>(
      act, nact, slotmap, jtail, nslots, nz_cur);
  return cudaGetLastError();
}

cudaError_t launch_joint_count_unslotted(const int* act, int nact, const int* slotmap, int* cnt,
                                         cudaStream_t s) {
  if (nact <= 0) return cudaSuccess;
  joint_count_unslotted_kernel<<<std::max(1, std::min(296, (nact + 255) / 256)), 256, 0, s>>>(
      act, nact, slotmap, cnt);
  return cudaGetLastError();
}

cudaError_t launch_joint_work(const int* act, int nact, const int* slotmap, int* work, int* nwork,
                              cudaStream_t s) {
  if (nact <= 0) return cudaSuccess;
  joint_work_kernel<<<std::max(1, std::min(296, (nact + 255) / 256)), 256, 0, s>>>(act, nact, slotmap,
                                                                                 work, nwork);
  return cudaGetLastError();
}

cudaError_t launch_joint_add_sweeps(const int* act, int nact, int inner, int* sweeps, cudaStream_t s) {
  if (nact <= 0 || inner <= 0) return cudaSuccess;
  joint_add_sweeps_kernel<<<std::max(1, std::min(296, (nact + 255) / 256)), 256, 0, s>>>(act, nact,
                                                                                       inner, sweeps);
  return cudaGetLastError();
}

cudaError_t launch_joint_init(const double* Xb, int64_t col_begin, int m, int n_pad, int nchunk,
                              int* act, double* sigma, double* Ej, cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  joint_init_kernel<<<m, 128, 0, s>>>(Xb, col_begin, m, n_pad, nchunk, act, sigma, Ej);
  return cudaGetLastError();
}

cudaError_t launch_joint_sigma(const double* Xb, int64_t col_begin, const int* act, int nact,
                               const int* nz_rows, const double* nz_vals, const int* nz_count,
                               const int* nz_cur, int nzcap, int n, int n_pad, int nchunk,
                               double sqrt_n, double sigma_floor, double tol, int capped,
                               double* sigma, int* iters, uint8_t* jflags, uint8_t* converged,
                               double* Ej, uint8_t* keep, cudaStream_t s) {
  if (nact <= 0) return cudaSuccess;
  const int wpb = 8;
  joint_sigma_kernel<<<(nact + wpb - 1) / wpb, wpb * 32, 0, s>>>(
      Xb, col_begin, act, nact, nz_rows, nz_vals, nz_count, nz_cur, nzcap, n, n_pad, nchunk,
      sqrt_n, sigma_floor, tol, capped, sigma, iters, jflags, converged, Ej, keep);
  return cudaGetLastError();
}

cudaError_t launch_joint_compact(const int* act, const uint8_t* keep, int nact, int* act_out,
                                 int* nact_out, cudaStream_t s) {
  joint_compact_kernel<<<1, 1024, 0, s>>>(act, keep, nact, act_out, nact_out);
  return cudaGetLastError();
}

}  // namespace spmesl
