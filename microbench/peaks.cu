// Roofline microbenchmarks for the SPMESL CD sweep on B200 (sm_100a).
// FP64 DFMA peak, FP64 DMMA (mma.sync m8n8k4) peak,
// L2-resident read bandwidth, HBM read bandwidth, plus a DMMA fragment-layout
// self-check (the CD kernel relies on the m8n8k4 .f64 fragment mapping).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o peaks peaks.cu
// Prints one JSON object on stdout.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, unsigned long long* cyc) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = k * 1e-3;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = fma(acc[k], b, a);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_kernel(double* out, int iters, unsigned long long* cyc) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c0[NACC], c1[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) { c0[k] = 0; c1[k] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NACC; ++k) dmma(c0[k], c1[k], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < NACC; ++k) s += c0[k] + c1[k];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
}

// One warp: D = A(8x4 row) * B(4x8 col) with the assumed fragment mapping.
__global__ void dmma_layout(const double* A, const double* B, double* D) {
  int lane = threadIdx.x;
  int g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t];      // A[m=g][k=t]
  double b = B[t * 8 + g];      // B[k=t][n=g]
  double d0 = 0, d1 = 0;
  dmma(d0, d1, a, b);
  D[g * 8 + 2 * t] = d0;        // D[m=g][n=2t]
  D[g * 8 + 2 * t + 1] = d1;
}

__global__ void read_kernel(const double2* __restrict__ buf, size_t n2, int reps, double* out) {
  double2 acc = make_double2(0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
      double2 v = __ldcg(buf + i);
      acc.x += v.x; acc.y += v.y;
    }
  if (acc.x + acc.y == 12345.678) out[0] = acc.x;
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  double* dout; CK(cudaMalloc(&dout, 64));
  unsigned long long* dcyc; CK(cudaMalloc(&dcyc, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu", prop.name, sms,
         prop.l2CacheSize, prop.sharedMemPerBlockOptin);

  // DFMA
  {
    int iters = 20000, threads = 256, blocks = sms * 8;
    dfma_kernel<<<blocks, threads>>>(dout, 100, dcyc);
    CK(cudaDeviceSynchronize());
    double best = 0, mhz = 0;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      dfma_kernel<<<blocks, threads>>>(dout, iters, dcyc);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      unsigned long long cyc; CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
      double fl = 2.0 * 8 * iters * (double)threads * blocks;
      double tf = fl / (ms * 1e-3) / 1e12;
      if (tf > best) { best = tf; mhz = cyc / (ms * 1e-3) / 1e6; }
    }
    printf(", \"dfma_tflops\": %.3f, \"dfma_clock_mhz_est\": %.0f", best, mhz);
    printf(", \"dfma_flop_per_clk_per_sm\": %.1f", best * 1e12 / (mhz * 1e6) / sms);
  }
  // DMMA with different accumulator counts (ILP) and warps/SM
  const int naccs[3] = {2, 4, 8};
  for (int v = 0; v < 3; ++v) {
    for (int wps = 4; wps <= 16; wps *= 2) {
      int iters = 4000, threads = 32 * wps, blocks = sms * 2;
      auto run = [&](int it) {
        if (naccs[v] == 2) dmma_kernel<2><<<blocks, threads / 2>>>(dout, it, dcyc);
        else if (naccs[v] == 4) dmma_kernel<4><<<blocks, threads / 2>>>(dout, it, dcyc);
        else dmma_kernel<8><<<blocks, threads / 2>>>(dout, it, dcyc);
      };
      run(10); CK(cudaDeviceSynchronize());
      double best = 0, mhz = 0;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0)); run(iters);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        unsigned long long cyc; CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
        double nwarps = (double)blocks * threads / 2 / 32;
        double fl = 2.0 * 256 * naccs[v] * (double)iters * nwarps;
        double tf = fl / (ms * 1e-3) / 1e12;
        if (tf > best) { best = tf; mhz = cyc / (ms * 1e-3) / 1e6; }
      }
      printf(", \"dmma_acc%d_w%d_tflops\": %.3f, \"dmma_acc%d_w%d_mhz\": %.0f", naccs[v], wps, best,
             naccs[v], wps, mhz);
    }
  }
  // DMMA layout check
  {
    double hA[32], hB[32], hD[64];
    for (int i = 0; i < 32; ++i) { hA[i] = (i * 7 % 11) - 5; hB[i] = (i * 5 % 13) - 6; }
    double *dA, *dB, *dD;
    CK(cudaMalloc(&dA, 256)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dD, 512));
    CK(cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice));
    dmma_layout<<<1, 32>>>(dA, dB, dD);
    CK(cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int m = 0; m < 8; ++m)
      for (int n = 0; n < 8; ++n) {
        double s = 0;
        for (int k = 0; k < 4; ++k) s += hA[m * 4 + k] * hB[k * 8 + n];
        maxerr = fmax(maxerr, fabs(s - hD[m * 8 + n]));
      }
    printf(", \"dmma_layout_maxerr\": %.3g", maxerr);
  }
  // L2-resident read bandwidth (48 MB buffer re-read) and HBM read bandwidth (4 GB)
  {
    size_t sizes[2] = {48ull << 20, 4ull << 30};
    const char* names[2] = {"l2_read_gbs", "hbm_read_gbs"};
    for (int s = 0; s < 2; ++s) {
      size_t bytes = sizes[s];
      double2* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
      int reps = s == 0 ? 20 : 1;
      int blocks = sms * 4, threads = 512;
      read_kernel<<<blocks, threads>>>(buf, bytes / 16, 1, dout);
      CK(cudaDeviceSynchronize());
      double best = 0;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        read_kernel<<<blocks, threads>>>(buf, bytes / 16, reps, dout);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
        if (gbs > best) best = gbs;
      }
      printf(", \"%s\": %.1f", names[s], best);
      CK(cudaFree(buf));
    }
  }
  printf("}\n");
  return 0;
}
