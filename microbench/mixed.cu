// Are FP64 DMMA (tensor) and DFMA (CUDA-core) separate pipes on B200?  Warps 0..A-1 run DMMA
// chains, warps A.. run DFMA chains, concurrently; report combined FP64 TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void mixed(int mma_warps, int iters, double* out) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp < mma_warps) {
    double c0[8] = {}, c1[8] = {};
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int k = 0; k < 8; ++k) dmma(c0[k], c1[k], a, b);
    for (int k = 0; k < 8; ++k) s += c0[k] + c1[k];
  } else {
    double acc[8];
    for (int k = 0; k < 8; ++k) acc[k] = k;
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
    for (int it = 0; it < iters * 8; ++it)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fma(acc[k], b, a);
    for (int k = 0; k < 8; ++k) s += acc[k];
  }
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  printf("{");
  for (int mw : {0, 4, 8, 12, 16}) {
    const int warps = 16;
    mixed<<<148, warps * 32>>>(mw, 10, out); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    mixed<<<148, warps * 32>>>(mw, iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // DMMA warp: iters*8 DMMA * 256 FMA; DFMA warp: iters*8*8 DFMA * 32 lanes
    double fl = 2.0 * 148 * ((double)mw * iters * 8 * 256 + (double)(warps - mw) * iters * 64 * 32);
    printf("%s\"mma_warps_%d\": %.2f", mw ? ", " : "", mw, fl / (ms * 1e-3) / 1e12);
  }
  printf("}\n");
  return 0;
}
