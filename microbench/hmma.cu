// Microbenchmark: legacy warp-level tensor-core MMA (mma.sync m16n8k16, f16/bf16 inputs, f32
// accumulate) throughput on B200 — the candidate engine for a certified low-precision
// screening pass.  Prints one JSON object.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma hmma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1;} } while (0)

template <int NACC, bool BF>
__global__ void hmma_kernel(float* out, int iters) {
  uint32_t a0 = 0x3c003c00u ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  uint32_t b0 = 0x3c003c00u ^ (threadIdx.x * 3), b1 = b0 + 5;
  float acc[NACC][4];
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NACC; ++k) {
      if (BF)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(acc[k][0]), "+f"(acc[k][1]), "+f"(acc[k][2]), "+f"(acc[k][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(acc[k][0]), "+f"(acc[k][1]), "+f"(acc[k][2]), "+f"(acc[k][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NACC; ++k) s += acc[k][0] + acc[k][1] + acc[k][2] + acc[k][3];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  float* d; CK(cudaMalloc(&d, 16));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  printf("{\"gpu\": \"%s\"", prop.name);
  for (int bf = 0; bf < 2; ++bf)
    for (int wps = 4; wps <= 16; wps *= 2) {
      const int iters = 20000, threads = 32 * wps, blocks = sms;
      auto run = [&](int it) {
        if (bf) hmma_kernel<8, true><<<blocks, threads>>>(d, it);
        else hmma_kernel<8, false><<<blocks, threads>>>(d, it);
      };
      run(10); CK(cudaDeviceSynchronize());
      float best = 0.f;
      for (int rep = 0; rep < 3; ++rep) {
        float ms;
        CK(cudaEventRecord(e0)); run(iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double fl = 2.0 * 16 * 8 * 16 * 8.0 * iters * (double)blocks * wps;
        const float tf = (float)(fl / (ms * 1e-3) / 1e12);
        if (tf > best) best = tf;
      }
      printf(", \"%s_m16n8k16_w%d_tflops\": %.1f", bf ? "bf16" : "f16", wps, best);
    }
  printf("}\n");
  return 0;
}
