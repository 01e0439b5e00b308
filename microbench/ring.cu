// Microbenchmark of the CD kernel's X-tile pipeline: one CTA per SM,
// 1 producer warp issuing cp.async.bulk of CHUNK-byte tiles into an NST-deep mbarrier ring,
// 8 consumer warps in 2 parity groups; each consumer warp does `dmma_per_chunk` DMMAs per
// chunk (operands from the chunk and a resident R tile) or none.  Reports achieved L2->SMEM
// bandwidth and DMMA TFLOP/s for: stream only, compute only (no waits), both.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ring ring.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(bytes), "r"(su(b)) : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// mode: 0 stream only, 1 compute only, 2 both
__global__ void __launch_bounds__(288, 1) ring(const double* X, size_t nchunks, int chunk_doubles,
                                               int NST, int mode, int kpairs, double* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 16;
  double* R = (double*)(sm + 256);                 // resident B operand (32 x 520 doubles)
  double* Xs = R + 32 * 520;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = threadIdx.x; e < 32 * 520; e += blockDim.x) R[e] = 1e-3 * (e % 17);
  __syncthreads();
  const uint32_t bytes = chunk_doubles * 8;
  if (warp == 8) {
    if (lane == 0 && mode != 1) {
      int s = 0; uint32_t ph = 0;
      for (size_t c = 0; c < nchunks; ++c) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect(&full[s], bytes);
        bulk(Xs + (size_t)s * chunk_doubles, X + (c % 8192) * chunk_doubles, bytes, &full[s]);
        if (++s == NST) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  const int grp = warp >> 2, wg = warp & 3, g = lane >> 2, t4 = lane & 3;
  const int m0 = 2 * (wg & 1), n0 = 2 * (wg >> 1);
  double acc[2][2][2] = {};
  int s = grp; uint32_t ph = 0;
  if (s >= NST) { s -= NST; ph ^= 1; }
  for (size_t c = grp; c < nchunks; c += 2) {
    if (mode != 1) mbar_wait(&full[s], ph);
    const double* xs = Xs + (size_t)s * chunk_doubles + (m0 * 8 + g) * 32 + 2 * t4;
    const double* rs = R + (n0 * 8 + g) * 520 + 2 * t4 + (c % 16) * 32;
    if (mode != 0) {
      for (int kp = 0; kp < kpairs; ++kp) {
        double2 a0 = *(const double2*)(xs + ((kp & 3) ^ (g & 1)) * 8);
        double2 a1 = *(const double2*)(xs + 8 * 32 + ((kp & 3) ^ (g & 1)) * 8);
        double2 b0 = *(const double2*)(rs + (kp & 3) * 8);
        double2 b1 = *(const double2*)(rs + 8 * 520 + (kp & 3) * 8);
        dmma(acc[0][0][0], acc[0][0][1], a0.x, b0.x); dmma(acc[0][1][0], acc[0][1][1], a0.x, b1.x);
        dmma(acc[1][0][0], acc[1][0][1], a1.x, b0.x); dmma(acc[1][1][0], acc[1][1][1], a1.x, b1.x);
        dmma(acc[0][0][0], acc[0][0][1], a0.y, b0.y); dmma(acc[0][1][0], acc[0][1][1], a0.y, b1.y);
        dmma(acc[1][0][0], acc[1][0][1], a1.y, b0.y); dmma(acc[1][1][0], acc[1][1][1], a1.y, b1.y);
      }
    }
    __syncwarp();
    if (mode != 1 && lane == 0) mbar_arrive(&empty[s]);
    s += 2; if (s >= NST) { s -= NST; ph ^= 1; }
  }
  double t = 0;
  for (int i = 0; i < 2; ++i) for (int j = 0; j < 2; ++j) t += acc[i][j][0] + acc[i][j][1];
  if (t == 1234.5) out[0] = t;
}

int main(int argc, char** argv) {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int chunk_doubles = 1024;                           // 32 x 32 doubles, 8 KB
  double* X; CK(cudaMalloc(&X, (size_t)8192 * chunk_doubles * 8));   // 64 MB, L2-resident
  CK(cudaMemset(X, 0, (size_t)8192 * chunk_doubles * 8));
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
  printf("{\"sms\": %d", sms);
  const size_t nchunks = 20000;
  for (int mode = 0; mode < 3; ++mode)
    for (int NST : {4, 6, 8, 10, 12})
      for (int kpairs : {4}) {
        size_t smem = 256 + 32 * 520 * 8 + (size_t)NST * chunk_doubles * 8;
        if (smem > 232448) continue;
        ring<<<sms, 288, smem>>>(X, 200, chunk_doubles, NST, mode, kpairs, out);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        ring<<<sms, 288, smem>>>(X, nchunks, chunk_doubles, NST, mode, kpairs, out);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        double gbs = (double)nchunks * chunk_doubles * 8 * sms / (ms * 1e-3) / 1e9;
        double tf = (double)nchunks * 4 * kpairs * 8 * 256 * 2 * sms / (ms * 1e-3) / 1e12;
        printf(", \"mode%d_nst%d\": {\"ms\": %.3f, \"l2_to_smem_gbs\": %.0f, \"dmma_tflops\": %.2f}", mode, NST, ms,
               mode == 1 ? 0.0 : gbs, mode == 0 ? 0.0 : tf);
      }
  printf("}\n");
  return 0;
}
