// Dev microbenchmark: how fast can a B200 write zeros to HBM (the 8 p^2-byte Theta fill)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fill fill.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
#include <initializer_list>

__global__ void st_kernel(double2* a, size_t n2) {
  const double2 z = make_double2(0.0, 0.0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    __stcs(a + i, z);
}
__global__ void st_kernel_v8(double4* a, size_t n4) {   // 32-byte stores
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double* p = (double*)(a + i);
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%1,%1,%1};\n" :: "l"(p), "d"(0.0) : "memory");
  }
}
template <int PIECE, int HINT>
__global__ void bulk_kernel(double* a, size_t count) {
  extern __shared__ __align__(128) double zb[];
  for (int e = threadIdx.x; e < PIECE; e += blockDim.x) zb[e] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane != 0) return;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(zb);
  const size_t np = (count + PIECE - 1) / PIECE;
  for (size_t k = (size_t)blockIdx.x * nw + warp; k < np; k += (size_t)gridDim.x * nw) {
    const size_t off = k * PIECE;
    const size_t cnt = (count - off) < PIECE ? (count - off) : PIECE;
    if (HINT)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(a + off), "r"(src), "r"((uint32_t)(cnt * 8)), "l"(pol) : "memory");
    else
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(a + off), "r"(src), "r"((uint32_t)(cnt * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// contiguous range per CTA (each CTA fills [bid*count/G, (bid+1)*count/G))
template <int PIECE>
__global__ void bulk_contig(double* a, size_t count) {
  extern __shared__ __align__(128) double zb[];
  for (int e = threadIdx.x; e < PIECE; e += blockDim.x) zb[e] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t lo = (count * blockIdx.x / gridDim.x) & ~(size_t)1, hi = (blockIdx.x + 1 == gridDim.x) ? count : ((count * (blockIdx.x + 1) / gridDim.x) & ~(size_t)1);
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(zb);
  for (size_t off = lo; off < hi; off += PIECE) {
    const size_t cnt = (hi - off) < PIECE ? (hi - off) : PIECE;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(a + off), "r"(src), "r"((uint32_t)(cnt * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
// S contiguous streams per CTA issued round-robin by ONE thread (as a producer warp would)
template <int PIECE>
__global__ void bulk_streams(double* a, size_t count, int S) {
  extern __shared__ __align__(128) double zb[];
  for (int e = threadIdx.x; e < PIECE; e += blockDim.x) zb[e] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(zb);
  const size_t nstream = (size_t)gridDim.x * S;
  size_t cur[16], end[16];
  for (int u = 0; u < S; ++u) {
    const size_t sid = (size_t)blockIdx.x * S + u;
    cur[u] = (count * sid / nstream) & ~(size_t)1;
    end[u] = (sid + 1 == nstream) ? count : ((count * (sid + 1) / nstream) & ~(size_t)1);
  }
  bool any = true;
  while (any) {
    any = false;
    for (int u = 0; u < S; ++u) {
      if (cur[u] >= end[u]) continue;
      any = true;
      const size_t cnt = (end[u] - cur[u]) < PIECE ? (end[u] - cur[u]) : PIECE;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(a + cur[u]), "r"(src), "r"((uint32_t)(cnt * 8)) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      cur[u] += cnt;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__global__ void st_contig(double* a, size_t count) {
  const size_t lo = (count * blockIdx.x / gridDim.x) & ~(size_t)3, hi = (blockIdx.x + 1 == gridDim.x) ? count : ((count * (blockIdx.x + 1) / gridDim.x) & ~(size_t)3);
  for (size_t i = lo + 4 * threadIdx.x; i < hi; i += 4 * blockDim.x)
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%1,%1,%1};\n" :: "l"(a + i), "d"(0.0) : "memory");
}

int main() {
  const size_t count = (size_t)20000 * 20000;  // 3.2 GB
  double* a;
  cudaMalloc(&a, count * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto f) {
    for (int w = 0; w < 2; ++w) f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("%-40s %.3f ms  %.0f GB/s %s\n", name, best, count * 8 / (best * 1e6), err ? cudaGetErrorString(err) : "");
  };
  timeit("cudaMemsetAsync", [&] { cudaMemsetAsync(a, 0, count * 8); });
  cudaFuncSetAttribute(bulk_kernel<2048, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * 8);
  for (int g : std::initializer_list<int>{})
    for (int t : {256, 512, 1024}) {
      char nm[64]; snprintf(nm, 64, "st.cs v2 grid %d x %d", g, t);
      timeit(nm, [&] { st_kernel<<<g, t>>>((double2*)a, count / 2); });
    }
  for (int g : {1184, 2368}) {
    char nm[64]; snprintf(nm, 64, "st.cs v4.f64 grid %d x 512", g);
    timeit(nm, [&] { st_kernel_v8<<<g, 512>>>((double4*)a, count / 4); });
  }
  cudaFuncSetAttribute(bulk_streams<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * 8);
  for (int S : {1, 2, 4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "bulk 16K streams grid 148 S %d", S);
    timeit(nm, [&] { bulk_streams<2048><<<148, 32, 2048 * 8>>>(a, count, S); });
  }
  cudaFuncSetAttribute(bulk_contig<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * 8);
  cudaFuncSetAttribute(bulk_contig<8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8);
  for (int g : {148, 296, 592, 1184, 2368}) {
    char nm[64];
    snprintf(nm, 64, "bulk contig 16K grid %d", g);
    timeit(nm, [&] { bulk_contig<2048><<<g, 32, 2048 * 8>>>(a, count); });
    snprintf(nm, 64, "bulk contig 64K grid %d", g);
    timeit(nm, [&] { bulk_contig<8192><<<g, 32, 8192 * 8>>>(a, count); });
    snprintf(nm, 64, "st.v4 contig grid %d x 512", g);
    timeit(nm, [&] { st_contig<<<g, 512>>>(a, count); });
  }
  for (int g : {1184, 2368})
    for (int w : {1}) {
      char nm[64];
      snprintf(nm, 64, "bulk 16K grid-stride grid %d warps %d", g, w);
      timeit(nm, [&] { bulk_kernel<2048, 0><<<g, 32 * w, 2048 * 8>>>(a, count); });
    }
  return 0;
  cudaFuncSetAttribute(bulk_kernel<2048, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * 8);
  cudaFuncSetAttribute(bulk_kernel<4096, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 8);
  cudaFuncSetAttribute(bulk_kernel<8192, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8);
  cudaFuncSetAttribute(bulk_kernel<2048, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * 8);
  for (int g : {148, 296, 592})
    for (int w : {1, 2, 4}) {
      char nm[64];
      snprintf(nm, 64, "bulk 16K hint grid %d warps %d", g, w);
      timeit(nm, [&] { bulk_kernel<2048, 1><<<g, 32 * w, 2048 * 8>>>(a, count); });
      snprintf(nm, 64, "bulk 16K nohint grid %d warps %d", g, w);
      timeit(nm, [&] { bulk_kernel<2048, 0><<<g, 32 * w, 2048 * 8>>>(a, count); });
      snprintf(nm, 64, "bulk 32K hint grid %d warps %d", g, w);
      timeit(nm, [&] { bulk_kernel<4096, 1><<<g, 32 * w, 4096 * 8>>>(a, count); });
      snprintf(nm, 64, "bulk 64K hint grid %d warps %d", g, w);
      timeit(nm, [&] { bulk_kernel<8192, 1><<<g, 32 * w, 8192 * 8>>>(a, count); });
    }
  return 0;
}
