// Certified low-precision screening for the Gram solver.
//
// The first sweep of column c changes some b_jc iff |S_jc| > lambda0 for some j != c
// (sigma^(0) = 1), S = X~^T X~ / n.  Deciding that needs S only to the extent of a
// comparison, so it is done on the f16 tensor cores (tcgen05.mma kind::f16 with the f32
// accumulator in TMEM) with a rigorous error bound, and only the columns that cannot be certified hit-free get their exact
// FP64 Gram column (DMMA, gram_pass in tail.cu, which also takes the exact decision).  No
// low-precision value ever enters the iterates.
//
// Bound.  y_k = x~_k / sqrt(N_k) with N_k = x~_k^T x~_k / n, so y_k^T y_k = n and
// R = Y^T Y / n is the correlation-scaled S: S_jc = R_jc sqrt(N_j N_c), |R_jc| <= 1.
// y_hat = fp16(y) (|y| <= sqrt(n) < 65504): |y_hat - y| <= u |y| + 2^-25 (u = 2^-11; the
// absolute term covers subnormals).  Products of two f16 values are exact in f32; allow every
// f32 accumulation step a relative error 2^-23 (round or truncate).  With sum_i |y_ij y_ic| <= n
// (Cauchy-Schwarz):
//   |R_hat_jc - R_jc| <= 2.1 u + n_pad 2^-22 + 2^-23 + 2^-20 =: eps      (n_pad <= 2^16)
// The pair is certified hit-free when (|R_hat_jc| + eps)(1 + 2^-40) sqrt(N_j N_c) <= lambda0.
// In terms of the raw accumulator acc = n R_hat_jc the epilogue tests
//   |acc| <= fma_rd(lam_n_j, inv_c, -epsn),  lam_n_j = rd(n lambda0 / sqrt(N_j)),
//   inv_c = rd(1 / sqrt(N_c)), epsn = ru(n eps)
// (every factor rounded so the f32 threshold can only come out smaller).
//
// Layout of Y16: tiles of 128 variables x 64 samples, one contiguous 16 KB block per tile
// ([nblk128][nchunk64][128][64] halves), each 128-byte row's 16-byte chunks XOR-swizzled by
// (row & 7): the canonical K-major SWIZZLE_128B layout tcgen05.mma reads.
#include <algorithm>
#include <cstdlib>
#include <cuda_fp16.h>
#include "spmesl_internal.cuh"

namespace spmesl {

namespace {

constexpr int S16_TB = 128;                 // variables per tile side
constexpr int S16_KC = 64;                  // samples per chunk
constexpr int S16_TILE_HALVES = S16_TB * S16_KC;     // 8192 halves = 16 KB
#ifndef SPMESL_S16_ZPIECE
#define SPMESL_S16_ZPIECE 2048
#endif
constexpr int S16_ZPIECE = SPMESL_S16_ZPIECE;   // doubles per Theta zero-fill bulk store

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait_s(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(su32(bar)), "r"(parity) : "memory");
}

// Theta's zero fill is spread over the producer's chunks in proportion, so the 8 p^2-byte write
// (the kernel's HBM floor at large p) overlaps the whole contraction instead of trailing it.
__device__ __forceinline__ size_t zero_quota(const Screen16Params& P, size_t npieces, int nchunk) {
  const int bid = blockIdx.x, G = gridDim.x;
  const int ntiles = P.tile_end - P.tile_begin;
  const size_t my_chunks = (size_t)(ntiles > bid ? (ntiles - bid + G - 1) / G : 0) * nchunk;
  const size_t my_pieces = npieces > (size_t)bid ? (npieces - bid + G - 1) / G : 0;
  return my_chunks ? (my_pieces + my_chunks - 1) / my_chunks : 0;
}
__device__ __forceinline__ void zero_pieces(const Screen16Params& P, const double* zbuf, size_t& zp,
                                            size_t npieces, size_t k) {
  for (; k > 0 && zp < npieces; --k) {
    const size_t off = zp * S16_ZPIECE;
    const size_t cnt = min((size_t)S16_ZPIECE, P.zero_count - off);
#ifndef SPMESL_S16_NO_EVICT_FIRST
    // evict-first: the 8 p^2 bytes streaming through L2 should not push out the f16 tiles
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(
                     P.zero_ptr + off),
                 "r"(su32(zbuf)), "r"((uint32_t)(cnt * 8)), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(P.zero_ptr + off),
                 "r"(su32(zbuf)), "r"((uint32_t)(cnt * 8))
                 : "memory");
#endif
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    zp += gridDim.x;
  }
}

// ------------------------------------------------------------------ tcgen05 version
// The same screening contraction on the 5th-generation tensor cores: the 128 x 64 f16 tiles of
// Y16 are already the canonical K-major SWIZZLE_128B layout (128-byte rows, 16-byte chunks
// XOR-ed with row & 7, 1024-byte aligned; two consecutive tiles form the 256-row layout), so
// one thread issues tcgen05.mma (M = 128, N = BN, K = 16) straight from the TMA-filled ring
// into a TMEM accumulator (two BN-column buffers: the epilogue of tile t overlaps the MMAs of
// tile t + 1), and eight epilogue warps read it back with tcgen05.ld.  Roles: warp 0 TMA
// producer (+ Theta zero fill), warp 1 MMA issuer and TMEM owner, warps 2-9 epilogue (two per
// TMEM lane quarter, each half of the columns).
// BN = 256: tiles of 128 rows x 256 columns, 1.5 B of operand traffic per output
// instead of 2 (the kernel is bound by L2 -> SM operand traffic, not by the tensor cores).
// Tile set: column block Jb (256 wide) pairs with row blocks I = 0 .. min(2 Jb + 1, ntb - 1),
// which covers every pair of the upper triangle (plus one redundant 128 x 128 sub-block below
// the diagonal per column block).
constexpr int T5_EPI_WARPS = 8;
constexpr int T5_THREADS = (2 + T5_EPI_WARPS) * 32;

constexpr int BN = 256;
constexpr int T5_NST = 3;                   // operand ring stages (3 x 48 KB; 4 measured the same)
constexpr size_t t5_smem() {
  return 1024 + (size_t)T5_NST * (1 + BN / 128) * S16_TILE_HALVES * 2 + (size_t)S16_ZPIECE * 8;
}

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu)      // start address
         | ((uint64_t)1 << 16)                    // leading byte offset (16 B; unused for SW128 K)
         | ((uint64_t)(1024 >> 4) << 32)          // stride byte offset: 8 rows x 128 B
         | ((uint64_t)1 << 46)                    // descriptor version (sm_100)
         | ((uint64_t)2 << 61);                   // SWIZZLE_128B
}

// wide tile t -> (row block I, 256-column block Jb); column block Jb holds min(2 Jb + 2, ntb)
// tiles, so tiles before block Jb number Jb (Jb + 1) (only the last block can be capped)
__device__ __forceinline__ void wide_tile(int t, int& I, int& Jb) {
  int jb = (int)((sqrt(4.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((jb + 1) * (jb + 2) <= t) ++jb;
  while (jb * (jb + 1) > t) --jb;
  Jb = jb;
  I = t - jb * (jb + 1);
}

__global__ void __launch_bounds__(T5_THREADS, 1) screen16_tc_kernel(const Screen16Params P) {
  if (P.zero_last && blockIdx.x == 0 && threadIdx.x == 0) *P.zero_last = 0.0;
  constexpr int NBT = BN / 128;                    // B sub-tiles per stage
  constexpr int NST = T5_NST;
  constexpr int STAGE_HALVES = (1 + NBT) * S16_TILE_HALVES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // [0, 1024): barriers + TMEM address; ring at 1024 (1024-aligned tiles); zero piece after it
  uint64_t* full = (uint64_t*)smem_raw;
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  __half* ring = (__half*)(smem_raw + 1024);
  double* zbuf = (double*)(ring + (size_t)NST * STAGE_HALVES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nchunk = P.nchunk64;
  if (P.zero_ptr) {
    for (int e = tid; e < S16_ZPIECE; e += blockDim.x) zbuf[e] = 0.0;
    // the producer's bulk stores (async proxy) read zbuf: every writer orders its generic-proxy
    // stores before them, then the barrier below publishes that to the producer
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&empty[s])), "r"(1));
    }
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&tfull[b])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&tempty[b])), "r"(T5_EPI_WARPS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (warp == 1) {   // TMEM: 2 accumulators x BN columns (f32), 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *(volatile uint32_t*)tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const size_t npieces = P.zero_ptr ? (P.zero_count + S16_ZPIECE - 1) / S16_ZPIECE : 0;
      size_t zp = blockIdx.x;
      const size_t zquota = zero_quota(P, npieces, nchunk);
      for (int t = P.tile_begin + blockIdx.x; t < P.tile_end; t += gridDim.x) {
        int I, Jb;
        wide_tile(t, I, Jb);
        for (int q = 0; q < nchunk; ++q) {
          mbar_wait_s(&empty[s], ph ^ 1u);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&full[s])),
                       "r"((uint32_t)STAGE_HALVES * 2u)
                       : "memory");
          __half* dst = ring + (size_t)s * STAGE_HALVES;
#pragma unroll
          for (int u = 0; u <= NBT; ++u) {   // A tile, then the NBT tiles of the column block
            const int blk = u == 0 ? I : Jb * NBT + (u - 1);
            const __half* src = P.Y16 + ((size_t)blk * nchunk + q) * S16_TILE_HALVES;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    su32(dst + (size_t)u * S16_TILE_HALVES)),
                "l"(src), "r"((uint32_t)S16_TILE_HALVES * 2u), "r"(su32(&full[s]))
                : "memory");
          }
          zero_pieces(P, zbuf, zp, npieces, zquota);   // Theta's zero fill rides along
          if (++s == NST) { s = 0; ph ^= 1u; }
        }
      }
      zero_pieces(P, zbuf, zp, npieces, npieces);
      asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    // instruction descriptor: D f32, A = B = f16, both K-major, N = BN, M = 128
    const uint32_t idesc = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((128u >> 4) << 24);
    int s = 0, it = 0;
    uint32_t ph = 0;
    uint32_t ph_te[2] = {0u, 0u};
    for (int t = P.tile_begin + blockIdx.x; t < P.tile_end; t += gridDim.x, ++it) {
      const int ab = it & 1;
      mbar_wait_s(&tempty[ab], ph_te[ab] ^ 1u);     // the epilogue has drained this buffer
      ph_te[ab] ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t dtm = tmem + (uint32_t)(ab * BN);
      for (int q = 0; q < nchunk; ++q) {
        mbar_wait_s(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const uint32_t sa = su32(ring + (size_t)s * STAGE_HALVES);
          const uint32_t sb = sa + S16_TILE_HALVES * 2;
#pragma unroll
          for (int kk = 0; kk < S16_KC / 16; ++kk) {
            const uint64_t da = umma_desc_sw128(sa + kk * 32);
            const uint64_t db = umma_desc_sw128(sb + kk * 32);
            const uint32_t acc = (q > 0 || kk > 0) ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtm),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          // the stage is free once these MMAs have read it
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           su32(&empty[s]))
                       : "memory");
        }
        __syncwarp();
        if (++s == NST) { s = 0; ph ^= 1u; }
      }
      if (lane == 0)   // accumulator complete
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         su32(&tfull[ab]))
                     : "memory");
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2-9)
    const int qd = warp & 3;                     // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;            // column half of the tile
    constexpr int GPW = BN / 64;                 // 32-column groups per warp
    int it = 0;
    uint32_t ph_tf[2] = {0u, 0u};
    for (int t = P.tile_begin + blockIdx.x; t < P.tile_end; t += gridDim.x, ++it) {
      int I, Jb;
      wide_tile(t, I, Jb);
      const int ab = it & 1;
      mbar_wait_s(&tfull[ab], ph_tf[ab]);
      ph_tf[ab] ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int j = I * S16_TB + 32 * qd + lane;          // this thread's row of the tile
      const bool jok = j < P.p;
      const float rA = jok ? P.lam_n[j] : 0.f;
#pragma unroll 1
      for (int cg = GPW * half; cg < GPW * half + GPW; ++cg) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(32 * qd) << 16) + (uint32_t)(ab * BN + 32 * cg);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
              "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
              "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (jok && P.acc_out) {   // (test-only: the raw accumulators n R_hat_jc)
          const int c0 = Jb * BN + 32 * cg;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            P.acc_out[(size_t)(c0 + i) * (size_t)P.acc_ld + (size_t)j] = __uint_as_float(v[i]);
        }
        if (jok) {
          // the certification threshold (header); the 32 columns' factors are warp-uniform loads
          const int c0 = Jb * BN + 32 * cg;
          const bool diag_sub = (c0 >> 7) == I;           // the 128 x 128 diagonal sub-block
          const float4* iv = reinterpret_cast<const float4*>(P.inv_sq + c0);
          uint32_t hits = 0;
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4) {
            const float4 f = __ldg(iv + k4);
            hits |= (uint32_t)(fabsf(__uint_as_float(v[4 * k4 + 0])) > __fmaf_rd(rA, f.x, -P.epsn)) << (4 * k4 + 0);
            hits |= (uint32_t)(fabsf(__uint_as_float(v[4 * k4 + 1])) > __fmaf_rd(rA, f.y, -P.epsn)) << (4 * k4 + 1);
            hits |= (uint32_t)(fabsf(__uint_as_float(v[4 * k4 + 2])) > __fmaf_rd(rA, f.z, -P.epsn)) << (4 * k4 + 2);
            hits |= (uint32_t)(fabsf(__uint_as_float(v[4 * k4 + 3])) > __fmaf_rd(rA, f.w, -P.epsn)) << (4 * k4 + 3);
          }
          if (diag_sub && (unsigned)(j - c0) < 32u) hits &= ~(1u << (j - c0));   // c == j
          while (hits) {   // rare
            const int i = __ffs(hits) - 1;
            hits &= hits - 1;
            P.cand[c0 + i] = 1;
            if (!diag_sub) P.cand[j] = 1;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&tempty[ab])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * BN));
}

// Candidate list on the device (no host round trip): U[0..nU) = {c : cand[c]} in any order
// (every consumer indexes its results by c), gstate[c] = 2 for candidates (their Gram column
// will be present), 0 otherwise.
__global__ void cand_compact_kernel(const uint8_t* __restrict__ cand, int p, int cb, int ce,
                                    int* __restrict__ U, int* __restrict__ nU,
                                    int* __restrict__ gstate) {
  const int lane = threadIdx.x & 31;
  for (int base = blockIdx.x * blockDim.x; base < p; base += gridDim.x * blockDim.x) {
    const int c = base + threadIdx.x;
    const bool f = c >= cb && c < ce && cand[c];
    if (c < p) gstate[c] = f ? 2 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    int first = 0;
    if (lane == 0 && bal) first = atomicAdd(nU, __popc(bal));
    first = __shfl_sync(0xffffffffu, first, 0);
    if (f) U[first + __popc(bal & ((1u << lane) - 1u))] = c;
  }
}

}  // namespace

cudaError_t launch_cand_compact(const uint8_t* cand, int p, int* U, int* nU, int* gstate,
                                cudaStream_t s, int cb, int ce) {
  const int blocks = std::max(1, std::min(296, (p + 255) / 256));
  if (ce < 0) ce = p;
  cand_compact_kernel<<<blocks, 256, 0, s>>>(cand, p, cb, ce, U, nU, gstate);
  return cudaGetLastError();
}

// Y16 holds an even number of 128-row tiles (the 256-column blocks read two; the padding
// tiles are zero)
size_t screen16_y_halves(int64_t p, int n_pad) {
  const int64_t nb = (p + 2 * S16_TB - 1) / (2 * S16_TB) * 2;
  const int64_t nc = (n_pad + S16_KC - 1) / S16_KC;
  return (size_t)(nb * nc * S16_TILE_HALVES);
}

double screen16_eps(int n_pad) {
  return 2.1 * 0x1p-11 + (double)n_pad * 0x1p-22 + 0x1p-23 + 0x1p-20;
}

int64_t screen16_pad(int64_t p) { return (p + 2 * S16_TB - 1) / (2 * S16_TB) * (2 * S16_TB); }

int screen16_tile_count(int64_t p) {
  const int64_t nT = (p + S16_TB - 1) / S16_TB;
  const int64_t ncb = (nT + 1) / 2;
  int64_t tot = 0;
  for (int64_t jb = 0; jb < ncb; ++jb) tot += std::min<int64_t>(2 * jb + 2, nT);
  return (int)tot;
}

cudaError_t launch_screen16(const Screen16Params& P, int grid, cudaStream_t s) {
  if (P.tile_end <= P.tile_begin) return cudaSuccess;
  static_assert(T5_EPI_WARPS == 8, "epilogue: two warps per TMEM lane quarter");
  cudaError_t e = cudaFuncSetAttribute(screen16_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)t5_smem());
  if (e != cudaSuccess) return e;
  screen16_tc_kernel<<<grid, T5_THREADS, t5_smem(), s>>>(P);
  return cudaGetLastError();
}

}  // namespace spmesl
