// Projection pass W = A^T Z on the 5th-generation tensor cores (sm_100a).
//
// tenrec/sketch.py:262-263 forms w = a^T z (n x s) and m = w^T w for the
// Rayleigh-Ritz step; s = (q+1) b is 20-40, so this is the one genuinely dense
// contraction of the Krylov iteration (2s flops per streamed element).  Here:
//   * A tile  = 128 columns of the unfolding x 32 rows (K), K-major, 128B
//     swizzle, filled by cp.async; its low part A_lo = A - tf32(A) is written
//     next to it by the threads (3xTF32: A Z_hi + A Z_lo + A_lo Z_hi, fp32-
//     faithful; the tensor core truncates fp32 operands to tf32).
//   * Z_hi / Z_lo tiles = 32 (N, s padded) x 32 rows, same layout.
//   * tcgen05.mma.cta_group::1.kind::tf32, M=128 N=32 K=8, accumulator in TMEM
//     (32 columns), issued by one thread; tcgen05.commit releases each stage.
//   * epilogue per 128-column tile: tcgen05.ld -> W rows to HBM, and the
//     32 x 32 Gram W^T W of the tile accumulated in fp64 (the per-CTA partial
//     of M), so no separate pass over W is needed.
#pragma once

#include "common.cuh"
#include "panel.cuh"

namespace tr {

constexpr int kPjThreads = 128;
constexpr int kPjStages = 4;
constexpr int kPjTileBytes = 128 * 128;  // A tile: 128 rows x 128 B
constexpr int kPjZBytes = 32 * 128;      // Z tile: 32 rows x 128 B
constexpr int kPjStageBytes = 2 * kPjTileBytes + 2 * kPjZBytes;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;  // zero-fill when out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// byte offset of 16-byte chunk q of row r in a K-major SWIZZLE_128B tile
__device__ __forceinline__ uint32_t sw128(int r, int q) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((q ^ (r & 7)) << 4));
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, SBO = 1024 B (8-row atoms)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

// instruction descriptor: kind::tf32, fp32 accumulate, K-major A and B
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 32 consecutive fp32 TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Z (m x 32, column-major, zero beyond s) split into tf32 high / low parts
__global__ void k_split_z(const double* __restrict__ Z, int64_t m, int s,
                          float* __restrict__ zhi, float* __restrict__ zlo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * 32) return;
  const int j = (int)(e / m);
  const double z = j < s ? Z[e] : 0.0;
  const float f = (float)z;
  const float hi = __uint_as_float(__float_as_uint(f) & 0xFFFFE000u);
  zhi[e] = hi;
  zlo[e] = (float)(z - (double)hi);
}

// W (n x s row-major) = A^T Z ; part[blk] (32 x 32, fp64) = sum over this CTA's
// columns of w w^T.  Requires m % 32 == 0 and 16-byte aligned A.
__global__ void __launch_bounds__(kPjThreads, 1)
    k_proj_tc(const float* __restrict__ A, int64_t m, int64_t n, const float* __restrict__ zhi,
              const float* __restrict__ zlo, int s, float* __restrict__ W,
              double* __restrict__ part) {
  extern __shared__ __align__(1024) unsigned char pj_raw[];
  __shared__ __align__(8) uint64_t mma_done[kPjStages];
  __shared__ __align__(8) uint64_t acc_ready;
  __shared__ uint32_t tmem_base_s;
  __shared__ float wtile[128][33];
  unsigned char* smem = (unsigned char*)(((uintptr_t)pj_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t ntiles = (n + 127) / 128;
  const int kt = (int)(m / 32);
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t iters = my_tiles * kt;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        smem_u32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kPjStages; ++i) mbar_init(&mma_done[i], 1);
    mbar_init(&acc_ready, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const uint32_t idesc = idesc_tf32(128, 32);

  // issue the cp.async loads of iteration `it` into its stage
  auto load = [&](int64_t it) {
    if (it < iters) {
      const int64_t tile = blockIdx.x + (it / kt) * gridDim.x;
      const int64_t k0 = (it % kt) * 32;
      const int64_t c0 = tile * 128;
      const uint32_t st = sbase + (uint32_t)((it % kPjStages) * kPjStageBytes);
#pragma unroll
      for (int u = 0; u < 8; ++u) {  // A: 128 rows x 8 chunks
        const int e = tid + kPjThreads * u;
        const int r = e >> 3, q = e & 7;
        const int64_t col = c0 + r;
        const bool ok = col < n;
        cp_async16(st + sw128(r, q), A + (ok ? col : 0) * m + k0 + 4 * q, ok);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {  // Z_hi, Z_lo: 32 rows x 8 chunks each
        const int e = tid + kPjThreads * u;
        const int r = e >> 3, q = e & 7;
        cp_async16(st + 2 * kPjTileBytes + sw128(r, q), zhi + (int64_t)r * m + k0 + 4 * q, true);
        cp_async16(st + 2 * kPjTileBytes + kPjZBytes + sw128(r, q), zlo + (int64_t)r * m + k0 + 4 * q,
                   true);
      }
    }
    cp_async_commit();
  };

  for (int i = 0; i < kPjStages - 1; ++i) load(i);
  double g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) g[i] = 0.0;
  uint32_t acc_phase = 0;

  for (int64_t it = 0; it < iters; ++it) {
    const int sidx = (int)(it % kPjStages);
    const uint32_t st = sbase + (uint32_t)(sidx * kPjStageBytes);
    // refill the stage consumed by the previous iteration (its MMAs are older)
    if (it >= 1) {
      const int64_t prev = it - 1;
      mbar_wait(&mma_done[prev % kPjStages], (uint32_t)((prev / kPjStages) & 1));
    }
    load(it + kPjStages - 1);
    cp_async_wait<kPjStages - 1>();
    // A_lo = A - tf32(A) for this thread's chunks
    unsigned char* sp = smem + sidx * kPjStageBytes;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + kPjThreads * u;
      const uint32_t off = sw128(e >> 3, e & 7);
      const float4 a = *reinterpret_cast<const float4*>(sp + off);
      float4 lo;
      lo.x = a.x - __uint_as_float(__float_as_uint(a.x) & 0xFFFFE000u);
      lo.y = a.y - __uint_as_float(__float_as_uint(a.y) & 0xFFFFE000u);
      lo.z = a.z - __uint_as_float(__float_as_uint(a.z) & 0xFFFFE000u);
      lo.w = a.w - __uint_as_float(__float_as_uint(a.w) & 0xFFFFE000u);
      *reinterpret_cast<float4*>(sp + kPjTileBytes + off) = lo;
    }
    fence_async_smem();
    __syncthreads();
    const bool first_k = (it % kt) == 0;
    const bool last_k = (it % kt) == kt - 1;
    if (tid == 0) {
      tc_fence_after();
      const uint64_t dA = umma_desc_sw128(st);
      const uint64_t dAl = umma_desc_sw128(st + kPjTileBytes);
      const uint64_t dZh = umma_desc_sw128(st + 2 * kPjTileBytes);
      const uint64_t dZl = umma_desc_sw128(st + 2 * kPjTileBytes + kPjZBytes);
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // K = 8 per MMA: +32 B in the swizzled row
        const uint64_t adv = (uint64_t)(2 * k);
        umma_tf32(tmem, dA + adv, dZh + adv, idesc, (first_k && k == 0) ? 0u : 1u);
        umma_tf32(tmem, dA + adv, dZl + adv, idesc, 1u);
        umma_tf32(tmem, dAl + adv, dZh + adv, idesc, 1u);
      }
      umma_commit(&mma_done[sidx]);
      if (last_k) umma_commit(&acc_ready);
    }
    if (last_k) {
      mbar_wait(&acc_ready, acc_phase);
      acc_phase ^= 1;
      tc_fence_after();
      float w[32];
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), w);
      const int64_t tile = blockIdx.x + (it / kt) * gridDim.x;
      const int64_t col = tile * 128 + tid;
      if (col < n) {
        for (int j = 0; j < s; ++j) W[col * s + j] = w[j];
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) wtile[tid][j] = (col < n) ? w[j] : 0.f;
      tc_fence_before();
      __syncthreads();
      // tile Gram: thread owns 8 entries e = tid + 128 u of the 32 x 32 block
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = tid + kPjThreads * u;
        const int j = e >> 5, k = e & 31;
        double a = 0.0;
        for (int r = 0; r < 128; ++r) a += (double)wtile[r][j] * (double)wtile[r][k];
        g[u] += a;
      }
      __syncthreads();
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = tid + kPjThreads * u;
    const int j = e >> 5, k = e & 31;
    if (j < s && k < s) part[(int64_t)blockIdx.x * s * s + j * s + k] = g[u];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  }
}

}  // namespace tr
