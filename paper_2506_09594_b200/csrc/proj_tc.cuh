// Projection pass W = A^T Z on the 5th-generation tensor cores (sm_100a).
//
// tenrec/sketch.py:262-263 forms w = a^T z (n x s) and m = w^T w for the
// Rayleigh-Ritz step; s = (q+1) b is 20-40, so this is the one genuinely dense
// contraction of the Krylov iteration (2s flops per streamed element).
// Warp-specialised persistent kernel, one CTA per SM:
//   warp 0     TMA producer: A tile = 128 columns of the unfolding x 32 rows
//              (K), K-major 128B-swizzled by the tensor map, plus the matching
//              32-row chunks of Z_hi / Z_lo, into a kPwStages-deep ring;
//   warps 2-9  split A_lo = A - tf32(A) of each landed tile straight into
//              TENSOR MEMORY (tcgen05.st: lane = tile row, 32 columns = the 32
//              K values) -- 3xTF32: A Z_hi + A Z_lo + A_lo Z_hi, fp32-faithful.
//              A_lo never round-trips through shared memory (the smem-resident
//              version moved 6.25 smem bytes per streamed byte, over the
//              128 B/clk port at the HBM rate; this one 4.25);
//   warp 1     one thread issues tcgen05.mma.cta_group::1.kind::tf32:
//              A[smem] x [Z_hi | Z_lo] (M=128 N=64 K=8) as soon as the TMA tile
//              lands, then A_lo[tmem] x Z_hi (N=32) once the split is in TMEM,
//              into a double-buffered TMEM accumulator; frees ring slots with
//              tcgen05.commit;
//   warps 10-13 epilogue: tcgen05.ld of a finished tile -> W rows in HBM and
//              the tile's 32 x 32 Gram W^T W accumulated in fp64 (the per-CTA
//              partial of M), while the next tile accumulates in the other
//              TMEM buffer.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "panel.cuh"

namespace tr {

constexpr int kPjTileBytes = 128 * 128;  // A tile: 128 rows x 128 B
constexpr int kPjZBytes = 32 * 128;      // Z tile: 32 rows x 128 B

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

// same with the A operand in tensor memory (lane = M row, one K value per column)
__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate));
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

// 32 consecutive 32-bit TMEM columns of this thread's lane <- v
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
      "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
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

constexpr int kPwStages = 8;   // TMA ring: A, Z_hi, Z_lo
constexpr int kPwLo = 8;       // A_lo ring in tensor memory (split warps -> MMA): 32 columns each
constexpr int kPwThreads = 448;
constexpr int kPwStageBytes = kPjTileBytes + 2 * kPjZBytes;
constexpr int kPwSmemBytes = kPwStages * kPwStageBytes;
constexpr int kPwTmemCols = 512;   // 2 accumulators x 64 + 2 lo accumulators x 32 + kPwLo x 32
constexpr int kPwTmemAccLo = 128;  // accumulators of A_lo Z_hi
constexpr int kPwTmemLo = 192;     // first A_lo column

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// W (n x s, row stride ldw) = A^T Z and part[blk] = this CTA's share of W^T W
// (s x s, fp64; part == nullptr: W only).  A: m x n column-major (tensor map mapA, box 32 x 128); Z_hi / Z_lo:
// m x 32 column-major (maps, box 32 x 32).  m % 32 == 0.
__global__ void __launch_bounds__(kPwThreads, 1)
    k_proj_ws(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapZh,
              const __grid_constant__ CUtensorMap mapZl, int64_t m, int64_t n, int s,
              float* __restrict__ W, double* __restrict__ part, int ldw) {
  extern __shared__ __align__(1024) unsigned char pw_raw[];
  __shared__ __align__(8) uint64_t full[kPwStages], empty[kPwStages];
  __shared__ __align__(8) uint64_t lo_ready[kPwLo], lo_empty[kPwLo];
  __shared__ __align__(8) uint64_t tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_s;
  unsigned char* smem = (unsigned char*)(((uintptr_t)pw_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + 127) / 128;
  const int kt = (int)(m / 32);
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t iters = my_tiles * kt;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        smem_u32(&tmem_base_s)), "n"(kPwTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPwStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kPwLo; ++i) {
      mbar_init(&lo_ready[i], 128);
      mbar_init(&lo_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      for (int64_t it = 0; it < iters; ++it) {
        const int st = (int)(it % kPwStages);
        const uint32_t ph = (uint32_t)((it / kPwStages) & 1);
        mbar_wait(&empty[st], ph ^ 1);
        const int64_t tile = blockIdx.x + (it / kt) * gridDim.x;
        const int k0 = (int)((it % kt) * 32);
        const uint32_t sa = sbase + (uint32_t)(st * kPwStageBytes);
        mbar_arrive_expect_tx(&full[st], kPjTileBytes + 2 * kPjZBytes);
        tma_load_2d(sa, &mapA, k0, (int)(tile * 128), &full[st]);
        tma_load_2d(sa + kPjTileBytes, &mapZh, k0, 0, &full[st]);
        tma_load_2d(sa + kPjTileBytes + kPjZBytes, &mapZl, k0, 0, &full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      // A x [Z_hi | Z_lo] as ONE N = 64 MMA (the two Z tiles sit next to each
      // other: 64 K-major rows), A_lo x Z_hi as an N = 32 MMA into the first
      // half: A is read from shared memory twice per K-step instead of three times
      const uint32_t idesc64 = idesc_tf32(128, 64);
      const uint32_t idesc = idesc_tf32(128, 32);
      for (int64_t t = 0; t < my_tiles; ++t) {
        const int acc = (int)(t & 1);
        mbar_wait(&tempty[acc], (uint32_t)(((t >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * 64);
        for (int kk = 0; kk < kt; ++kk) {
          const int64_t it = t * kt + kk;
          const int st = (int)(it % kPwStages);
          const int ls = (int)(it % kPwLo);
          const uint32_t sa = sbase + (uint32_t)(st * kPwStageBytes);
          const uint64_t dA = umma_desc_sw128(sa);
          const uint64_t dZh = umma_desc_sw128(sa + kPjTileBytes);
          mbar_wait(&full[st], (uint32_t)((it / kPwStages) & 1));
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // K = 8 per MMA: +32 B in the swizzled row
            const uint64_t adv = (uint64_t)(2 * k);
            umma_tf32(d, dA + adv, dZh + adv, idesc64, (kk == 0 && k == 0) ? 0u : 1u);
          }
          mbar_wait(&lo_ready[ls], (uint32_t)((it / kPwLo) & 1));
          tc_fence_after();
          const uint32_t ta = tmem + (uint32_t)(kPwTmemLo + 32 * ls);
#pragma unroll
          for (int k = 0; k < 4; ++k)  // K = 8 per MMA: 8 TMEM columns of A_lo
            umma_tf32_ts(tmem + (uint32_t)(kPwTmemAccLo + 32 * acc), ta + (uint32_t)(8 * k),
                         dZh + (uint64_t)(2 * k), idesc, (kk == 0 && k == 0) ? 0u : 1u);
          umma_commit(&empty[st]);
          umma_commit(&lo_empty[ls]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp < 10) {  // ---- A_lo split into tensor memory ----
    // this warp may touch TMEM lanes 32 (warp % 4) ..: thread = tile row (M index).
    // Two warps per lane quarter take alternate K-steps: the chain of one step
    // (wait, 8 LDS.128, split, tcgen05.st + wait::st, arrive) is longer than
    // the step's share of the HBM stream.
    const int row = 32 * (warp & 3) + lane;
    for (int64_t it = (warp - 2) >> 2; it < iters; it += 2) {
      const int st = (int)(it % kPwStages);
      const int ls = (int)(it % kPwLo);
      mbar_wait(&lo_empty[ls], (uint32_t)(((it / kPwLo) & 1) ^ 1));
      mbar_wait(&full[st], (uint32_t)((it / kPwStages) & 1));
      tc_fence_after();
      // row `row` of the 128B-swizzled tile: 16-byte chunk c sits at c ^ (row & 7)
      const unsigned char* sp = smem + st * kPwStageBytes + row * 128;
      uint32_t lo[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 a = *reinterpret_cast<const float4*>(sp + ((c ^ (row & 7)) << 4));
        lo[4 * c + 0] = __float_as_uint(a.x - __uint_as_float(__float_as_uint(a.x) & 0xFFFFE000u));
        lo[4 * c + 1] = __float_as_uint(a.y - __uint_as_float(__float_as_uint(a.y) & 0xFFFFE000u));
        lo[4 * c + 2] = __float_as_uint(a.z - __uint_as_float(__float_as_uint(a.z) & 0xFFFFE000u));
        lo[4 * c + 3] = __float_as_uint(a.w - __uint_as_float(__float_as_uint(a.w) & 0xFFFFE000u));
      }
      tmem_st32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(kPwTmemLo + 32 * ls), lo);
      tc_fence_before();
      mbar_arrive(&lo_ready[ls]);
    }
  } else {  // ---- epilogue: TMEM lane quarter (warp % 4) ----
    __shared__ float wt[128][33];
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const int et = threadIdx.x - 320;  // 0..127: Gram entries et + 128 u
    double g[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) g[u] = 0.0;
    for (int64_t t = 0; t < my_tiles; ++t) {
      const int acc = (int)(t & 1);
      mbar_wait(&tfull[acc], (uint32_t)((t >> 1) & 1));
      tc_fence_after();
      float w[32], wl[32];
      tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * 64), w);
      tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * 64 + 32), wl);
#pragma unroll
      for (int j = 0; j < 32; ++j) w[j] += wl[j];  // A Z_hi + A Z_lo
      tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(kPwTmemAccLo + 32 * acc), wl);
#pragma unroll
      for (int j = 0; j < 32; ++j) w[j] += wl[j];  // + A_lo Z_hi
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      const int64_t col = (blockIdx.x + t * gridDim.x) * 128 + row;
      if (col < n) {
        float* dst = W + col * ldw;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < s) dst[j] = w[j];
      }
      if (part == nullptr) continue;  // column block of a wider W: Gram formed afterwards
      asm volatile("bar.sync 1, 128;" ::: "memory");  // previous tile's Gram reads done
#pragma unroll
      for (int j = 0; j < 32; ++j) wt[row][j] = col < n ? w[j] : 0.f;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int r = 0; r < 128; ++r) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = et + 128 * u;
          g[u] += (double)wt[r][e >> 5] * (double)wt[r][e & 31];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = et + 128 * u, j = e >> 5, k = e & 31;
      if (part != nullptr && j < s && k < s) part[(int64_t)blockIdx.x * s * s + j * s + k] = g[u];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kPwTmemCols));
  }
}

}  // namespace tr
