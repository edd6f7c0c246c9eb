// Re-expansion GEMM of the randomized t-SVT on the 5th-generation tensor cores:
//   out (n1 x N, column-major) = F0 (n1 x K) * C1 (K x N),  K = r0 <= 32
// (TuckerFactors.reconstruct along mode 0, tenrec/sketch.py:45-53; N = n2 * faces).
//
// K is tiny (25 on the bench), so the CUDA-core kernel (k_gemm_expand) is FFMA
// issue-bound at ~1/3 of the HBM write rate.  Here every 128 x 128 output tile
// costs 8 tcgen05.mma (3xTF32, fp32-faithful) and the pass is bound by the
// 4 B-per-element output write:
//   * F0 and C1 are stored K-major, K padded to 32 floats (one 128-byte
//     swizzle atom per row), split into tf32 high / low parts by their
//     producers (k_split_rows, k_expand_mode1<.., true>);
//   * warp 0: TMA producer -- the CTA's 128 rows of F0 (hi, lo) once, then C1
//     tiles (128 columns x 32 K, hi and lo adjacent = one 256-row B operand)
//     into a kEtStages-deep ring;
//   * warp 1: one thread issues, per K = 8 step, A_hi C1_hi + A_hi C1_lo +
//     A_lo C1_hi (M = 128, N = 128) into a double-buffered TMEM accumulator
//     (2 x 128 columns);
//   * warps 2-17: epilogue -- one tcgen05.ld of 32 columns per warp (lane
//     quarter x column quarter), the accumulator released at once, then coalesced
//     stores (each warp instruction writes 32 consecutive rows of a column).
// CTA i works on row block i % (n1 / 128) and strides over column tiles, so the
// CTAs of one column tile run together and C1 tiles are re-read from L2.
#pragma once

#include "proj_tc.cuh"

namespace tr {

// 64 consecutive fp32 TMEM columns of this thread's lane (one wait)
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&v)[64]) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]),
        "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]),
        "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),
        "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]),
        "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

constexpr int kEtStages = 5;        // C1 ring depth (direct-store epilogue)
constexpr int kEtStagesTs = 3;      // C1 ring depth next to the TMA-store staging
constexpr int kEtEpiWarps = 16;  // 4 per TMEM lane quarter, 128 / 4 columns each
constexpr int kEtThreads = 64 + 32 * kEtEpiWarps;  // producer, MMA, epilogue warps
constexpr int kEtABytes = 128 * 128;          // 128 rows x 32 fp32
constexpr int kEtStageBytes = 2 * 128 * 128;  // C1_hi + C1_lo tile
constexpr int kEtSmemBytes = 2 * kEtABytes + kEtStages * kEtStageBytes;
// TMA-store variant: 3 ring stages + one 32 x 32 fp32 staging box per epilogue warp
constexpr int kEtSmemBytesTs = 2 * kEtABytes + kEtStagesTs * kEtStageBytes + kEtEpiWarps * 4096;

// rows (K-major, 32-float rows): hi[r * 32 + k] = tf32(x), lo = x - hi, for the
// n x K fp64 column-major factor F (zero for k >= K)
__global__ void k_split_rows(const double* __restrict__ F, int64_t n, int K,
                             float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * 32) return;
  const int64_t r = e >> 5;
  const int k = (int)(e & 31);
  const double x = k < K ? F[r + n * k] : 0.0;
  const float h = __uint_as_float(__float_as_uint((float)x) & 0xFFFFE000u);
  hi[e] = h;
  lo[e] = (float)(x - (double)h);
}

// C1 = core x_1 F1 (as k_expand_mode1), written K-major with K padded to 32
// and split into tf32 hi / lo: hi[a + 32 (i2 + n2 f)], zero for a >= r0.
__global__ void __launch_bounds__(128) k_expand_mode1_split(const double* __restrict__ core,
                                                            int r0, int r1, int64_t nf,
                                                            const double* __restrict__ F1,
                                                            int64_t n2, float* __restrict__ hi,
                                                            float* __restrict__ lo) {
  __shared__ double cs[32 * 64];
  const int64_t tiles = (n2 + 127) / 128;
  const int64_t f = blockIdx.x / tiles;
  const int64_t i2 = (blockIdx.x % tiles) * 128 + threadIdx.x;
  for (int e = threadIdx.x; e < r0 * r1; e += blockDim.x) cs[e] = core[e + (int64_t)r0 * r1 * f];
  __syncthreads();
  if (i2 >= n2 || f >= nf) return;
  double acc[32];
#pragma unroll
  for (int a = 0; a < 32; ++a) acc[a] = 0.0;
  for (int b = 0; b < r1; ++b) {
    const double fv = F1[i2 + n2 * b];
#pragma unroll
    for (int a = 0; a < 32; ++a)
      if (a < r0) acc[a] += cs[a + r0 * b] * fv;
  }
  float4* h4 = reinterpret_cast<float4*>(hi + 32 * (i2 + n2 * f));
  float4* l4 = reinterpret_cast<float4*>(lo + 32 * (i2 + n2 * f));
#pragma unroll
  for (int a = 0; a < 32; a += 4) {
    float hv[4], lv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double x = acc[a + u];
      hv[u] = __uint_as_float(__float_as_uint((float)x) & 0xFFFFE000u);
      lv[u] = (float)(x - (double)hv[u]);
    }
    h4[a / 4] = make_float4(hv[0], hv[1], hv[2], hv[3]);
    l4[a / 4] = make_float4(lv[0], lv[1], lv[2], lv[3]);
  }
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          (uint64_t)map),
      "r"(c0), "r"(c1), "r"(src)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// TS: the epilogue stages each warp's 32 x 32 block in shared memory and
// writes it with a TMA tensor store (mapOut: out, n1 x N, box 32 x 32);
// otherwise direct coalesced st.global.
template <bool TS>
__global__ void __launch_bounds__(kEtThreads, 1)
    k_expand_tc(const __grid_constant__ CUtensorMap mapAh, const __grid_constant__ CUtensorMap mapAl,
                const __grid_constant__ CUtensorMap mapBh, const __grid_constant__ CUtensorMap mapBl,
                const __grid_constant__ CUtensorMap mapOut, int64_t n1, int64_t N,
                float* __restrict__ out) {
  constexpr int NST = TS ? kEtStagesTs : kEtStages;
  extern __shared__ __align__(1024) unsigned char et_raw[];
  __shared__ __align__(8) uint64_t full[NST], empty[NST], abar;
  __shared__ __align__(8) uint64_t tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_s;
  unsigned char* smem = (unsigned char*)(((uintptr_t)et_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sAh = sbase, sAl = sbase + kEtABytes, sB = sbase + 2 * kEtABytes;
  (void)out;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nrb = (int)(n1 / 128);
  const int rb = (int)(blockIdx.x % nrb);
  const int64_t cstride = gridDim.x / nrb;  // CTAs per row block (host: grid % nrb == 0)
  const int64_t c0 = blockIdx.x / nrb;
  const int64_t ntc = (N + 127) / 128;
  const int64_t my_tiles = ntc > c0 ? (ntc - 1 - c0) / cstride + 1 : 0;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&abar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kEtEpiWarps);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      mbar_arrive_expect_tx(&abar, 2 * kEtABytes);
      tma_load_2d(sAh, &mapAh, 0, rb * 128, &abar);
      tma_load_2d(sAl, &mapAl, 0, rb * 128, &abar);
      for (int64_t t = 0; t < my_tiles; ++t) {
        const int st = (int)(t % NST);
        const uint32_t ph = (uint32_t)((t / NST) & 1);
        mbar_wait(&empty[st], ph ^ 1);
        const int col = (int)((c0 + t * cstride) * 128);
        const uint32_t sb = sB + (uint32_t)(st * kEtStageBytes);
        mbar_arrive_expect_tx(&full[st], kEtStageBytes);
        tma_load_2d(sb, &mapBh, 0, col, &full[st]);
        tma_load_2d(sb + kEtStageBytes / 2, &mapBl, 0, col, &full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      const uint32_t idesc128 = idesc_tf32(128, 128);
      mbar_wait(&abar, 0);
      tc_fence_after();
      const uint64_t dAh = umma_desc_sw128(sAh), dAl = umma_desc_sw128(sAl);
      for (int64_t t = 0; t < my_tiles; ++t) {
        const int acc = (int)(t & 1);
        const int st = (int)(t % NST);
        mbar_wait(&tempty[acc], (uint32_t)(((t >> 1) & 1) ^ 1));
        mbar_wait(&full[st], (uint32_t)((t / NST) & 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * 128);
        const uint64_t dBh = umma_desc_sw128(sB + (uint32_t)(st * kEtStageBytes));
        const uint64_t dBl = umma_desc_sw128(sB + (uint32_t)(st * kEtStageBytes + kEtStageBytes / 2));
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // K = 8 per MMA: +32 B in the swizzled row
          const uint64_t adv = (uint64_t)(2 * k);
          // 3xTF32 into one accumulator: A_hi B_hi + A_hi B_lo + A_lo B_hi
          umma_tf32(d, dAh + adv, dBh + adv, idesc128, k == 0 ? 0u : 1u);
          umma_tf32(d, dAh + adv, dBl + adv, idesc128, 1u);
          umma_tf32(d, dAl + adv, dBh + adv, idesc128, 1u);
        }
        umma_commit(&empty[st]);
        umma_commit(&tfull[acc]);
      }
    }
  } else {  // ---- epilogue: TMEM lane quarter (warp % 4) = 32 rows, 32 columns per warp ----
    constexpr int CW = 128 / (kEtEpiWarps / 4);
    const int q = warp & 3, part = (warp - 2) >> 2;
    const int64_t row = (int64_t)rb * 128 + 32 * q + lane;
    for (int64_t t = 0; t < my_tiles; ++t) {
      const int acc = (int)(t & 1);
      mbar_wait(&tfull[acc], (uint32_t)((t >> 1) & 1));
      tc_fence_after();
      const int64_t col0 = (c0 + t * cstride) * 128 + CW * part;
      float a[CW];
      tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * 128 + CW * part), a);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);  // the accumulator is in registers: free it early
      if (TS) {
        // this warp's box: rows 32 q .. of the row block, columns col0 .. col0 + 31
        float* box = reinterpret_cast<float*>(smem + 2 * kEtABytes + NST * kEtStageBytes) +
                     (warp - 2) * 1024;
        if (lane == 0) tma_store_wait_read();  // the previous tile's store has read the box
        __syncwarp();
#pragma unroll
        for (int j = 0; j < CW; ++j) box[j * 32 + lane] = a[j];
        fence_async_smem();
        __syncwarp();
        if (lane == 0)
          tma_store_2d(&mapOut, smem_u32(box), (int)(rb * 128 + 32 * q), (int)col0);
      } else if (row < n1) {
        float* o = out + row + n1 * col0;
#pragma unroll
        for (int j = 0; j < CW; ++j)
          if (col0 + j < N) o[n1 * j] = a[j];
      }
    }
    if (TS && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

}  // namespace tr
