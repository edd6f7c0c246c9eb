// Krylov streaming passes over a tall fp32 unfolding A (m x n, column-major)
// on the tensor cores, 3xTF32 (fp32-faithful), for tenrec/sketch.py:253-259:
//
//   MODE 0 (sketch):  Y = A G          (G: Philox Gaussian sketch rows)
//   MODE 1 (gram):    Y = A (A^T P)    (one power of A A^T in ONE pass over A)
//
// Why this shape.  Per streamed element the pass does 2b (sketch) or 4b (gram)
// flops with b = 7..8, i.e. 7-14 flop/byte: on the CUDA cores the A^T P half
// needs a 256-thread reduction per column and the old kernel (panel.cuh) ran
// issue-bound at IPC ~2 (2.5 TB/s).  Both halves are skinny products whose
// reduction dimension the tensor core does for free, so each warp issues
// warp-level m16n8k8 TF32 MMAs, which leaves the pass HBM-bound.  tcgen05 is
// not used here: its minimum M of 64 needs a whole m x 64-column chunk (and its
// A_lo twin) resident for both products, which does not fit next to a TMA ring
// for m = 1024, and at this arithmetic intensity the warp-level path's
// 0.45 MMA/clk/SM (tools/mma_probe.cu) already exceeds what HBM can feed.
//
// Structure (persistent, one CTA per SM, 16 compute warps + 2 helpers):
//   * producer warp: chunks of 8 columns land in a 6-deep ring by the bulk
//     copy engine (one cp.async.bulk per column into a slot of S = m' + 8
//     floats, S = 8 mod 32: every fragment load below is conflict-free);
//   * compute warp w owns rows [32 RG w, 32 RG (w+1)); its P fragments (hi/lo)
//     and its rows of Y stay in registers for the whole pass;
//   * step 1 (gram): D (16 x 8) = [P_hi; P_lo]^T (rows) x A_chunk (rows x 8
//     columns), 2 MMAs per 8-row step (A_hi and A_lo); T partial = D_hi + D_lo
//     in-lane; per-warp partials -> smem;
//   * reducer warp: T = sum of the 16 partials in a fixed order
//     (deterministic), split into T_hi / T_lo;
//   * step 2: Y_rows += A_rows,chunk T (M = 16 rows, K = 8 columns), 3 MMAs;
//   * the compute warps run step 1 of chunk i before step 2 of chunk i-1, so
//     the reduction overlaps the MMAs; all hand-offs are mbarriers (no CTA
//     barrier in the loop).  Sketch mode: T = the chunk's sketch rows,
//     precomputed by k_sketch_rows and bulk-copied next to the chunk.
// The streamed operand is split by truncation (hi = tf32 bits, exact lo = A -
// hi; 2 ALU ops), the small operands by round-to-nearest.
// Per-CTA results go to `partial` (m x b, fp64), reduced afterwards.
#pragma once

#include "proj_tc.cuh"

namespace tr {

constexpr int kPmCols = 8;   // columns per chunk (= N of step 1, K of step 2)
constexpr int kPmWarps = 16;  // compute warps
constexpr int kPmThreads = (kPmWarps + 2) * 32;  // + reducer + producer
constexpr int kPmMaxStages = 8;
constexpr int kPmTE = kPmCols * 8;  // T entries per chunk (8 columns x 8 sketch columns)
constexpr int kPmRS = kPmTE + 8;    // per-warp partial stride

__device__ __forceinline__ uint32_t f2tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// x = hi + lo with hi a tf32 value (round to nearest); lo keeps fp32 bits
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = f2tf32(x);
  lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32_16x8x8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// d += A B in 3xTF32: A_hi B_hi + A_hi B_lo + A_lo B_hi
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                     uint32_t bh0, uint32_t bh1, uint32_t bl0, uint32_t bl1) {
  mma_tf32_16x8x8(d, al[0], al[1], al[2], al[3], bh0, bh1);
  mma_tf32_16x8x8(d, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
  mma_tf32_16x8x8(d, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
}

__device__ __forceinline__ void fence_async_smem_pm() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// x = hi + lo by truncation: hi keeps the tf32 bits, lo = x - hi is exact
__device__ __forceinline__ void split_trunc(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xFFFFE000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}

// mbarrier wait / arrive on a precomputed shared-window address (the generic ->
// shared conversion of a barrier pointer costs an S2UR + two address ops at
// every use; the compute-warp loop does ~7 barrier operations per chunk)
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t phase) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

struct PanelMmaArgs {
  int64_t m, n;
  int b;
  int S;    // column slot stride in floats (round_up(m, 32) + 8)
  int nst;  // ring depth
  int64_t nchunks;
  // sketch columns [j0, j0 + b) of a block of b_all: both products are
  // column-separable (Y_j = A G_j, Y_j = A (A^T P_j)), so a block wider than
  // the 8-column MMA tile runs as several passes writing their columns of the
  // per-CTA partial (stride b_all * m)
  int j0 = 0, b_all = 0;
};

// slot covers every row a compute warp touches (rows >= m stay zero), S = 8 mod 32
__host__ __device__ constexpr int panel_mma_slot(int64_t m) {
  return (int)(m <= 512 ? 512 + 8 : 1024 + 8);
}

// rows[c * b + j] = sketch entry (c, j) of physical column c (logical-column
// remap, override or Philox), zero for c >= n (up to the chunk pad)
// (columns [j0, j0 + b) of a sketch of b_all columns; rows[c * b + j])
// One thread per column: the column's b entries are consecutive Philox indices
// cl * b_all + j0 .. + b - 1, so neighbouring entries share a Box-Muller pair
// (gauss_pair yields indices 2 p and 2 p + 1 at once) -- about half the
// Philox / log / sincos evaluations of one gauss_at per entry -- and the
// logical-column remap costs two divisions per column instead of four per entry.
__global__ void k_sketch_rows(int64_t n, int b, SketchSpec sk, const float* __restrict__ gover,
                              float* __restrict__ rows, int j0, int b_all) {
  const int64_t npad = (n + kPmCols - 1) / kPmCols * kPmCols;
  const int64_t eff = sk.inner_eff ? *sk.inner_eff : sk.inner;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < npad;
       c += (int64_t)gridDim.x * blockDim.x) {
    float* out = rows + c * b;
    bool live = false;
    int64_t cl = 0;
    if (c < n) {
      const int64_t col = c + sk.col0;  // global column
      int64_t lo, f;
      if (((col | sk.inner) >> 31) == 0) {
        const uint32_t q = (uint32_t)col / (uint32_t)sk.inner;
        f = q;
        lo = (uint32_t)col - q * (uint32_t)sk.inner;
      } else {
        f = col / sk.inner;
        lo = col - f * sk.inner;
      }
      live = lo < eff;
      cl = lo + eff * f;
    }
    if (!live) {
      for (int j = 0; j < b; ++j) out[j] = 0.f;
      continue;
    }
    const uint64_t i0 = (uint64_t)(cl * b_all + j0);
    if (gover) {
      for (int j = 0; j < b; ++j) out[j] = gover[i0 + j];
      continue;
    }
    uint64_t have = ~0ull;  // pair index held in (z0, z1)
    double z0 = 0.0, z1 = 0.0;
    for (int j = 0; j < b; ++j) {
      const uint64_t idx = i0 + j, pr = idx >> 1;
      if (pr != have) {
        gauss_pair(sk.seed, sk.stream, pr, z0, z1);
        have = pr;
      }
      out[j] = (float)((idx & 1) ? z1 : z0);
    }
  }
}

// Step 1 of one chunk (S1: As1) and step 2 of an older chunk (S2: As2) in
// one instruction stream: per 32-row group the fragment loads come first, then
// the MMAs alternate between the 4 step-1 chains (hi / lo x step parity) and
// the 2 step-2 tiles so no MMA waits on the one just before it.
template <int RG, bool S1, bool S2>
__device__ __forceinline__ void panel_fused(const float* __restrict__ As1,
                                            const float* __restrict__ As2, int S, int rw0, int g,
                                            int t, const uint32_t (&pf)[RG][4][4],
                                            float (&d)[4][4], float (&y)[RG][2][4],
                                            const uint32_t (&bh)[2], const uint32_t (&bl)[2]) {
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    const int rb = rw0 + 32 * rg;
    uint32_t h1[4][2], l1[4][2];  // step 1: column g, rows 2t / 2t+1 of step ks
    uint32_t h2[2][4], l2[2][4];  // step 2: tile tl fragment a0..a3
    if (S1) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const float2 x = *reinterpret_cast<const float2*>(As1 + g * S + rb + 8 * ks + 2 * t);
        split_trunc(x.x, h1[ks][0], l1[ks][0]);
        split_trunc(x.y, h1[ks][1], l1[ks][1]);
      }
    }
    if (S2) {
#pragma unroll
      for (int tl = 0; tl < 2; ++tl) {
        const int r0 = rb + 16 * tl + 2 * g;  // fragment rows g / g+8 = rows r0 / r0+1
        const float2 x0 = *reinterpret_cast<const float2*>(As2 + t * S + r0);
        const float2 x1 = *reinterpret_cast<const float2*>(As2 + (t + 4) * S + r0);
        split_trunc(x0.x, h2[tl][0], l2[tl][0]);
        split_trunc(x0.y, h2[tl][1], l2[tl][1]);
        split_trunc(x1.x, h2[tl][2], l2[tl][2]);
        split_trunc(x1.y, h2[tl][3], l2[tl][3]);
      }
    }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const uint32_t(&a)[4] = pf[rg][ks];
      if (S1) mma_tf32_16x8x8(d[2 * (ks & 1)], a[0], a[1], a[2], a[3], h1[ks][0], h1[ks][1]);
#pragma unroll
      for (int tl = 0; tl < 2; ++tl) {
        if (S2 && ks == 0)  // A_lo T_hi
          mma_tf32_16x8x8(y[rg][tl], l2[tl][0], l2[tl][1], l2[tl][2], l2[tl][3], bh[0], bh[1]);
        if (S2 && ks == 1)  // A_hi T_lo
          mma_tf32_16x8x8(y[rg][tl], h2[tl][0], h2[tl][1], h2[tl][2], h2[tl][3], bl[0], bl[1]);
        if (S2 && ks == 2)  // A_hi T_hi
          mma_tf32_16x8x8(y[rg][tl], h2[tl][0], h2[tl][1], h2[tl][2], h2[tl][3], bh[0], bh[1]);
        if (S1 && tl == 0)
          mma_tf32_16x8x8(d[2 * (ks & 1) + 1], a[0], a[1], a[2], a[3], l1[ks][0], l1[ks][1]);
      }
    }
  }
}

__device__ __forceinline__ uint32_t pm_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// shared::cluster address of `p` (a local shared variable) in CTA `rank`
__device__ __forceinline__ uint32_t pm_mapa(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}

__device__ __forceinline__ void pm_st_cluster(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

__device__ __forceinline__ void pm_arrive_remote(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   bar_cluster_addr)
               : "memory");
}

__device__ __forceinline__ void pm_wait_cluster(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
}

// RG = 32-row groups per compute warp (m <= 512 RG); b <= 8.
// MODE 0: `coef` = k_sketch_rows output; MODE 1: P (m x b column-major).
// CL = 2: the rows are split over a 2-CTA cluster (m <= 2048; each CTA streams
// its half of every column chunk); in the gram mode the two halves of each
// chunk's T partial are exchanged through distributed shared memory and
// summed in CTA order on both sides, so T -- and Y -- are bit-identical to a
// single CTA's fixed-order sum of the same warps.
template <int RG, int MODE, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kPmThreads, 1)
    k_panel_mma(const float* __restrict__ A, const float* __restrict__ P,
                const float* __restrict__ coef, PanelMmaArgs pa, double* __restrict__ partial) {
  extern __shared__ __align__(128) unsigned char pm_smem[];
  __shared__ __align__(8) uint64_t full[kPmMaxStages], empty[kPmMaxStages];
  __shared__ __align__(8) uint64_t redfull[2], redempty[2], tready[2], tempty[2];
  __shared__ __align__(8) uint64_t xfull[2], xempty[2];  // CL = 2: the peer's T partial
  __shared__ float xbuf[2][kPmTE];
  const uint32_t crank = CL > 1 ? pm_cluster_rank() : 0u;
  const int S = pa.S;
  const int64_t mfull = pa.m;  // rows of A, P, Y
  // this CTA's rows [mrow0, mrow0 + m): the first half rounded to 4 (16-byte copies)
  const int64_t mh = CL > 1 ? ((pa.m + 1) / 2 + 3) / 4 * 4 : pa.m;
  const int64_t mrow0 = crank == 0 ? 0 : mh;
  const int64_t m = crank == 0 ? mh : pa.m - mh;
  const int b = pa.b;
  const int nst = pa.nst;
  const size_t stage_elems = (size_t)kPmCols * S;
  float* stages = reinterpret_cast<float*>(pm_smem);
  float* cst = stages + nst * stage_elems;  // MODE 0: nst x (8 x b) sketch rows
  float* red = cst;                         // MODE 1: 2 x kPmWarps x kPmRS partials
  float* thi = red + 2 * kPmWarps * kPmRS;  // MODE 1: 2 x kPmTE
  float* tlo = thi + 2 * kPmTE;             // MODE 1: 2 x kPmTE
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t G = gridDim.x / CL;        // clusters (one chunk sequence each)
  const int64_t cid = blockIdx.x / CL;
  const int64_t my_chunks = pa.nchunks > cid ? (pa.nchunks - 1 - cid) / G + 1 : 0;

  // zeroed ring: padding rows and the absent columns of a partial chunk stay finite
  {
    float4* z = reinterpret_cast<float4*>(stages);
    const size_t n4 = nst * stage_elems / 4;
    for (size_t e = tid; e < n4; e += kPmThreads) z[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  fence_async_smem_pm();
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPmWarps * 32);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&redfull[k], kPmWarps * 32);
      mbar_init(&redempty[k], 32);
      mbar_init(&tready[k], 32);
      mbar_init(&tempty[k], kPmWarps * 32);
      mbar_init(&xfull[k], 32);
      mbar_init(&xempty[k], 32);
    }
    fence_barrier_init();
  }
  if (CL > 1) {
    // every CTA's barriers exist before the peer's first remote arrive
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
  } else {
    __syncthreads();
  }

  if (warp == kPmWarps + 1) {  // ---- producer (one thread; no divisions in the loop) ----
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(m * sizeof(float));
      const uint32_t cbytes = (uint32_t)(kPmCols * b * sizeof(float));
      const int64_t cstep = G * kPmCols;
      int64_t c0 = cid * kPmCols;
      const float* src = A + c0 * mfull + mrow0;
      int s = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it < my_chunks; ++it) {
        mbar_wait(&empty[s], ph ^ 1u);
        const int cols = (int)((pa.n - c0) < kPmCols ? (pa.n - c0) : kPmCols);
        mbar_arrive_expect_tx(&full[s], bytes * (uint32_t)cols + (MODE == 0 ? cbytes : 0u));
        float* dst = stages + s * stage_elems;
        if (cols == kPmCols) {
#pragma unroll
          for (int c = 0; c < kPmCols; ++c) bulk_g2s(dst + c * S, src + c * mfull, bytes, &full[s]);
        } else {
          for (int c = 0; c < cols; ++c) bulk_g2s(dst + c * S, src + c * mfull, bytes, &full[s]);
        }
        if (MODE == 0) bulk_g2s(cst + s * kPmCols * b, coef + c0 * b, cbytes, &full[s]);
        c0 += cstep;
        src += cstep * mfull;
        if (++s == nst) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp == kPmWarps) {  // ---- reducer (gram) ----
    if (MODE == 1) {
      const uint32_t peer = crank ^ 1u;
      for (int64_t it = 0; it < my_chunks; ++it) {
        const int k = (int)(it & 1);
        const uint32_t ph = (uint32_t)((it >> 1) & 1);
        const int64_t c0 = (cid + it * G) * kPmCols;
        const int cols = (int)((pa.n - c0) < kPmCols ? (pa.n - c0) : kPmCols);
        mbar_wait(&redfull[k], ph);
        mbar_wait(&tempty[k], ph ^ 1);
        const float* rk = red + k * kPmWarps * kPmRS;
        float v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = lane + 32 * h;  // e = j * 8 + column
          float x = 0.f;
#pragma unroll
          for (int w = 0; w < kPmWarps; ++w) x += rk[w * kPmRS + e];
          v[h] = x;
        }
        if (CL > 1) {
          // this half's partial -> the peer's xbuf[k]; the peer's -> ours; sum in CTA order
          pm_wait_cluster(&xempty[k], ph ^ 1);  // the peer has consumed its xbuf[k]
#pragma unroll
          for (int h = 0; h < 2; ++h) pm_st_cluster(pm_mapa(&xbuf[k][lane + 32 * h], peer), v[h]);
          pm_arrive_remote(pm_mapa(&xfull[k], peer));
          pm_wait_cluster(&xfull[k], ph);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float o = xbuf[k][lane + 32 * h];
            v[h] = crank == 0 ? v[h] + o : o + v[h];
          }
          pm_arrive_remote(pm_mapa(&xempty[k], peer));  // our xbuf[k] may be refilled
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = lane + 32 * h;
          float x = v[h];
          if ((e & 7) >= cols || (e >> 3) >= b) x = 0.f;
          const uint32_t hv = f2tf32(x);
          thi[k * kPmTE + e] = __uint_as_float(hv);
          tlo[k * kPmTE + e] = x - __uint_as_float(hv);
        }
        mbar_arrive(&redempty[k]);
        mbar_arrive(&tready[k]);
      }
    }
  } else {
    // ---- compute warps ----
    // step-1 A operand = [P_hi; P_lo]^T: a0 / a2 = P_hi (sketch column g) at rows
    // 2t / 2t+1 of the 8-row step, a1 / a3 = P_lo
    uint32_t pf[RG][4][4];
#pragma unroll
    for (int rg = 0; rg < RG; ++rg)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t r = 32 * (warp * RG + rg) + 8 * ks + 2 * t + h;
          const float p = (MODE == 1 && r < m && g < b) ? P[mrow0 + r + mfull * g] : 0.f;
          split_tf32(p, pf[rg][ks][2 * h], pf[rg][ks][2 * h + 1]);
        }
    float y[RG][2][4];
#pragma unroll
    for (int rg = 0; rg < RG; ++rg)
#pragma unroll
      for (int tl = 0; tl < 2; ++tl)
#pragma unroll
        for (int i = 0; i < 4; ++i) y[rg][tl][i] = 0.f;
    const int rw0 = 32 * RG * warp;  // first row of this warp (rows >= m read zero padding)

    // stage / phase of chunk `it` and of chunk it-2 (step 2 lags two chunks).
    // Everything the loop addresses is a precomputed shared-window offset, the
    // counters are 32-bit (a CTA's chunk count is far below 2^31).
    int s_cur = 0, s_old = 0;
    uint32_t ph_cur = 0;
    const uint32_t zero2[2] = {0u, 0u};
    const uint32_t full_a = smem_u32(&full[0]), empty_a = smem_u32(&empty[0]);
    const uint32_t redfull_a = smem_u32(&redfull[0]), redempty_a = smem_u32(&redempty[0]);
    const uint32_t tready_a = smem_u32(&tready[0]), tempty_a = smem_u32(&tempty[0]);
    const int nch = (int)my_chunks;
    const int nit = nch + (MODE == 1 ? 2 : 0);
    const int te0 = g * 8 + t;  // T[column t][sketch column g]
    float* const rw_base = red + warp * kPmRS + g * 8 + 2 * t;
    for (int it = 0; it < nit; ++it) {
      const bool has1 = it < nch;              // chunk it: step 1 (gram) / step 2 (sketch)
      const bool has2 = MODE == 1 && it >= 2;  // chunk it-2: step 2 (gram)
      const int kb = it & 1;
      if (has1) mbar_wait_a(full_a + 8u * (uint32_t)s_cur, ph_cur);
      const float* As1 = stages + s_cur * stage_elems;
      uint32_t bh[2], bl[2];
      if (MODE == 1) {
        if (has2) {
          mbar_wait_a(tready_a + 8u * (uint32_t)kb, (uint32_t)(((it - 2) >> 1) & 1));
          const float* th = thi + kb * kPmTE + te0;
          const float* tl = tlo + kb * kPmTE + te0;
          bh[0] = __float_as_uint(th[0]);
          bh[1] = __float_as_uint(th[4]);
          bl[0] = __float_as_uint(tl[0]);
          bl[1] = __float_as_uint(tl[4]);
          mbar_arrive_a(tempty_a + 8u * (uint32_t)kb);
        }
        float d[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int i = 0; i < 4; ++i) d[u][i] = 0.f;
        const float* As2 = stages + s_old * stage_elems;
        if (has1 && has2)
          panel_fused<RG, true, true>(As1, As2, S, rw0, g, t, pf, d, y, bh, bl);
        else if (has1)
          panel_fused<RG, true, false>(As1, As2, S, rw0, g, t, pf, d, y, zero2, zero2);
        else if (has2)  // (neither: a one-chunk CTA between its step 1 and its step 2)
          panel_fused<RG, false, true>(As1, As2, S, rw0, g, t, pf, d, y, bh, bl);
        if (has2) {
          mbar_arrive_a(empty_a + 8u * (uint32_t)s_old);
          s_old = s_old + 1 == nst ? 0 : s_old + 1;
        }
        if (has1) {
          // d[0..1] rows g (P_hi), d[2..3] rows g+8 (P_lo): T partial (sketch column g, columns 2t / 2t+1)
          mbar_wait_a(redempty_a + 8u * (uint32_t)kb, (uint32_t)(((it >> 1) & 1) ^ 1));
          *reinterpret_cast<float2*>(rw_base + kb * (kPmWarps * kPmRS)) =
              make_float2(((d[0][0] + d[1][0]) + (d[2][0] + d[3][0])) +
                              ((d[0][2] + d[1][2]) + (d[2][2] + d[3][2])),
                          ((d[0][1] + d[1][1]) + (d[2][1] + d[3][1])) +
                              ((d[0][3] + d[1][3]) + (d[2][3] + d[3][3])));
          mbar_arrive_a(redfull_a + 8u * (uint32_t)kb);
        }
      } else {
        const float* cr = cst + s_cur * kPmCols * b;
        const float v0 = g < b ? cr[t * b + g] : 0.f;
        const float v1 = g < b ? cr[(t + 4) * b + g] : 0.f;
        split_tf32(v0, bh[0], bl[0]);
        split_tf32(v1, bh[1], bl[1]);
        float d[4][4];
        panel_fused<RG, false, true>(As1, As1, S, rw0, g, t, pf, d, y, bh, bl);
        mbar_arrive_a(empty_a + 8u * (uint32_t)s_cur);
      }
      if (has1) {
        s_cur = s_cur + 1 == nst ? 0 : s_cur + 1;
        ph_cur ^= s_cur == 0 ? 1u : 0u;
      }
    }

    // y: (row r0, sketch column 2t / 2t+1), (row r0+1, ...); the partial of a
    // cluster covers all mfull rows (each CTA its own)
    double* out = partial + cid * pa.b_all * mfull + (int64_t)pa.j0 * mfull + mrow0;
#pragma unroll
    for (int rg = 0; rg < RG; ++rg)
#pragma unroll
      for (int tl = 0; tl < 2; ++tl)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t row = 32 * (warp * RG + rg) + 16 * tl + 2 * g + (i >> 1);
          const int j = 2 * t + (i & 1);
          if (row < m && j < b) out[(int64_t)j * mfull + row] = (double)y[rg][tl][i];
        }
  }
  if (CL > 1) {
    // no CTA leaves while its peer may still arrive on its barriers
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
  }
}

}  // namespace tr
