// Fused streaming passes over a tall unfolding A (m x n, column-major) for the
// block Krylov iteration of tenrec/sketch.py:253-259.
//
//   MODE_SKETCH:  Y = A G          (G: Gaussian sketch generated on the fly)
//   MODE_GRAM:    Y = A (A^T P)    (one power of A A^T in ONE pass over A)
//
// A is streamed through shared memory in contiguous column chunks by the TMA
// bulk-copy engine (cp.async.bulk + mbarrier transaction counts), NSTAGE deep,
// by a persistent grid of one CTA per SM.  Each thread owns 4 consecutive rows
// (x QMAX row quads) and keeps them and the matching rows of P in registers:
//   phase 1 (GRAM): partial (A^T P) of the chunk from the thread's rows, summed
//                   across the CTA by a transposing warp reduction + smem;
//   phase 2:        rank-b update of the thread's rows of Y.
// Per element of A: 2b (sketch) or 4b (gram) FMAs, 0 extra HBM traffic.
// Per-CTA results go to `partial` (reduced deterministically afterwards).
#pragma once

#include "common.cuh"
#include "lrta_kernels.cuh"

namespace tr {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}

// global -> shared bulk copy completing on `bar` (bytes % 16 == 0, 16B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Transposing warp reduction of 32 values per lane: afterwards lane l holds
// the warp-wide sum of v[l] in v[0].  31 shuffles for 32 sums.
template <typename T>
__device__ __forceinline__ T warp_transpose_reduce32(T (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16, n = 32; o >= 1; o >>= 1, n >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const T send = upper ? v[i] : v[i + n / 2];
      const T keep = upper ? v[i + n / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0];
}

// 4 consecutive elements from a 16-byte aligned shared address
__device__ __forceinline__ void lds4(const float* p, float (&a)[4]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  a[0] = v.x;
  a[1] = v.y;
  a[2] = v.z;
  a[3] = v.w;
}
__device__ __forceinline__ void lds4(const double* p, double (&a)[4]) {
  const double2 v0 = reinterpret_cast<const double2*>(p)[0];
  const double2 v1 = reinterpret_cast<const double2*>(p)[1];
  a[0] = v0.x;
  a[1] = v0.y;
  a[2] = v1.x;
  a[3] = v1.y;
}

constexpr int kPanelThreads = 256;
constexpr int kPanelStages = 4;

struct PanelArgs {
  int64_t m, n;
  int b;
  int cc;              // columns per chunk
  int64_t nchunks;
  SketchSpec sk;       // sketch: logical column remap + Philox stream
};

// MODE 0 = sketch (coef from Philox / gover), 1 = gram (coef = A_chunk^T P).
template <typename T, int B, int QMAX, int MODE>
__global__ void __launch_bounds__(kPanelThreads, 1)
    k_panel(const T* __restrict__ A, const T* __restrict__ P, const T* __restrict__ gover,
            PanelArgs pa, double* __restrict__ partial) {
  extern __shared__ __align__(128) unsigned char panel_smem[];
  __shared__ __align__(8) uint64_t full[kPanelStages];
  const int cc = pa.cc;
  const int64_t m = pa.m;
  const size_t stage_elems = (size_t)m * cc;
  T* stages = reinterpret_cast<T*>(panel_smem);
  T* coef = stages + kPanelStages * stage_elems;        // cc x B
  T* red = coef + (size_t)cc * B;                        // 8 warps x (cc * B)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x;
  const int64_t my_chunks = pa.nchunks > (int64_t)blockIdx.x
                                ? (pa.nchunks - 1 - blockIdx.x) / G + 1 : 0;

  if (tid == 0) {
    for (int s = 0; s < kPanelStages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int64_t it) {
    const int64_t ch = blockIdx.x + it * G;
    const int64_t c0 = ch * cc;
    const int64_t cols = (pa.n - c0) < cc ? (pa.n - c0) : cc;
    const uint32_t bytes = (uint32_t)(cols * m * sizeof(T));
    const int s = (int)(it % kPanelStages);
    mbar_arrive_expect_tx(&full[s], bytes);
    bulk_g2s(stages + s * stage_elems, A + c0 * m, bytes, &full[s]);
  };
  if (tid == 0)
    for (int64_t it = 0; it < my_chunks && it < kPanelStages; ++it) issue(it);

  // this thread's rows: 4*tid + 1024*q + r
  T prow[QMAX][4][B];
  T acc[QMAX][4][B];
#pragma unroll
  for (int q = 0; q < QMAX; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < B; ++j) {
        acc[q][r][j] = T(0);
        const int64_t row = 4 * tid + 1024 * q + r;
        prow[q][r][j] = (MODE == 1 && row < m && j < pa.b) ? P[row + m * j] : T(0);
      }
  const int64_t eff = pa.sk.inner_eff ? *pa.sk.inner_eff : pa.sk.inner;

  for (int64_t it = 0; it < my_chunks; ++it) {
    const int64_t ch = blockIdx.x + it * G;
    const int64_t c0 = ch * cc;
    const int cols = (int)((pa.n - c0) < cc ? (pa.n - c0) : cc);
    const int s = (int)(it % kPanelStages);
    if (MODE == 0) {
      // Gaussian coefficients of this chunk (logical column index)
      for (int e = tid; e < cc * B; e += kPanelThreads) {
        const int c = e / B, j = e % B;
        T v = T(0);
        if (c < cols && j < pa.b) {
          const int64_t col = c0 + c + pa.sk.col0;  // global column
          const int64_t lo = col % pa.sk.inner, f = col / pa.sk.inner;
          if (lo < eff) {
            const int64_t cl = lo + eff * f;
            v = gover ? gover[cl * pa.b + j]
                      : (T)gauss_at(pa.sk.seed, pa.sk.stream, (uint64_t)(cl * pa.b + j));
          }
        }
        coef[e] = v;
      }
    }
    mbar_wait(&full[s], (uint32_t)((it / kPanelStages) & 1));
    const T* As = stages + s * stage_elems;
    if (MODE == 1) {
      // phase 1: coef[c][j] = sum_rows A[row, c] P[row, j], groups of 32 (c, j)
      constexpr int CPG = 32 / B;  // columns per reduction group
      for (int g0 = 0; g0 < cc; g0 += CPG) {
        T v[32];
#pragma unroll
        for (int cg = 0; cg < CPG; ++cg) {
          const int c = g0 + cg;
          T a[QMAX][4];
#pragma unroll
          for (int q = 0; q < QMAX; ++q) {
            const int64_t row0 = 4 * tid + 1024 * q;
            if (c < cols && row0 < m) {
              lds4(As + (size_t)c * m + row0, a[q]);
            } else {
#pragma unroll
              for (int r = 0; r < 4; ++r) a[q][r] = T(0);
            }
          }
#pragma unroll
          for (int j = 0; j < B; ++j) {
            T t = T(0);
#pragma unroll
            for (int q = 0; q < QMAX; ++q)
#pragma unroll
              for (int r = 0; r < 4; ++r) t += a[q][r] * prow[q][r][j];
            v[cg * B + j] = t;
          }
        }
        const T sum = warp_transpose_reduce32(v);
        // cc need not be a multiple of CPG (fp64, m = 1024: cc = 6): no store past this warp's row
        if (g0 * B + lane < cc * B) red[warp * (cc * B) + g0 * B + lane] = sum;
      }
      __syncthreads();
      for (int e = tid; e < cc * B; e += kPanelThreads) {
        T t = T(0);
#pragma unroll
        for (int w = 0; w < kPanelThreads / 32; ++w) t += red[w * (cc * B) + e];
        coef[e] = t;
      }
    }
    __syncthreads();
    // phase 2: rank-b update of this thread's rows
    for (int c = 0; c < cols; ++c) {
      T cf[B];
#pragma unroll
      for (int j = 0; j < B; ++j) cf[j] = coef[c * B + j];
#pragma unroll
      for (int q = 0; q < QMAX; ++q) {
        const int64_t row0 = 4 * tid + 1024 * q;
        if (row0 < m) {
          T a[4];
          lds4(As + (size_t)c * m + row0, a);
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int j = 0; j < B; ++j) acc[q][r][j] += a[r] * cf[j];
        }
      }
    }
    __syncthreads();  // stage s and coef free
    if (tid == 0 && it + kPanelStages < my_chunks) issue(it + kPanelStages);
  }
  double* out = partial + (int64_t)blockIdx.x * pa.b * m;
#pragma unroll
  for (int q = 0; q < QMAX; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t row = 4 * tid + 1024 * q + r;
#pragma unroll
      for (int j = 0; j < B; ++j)  // static indices keep acc in registers
        if (row < m && j < pa.b) out[(int64_t)j * m + row] = (double)acc[q][r][j];
    }
}

}  // namespace tr
