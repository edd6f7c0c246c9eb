// Kernels of the generic Tucker engine (tucker.cuh): any processing order,
// fixed-rank (block Krylov) or fixed-accuracy (block Lanczos bidiagonalisation)
// compression, tenrec/sketch.py:211-427.
//
// The engine works on explicit mode-k unfoldings: a batched transpose moves
// mode k to the front (the reference's unfold column order: remaining modes
// ascending, earliest fastest, core.py:44-55) and folds the new core back.
// The skinny products of the Lanczos recurrences are tall (n rows) times
// small (<= 64 columns) and run as row-blocked fp64 kernels whose reductions
// go through per-block partials summed in a fixed order (deterministic).
#pragma once

#include "common.cuh"

namespace tr {

// out[c + C (r + R b)] = in[r + R (c + C b)]: batched transpose of R x C
// column-major matrices (batch b), 32 x 32 shared tiles.
template <typename TI, typename TO>
__global__ void __launch_bounds__(256) k_batched_transpose(const TI* __restrict__ in,
                                                           TO* __restrict__ out, int64_t R,
                                                           int64_t C, int64_t tiles_r,
                                                           int64_t tiles_c) {
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  int64_t t = blockIdx.x;
  const int64_t tr_ = t % tiles_r;
  t /= tiles_r;
  const int64_t tc = t % tiles_c;
  const int64_t b = t / tiles_c;
  const int64_t r0 = tr_ * 32, c0 = tc * 32;
  const TI* src = in + b * R * C;
  TO* dst = out + b * R * C;
  for (int j = ty; j < 32; j += 8) {
    const int64_t r = r0 + tx, c = c0 + j;
    tile[j][tx] = (r < R && c < C) ? (double)src[r + R * c] : 0.0;
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    const int64_t c = c0 + tx, r = r0 + j;
    if (r < R && c < C) dst[c + C * r] = (TO)tile[tx][j];
  }
}

// Z[i + ldz j] = beta Z[i + ldz j] + alpha sum_{t<k} X[i + ldx t] Y[t + ldy j]
// (i < rows, j < c): tall X (rows x k, k <= 64) times a small Y (k x c, c <= 64).
template <typename TX>
__global__ void __launch_bounds__(256) k_tall_small(const TX* __restrict__ X, int64_t ldx,
                                                    int64_t rows, int k,
                                                    const double* __restrict__ Y, int ldy, int c,
                                                    double alpha, double beta,
                                                    double* __restrict__ Z, int64_t ldz) {
  __shared__ double ys[64 * 64];
  for (int e = threadIdx.x; e < k * c; e += blockDim.x) {
    const int t = e % k, j = e / k;
    ys[t + 64 * j] = Y[t + (int64_t)ldy * j];
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride) {
    double x[64];
#pragma unroll 8
    for (int t = 0; t < k; ++t) x[t] = (double)X[i + ldx * t];
    for (int j = 0; j < c; ++j) {
      double acc = 0.0;
      for (int t = 0; t < k; ++t) acc = fma(x[t], ys[t + 64 * j], acc);
      double* zp = Z + i + ldz * j;
      *zp = (beta == 0.0 ? 0.0 : beta * *zp) + alpha * acc;
    }
  }
}

// part[blk][t + K j] = sum over the block's rows i of X[i + ldx t] Z[i + ldz j]
// (t < K, j < c <= 32).  grid = (ceil(K / 32), nblk); 32 rows per smem stage.
template <typename TX>
__global__ void __launch_bounds__(256) k_tall_tn_partial(const TX* __restrict__ X, int64_t ldx,
                                                         int64_t rows, int K,
                                                         const double* __restrict__ Zm,
                                                         int64_t ldz, int c,
                                                         int64_t rows_per_blk,
                                                         double* __restrict__ part) {
  __shared__ double xs[32][33];
  __shared__ double zs[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + tx;
  const int64_t rb = (int64_t)blockIdx.y * rows_per_blk;
  const int64_t re = min(rows, rb + rows_per_blk);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i0 = rb; i0 < re; i0 += 32) {
    __syncthreads();
    for (int q = ty; q < 32; q += 8) {
      const int64_t i = i0 + tx;
      const int tt = blockIdx.x * 32 + q;
      xs[q][tx] = (i < re && tt < K) ? (double)X[i + ldx * tt] : 0.0;
      zs[q][tx] = (i < re && q < c) ? Zm[i + ldz * q] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = ty + 8 * u;
      double a = acc[u];
#pragma unroll 8
      for (int r = 0; r < 32; ++r) a = fma(xs[tx][r], zs[j][r], a);
      acc[u] = a;
    }
  }
  if (t < K) {
    double* out = part + (int64_t)blockIdx.y * K * c;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = ty + 8 * u;
      if (j < c) out[t + (int64_t)K * j] = acc[u];
    }
  }
}

// Core rows of a factor block, folded: for column c = lo + inner f of the
// mode-k unfolding (lo < inner = prod of the modes before k) and factor column
// j0 + j (j < cnt <= 64), out[lo + inner (j0 + j + r f)] = sum_i A[i + m c] U[i + m j]
// -- the new core f^T a written straight into its natural layout
// (sketch.py:397-399).  One warp per unfolding column, fp64 accumulation.
template <typename T>
__global__ void __launch_bounds__(256) k_project_rows(const T* __restrict__ A, int64_t m,
                                                      int64_t n, const double* __restrict__ U,
                                                      int cnt, int j0, int r, int64_t inner,
                                                      double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < n; c += nwarps) {
    double acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0;
    for (int64_t i = lane; i < m; i += 32) {
      const double a = (double)A[i + m * c];
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if (j < cnt) acc[j] = fma(a, U[i + m * j], acc[j]);
    }
    const int64_t lo = c % inner, f = c / inner;
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      if (j < cnt) {
        const double v = warp_sum(acc[j]);
        if (lane == 0) out[lo + inner * (j0 + j + (int64_t)r * f)] = v;
      }
    }
  }
}

// Z[i + m j] = sum_{t<k} F[i + m t] X[t + k j]: the mode product of the
// re-expansion (m x k factor times k x ncols core unfolding), 64 x 64 output
// tiles, k staged through shared memory in chunks of 16.
template <typename TO>
__global__ void __launch_bounds__(256) k_gemm_smallk(const double* __restrict__ F, int64_t m,
                                                     int k, const double* __restrict__ X,
                                                     int64_t ncols, TO* __restrict__ Z,
                                                     int64_t tiles_m) {
  __shared__ double fs[16][64 + 1];
  __shared__ double xs[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16, 4 x 4 per thread
  const int64_t i0 = (int64_t)(blockIdx.x % tiles_m) * 64;
  const int64_t j0 = (int64_t)(blockIdx.x / tiles_m) * 64;
  double acc[4][4] = {};
  for (int t0 = 0; t0 < k; t0 += 16) {
    __syncthreads();
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int t = e / 64, r = e % 64;
      fs[t][r] = (t0 + t < k && i0 + r < m) ? F[i0 + r + m * (t0 + t)] : 0.0;
      xs[t][r] = (t0 + t < k && j0 + r < ncols) ? X[(t0 + t) + (int64_t)k * (j0 + r)] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = fs[t][tx + 16 * u];
        b[u] = xs[t][ty + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t i = i0 + tx + 16 * u, j = j0 + ty + 16 * v;
      if (i < m && j < ncols) Z[i + m * j] = (TO)acc[u][v];
    }
}

// G[c + n t] = N(0,1) at Philox (seed, stream, c * cols + t): the (n, cols)
// draw of numpy's standard_normal((n, cols)) fill order, stored column-major.
__global__ void k_gauss_block(uint64_t seed, uint64_t stream, int64_t n, int cols,
                              double* __restrict__ G) {
  const int64_t total = n * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / cols;
    const int t = (int)(e % cols);
    G[c + n * t] = gauss_at(seed, stream, (uint64_t)e);
  }
}

// Per-block sums of squares of x[0..n) (fixed order; summed by k_reduce_partials).
template <typename T>
__global__ void __launch_bounds__(256) k_sumsq_partial(const T* __restrict__ x, int64_t n,
                                                       double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)x[i];
    s = fma(v, v, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Column signs of a factor (the canonical convention shared with the oracle,
// oracle/lrta.py canonicalize_columns): column j is flipped so that its
// largest-|entry| (first index on ties) is positive.  One CTA per column.
__global__ void __launch_bounds__(256) k_canonical_signs(double* __restrict__ F, int64_t m) {
  __shared__ double bv[256];
  __shared__ int64_t bi[256];
  double* col = F + m * blockIdx.x;
  double best = -1.0;
  int64_t arg = 0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double a = fabs(col[i]);
    if (a > best) {
      best = a;
      arg = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = arg;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double a = bv[threadIdx.x + o];
      const int64_t ia = bi[threadIdx.x + o];
      if (a > bv[threadIdx.x] || (a == bv[threadIdx.x] && ia < bi[threadIdx.x])) {
        bv[threadIdx.x] = a;
        bi[threadIdx.x] = ia;
      }
    }
    __syncthreads();
  }
  const bool flip = col[bi[0]] < 0.0;
  __syncthreads();
  if (flip)
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) col[i] = -col[i];
}

// rows [r0, r1) of an ld x ld matrix set to zero (the truncated R of a block)
__global__ void k_zero_rows(double* __restrict__ R, int ld, int r0, int r1) {
  for (int e = threadIdx.x; e < ld * ld; e += blockDim.x) {
    const int i = e % ld;
    if (i >= r0 && i < r1) R[e] = 0.0;
  }
}

// columns [c0, c1) of an ld x ld matrix set to zero
__global__ void k_zero_cols(double* __restrict__ L, int ld, int rows, int c0, int c1) {
  (void)rows;
  for (int e = threadIdx.x; e < ld * ld; e += blockDim.x) {
    const int j = e / ld;
    if (j >= c0 && j < c1) L[e] = 0.0;
  }
}

// out (ld_out x ld_out) = [in^T, 0]: out[i + ld_out j] = in[j + ld_in i] for
// i < cols_in, j < rows_in, zero elsewhere (l_next = l_t^T, sketch.py:342)
__global__ void k_transpose_small(const double* __restrict__ in, int ld_in, int rows_in,
                                  int cols_in, double* __restrict__ out, int ld_out) {
  for (int e = threadIdx.x; e < ld_out * ld_out; e += blockDim.x) {
    const int i = e % ld_out, j = e / ld_out;
    out[e] = (i < cols_in && j < rows_in) ? in[j + ld_in * i] : 0.0;
  }
}

// partial[p][j][i] = sum_{c in split p} A[i + m c] V[c + n j] in fp64 (j < b <= B):
// the A v pass of the bidiagonalisation with fp64 accumulation for either
// streaming precision (its deflation test runs at 1e-10 ||A||, far below fp32
// rounding).  One row per thread, V tiles of 32 columns in shared memory.
template <typename T, int B>
__global__ void __launch_bounds__(256) k_av_partial(const T* __restrict__ A, int64_t m, int64_t n,
                                                    int b, const double* __restrict__ V,
                                                    int64_t cols_per_split,
                                                    double* __restrict__ partial) {
  __shared__ double vs[32][B];
  const int64_t row = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t cb = (int64_t)blockIdx.y * cols_per_split;
  const int64_t ce = min(n, cb + cols_per_split);
  double acc[B];
#pragma unroll
  for (int j = 0; j < B; ++j) acc[j] = 0.0;
  for (int64_t c0 = cb; c0 < ce; c0 += 32) {
    const int cnt = (int)(ce - c0 < 32 ? (ce - c0) : 32);
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * B; e += 256) {
      const int cc = e % 32, j = e / 32;
      vs[cc][j] = (cc < cnt && j < b) ? V[c0 + cc + n * j] : 0.0;
    }
    __syncthreads();
    if (row < m) {
      const T* ap = A + row + m * c0;
      for (int cc = 0; cc < cnt; ++cc) {
        const double a = (double)ap[m * cc];
#pragma unroll
        for (int j = 0; j < B; ++j) acc[j] = fma(a, vs[cc][j], acc[j]);
      }
    }
  }
  if (row < m) {
    double* out = partial + (int64_t)blockIdx.y * b * m;
    for (int j = 0; j < b; ++j) out[(int64_t)j * m + row] = acc[j];
  }
}

}  // namespace tr
