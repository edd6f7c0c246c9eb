// Kernels of the randomized t-SVT (tenrec/sketch.py:211-270, 430-456) on B200.
//
// Every large unfolding is an m x n column-major matrix A (lda = m): the
// mode-0 unfolding of the input is the tensor itself, and the mode-1
// unfolding of the mode-0 core is produced directly in that layout by
// k_core_from_w.  Small dense algebra (Krylov basis, Rayleigh-Ritz, core
// SVDs) runs in fp64 regardless of the streaming precision T.
#pragma once

#include "common.cuh"
#include "prox.cuh"

namespace tr {

// Logical column of a (possibly rank-padded) unfolding: padded column
// c = lo + inner * f maps to lo + inner_eff * f (the reference's unpadded
// unfolding) when lo < inner_eff; columns with lo >= inner_eff are zero.
struct SketchSpec {
  uint64_t seed;
  uint64_t stream;
  int64_t inner;
  const int64_t* inner_eff;  // device scalar or nullptr
  int64_t col0 = 0;          // global index of local column 0 (sharded unfoldings)
};

// partial[p][j][i] = sum_{c in split p} A[i + m c] * C(c, j)
// C(c, j) = coef[c*b + j] when coef != nullptr, else the Gaussian sketch entry
// (override `gover` or Philox) at the logical column.
template <typename T, int B>
__global__ void __launch_bounds__(256) k_rank_update(
    const T* __restrict__ A, int64_t m, int64_t n, int b, const T* __restrict__ coef,
    const T* __restrict__ gover, SketchSpec sk, int64_t cols_per_split,
    double* __restrict__ partial) {
  __shared__ T cs[32][B];
  const int64_t row = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t cb = (int64_t)blockIdx.y * cols_per_split;
  const int64_t ce = min(n, cb + cols_per_split);
  const int64_t eff = sk.inner_eff ? *sk.inner_eff : sk.inner;
  T acc[B];
#pragma unroll
  for (int j = 0; j < B; ++j) acc[j] = T(0);
  for (int64_t c0 = cb; c0 < ce; c0 += 32) {
    const int cnt = (int)(ce - c0 < 32 ? (ce - c0) : 32);
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * B; e += 256) {
      const int cc = e / B, j = e % B;
      T v = T(0);
      if (cc < cnt && j < b) {
        const int64_t c = c0 + cc;
        if (coef) {
          v = coef[c * b + j];
        } else {
          const int64_t lo = (c + sk.col0) % sk.inner, f = (c + sk.col0) / sk.inner;
          if (lo < eff) {
            const int64_t cl = lo + eff * f;
            v = gover ? gover[cl * b + j] : (T)gauss_at(sk.seed, sk.stream, (uint64_t)(cl * b + j));
          }
        }
      }
      cs[cc][j] = v;
    }
    __syncthreads();
    if (row < m) {
      const T* ap = A + row + m * c0;
#pragma unroll 4
      for (int cc = 0; cc < cnt; ++cc) {
        const T a = ap[m * cc];
#pragma unroll
        for (int j = 0; j < B; ++j) acc[j] += a * cs[cc][j];
      }
    }
  }
  if (row < m) {
    double* out = partial + (int64_t)blockIdx.y * b * m;
    for (int j = 0; j < b; ++j) out[(int64_t)j * m + row] = (double)acc[j];
  }
}

// W[c*s + j] = sum_i A[i + m c] * Z[i + m j]  (one warp per column)
template <typename T, int S>
__global__ void __launch_bounds__(256) k_dot_cols(const T* __restrict__ A, int64_t m,
                                                  int64_t n, const T* __restrict__ Z, int s,
                                                  T* __restrict__ W) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < n; c += nwarps) {
    T acc[S];
#pragma unroll
    for (int j = 0; j < S; ++j) acc[j] = T(0);
    for (int64_t i = lane; i < m; i += 32) {
      const T a = A[i + m * c];
#pragma unroll
      for (int j = 0; j < S; ++j)
        if (j < s) acc[j] += a * Z[i + m * j];
    }
#pragma unroll
    for (int j = 0; j < S; ++j) {
      if (j < s) {
        const T v = warp_sum(acc[j]);
        if (lane == 0) W[c * s + j] = v;
      }
    }
  }
}

// part[blk][j*s + k] = sum over the block's rows c of W[c*s+j] * W[c*s+k]
template <typename T>
__global__ void __launch_bounds__(256) k_wtw(const T* __restrict__ W, int64_t n, int s,
                                             int64_t rows_per_blk, double* __restrict__ part) {
  extern __shared__ double sw[];  // 32 x s
  const int64_t rb = (int64_t)blockIdx.x * rows_per_blk;
  const int64_t re = min(n, rb + rows_per_blk);
  const int ss = s * s;
  double acc[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) acc[t] = 0.0;
  for (int64_t r0 = rb; r0 < re; r0 += 32) {
    const int cnt = (int)(re - r0 < 32 ? (re - r0) : 32);
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * s; e += 256) {
      const int rr = e / s;
      sw[e] = rr < cnt ? (double)W[(r0 + rr) * s + (e % s)] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int e = threadIdx.x + 256 * t;
      if (e < ss) {
        const int j = e / s, k = e % s;
        double a = 0.0;
        for (int rr = 0; rr < cnt; ++rr) a += sw[rr * s + j] * sw[rr * s + k];
        acc[t] += a;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int e = threadIdx.x + 256 * t;
    if (e < ss) part[(int64_t)blockIdx.x * ss + e] = acc[t];
  }
}

// Same partials for s <= 32: thread t of each 64-thread row group owns the
// 4 x 4 block (4 (t/8) + a, 4 (t%8) + b) of the Gram, 16 independent fp64
// accumulators; the 4 row groups of the CTA are combined in shared memory.
template <typename T>
__global__ void __launch_bounds__(256) k_wtw32(const T* __restrict__ W, int64_t n, int s,
                                               int64_t rows_per_blk, double* __restrict__ part) {
  __shared__ double red[3][32 * 32];
  const int grp = threadIdx.x >> 6, t = threadIdx.x & 63;
  const int j0 = 4 * (t >> 3), k0 = 4 * (t & 7);
  const int64_t rb = (int64_t)blockIdx.x * rows_per_blk;
  const int64_t re = min(n, rb + rows_per_blk);
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  if (j0 < s && k0 < s) {
    for (int64_t r = rb + grp; r < re; r += 4) {
      const T* row = W + r * s;
      double x[4], y[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        x[a] = j0 + a < s ? (double)row[j0 + a] : 0.0;
        y[a] = k0 + a < s ? (double)row[k0 + a] : 0.0;
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += x[a] * y[b];
    }
  }
  if (grp > 0)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) red[grp - 1][(j0 + a) * 32 + k0 + b] = acc[a][b];
  __syncthreads();
  if (grp == 0)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = j0 + a, k = k0 + b;
        if (j < s && k < s) {
          const int e = j * 32 + k;
          part[(int64_t)blockIdx.x * s * s + j * s + k] =
              ((acc[a][b] + red[0][e]) + red[1][e]) + red[2][e];
        }
      }
}

// out[e] = sum_p part[p*len + e]  (fixed summation order: deterministic).
// One warp per 32 consecutive outputs x 8 partial groups: lanes stream
// coalesced rows, each warp owns a slice of the partials, smem tree at the end.
__global__ void __launch_bounds__(256) k_reduce_partials(const double* __restrict__ part,
                                                         int nparts, int64_t len,
                                                         double* __restrict__ out) {
  __shared__ double acc[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < len)
    for (int p = warp; p < nparts; p += 8) s += part[(int64_t)p * len + e];
  acc[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && e < len) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += acc[w][lane];
    out[e] = t;
  }
}

// k_reduce_partials + k_normalize_piece in one launch (the Krylov step's
// tail, sketch.py:257-258): block b sums the partials of elements
// [32 b, 32 b + 32) in the same order as k_reduce_partials, stores them and its
// sum of squares; the last block to finish (ticket counter, reset by it)
// adds the block sums in index order and scales every element by 1/||K||_F.
// One launch instead of two per Krylov step; deterministic.
template <typename T>
__global__ void __launch_bounds__(256) k_reduce_normalize(const double* __restrict__ part,
                                                          int nparts, int64_t len,
                                                          double* __restrict__ kslot,
                                                          T* __restrict__ p,
                                                          double* __restrict__ bsum,
                                                          unsigned int* __restrict__ ticket) {
  __shared__ double acc[8][32];
  __shared__ bool last;
  __shared__ double inv_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < len)
    for (int q = warp; q < nparts; q += 8) s += part[(int64_t)q * len + e];
  acc[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    if (e < len) {
#pragma unroll
      for (int w = 0; w < 8; ++w) t += acc[w][lane];
      kslot[e] = t;
    }
    const double sq = warp_sum(t * t);
    if (lane == 0) {
      bsum[blockIdx.x] = sq;
      __threadfence();
      last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (warp == 0) {
    double t = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) t += bsum[b];
    t = warp_sum(t);
    if (lane == 0) {
      const double nrm = sqrt(t);
      inv_s = nrm > 0.0 ? 1.0 / nrm : 0.0;
      *ticket = 0u;
    }
  }
  __syncthreads();
  const double inv = inv_s;
  for (int64_t i0 = threadIdx.x; i0 < len; i0 += 8 * (int64_t)blockDim.x) {
    double v[8];  // 8 independent loads in flight before the stores
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      v[u] = i < len ? __ldcg(kslot + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      if (i < len) {
        const double x = inv > 0.0 ? v[u] * inv : v[u];
        kslot[i] = x;
        p[i] = (T)x;
      }
    }
  }
}

// Fast fp64 reciprocal / reciprocal square root: fp32 seed + two Newton steps
// (~1 ulp; the IEEE-rounded slow paths dominate Jacobi round latency otherwise).
// Valid for |x| in the fp32 normal range, which the callers guarantee.
__device__ __forceinline__ double fast_rcp(double x) {
  double r = (double)__frcp_rn((float)x);
  r = r * (2.0 - x * r);
  r = r * (2.0 - x * r);
  return r;
}
__device__ __forceinline__ double fast_rsqrt(double x) {
  double r = (double)rsqrtf((float)x);
  r = r * (1.5 - 0.5 * x * r * r);
  r = r * (1.5 - 0.5 * x * r * r);
  r = r * (1.5 - 0.5 * x * r * r);
  return r;
}

// Jacobi rotation (c, s) annihilating a_pq of [[app, apq], [apq, aqq]]
// (t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = (aqq - app) / (2 apq)).
__device__ __forceinline__ void jacobi_cs(double app, double aqq, double apq, double& c,
                                          double& s) {
  const double ra = fabs(apq);
  const double inv = (ra > 1e-30 && ra < 1e30) ? fast_rcp(apq) : 1.0 / apq;
  const double tau = (aqq - app) * 0.5 * inv;
  double t;
  const double at = fabs(tau);
  if (at > 1e15) {
    t = 0.5 / tau;  // sqrt(1 + tau^2) ~ |tau|
  } else if (at < 1e-30) {
    t = 1.0;
  } else {
    const double h = 1.0 + tau * tau;
    const double sq = h * fast_rsqrt(h);
    t = (tau >= 0 ? 1.0 : -1.0) * fast_rcp(at + sq);
  }
  c = fast_rsqrt(1.0 + t * t);
  s = t * c;
}

// Same rotation with the tangent formed in fp32 (MUFU rcp/sqrt) and c, s
// completed in fp64 from it: the rotation stays exactly orthogonal in fp64;
// only the annihilation of a_pq is fp32-accurate, which the following sweeps
// absorb.  Shortens the serial latency chain of a Jacobi round.
__device__ __forceinline__ void jacobi_cs_fast(double app, double aqq, double apq, double& c,
                                               double& s) {
  // fast_rcp starts from an fp32 reciprocal: outside [1e-30, 1e30] use the
  // IEEE division (a tiny or huge a_pq would give inf / 0 there)
  const double ra = fabs(apq);
  const double r = (aqq - app) * 0.5 * ((ra > 1e-30 && ra < 1e30) ? fast_rcp(apq) : 1.0 / apq);
  const float rf = (float)r;
  float tf;
  if (fabsf(rf) > 1e15f) tf = 0.5f / rf;
  else tf = copysignf(1.0f, rf) / (fabsf(rf) + sqrtf(1.0f + rf * rf));
  const double t = (double)tf;
  c = fast_rsqrt(1.0 + t * t);
  s = t * c;
}

// Krylov piece normalisation (sketch.py:257-258): piece = blk / ||blk||_F.
template <typename T>
__global__ void __launch_bounds__(1024) k_normalize_piece(double* __restrict__ kslot,
                                                          int64_t len, T* __restrict__ p) {
  __shared__ double red[32];
  double ss = 0.0;
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) ss += kslot[e] * kslot[e];
  const double nrm = sqrt(block_sum(ss, red));
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
    const double v = nrm > 0.0 ? kslot[e] / nrm : kslot[e];
    kslot[e] = v;
    p[e] = (T)v;
  }
}

// Sum `nv` per-thread values across the block into out[0..nv) (smem).
// red must hold 32 * 64 doubles; nv <= 64.
__device__ inline void block_sum_vec(const double* v, int nv, double* red, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int j = 0; j < nv; ++j) {
    const double t = warp_sum(v[j]);
    if (lane == 0) red[wid * 64 + j] = t;
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w * 64 + threadIdx.x];
    out[threadIdx.x] = t;
  }
  __syncthreads();
}

// Orthonormal basis of the Krylov block (sketch.py:167-185): pivoted
// Gram-Schmidt with the reference's deflation rule (stop once the largest
// remaining column norm falls below 1e-14 * ||K||_F, the |R_kk| test of
// Algorithm 2) and a second projection pass for full orthogonality.
// Single CTA of 1024 threads; K and the work copy live in L2.
template <typename T>
__global__ void __launch_bounds__(1024) k_orth(const double* __restrict__ K, int64_t m, int s,
                                               double* __restrict__ work,
                                               double* __restrict__ Z, T* __restrict__ Zt,
                                               int64_t* __restrict__ info) {
  __shared__ double red[32 * 64];
  __shared__ double vec[64];
  __shared__ int piv;
  __shared__ int s_eff;
  double loc[64];
  double ss = 0.0;
  for (int64_t e = threadIdx.x; e < m * s; e += blockDim.x) {
    const double v = K[e];
    work[e] = v;
    Z[e] = 0.0;
    ss += v * v;
  }
  const double tol = 1e-14 * sqrt(block_sum(ss, red));
  if (threadIdx.x == 0) s_eff = s;
  __syncthreads();
  for (int k = 0; k < s; ++k) {
    // residual column norms of k..s-1
    for (int j = 0; j < 64; ++j) loc[j] = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x)
      for (int j = k; j < s; ++j) {
        const double v = work[i + m * j];
        loc[j - k] += v * v;
      }
    block_sum_vec(loc, s - k, red, vec);
    if (threadIdx.x == 0) {
      int best = 0;
      for (int j = 1; j < s - k; ++j)
        if (vec[j] > vec[best]) best = j;
      piv = k + best;
      const double nb = sqrt(vec[best]);
      if (!(nb >= tol) || nb == 0.0) s_eff = k;
    }
    __syncthreads();
    if (s_eff == k) break;
    const int p = piv;
    if (p != k)
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const double a = work[i + m * k];
        work[i + m * k] = work[i + m * p];
        work[i + m * p] = a;
      }
    __syncthreads();
    // second projection of the pivot column against the accepted basis
    for (int j = 0; j < 64; ++j) loc[j] = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      const double v = work[i + m * k];
      for (int l = 0; l < k; ++l) loc[l] += Z[i + m * l] * v;
    }
    block_sum_vec(loc, k, red, vec);
    double nn = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      double v = work[i + m * k];
      for (int l = 0; l < k; ++l) v -= vec[l] * Z[i + m * l];
      work[i + m * k] = v;
      nn += v * v;
    }
    const double nrm = sqrt(block_sum(nn, red));
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) Z[i + m * k] = work[i + m * k] / nrm;
    __syncthreads();
    // project the remaining columns (modified Gram-Schmidt step)
    for (int j = 0; j < 64; ++j) loc[j] = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      const double q = Z[i + m * k];
      for (int j = k + 1; j < s; ++j) loc[j - k - 1] += q * work[i + m * j];
    }
    block_sum_vec(loc, s - k - 1, red, vec);
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      const double q = Z[i + m * k];
      for (int j = k + 1; j < s; ++j) work[i + m * j] -= vec[j - k - 1] * q;
    }
    __syncthreads();
  }
  for (int64_t e = threadIdx.x; e < m * s; e += blockDim.x) Zt[e] = (T)Z[e];
  if (threadIdx.x == 0) info[0] = s_eff;
}

#ifdef TR_RITZ_PROBE
__device__ long long g_ritz_probe[4];
#endif

// Rayleigh-Ritz (sketch.py:261-265) for s_eff <= 32 by QR-preconditioned
// one-sided Jacobi (Drmac-Veselic): a complete-pivoting Cholesky P M P^T =
// R^T R, then one-sided (Hestenes) Jacobi on the columns of R^T.  The columns
// of R^T V become orthogonal -- normalised, they are the eigenvectors of
// P M P^T, their squared norms the eigenvalues.  The Krylov Gram matrices are
// strongly graded (eigenvalues over many decades), for which the pivoted
// factor is nearly orthogonal already: a few sweeps instead of the ~8 of
// two-sided Jacobi on M.  16 threads per column pair, one barrier per round.
// V (s x r) = the top r_eff eigenvectors (rows un-permuted), descending; signs
// are fixed by k_ritz_apply.  A numerically rank-deficient M (pivot below
// 1e-15 of the largest diagonal) leaves its null space to an orthonormal
// completion -- eigenvalue-0 Ritz vectors the reference's eigh also fixes
// arbitrarily.
__global__ void __launch_bounds__(256) k_ritz_pc(const double* __restrict__ Mfull, int s, int r,
                                                 double* __restrict__ V,
                                                 int64_t* __restrict__ info) {
  constexpr int LD = 33;
  __shared__ double A[32 * LD], B[32 * LD];
  __shared__ unsigned char sched[31][16][2];
  __shared__ int perm[32], order[32];
  __shared__ double nrm[32];
  __shared__ int piv_s, rank_s;
  __shared__ double dmax_s;
  const int n = (int)info[0];  // s_eff
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 32 * 32; e += 256) {
    const int i = e & 31, j = e >> 5;
    A[i + LD * j] = (i < n && j < n) ? Mfull[i + s * j] : 0.0;
    B[i + LD * j] = 0.0;
  }
  if (tid < 32) perm[tid] = tid;
  if (tid == 0) rank_s = n;
  __syncthreads();
  if (warp == 0) {
    double d = lane < n ? A[lane + LD * lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    if (lane == 0) dmax_s = d;
  }
  __syncthreads();
  const double tol = 1e-15 * dmax_s;
#ifdef TR_RITZ_PROBE
  const long long t_c0 = clock64();
#endif
  // ---- complete-pivoting Cholesky ----
  for (int k = 0; k < n; ++k) {
    if (warp == 0) {
      double v = (lane >= k && lane < n) ? A[lane + LD * lane] : -1.0;
      int idx = lane;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) {
          v = ov;
          idx = oi;
        }
      }
      if (lane == 0) {
        piv_s = idx;
        if (!(v > tol)) rank_s = k;
      }
    }
    __syncthreads();
    if (rank_s == k) break;
    const int p = piv_s;
    if (p != k) {
      // symmetric swap of rows / columns k, p of the Schur complement, rows of R^T
      for (int i = tid; i < n; i += 256) {
        double t = A[k + LD * i];
        A[k + LD * i] = A[p + LD * i];
        A[p + LD * i] = t;
      }
      __syncthreads();
      for (int i = tid; i < n; i += 256) {
        double t = A[i + LD * k];
        A[i + LD * k] = A[i + LD * p];
        A[i + LD * p] = t;
      }
      for (int j = tid; j < k; j += 256) {
        double t = B[k + LD * j];
        B[k + LD * j] = B[p + LD * j];
        B[p + LD * j] = t;
      }
      if (tid == 0) {
        const int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
      __syncthreads();
    }
    const double dk = sqrt(A[k + LD * k]);
    for (int j = k + tid; j < n; j += 256) B[j + LD * k] = j == k ? dk : A[k + LD * j] / dk;
    __syncthreads();
    const int w = n - k - 1;
    for (int e = tid; e < w * w; e += 256) {
      const int i = k + 1 + e % w, j = k + 1 + e / w;
      A[i + LD * j] -= B[i + LD * k] * B[j + LD * k];
    }
    __syncthreads();
  }
  const int rank = rank_s;
#ifdef TR_RITZ_PROBE
  const long long t_c1 = clock64();
  int nsweeps = 0;
#endif
  // ---- one-sided Jacobi on the columns of R^T (n rows, rank columns) ----
  const int ne = rank + (rank & 1);
  const int npairs = ne / 2;
  for (int e = tid; e < (ne - 1) * npairs; e += 256) {
    const int rnd = e / npairs, kk = e - rnd * npairs;
    int p = rr_player(kk, rnd, ne), q = rr_player(ne - 1 - kk, rnd, ne);
    if (p > q) {
      const int t = p;
      p = q;
      q = t;
    }
    sched[rnd][kk][0] = (unsigned char)p;
    sched[rnd][kk][1] = (unsigned char)q;
  }
  __syncthreads();
  const int kp = tid >> 4, j = tid & 15;  // pair kp, rows j and j + 16
  // next round's pair is fetched before the barrier (off the round's serial chain)
  int pn = 0, qn = rank;
  if (kp < npairs && ne >= 2) {
    pn = sched[0][kp][0];
    qn = sched[0][kp][1];
  }
  for (int sweep = 0; sweep < 40 && ne >= 2; ++sweep) {
    int big = 0;  // a pair of this sweep met |cos| > 1e-8
    for (int rnd = 0; rnd < ne - 1; ++rnd) {
      const int p = pn, q = qn;
      const bool live = q < rank;  // uniform over the pair's 16 lanes; idle slots carry zeros
      if (kp < npairs) {
        const int nr = rnd + 1 < ne - 1 ? rnd + 1 : 0;
        pn = sched[nr][kp][0];
        qn = sched[nr][kp][1];
      }
      const double ap0 = live ? B[j + LD * p] : 0.0, ap1 = live ? B[j + 16 + LD * p] : 0.0;
      const double aq0 = live ? B[j + LD * q] : 0.0, aq1 = live ? B[j + 16 + LD * q] : 0.0;
      double al = fma(ap0, ap0, ap1 * ap1), be = fma(aq0, aq0, aq1 * aq1),
             ga = fma(ap0, aq0, ap1 * aq1);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
      const double g2 = ga * ga, ab = al * be;
      if (g2 > 1e-30 * ab) {  // |cos| > 1e-15 (false for idle slots and zero columns)
        big |= g2 > 1e-16 * ab;
        // Tangent in fp32 from MUFU rsqrt / rcp on the pair scaled by a power of
        // two to max(alpha, beta) in [1, 2) (no range guards; |gamma| <= the
        // scaled geometric mean, and a rotating pair keeps z and gamma far from
        // fp32 underflow together): t = sign(z) gamma / (|z| + sqrt(z^2 + gamma^2)),
        // z = (beta - alpha) / 2.  c = (1 + t^2)^{-1/2} is completed in fp64 from
        // the t actually used: the rotation is orthogonal to fp64 rounding, only
        // the annihilation is fp32-accurate (the next sweep absorbs it).
        const double sc = __hiloint2double(0x7fe00000 - (__double2hiint(fmax(al, be)) & 0x7ff00000), 0);
        const float zf = (float)(0.5 * (be - al) * sc), gf = (float)(ga * sc);
        const float hf = fmaf(zf, zf, gf * gf);
        float rs, invd, cs;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(hf));
        const float df = fabsf(zf) + hf * rs;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(invd) : "f"(df));
        const float tf = gf * copysignf(invd, zf);
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(cs) : "f"(fmaf(tf, tf, 1.0f)));
        const double t = (double)tf;
        const double x1 = fma(t, t, 1.0);  // in [1, 2]
        const double c0 = (double)cs;
        const double er = fma(-x1, c0 * c0, 1.0);  // one cubic step: seed error ~2^-21
        const double c = fma(c0 * er, fma(0.375, er, 0.5), c0);
        const double sn = c * t;
        B[j + LD * p] = fma(c, ap0, -sn * aq0);
        B[j + 16 + LD * p] = fma(c, ap1, -sn * aq1);
        B[j + LD * q] = fma(sn, ap0, c * aq0);
        B[j + 16 + LD * q] = fma(sn, ap1, c * aq1);
      }
      if (rnd < ne - 2) __syncthreads();
    }
    // quadratic convergence: once every pair of a sweep met |cos| <= 1e-8 the
    // rotated pairs are left at <= 1e-15 and the rest moved by second-order
    // terms only -- no verification sweep
    const int any = __syncthreads_or(big);
#ifdef TR_RITZ_PROBE
    ++nsweeps;
#endif
    if (!any) break;
  }
#ifdef TR_RITZ_PROBE
  if (tid == 0) {
    info[4] = t_c1 - t_c0;
    info[5] = clock64() - t_c1;
    info[6] = nsweeps;
    info[7] = rank;
  }
#endif
  // ---- eigenpairs: normalised columns (eigenvalue = squared norm), descending ----
  if (tid < 32) {
    double x = 0.0;
    if (tid < rank)
      for (int i = 0; i < n; ++i) x += B[i + LD * tid] * B[i + LD * tid];
    nrm[tid] = tid < rank ? x : -1.0;
  }
  __syncthreads();
  if (tid < 32) {
    int rk = 0;
    const double me = nrm[tid];
    for (int c = 0; c < rank; ++c) {
      const double o = nrm[c];
      rk += (o > me || (o == me && c < tid)) ? 1 : 0;
    }
    if (tid < rank) order[rk] = tid;
  }
  __syncthreads();
  // normalise the kept columns into A (rows un-permuted): A[perm[i], c] = B[i, order[c]] / norm
  for (int e = tid; e < 32 * 32; e += 256) A[e] = 0.0;
  __syncthreads();
  for (int e = tid; e < n * rank; e += 256) {
    const int i = e % n, c = e / n;
    const int src = order[c];
    A[perm[i] + LD * c] = B[i + LD * src] / sqrt(nrm[src]);
  }
  __syncthreads();
  const int re = min(r, n);
  // orthonormal completion beyond the numerical rank (Gram-Schmidt of unit vectors)
  if (re > rank && warp == 0) {
    int c = rank;
    for (int u = 0; u < n && c < re; ++u) {
      double x = lane == u ? 1.0 : 0.0;
      for (int q = 0; q < c; ++q) {
        double dot = lane < n ? A[lane + LD * q] * (lane == u ? 1.0 : 0.0) : 0.0;
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        x -= dot * (lane < n ? A[lane + LD * q] : 0.0);
      }
      double x2 = lane < n ? x * x : 0.0;
      for (int o = 16; o > 0; o >>= 1) x2 += __shfl_xor_sync(0xffffffffu, x2, o);
      if (x2 > 1e-2) {
        if (lane < n) A[lane + LD * c] = x / sqrt(x2);
        ++c;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < s * r; e += 256) {
    const int row = e % s, col = e / s;
    V[e] = (col < re && row < n) ? A[row + LD * col] : 0.0;
  }
  if (tid == 0) info[1] = re;
}

// Rayleigh-Ritz (sketch.py:261-265): eigenvectors of M = W^T W by parallel
// cyclic Jacobi, descending order, F = Z V; then the canonical sign (largest
// |entry| of every factor column positive, first index on ties).
template <typename T>
__global__ void __launch_bounds__(256) k_ritz(const double* __restrict__ Mfull, int s,
                                              const double* __restrict__ Z, int64_t m, int r,
                                              double* __restrict__ V, double* __restrict__ F,
                                              T* __restrict__ Ft, int64_t* __restrict__ info) {
  extern __shared__ double ritz_smem[];  // A and Q, 64 x 65 each
  double* A = ritz_smem;
  double* Q = ritz_smem + 64 * 65;
  __shared__ double cs_c[32], cs_s[32];
  __shared__ int pp[32], pq[32];
  __shared__ double evals[64];
  __shared__ int order[64];
  __shared__ double sgn[64];
  __shared__ int rot_any;
  if (threadIdx.x == 0) rot_any = 0;
  __shared__ double red[32];
  const int n = (int)info[0];  // s_eff
  const int ld = 65;
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int i = e % 64, j = e / 64;
    A[i + ld * j] = (i < n && j < n) ? Mfull[i + s * j] : 0.0;
    Q[i + ld * j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int ne = n + (n & 1);
  double diag2 = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) diag2 += A[i + ld * i] * A[i + ld * i];
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int a = i % n, b = i / n;
    if (a != b) diag2 += A[a + ld * b] * A[a + ld * b];
  }
  const double mnorm = sqrt(block_sum(diag2, red));
#ifdef TR_RITZ_PROBE
  long long t_j0 = clock64();
#endif
  if (ne <= 32 && blockDim.x >= 256) {
    // n <= 32: fixed roles, decoded once -- thread t owns the 2x2 block
    // (t >> 4, t & 15) of the round's J^T A J and the Q row pairs
    // (row t & 31, pairs (t >> 5) and (t >> 5) + 8); two barriers per round.
    const int npairs = ne / 2;
    const int t = threadIdx.x;
    __shared__ unsigned char sched[31][16][2];  // round-robin pairs (p < q) of every round
    for (int e = t; e < (ne - 1) * npairs; e += blockDim.x) {
      const int rnd = e / npairs, k = e - rnd * npairs;
      int p = rr_player(k, rnd, ne), q = rr_player(ne - 1 - k, rnd, ne);
      if (p > q) { const int tt = p; p = q; q = tt; }
      sched[rnd][k][0] = (unsigned char)p;
      sched[rnd][k][1] = (unsigned char)q;
    }
    __syncthreads();
    const double mthr = 1e-16 * mnorm;
    const int bk1 = t >> 4, bk2 = t & 15;
    const bool blk = t < 256 && bk1 <= bk2 && bk2 < npairs;
    const int qi = t & 31, qk0 = (t >> 5) & 7;
    const bool qrow = t < 256 && qi < n;
    for (int sweep = 0; sweep < 40 && ne >= 2; ++sweep) {
      for (int rnd = 0; rnd < ne - 1; ++rnd) {
        if (t < npairs) {
          const int p = sched[rnd][t][0], q = sched[rnd][t][1];
          double c = 1.0, sn = 0.0;
          if (q < n) {
            const double apq = A[p + ld * q];
            const double app = A[p + ld * p], aqq = A[q + ld * q];
            // |apq| > 1e-15 sqrt|app aqq|  <=>  apq^2 > 1e-30 |app aqq|
            if (apq * apq > 1e-30 * fabs(app * aqq) && fabs(apq) > mthr) {
              rot_any = 1;
              jacobi_cs_fast(app, aqq, apq, c, sn);
            }
          }
          pp[t] = p;
          pq[t] = q;
          cs_c[t] = c;
          cs_s[t] = sn;
        }
        __syncthreads();
        if (blk) {
          const double s1 = cs_s[bk1], s2 = cs_s[bk2];
          if (s1 != 0.0 || s2 != 0.0) {
            const double c1 = cs_c[bk1], c2 = cs_c[bk2];
            const int p1 = pp[bk1], q1 = pq[bk1], p2 = pp[bk2], q2 = pq[bk2];
            const double a = A[p1 + ld * p2], b = A[p1 + ld * q2];
            const double c = A[q1 + ld * p2], d = A[q1 + ld * q2];
            const double ap = c2 * a - s2 * b, bq = s2 * a + c2 * b;
            const double cp = c2 * c - s2 * d, dq = s2 * c + c2 * d;
            const double npp = c1 * ap - s1 * cp, npq = c1 * bq - s1 * dq;
            const double nqp = s1 * ap + c1 * cp, nqq = s1 * bq + c1 * dq;
            A[p1 + ld * p2] = npp;
            A[p1 + ld * q2] = npq;
            A[q1 + ld * p2] = nqp;
            A[q1 + ld * q2] = nqq;
            if (bk1 != bk2) {
              A[p2 + ld * p1] = npp;
              A[q2 + ld * p1] = npq;
              A[p2 + ld * q1] = nqp;
              A[q2 + ld * q1] = nqq;
            }
          }
        }
        if (qrow) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int k = qk0 + 8 * u;
            if (k < npairs) {
              const double sn = cs_s[k];
              if (sn != 0.0) {
                const double c = cs_c[k];
                const int p = pp[k], q = pq[k];
                const double qp = Q[qi + ld * p], qq = Q[qi + ld * q];
                Q[qi + ld * p] = c * qp - sn * qq;
                Q[qi + ld * q] = sn * qp + c * qq;
              }
            }
          }
        }
        __syncthreads();
      }
      const int any = rot_any;
      __syncthreads();
      if (threadIdx.x == 0) rot_any = 0;
      __syncthreads();
      if (!any) break;
    }
  } else {
    for (int sweep = 0; sweep < 40 && ne >= 2; ++sweep) {
      for (int rnd = 0; rnd < ne - 1; ++rnd) {
        const int npairs = ne / 2;
        if (threadIdx.x < npairs) {
          int p = rr_player(threadIdx.x, rnd, ne), q = rr_player(ne - 1 - threadIdx.x, rnd, ne);
          if (p > q) { const int t = p; p = q; q = t; }
          double c = 1.0, sn = 0.0;
          if (q < n) {
            const double apq = A[p + ld * q];
            const double app = A[p + ld * p], aqq = A[q + ld * q];
            // skip pairs already decoupled to working precision, relative to the
            // pair and to ||M|| (rotating rounding noise never converges)
            if (fabs(apq) > 1e-15 * sqrt(fabs(app * aqq)) && fabs(apq) > 1e-16 * mnorm) {
              rot_any = 1;
              jacobi_cs(app, aqq, apq, c, sn);
            }
          }
          pp[threadIdx.x] = p;
          pq[threadIdx.x] = q;
          cs_c[threadIdx.x] = c;
          cs_s[threadIdx.x] = sn;
        }
        __syncthreads();
        // one pass per round: the rotations of a round act on disjoint index
        // pairs, so J^T A J splits into independent 2x2 blocks
        // B'(k1,k2) = J_k1^T B(k1,k2) J_k2 (upper blocks, mirrored), and Q <- Q J
        // row by row; only the live n x n part is touched.
        for (int e = threadIdx.x; e < npairs * npairs + npairs * n; e += blockDim.x) {
          if (e < npairs * npairs) {
            const int k1 = e / npairs, k2 = e - k1 * npairs;
            if (k1 > k2) continue;
            const double s1 = cs_s[k1], s2 = cs_s[k2];
            if (s1 == 0.0 && s2 == 0.0) continue;
            const double c1 = cs_c[k1], c2 = cs_c[k2];
            const int p1 = pp[k1], q1 = pq[k1], p2 = pp[k2], q2 = pq[k2];
            const double a = A[p1 + ld * p2], b = A[p1 + ld * q2];
            const double c = A[q1 + ld * p2], d = A[q1 + ld * q2];
            // columns (B J2), then rows (J1^T .)
            const double ap = c2 * a - s2 * b, bq = s2 * a + c2 * b;
            const double cp = c2 * c - s2 * d, dq = s2 * c + c2 * d;
            const double npp = c1 * ap - s1 * cp, npq = c1 * bq - s1 * dq;
            const double nqp = s1 * ap + c1 * cp, nqq = s1 * bq + c1 * dq;
            A[p1 + ld * p2] = npp;
            A[p1 + ld * q2] = npq;
            A[q1 + ld * p2] = nqp;
            A[q1 + ld * q2] = nqq;
            if (k1 != k2) {
              A[p2 + ld * p1] = npp;
              A[q2 + ld * p1] = npq;
              A[p2 + ld * q1] = nqp;
              A[q2 + ld * q1] = nqq;
            }
          } else {
            const int e2 = e - npairs * npairs;
            const int k = e2 / n, i = e2 - k * n;
            const double sn = cs_s[k];
            if (sn == 0.0) continue;
            const double c = cs_c[k];
            const int p = pp[k], q = pq[k];
            const double qp = Q[i + ld * p], qq = Q[i + ld * q];
            Q[i + ld * p] = c * qp - sn * qq;
            Q[i + ld * q] = sn * qp + c * qq;
          }
        }
        __syncthreads();
      }
      // converged once a whole sweep needed no rotation (every |a_pq| is below
      // 1e-15 sqrt(|a_pp a_qq|), the classical Jacobi stopping rule)
      const int any = rot_any;
      __syncthreads();
      if (threadIdx.x == 0) rot_any = 0;
      __syncthreads();
      if (!any) break;
    }
  }
#ifdef TR_RITZ_PROBE
  if (threadIdx.x == 0) g_ritz_probe[0] = clock64() - t_j0;
#endif
  // descending order (stable on ties, like reversing eigh's ascending output)
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      evals[i] = A[i + ld * i];
      order[i] = i;
    }
    for (int i = 1; i < n; ++i) {
      const int oi = order[i];
      int j = i - 1;
      while (j >= 0 && evals[order[j]] < evals[oi]) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = oi;
    }
  }
  __syncthreads();
  const int re = min(r, n);
  if (n <= 32 && r <= 32 && F == nullptr) {
    // F, its canonical signs and V's signs come from k_ritz_apply (many CTAs)
    for (int e = threadIdx.x; e < s * r; e += blockDim.x) {
      const int j = e % s, k = e / s;
      V[e] = (k < re && j < n) ? Q[j + ld * order[k]] : 0.0;
    }
    if (threadIdx.x == 0) info[1] = re;
    return;
  } else {
  // F = Z V (m x r): one row of Z per thread, held in registers (independent loads)
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    if (n <= 32) {
      double z[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) z[j] = j < n ? Z[i + m * j] : 0.0;
      for (int k = 0; k < r; ++k) {
        double f = 0.0;
        if (k < re) {
          const int col = order[k];
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < n) f += z[j] * Q[j + ld * col];
        }
        F[i + m * k] = f;
      }
    } else {
      for (int k = 0; k < r; ++k) {
        double f = 0.0;
        if (k < re) {
          const int col = order[k];
          for (int j = 0; j < n; ++j) f += Z[i + m * j] * Q[j + ld * col];
        }
        F[i + m * k] = f;
      }
    }
  }
  __syncthreads();
#ifdef TR_RITZ_PROBE
  if (threadIdx.x == 0) g_ritz_probe[1] = clock64() - t_j0;
#endif
  // canonical sign: one warp per column, argmax |F| with first-index ties
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = warp; k < r; k += nw) {
      double best = -1.0, bval = 0.0;
      int64_t bidx = INT64_MAX;
      for (int64_t i = lane; i < m; i += 32) {
        const double f = F[i + m * k];
        if (fabs(f) > best) {
          best = fabs(f);
          bval = f;
          bidx = i;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const double ov = __shfl_xor_sync(0xffffffffu, bval, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (ob > best || (ob == best && oi < bidx)) {
          best = ob;
          bval = ov;
          bidx = oi;
        }
      }
      if (lane == 0) sgn[k] = bval < 0.0 ? -1.0 : 1.0;
    }
  }
  }  // n > 32 or r > 32
  __syncthreads();
  for (int64_t e = threadIdx.x; e < m * r; e += blockDim.x) {
    const double f = F[e] * sgn[e / m];
    F[e] = f;
    Ft[e] = (T)f;
  }
  for (int e = threadIdx.x; e < s * r; e += blockDim.x) {
    const int j = e % s, k = e / s;
    V[e] = (k < re && j < n) ? Q[j + ld * order[k]] * sgn[k] : 0.0;
  }
  if (threadIdx.x == 0) info[1] = re;
#ifdef TR_RITZ_PROBE
  if (threadIdx.x == 0) g_ritz_probe[2] = clock64() - t_j0;
#endif
}

// Rayleigh-Ritz factor F = Z V_top (m x r, n, r <= 32) and its canonical sign
// (largest-|entry| of every column positive, first index on ties), spread
// over CTAs of 32 rows: each CTA forms its rows and a per-column argmax; the
// last CTA (ticket) combines them in row-block order, flips V's columns and
// rescales F / Ft.  V holds V_top (s x r, unsigned) on entry, signed on exit.
template <typename T>
__global__ void __launch_bounds__(256) k_ritz_apply(const double* __restrict__ Z, int64_t m, int s,
                                                    double* __restrict__ V, int r,
                                                    const int64_t* __restrict__ info,
                                                    double* __restrict__ F, T* __restrict__ Ft,
                                                    double* __restrict__ pbv,
                                                    int64_t* __restrict__ pbi,
                                                    unsigned int* __restrict__ ticket) {
  __shared__ double zs[32][33];
  __shared__ double vs[32][33];
  __shared__ double sg[32];
  __shared__ bool last;
  const int n = (int)info[0];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int i = e & 31, j = e >> 5;
    zs[i][j] = (r0 + i < m && j < n) ? Z[r0 + i + m * j] : 0.0;
    vs[i][j] = (i < n && j < r) ? V[i + (int64_t)s * j] : 0.0;  // vs[j_row][k_col]
  }
  __syncthreads();
  // thread (row lane, columns warp + 8 c): rows of this block, 4 columns each
  const int64_t row = r0 + lane;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int k = warp + 8 * c;
    double f = 0.0;
#pragma unroll
    for (int j = 0; j < 32; ++j) f += zs[lane][j] * vs[j][k];
    if (row < m && k < r) F[row + m * k] = f;
    // warp argmax over the block's 32 rows (first index on ties)
    double b = (row < m) ? f : 0.0;
    int64_t ix = (row < m) ? row : INT64_MAX;
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, b, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, ix, o);
      if (fabs(ob) > fabs(b) || (fabs(ob) == fabs(b) && oi < ix)) {
        b = ob;
        ix = oi;
      }
    }
    if (lane == 0 && k < r) {
      pbv[(int64_t)blockIdx.x * 32 + k] = b;
      pbi[(int64_t)blockIdx.x * 32 + k] = ix;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // column k: combine the blocks' candidates, 8 threads per column
  {
    const int k = tid >> 3, part = tid & 7;
    double b = 0.0;
    int64_t ix = INT64_MAX;
    if (k < r)
      for (int64_t q = part; q < (int64_t)gridDim.x; q += 8) {
        const double ob = __ldcg(pbv + q * 32 + k);
        const int64_t oi = __ldcg(pbi + q * 32 + k);
        if (fabs(ob) > fabs(b) || (fabs(ob) == fabs(b) && oi < ix)) {
          b = ob;
          ix = oi;
        }
      }
    for (int o = 4; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, b, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, ix, o);
      if (fabs(ob) > fabs(b) || (fabs(ob) == fabs(b) && oi < ix)) {
        b = ob;
        ix = oi;
      }
    }
    if (part == 0 && k < 32) sg[k] = b < 0.0 ? -1.0 : 1.0;
  }
  __syncthreads();
  for (int e = tid; e < s * r; e += blockDim.x) V[e] *= sg[e / s];
  // F / Ft rescale, 8 independent loads in flight per thread
  const int64_t tot = m * r;
  for (int64_t e0 = tid; e0 < tot; e0 += 8 * (int64_t)blockDim.x) {
    double fv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t e = e0 + (int64_t)u * blockDim.x;
      fv[u] = e < tot ? __ldcg(F + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t e = e0 + (int64_t)u * blockDim.x;
      if (e < tot) {
        const double f = fv[u] * sg[e / m];
        F[e] = f;
        Ft[e] = (T)f;
      }
    }
  }
  if (tid == 0) *ticket = 0u;
}

// The same for fp32 W rows of s <= 32 values with the CTA's 256 rows staged
// through shared memory by coalesced loads (row stride s | 1: conflict-free
// reads): a thread reading its own row straight from global memory touches
// s cache lines per load instruction (48 us for the 131072 x 28 W of the bench
// t-SVT, against ~10 us here).
template <typename TO>
__global__ void __launch_bounds__(256) k_core_from_w_s(const float* __restrict__ W, int64_t n, int s,
                                                       const double* __restrict__ V, int r,
                                                       int64_t inner, TO* __restrict__ out) {
  __shared__ double vs[32 * 32];
  __shared__ float ws[256 * 33];
  const int tid = threadIdx.x, ld = s | 1;
  for (int e = tid; e < s * r; e += 256) vs[e] = V[e];
  const int64_t c0 = (int64_t)blockIdx.x * 256;
  const int cols = (int)(n - c0 < 256 ? n - c0 : 256);
  const float* src = W + c0 * s;
  for (int e = tid; e < cols * s; e += 256) {
    const int row = e / s, j = e - row * s;
    ws[row * ld + j] = src[e];
  }
  __syncthreads();
  if (tid >= cols) return;
  const int64_t c = c0 + tid;
  const int64_t lo = c % inner, f = c / inner;
  double w[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) w[j] = j < s ? (double)ws[tid * ld + j] : 0.0;
  for (int i = 0; i < r; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < s) acc += w[j] * vs[j + s * i];
    out[lo + inner * (i + (int64_t)r * f)] = (TO)acc;
  }
}

// core rows from W: out[lo + inner*(i + r*f)] = sum_j W[c*s + j] V[j + s*i],
// c = lo + inner * f.  Realises F^T A (sketch.py:267-269) without another pass.
// One thread per unfolding column c: its W row (s values) times V (s x r,
// in shared memory) gives the r core entries of that column.
template <typename T, typename TO>
__global__ void __launch_bounds__(256) k_core_from_w(const T* __restrict__ W, int64_t n, int s,
                                                     const double* __restrict__ V, int r,
                                                     int64_t inner, TO* __restrict__ out) {
  __shared__ double vs[64 * 64];
  for (int e = threadIdx.x; e < s * r; e += blockDim.x) vs[e] = V[e];
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int64_t lo = c % inner, f = c / inner;
  double w[64];
#pragma unroll
  for (int j = 0; j < 64; ++j)
    if (j < s) w[j] = (double)W[c * s + j];
  for (int i = 0; i < r; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (j < s) acc += w[j] * vs[j + s * i];
    out[lo + inner * (i + (int64_t)r * f)] = (TO)acc;
  }
}

// C1[a + r0*(i2 + n2*f)] = sum_b core[a + r0*(b + r1*f)] * F1[i2 + n2*b]
// C1 (r0 x n2 x nf) = core x_1 F1: C1[a, i2, f] = sum_b core[a, b, f] F1[i2, b]
// (the mode-1 expansion ahead of k_gemm_expand, sketch.py:61).  One thread per
// (i2, f) column of C1: the face's r0 x r1 core block sits in shared memory
// (one block of 128 columns shares a face), the thread keeps its r0 outputs in
// registers, reads its r1 values of F1 once (coalesced over i2) and writes a
// contiguous column.  r0 <= 64.
template <typename T>
__global__ void __launch_bounds__(128) k_expand_mode1(const double* __restrict__ core, int r0,
                                                      int r1, int64_t nf,
                                                      const double* __restrict__ F1, int64_t n2,
                                                      T* __restrict__ C1) {
  __shared__ double cs[64 * 64];
  const int64_t tiles = (n2 + 127) / 128;
  const int64_t f = blockIdx.x / tiles;
  const int64_t i2 = (blockIdx.x % tiles) * 128 + threadIdx.x;
  for (int e = threadIdx.x; e < r0 * r1; e += blockDim.x) cs[e] = core[e + (int64_t)r0 * r1 * f];
  __syncthreads();
  if (i2 >= n2 || f >= nf) return;
  double acc[64];
#pragma unroll
  for (int a = 0; a < 64; ++a) acc[a] = 0.0;
  for (int b = 0; b < r1; ++b) {
    const double fv = F1[i2 + n2 * b];
#pragma unroll
    for (int a = 0; a < 64; ++a)
      if (a < r0) acc[a] += cs[a + r0 * b] * fv;
  }
  T* out = C1 + (int64_t)r0 * (i2 + n2 * f);
#pragma unroll
  for (int a = 0; a < 64; ++a)
    if (a < r0) out[a] = (T)acc[a];
}

// out (n1 x N, col-major) = F0 (n1 x K) * C1 (K x N); K <= 64.
// Persistent CTAs, each pinned to one block of 32*RA rows whose F0 rows stay
// in shared memory, looping over (8*CB)-column tiles of C1 (double-buffered
// with cp.async).  Thread (lane, warp) owns rows lane + 32a (a < RA: coalesced
// stores) and columns CB*warp + b (b < CB: broadcast shared reads).  Both
// operands are stored k-contiguous with K padded to Kp (a multiple of the
// 16-byte vector width VK), so VK consecutive k come in one 16-byte load:
// per VK k-steps a thread issues RA + CB vector loads for VK*RA*CB FMAs.
template <typename T, int RA, int CB>
__global__ void __launch_bounds__(256, 1) k_gemm_expand(const T* __restrict__ F0, int64_t n1,
                                                        int K, const T* __restrict__ C1,
                                                        int64_t N, T* __restrict__ out) {
  constexpr int ROWS = 32 * RA, COLS = 8 * CB, VK = 16 / (int)sizeof(T);
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  extern __shared__ __align__(16) unsigned char gemm_smem[];
  const int Kp = (K + VK - 1) / VK * VK;
  T* fa = reinterpret_cast<T*>(gemm_smem);  // [row][Kp]
  T* cbuf = fa + (size_t)ROWS * Kp;         // 2 x [col][Kp]
  const int tile_el = COLS * Kp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nrb = (n1 + ROWS - 1) / ROWS, nct = (N + COLS - 1) / COLS;
  const int64_t rb = blockIdx.x % nrb, cstep = gridDim.x / nrb;
  const int64_t r0 = rb * ROWS;
  if ((int64_t)blockIdx.x >= cstep * nrb) return;
  for (int e = threadIdx.x; e < 2 * tile_el; e += blockDim.x) cbuf[e] = T(0);  // k padding
  __syncthreads();
  // C1 tile ct -> buffer (column j, k) at j*Kp + k; columns past N zeroed
  auto fill = [&](int64_t ct, T* dst) {
    if (ct < nct) {
      const int64_t c0 = ct * COLS;
      const int ncol = (int)((N - c0) < COLS ? (N - c0) : COLS);
      const T* src = C1 + (int64_t)K * c0;
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
      for (int e = threadIdx.x; e < ncol * K; e += blockDim.x) {
        const int j = e / K, k = e - j * K;
        if (sizeof(T) == 4) cpa4(d + (j * Kp + k) * 4, src + e);
        else cpa8(d + (j * Kp + k) * 8, src + e);
      }
      for (int e = ncol * Kp + threadIdx.x; e < tile_el; e += blockDim.x) dst[e] = T(0);
    }
    cpa_commit();
  };
  int64_t ct = blockIdx.x / nrb;
  fill(ct, cbuf);
  for (int e = threadIdx.x; e < ROWS * Kp; e += blockDim.x) {
    const int i = e / Kp, k = e - i * Kp;
    fa[e] = (r0 + i < n1 && k < K) ? F0[r0 + i + n1 * k] : T(0);
  }
  for (int buf = 0; ct < nct; ct += cstep, buf ^= 1) {
    fill(ct + cstep, cbuf + (buf ^ 1) * tile_el);
    cpa_wait1();
    __syncthreads();
    const T* cb = cbuf + buf * tile_el + (size_t)Kp * CB * warp;  // this warp's columns
    T acc[RA][CB];
#pragma unroll
    for (int a = 0; a < RA; ++a)
#pragma unroll
      for (int b = 0; b < CB; ++b) acc[a][b] = T(0);
    for (int k0 = 0; k0 < Kp; k0 += VK) {
      T fr[RA][VK];
#pragma unroll
      for (int a = 0; a < RA; ++a) {
        const V v = *reinterpret_cast<const V*>(fa + (lane + 32 * a) * Kp + k0);
        if constexpr (VK == 4) {
          fr[a][0] = v.x; fr[a][1] = v.y; fr[a][2] = v.z; fr[a][3] = v.w;
        } else {
          fr[a][0] = v.x; fr[a][1] = v.y;
        }
      }
#pragma unroll
      for (int b = 0; b < CB; ++b) {
        const V w = *reinterpret_cast<const V*>(cb + b * Kp + k0);
        T cr[VK];
        if constexpr (VK == 4) {
          cr[0] = w.x; cr[1] = w.y; cr[2] = w.z; cr[3] = w.w;
        } else {
          cr[0] = w.x; cr[1] = w.y;
        }
#pragma unroll
        for (int kk = 0; kk < VK; ++kk)
#pragma unroll
          for (int a = 0; a < RA; ++a) acc[a][b] += fr[a][kk] * cr[kk];
      }
    }
    const int64_t c0 = ct * COLS;
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int64_t col = c0 + CB * warp + b;
      if (col >= N) continue;
#pragma unroll
      for (int a = 0; a < RA; ++a) {
        const int64_t row = r0 + lane + 32 * a;
        if (row < n1) out[row + n1 * col] = acc[a][b];
      }
    }
    __syncthreads();  // buffer `buf` is refilled next iteration
  }
  cpa_wait0();
}

}  // namespace tr
