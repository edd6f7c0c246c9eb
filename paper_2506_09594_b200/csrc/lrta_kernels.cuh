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
          const int64_t lo = c % sk.inner, f = c / sk.inner;
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

// Rayleigh-Ritz (sketch.py:261-265): eigenvectors of M = W^T W by parallel
// cyclic Jacobi, descending order, F = Z V; then the canonical sign (largest
// |entry| of every factor column positive, first index on ties).
template <typename T>
__global__ void __launch_bounds__(512) k_ritz(const double* __restrict__ Mfull, int s,
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
      // columns: A <- A J, Q <- Q J
      for (int e = threadIdx.x; e < npairs * 64; e += blockDim.x) {
        const int k = e / 64, i = e % 64;
        const int p = pp[k], q = pq[k];
        const double c = cs_c[k], sn = cs_s[k];
        if (sn != 0.0) {
          const double ap = A[i + ld * p], aq = A[i + ld * q];
          A[i + ld * p] = c * ap - sn * aq;
          A[i + ld * q] = sn * ap + c * aq;
          const double qp = Q[i + ld * p], qq = Q[i + ld * q];
          Q[i + ld * p] = c * qp - sn * qq;
          Q[i + ld * q] = sn * qp + c * qq;
        }
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int e = threadIdx.x; e < npairs * 64; e += blockDim.x) {
        const int k = e / 64, j = e % 64;
        const int p = pp[k], q = pq[k];
        const double c = cs_c[k], sn = cs_s[k];
        if (sn != 0.0) {
          const double ap = A[p + ld * j], aq = A[q + ld * j];
          A[p + ld * j] = c * ap - sn * aq;
          A[q + ld * j] = sn * ap + c * aq;
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
    if (threadIdx.x == 0) atomicAdd(&g_dbg[0], 1);  // ritz sweeps
    if (!any) break;
  }
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
template <typename T>
__global__ void k_expand_mode1(const double* __restrict__ core, int r0, int r1, int64_t nf,
                               const double* __restrict__ F1, int64_t n2, T* __restrict__ C1) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)r0 * n2 * nf) return;
  const int a = (int)(t % r0);
  const int64_t rest = t / r0;
  const int64_t i2 = rest % n2, f = rest / n2;
  double acc = 0.0;
  for (int b = 0; b < r1; ++b) acc += core[a + (int64_t)r0 * (b + (int64_t)r1 * f)] * F1[i2 + n2 * b];
  C1[t] = (T)acc;
}

// out (n1 x N, col-major) = F0 (n1 x K) * C1 (K x N); K <= 64.
// 64x64 CTA tile, 256 threads, 4x4 register tile per thread.
template <typename T>
__global__ void __launch_bounds__(256) k_gemm_expand(const T* __restrict__ F0, int64_t n1,
                                                     int K, const T* __restrict__ C1,
                                                     int64_t N, T* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char gemm_smem[];
  T(*fa)[65] = reinterpret_cast<T(*)[65]>(gemm_smem);                    // [k][row]
  T(*cb)[65] = reinterpret_cast<T(*)[65]>(gemm_smem + 64 * 65 * sizeof(T));  // [k][col]
  const int64_t r0 = (int64_t)blockIdx.x * 64, c0 = (int64_t)blockIdx.y * 64;
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int i = e % 64, k = e / 64;
    fa[k][i] = (k < K && r0 + i < n1) ? F0[r0 + i + n1 * k] : T(0);
    const int kk = e % 64, j = e / 64;
    cb[kk][j] = (kk < K && c0 + j < N) ? C1[kk + (int64_t)K * (c0 + j)] : T(0);
  }
  __syncthreads();
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
  for (int k = 0; k < K; ++k) {
    T fr[4], cr[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) fr[a] = fa[k][tx + 16 * a];
#pragma unroll
    for (int b = 0; b < 4; ++b) cr[b] = cb[k][ty + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] += fr[a] * cr[b];
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int64_t col = c0 + ty + 16 * b;
    if (col >= N) continue;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t row = r0 + tx + 16 * a;
      if (row < n1) out[row + n1 * col] = acc[a][b];
    }
  }
}

}  // namespace tr
