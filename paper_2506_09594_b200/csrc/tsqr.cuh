// Orthonormal basis of the Krylov block by TSQR + rank-revealing QR of R.
//
// The reference (tenrec/sketch.py:146-185) takes a column-pivoted Householder
// QR of the m x s Krylov block K, keeps the columns with |R_kk| >= 1e-14 ||K||_F
// and re-orthonormalises.  Column pivoting depends on K only through K^T K =
// R^T R, so the same pivot sequence, deflation count and span come out of
//   1. an unpivoted Householder QR of row blocks of K in parallel (k_tsqr_local),
//   2. a QR of the stacked block R factors, then a pivoted QR of the s x s R
//      with the reference's deflation test (k_tsqr_top),
//   3. Z = Q_local * Q_top * Q_piv[:, :s_eff] formed block by block (k_tsqr_form).
// TSQR is backward stable, so the basis is orthonormal to working precision
// however ill-conditioned the Krylov block is.  All arithmetic is fp64.
#pragma once

#include "common.cuh"

namespace tr {

// In-place Householder QR of a rows x cols column-major block in shared memory
// (leading dimension ld).  LAPACK dgeqrf conventions: R on and above the
// diagonal, reflector tails below it (implicit unit head), tau[k] per column.
__device__ inline void smem_householder(double* A, int rows, int cols, int ld, double* tau) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int kmax = rows < cols ? rows : cols;
  for (int k = 0; k < kmax; ++k) {
    if (warp == 0) {
      double sig = 0.0;
      for (int i = k + 1 + lane; i < rows; i += 32) sig += A[i + ld * k] * A[i + ld * k];
      sig = warp_sum(sig);
      const double alpha = A[k + ld * k];
      double t = 0.0, beta = alpha, scale = 0.0;
      if (sig > 0.0) {
        const double nrm = sqrt(alpha * alpha + sig);
        beta = alpha >= 0.0 ? -nrm : nrm;
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
        for (int i = k + 1 + lane; i < rows; i += 32) A[i + ld * k] *= scale;
      }
      __syncwarp();
      if (lane == 0) {
        tau[k] = t;
        A[k + ld * k] = beta;
      }
    }
    __syncthreads();
    const double tk = tau[k];
    if (tk != 0.0) {
      for (int j = k + 1 + warp; j < cols; j += nw) {
        double w = lane == 0 ? A[k + ld * j] : 0.0;
        for (int i = k + 1 + lane; i < rows; i += 32) w += A[i + ld * k] * A[i + ld * j];
        w = warp_sum(w) * tk;
        if (lane == 0) A[k + ld * j] -= w;
        for (int i = k + 1 + lane; i < rows; i += 32) A[i + ld * j] -= w * A[i + ld * k];
      }
    }
    __syncthreads();
  }
}

// C <- Q C with Q = H_0 H_1 ... H_{kmax-1} from smem_householder (reflectors in V).
__device__ inline void smem_apply_q(const double* V, int rows, int kmax, int ldv,
                                    const double* tau, double* C, int ccols, int ldc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = kmax - 1; k >= 0; --k) {
    const double tk = tau[k];
    if (tk != 0.0) {
      for (int j = warp; j < ccols; j += nw) {
        double w = lane == 0 ? C[k + ldc * j] : 0.0;
        for (int i = k + 1 + lane; i < rows; i += 32) w += V[i + ldv * k] * C[i + ldc * j];
        w = warp_sum(w) * tk;
        if (lane == 0) C[k + ldc * j] -= w;
        for (int i = k + 1 + lane; i < rows; i += 32) C[i + ldc * j] -= w * V[i + ldv * k];
      }
    }
    __syncthreads();
  }
}

// Stage 1: block b owns rows [b*RB, min(m, (b+1)*RB)).  Writes its reflectors
// (same layout as K) and tau, and its R factor into rows [b*s, b*s+s) of the
// (nb*s) x s stack (zero below the diagonal / beyond the block's row count).
__global__ void __launch_bounds__(1024) k_tsqr_local(const double* __restrict__ K, int64_t m, int s,
                                                    int RB, double* __restrict__ Vout,
                                                    double* __restrict__ tauout,
                                                    double* __restrict__ Rstack, int64_t ldr) {
  extern __shared__ double tsqr_smem[];
  const int ld = RB + 1;
  double* A = tsqr_smem;
  double* tau = A + (int64_t)ld * s;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int rows = (int)((m - r0) < RB ? (m - r0) : RB);
  for (int e = threadIdx.x; e < rows * s; e += blockDim.x) {
    const int i = e % rows, j = e / rows;
    A[i + ld * j] = K[r0 + i + m * j];
  }
  __syncthreads();
  smem_householder(A, rows, s, ld, tau);
  for (int e = threadIdx.x; e < rows * s; e += blockDim.x) {
    const int i = e % rows, j = e / rows;
    Vout[r0 + i + m * j] = A[i + ld * j];
  }
  for (int k = threadIdx.x; k < s; k += blockDim.x) tauout[(int64_t)blockIdx.x * s + k] = k < rows ? tau[k] : 0.0;
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
    const int i = e % s, j = e / s;
    Rstack[(int64_t)blockIdx.x * s + i + ldr * j] = (i <= j && i < rows) ? A[i + ld * j] : 0.0;
  }
}

// Stage 2 (one CTA): QR of the stack, pivoted QR of its s x s R with the
// reference's deflation rule, and C = Q_top [Q_piv[:, :s_eff]; 0] (zero
// columns beyond s_eff).  info[0] <- s_eff.
//   tol_abs > 0   absolute deflation tolerance (defl_qr(a, tol), sketch.py:146-164)
//   tol_abs == 0  1e-14 ||K||_F (the Krylov basis rule, sketch.py:179)
//   tol_abs < 0   no deflation (every column kept)
//   pivot == 0    plain Householder QR (np.linalg.qr) instead of geqp3 pivoting
//   Rout          optional s x s: rows < s_eff hold R with the pivoting undone
//                 (r_out[:, piv] = r[:s_eff, :]), rows >= s_eff zero
__global__ void __launch_bounds__(1024) k_tsqr_top(const double* __restrict__ Rstack, int nrows,
                                                  int s, double* __restrict__ Cout,
                                                  int64_t* __restrict__ info, double tol_abs,
                                                  int pivot, double* __restrict__ Rout) {
  extern __shared__ double tsqr_smem[];
  const int ld = nrows + 1;
  double* S = tsqr_smem;                       // nrows x s stack -> reflectors
  double* C = S + (int64_t)ld * s;             // nrows x s result
  double* Rp = C + (int64_t)ld * s;            // s x s pivoted work (ld s+1)
  double* tauS = Rp + (int64_t)(s + 1) * s;    // s
  double* tauP = tauS + s;                     // s
  double* cn = tauP + s;                       // s column norms
  __shared__ int perm[64];
  __shared__ int s_eff_s;
  __shared__ int best_s;
  __shared__ double red[32];
  const int lrp = s + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = threadIdx.x; e < nrows * s; e += blockDim.x) {
    const int i = e % nrows, j = e / nrows;
    S[i + ld * j] = Rstack[i + (int64_t)nrows * j];
  }
  __syncthreads();
  smem_householder(S, nrows, s, ld, tauS);
  // ||K||_F = ||R||_F
  double f2 = 0.0;
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
    const int i = e % s, j = e / s;
    if (i <= j) f2 += S[i + ld * j] * S[i + ld * j];
  }
  const double fro = sqrt(block_sum(f2, red));
  const double tol = tol_abs > 0.0 ? tol_abs : tol_abs == 0.0 ? 1e-14 * fro : -1.0;
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
    const int i = e % s, j = e / s;
    Rp[i + lrp * j] = i <= j ? S[i + ld * j] : 0.0;
  }
  if (threadIdx.x < s) perm[threadIdx.x] = threadIdx.x;
  if (threadIdx.x == 0) s_eff_s = s;
  __syncthreads();
  // pivoted Householder on Rp (rank revealing, geqp3-style pivot = max norm)
  for (int k = 0; k < s; ++k) {
    for (int j = k + warp; j < s; j += nw) {
      double t = 0.0;
      for (int i = k + lane; i < s; i += 32) t += Rp[i + lrp * j] * Rp[i + lrp * j];
      t = warp_sum(t);
      if (lane == 0) cn[j] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int best = k;
      if (pivot)
        for (int j = k + 1; j < s; ++j)
          if (cn[j] > cn[best]) best = j;
      const double nb = sqrt(cn[best]);
      if (tol >= 0.0 && (!(nb >= tol) || nb == 0.0)) {
        s_eff_s = k;
      } else {
        const int t = perm[k];
        perm[k] = perm[best];
        perm[best] = t;
      }
      best_s = best;
    }
    __syncthreads();
    if (s_eff_s == k) break;
    const int best = best_s;
    if (best != k)
      for (int i = threadIdx.x; i < s; i += blockDim.x) {
        const double t = Rp[i + lrp * k];
        Rp[i + lrp * k] = Rp[i + lrp * best];
        Rp[i + lrp * best] = t;
      }
    __syncthreads();
    // one Householder step on column k of Rp
    if (warp == 0) {
      double sig = 0.0;
      for (int i = k + 1 + lane; i < s; i += 32) sig += Rp[i + lrp * k] * Rp[i + lrp * k];
      sig = warp_sum(sig);
      const double alpha = Rp[k + lrp * k];
      double t = 0.0, beta = alpha;
      if (sig > 0.0) {
        const double nrm = sqrt(alpha * alpha + sig);
        beta = alpha >= 0.0 ? -nrm : nrm;
        t = (beta - alpha) / beta;
        const double scale = 1.0 / (alpha - beta);
        for (int i = k + 1 + lane; i < s; i += 32) Rp[i + lrp * k] *= scale;
      }
      __syncwarp();
      if (lane == 0) {
        tauP[k] = t;
        Rp[k + lrp * k] = beta;
      }
    }
    __syncthreads();
    const double tk = tauP[k];
    if (tk != 0.0)
      for (int j = k + 1 + warp; j < s; j += nw) {
        double w = lane == 0 ? Rp[k + lrp * j] : 0.0;
        for (int i = k + 1 + lane; i < s; i += 32) w += Rp[i + lrp * k] * Rp[i + lrp * j];
        w = warp_sum(w) * tk;
        if (lane == 0) Rp[k + lrp * j] -= w;
        for (int i = k + 1 + lane; i < s; i += 32) Rp[i + lrp * j] -= w * Rp[i + lrp * k];
      }
    __syncthreads();
  }
  const int se = s_eff_s;
  if (Rout)
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
      const int i = e % s, j = e / s;
      Rout[i + (int64_t)s * perm[j]] = (i < se && i <= j) ? Rp[i + lrp * j] : 0.0;
    }
  // C = [Q_piv[:, :se]; 0] (columns >= se zero), then C <- Q_top C
  for (int e = threadIdx.x; e < nrows * s; e += blockDim.x) {
    const int i = e % nrows, j = e / nrows;
    C[i + ld * j] = (i == j && j < se) ? 1.0 : 0.0;
  }
  __syncthreads();
  smem_apply_q(Rp, s, se, lrp, tauP, C, se, ld);
  smem_apply_q(S, nrows, nrows < s ? nrows : s, ld, tauS, C, se, ld);
  for (int e = threadIdx.x; e < nrows * s; e += blockDim.x) {
    const int i = e % nrows, j = e / nrows;
    Cout[i + (int64_t)nrows * j] = j < se ? C[i + ld * j] : 0.0;
  }
  if (threadIdx.x == 0) info[0] = se;
}

// Stage 3: Z rows of block b = Q_b [C_b; 0] with C_b = C[b*s : b*s+s, :].
template <typename T>
__global__ void __launch_bounds__(1024) k_tsqr_form(const double* __restrict__ V,
                                                   const double* __restrict__ tauin,
                                                   const double* __restrict__ C, int nrows_c,
                                                   int64_t m, int s, int RB,
                                                   double* __restrict__ Z, T* __restrict__ Zt) {
  extern __shared__ double tsqr_smem[];
  const int ld = RB + 1;
  double* Vs = tsqr_smem;
  double* Zs = Vs + (int64_t)ld * s;
  double* tau = Zs + (int64_t)ld * s;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int rows = (int)((m - r0) < RB ? (m - r0) : RB);
  for (int e = threadIdx.x; e < rows * s; e += blockDim.x) {
    const int i = e % rows, j = e / rows;
    Vs[i + ld * j] = V[r0 + i + m * j];
    Zs[i + ld * j] = i < s ? C[(int64_t)blockIdx.x * s + i + (int64_t)nrows_c * j] : 0.0;
  }
  for (int k = threadIdx.x; k < s; k += blockDim.x) tau[k] = tauin[(int64_t)blockIdx.x * s + k];
  __syncthreads();
  smem_apply_q(Vs, rows, rows < s ? rows : s, ld, tau, Zs, s, ld);
  for (int e = threadIdx.x; e < rows * s; e += blockDim.x) {
    const int i = e % rows, j = e / rows;
    const double z = Zs[i + ld * j];
    Z[r0 + i + m * j] = z;
    if (Zt) Zt[r0 + i + m * j] = (T)z;
  }
}

}  // namespace tr
