// Orthonormal basis of the Krylov block in ONE launch: a 4-CTA cluster TSQR.
//
// Same mathematics as tsqr.cuh (tenrec/sketch.py:146-185): unpivoted
// Householder QR of the m x s block K, a pivoted QR of its R with the
// reference's deflation rule |R_kk| >= 1e-14 ||K||_F, and
// Z = Q_K [Q_piv[:, :s_eff]; 0].  What changes is the execution model (the
// 3-kernel TSQR spent ~160 us per stage on barriers and serial column loops):
//   * CTA c of the cluster owns rows [256 c, 256 c + 256); warp w holds
//     columns w and w + 16 in registers, lane l rows l + 32 r (r < 8);
//   * a Householder step is one warp reduction per column (the Gram entry of
//     column k with every other column over the rows below k), two CTA
//     barriers, and the reflector / v^T a_j / rank-1 update all follow from
//     that Gram row -- no second reduction;
//   * applying a factor's reflectors to another block needs no barrier at
//     all: the reflectors sit in shared memory and every warp walks its own
//     columns through them;
//   * the four R factors meet in CTA 0 through distributed shared memory, the
//     pivoted QR of the s x s R runs in one warp, and the C blocks go back the
//     same way; every CTA then forms its rows of Z.
// All arithmetic is fp64; the reduction order is fixed (deterministic).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace tr {

#ifdef TR_ORTH_PROBE
__device__ long long g_orth_probe[8];
#define OC_MARK(i) \
  if (threadIdx.x == 0 && cl.block_rank() == 0) g_orth_probe[i] = clock64() - oc_t0;
#else
#define OC_MARK(i)
#endif

constexpr int kOcThreads = 512;  // 16 warps
constexpr int kOcWarps = kOcThreads / 32;
constexpr int kOcRows = 256;          // rows per CTA
constexpr int kOcRpl = kOcRows / 32;  // rows per lane
constexpr int kOcCtas = 4;            // cluster size: m <= 1024
constexpr int kOcS = 32;              // max block width (2 columns per warp)
constexpr int kOcStack = kOcCtas * kOcS;  // max stacked rows
constexpr int kOcLdp = kOcS + 1;          // pivoted-R / E column stride

// a[r] for a runtime r (keeps a in registers)
template <int N>
__device__ __forceinline__ double selr(const double (&a)[N], int r) {
  double v = 0.0;
#pragma unroll
  for (int q = 0; q < N; ++q) v = (q == r) ? a[q] : v;
  return v;
}

// In-place Householder QR of the nrows x s block held column-wise (a[c][r] =
// row lane + 32 r of column warp + kOcWarps c).  LAPACK conventions: R on and
// above the diagonal, reflector tails below (unit head implied), tau[k] in smem.
// colk: 32 RPL doubles, gk: kOcS doubles of scratch.
template <int RPL>
__device__ inline void col_householder(double (&a)[2][RPL], int nrows, int s, double* colk,
                                       double* gk, double* tau) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kmax = nrows < s ? nrows : s;
  if (kmax <= 0) return;
#pragma unroll
  for (int c = 0; c < 2; ++c)  // publish column 0
    if (warp + kOcWarps * c == 0)
#pragma unroll
      for (int r = 0; r < RPL; ++r) colk[lane + 32 * r] = a[c][r];
  __syncthreads();
  for (int k = 0; k < kmax; ++k) {
    double cv[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) cv[r] = colk[lane + 32 * r];
    const double alpha = colk[k];
    // phase A: Gram entries of column k with my columns over rows > k
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int j = warp + kOcWarps * c;
      if (j >= k && j < s) {  // warp-uniform
        double p = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int row = lane + 32 * r;
          if (row > k && row < nrows) p += cv[r] * a[c][r];
        }
        p = warp_sum(p);
        if (lane == 0) gk[j] = p;
      }
    }
    __syncthreads();
    const double sig = gk[k];
    double tk = 0.0, beta = alpha, scale = 0.0;
    if (sig > 0.0) {
      const double nrm = sqrt(alpha * alpha + sig);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tk = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    const int kl = k & 31, kr = k >> 5;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int j = warp + kOcWarps * c;
      if (j > k && j < s) {
        const double akj = __shfl_sync(0xffffffffu, selr(a[c], kr), kl);
        const double w = tk * (akj + scale * gk[j]);  // tau v^T a_j
        const double ws = w * scale;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int row = lane + 32 * r;
          if (row > k && row < nrows) a[c][r] -= cv[r] * ws;
          else if (row == k) a[c][r] -= w;
        }
      } else if (j == k) {
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int row = lane + 32 * r;
          if (row > k && row < nrows) a[c][r] = cv[r] * scale;
          else if (row == k) a[c][r] = beta;
        }
      }
      if (j == k + 1 && j < s)  // publish the next pivot column (all reads of colk are done)
#pragma unroll
        for (int r = 0; r < RPL; ++r) colk[lane + 32 * r] = a[c][r];
    }
    if (threadIdx.x == 0) tau[k] = tk;
    __syncthreads();
  }
}

// c <- Q c for Q = H_0 ... H_{kmax-1}: reflector k = column k of V (column-major,
// stride ldv, rows < nrows; unit head), taus in smem.  Each warp walks its own
// columns of c (cc[q][r] = row lane + 32 r of column warp + kOcWarps q) through
// the reflectors; no barriers.
template <int RPL>
__device__ inline void col_apply_q(const double* V, int ldv, int nrows, int kmax, const double* tau,
                                   double (&cc)[2][RPL], int ncols) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = kmax - 1; k >= 0; --k) {
    const double tk = tau[k];
    if (tk == 0.0) continue;
    double v[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int row = lane + 32 * r;
      v[r] = row == k ? 1.0 : ((row > k && row < nrows) ? V[k * ldv + row] : 0.0);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = warp + kOcWarps * q;
      if (j < ncols) {
        double p = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) p += v[r] * cc[q][r];
        p = tk * warp_sum(p);
#pragma unroll
        for (int r = 0; r < RPL; ++r) cc[q][r] -= v[r] * p;
      }
    }
  }
}

// K (m x s, column-major fp64) -> Z (m x s; columns >= s_eff zero) and Zt.
// info[0] <- s_eff.  Launch: one cluster of kOcCtas CTAs x kOcThreads.
template <typename T>
__global__ void __cluster_dims__(kOcCtas, 1, 1) __launch_bounds__(kOcThreads, 1)
    k_orth_cluster(const double* __restrict__ K, int64_t m, int s, double* __restrict__ Z,
                   T* __restrict__ Zt, int64_t* __restrict__ info, float* __restrict__ zhi,
                   float* __restrict__ zlo) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double oc_smem[];
  double* vloc = oc_smem;                // kOcS x kOcRows: local reflectors (col-major)
  double* stk = vloc + kOcS * kOcRows;   // kOcS x kOcStack: R stack, then its reflectors
  double* cblk = stk + kOcS * kOcStack;  // kOcS x kOcS: this CTA's C block (col-major)
  double* rp = cblk + kOcS * kOcS;       // kOcS x kOcLdp: pivoted R (col-major)
  double* eb = rp + kOcS * kOcLdp;       // kOcS x kOcLdp: Q_piv[:, :se]
  double* colk = eb + kOcS * kOcLdp;     // kOcRows
  double* gk = colk + kOcRows;           // kOcS
  double* tau = gk + kOcS;               // kOcS (local)
  double* taut = tau + kOcS;             // kOcS (stack)
  double* taup = taut + kOcS;            // kOcS (pivoted)
  double* bscr = taup + kOcS;            // 32 (block_sum scratch)
  __shared__ int se_s;
  const int c = (int)cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = (int64_t)c * kOcRows;
  const int64_t left = m - row0;
  const int rows_c = left <= 0 ? 0 : (left < kOcRows ? (int)left : kOcRows);
#ifdef TR_ORTH_PROBE
  const long long oc_t0 = clock64();
#endif
  // cluster-wide "all CTAs running" before the first remote shared-memory store
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

  // ---- 1. local QR of this CTA's rows ----
  double a[2][kOcRpl];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = warp + kOcWarps * q;
#pragma unroll
    for (int r = 0; r < kOcRpl; ++r) {
      const int row = lane + 32 * r;
      a[q][r] = (row < rows_c && j < s) ? K[row0 + row + m * j] : 0.0;
    }
  }
  col_householder<kOcRpl>(a, rows_c, s, colk, gk, tau);
  OC_MARK(0)
  const int kloc = rows_c < s ? rows_c : s;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = warp + kOcWarps * q;
#pragma unroll
    for (int r = 0; r < kOcRpl; ++r) vloc[j * kOcRows + lane + 32 * r] = a[q][r];
  }
  // R_c (rows < s) -> CTA 0's stack rows c*s .. c*s+s-1 (col-major, stride kOcStack)
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  {
    double* st0 = cl.map_shared_rank(stk, 0);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = warp + kOcWarps * q;
      if (j < s && lane < s)  // row lane (r = 0); s <= 32
        st0[j * kOcStack + c * s + lane] = (lane <= j && lane < rows_c) ? a[q][0] : 0.0;
    }
  }
  cl.sync();
  OC_MARK(1)

  if (c == 0) {
    // ---- 2. QR of the stack (kOcCtas*s x s) ----
    constexpr int RS = kOcStack / 32;
    const int nst = kOcCtas * s;
    double y[2][RS];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = warp + kOcWarps * q;
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const int row = lane + 32 * r;
        y[q][r] = (row < nst && j < s) ? stk[j * kOcStack + row] : 0.0;
      }
    }
    col_householder<RS>(y, nst, s, colk, gk, taut);
    double f = 0.0;  // ||K||_F^2 = ||R||_F^2
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = warp + kOcWarps * q;
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const int row = lane + 32 * r;
        if (j < s) {
          stk[j * kOcStack + row] = y[q][r];  // reflectors below the diagonal
          if (row <= j) f += y[q][r] * y[q][r];
          if (row < s) rp[j * kOcLdp + row] = row <= j ? y[q][r] : 0.0;
        }
      }
    }
    const double tol = 1e-14 * sqrt(block_sum(f, bscr));  // barriers: rp, stk ready
    OC_MARK(2)
    // ---- 3. pivoted QR of R (one warp) ----
    if (warp == 0) {
      int se = s;
      for (int k = 0; k < s; ++k) {
        double cn = -1.0;
        if (lane >= k && lane < s) {  // lane = column
          cn = 0.0;
          for (int r = k; r < s; ++r) cn += rp[lane * kOcLdp + r] * rp[lane * kOcLdp + r];
        }
        double best = cn;
        int bidx = lane;
        for (int o = 16; o > 0; o >>= 1) {  // max norm, lowest index on ties
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
          if (ob > best || (ob == best && oi < bidx)) {
            best = ob;
            bidx = oi;
          }
        }
        const double nb = sqrt(best > 0.0 ? best : 0.0);
        if (!(nb >= tol) || nb == 0.0) {
          se = k;
          break;
        }
        if (bidx != k && lane < s) {  // swap columns k and bidx (lane = row)
          const double t0 = rp[k * kOcLdp + lane];
          rp[k * kOcLdp + lane] = rp[bidx * kOcLdp + lane];
          rp[bidx * kOcLdp + lane] = t0;
        }
        __syncwarp();
        const double av = (lane > k && lane < s) ? rp[k * kOcLdp + lane] : 0.0;
        const double sig = warp_sum(av * av);
        const double alpha = rp[k * kOcLdp + k];
        double tk = 0.0, beta = alpha, scale = 0.0;
        if (sig > 0.0) {
          const double nrm = sqrt(alpha * alpha + sig);
          beta = alpha >= 0.0 ? -nrm : nrm;
          tk = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        __syncwarp();
        if (lane > k && lane < s) rp[k * kOcLdp + lane] = av * scale;
        if (lane == k) rp[k * kOcLdp + k] = beta;
        if (lane == 0) taup[k] = tk;
        __syncwarp();
        if (lane > k && lane < s && tk != 0.0) {  // lane = column j
          double w = rp[lane * kOcLdp + k];
          for (int r = k + 1; r < s; ++r) w += rp[k * kOcLdp + r] * rp[lane * kOcLdp + r];
          w *= tk;
          rp[lane * kOcLdp + k] -= w;
          for (int r = k + 1; r < s; ++r) rp[lane * kOcLdp + r] -= w * rp[k * kOcLdp + r];
        }
        __syncwarp();
      }
      // E = Q_piv [I_se; 0] (s x se), lane = column of E
      if (lane < se)
        for (int r = 0; r < s; ++r) eb[lane * kOcLdp + r] = r == lane ? 1.0 : 0.0;
      __syncwarp();
      for (int k = se - 1; k >= 0; --k) {
        const double tk = taup[k];
        if (tk != 0.0 && lane < se) {
          double w = eb[lane * kOcLdp + k];
          for (int r = k + 1; r < s; ++r) w += rp[k * kOcLdp + r] * eb[lane * kOcLdp + r];
          w *= tk;
          eb[lane * kOcLdp + k] -= w;
          for (int r = k + 1; r < s; ++r) eb[lane * kOcLdp + r] -= w * rp[k * kOcLdp + r];
        }
        __syncwarp();
      }
      if (lane == 0) se_s = se;
    }
    __syncthreads();
    OC_MARK(3)
    const int se = se_s;
    // ---- 4. C = Q_stack [E; 0] (kOcCtas*s x se); rows -> the owning CTAs ----
    double cc[2][RS];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = warp + kOcWarps * q;
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const int row = lane + 32 * r;
        cc[q][r] = (row < s && j < se) ? eb[j * kOcLdp + row] : 0.0;
      }
    }
    col_apply_q<RS>(stk, kOcStack, nst, nst < s ? nst : s, taut, cc, se);
    OC_MARK(4)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = warp + kOcWarps * q;
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const int row = lane + 32 * r;
        if (row < nst && j < s) {
          double* cb = cl.map_shared_rank(cblk, row / s);
          cb[j * kOcS + row % s] = j < se ? cc[q][r] : 0.0;
        }
      }
    }
    if (threadIdx.x == 0)
      for (int d = 0; d < kOcCtas; ++d) *cl.map_shared_rank(&se_s, d) = se;
  }
  cl.sync();

  OC_MARK(5)
  // ---- 5. Z rows of this CTA = Q_c [C_c; 0] ----
  const int se = se_s;
  double zz[2][kOcRpl];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = warp + kOcWarps * q;
#pragma unroll
    for (int r = 0; r < kOcRpl; ++r) {
      const int row = lane + 32 * r;
      zz[q][r] = (row < s && j < se) ? cblk[j * kOcS + row] : 0.0;
    }
  }
  col_apply_q<kOcRpl>(vloc, kOcRows, rows_c, kloc, tau, zz, se);
  OC_MARK(6)
  // zhi / zlo (optional): the tf32 high / low split of Z as an m x 32 block (zero
  // columns beyond s_eff) for the tensor-core projection -- k_split_z fused here
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = warp + kOcWarps * q;  // < 32: the two passes cover every column of the split
#pragma unroll
    for (int r = 0; r < kOcRpl; ++r) {
      const int row = lane + 32 * r;
      if (row < rows_c) {
        const double v = (j < s && j < se) ? zz[q][r] : 0.0;
        if (j < s) {
          Z[row0 + row + m * j] = v;
          Zt[row0 + row + m * j] = (T)v;
        }
        if (zhi != nullptr) {
          const float hi = __uint_as_float(__float_as_uint((float)v) & 0xFFFFE000u);
          zhi[row0 + row + m * j] = hi;
          zlo[row0 + row + m * j] = (float)(v - (double)hi);
        }
      }
    }
  }
  if (c == 0 && threadIdx.x == 0) info[0] = se;
  cl.sync();  // no CTA exits while a peer may still address its shared memory
}

constexpr size_t kOcSmem = (size_t)(kOcS * kOcRows + kOcS * kOcStack + kOcS * kOcS +
                                    2 * kOcS * kOcLdp + kOcRows + 5 * kOcS + 32) *
                           sizeof(double);

}  // namespace tr
