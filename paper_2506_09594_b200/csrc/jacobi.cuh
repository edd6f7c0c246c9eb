// Warp-level one-sided (Hestenes) Jacobi SVD of a small complex matrix.
//
// One warp factors an r0 x r1 matrix (r0, r1 <= 32): lane j keeps column j in
// registers, the accumulated right rotations V live in shared memory.  Each
// round pairs every lane with its round-robin partner; partners exchange
// columns by shuffles, compute the same rotation bit-for-bit (identical
// operand order) and update their own column.  No block barriers, no
// cross-lane reductions -- the latency of a round is a few hundred cycles.
//
// On return X <- X V has orthogonal columns (norm = singular value) and V is
// unitary: X_in = X_out V^H.
#pragma once

#include "common.cuh"

namespace tr {

constexpr int kJW = 32;      // max columns / rows handled by one warp
constexpr int kVld = kJW + 1; // padded row stride of V in shared memory

// xr/xi: this lane's column (rows < r0).  Vr/Vi: [k * kVld + j] = V[k][j]
// (row k, column j), Wr/Wi the second buffer of the same size; on return
// Vr/Vi point at the buffer holding V (the pointers are swapped per round).
__device__ inline void warp_jacobi(double (&xr)[kJW], double (&xi)[kJW], double*& Vr, double*& Vi,
                                   double* Wr, double* Wi, int r0, int r1, int max_sweeps = 40) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < r1; ++k) {
    if (lane < r1) {
      Vr[k * kVld + lane] = (k == lane) ? 1.0 : 0.0;
      Vi[k * kVld + lane] = 0.0;
    }
  }
  double fro = 0.0;
#pragma unroll
  for (int i = 0; i < kJW; ++i)
    if (i < r0 && lane < r1) fro += xr[i] * xr[i] + xi[i] * xi[i];
  fro = warp_sum(fro);
  const int ne = r1 + (r1 & 1);
  __syncwarp();
  for (int sweep = 0; sweep < max_sweeps && ne >= 2; ++sweep) {
    int rotated = 0;
    for (int rnd = 0; rnd < ne - 1; ++rnd) {
      // my slot k in this round, and my partner's player index
      int k;
      if (lane == 0) k = 0;
      else k = ((lane - 1 - rnd) % (ne - 1) + (ne - 1)) % (ne - 1) + 1;
      const int partner = rr_player(ne - 1 - k, rnd, ne);
      const bool active = lane < r1 && partner < r1 && lane < ne;
      const int src = (partner < 32) ? partner : lane;
      const bool is_p = lane < partner;
      double na = 0.0;
#pragma unroll
      for (int i = 0; i < kJW; ++i)
        if (i < r0) na += xr[i] * xr[i] + xi[i] * xi[i];
      const double nb = __shfl_sync(0xffffffffu, na, src);
      double gr = 0.0, gi = 0.0;  // gamma = sum conj(x_p) x_q
#pragma unroll
      for (int i = 0; i < kJW; ++i) {
        const double pr = __shfl_sync(0xffffffffu, xr[i], src);
        const double pi = __shfl_sync(0xffffffffu, xi[i], src);
        if (i < r0) {
          const double ar = is_p ? xr[i] : pr, ai = is_p ? xi[i] : pi;
          const double br = is_p ? pr : xr[i], bi = is_p ? pi : xi[i];
          gr += ar * br + ai * bi;
          gi += ar * bi - ai * br;
        }
      }
      const double al = is_p ? na : nb, be = is_p ? nb : na;
      const double g = sqrt(gr * gr + gi * gi);
      double c = 1.0, s = 0.0, phr = 1.0, phi = 0.0;
      if (active && g > 1e-15 * sqrt(al * be) && g > 1e-17 * fro) {  // fro = ||X||_F^2
        const double zeta = (be - al) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        c = 1.0 / sqrt(1.0 + t * t);
        s = c * t;
        phr = gr / g;
        phi = gi / g;
        rotated = 1;
      }
      // [x_p, x_q] <- [x_p, x_q] [[c, s e^{i phi}], [-s e^{-i phi}, c]]
      // lane p: x_p - s e^{-i phi} x_q ; lane q: s e^{i phi} x_p + c x_q
      const double fr = s * phr, fi = is_p ? -s * phi : s * phi;  // coefficient on partner
      const double sg = is_p ? -1.0 : 1.0;
#pragma unroll
      for (int i = 0; i < kJW; ++i) {
        const double pr = __shfl_sync(0xffffffffu, xr[i], src);
        const double pi = __shfl_sync(0xffffffffu, xi[i], src);
        if (i < r0 && s != 0.0) {
          const double ur = fr * pr - fi * pi, ui = fr * pi + fi * pr;
          xr[i] = c * xr[i] + sg * ur;
          xi[i] = c * xi[i] + sg * ui;
        }
      }
      // V columns: same rotation; read the current buffer, write the other one
      if (lane < r1) {
        for (int kk = 0; kk < r1; ++kk) {
          const double orr = Vr[kk * kVld + lane], oi = Vi[kk * kVld + lane];
          double nr = orr, ni = oi;
          if (s != 0.0) {
            const double pr = Vr[kk * kVld + src], pi = Vi[kk * kVld + src];
            const double ur = fr * pr - fi * pi, ui = fr * pi + fi * pr;
            nr = c * orr + sg * ur;
            ni = c * oi + sg * ui;
          }
          Wr[kk * kVld + lane] = nr;
          Wi[kk * kVld + lane] = ni;
        }
      }
      __syncwarp();
      double* t = Vr;
      Vr = Wr;
      Wr = t;
      t = Vi;
      Vi = Wi;
      Wi = t;
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
  }
}

// One warp per face: X (r0 x r1 complex, column-major, faces + f*r0*r1)
// becomes X diag(prox(sigma)/sigma) V^H = U prox(S) V^H.  r0, r1 <= 32.
__global__ void __launch_bounds__(128) k_face_svt_warp(double2* __restrict__ faces, int r0, int r1,
                                                       int64_t nfaces, Penalty pen, double tau) {
  extern __shared__ double jac_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  double* Vr = jac_smem + (size_t)warp * 4 * kJW * kVld;
  double* Vi = Vr + kJW * kVld;
  double* Yr = Vi + kJW * kVld;  // second V buffer during Jacobi, then X diag(w)
  double* Yi = Yr + kJW * kVld;
  if (f >= nfaces) return;
  double2* src = faces + f * r0 * r1;
  double xr[kJW], xi[kJW];
#pragma unroll
  for (int i = 0; i < kJW; ++i) {
    xr[i] = 0.0;
    xi[i] = 0.0;
    if (i < r0 && lane < r1) {
      const double2 v = src[i + r0 * lane];
      xr[i] = v.x;
      xi[i] = v.y;
    }
  }
  double* Vr0 = Vr;
  warp_jacobi(xr, xi, Vr, Vi, Yr, Yi, r0, r1);
  if (Vr != Vr0) {  // V ended in the second buffer: Y goes into the first
    Yr = Vr0;
    Yi = Vr0 + kJW * kVld;
  }
  double s2 = 0.0;
#pragma unroll
  for (int i = 0; i < kJW; ++i)
    if (i < r0) s2 += xr[i] * xr[i] + xi[i] * xi[i];
  const double sg = sqrt(s2);
  const double w = (lane < r1 && sg > 0.0) ? prox(pen, tau, sg) / sg : 0.0;
#pragma unroll
  for (int i = 0; i < kJW; ++i)
    if (i < r0) {
      Yr[i * kVld + lane] = w * xr[i];
      Yi[i * kVld + lane] = w * xi[i];
    }
  __syncwarp();
  // out[:, k] (lane k) = sum_j Y[:, j] conj(V[k][j])
  if (lane < r1) {
    for (int i = 0; i < r0; ++i) {
      double ar = 0.0, ai = 0.0;
      for (int j = 0; j < r1; ++j) {
        const double yr = Yr[i * kVld + j], yi = Yi[i * kVld + j];
        const double vr = Vr[lane * kVld + j], vi = Vi[lane * kVld + j];
        ar += yr * vr + yi * vi;
        ai += yi * vr - yr * vi;
      }
      src[i + r0 * lane] = make_double2(ar, ai);
    }
  }
}

}  // namespace tr

namespace tr {

// Rayleigh-Ritz with the warp Jacobi (s_eff <= 32): eigenvectors of the
// symmetric PSD M = W^T W (one-sided Jacobi on M: x_j = lambda_j v_j), top r
// in descending order, F = Z V_top, canonical sign per column (largest-|entry|
// positive, first index on ties).  Replaces k_ritz for small Krylov blocks.
template <typename T>
__global__ void __launch_bounds__(256) k_ritz_warp(const double* __restrict__ Mfull, int s,
                                                    const double* __restrict__ Z, int64_t m, int r,
                                                    double* __restrict__ V, double* __restrict__ F,
                                                    T* __restrict__ Ft, int64_t* __restrict__ info) {
  extern __shared__ double jac_smem[];
  __shared__ double lam[kJW];
  __shared__ int order[kJW];
  __shared__ double sgn[64];
  __shared__ int vbuf;
  __shared__ double Vt[kJW * 64];  // V_top, [j + kJW * k]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n = (int)info[0];
  if (warp == 0) {
    double xr[kJW], xi[kJW];
#pragma unroll
    for (int i = 0; i < kJW; ++i) {
      xr[i] = (i < n && lane < n) ? Mfull[i + s * lane] : 0.0;
      xi[i] = 0.0;
    }
    double* Vr = jac_smem;
    double* Vi = Vr + kJW * kVld;
    double* Wr = Vi + kJW * kVld;
    double* Wi = Wr + kJW * kVld;
    warp_jacobi(xr, xi, Vr, Vi, Wr, Wi, n, n);
    double nrm = 0.0;
#pragma unroll
    for (int i = 0; i < kJW; ++i) nrm += xr[i] * xr[i];
    lam[lane] = sqrt(nrm);
    if (lane == 0) vbuf = (Vr == jac_smem) ? 0 : 2;
    __syncwarp();
    if (lane == 0) {
      for (int i = 0; i < n; ++i) order[i] = i;
      for (int i = 1; i < n; ++i) {
        const int oi = order[i];
        int j = i - 1;
        while (j >= 0 && lam[order[j]] < lam[oi]) {
          order[j + 1] = order[j];
          --j;
        }
        order[j + 1] = oi;
      }
    }
  }
  __syncthreads();
  const int re = r < n ? r : n;
  const double* Vr = jac_smem + vbuf * kJW * kVld;
  for (int e = threadIdx.x; e < kJW * r; e += blockDim.x) {
    const int j = e % kJW, k = e / kJW;
    Vt[e] = (k < re && j < n) ? Vr[j * kVld + order[k]] : 0.0;
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < m * r; e += blockDim.x) {
    const int64_t i = e % m;
    const int k = (int)(e / m);
    double f = 0.0;
    for (int j = 0; j < n; ++j) f += Z[i + m * j] * Vt[j + kJW * k];
    F[e] = f;
  }
  __syncthreads();
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
  __syncthreads();
  for (int64_t e = threadIdx.x; e < m * r; e += blockDim.x) {
    const double f = F[e] * sgn[e / m];
    F[e] = f;
    Ft[e] = (T)f;
  }
  for (int e = threadIdx.x; e < s * r; e += blockDim.x) {
    const int j = e % s, k = e / s;
    V[e] = (j < kJW) ? Vt[j + kJW * k] * sgn[k] : 0.0;
  }
  if (threadIdx.x == 0) info[1] = re;
}

}  // namespace tr
