// Transform-domain singular value thresholding of a small core tensor
// (tenrec/shrink.py:76-106 with the transforms of tenrec/transform.py:109-165).
//
// The trailing-mode transform is a chain of mode products with a complex
// matrix U_i (DFT, orthonormal DCT-II or an explicit unitary-up-to-scale
// matrix); the inverse uses U_i^H / alpha_i in reverse order.  Each face is
// thresholded by a one-sided (Hestenes) complex Jacobi SVD in one CTA; the FFT
// conjugate-mirror faces are then overwritten by the conjugate of their
// canonical partner exactly as the reference assembles them.
#pragma once

#include "common.cuh"
#include "lrta_kernels.cuh"
#include "prox.cuh"

namespace tr {

struct cplx {
  double re, im;
};

__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__device__ __forceinline__ cplx cconj(cplx a) { return {a.re, -a.im}; }

// U[k*n + j] for kind 0 = DFT, 1 = orthonormal DCT-II (tenrec/transform.py:115-121).
__global__ void k_build_transform(int kind, int n, cplx* __restrict__ U) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int k = e / n, j = e % n;
  if (kind == 0) {
    // exp(-2 pi i k j / n), argument reduced exactly modulo n
    const long long kj = ((long long)k * j) % n;
    double s, c;
    sincospi(-2.0 * (double)kj / (double)n, &s, &c);
    U[e] = {c, s};
  } else {
    double c = cospi((double)(2 * j + 1) * (double)k / (2.0 * n)) * sqrt(2.0 / n);
    if (k == 0) c *= sqrt(0.5);
    U[e] = {c, 0.0};
  }
}

// FFT faces: every non-canonical face (mirror < f) becomes conj(face[mirror]).
// trailing dims t[0..nt) column-major flattening (tenrec/transform.py:169-183).
struct Trailing {
  int nt;
  int64_t d[8];
};

__device__ __forceinline__ int64_t mirror_face(int64_t f, const Trailing& tr) {
  int64_t out = 0, mul = 1, rem = f;
  for (int i = 0; i < tr.nt; ++i) {
    const int64_t n = tr.d[i];
    const int64_t t = rem % n;
    rem /= n;
    out += ((n - t) % n) * mul;
    mul *= n;
  }
  return out;
}

// One CTA per face: X (r0 x r1 complex, column-major at faces + f*r0*r1) is
// replaced by U prox(S) V^H (one-sided Jacobi).  The working copy X and the
// rotations V live in shared memory (r0, r1 <= 64: k_face_svt) or in global
// scratch (larger faces, the deterministic t-SVT of a whole tensor:
// k_face_svt_g); wsc holds r1 weights.
__device__ inline void face_svt_body(cplx* __restrict__ X, cplx* __restrict__ V,
                                     double* __restrict__ wsc, cplx* __restrict__ src, int r0,
                                     int r1, Penalty pen, double tau) {
  __shared__ int rot_any;
  for (int e = threadIdx.x; e < r0 * r1; e += blockDim.x) X[e] = src[e];
  for (int e = threadIdx.x; e < r1 * r1; e += blockDim.x)
    V[e] = {(e % r1) == (e / r1) ? 1.0 : 0.0, 0.0};
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  __shared__ double fred[32];
  double f2 = 0.0;
  for (int e = threadIdx.x; e < r0 * r1; e += blockDim.x) f2 += X[e].re * X[e].re + X[e].im * X[e].im;
  const double fnorm2 = block_sum(f2, fred);
  const int ne = r1 + (r1 & 1);
  const int npairs = ne / 2;
  for (int sweep = 0; sweep < 60 && ne >= 2; ++sweep) {
    if (threadIdx.x == 0) rot_any = 0;
    __syncthreads();
    for (int rnd = 0; rnd < ne - 1; ++rnd) {
      for (int k = warp; k < npairs; k += nw) {
        int p = rr_player(k, rnd, ne), q = rr_player(ne - 1 - k, rnd, ne);
        if (p > q) { const int t = p; p = q; q = t; }
        if (q >= r1) continue;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        for (int i = lane; i < r0; i += 32) {
          const cplx xp = X[i + r0 * p], xq = X[i + r0 * q];
          al += xp.re * xp.re + xp.im * xp.im;
          be += xq.re * xq.re + xq.im * xq.im;
          gr += xp.re * xq.re + xp.im * xq.im;  // conj(xp) * xq
          gi += xp.re * xq.im - xp.im * xq.re;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        gr = warp_sum(gr);
        gi = warp_sum(gi);
        const double g2 = gr * gr + gi * gi;
        // decoupled to working precision relative to the pair and to the face
        if (!(g2 > 1e-30 * al * be) || !(g2 > 1e-34 * fnorm2 * fnorm2) || !(g2 > 1e-300)) continue;
        const double rg = (g2 > 1e-36 && g2 < 1e36) ? fast_rsqrt(g2) : 1.0 / sqrt(g2);
        const double g = g2 * rg;
        double c, s;
        jacobi_cs_fast(al, be, g, c, s);  // tau = (beta - alpha) / (2 |gamma|), fp32 tangent
        const cplx ph = {gr * rg, gi * rg};  // e^{i phi}
        // [xp, xq] <- [xp, xq] [[c, s e^{i phi}], [-s e^{-i phi}, c]]
        const cplx spn = {s * ph.re, s * ph.im};   // s e^{i phi}
        const cplx smn = {s * ph.re, -s * ph.im};  // s e^{-i phi}
        for (int i = lane; i < r0; i += 32) {
          const cplx xp = X[i + r0 * p], xq = X[i + r0 * q];
          const cplx a = cmul(smn, xq), b2 = cmul(spn, xp);
          X[i + r0 * p] = {c * xp.re - a.re, c * xp.im - a.im};
          X[i + r0 * q] = {b2.re + c * xq.re, b2.im + c * xq.im};
        }
        for (int i = lane; i < r1; i += 32) {
          const cplx vp = V[i + r1 * p], vq = V[i + r1 * q];
          const cplx a = cmul(smn, vq), b2 = cmul(spn, vp);
          V[i + r1 * p] = {c * vp.re - a.re, c * vp.im - a.im};
          V[i + r1 * q] = {b2.re + c * vq.re, b2.im + c * vq.im};
        }
        if (lane == 0) rot_any = 1;
      }
      __syncthreads();
    }
    if (!rot_any) break;
    __syncthreads();
  }
  // sigma_j = ||x_j||; weight prox(sigma)/sigma
  for (int j = warp; j < r1; j += nw) {
    double s2 = 0.0;
    for (int i = lane; i < r0; i += 32) s2 += X[i + r0 * j].re * X[i + r0 * j].re +
                                              X[i + r0 * j].im * X[i + r0 * j].im;
    s2 = warp_sum(s2);
    if (lane == 0) {
      const double sg = sqrt(s2);
      wsc[j] = sg > 0.0 ? prox(pen, tau, sg) / sg : 0.0;
    }
  }
  __syncthreads();
  // out = X diag(w) V^H
  for (int e = threadIdx.x; e < r0 * r1; e += blockDim.x) {
    const int i = e % r0, k = e / r0;
    double ar = 0.0, ai = 0.0;
    for (int j = 0; j < r1; ++j) {
      const double w = wsc[j];
      if (w == 0.0) continue;
      const cplx x = X[i + r0 * j];
      const cplx v = V[k + r1 * j];  // conj(v) used
      ar += w * (x.re * v.re + x.im * v.im);
      ai += w * (x.im * v.re - x.re * v.im);
    }
    src[e] = {ar, ai};
  }
}

// out[lo + st*(k + n*hi)] = sum_j M(k, j) in[lo + st*(j + n*hi)] with
// M = U (inverse = 0) or U^H / alpha (inverse = 1).  `in_real` reads a real
// input; `out_real` writes the real part only.  Four lanes per output split
// the j sum (j = sub, sub + 4, ...) and combine it with two xor shuffles in a
// fixed order: 4x the parallelism and a 4x shorter dependent chain for the
// small core transforms (n = transform length, total = core size).
// skip_tr.nt > 0 (last forward FFT product): outputs of faces that the mirror
// step overwrites afterwards are not formed (face = t / face_len).
__global__ void k_mode_product(const void* __restrict__ in_, int in_real, void* __restrict__ out_,
                               int out_real, int64_t st, int n, int64_t hi_count,
                               const cplx* __restrict__ U, int inverse, double alpha,
                               int64_t face_len, Trailing skip_tr) {
  const int64_t tq = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int sub = (int)(tq & 3);
  const int64_t t = tq >> 2;
  const int64_t total = st * n * hi_count;
  const bool live = t < total && !(skip_tr.nt > 0 && mirror_face(t / face_len, skip_tr) < t / face_len);
  const int64_t tt = live ? t : 0;
  const int64_t lo = tt % st;
  const int k = (int)((tt / st) % n);
  const int64_t hi = tt / (st * n);
  double ar = 0.0, ai = 0.0;
  if (live) {
    for (int j = sub; j < n; j += 4) {
      cplx u = inverse ? cconj(U[j * n + k]) : U[k * n + j];
      const int64_t src = lo + st * (j + (int64_t)n * hi);
      cplx x;
      if (in_real) x = {((const double*)in_)[src], 0.0};
      else x = ((const cplx*)in_)[src];
      ar += u.re * x.re - u.im * x.im;
      ai += u.re * x.im + u.im * x.re;
    }
  }
  ar += __shfl_xor_sync(0xffffffffu, ar, 1);
  ai += __shfl_xor_sync(0xffffffffu, ai, 1);
  ar += __shfl_xor_sync(0xffffffffu, ar, 2);
  ai += __shfl_xor_sync(0xffffffffu, ai, 2);
  if (!live || sub != 0) return;
  if (inverse) {
    ar /= alpha;
    ai /= alpha;
  }
  if (out_real) ((double*)out_)[t] = ar;
  else ((cplx*)out_)[t] = {ar, ai};
}

// skip (FFT transforms, mirror_tr.nt > 0): faces whose mirror is an earlier
// face are overwritten by k_mirror_fix, so their CTAs exit at once and leave
// the SMs to the other mode streams.
__device__ __forceinline__ bool face_is_mirror_copy(int64_t f, const Trailing& mirror_tr) {
  return mirror_tr.nt > 0 && mirror_face(f, mirror_tr) < f;
}

__global__ void __launch_bounds__(1024) k_face_svt(cplx* __restrict__ faces, int r0, int r1,
                                                    Penalty pen, double tau, Trailing mirror_tr) {
  if (face_is_mirror_copy(blockIdx.x, mirror_tr)) return;
  extern __shared__ double svt_smem[];
  cplx* X = reinterpret_cast<cplx*>(svt_smem);  // r0 x r1, ld = r0
  cplx* V = X + r0 * r1;                        // r1 x r1, ld = r1
  __shared__ double wsc[64];
  face_svt_body(X, V, wsc, faces + (int64_t)blockIdx.x * r0 * r1, r0, r1, pen, tau);
}

// faces larger than 64: X / V in global scratch (xw: faces-sized, vw: r1^2 per face)
__global__ void __launch_bounds__(1024) k_face_svt_g(cplx* __restrict__ faces, cplx* __restrict__ xw,
                                                      cplx* __restrict__ vw, int r0, int r1,
                                                      Penalty pen, double tau, Trailing mirror_tr) {
  if (face_is_mirror_copy(blockIdx.x, mirror_tr)) return;
  extern __shared__ double wsc_g[];  // r1 weights
  const int64_t f = blockIdx.x;
  face_svt_body(xw + f * r0 * r1, vw + f * (int64_t)r1 * r1, wsc_g, faces + f * r0 * r1, r0, r1,
                pen, tau);
}

__global__ void k_mirror_fix(cplx* __restrict__ faces, int64_t face_len, int64_t nf, Trailing tr) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= face_len * nf) return;
  const int64_t f = t / face_len, e = t % face_len;
  const int64_t mf = mirror_face(f, tr);
  if (mf < f) faces[t] = cconj(faces[mf * face_len + e]);
}

}  // namespace tr
