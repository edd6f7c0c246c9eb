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

// The same product with both operands staged in shared memory: a TL x n tile of
// `in` (TL consecutive lo, all j, one hi) and the KB rows of M the CTA's outputs
// need (conjugated for the inverse), so `in` is read from L2 n / KB times instead
// of n times and the inner loop is two LDS.128 per complex FMA (k_mode_product
// re-reads `in` for every output: 164 MB of L2 traffic for the 25 x 25 x 128
// bench core, and slower still next to the streaming passes of the other mode
// streams).  blockIdx = (lo tile, hi, k block); thread = (lo, k): one output.
constexpr int kMpTL = 8, kMpKB = 32;
inline size_t mode_product_smem(int n) {
  return ((size_t)n * kMpTL + (size_t)kMpKB * (n + 1)) * sizeof(cplx);
}
__global__ void __launch_bounds__(kMpTL* kMpKB) k_mode_product_t(
    const void* __restrict__ in_, int in_real, void* __restrict__ out_, int out_real, int64_t st,
    int n, int64_t hi_count, const cplx* __restrict__ U, int inverse, double alpha,
    int64_t face_len, Trailing skip_tr) {
  constexpr int TL = kMpTL, KB = kMpKB, NT = TL * KB;
  extern __shared__ double mpt_smem[];
  cplx* tile = reinterpret_cast<cplx*>(mpt_smem);  // [j][TL]
  cplx* Us = tile + (size_t)n * TL;                // [KB][n + 1]: M(k0 + kk, j)
  const int tid = threadIdx.x;
  const int64_t lo0 = (int64_t)blockIdx.x * TL, hi = blockIdx.y;
  const int k0 = (int)blockIdx.z * KB;
  for (int e = tid; e < n * TL; e += NT) {
    const int j = e / TL, ll = e % TL;
    const int64_t lo = lo0 + ll;
    cplx v = {0.0, 0.0};
    if (lo < st) {
      const int64_t src = lo + st * (j + (int64_t)n * hi);
      if (in_real) v.re = ((const double*)in_)[src];
      else v = ((const cplx*)in_)[src];
    }
    tile[e] = v;
  }
  if (inverse) {  // M(k, j) = conj(U[j, k]): KB consecutive k are contiguous in U
    for (int e = tid; e < n * KB; e += NT) {
      const int j = e / KB, kk = e % KB;
      cplx u = {0.0, 0.0};
      if (k0 + kk < n) u = cconj(U[(int64_t)j * n + k0 + kk]);
      Us[kk * (n + 1) + j] = u;
    }
  } else {
    for (int e = tid; e < n * KB; e += NT) {
      const int kk = e / n, j = e % n;
      cplx u = {0.0, 0.0};
      if (k0 + kk < n) u = U[(int64_t)(k0 + kk) * n + j];
      Us[kk * (n + 1) + j] = u;
    }
  }
  __syncthreads();
  const int ll = tid % TL, kq = tid / TL;
  const int64_t lo = lo0 + ll;
  const int k = k0 + kq;
  if (lo >= st || k >= n) return;
  const int64_t t = lo + st * (k + (int64_t)n * hi);
  if (skip_tr.nt > 0 && mirror_face(t / face_len, skip_tr) < t / face_len) return;
  // two independent accumulator sets (even / odd j) halve the dependent chain
  double ar0 = 0.0, ai0 = 0.0, ar1 = 0.0, ai1 = 0.0;
  const cplx* urow = Us + kq * (n + 1);
  int j = 0;
#pragma unroll 4
  for (; j + 1 < n; j += 2) {
    const cplx u0 = urow[j], u1 = urow[j + 1];
    const cplx x0 = tile[j * TL + ll], x1 = tile[(j + 1) * TL + ll];
    ar0 = fma(u0.re, x0.re, fma(-u0.im, x0.im, ar0));
    ai0 = fma(u0.re, x0.im, fma(u0.im, x0.re, ai0));
    ar1 = fma(u1.re, x1.re, fma(-u1.im, x1.im, ar1));
    ai1 = fma(u1.re, x1.im, fma(u1.im, x1.re, ai1));
  }
  if (j < n) {
    const cplx u0 = urow[j];
    const cplx x0 = tile[j * TL + ll];
    ar0 = fma(u0.re, x0.re, fma(-u0.im, x0.im, ar0));
    ai0 = fma(u0.re, x0.im, fma(u0.im, x0.re, ai0));
  }
  double ar = ar0 + ar1, ai = ai0 + ai1;
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

#ifdef TR_FACE_PROBE
__device__ long long g_face_probe[4];
#endif

// Faces up to 32 x 32 (the Tucker cores of the randomized t-SVT): one CTA of
// 16 * LPP threads per face, LPP (8 or 16) lanes per Jacobi pair (lane l owns
// rows l, l + LPP, ... of both columns), so the 16 pair slots of a round fill
// 4 or 8 warps and the serial chain of a round is log2(LPP) shuffle steps, one
// short rotation and one barrier.  A single warp issues an fp64 instruction
// every ~4.5 cycles (measured), so LPP = 16 -- two warps per SM sub-partition,
// two rows per lane -- halves the per-warp instruction stream of LPP = 8.
//   * the face is scaled by a power of two to ||X||_F in [0.5, 1), so the
//     rotation's tangent can be formed in fp32 from MUFU rsqrt / rcp without
//     range guards: w = t e^{i phi} = sign(z) gamma / (|z| + sqrt(z^2 + |gamma|^2)),
//     z = (beta - alpha) / 2;  c = (1 + |w|^2)^{-1/2} is completed in fp64 from
//     the w actually used, so every rotation is unitary to fp64 rounding and only
//     the annihilation of gamma is fp32-accurate (the next sweep absorbs it);
//   * no V accumulation: with Xf = X V (orthogonal columns, norms sigma_j),
//     U prox(S) V^H = Xf diag(prox(sigma_j) / sigma_j^3) Xf^H X, two small
//     products at the end.  The error of a direction with a small sigma_j is
//     eps * sigma_max / sigma_j relative, weighted by prox(sigma_j) <= sigma_j:
//     eps * sigma_max absolute, the same as the explicit-V form;
//   * Jacobi converges quadratically: once every pair of a sweep met
//     |cos| <= 1e-8 the rotated pairs are left at <= 1e-15 and the others moved
//     by second-order terms only, so no verification sweep is run.
template <int LPP>
__global__ void __launch_bounds__(16 * LPP) k_face_svt8(cplx* __restrict__ faces, int r0, int r1,
                                                        Penalty pen, double tau,
                                                        Trailing mirror_tr) {
  constexpr int NT = 16 * LPP, RPL = 32 / LPP;
  if (face_is_mirror_copy(blockIdx.x, mirror_tr)) return;
  extern __shared__ double svt8_smem[];
  cplx* X = reinterpret_cast<cplx*>(svt8_smem);  // r0 x r1 working copy (scaled), ld = r0
  cplx* X0 = X + r0 * r1;                        // r0 x r1 scaled input
  cplx* Tm = X0 + r0 * r1;                       // r1 x r1: diag(w) Xf^H X0
  __shared__ unsigned char sched[31][16][2];
  __shared__ double wsc[32];
  __shared__ double fred[32];
  cplx* src = faces + (int64_t)blockIdx.x * r0 * r1;
  // the conjugate-mirror partner of this canonical face (k_mirror_fix fused here)
  cplx* mir = nullptr;
  if (mirror_tr.nt > 0) {
    const int64_t mf = mirror_face(blockIdx.x, mirror_tr);
    if (mf != (int64_t)blockIdx.x) mir = faces + mf * r0 * r1;
  }
  const int tid = threadIdx.x;
  const int ne = r1 + (r1 & 1), npairs = ne / 2;
  for (int e = tid; e < (ne - 1) * npairs; e += NT) {
    const int rnd = e / npairs, kk = e - rnd * npairs;
    int p = rr_player(kk, rnd, ne), q = rr_player(ne - 1 - kk, rnd, ne);
    if (p > q) { const int t = p; p = q; q = t; }
    sched[rnd][kk][0] = (unsigned char)p;
    sched[rnd][kk][1] = (unsigned char)q;
  }
  double f2 = 0.0;
  for (int e = tid; e < r0 * r1; e += NT) {
    const cplx v = src[e];
    X[e] = v;
    f2 += v.re * v.re + v.im * v.im;
  }
  const double fn2 = block_sum(f2, fred);
  // zero face: prox(0) = 0, the face stays zero (non-finite input is left as is)
  if (!(fn2 > 0.0) || !(fn2 < 1e300)) {
    if (mir)
      for (int e = tid; e < r0 * r1; e += NT) mir[e] = cconj(X[e]);
    return;
  }
  int ex;
  frexp(sqrt(fn2), &ex);
  const double scale = ldexp(1.0, -ex), unscale = ldexp(1.0, ex);
  for (int e = tid; e < r0 * r1; e += NT) {
    cplx v = X[e];
    v.re *= scale;
    v.im *= scale;
    X[e] = v;
    X0[e] = v;
  }
  const double thr_abs = 1e-34 * (fn2 * scale * scale) * (fn2 * scale * scale);
  __syncthreads();
  const int kp = tid / LPP, l = tid % LPP;
#ifdef TR_FACE_PROBE
  const long long t_j0 = clock64();
  int nsweeps = 0;
#endif
  // next round's pair is fetched before the barrier (off the round's serial chain)
  int pn = 0, qn = r1;
  if (kp < npairs && ne >= 2) {
    pn = sched[0][kp][0];
    qn = sched[0][kp][1];
  }
  for (int sweep = 0; sweep < 60 && ne >= 2; ++sweep) {
    int big = 0;  // a pair of this sweep met |cos| > 1e-8
    for (int rnd = 0; rnd < ne - 1; ++rnd) {
      const int p = pn, q = qn;
      const bool live = q < r1;  // uniform over the pair's lanes; idle slots carry zeros
      if (kp < npairs) {
        const int nr = rnd + 1 < ne - 1 ? rnd + 1 : 0;
        pn = sched[nr][kp][0];
        qn = sched[nr][kp][1];
      }
      cplx xp[RPL], xq[RPL];
      double pa[RPL], pb[RPL], pr[RPL], pi[RPL];
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int i = l + LPP * u;
        const bool in = live && i < r0;
        xp[u] = in ? X[i + r0 * p] : cplx{0.0, 0.0};
        xq[u] = in ? X[i + r0 * q] : cplx{0.0, 0.0};
        pa[u] = fma(xp[u].re, xp[u].re, xp[u].im * xp[u].im);
        pb[u] = fma(xq[u].re, xq[u].re, xq[u].im * xq[u].im);
        pr[u] = fma(xp[u].re, xq[u].re, xp[u].im * xq[u].im);  // conj(xp) * xq
        pi[u] = fma(xp[u].re, xq[u].im, -(xp[u].im * xq[u].re));
      }
      double al, be, gr, gi;
      if constexpr (RPL == 4) {
        al = (pa[0] + pa[1]) + (pa[2] + pa[3]);
        be = (pb[0] + pb[1]) + (pb[2] + pb[3]);
        gr = (pr[0] + pr[1]) + (pr[2] + pr[3]);
        gi = (pi[0] + pi[1]) + (pi[2] + pi[3]);
      } else {
        al = pa[0] + pa[1];
        be = pb[0] + pb[1];
        gr = pr[0] + pr[1];
        gi = pi[0] + pi[1];
      }
#pragma unroll
      for (int o = LPP / 2; o > 0; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        gr += __shfl_xor_sync(0xffffffffu, gr, o);
        gi += __shfl_xor_sync(0xffffffffu, gi, o);
      }
      const double g2 = fma(gr, gr, gi * gi);
      const double ab = al * be;
      // decoupled to working precision relative to the pair and to the face
      if (g2 > 1e-30 * ab && g2 > thr_abs) {
        big |= g2 > 1e-16 * ab;
        const float zf = (float)(0.5 * (be - al));
        const float grf = (float)gr, gif = (float)gi;
        const float hf = fmaf(zf, zf, fmaf(grf, grf, gif * gif));
        float rs, invd, cs;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(hf));
        const float df = fabsf(zf) + hf * rs;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(invd) : "f"(df));
        const float sg = copysignf(invd, zf);
        const float wrf = grf * sg, wif = gif * sg;
        // fp32 seed of c beside the fp64 conversion of w; one cubic step
        // (seed error e ~ 2^-21, remaining error ~ e^3)
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(cs) : "f"(fmaf(wrf, wrf, fmaf(wif, wif, 1.0f))));
        const double wr = (double)wrf, wi = (double)wif;
        const double x1 = 1.0 + fma(wr, wr, wi * wi);  // in [1, 2]
        const double c0 = (double)cs;
        const double er = fma(-x1, c0 * c0, 1.0);
        const double c = fma(c0 * er, fma(0.375, er, 0.5), c0);
        const double sr = c * wr, si = c * wi;  // S = s e^{i phi}
        // xp' = c xp - conj(S) xq,  xq' = S xp + c xq
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int i = l + LPP * u;
          cplx a, b;
          a.re = fma(c, xp[u].re, -fma(sr, xq[u].re, si * xq[u].im));
          a.im = fma(c, xp[u].im, -fma(sr, xq[u].im, -(si * xq[u].re)));
          b.re = fma(c, xq[u].re, fma(sr, xp[u].re, -(si * xp[u].im)));
          b.im = fma(c, xq[u].im, fma(sr, xp[u].im, si * xp[u].re));
          if (i < r0) {  // live: g2 > 0
            X[i + r0 * p] = a;
            X[i + r0 * q] = b;
          }
        }
      }
      if (rnd < ne - 2) __syncthreads();
    }
    const int any = __syncthreads_or(big);
#ifdef TR_FACE_PROBE
    ++nsweeps;
#endif
    if (!any) break;
  }
#ifdef TR_FACE_PROBE
  if (tid == 0 && blockIdx.x == 0) {
    g_face_probe[0] = clock64() - t_j0;
    g_face_probe[1] = nsweeps;
  }
#endif
  // sigma_j = ||xf_j|| / scale; wsc[j] = prox(sigma_j) / (sigma_j * ||xf_j||^2)
  for (int j0 = 0; j0 < r1; j0 += 16) {
    const int j = j0 + kp;
    double s2 = 0.0;
    if (j < r1)
      for (int i = l; i < r0; i += LPP) {
        const cplx v = X[i + r0 * j];
        s2 += v.re * v.re + v.im * v.im;
      }
#pragma unroll
    for (int o = LPP / 2; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (l == 0 && j < r1) {
      const double sg = sqrt(s2) * unscale;
      wsc[j] = (s2 > 1e-280 && sg > 0.0) ? prox(pen, tau, sg) / (sg * s2) : 0.0;
    }
  }
  __syncthreads();
  // Tm = diag(wsc) Xf^H X0
  for (int e = tid; e < r1 * r1; e += NT) {
    const int j = e % r1, k = e / r1;
    const double w = wsc[j];
    double ar = 0.0, ai = 0.0;
    if (w != 0.0)
      for (int i = 0; i < r0; ++i) {
        const cplx a = X[i + r0 * j], b = X0[i + r0 * k];
        ar += a.re * b.re + a.im * b.im;  // conj(a) * b
        ai += a.re * b.im - a.im * b.re;
      }
    Tm[e] = {w * ar, w * ai};
  }
  __syncthreads();
  // out = Xf Tm (the power-of-two scale cancels: Xf and X0 carry it, wsc has 1 / ||xf||^2)
  for (int e = tid; e < r0 * r1; e += NT) {
    const int i = e % r0, k = e / r0;
    double ar = 0.0, ai = 0.0;
    for (int j = 0; j < r1; ++j) {
      const cplx a = X[i + r0 * j], b = Tm[j + r1 * k];
      ar += a.re * b.re - a.im * b.im;
      ai += a.re * b.im + a.im * b.re;
    }
    const cplx o = {ar * unscale, ai * unscale};
    src[e] = o;
    if (mir) mir[e] = cconj(o);
  }
}

__global__ void k_mirror_fix(cplx* __restrict__ faces, int64_t face_len, int64_t nf, Trailing tr) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= face_len * nf) return;
  const int64_t f = t / face_len, e = t % face_len;
  const int64_t mf = mirror_face(f, tr);
  if (mf < f) faces[t] = cconj(faces[mf * face_len + e]);
}

}  // namespace tr
