// Batched FFTs along one axis of a column-major tensor, and the FFT-diagonal
// solve of tenrec/gradient.py:90-106:
//     (I + sum_{k in Gamma} D_k^T D_k) L = rhs,   D_k = forward circular difference
// which is diagonal under the full d-dimensional DFT with eigenvalues
// 1 + sum_k 4 sin^2(pi j_k / n_k) (gradient.py:63-80).
//
// Layout: element (lo, k, hi) of an axis of length n with lo-stride st lives at
// lo + st * (k + n * hi).  One CTA loads a tile of `L` lines (consecutive lo
// when st > 1 for coalescing, consecutive hi when the axis is contiguous) into
// shared memory, transforms every line there (radix-2 DIT for powers of two,
// direct DFT otherwise), and writes it back.  The last-axis pass of the solve
// does forward FFT -> divide -> inverse FFT without leaving shared memory.
#pragma once

#include "common.cuh"

namespace tr {

template <typename T>
struct cpx {
  T re, im;
};

template <typename T>
__device__ __forceinline__ cpx<T> cadd(cpx<T> a, cpx<T> b) { return {a.re + b.re, a.im + b.im}; }
template <typename T>
__device__ __forceinline__ cpx<T> csub(cpx<T> a, cpx<T> b) { return {a.re - b.re, a.im - b.im}; }
template <typename T>
__device__ __forceinline__ cpx<T> cmulc(cpx<T> a, cpx<T> b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}

// tw[k] = exp(-2 pi i k / n), k < n, computed in fp64 with exact argument reduction
template <typename T>
__global__ void k_twiddles(int n, cpx<T>* __restrict__ tw) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double s, c;
  sincospi(-2.0 * (double)k / (double)n, &s, &c);
  tw[k] = {(T)c, (T)s};
}

struct SolveSpec {
  int active;          // last-axis pass of the diagonal solve
  int d;               // tensor order
  int64_t dims[10];
  int64_t lam_off[10];  // offset of axis k's 4 sin^2(pi j / n_k) table in lam, -1 if k not in Gamma
};

__device__ __forceinline__ int brev(int x, int bits) { return (int)(__brev((unsigned)x) >> (32 - bits)); }

// in-place transform of the L lines held in shared memory; element (l, k) at l*ls + k*ks
template <typename T>
__device__ void smem_lines_fft(cpx<T>* buf, cpx<T>* tmp, int L, int n, int64_t ls, int64_t ks,
                               const cpx<T>* __restrict__ tw, bool inverse, bool pow2, int bits) {
  const int nt = blockDim.x;
  if (n == 1) return;
  if (pow2) {
    // bit-reversal permutation (swap pairs once)
    for (int e = threadIdx.x; e < L * n; e += nt) {
      const int l = e / n, k = e % n;
      const int r = brev(k, bits);
      if (r > k) {
        const cpx<T> a = buf[l * ls + k * ks];
        buf[l * ls + k * ks] = buf[l * ls + r * ks];
        buf[l * ls + r * ks] = a;
      }
    }
    __syncthreads();
    for (int len = 2; len <= n; len <<= 1) {
      const int half = len >> 1, step = n / len;
      for (int e = threadIdx.x; e < L * (n >> 1); e += nt) {
        const int l = e / (n >> 1), b = e % (n >> 1);
        const int i = (b / half) * len + (b % half), j = i + half;
        cpx<T> w = tw[(b % half) * step];
        if (inverse) w.im = -w.im;
        const cpx<T> t = cmulc(w, buf[l * ls + j * ks]);
        const cpx<T> u = buf[l * ls + i * ks];
        buf[l * ls + i * ks] = cadd(u, t);
        buf[l * ls + j * ks] = csub(u, t);
      }
      __syncthreads();
    }
  } else {
    // direct DFT through tmp (same shape as buf)
    for (int e = threadIdx.x; e < L * n; e += nt) {
      const int l = e / n, k = e % n;
      cpx<T> acc = {T(0), T(0)};
      int idx = 0;
      for (int j = 0; j < n; ++j) {
        cpx<T> w = tw[idx];
        if (inverse) w.im = -w.im;
        acc = cadd(acc, cmulc(w, buf[l * ls + j * ks]));
        idx += k;
        if (idx >= n) idx -= n;
      }
      tmp[l * ls + k * ks] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < L * n; e += nt) {
      const int l = e / n, k = e % n;
      buf[l * ls + k * ks] = tmp[l * ls + k * ks];
    }
    __syncthreads();
  }
}

// One pass along an axis.  in_real: input is real T; out_real: write Re * out_scale.
template <typename T>
__global__ void __launch_bounds__(256) k_fft_axis(const void* __restrict__ in, int in_real,
                                                  void* __restrict__ out, int out_real,
                                                  double out_scale, int64_t st, int n, int64_t hi,
                                                  int L, const cpx<T>* __restrict__ tw, int inverse,
                                                  SolveSpec ss, const double* __restrict__ lam) {
  extern __shared__ __align__(16) unsigned char fft_smem[];
  cpx<T>* buf = reinterpret_cast<cpx<T>*>(fft_smem);
  const bool pow2 = (n & (n - 1)) == 0;
  cpx<T>* tmp = buf + (size_t)L * n;
  int bits = 0;
  while ((1 << bits) < n) ++bits;
  // line l of this CTA -> (lo, hi)
  int64_t lo0, hi0;
  bool lo_lines;
  if (st == 1) {
    lo_lines = false;
    lo0 = 0;
    hi0 = (int64_t)blockIdx.x * L;
  } else {
    lo_lines = true;
    const int64_t nlob = (st + L - 1) / L;
    lo0 = (int64_t)(blockIdx.x % nlob) * L;
    hi0 = blockIdx.x / nlob;
  }
  // smem layout: lo-lines -> [k][l] (coalesced along lo), hi-lines -> [l][k]
  const int64_t ls = lo_lines ? 1 : n, ks = lo_lines ? L : 1;
  for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
    int l, k;
    if (lo_lines) { l = e % L; k = e / L; } else { l = e / n; k = e % n; }
    const int64_t lo = lo_lines ? lo0 + l : 0;
    const int64_t hh = lo_lines ? hi0 : hi0 + l;
    cpx<T> v = {T(0), T(0)};
    if (lo < st && hh < hi) {
      const int64_t g = lo + st * (k + (int64_t)n * hh);
      if (in_real) v.re = reinterpret_cast<const T*>(in)[g];
      else v = reinterpret_cast<const cpx<T>*>(in)[g];
    }
    buf[l * ls + k * ks] = v;
  }
  __syncthreads();
  smem_lines_fft<T>(buf, tmp, L, n, ls, ks, tw, inverse != 0, pow2, bits);
  if (ss.active) {
    // divide by 1 + sum_k lam_k(j_k); the transformed axis is the last one
    for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
      int l, k;
      if (lo_lines) { l = e % L; k = e / L; } else { l = e / n; k = e % n; }
      const int64_t lo = lo_lines ? lo0 + l : 0;
      double den = 1.0;
      int64_t rem = lo;
      for (int a = 0; a < ss.d - 1; ++a) {
        const int64_t j = rem % ss.dims[a];
        rem /= ss.dims[a];
        if (ss.lam_off[a] >= 0) den += lam[ss.lam_off[a] + j];
      }
      if (ss.lam_off[ss.d - 1] >= 0) den += lam[ss.lam_off[ss.d - 1] + k];
      const T inv = (T)(1.0 / den);
      cpx<T> v = buf[l * ls + k * ks];
      buf[l * ls + k * ks] = {v.re * inv, v.im * inv};
    }
    __syncthreads();
    smem_lines_fft<T>(buf, tmp, L, n, ls, ks, tw, true, pow2, bits);
  }
  for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
    int l, k;
    if (lo_lines) { l = e % L; k = e / L; } else { l = e / n; k = e % n; }
    const int64_t lo = lo_lines ? lo0 + l : 0;
    const int64_t hh = lo_lines ? hi0 : hi0 + l;
    if (lo < st && hh < hi) {
      const int64_t g = lo + st * (k + (int64_t)n * hh);
      const cpx<T> v = buf[l * ls + k * ks];
      if (out_real) reinterpret_cast<T*>(out)[g] = (T)(v.re * out_scale);
      else reinterpret_cast<cpx<T>*>(out)[g] = v;
    }
  }
}

// 4 sin^2(pi j / n) for j < n
__global__ void k_lap_eig(int n, double* __restrict__ lam) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double s = sinpi((double)j / (double)n);
  lam[j] = 4.0 * s * s;
}

}  // namespace tr
