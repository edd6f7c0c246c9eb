// Elementwise / stencil kernels of the ADMM solvers (tenrec/solvers.py:204-284,
// tenrec/onebit.py:141-220), each fused with the Eq. (24) residual reductions
// it can produce from the values it already has in registers.
#pragma once

#include "common.cuh"
#include "prox.cuh"

namespace tr {

constexpr int kMaxOrder = 10;
constexpr int kRedThreads = 256;

struct Geom {
  int d;
  int64_t dims[kMaxOrder];
  int64_t st[kMaxOrder];
  int64_t N;
};

// index of the circular neighbour of i along axis a (dir = +1 next, -1 previous)
__device__ __forceinline__ int64_t nbr(int64_t i, const Geom& g, int a, int dir) {
  const int64_t n = g.dims[a], s = g.st[a];
  const int64_t j = (i / s) % n;
  if (dir > 0) return j + 1 < n ? i + s : i - s * (n - 1);
  return j > 0 ? i - s : i + s * (n - 1);
}

template <typename T>
struct ModePtrs {
  int count;
  int axis[kMaxOrder];  // -1 = identity chain (pure low-rank ablation)
  T* p[kMaxOrder];
};

// per-block partial reductions: NQ values, `is_max` bitmask selects max vs sum
template <int NQ>
__device__ __forceinline__ void block_partials(double (&v)[NQ], unsigned is_max, double* red,
                                               double* __restrict__ part) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double r = (is_max >> q) & 1 ? block_max(v[q], red) : block_sum(v[q], red);
    if (threadIdx.x == 0) part[(int64_t)blockIdx.x * NQ + q] = r;
  }
}

__global__ void k_final_reduce(const double* __restrict__ part, int nblocks, int nq,
                               unsigned is_max, double* __restrict__ out) {
  __shared__ double red[32];
  for (int q = 0; q < nq; ++q) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
      const double x = part[(int64_t)b * nq + q];
      v = (is_max >> q) & 1 ? fmax(v, x) : v + x;
    }
    v = (is_max >> q) & 1 ? block_max(v, red) : block_sum(v, red);
    if (threadIdx.x == 0) out[q] = v;
  }
}

// rhs of the L- (or Z-) subproblem (solvers.py:231-233, onebit.py:182-184):
//   b = A - B + y / mu ;  rhs = b + sum_k D_k^T (g_k - lag_k / mu)
// pure low-rank chain: out = 0.5 * (b + g - lag / mu)  (solvers.py:194-195), the final L.
template <typename T>
__global__ void k_admm_rhs(Geom g, const T* __restrict__ A, const T* __restrict__ B,
                           const T* __restrict__ y, double mu, ModePtrs<T> gm, ModePtrs<T> lag,
                           T* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.N; i += stride) {
    const T bv = (B ? (A[i] - B[i]) : A[i]) + y[i] / (T)mu;
    if (gm.count == 1 && gm.axis[0] < 0) {
      out[i] = (T)0.5 * (bv + (gm.p[0][i] - lag.p[0][i] / (T)mu));
      continue;
    }
    T acc = bv;
    for (int k = 0; k < gm.count; ++k) {
      const int a = gm.axis[k];
      const int64_t ip = nbr(i, g, a, -1);
      const T gi = gm.p[k][i] - lag.p[k][i] / (T)mu;
      const T gp = gm.p[k][ip] - lag.p[k][ip] / (T)mu;
      acc += gp - gi;
    }
    out[i] = acc;
  }
}

// LRTA input of mode k: X = D_k L + lag_k / mu (identity chain: L + lag / mu)
template <typename T>
__global__ void k_lrta_input(Geom g, const T* __restrict__ l, int axis, const T* __restrict__ lag,
                             double mu, T* __restrict__ X) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.N; i += stride) {
    const T gl = axis < 0 ? l[i] : l[nbr(i, g, axis, +1)] - l[i];
    X[i] = gl + lag[i] / (T)mu;
  }
}

// multiplier update of mode k (solvers.py:247-248) with its residuals:
//   lag += mu (D_k L - G_new);  partial q: 0 max|DL-G|, 1 sum (DL-G)^2,
//   2 max|G_new-G_old|, 3 sum (G_new-G_old)^2, 4 sum lag_new^2
template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_lag_update(Geom g, const T* __restrict__ l, int axis,
                                                            const T* __restrict__ gnew,
                                                            const T* __restrict__ gold,
                                                            T* __restrict__ lag, double mu,
                                                            double* __restrict__ part) {
  __shared__ double red[32];
  double v[5] = {0, 0, 0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.N; i += stride) {
    const T gl = axis < 0 ? l[i] : l[nbr(i, g, axis, +1)] - l[i];
    const T gn = gnew[i];
    const T gap = gl - gn;
    const T ln = lag[i] + (T)mu * gap;
    lag[i] = ln;
    const double dg = (double)gn - (double)gold[i];
    v[0] = fmax(v[0], fabs((double)gap));
    v[1] += (double)gap * (double)gap;
    v[2] = fmax(v[2], fabs(dg));
    v[3] += dg * dg;
    v[4] += (double)ln * (double)ln;
  }
  block_partials<5>(v, 0b00101u, red, part);
}

// group scales of the structured noise shrinkage (shrink.py:49-54) of
// mask * h, h = mobs - l + y / mu:  scale = prox(level, ||group||) / ||group||.
// structure 1 = tube (i0, i1) over trailing modes, 2 = slice (face) over (i0, i1).
template <typename T>
__global__ void k_group_scale(Geom g, int structure, const T* __restrict__ mobs,
                              const uint8_t* __restrict__ mask, const T* __restrict__ l,
                              const T* __restrict__ y, double mu, Penalty pen, double level,
                              double* __restrict__ scale) {
  const int64_t face = g.dims[0] * g.dims[1];
  const int64_t nf = g.N / face;
  if (structure == 1) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= face) return;
    double s2 = 0.0;
    for (int64_t f = 0; f < nf; ++f) {
      const int64_t i = t + face * f;
      const double h = mask[i] ? (double)(mobs[i] - l[i] + y[i] / (T)mu) : 0.0;
      s2 += h * h;
    }
    const double gn = sqrt(s2);
    scale[t] = gn > 0 ? prox(pen, level, gn) / gn : 0.0;
  } else {
    __shared__ double red[32];
    const int64_t f = blockIdx.x;
    double s2 = 0.0;
    for (int64_t e = threadIdx.x; e < face; e += blockDim.x) {
      const int64_t i = e + face * f;
      const double h = mask[i] ? (double)(mobs[i] - l[i] + y[i] / (T)mu) : 0.0;
      s2 += h * h;
    }
    const double gn = sqrt(block_sum(s2, red));
    if (threadIdx.x == 0) scale[f] = gn > 0 ? prox(pen, level, gn) / gn : 0.0;
  }
}

// noise and dual updates (solvers.py:239-246) with residuals:
//   h = mobs - l + y/mu ; E = mask*shrink(mask*h) + (1-mask)*h ; y += mu (mobs - l - E)
//   structure 0 entry / 1 tube / 2 slice / 3 noise-free (E = 0 on the mask)
//   partial q: 0 max|l-lold| 1 sum 2 max|E-Eold| 3 sum 4 max|fit| 5 sum 6 sum y^2
template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_noise_dual(Geom g, int structure,
                                                            const T* __restrict__ mobs,
                                                            const uint8_t* __restrict__ mask,
                                                            const T* __restrict__ l,
                                                            const T* __restrict__ lold,
                                                            T* __restrict__ e, T* __restrict__ y,
                                                            double mu, Penalty pen, double level,
                                                            const double* __restrict__ scale,
                                                            double* __restrict__ part) {
  __shared__ double red[32];
  double v[7] = {0, 0, 0, 0, 0, 0, 0};
  const int64_t face = g.dims[0] * g.dims[1];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.N; i += stride) {
    const T mi = mobs[i], li = l[i], yi = y[i];
    const T h = mi - li + yi / (T)mu;
    T en;
    if (!mask[i]) {
      en = h;
    } else if (structure == 3) {
      en = T(0);
    } else if (structure == 0) {
      en = (T)prox(pen, level, (double)h);
    } else {
      const double sc = structure == 1 ? scale[i % face] : scale[i / face];
      en = (T)((double)h * sc);
    }
    const T fit = mi - li - en;
    const T yn = yi + (T)mu * fit;
    const double dl = (double)li - (double)lold[i];
    const double de = (double)en - (double)e[i];
    e[i] = en;
    y[i] = yn;
    v[0] = fmax(v[0], fabs(dl));
    v[1] += dl * dl;
    v[2] = fmax(v[2], fabs(de));
    v[3] += de * de;
    v[4] = fmax(v[4], fabs((double)fit));
    v[5] += (double)fit * (double)fit;
    v[6] += (double)yn * (double)yn;
  }
  block_partials<7>(v, 0b0010101u, red, part);
}

// one-bit data-fit update (onebit.py:128-138, 172-180):
//   L = clip((J1 + m mu Z - m Y [- J2 S]) / (J2 + m mu), -alpha, alpha)
//   robust: S = observed ? prox(lam2 m / c, J1/c - L) : 0   (c = J2)
//   partial q: 0 sum (L-Lold)^2  1 sum Lold^2  2 max|L-Lold|
template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_onebit_fit(int64_t N, const T* __restrict__ j1,
                                                            const T* __restrict__ j2, double m,
                                                            double mu, const T* __restrict__ z,
                                                            const T* __restrict__ y, double alpha,
                                                            const T* __restrict__ lold,
                                                            T* __restrict__ lnew,
                                                            T* __restrict__ s, int robust,
                                                            Penalty psi, double lam2,
                                                            double* __restrict__ part) {
  __shared__ double red[32];
  double v[3] = {0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    const T c = j2[i];
    T num = j1[i] + (T)(m * mu) * z[i] - (T)m * y[i];
    if (robust) num = num - c * s[i];
    T ln = num / (c + (T)(m * mu));
    ln = ln < (T)(-alpha) ? (T)(-alpha) : (ln > (T)alpha ? (T)alpha : ln);
    lnew[i] = ln;
    if (robust) {
      T sn = T(0);
      if (c > T(0)) {
        const T w = j1[i] / (c > T(1) ? c : T(1)) - ln;
        sn = (T)prox(psi, lam2 * m / (double)c, (double)w);
      }
      s[i] = sn;
    }
    const double lo = (double)lold[i];
    const double d = (double)ln - lo;
    v[0] += d * d;
    v[1] += lo * lo;
    v[2] = fmax(v[2], fabs(d));
  }
  block_partials<3>(v, 0b100u, red, part);
}

// one-bit dual update Y += mu (L - Z) (onebit.py:190) with max|L - Z| and ||Y||^2
template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_onebit_dual(int64_t N, const T* __restrict__ l,
                                                             const T* __restrict__ z,
                                                             T* __restrict__ y, double mu,
                                                             double* __restrict__ part) {
  __shared__ double red[32];
  double v[2] = {0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    const T gap = l[i] - z[i];
    const T yn = y[i] + (T)mu * gap;
    y[i] = yn;
    v[0] = fmax(v[0], fabs((double)gap));
    v[1] += (double)yn * (double)yn;
  }
  block_partials<2>(v, 0b01u, red, part);
}

template <typename T>
__global__ void k_fill(T* __restrict__ p, int64_t n, T v) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
}

// real T <-> fp64 (deterministic small-face t-SVT path)
template <typename A, typename B>
__global__ void k_convert(const A* __restrict__ in, B* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (B)in[i];
}

}  // namespace tr
