// Elementwise / stencil kernels of the ADMM solvers (tenrec/solvers.py:204-284,
// tenrec/onebit.py:141-220), each fused with the Eq. (24) residual reductions
// it can produce from the values it already holds.
//
// Kernels walk the tensor line by line (a line = the contiguous axis-0 fiber):
// the multi-index of a line, and so the circular-neighbour offsets along the
// other axes, is computed once per line, then the threads of the block stream
// along the line (coalesced).  Penalty kinds are template parameters so each
// instantiation carries only its own proximity operator.
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
  int64_t lst[kMaxOrder];  // st[a] / dims[0]: stride of axis a in the line index
  int64_t N;
  // sharded last axis (multi-GPU): the arrays a stencil reads along axis
  // `halo` carry one ghost face before and after their own faces, filled by the
  // neighbouring ranks, so the circular neighbour of a boundary face is the
  // ghost (no local wrap).  -1: every axis is whole and periodic.
  int halo = -1;
  // line-walk order of the resident line kernels (for_each_chunk): with
  // walk_last > 1 the last axis is visited fastest, so a line's neighbours
  // along the last axis -- whole faces (MBs) apart in memory -- are the
  // previous / next line of the walk and still in L2, while the ones along
  // the inner axes stay within a few MB of the walk.  0: memory order.
  int64_t walk_last = 0;
};

// offsets of the previous / next element along axis a (a >= 1) for a line
// whose axis-a coordinate is j
__device__ __forceinline__ void axis_offsets(const Geom& g, int a, int64_t j, int64_t& prev,
                                             int64_t& next) {
  const int64_t n = g.dims[a], s = g.st[a];
  if (a == g.halo) {
    prev = -s;
    next = s;
    return;
  }
  prev = j > 0 ? -s : s * (n - 1);
  next = j + 1 < n ? s : -s * (n - 1);
}

// coordinate of the line (index of axes 1..d-1 flattened) along axis a >= 1;
// 32-bit division when the line count allows (it does for any tensor < 2^31 lines)
__device__ __forceinline__ int64_t line_coord(const Geom& g, int64_t line, int a) {
  const int64_t lst = g.lst[a];
  if (line < (1ll << 31) && lst < (1ll << 31) && g.dims[a] < (1ll << 31))
    return (int64_t)(((uint32_t)line / (uint32_t)lst) % (uint32_t)g.dims[a]);
  return (line / lst) % g.dims[a];
}

template <typename T>
struct ModePtrs {
  int count;
  int axis[kMaxOrder];  // -1 = identity chain (pure low-rank ablation)
  T* p[kMaxOrder];
};

// V consecutive elements of one line (V = 4: 16-byte accesses when the host
// checked n0 % 4 == 0 and 16-byte aligned buffers; V = 1 otherwise).
template <typename T, int V>
struct Vec {
  T x[V];
};

template <typename T, int V>
__device__ __forceinline__ Vec<T, V> ldv(const T* p) {
  Vec<T, V> r;
  if constexpr (V == 4 && sizeof(T) == 4) {
    const float4 f = *reinterpret_cast<const float4*>(p);
    r.x[0] = f.x; r.x[1] = f.y; r.x[2] = f.z; r.x[3] = f.w;
  } else if constexpr (V == 4 && sizeof(T) == 8) {
    const double2 a = reinterpret_cast<const double2*>(p)[0];
    const double2 b = reinterpret_cast<const double2*>(p)[1];
    r.x[0] = a.x; r.x[1] = a.y; r.x[2] = b.x; r.x[3] = b.y;
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) r.x[j] = p[j];
  }
  return r;
}

// read-only variant (ld.global.nc): the compiler may schedule these loads
// across the kernel's stores, which raises memory-level parallelism
template <typename T, int V>
__device__ __forceinline__ Vec<T, V> ldv_nc(const T* p) {
  Vec<T, V> r;
  if constexpr (V == 4 && sizeof(T) == 4) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(p));
    r.x[0] = f.x; r.x[1] = f.y; r.x[2] = f.z; r.x[3] = f.w;
  } else if constexpr (V == 4 && sizeof(T) == 8) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    r.x[0] = a.x; r.x[1] = a.y; r.x[2] = b.x; r.x[3] = b.y;
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) r.x[j] = __ldg(p + j);
  }
  return r;
}

template <typename T, int V>
__device__ __forceinline__ void stv(T* p, const T (&v)[V]) {
  if constexpr (V == 4 && sizeof(T) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (V == 4 && sizeof(T) == 8) {
    reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) p[j] = v[j];
  }
}

template <int V>
__device__ __forceinline__ void ld_mask(const uint8_t* p, bool (&m)[V]) {
  if constexpr (V == 4) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = ((w >> (8 * j)) & 0xffu) != 0;
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) m[j] = p[j] != 0;
  }
}

// A line (axis-0 fiber) and its coordinates along axes 1..d-1.
struct LineCo {
  int64_t line;
  int co[kMaxOrder];
};

// Walk every V-element chunk of every axis-0 line: f(lc, i0).  Long lines:
// grid-stride over the lines in memory order with a RESIDENT grid (the host
// sizes it to SMs x occupancy), so every block advances in lockstep and a
// line's neighbours along the outer axes (+-1 line, +-n1 lines, ...) are read
// by some block within about one iteration -- the stencil re-reads hit L2.
// Short lines pack several per pass.
template <int V, typename F>
__device__ __forceinline__ void for_each_chunk(const Geom& g, F&& f) {
  const int64_t n0 = g.dims[0], lines = g.N / n0;
  const int cpl = (int)(n0 / V);
  LineCo lc;
  if (cpl >= (int)blockDim.x) {
    const int64_t wl = g.walk_last, per = wl > 1 ? lines / wl : lines;
    // walk position v = vr + wl * vq visits line vr * per + vq (last axis fastest);
    // (vr, vq) advance incrementally: no 64-bit division per line
    const int64_t dq = wl > 1 ? (int64_t)gridDim.x / wl : 0, dr = wl > 1 ? (int64_t)gridDim.x % wl : 0;
    int64_t vq = wl > 1 ? (int64_t)blockIdx.x / wl : 0, vr = wl > 1 ? (int64_t)blockIdx.x % wl : 0;
    for (int64_t v = blockIdx.x; v < lines; v += gridDim.x) {
      lc.line = wl > 1 ? vr * per + vq : v;
      if (wl > 1 && lines < (1ll << 31)) {
        // coordinates straight from the walk position: the last axis is vr, the
        // inner axes unflatten vq (no division at all for an order-3 tensor)
        lc.co[g.d - 1] = (int)vr;
        uint32_t rem = (uint32_t)vq;
        for (int a = 1; a < g.d - 2; ++a) {
          const uint32_t n = (uint32_t)g.dims[a], q = rem / n;
          lc.co[a] = (int)(rem - q * n);
          rem = q;
        }
        if (g.d >= 3) lc.co[g.d - 2] = (int)rem;
      } else {
        for (int a = 1; a < g.d; ++a) lc.co[a] = (int)line_coord(g, lc.line, a);
      }
      vq += dq;
      vr += dr;
      if (vr >= wl) {
        vr -= wl;
        ++vq;
      }
      for (int c = threadIdx.x; c < cpl; c += blockDim.x) f(lc, (int64_t)c * V);
    }
  } else {
    const int lpi = (int)blockDim.x / cpl;
    const int sub = (int)threadIdx.x / cpl, c = (int)threadIdx.x - sub * cpl;
    if (sub >= lpi) return;
    for (int64_t l0 = (int64_t)blockIdx.x * lpi; l0 < lines; l0 += (int64_t)gridDim.x * lpi) {
      lc.line = l0 + sub;
      if (lc.line >= lines) continue;
      for (int a = 1; a < g.d; ++a) lc.co[a] = (int)line_coord(g, lc.line, a);
      f(lc, (int64_t)c * V);
    }
  }
}

// forward difference D_a x at the V elements of a chunk (x already loaded);
// a < 0: identity chain
template <typename T, int V>
__device__ __forceinline__ void fwd_diff(const Geom& g, const T* x, int a, const LineCo& lc,
                                         int64_t base, int64_t i0, const Vec<T, V>& xv,
                                         T (&out)[V]) {
  const int64_t n0 = g.dims[0];
  if (a < 0) {
#pragma unroll
    for (int j = 0; j < V; ++j) out[j] = xv.x[j];
  } else if (a == 0) {
    const T last = __ldg(x + base + (i0 + V < n0 ? i0 + V : 0));
#pragma unroll
    for (int j = 0; j < V; ++j) out[j] = (j + 1 < V ? xv.x[j + 1] : last) - xv.x[j];
  } else {
    int64_t pv, nx;
    axis_offsets(g, a, lc.co[a], pv, nx);
    const Vec<T, V> xn = ldv_nc<T, V>(x + base + i0 + nx);
#pragma unroll
    for (int j = 0; j < V; ++j) out[j] = xn.x[j] - xv.x[j];
  }
}

template <int KIND>
__device__ __forceinline__ double prox_k(double p0, double p1, double mu, double v) {
  Penalty pen{KIND, p0, p1};
  return prox(pen, mu, v);
}

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

// One warp per quantity (fixed order: lane-strided partials, then the xor tree):
// the quantities reduce side by side instead of one block-wide reduction each.
__global__ void k_final_reduce(const double* __restrict__ part, int nblocks, int nq,
                               unsigned is_max, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int q = warp; q < nq; q += nw) {
    const bool mx = (is_max >> q) & 1;
    double v = 0.0;
    for (int b = lane; b < nblocks; b += 32) {
      const double x = part[(int64_t)b * nq + q];
      v = mx ? fmax(v, x) : v + x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, v, o);
      v = mx ? fmax(v, x) : v + x;
    }
    if (lane == 0) out[q] = v;
  }
}

// rhs of the L- (or Z-) subproblem (solvers.py:231-233, onebit.py:182-184):
//   b = A - B + y / mu ;  rhs = b + sum_k D_k^T (g_k - lag_k / mu)
// pure low-rank chain: out = 0.5 * (b + g - lag / mu)  (solvers.py:194-195), the final L.
template <typename T, int V>
__global__ void __launch_bounds__(kRedThreads) k_admm_rhs(Geom g, const T* __restrict__ A,
                                                          const T* __restrict__ B,
                                                          const T* __restrict__ y, double mu,
                                                          ModePtrs<T> gm, ModePtrs<T> lag,
                                                          T* __restrict__ out) {
  const int64_t n0 = g.dims[0];
  const T imu = (T)(1.0 / mu);
  const bool pure = gm.count == 1 && gm.axis[0] < 0;
  for_each_chunk<V>(g, [&](const LineCo& lc, int64_t i0) {
    const int64_t line = lc.line;
    const int64_t base = line * n0, i = base + i0;
    const Vec<T, V> av = ldv<T, V>(A + i), yv = ldv<T, V>(y + i);
    Vec<T, V> bv;
    if (B) bv = ldv<T, V>(B + i);
    T acc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = (B ? (av.x[j] - bv.x[j]) : av.x[j]) + yv.x[j] * imu;
    if (pure) {
      const Vec<T, V> gv = ldv<T, V>(gm.p[0] + i), lv = ldv<T, V>(lag.p[0] + i);
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = (T)0.5 * (acc[j] + (gv.x[j] - lv.x[j] * imu));
      stv<T, V>(out + i, acc);
      return;
    }
#pragma unroll
    for (int k = 0; k < kMaxOrder; ++k) {
      if (k < gm.count) {
        const int a = gm.axis[k];
        const Vec<T, V> gv = ldv<T, V>(gm.p[k] + i), lv = ldv<T, V>(lag.p[k] + i);
        T gi[V], gp[V];
#pragma unroll
        for (int j = 0; j < V; ++j) gi[j] = gv.x[j] - lv.x[j] * imu;
        if (a == 0) {
          const int64_t ip = base + (i0 > 0 ? i0 - 1 : n0 - 1);
          gp[0] = gm.p[k][ip] - lag.p[k][ip] * imu;
#pragma unroll
          for (int j = 1; j < V; ++j) gp[j] = gi[j - 1];
        } else {
          int64_t pv, nx;
          axis_offsets(g, a, lc.co[a], pv, nx);
          const Vec<T, V> gq = ldv<T, V>(gm.p[k] + i + pv), lq = ldv<T, V>(lag.p[k] + i + pv);
#pragma unroll
          for (int j = 0; j < V; ++j) gp[j] = gq.x[j] - lq.x[j] * imu;
        }
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] += gp[j] - gi[j];
      }
    }
    stv<T, V>(out + i, acc);
  });
}

// LRTA inputs of every mode (one pass over L): X_k = D_k L + lag_k / mu
// (identity chain: L + lag / mu) for up to 4 modes (the host launches groups).
// All loads of a chunk are issued before its stores.
template <typename T, int V>
__global__ void __launch_bounds__(kRedThreads) k_lrta_input(Geom g, const T* __restrict__ l,
                                                            ModePtrs<T> lag, ModePtrs<T> X,
                                                            double mu) {
  constexpr int MM = 4;
  const T imu = (T)(1.0 / mu);
  const int64_t n0 = g.dims[0];
  const int nm = lag.count;
  for_each_chunk<V>(g, [&](const LineCo& lc, int64_t i0) {
    const int64_t base = lc.line * n0, i = base + i0;
    const Vec<T, V> lv = ldv_nc<T, V>(l + i);
    Vec<T, V> mv[MM], xn[MM];
#pragma unroll
    for (int k = 0; k < MM; ++k) {
      if (k < nm) {
        const int a = lag.axis[k];
        mv[k] = ldv_nc<T, V>(lag.p[k] + i);
        if (a == 0) {
          xn[k].x[0] = __ldg(l + base + (i0 + V < n0 ? i0 + V : 0));
        } else if (a > 0) {
          int64_t pv, nx;
          axis_offsets(g, a, lc.co[a], pv, nx);
          xn[k] = ldv_nc<T, V>(l + i + nx);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < MM; ++k) {
      if (k < nm) {
        const int a = lag.axis[k];
        T o[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const T gl = a < 0 ? lv.x[j]
                             : (a == 0 ? (j + 1 < V ? lv.x[j + 1] : xn[k].x[0]) : xn[k].x[j]) - lv.x[j];
          o[j] = gl + mv[k].x[j] * imu;
        }
        stv<T, V>(X.p[k] + i, o);
      }
    }
  });
}

// multiplier updates of NM modes (solvers.py:247-248) with their residuals:
//   lag_k += mu (D_k L - G_new,k);  partial 5k+q: 0 max|DL-G|, 1 sum (DL-G)^2,
//   2 max|G_new-G_old|, 3 sum (G_new-G_old)^2, 4 sum lag_new^2
template <typename T, int V, int NM>
__global__ void __launch_bounds__(kRedThreads) k_lag_update(Geom g, const T* __restrict__ l,
                                                            ModePtrs<T> gnew, ModePtrs<T> gold,
                                                            ModePtrs<T> lag, double mu,
                                                            double* __restrict__ part) {
  __shared__ double red[32];
  double v[5 * NM];
#pragma unroll
  for (int q = 0; q < 5 * NM; ++q) v[q] = 0.0;
  const int64_t n0 = g.dims[0];
  const T tmu = (T)mu;
  for_each_chunk<V>(g, [&](const LineCo& lc, int64_t i0) {
    const int64_t line = lc.line;
    const int64_t base = line * n0, i = base + i0;
    const Vec<T, V> lv = ldv<T, V>(l + i);
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      T gl[V];
      fwd_diff<T, V>(g, l, lag.axis[k], lc, base, i0, lv, gl);
      const Vec<T, V> gn = ldv<T, V>(gnew.p[k] + i), go = ldv<T, V>(gold.p[k] + i);
      const Vec<T, V> lo = ldv<T, V>(lag.p[k] + i);
      T ln[V];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const T gap = gl[j] - gn.x[j];
        ln[j] = lo.x[j] + tmu * gap;
        const double dg = (double)gn.x[j] - (double)go.x[j];
        v[5 * k + 0] = fmax(v[5 * k + 0], fabs((double)gap));
        v[5 * k + 1] += (double)gap * (double)gap;
        v[5 * k + 2] = fmax(v[5 * k + 2], fabs(dg));
        v[5 * k + 3] += dg * dg;
        v[5 * k + 4] += (double)ln[j] * (double)ln[j];
      }
      stv<T, V>(lag.p[k] + i, ln);
    }
  });
  constexpr unsigned kMaxMask = 0b00101u;
  unsigned mask = 0;
#pragma unroll
  for (int k = 0; k < NM; ++k) mask |= kMaxMask << (5 * k);
  block_partials<5 * NM>(v, mask, red, part);
}

// group scales of the structured noise shrinkage (shrink.py:49-54) of
// mask * h, h = mobs - l + y / mu:  scale = prox(level, ||group||) / ||group||.
// structure 1 = tube (i0, i1) over trailing modes, 2 = slice (face) over (i0, i1).
template <typename T, int KIND>
__global__ void k_group_scale(Geom g, int structure, const T* __restrict__ mobs,
                              const uint8_t* __restrict__ mask, const T* __restrict__ l,
                              const T* __restrict__ y, double mu, double p0, double p1,
                              double level, double* __restrict__ scale) {
  const T imu = (T)(1.0 / mu);
  const int64_t face = g.dims[0] * g.dims[1];
  const int64_t nf = g.N / face;
  if (structure == 1) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= face) return;
    double s2 = 0.0;
    for (int64_t f = 0; f < nf; ++f) {
      const int64_t i = t + face * f;
      const double h = mask[i] ? (double)(mobs[i] - l[i] + y[i] * imu) : 0.0;
      s2 += h * h;
    }
    const double gn = sqrt(s2);
    scale[t] = gn > 0 ? prox_k<KIND>(p0, p1, level, gn) / gn : 0.0;
  } else {
    __shared__ double red[32];
    const int64_t f = blockIdx.x;
    double s2 = 0.0;
    for (int64_t e = threadIdx.x; e < face; e += blockDim.x) {
      const int64_t i = e + face * f;
      const double h = mask[i] ? (double)(mobs[i] - l[i] + y[i] * imu) : 0.0;
      s2 += h * h;
    }
    const double gn = sqrt(block_sum(s2, red));
    if (threadIdx.x == 0) scale[f] = gn > 0 ? prox_k<KIND>(p0, p1, level, gn) / gn : 0.0;
  }
}

// noise and dual updates (solvers.py:239-246) with residuals:
//   h = mobs - l + y/mu ; E = mask*shrink(mask*h) + (1-mask)*h ; y += mu (mobs - l - E)
//   structure 0 entry / 1 tube / 2 slice / 3 noise-free (E = 0 on the mask)
//   partial q: 0 max|l-lold| 1 sum 2 max|E-Eold| 3 sum 4 max|fit| 5 sum 6 sum y^2
// Prox in the streaming precision for the closed-form families (l1, firm,
// mcp, scad); the iterative / candidate families (lq, capped-lq, log) stay fp64.
template <int KIND, typename T>
__device__ __forceinline__ T prox_t(T p0, double p0d, double p1d, T mu, double mud, T v) {
  if (KIND <= 3) {
    if (mu == T(0)) return v;
    const T a = v < T(0) ? -v : v;
    T r;
    if (KIND == 0) {
      r = a > mu ? a - mu : T(0);
    } else if (KIND == 1 || KIND == 2) {
      r = a <= mu ? T(0) : (a < p0 * mu ? p0 * (a - mu) / (p0 - T(1)) : a);
    } else {
      r = a <= T(2) * mu ? (a > mu ? a - mu : T(0))
                         : (a <= p0 * mu ? ((p0 - T(1)) * a - p0 * mu) / (p0 - T(2)) : a);
    }
    return v > T(0) ? r : (v < T(0) ? -r : T(0));
  } else {
    return (T)prox_k<KIND>(p0d, p1d, mud, (double)v);
  }
}

// STRUCT: 0 entry, 1 tube, 2 slice, 3 noise-free (E = 0 on the mask)
template <typename T, int KIND, int STRUCT, int V>
__global__ void __launch_bounds__(kRedThreads) k_noise_dual(Geom g, const T* __restrict__ mobs,
                                                            const uint8_t* __restrict__ mask,
                                                            const T* __restrict__ l,
                                                            const T* __restrict__ lold,
                                                            T* __restrict__ e, T* __restrict__ y,
                                                            double mu, double p0, double p1,
                                                            double level,
                                                            const double* __restrict__ scale,
                                                            double* __restrict__ part) {
  __shared__ double red[32];
  // per-thread partials in T (fp32 sums over <= a few hundred elements), per-block fp64
  T v[7] = {T(0), T(0), T(0), T(0), T(0), T(0), T(0)};
  const int64_t face = g.dims[0] * g.dims[1];
  const int64_t n0 = g.dims[0];
  const T tmu = (T)mu, tlev = (T)level, tp0 = (T)p0, timu = (T)(1.0 / mu);
  for_each_chunk<V>(g, [&](const LineCo& lc, int64_t i0) {
    const int64_t line = lc.line;
    const int64_t i = line * n0 + i0;
    const Vec<T, V> mv = ldv<T, V>(mobs + i), lv = ldv<T, V>(l + i), yv = ldv<T, V>(y + i);
    const Vec<T, V> ev = ldv<T, V>(e + i), ov = ldv<T, V>(lold + i);
    bool obs[V];
    ld_mask<V>(mask + i, obs);
    T en[V], yn[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const T mi = mv.x[j], li = lv.x[j], yi = yv.x[j];
      const T h = mi - li + yi * timu;
      T ej;
      if (!obs[j]) {
        ej = h;
      } else if (STRUCT == 3) {
        ej = T(0);
      } else if (STRUCT == 0) {
        ej = prox_t<KIND, T>(tp0, p0, p1, tlev, level, h);
      } else {
        const double sc = STRUCT == 1 ? scale[(i + j) % face] : scale[(i + j) / face];
        ej = (T)((double)h * sc);
      }
      const T fit = mi - li - ej;
      en[j] = ej;
      yn[j] = yi + tmu * fit;
      const T dl = li - ov.x[j], de = ej - ev.x[j];
      v[0] = fmax(v[0], fabs(dl));
      v[1] += dl * dl;
      v[2] = fmax(v[2], fabs(de));
      v[3] += de * de;
      v[4] = fmax(v[4], fabs(fit));
      v[5] += fit * fit;
      v[6] += yn[j] * yn[j];
    }
    stv<T, V>(e + i, en);
    stv<T, V>(y + i, yn);
  });
  double vd[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) vd[q] = (double)v[q];
  block_partials<7>(vd, 0b0010101u, red, part);
}

// Tail of ADMM sweep t and head of sweep t+1 in ONE pass (solvers.py:244-248,
// then 230-232 of the next iteration), for the gradient chain with <= 4 modes:
//   lag'_k = lag_k + mu (D_k L - G_k)          written to lagw_k (double buffer:
//                                              neighbours still read lag_k)
//   E', Y'  exactly as k_noise_dual
//   rhs'    = A - E' + Y'/mu' + sum_k D_k^T (G_k - lag'_k / mu'),  mu' = min(mu_max, growth mu)
// D_k^T at i needs lag'_k at ip = i - e_k; it is recomputed from lag_k, G_k, L
// at ip with the very expression the owner of ip evaluates, so rhs' is
// bit-identical to k_admm_rhs of the next sweep.  Partials per block: 5 per
// mode slot (k_lag_update's, 4 slots) then the 7 of k_noise_dual.
// NOISE = false: E' and Y' were already written in place by k_noise_dual
// (launched on the main stream while the per-mode t-SVTs ran); the pass reads
// them instead of recomputing them and leaves the 7 noise partials at zero.
template <typename T, int KIND, int STRUCT, bool NOISE = true, int V = 4, int MINB = 1>
__global__ void __launch_bounds__(kRedThreads, MINB) k_sweep_tail(
    Geom g, const T* __restrict__ mobs, const uint8_t* __restrict__ mask, const T* __restrict__ l,
    const T* __restrict__ lold, T* __restrict__ e, T* __restrict__ y, ModePtrs<T> gn, ModePtrs<T> go,
    ModePtrs<T> lag, ModePtrs<T> lagw, double mu, double mu_next, double p0, double p1,
    double level, const double* __restrict__ scale, T* __restrict__ rhs,
    double* __restrict__ part) {
  constexpr int MM = 4;  // mode slots
  __shared__ double red[32];
  // per-thread partials in T (sums over a few hundred elements), per-block fp64
  T vl[5 * MM], vn[7];
#pragma unroll
  for (int q = 0; q < 5 * MM; ++q) vl[q] = T(0);
#pragma unroll
  for (int q = 0; q < 7; ++q) vn[q] = T(0);
  const int nm = gn.count;
  const int64_t n0 = g.dims[0], face = g.dims[0] * g.dims[1];
  const T tmu = (T)mu, tlev = (T)level, tp0 = (T)p0, timu = (T)(1.0 / mu);
  const T imu2 = (T)(1.0 / mu_next);
  for_each_chunk<V>(g, [&](const LineCo& lc, int64_t i0) {
    const int64_t base = lc.line * n0, i = base + i0;
    // ---- every load of the chunk first (memory-level parallelism) ----
    const Vec<T, V> lv = ldv_nc<T, V>(l + i), mv = ldv_nc<T, V>(mobs + i);
    Vec<T, V> ov;
    if (NOISE) ov = ldv_nc<T, V>(lold + i);
    const Vec<T, V> yv = ldv<T, V>(y + i), ev = ldv<T, V>(e + i);
    bool obs[V];
    if (NOISE) ld_mask<V>(mask + i, obs);
    Vec<T, V> gnv[MM], gov[MM], lgv[MM], lnx[MM], lpv[MM], gpv[MM], mpv[MM];
#pragma unroll
    for (int k = 0; k < MM; ++k) {
      if (k < nm) {
        const int a = lag.axis[k];
        gnv[k] = ldv_nc<T, V>(gn.p[k] + i);
        gov[k] = ldv_nc<T, V>(go.p[k] + i);
        lgv[k] = ldv_nc<T, V>(lag.p[k] + i);
        if (a == 0) {
          const int64_t inext = base + (i0 + V < n0 ? i0 + V : 0);
          const int64_t ip = base + (i0 > 0 ? i0 - 1 : n0 - 1);
          lnx[k].x[0] = __ldg(l + inext);
          lpv[k].x[0] = __ldg(l + ip);
          gpv[k].x[0] = __ldg(gn.p[k] + ip);
          mpv[k].x[0] = __ldg(lag.p[k] + ip);
        } else {
          int64_t pv, nx;
          axis_offsets(g, a, lc.co[a], pv, nx);
#ifdef TR_TAIL_PROBE_SKIP_AXIS
          if (a >= TR_TAIL_PROBE_SKIP_AXIS) pv = nx = 0;
#endif
          lnx[k] = ldv_nc<T, V>(l + i + nx);
          lpv[k] = ldv_nc<T, V>(l + i + pv);
          gpv[k] = ldv_nc<T, V>(gn.p[k] + i + pv);
          mpv[k] = ldv_nc<T, V>(lag.p[k] + i + pv);
        }
      }
    }
    // ---- noise and dual (k_noise_dual) ----
    T en[V], yn[V], acc[V];
    if (!NOISE) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        en[j] = ev.x[j];  // already E', Y'
        yn[j] = yv.x[j];
        acc[j] = (mv.x[j] - en[j]) + yn[j] * imu2;
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (!NOISE) break;
      const T mi = mv.x[j], li = lv.x[j], yi = yv.x[j];
      const T h = mi - li + yi * timu;
      T ej;
      if (!obs[j]) {
        ej = h;
      } else if (STRUCT == 3) {
        ej = T(0);
      } else if (STRUCT == 0) {
        ej = prox_t<KIND, T>(tp0, p0, p1, tlev, level, h);
      } else {
        const double sc = STRUCT == 1 ? scale[(i + j) % face] : scale[(i + j) / face];
        ej = (T)((double)h * sc);
      }
      const T fit = mi - li - ej;
      en[j] = ej;
      yn[j] = yi + tmu * fit;
      const T dl = li - ov.x[j], de = ej - ev.x[j];
      vn[0] = fmax(vn[0], fabs(dl));
      vn[1] += dl * dl;
      vn[2] = fmax(vn[2], fabs(de));
      vn[3] += de * de;
      vn[4] = fmax(vn[4], fabs(fit));
      vn[5] += fit * fit;
      vn[6] += yn[j] * yn[j];
      acc[j] = (mi - ej) + yn[j] * imu2;  // b' = A - E' + Y' / mu'
    }
    if (NOISE) {
      stv<T, V>(e + i, en);
      stv<T, V>(y + i, yn);
    }
    // ---- multipliers (k_lag_update) and the next rhs (k_admm_rhs) ----
#pragma unroll
    for (int k = 0; k < MM; ++k) {
      if (k < nm) {
        const int a = lag.axis[k];
        T gl[V], ln[V], gi[V], gp[V];
#pragma unroll
        for (int j = 0; j < V; ++j)  // D_a L (as fwd_diff)
          gl[j] = (a == 0 ? (j + 1 < V ? lv.x[j + 1] : lnx[k].x[0]) : lnx[k].x[j]) - lv.x[j];
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const T gap = gl[j] - gnv[k].x[j];
          ln[j] = lgv[k].x[j] + tmu * gap;
          const T dg = gnv[k].x[j] - gov[k].x[j];
          vl[5 * k + 0] = fmax(vl[5 * k + 0], fabs(gap));
          vl[5 * k + 1] += gap * gap;
          vl[5 * k + 2] = fmax(vl[5 * k + 2], fabs(dg));
          vl[5 * k + 3] += dg * dg;
          vl[5 * k + 4] += ln[j] * ln[j];
          gi[j] = gnv[k].x[j] - ln[j] * imu2;
        }
        stv<T, V>(lagw.p[k] + i, ln);
        // lag' at ip = i - e_a, with its owner's expression (D_a L at ip = L[i] - L[ip])
        if (a == 0) {
          const T gap = (lv.x[0] - lpv[k].x[0]) - gpv[k].x[0];
          const T lnp = mpv[k].x[0] + tmu * gap;
          gp[0] = gpv[k].x[0] - lnp * imu2;
#pragma unroll
          for (int j = 1; j < V; ++j) gp[j] = gi[j - 1];
        } else {
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const T gap = (lv.x[j] - lpv[k].x[j]) - gpv[k].x[j];
            const T lnp = mpv[k].x[j] + tmu * gap;
            gp[j] = gpv[k].x[j] - lnp * imu2;
          }
        }
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] += gp[j] - gi[j];
      }
    }
    stv<T, V>(rhs + i, acc);
  });
  double vd[27];
#pragma unroll
  for (int q = 0; q < 20; ++q) vd[q] = (double)vl[q];
#pragma unroll
  for (int q = 0; q < 7; ++q) vd[20 + q] = (double)vn[q];
  constexpr unsigned kMax = 0b00101u | (0b00101u << 5) | (0b00101u << 10) | (0b00101u << 15) |
                            (0b0010101u << 20);
  block_partials<27>(vd, kMax, red, part);
}

// one-bit data-fit update (onebit.py:128-138, 172-180):
//   L = clip((J1 + m mu Z - m Y [- J2 S]) / (J2 + m mu), -alpha, alpha)
//   robust: S = observed ? prox(lam2 m / c, J1/c - L) : 0   (c = J2)
//   partial q: 0 sum (L-Lold)^2  1 sum Lold^2  2 max|L-Lold|
template <typename T, int KIND>
__global__ void __launch_bounds__(kRedThreads) k_onebit_fit(int64_t N, const T* __restrict__ j1,
                                                            const T* __restrict__ j2, double m,
                                                            double mu, const T* __restrict__ z,
                                                            const T* __restrict__ y, double alpha,
                                                            const T* __restrict__ lold,
                                                            T* __restrict__ lnew,
                                                            T* __restrict__ s, int robust,
                                                            double p0, double p1, double lam2,
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
        sn = (T)prox_k<KIND>(p0, p1, lam2 * m / (double)c, (double)w);
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

// real T <-> fp64 (deterministic small-face t-SVT path)
template <typename A, typename B>
__global__ void k_convert(const A* __restrict__ in, B* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (B)in[i];
}

// launch a KIND-templated kernel for a runtime penalty kind
#define TR_PEN_DISPATCH(kind, CALL) \
  switch (kind) {                   \
    case 0: CALL(0); break;         \
    case 1: CALL(1); break;         \
    case 2: CALL(2); break;         \
    case 3: CALL(3); break;         \
    case 4: CALL(4); break;         \
    case 5: CALL(5); break;         \
    default: CALL(6); break;        \
  }

}  // namespace tr
