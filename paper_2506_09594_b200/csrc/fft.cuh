// Batched FFTs along one axis of a column-major tensor, and the FFT-diagonal
// solve of tenrec/gradient.py:90-106:
//     (I + sum_{k in Gamma} D_k^T D_k) L = rhs,   D_k = forward circular difference
// which is diagonal under the full d-dimensional DFT with eigenvalues
// 1 + sum_k 4 sin^2(pi j_k / n_k) (gradient.py:63-80).
//
// Layout: element (lo, k, hi) of an axis of length n with lo-stride st lives at
// lo + st * (k + n * hi).  One CTA loads a tile of `L` lines (consecutive lo
// when st > 1 for coalescing, consecutive hi when the axis is contiguous) into
// shared memory and transforms every line there:
//   * powers of two: radix-4 Stockham autosort (radix-2 last stage when log2 n
//     is odd), each thread holding its groups in registers, twiddles in smem;
//   * other lengths: direct DFT.
// Axis 0 is real-to-complex on the way in (n0/2+1 bins, the conjugate-even half
// spectrum of a real tensor) and complex-to-real on the way out.  The last-axis
// pass of the solve does forward FFT -> divide -> inverse FFT in shared memory.
#pragma once

#include "common.cuh"

namespace tr {

template <typename T>
struct __align__(2 * sizeof(T)) cpx {
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
template <typename T>
__device__ __forceinline__ cpx<T> cconjt(cpx<T> a) { return {a.re, -a.im}; }

enum FftMode { FFT_C2C = 0, FFT_R2C = 1, FFT_C2R = 2 };

__host__ __device__ constexpr int bitrev_c(int i, int bits) {
  return bits == 0 ? 0 : (((i & 1) << (bits - 1)) | bitrev_c(i >> 1, bits - 1));
}

template <int N>
__host__ __device__ constexpr int log2_c() {
  return N <= 1 ? 0 : 1 + log2_c<N / 2>();
}

// One radix-2 stage (butterfly span LEN) of reg_fft, fully unrolled.
template <typename T, int N, int TS, int LEN>
__device__ __forceinline__ void reg_fft_stage(cpx<T> (&v)[N], const cpx<T>* ts, bool inverse) {
#pragma unroll
  for (int i = 0; i < N; i += LEN)
#pragma unroll
    for (int j = 0; j < LEN / 2; ++j) {
      constexpr int STEP = N / LEN;
      const int widx = j * STEP;  // of N
      const cpx<T> u = v[i + j];
      const cpx<T> x = v[i + j + LEN / 2];
      cpx<T> t;
      if (widx == 0) {
        t = x;
      } else if (4 * widx == N) {  // w = -i (forward) / +i (inverse)
        t = inverse ? cpx<T>{-x.im, x.re} : cpx<T>{x.im, -x.re};
      } else {
        cpx<T> w = ts[widx * TS];
        if (inverse) w.im = -w.im;
        t = cmulc(w, x);
      }
      v[i + j] = cadd(u, t);
      v[i + j + LEN / 2] = csub(u, t);
    }
  if constexpr (LEN < N) reg_fft_stage<T, N, TS, 2 * LEN>(v, ts, inverse);
}

// In-register radix-2 FFT of N = 2^k points (unnormalised; ts = the N-point
// forward table -- or any table of which every TS-th entry is, TS = 1 by
// default -- conjugated for the inverse).  Every index is a compile-time
// constant (stages unrolled by template recursion), so the line stays in
// registers and the trivial twiddles (1, -i) cost nothing.
template <typename T, int N, int TS = 1>
__device__ __forceinline__ void reg_fft(cpx<T> (&v)[N], const cpx<T>* ts, bool inverse) {
  constexpr int LB = log2_c<N>();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    // bit reversal as a bit-reverse intrinsic of a constant (folded after unrolling)
    const int j = LB == 0 ? 0 : (int)(__brev((unsigned)i) >> (32 - LB));
    if (j > i) {
      const cpx<T> t = v[i];
      v[i] = v[j];
      v[j] = t;
    }
  }
  if constexpr (N >= 2) reg_fft_stage<T, N, TS, 2>(v, ts, inverse);
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

// q = a / b, r = a % b with a 32-bit division when both fit (a 64-bit division is
// ~100 instructions per thread -- a sizeable share of a register-FFT tile)
__device__ __forceinline__ void divmod_fast(int64_t a, int64_t b, int64_t& q, int64_t& r) {
  if (((a | b) >> 31) == 0) {
    const uint32_t qq = (uint32_t)a / (uint32_t)b;
    q = qq;
    r = (uint32_t)a - qq * (uint32_t)b;
  } else {
    q = a / b;
    r = a - q * b;
  }
}

struct SolveSpec {
  int active;           // last-axis pass of the diagonal solve
  int d;                // tensor order
  int64_t dims[10];     // spectrum dims (axis 0 = n0/2+1 in the half-spectrum layout)
  int64_t lam_off[10];  // offset of axis k's 4 sin^2(pi j / n_k) table, -1 if k not in Gamma
  int64_t lo_base = 0;  // global index of local lo-element 0 (the all-to-all layout of a
                        // sharded solve: this rank's slice of the axes before the last)
};

// Four-step C2C pass for N = P * N2 points (P <= N2, both powers of two), in
// place: n = n1 + P n2, k = k2 + N2 k1.  A line is served by P threads; thread
// n1 holds x[n1 + P n2] (n2 < N2) in registers, runs the inner N2-point FFT,
// applies W_N^(n1 k2), and the line's P x N2 matrix is transposed through
// shared memory so that each thread ends with N2 / P columns k2 = n1 + P c of
// all P rows for the outer P-point FFTs: X[k2 + N2 k1].  Two register FFTs and
// one shared-memory exchange per pass -- against four smem round trips of the
// radix-8 tile kernel.
//   STRIDED = false: contiguous lines (line l at l * N); a warp reads and
//     writes 32 / P runs of P consecutive points.  P >= 8.
//   STRIDED = true: lines at lo-stride st (element (lo, k) at lo + st (k + N h));
//     the 256 / P lines of a CTA are consecutive lo, so a warp reads and writes
//     32 consecutive lo of one point.  P <= 8.
// `ss.active` (the last-axis pass of the solve): forward, divide by
// 1 + sum_k 4 sin^2, inverse (through one more exchange), as k_fft_t.
template <int N2>
__host__ __device__ constexpr int fft4_smem_cpx() {
  return N2 + 256 * (N2 + 1);  // N2-point table + exchange
}

// One four-step transform of the register line v (input layout: v[j] =
// x[n1 + P j], n1 = this thread's row) into u (output layout: u[c][k1] =
// X[k2 + N2 k1], k2 = n1 + P c) through the exchange buffer.
template <typename T, int P, int N2, bool STRIDED>
__device__ __forceinline__ int fft4_xa(int g, int n1, int k2) {
  return STRIDED ? (n1 * N2 + k2) * (256 / P) + g : g * (P * (N2 + 1)) + n1 * (N2 + 1) + k2;
}

// (twiddles W_N^m read as tw[TWS m]: the n0-point table of a real pass serves
// its N = n0 / 2-point complex transform with TWS = 2)
template <typename T, int P, int N2, bool STRIDED, int TWS>
__device__ __forceinline__ void four_step_tw(cpx<T> (&v)[N2], cpx<T> (&u)[N2 / P][P],
                                             const cpx<T>* tsn, const cpx<T>* __restrict__ tw,
                                             cpx<T>* xch, int g, int p, bool inv) {
  constexpr int N = N2 * P, CP = N2 / P;
  reg_fft<T, N2>(v, tsn, inv);
#pragma unroll
  for (int k2 = 1; k2 < N2; ++k2) {  // W_N^(n1 k2)
    cpx<T> w = tw[TWS * ((p * k2) % N)];
    if (inv) w.im = -w.im;
    v[k2] = cmulc(v[k2], w);
  }
#pragma unroll
  for (int k2 = 0; k2 < N2; ++k2) xch[fft4_xa<T, P, N2, STRIDED>(g, p, k2)] = v[k2];
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CP; ++c)
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) u[c][n1] = xch[fft4_xa<T, P, N2, STRIDED>(g, n1, p + P * c)];
#pragma unroll
  for (int c = 0; c < CP; ++c) reg_fft<T, P, N2 / P>(u[c], tsn, inv);
}

// The inverse of four_step straight from its output layout (u[c][k1] =
// X[k2 + N2 k1], k2 = n1 + P c) back to the input layout (v[j] = x[n1 + P j]):
// x[n1 + P n2] = sum_k2 W_N2^(-n2 k2) W_N^(-n1 k2) sum_k1 X[k2 + N2 k1] W_P^(-n1 k1)
// -- outer P-point FFTs in registers, twiddle, ONE exchange, inner N2-point FFT.
template <typename T, int P, int N2, bool STRIDED>
__device__ __forceinline__ void four_step_inv_out(cpx<T> (&u)[N2 / P][P], cpx<T> (&v)[N2],
                                                  const cpx<T>* tsn, const cpx<T>* __restrict__ tw,
                                                  cpx<T>* xch, int g, int p) {
  constexpr int N = N2 * P, CP = N2 / P;
#pragma unroll
  for (int c = 0; c < CP; ++c) {
    reg_fft<T, P, N2 / P>(u[c], tsn, true);  // u[c][n1] = sum_k1 X[k2 + N2 k1] W_P^(-n1 k1)
#pragma unroll
    for (int n1 = 1; n1 < P; ++n1) {
      cpx<T> w = tw[(n1 * (p + P * c)) % N];
      w.im = -w.im;
      u[c][n1] = cmulc(u[c][n1], w);
    }
  }
#pragma unroll
  for (int c = 0; c < CP; ++c)
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) xch[fft4_xa<T, P, N2, STRIDED>(g, n1, p + P * c)] = u[c][n1];
  __syncthreads();
#pragma unroll
  for (int k2 = 0; k2 < N2; ++k2) v[k2] = xch[fft4_xa<T, P, N2, STRIDED>(g, p, k2)];
  reg_fft<T, N2>(v, tsn, true);
}

template <typename T, int P, int N2, bool STRIDED>
__device__ __forceinline__ void four_step(cpx<T> (&v)[N2], cpx<T> (&u)[N2 / P][P],
                                          const cpx<T>* tsn, const cpx<T>* __restrict__ tw,
                                          cpx<T>* xch, int g, int p, bool inv) {
  four_step_tw<T, P, N2, STRIDED, 1>(v, u, tsn, tw, xch, g, p, inv);
}

template <typename T, int P, int N2, bool STRIDED, int MINB>
__global__ void __launch_bounds__(256, MINB) k_fft4(cpx<T>* __restrict__ data, int64_t st,
                                                    int64_t hi, const cpx<T>* __restrict__ tw,
                                                    int inverse, SolveSpec ss,
                                                    const double* __restrict__ lam) {
  constexpr int N = N2 * P, G = 256 / P, CP = N2 / P;
  static_assert(P <= N2, "four-step split");
  static_assert(STRIDED ? P <= 8 : P >= 8, "layout / coalescing constraint");
  extern __shared__ __align__(16) unsigned char fft4_smem[];
  cpx<T>* tsn = reinterpret_cast<cpx<T>*>(fft4_smem);
  cpx<T>* xch = tsn + N2;
  __shared__ double den[G];
  const int tid = threadIdx.x;
  const int p = STRIDED ? tid / G : tid % P;
  const int g = STRIDED ? tid % G : tid / P;
  for (int k = tid; k < N2; k += 256) tsn[k] = tw[k * P];  // W_N2^k = W_N^(P k)
  const int64_t nlines = STRIDED ? st * hi : hi;
  const int64_t ntiles = (nlines + G - 1) / G;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t line = tile * G + g;
    const bool ok = line < nlines;
    int64_t base, es, lo = 0;
    if (STRIDED) {
      int64_t h;
      divmod_fast(line, st, h, lo);
      base = lo + st * (int64_t)N * h;
      es = st;
    } else {
      base = line * (int64_t)N;
      es = 1;
    }
    __syncthreads();  // table ready / previous tile's exchange reads done
    cpx<T> v[N2];
#pragma unroll
    for (int j = 0; j < N2; ++j)
      v[j] = ok ? data[base + es * (p + P * j)] : cpx<T>{T(0), T(0)};
    cpx<T> u[CP][P];
    if (!ss.active) {
      four_step<T, P, N2, STRIDED>(v, u, tsn, tw, xch, g, p, inverse != 0);
    } else {
      if (p == 0) {
        double dsum = 1.0;
        int64_t rem = ss.lo_base + lo;
        for (int a = 0; a < ss.d - 1; ++a) {
          int64_t j;
          divmod_fast(rem, ss.dims[a], rem, j);
          if (ss.lam_off[a] >= 0) dsum += lam[ss.lam_off[a] + j];
        }
        den[g] = dsum;
      }
      four_step<T, P, N2, STRIDED>(v, u, tsn, tw, xch, g, p, false);
      // X[k2 + N2 k1], k2 = p + P c: divide, then the inverse from this layout
      __syncthreads();  // exchange reads done before it is rewritten; den ready
      const double dl = den[g];
      const int lo_off = ss.lam_off[ss.d - 1];
#pragma unroll
      for (int c = 0; c < CP; ++c)
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) {
          const int k = p + P * c + N2 * k1;
          const T sc = (T)(1.0 / (dl + (lo_off >= 0 ? lam[lo_off + k] : 0.0)));
          u[c][k1] = cpx<T>{u[c][k1].re * sc, u[c][k1].im * sc};
        }
      four_step_inv_out<T, P, N2, STRIDED>(u, v, tsn, tw, xch, g, p);
      if (ok) {
#pragma unroll
        for (int j = 0; j < N2; ++j) data[base + es * (p + P * j)] = v[j];
      }
      continue;
    }
    if (ok) {
#pragma unroll
      for (int c = 0; c < CP; ++c)
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) data[base + es * (p + P * c + N2 * k1)] = u[c][k1];
    }
  }
}

// Axis-0 real passes of the solve with the four-step core: a real line of
// n0 = 2N points is the complex line z[j] = x[2j] + i x[2j+1] of N = P N2
// points.
//   R2C: Z = FFT_N(z), then X[k] = E + w^k O, X[N-k] = conj(E - w^k O) with
//        E = (Z[k] + conj Z[N-k]) / 2, O = -i (Z[k] - conj Z[N-k]) / 2, w the
//        n0-point root; the N + 1 bins go to the half spectrum in the swapped
//        layout: bin k of line (i1, rest) at i1 + tr_n1 (k + (N+1) rest).
//   C2R: the inverse (Z[k] = E + i O from the bin pairs, inverse FFT_N, the
//        real line scaled by out_scale).
// G = 256 / P lines per CTA (consecutive i1), so every bin of the half
// spectrum is read / written as G consecutive complex values.
template <typename T, int P, int N2, int MINB>
__global__ void __launch_bounds__(256, MINB) k_fft4_real(const void* in, void* out, int mode,
                                                         double out_scale, int64_t lines,
                                                         int64_t tr_n1,
                                                         const cpx<T>* __restrict__ tw) {
  // natural-order staging stride NB = N + 1 = 1 mod 16 complex: the G lines of
  // one bin fall in distinct banks
  constexpr int N = P * N2, G = 256 / P, CP = N2 / P, NB = N + 1, LS = NB;
  static_assert(G * LS <= 256 * (N2 + 1), "staging fits the exchange buffer");
  extern __shared__ __align__(16) unsigned char fft4_smem[];
  cpx<T>* tsn = reinterpret_cast<cpx<T>*>(fft4_smem);
  cpx<T>* xch = tsn + N2;
  const int tid = threadIdx.x;
  const int p = tid % P, g = tid / P;
  for (int k = tid; k < N2; k += 256) tsn[k] = tw[2 * k * P];  // W_N2 = W_n0^(2 P)
  // the N-point table of the inner four-step: W_N^m = W_n0^(2 m)
  const int64_t ntiles = (lines + G - 1) / G;
  const T osc = (T)out_scale;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t line0 = tile * G;
    __syncthreads();
    cpx<T> v[N2];
    cpx<T> u[CP][P];
    if (mode == FFT_R2C) {
      const int64_t line = line0 + g;
      const bool ok = line < lines;
      const cpx<T>* zl = reinterpret_cast<const cpx<T>*>(in) + line * (int64_t)N;
#pragma unroll
      for (int j = 0; j < N2; ++j) v[j] = ok ? zl[p + P * j] : cpx<T>{T(0), T(0)};
      four_step_tw<T, P, N2, false, 2>(v, u, tsn, tw, xch, g, p, false);
      __syncthreads();
#pragma unroll
      for (int c = 0; c < CP; ++c)
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) xch[g * LS + p + P * c + N2 * k1] = u[c][k1];
      __syncthreads();
      // bins k = 0 .. N (pairs k, N - k): thread -> (line t % G, bin t / G + step j)
      cpx<T>* Xo = reinterpret_cast<cpx<T>*>(out);
      const int gl = tid % G;
      const int64_t ln = line0 + gl;
      if (ln < lines) {
        int64_t lq, lr;
        divmod_fast(ln, tr_n1, lq, lr);
        const int64_t lb = lr + tr_n1 * (int64_t)NB * lq;
        for (int k = tid / G; k <= N / 2; k += P) {
          const cpx<T> a = xch[gl * LS + k];
          const cpx<T> bb = cconjt(xch[gl * LS + ((N - k) & (N - 1))]);
          const cpx<T> E = {(a.re + bb.re) * T(0.5), (a.im + bb.im) * T(0.5)};
          const cpx<T> D = {(a.re - bb.re) * T(0.5), (a.im - bb.im) * T(0.5)};
          const cpx<T> O = {D.im, -D.re};
          const cpx<T> WO = cmulc(tw[k], O);
          Xo[lb + tr_n1 * k] = cadd(E, WO);
          if (k < N / 2 || k == 0) Xo[lb + tr_n1 * (N - k)] = {E.re - WO.re, WO.im - E.im};
        }
      }
    } else {
      // C2R: stage the N + 1 bins of the G lines, pair them into Z in place
      const cpx<T>* Xi = reinterpret_cast<const cpx<T>*>(in);
      const int gl = tid % G;
      const int64_t ln = line0 + gl;
      if (ln < lines) {
        int64_t lq, lr;
        divmod_fast(ln, tr_n1, lq, lr);
        const int64_t lb = lr + tr_n1 * (int64_t)NB * lq;
        constexpr int IT = (NB + P - 1) / P;
        cpx<T> st[IT];  // all loads in flight before the shared-memory stores
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          const int k = tid / G + P * it;
          if (k < NB) st[it] = Xi[lb + tr_n1 * k];
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          const int k = tid / G + P * it;
          if (k < NB) xch[gl * LS + k] = st[it];
        }
      }
      __syncthreads();
      if (ln < lines)
        for (int k = tid / G; k <= N / 2; k += P) {
          // Z[k] = E + i O, Z[N-k] = conj(E - i O) with E = (X[k] + conj X[N-k]) / 2,
          // O = conj(w^k) (X[k] - conj X[N-k]) / 2
          const cpx<T> a = xch[gl * LS + k];
          const cpx<T> bb = cconjt(xch[gl * LS + N - k]);
          const cpx<T> E = {(a.re + bb.re) * T(0.5), (a.im + bb.im) * T(0.5)};
          const cpx<T> D = {(a.re - bb.re) * T(0.5), (a.im - bb.im) * T(0.5)};
          const cpx<T> O = cmulc(D, cconjt(tw[k]));
          const cpx<T> z1 = {E.re - O.im, E.im + O.re};
          const cpx<T> z2 = {E.re + O.im, O.re - E.im};
          xch[gl * LS + k] = z1;
          if (k > 0 && k < N / 2) xch[gl * LS + N - k] = z2;
          if (k == N / 2) xch[gl * LS + k] = z1;
        }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < N2; ++j) v[j] = xch[g * LS + p + P * j];
      __syncthreads();
      four_step_tw<T, P, N2, false, 2>(v, u, tsn, tw, xch, g, p, true);
      const int64_t line = line0 + g;
      if (line < lines) {
        cpx<T>* zo = reinterpret_cast<cpx<T>*>(out) + line * (int64_t)N;
#pragma unroll
        for (int c = 0; c < CP; ++c)
#pragma unroll
          for (int k1 = 0; k1 < P; ++k1)
            zo[p + P * c + N2 * k1] = cpx<T>{u[c][k1].re * osc, u[c][k1].im * osc};
      }
    }
  }
}

// C2C pass along a short power-of-two axis (N <= 32) with lo-stride st >= 32,
// in place: one thread per line, the whole line in registers, every load and
// store a coalesced warp access (consecutive threads = consecutive lo).  No
// shared-memory tile or barrier -- the tile kernels below spend most of their
// issue slots on those for short axes.  `ss.active`: forward, divide,
// inverse (the solve along the last axis).
template <typename T, int N>
__global__ void __launch_bounds__(256) k_fft_reg(cpx<T>* __restrict__ data, int64_t st,
                                                 int64_t hi, const cpx<T>* __restrict__ tw,
                                                 int inverse, SolveSpec ss,
                                                 const double* __restrict__ lam) {
  __shared__ cpx<T> ts[N];
  __shared__ double lamk[N];
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    ts[k] = tw[k];
    lamk[k] = (ss.active && ss.lam_off[ss.d - 1] >= 0) ? lam[ss.lam_off[ss.d - 1] + k] : 0.0;
  }
  __syncthreads();
  const int64_t total = st * hi;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = e % st, h = e / st;
    cpx<T>* p = data + lo + st * (int64_t)N * h;
    cpx<T> v[N];
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = p[st * k];
    reg_fft<T, N>(v, ts, ss.active ? false : inverse != 0);
    if (ss.active) {
      double den = 1.0;
      int64_t rem = ss.lo_base + lo;
      for (int a = 0; a < ss.d - 1; ++a) {
        const int64_t j = rem % ss.dims[a];
        rem /= ss.dims[a];
        if (ss.lam_off[a] >= 0) den += lam[ss.lam_off[a] + j];
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const T inv = (T)(1.0 / (den + lamk[k]));
        v[k].re *= inv;
        v[k].im *= inv;
      }
      reg_fft<T, N>(v, ts, true);
    }
#pragma unroll
    for (int k = 0; k < N; ++k) p[st * k] = v[k];
  }
}

// Stockham radix-4/2 FFT of the L lines in smem (element (l, k) at l*ls + k*ks),
// in place: every stage reads all groups into registers, syncs, writes.
// twiddles: ts[m] = exp(-2 pi i m / n) for m < n (smem); inverse conjugates.
template <typename T, int GMAX>
__device__ void stockham_lines(cpx<T>* buf, int L, int n, int64_t ls, int64_t ks,
                               const cpx<T>* ts, bool inverse, bool lo_major) {
  int Ns = 1;
  while (Ns < n) {
    const int R = (n / Ns) % 4 == 0 ? 4 : 2;
    const int groups = n / R;
    const int total = L * groups;
    cpx<T> v[GMAX][4];
    int cnt = 0;
    // load phase
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      const int e = threadIdx.x + g * blockDim.x;
      if (e < total) {
        const int l = lo_major ? e % L : e / groups;
        const int j = lo_major ? e / L : e % groups;
        const int jm = j % Ns;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r < R) {
            cpx<T> x = buf[l * ls + (int64_t)(j + r * groups) * ks];
            if (r > 0 && jm > 0) {
              cpx<T> w = ts[(jm * r * (n / (Ns * R))) % n];
              if (inverse) w.im = -w.im;
              x = cmulc(x, w);
            }
            v[g][r] = x;
          }
        }
        cnt = g + 1;
      }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      if (g < cnt) {
        const int e = threadIdx.x + g * blockDim.x;
        const int l = lo_major ? e % L : e / groups;
        const int j = lo_major ? e / L : e % groups;
        const int jm = j % Ns;
        const int64_t base = (int64_t)((j / Ns) * Ns * R + jm);
        if (R == 4) {
          const cpx<T> a0 = cadd(v[g][0], v[g][2]), a1 = csub(v[g][0], v[g][2]);
          const cpx<T> a2 = cadd(v[g][1], v[g][3]);
          const cpx<T> d = csub(v[g][1], v[g][3]);
          // forward: a3 = -i d ; inverse: +i d
          const cpx<T> a3 = inverse ? cpx<T>{-d.im, d.re} : cpx<T>{d.im, -d.re};
          buf[l * ls + (base + 0 * Ns) * ks] = cadd(a0, a2);
          buf[l * ls + (base + 1 * Ns) * ks] = cadd(a1, a3);
          buf[l * ls + (base + 2 * Ns) * ks] = csub(a0, a2);
          buf[l * ls + (base + 3 * Ns) * ks] = csub(a1, a3);
        } else {
          buf[l * ls + (base + 0 * Ns) * ks] = cadd(v[g][0], v[g][1]);
          buf[l * ls + (base + 1 * Ns) * ks] = csub(v[g][0], v[g][1]);
        }
      }
    }
    __syncthreads();
    Ns *= R;
  }
}

// Shift/mask version of stockham_lines for power-of-two L and n (lL = log2 L,
// ln = log2 n) with 32-bit shared-memory indices: no integer division in the
// butterfly loops.  Layout: lo_major -> element (l, k) at (k << lL) + l,
// otherwise (l << ln) + k.
// Per-stage twiddle tables for the radix-4/2 Stockham sequence of an n-point
// transform: stage (Ns, R) holds w^{jm r n/(Ns R)} at jm*(R-1) + r-1, so a
// warp's twiddle reads are consecutive (stride R-1) instead of all hitting one
// bank.  Total size < n.  `full` = exp(-2 pi i m / n) table (global).
template <typename T>
__device__ void build_stage_twiddles(cpx<T>* st_tab, int ln, const cpx<T>* full, int full_step) {
  int lNs = 0, off = 0;
  while (lNs < ln) {
    const int lR = (ln - lNs) >= 2 ? 2 : 1;
    const int R = 1 << lR, Ns = 1 << lNs;
    const int tws = ln - lNs - lR;
    for (int e = threadIdx.x; e < Ns * (R - 1); e += blockDim.x) {
      const int jm = e / (R - 1), r = e % (R - 1) + 1;
      st_tab[off + e] = full[((jm * r) << tws) * full_step];
    }
    off += Ns * (R - 1);
    lNs += lR;
  }
}

template <typename T, int GMAX>
__device__ void stockham_p2(cpx<T>* buf, int lL, int ln, const cpx<T>* st_tab, bool inverse,
                            bool lo_major) {
  const int n = 1 << ln;
  int lNs = 0, toff = 0;
  while (lNs < ln) {
    const int lR = (ln - lNs) >= 2 ? 2 : 1;
    const int lg = ln - lR;  // log2(groups)
    const int total = 1 << (lL + lg);
    const int rm1 = (1 << lR) - 1;
    const int nsm = (1 << lNs) - 1;
    cpx<T> v[GMAX][4];
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      const int e = threadIdx.x + g * blockDim.x;
      if (e < total) {
        const int l = lo_major ? (e & ((1 << lL) - 1)) : (e >> lg);
        const int j = lo_major ? (e >> lL) : (e & ((1 << lg) - 1));
        const int jm = j & nsm;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r < (1 << lR)) {
            const int k = j + (r << lg);
            cpx<T> x = buf[lo_major ? (k << lL) + l : (l << ln) + k];
            if (r > 0 && jm > 0) {
              cpx<T> w = st_tab[toff + jm * rm1 + r - 1];
              if (inverse) w.im = -w.im;
              x = cmulc(x, w);
            }
            v[g][r] = x;
          }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      const int e = threadIdx.x + g * blockDim.x;
      if (e < total) {
        const int l = lo_major ? (e & ((1 << lL) - 1)) : (e >> lg);
        const int j = lo_major ? (e >> lL) : (e & ((1 << lg) - 1));
        const int base = ((j >> lNs) << (lNs + lR)) + (j & nsm);
        auto at = [&](int r) -> cpx<T>& {
          const int k = base + (r << lNs);
          return buf[lo_major ? (k << lL) + l : (l << ln) + k];
        };
        if (lR == 2) {
          const cpx<T> a0 = cadd(v[g][0], v[g][2]), a1 = csub(v[g][0], v[g][2]);
          const cpx<T> a2 = cadd(v[g][1], v[g][3]);
          const cpx<T> d = csub(v[g][1], v[g][3]);
          const cpx<T> a3 = inverse ? cpx<T>{-d.im, d.re} : cpx<T>{d.im, -d.re};
          at(0) = cadd(a0, a2);
          at(1) = cadd(a1, a3);
          at(2) = csub(a0, a2);
          at(3) = csub(a1, a3);
        } else {
          at(0) = cadd(v[g][0], v[g][1]);
          at(1) = csub(v[g][0], v[g][1]);
        }
      }
    }
    __syncthreads();
    toff += (1 << lNs) * rm1;
    lNs += lR;
  }
  (void)n;
}

// direct DFT of the lines (non power-of-two n), result back into buf via tmp
template <typename T>
__device__ void direct_lines(cpx<T>* buf, cpx<T>* tmp, int L, int n, int64_t ls, int64_t ks,
                             const cpx<T>* ts, bool inverse) {
  for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
    const int l = e / n, k = e % n;
    cpx<T> acc = {T(0), T(0)};
    int idx = 0;
    for (int j = 0; j < n; ++j) {
      cpx<T> w = ts[idx];
      if (inverse) w.im = -w.im;
      acc = cadd(acc, cmulc(w, buf[l * ls + (int64_t)j * ks]));
      idx += k;
      if (idx >= n) idx -= n;
    }
    tmp[l * ls + (int64_t)k * ks] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
    const int l = e / n, k = e % n;
    buf[l * ls + (int64_t)k * ks] = tmp[l * ls + (int64_t)k * ks];
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ void lines_fft(cpx<T>* buf, cpx<T>* tmp, int L, int n, int64_t ls,
                                          int64_t ks, const cpx<T>* ts, bool inverse,
                                          bool lo_major) {
  if (n == 1) return;
  if ((n & (n - 1)) == 0) {
    // host guarantees L * n <= 16 * blockDim.x, i.e. <= 8 radix-2 groups per thread
    stockham_lines<T, 8>(buf, L, n, ls, ks, ts, inverse, lo_major);
  } else {
    direct_lines<T>(buf, tmp, L, n, ls, ks, ts, inverse);
  }
}

// Pass modes


// One pass along an axis.
//  C2C: complex in/out, axis length n (lo-stride st, hi lines).
//  R2C (axis 0 only, n = n0 even, hn = n/2): real input lines of n, complex
//       output lines of hn+1 (half spectrum, contiguous).
//  C2R (axis 0 only): inverse of R2C, real output times out_scale.
// `ss.active` (C2C on the last axis): forward, divide, inverse.
template <typename T>
__global__ void __launch_bounds__(256) k_fft_axis(const void* in, void* out,  // may alias (in-place passes)
                                                  int mode, double out_scale, int64_t st, int n,
                                                  int64_t hi, int L,
                                                  const cpx<T>* __restrict__ tw, int inverse,
                                                  SolveSpec ss, const double* __restrict__ lam) {
  extern __shared__ __align__(16) unsigned char fft_smem[];
  // the transformed length (complex) and the element counts of in/out lines
  const int nt = (mode == FFT_C2C) ? n : n / 2;
  cpx<T>* ts = reinterpret_cast<cpx<T>*>(fft_smem);                 // nt twiddles
  cpx<T>* buf = ts + nt;                                             // L x nt
  cpx<T>* tmp = buf + (size_t)L * nt;                                // L x nt (non pow2)
  for (int m = threadIdx.x; m < nt; m += blockDim.x)
    ts[m] = tw[(mode == FFT_C2C) ? m : 2 * m];  // n-point table, even entries = nt-point
  int64_t lo0, hi0;
  const bool lo_lines = st > 1;
  if (!lo_lines) {
    lo0 = 0;
    hi0 = (int64_t)blockIdx.x * L;
  } else {
    const int64_t nlob = (st + L - 1) / L;
    lo0 = (int64_t)(blockIdx.x % nlob) * L;
    hi0 = blockIdx.x / nlob;
  }
  const int64_t ls = lo_lines ? 1 : nt, ks = lo_lines ? L : 1;
  const int hn = n / 2;
  // ---- load ----
  if (mode == FFT_R2C) {
    // z[k] = x[2k] + i x[2k+1]
    for (int e = threadIdx.x; e < L * nt; e += blockDim.x) {
      const int l = e / nt, k = e % nt;
      const int64_t line = hi0 + l;
      cpx<T> v = {T(0), T(0)};
      if (line < hi) {
        const T* x = reinterpret_cast<const T*>(in) + line * n;
        v = {x[2 * k], x[2 * k + 1]};
      }
      buf[l * ls + k * ks] = v;
    }
  } else if (mode == FFT_C2R) {
    // Z[k] = E[k] + i O[k],  E = (X[k] + conj X[h-k]) / 2,  O = w^-k (X[k] - conj X[h-k]) / 2
    for (int e = threadIdx.x; e < L * nt; e += blockDim.x) {
      const int l = e / nt, k = e % nt;
      const int64_t line = hi0 + l;
      cpx<T> v = {T(0), T(0)};
      if (line < hi) {
        const cpx<T>* X = reinterpret_cast<const cpx<T>*>(in) + line * (hn + 1);
        const cpx<T> a = X[k], b = cconjt(X[hn - k]);
        const cpx<T> E = {(a.re + b.re) * T(0.5), (a.im + b.im) * T(0.5)};
        cpx<T> w = tw[k];  // n-point twiddle e^{-2 pi i k / n}; need w^{-k} = conj
        w.im = -w.im;
        const cpx<T> D = {(a.re - b.re) * T(0.5), (a.im - b.im) * T(0.5)};
        const cpx<T> O = cmulc(D, w);
        v = {E.re - O.im, E.im + O.re};  // E + i O
      }
      buf[l * ls + k * ks] = v;
    }
  } else {
    for (int e = threadIdx.x; e < L * nt; e += blockDim.x) {
      int l, k;
      if (lo_lines) { l = e % L; k = e / L; } else { l = e / nt; k = e % nt; }
      const int64_t lo = lo_lines ? lo0 + l : 0;
      const int64_t hh = lo_lines ? hi0 : hi0 + l;
      cpx<T> v = {T(0), T(0)};
      if (lo < st && hh < hi) v = reinterpret_cast<const cpx<T>*>(in)[lo + st * (k + (int64_t)n * hh)];
      buf[l * ls + k * ks] = v;
    }
  }
  __syncthreads();
  lines_fft<T>(buf, tmp, L, nt, ls, ks, ts, (mode == FFT_C2R) || inverse != 0, lo_lines);
  if (ss.active) {
    for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
      int l, k;
      if (lo_lines) { l = e % L; k = e / L; } else { l = e / n; k = e % n; }
      const int64_t lo = lo_lines ? lo0 + l : 0;
      double den = 1.0;
      int64_t rem = ss.lo_base + lo;
      for (int a = 0; a < ss.d - 1; ++a) {
        const int64_t j = rem % ss.dims[a];
        rem /= ss.dims[a];
        if (ss.lam_off[a] >= 0) den += lam[ss.lam_off[a] + j];
      }
      if (ss.lam_off[ss.d - 1] >= 0) den += lam[ss.lam_off[ss.d - 1] + k];
      const T inv = (T)(1.0 / den);
      const cpx<T> v = buf[l * ls + k * ks];
      buf[l * ls + k * ks] = {v.re * inv, v.im * inv};
    }
    __syncthreads();
    lines_fft<T>(buf, tmp, L, n, ls, ks, ts, true, lo_lines);
  }
  // ---- store ----
  if (mode == FFT_R2C) {
    // X[k] = E[k] + w^k O[k], k = 0..h, with E = (Z[k] + conj Z[h-k]) / 2,
    // O = -i (Z[k] - conj Z[h-k]) / 2, Z[h] = Z[0]
    for (int e = threadIdx.x; e < L * (hn + 1); e += blockDim.x) {
      const int l = e / (hn + 1), k = e % (hn + 1);
      const int64_t line = hi0 + l;
      if (line >= hi) continue;
      const cpx<T> a = buf[l * ls + (k % nt) * ks];
      const cpx<T> b = cconjt(buf[l * ls + ((nt - k) % nt) * ks]);
      const cpx<T> E = {(a.re + b.re) * T(0.5), (a.im + b.im) * T(0.5)};
      const cpx<T> D = {(a.re - b.re) * T(0.5), (a.im - b.im) * T(0.5)};
      const cpx<T> O = {D.im, -D.re};  // -i D
      const cpx<T> wO = cmulc(tw[k % n], O);
      reinterpret_cast<cpx<T>*>(out)[line * (hn + 1) + k] = cadd(E, wO);
    }
  } else if (mode == FFT_C2R) {
    for (int e = threadIdx.x; e < L * nt; e += blockDim.x) {
      const int l = e / nt, k = e % nt;
      const int64_t line = hi0 + l;
      if (line >= hi) continue;
      const cpx<T> v = buf[l * ls + k * ks];
      T* x = reinterpret_cast<T*>(out) + line * n;
      x[2 * k] = (T)(v.re * out_scale);
      x[2 * k + 1] = (T)(v.im * out_scale);
    }
  } else {
    for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
      int l, k;
      if (lo_lines) { l = e % L; k = e / L; } else { l = e / n; k = e % n; }
      const int64_t lo = lo_lines ? lo0 + l : 0;
      const int64_t hh = lo_lines ? hi0 : hi0 + l;
      if (lo < st && hh < hi) {
        const cpx<T> v = buf[l * ls + k * ks];
        if (out_scale != 1.0) {
          reinterpret_cast<cpx<T>*>(out)[lo + st * (k + (int64_t)n * hh)] =
              {(T)(v.re * out_scale), (T)(v.im * out_scale)};
        } else {
          reinterpret_cast<cpx<T>*>(out)[lo + st * (k + (int64_t)n * hh)] = v;
        }
      }
    }
  }
}

// Persistent, double-buffered variant for power-of-two transform lengths:
// while tile t is transformed in one buffer, tile t+1 streams into the other
// (cp.async), so HBM stays busy through the butterflies.  Same modes and
// semantics as k_fft_axis.  Tile = L lines; `ntiles` tiles in total.
template <typename T>
__global__ void __launch_bounds__(256) k_fft_axis_p(const void* in, void* out,  // may alias (in-place passes)
                                                    int mode, double out_scale, int64_t st, int n,
                                                    int64_t hi, int L, int64_t ntiles,
                                                    const cpx<T>* __restrict__ tw, int inverse,
                                                    SolveSpec ss, const double* __restrict__ lam) {
  extern __shared__ __align__(16) unsigned char fft_smem[];
  const int nt = (mode == FFT_C2C) ? n : n / 2;
  const int hn = n / 2;
  const int bufc = L * (nt + 1);  // complex slots per buffer (C2R stages hn+1 per line)
  cpx<T>* ts = reinterpret_cast<cpx<T>*>(fft_smem);
  cpx<T>* bufs[2] = {ts + nt, ts + nt + bufc};
  for (int m = threadIdx.x; m < nt; m += blockDim.x) ts[m] = tw[(mode == FFT_C2C) ? m : 2 * m];
  const bool lo_lines = st > 1;
  const int64_t nlob = lo_lines ? (st + L - 1) / L : 1;
  const int64_t ls = lo_lines ? 1 : nt, ks = lo_lines ? L : 1;
  auto tile_origin = [&](int64_t t, int64_t& lo0, int64_t& hi0) {
    if (!lo_lines) {
      lo0 = 0;
      hi0 = t * L;
    } else {
      lo0 = (t % nlob) * L;
      hi0 = t / nlob;
    }
  };
  // async copy of tile t's input into buffer b
  auto load = [&](int64_t t, int b) {
    if (t < ntiles) {
      int64_t lo0, hi0;
      tile_origin(t, lo0, hi0);
      cpx<T>* buf = bufs[b];
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf);
      if (mode == FFT_R2C) {
        // L contiguous real lines of n = L * nt complex-sized slots, verbatim
        const int64_t lines = (hi - hi0) < L ? (hi - hi0) : L;
        const T* src = reinterpret_cast<const T*>(in) + hi0 * n;
        const int64_t bytes = lines * n * (int64_t)sizeof(T);
        for (int64_t o = threadIdx.x * 16; o < bytes; o += blockDim.x * 16)
          cpa16(sb + (uint32_t)o, reinterpret_cast<const unsigned char*>(src) + o);
      } else if (mode == FFT_C2R) {
        // L contiguous lines of hn+1 complex, staged as [l][hn+1]
        const int64_t lines = (hi - hi0) < L ? (hi - hi0) : L;
        const cpx<T>* src = reinterpret_cast<const cpx<T>*>(in) + hi0 * (hn + 1);
        for (int64_t e = threadIdx.x; e < lines * (hn + 1); e += blockDim.x) {
          if (sizeof(cpx<T>) == 8) cpa8(sb + (uint32_t)(e * sizeof(cpx<T>)), src + e);
          else cpa16(sb + (uint32_t)(e * sizeof(cpx<T>)), src + e);
        }
      } else {
        const cpx<T>* src = reinterpret_cast<const cpx<T>*>(in);
        for (int e = threadIdx.x; e < L * nt; e += blockDim.x) {
          int l, k;
          if (lo_lines) { l = e % L; k = e / L; } else { l = e / nt; k = e % nt; }
          const int64_t lo = lo_lines ? lo0 + l : 0;
          const int64_t hh = lo_lines ? hi0 : hi0 + l;
          if (lo < st && hh < hi) {
            const uint32_t d = sb + (uint32_t)((l * ls + k * ks) * sizeof(cpx<T>));
            const cpx<T>* s = src + lo + st * (k + (int64_t)n * hh);
            if (sizeof(cpx<T>) == 8) cpa8(d, s);
            else cpa16(d, s);
          }
        }
      }
    }
    cpa_commit();
  };
  int64_t t = blockIdx.x;
  load(t, 0);
  int b = 0;
  for (; t < ntiles; t += gridDim.x, b ^= 1) {
    load(t + gridDim.x, b ^ 1);
    cpa_wait1();
    __syncthreads();
    cpx<T>* buf = bufs[b];
    int64_t lo0, hi0;
    tile_origin(t, lo0, hi0);
    if (mode == FFT_C2R) {
      // staged X[l][0..hn] -> Z[l][k] = E + i O in place (Z needs X[k], X[hn-k])
      cpx<T> zv[8];
      int cnt = 0;
      for (int e = threadIdx.x; e < L * nt && cnt < 8; e += blockDim.x, ++cnt) {
        const int l = e / nt, k = e % nt;
        const cpx<T> a = buf[l * (hn + 1) + k], bb = cconjt(buf[l * (hn + 1) + hn - k]);
        const cpx<T> E = {(a.re + bb.re) * T(0.5), (a.im + bb.im) * T(0.5)};
        cpx<T> w = tw[k];
        w.im = -w.im;
        const cpx<T> D = {(a.re - bb.re) * T(0.5), (a.im - bb.im) * T(0.5)};
        const cpx<T> O = cmulc(D, w);
        zv[cnt] = {E.re - O.im, E.im + O.re};
      }
      __syncthreads();
      cnt = 0;
      for (int e = threadIdx.x; e < L * nt && cnt < 8; e += blockDim.x, ++cnt) buf[e] = zv[cnt];
      __syncthreads();
    }
    stockham_lines<T, 4>(buf, L, nt, ls, ks, ts, (mode == FFT_C2R) || inverse != 0, lo_lines);
    if (ss.active) {
      for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
        int l, k;
        if (lo_lines) { l = e % L; k = e / L; } else { l = e / n; k = e % n; }
        const int64_t lo = lo_lines ? lo0 + l : 0;
        double den = 1.0;
        int64_t rem = ss.lo_base + lo;
        for (int a = 0; a < ss.d - 1; ++a) {
          const int64_t j = rem % ss.dims[a];
          rem /= ss.dims[a];
          if (ss.lam_off[a] >= 0) den += lam[ss.lam_off[a] + j];
        }
        if (ss.lam_off[ss.d - 1] >= 0) den += lam[ss.lam_off[ss.d - 1] + k];
        const T inv = (T)(1.0 / den);
        const cpx<T> v = buf[l * ls + k * ks];
        buf[l * ls + k * ks] = {v.re * inv, v.im * inv};
      }
      __syncthreads();
      stockham_lines<T, 4>(buf, L, n, ls, ks, ts, true, lo_lines);
    }
    // ---- store ----
    if (mode == FFT_R2C) {
      for (int e = threadIdx.x; e < L * (hn + 1); e += blockDim.x) {
        const int l = e / (hn + 1), k = e % (hn + 1);
        const int64_t line = hi0 + l;
        if (line >= hi) continue;
        const cpx<T> a = buf[l * ls + (k % nt) * ks];
        const cpx<T> bb = cconjt(buf[l * ls + ((nt - k) % nt) * ks]);
        const cpx<T> E = {(a.re + bb.re) * T(0.5), (a.im + bb.im) * T(0.5)};
        const cpx<T> D = {(a.re - bb.re) * T(0.5), (a.im - bb.im) * T(0.5)};
        const cpx<T> O = {D.im, -D.re};
        const cpx<T> wO = cmulc(tw[k % n], O);
        reinterpret_cast<cpx<T>*>(out)[line * (hn + 1) + k] = cadd(E, wO);
      }
    } else if (mode == FFT_C2R) {
      for (int e = threadIdx.x; e < L * nt; e += blockDim.x) {
        const int l = e / nt, k = e % nt;
        const int64_t line = hi0 + l;
        if (line >= hi) continue;
        const cpx<T> v = buf[l * ls + k * ks];
        T* x = reinterpret_cast<T*>(out) + line * n;
        x[2 * k] = (T)(v.re * out_scale);
        x[2 * k + 1] = (T)(v.im * out_scale);
      }
    } else {
      for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
        int l, k;
        if (lo_lines) { l = e % L; k = e / L; } else { l = e / n; k = e % n; }
        const int64_t lo = lo_lines ? lo0 + l : 0;
        const int64_t hh = lo_lines ? hi0 : hi0 + l;
        if (lo < st && hh < hi) {
          cpx<T> v = buf[l * ls + k * ks];
          if (out_scale != 1.0) v = {(T)(v.re * out_scale), (T)(v.im * out_scale)};
          reinterpret_cast<cpx<T>*>(out)[lo + st * (k + (int64_t)n * hh)] = v;
        }
      }
    }
    __syncthreads();  // buffer b is reloaded two iterations later
  }
}

// Power-of-two persistent pass (L, nt powers of two; host checks).  Same
// semantics as k_fft_axis; double-buffered cp.async tiles, shift indexing,
// per-line solve denominators.
// tr_n1 > 0 (R2C / C2R only): the half spectrum is stored with axes 0 and 1
// swapped, bin k of line (i1, rest) at i1 + n1 * (k + (n/2+1) * rest), so the
// axis-1 pass runs on contiguous lines.
template <typename T>
__global__ void __launch_bounds__(256) k_fft_p2(const void* in, void* out,  // may alias (in-place passes)
                                                int mode, double out_scale, int64_t st, int n,
                                                int64_t hi, int lL, int64_t ntiles,
                                                const cpx<T>* __restrict__ tw, int inverse,
                                                SolveSpec ss, const double* __restrict__ lam,
                                                int64_t tr_n1) {
  extern __shared__ __align__(16) unsigned char fft_smem[];
  const int nt = (mode == FFT_C2C) ? n : n / 2;
  int ln = 0;
  while ((1 << ln) < nt) ++ln;
  const int L = 1 << lL;
  const int hn = n / 2;
  const int bufc = L * (nt + 1);
  cpx<T>* ts = reinterpret_cast<cpx<T>*>(fft_smem);  // per-stage twiddles (< nt entries)
  cpx<T>* const buf0 = ts + nt;                       // two tile buffers of bufc slots
  __shared__ double denl[16];
  __shared__ int64_t lbase[16];  // R2C output base of each line of the tile
  build_stage_twiddles<T>(ts, ln, tw, (mode == FFT_C2C) ? 1 : 2);
  const bool lo_lines = st > 1;
  const int64_t nlob = lo_lines ? (st + L - 1) >> lL : 1;
  auto origin = [&](int64_t t, int64_t& lo0, int64_t& hi0) {
    if (!lo_lines) {
      lo0 = 0;
      hi0 = t << lL;
    } else {
      lo0 = (t % nlob) << lL;
      hi0 = t / nlob;
    }
  };
  auto sidx = [&](int l, int k) -> int { return lo_lines ? (k << lL) + l : (l << ln) + k; };
  auto load = [&](int64_t t, int b) {
    if (t < ntiles) {
      int64_t lo0, hi0;
      origin(t, lo0, hi0);
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf0 + b * bufc);
      if (mode == FFT_R2C) {
        const int64_t lines = (hi - hi0) < L ? (hi - hi0) : L;
        const unsigned char* src = reinterpret_cast<const unsigned char*>(in) + hi0 * n * (int64_t)sizeof(T);
        const int64_t bytes = lines * n * (int64_t)sizeof(T);
        for (int64_t o = threadIdx.x * 16; o < bytes; o += blockDim.x * 16) cpa16(sb + (uint32_t)o, src + o);
      } else if (mode == FFT_C2R) {
        const cpx<T>* X = reinterpret_cast<const cpx<T>*>(in);
        const int cnt = L * (hn + 1);
        if (tr_n1) {
          // swapped layout: this thread always serves line l = tid mod L
          const int l = threadIdx.x & (L - 1);
          const int64_t line = hi0 + l;
          if (line < hi) {
            const int64_t gb = (line % tr_n1) + tr_n1 * (int64_t)(hn + 1) * (line / tr_n1);
            for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
              const int k = e >> lL;
              const uint32_t d = sb + (uint32_t)((l * (hn + 1) + k) * (int)sizeof(cpx<T>));
              if (sizeof(cpx<T>) == 8) cpa8(d, X + gb + tr_n1 * k);
              else cpa16(d, X + gb + tr_n1 * k);
            }
          }
        } else {
          for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
            const int l = e / (hn + 1), k = e % (hn + 1);
            if (hi0 + l >= hi) continue;
            const uint32_t d = sb + (uint32_t)(e * (int)sizeof(cpx<T>));
            if (sizeof(cpx<T>) == 8) cpa8(d, X + (hi0 + l) * (hn + 1) + k);
            else cpa16(d, X + (hi0 + l) * (hn + 1) + k);
          }
        }
      } else {
        const cpx<T>* src = reinterpret_cast<const cpx<T>*>(in);
        const int tot = L << ln;
        for (int e = threadIdx.x; e < tot; e += blockDim.x) {
          const int l = lo_lines ? (e & (L - 1)) : (e >> ln);
          const int k = lo_lines ? (e >> lL) : (e & (nt - 1));
          const int64_t lo = lo_lines ? lo0 + l : 0;
          const int64_t hh = lo_lines ? hi0 : hi0 + l;
          if (lo < st && hh < hi) {
            const uint32_t d = sb + (uint32_t)(sidx(l, k) * (int)sizeof(cpx<T>));
            const cpx<T>* s = src + lo + st * (k + (int64_t)n * hh);
            if (sizeof(cpx<T>) == 8) cpa8(d, s);
            else cpa16(d, s);
          }
        }
      }
    }
    cpa_commit();
  };
  int64_t t = blockIdx.x;
  load(t, 0);
  int b = 0;
  for (; t < ntiles; t += gridDim.x, b ^= 1) {
    load(t + gridDim.x, b ^ 1);
    cpa_wait1();
    int64_t lo0, hi0;
    origin(t, lo0, hi0);
    if (ss.active && threadIdx.x < L) {
      // per-line part of the denominator: axes 0..d-2 from the line's lo index
      double den = 1.0;
      int64_t rem = ss.lo_base + lo0 + threadIdx.x;
      for (int a = 0; a < ss.d - 1; ++a) {
        const int64_t j = rem % ss.dims[a];
        rem /= ss.dims[a];
        if (ss.lam_off[a] >= 0) den += lam[ss.lam_off[a] + j];
      }
      denl[threadIdx.x] = den;
    }
    if (mode == FFT_R2C && threadIdx.x < L) {
      const int64_t line = hi0 + threadIdx.x;
      lbase[threadIdx.x] = tr_n1 ? (line % tr_n1) + tr_n1 * (int64_t)(hn + 1) * (line / tr_n1)
                                 : line * (hn + 1);
    }
    __syncthreads();
    cpx<T>* buf = buf0 + b * bufc;
    if (mode == FFT_C2R) {
      // staged X[l][0..hn] -> Z[l][k] = E + i O (registers, then in place)
      cpx<T> zv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int e = threadIdx.x + c * blockDim.x;
        if (e < (L << ln)) {
          const int l = e >> ln, k = e & (nt - 1);
          const cpx<T> a = buf[l * (hn + 1) + k], bb = cconjt(buf[l * (hn + 1) + hn - k]);
          const cpx<T> E = {(a.re + bb.re) * T(0.5), (a.im + bb.im) * T(0.5)};
          cpx<T> w = tw[k];
          w.im = -w.im;
          const cpx<T> D = {(a.re - bb.re) * T(0.5), (a.im - bb.im) * T(0.5)};
          const cpx<T> O = cmulc(D, w);
          zv[c] = {E.re - O.im, E.im + O.re};
        }
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int e = threadIdx.x + c * blockDim.x;
        if (e < (L << ln)) buf[e] = zv[c];
      }
      __syncthreads();
    }
    stockham_p2<T, 4>(buf, lL, ln, ts, (mode == FFT_C2R) || inverse != 0, lo_lines);
    if (ss.active) {
      const int tot = L << ln;
      const int lo_off = ss.lam_off[ss.d - 1];
      for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int l = lo_lines ? (e & (L - 1)) : (e >> ln);
        const int k = lo_lines ? (e >> lL) : (e & (nt - 1));
        const double den = denl[l] + (lo_off >= 0 ? lam[lo_off + k] : 0.0);
        const T inv = (T)(1.0 / den);
        const cpx<T> v = buf[e];
        buf[e] = {v.re * inv, v.im * inv};
      }
      __syncthreads();
      stockham_p2<T, 4>(buf, lL, ln, ts, true, lo_lines);
    }
    // ---- store ----
    if (mode == FFT_R2C) {
      // element e -> (l, k); with the swapped layout l runs fastest so the L
      // lines' bin k land in one contiguous segment
      cpx<T>* Xo = reinterpret_cast<cpx<T>*>(out);
      const int cnt = L * (hn + 1);
      const int64_t kst = tr_n1 ? tr_n1 : 1;
      for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
        const int l = tr_n1 ? (e & (L - 1)) : e / (hn + 1);
        const int k = tr_n1 ? (e >> lL) : e % (hn + 1);
        if (hi0 + l >= hi) continue;
        const cpx<T> a = buf[(l << ln) + (k & (nt - 1))];
        const cpx<T> bb = cconjt(buf[(l << ln) + ((nt - k) & (nt - 1))]);
        const cpx<T> E = {(a.re + bb.re) * T(0.5), (a.im + bb.im) * T(0.5)};
        const cpx<T> D = {(a.re - bb.re) * T(0.5), (a.im - bb.im) * T(0.5)};
        const cpx<T> O = {D.im, -D.re};
        Xo[lbase[l] + kst * k] = cadd(E, cmulc(tw[k], O));
      }
    } else if (mode == FFT_C2R) {
      const int tot = L << ln;
      for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int l = e >> ln, k = e & (nt - 1);
        const int64_t line = hi0 + l;
        if (line >= hi) continue;
        const cpx<T> v = buf[e];
        T* x = reinterpret_cast<T*>(out) + line * n;
        x[2 * k] = (T)(v.re * out_scale);
        x[2 * k + 1] = (T)(v.im * out_scale);
      }
    } else {
      const int tot = L << ln;
      for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int l = lo_lines ? (e & (L - 1)) : (e >> ln);
        const int k = lo_lines ? (e >> lL) : (e & (nt - 1));
        const int64_t lo = lo_lines ? lo0 + l : 0;
        const int64_t hh = lo_lines ? hi0 : hi0 + l;
        if (lo < st && hh < hi) {
          cpx<T> v = buf[e];
          if (out_scale != 1.0) v = {(T)(v.re * out_scale), (T)(v.im * out_scale)};
          reinterpret_cast<cpx<T>*>(out)[lo + st * (k + (int64_t)n * hh)] = v;
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Compile-time specialised pass: nt = 2^LN points, L = 2^LL lines, L*nt = 2048
// (8 points per thread of 256).  Stockham stages of radix 8 (radix 4 where
// log2 nt is not a multiple of 3: 128 = 8.4.4, 1024 = 8.8.4.4, 2048 = 8.8.8.4),
// each thread running 8/R register butterflies per stage, so a 512-point line
// takes 3 shared-memory exchanges instead of 5.  Tile slots are padded by one
// per 16 (fpad) which makes the stride-Ns Stockham writes bank-conflict free.
// Shapes, shifts, twiddle offsets are constants: the stages unroll into
// straight-line code.
// ---------------------------------------------------------------------------
template <int LN>
struct R8Plan {
  static constexpr int n4 = (LN % 3 == 0) ? 0 : ((LN % 3 == 2) ? 1 : 2);
  static constexpr int n8 = (LN - 2 * n4) / 3;
  static constexpr int NST = n8 + n4;
  __host__ __device__ static constexpr int lr(int s) { return s < n8 ? 3 : 2; }
  __host__ __device__ static constexpr int lns(int s) {
    return s <= n8 ? 3 * s : 3 * n8 + 2 * (s - n8);
  }
  __host__ __device__ static constexpr int toff(int s) {
    int o = 0;
    for (int i = 0; i < s; ++i) o += (1 << lns(i)) * ((1 << lr(i)) - 1);
    return o;
  }
};

__device__ __forceinline__ int fpad(int i) { return i + (i >> 4); }
// padded tile slots for a 2048-point tile (+ the C2R staging overhang)
constexpr int kFftTileSlots = 2048 + 2048 / 16 + 32;
// slots of the real-transform twiddle table (NT/2 + 1, rounded to 16 bytes x 2)
__host__ __device__ constexpr int kFftRtwSlots(int nt) { return (nt / 2 + 1 + 1) & ~1; }

// per-stage twiddles of the radix-8/4 plan: stage s holds w^{jm r nt/(Ns R)}
// at toff(s) + jm (R-1) + r-1
template <typename T, int LN>
__device__ void build_r8_twiddles(cpx<T>* st_tab, const cpx<T>* full, int full_step) {
  using P = R8Plan<LN>;
#pragma unroll
  for (int s = 0; s < P::NST; ++s) {
    const int lR = P::lr(s), lNs = P::lns(s), R = 1 << lR;
    const int tws = LN - lNs - lR;
    for (int e = threadIdx.x; e < ((R - 1) << lNs); e += blockDim.x) {
      const int jm = e / (R - 1), r = e % (R - 1) + 1;
      st_tab[P::toff(s) + e] = full[((jm * r) << tws) * full_step];
    }
  }
}

// y *= exp(-+ 2 pi i m / 8) for m = 1, 2, 3 (INV: conjugate)
template <typename T, bool INV, int M>
__device__ __forceinline__ cpx<T> rot8(cpx<T> a) {
  constexpr T h = (T)0.70710678118654752440;
  if (M == 1) return INV ? cpx<T>{(a.re - a.im) * h, (a.re + a.im) * h}
                         : cpx<T>{(a.re + a.im) * h, (a.im - a.re) * h};
  if (M == 2) return INV ? cpx<T>{-a.im, a.re} : cpx<T>{a.im, -a.re};
  return INV ? cpx<T>{(-a.re - a.im) * h, (a.re - a.im) * h}
             : cpx<T>{(a.im - a.re) * h, (-a.re - a.im) * h};
}

// in-register DFT4 of x[o], x[o+s], x[o+2s], x[o+3s]; output k in place of input k
template <typename T, bool INV>
__device__ __forceinline__ void dft4(cpx<T>& x0, cpx<T>& x1, cpx<T>& x2, cpx<T>& x3) {
  const cpx<T> c0 = cadd(x0, x2), c1 = csub(x0, x2), c2 = cadd(x1, x3);
  const cpx<T> c3 = rot8<T, INV, 2>(csub(x1, x3));
  x0 = cadd(c0, c2);
  x2 = csub(c0, c2);
  x1 = cadd(c1, c3);
  x3 = csub(c1, c3);
}

// in-register DFT8 (decimation in frequency: X[2k] = DFT4(a), X[2k+1] = DFT4(b))
template <typename T, bool INV>
__device__ __forceinline__ void dft8(cpx<T>* x) {
  cpx<T> a0 = cadd(x[0], x[4]), a1 = cadd(x[1], x[5]), a2 = cadd(x[2], x[6]), a3 = cadd(x[3], x[7]);
  cpx<T> b0 = csub(x[0], x[4]);
  cpx<T> b1 = rot8<T, INV, 1>(csub(x[1], x[5]));
  cpx<T> b2 = rot8<T, INV, 2>(csub(x[2], x[6]));
  cpx<T> b3 = rot8<T, INV, 3>(csub(x[3], x[7]));
  dft4<T, INV>(a0, a1, a2, a3);
  dft4<T, INV>(b0, b1, b2, b3);
  x[0] = a0; x[2] = a1; x[4] = a2; x[6] = a3;
  x[1] = b0; x[3] = b1; x[5] = b2; x[7] = b3;
}

template <typename T, int LN, int LL, bool INV>
__device__ __forceinline__ void stockham8(cpx<T>* buf, const cpx<T>* st_tab, bool lo_major) {
  using P = R8Plan<LN>;
#pragma unroll
  for (int s = 0; s < P::NST; ++s) {
    const int lR = P::lr(s), lNs = P::lns(s), R = 1 << lR;
    const int lg = LN - lR;  // log2 butterflies per line
    const int nsm = (1 << lNs) - 1;
    const int NB = 8 / R;    // butterflies per thread
    cpx<T> v[8];
#pragma unroll
    for (int g = 0; g < NB; ++g) {
      const int e = threadIdx.x + g * 256;
      const int l = lo_major ? (e & ((1 << LL) - 1)) : (e >> lg);
      const int b = lo_major ? (e >> LL) : (e & ((1 << lg) - 1));
      const int jm = b & nsm;
      // read offsets r * 2^lg (x 2^LL when lo-major) are multiples of 16: the
      // padded slot of element r is p0 + r * (step + step / 16)
      const int p0 = fpad(lo_major ? (b << LL) + l : (l << LN) + b);
      const int rstep = lo_major ? (1 << (lg + LL)) : (1 << lg);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        cpx<T> x = buf[p0 + r * (rstep + (rstep >> 4))];
        if (r > 0 && s > 0) {
          cpx<T> w = st_tab[P::toff(s) + jm * (R - 1) + r - 1];
          if (INV) w.im = -w.im;
          x = cmulc(x, w);
        }
        v[g * R + r] = x;
      }
      if (R == 8) dft8<T, INV>(v);
      else dft4<T, INV>(v[g * 4 + 0], v[g * 4 + 1], v[g * 4 + 2], v[g * 4 + 3]);
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < NB; ++g) {
      const int e = threadIdx.x + g * 256;
      const int l = lo_major ? (e & ((1 << LL) - 1)) : (e >> lg);
      const int b = lo_major ? (e >> LL) : (e & ((1 << lg) - 1));
      const int base = ((b >> lNs) << (lNs + lR)) + (b & nsm);
      const int i0 = lo_major ? (base << LL) + l : (l << LN) + base;
      const int wstep = lo_major ? (1 << (lNs + LL)) : (1 << lNs);
      if ((wstep & 15) == 0) {
        const int q0 = fpad(i0);
#pragma unroll
        for (int r = 0; r < R; ++r) buf[q0 + r * (wstep + (wstep >> 4))] = v[g * R + r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) buf[fpad(i0 + r * wstep)] = v[g * R + r];
      }
    }
    __syncthreads();
  }
}

template <typename T, int LN, int LL>
__global__ void __launch_bounds__(256, 3) k_fft_t(const void* in, void* out,  // may alias
                                               int mode, double out_scale, int64_t st, int n,
                                               int64_t hi, int64_t ntiles,
                                               const cpx<T>* __restrict__ tw, int inverse,
                                               SolveSpec ss, const double* __restrict__ lam,
                                               int64_t tr_n1) {
  constexpr int NT = 1 << LN, L = 1 << LL, TOT = NT * L, PER = TOT / 256;
  static_assert(TOT == 2048, "tile must hold 2048 points");
  extern __shared__ __align__(16) unsigned char fft_smem[];
  const int hn = n / 2;
  constexpr int bufc = kFftTileSlots;
  constexpr int NP = NT / 2 + 1;  // bin pairs (k, NT - k) per line of a real transform
  const T osc = (T)out_scale;
  cpx<T>* ts = reinterpret_cast<cpx<T>*>(fft_smem);
  cpx<T>* const rtw = ts + NT;               // w^k, k <= NT/2, of the real transforms
  cpx<T>* const buf0 = rtw + kFftRtwSlots(NT);
  __shared__ double denl[16];
  __shared__ int64_t lbase[16];
  build_r8_twiddles<T, LN>(ts, tw, (mode == FFT_C2C) ? 1 : 2);
  if (mode != FFT_C2C)
    for (int k = threadIdx.x; k < NP; k += blockDim.x) rtw[k] = tw[k];
  const bool inv_first = (mode == FFT_C2R) || inverse != 0;
  constexpr int CS = (int)sizeof(cpx<T>);
  const bool lo_lines = st > 1;
  const int64_t nlob = lo_lines ? (st + L - 1) >> LL : 1;
  auto origin = [&](int64_t t, int64_t& lo0, int64_t& hi0) {
    if (!lo_lines) {
      lo0 = 0;
      hi0 = t << LL;
    } else {
      lo0 = (t % nlob) << LL;
      hi0 = t / nlob;
    }
  };
  const int tid = threadIdx.x;
  auto load = [&](int64_t t, int b) {
    if (t < ntiles) {
      int64_t lo0, hi0;
      origin(t, lo0, hi0);
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf0 + b * bufc);
      if (mode == FFT_R2C) {
        const int64_t lines = (hi - hi0) < L ? (hi - hi0) : L;
        const unsigned char* src =
            reinterpret_cast<const unsigned char*>(in) + hi0 * n * (int64_t)sizeof(T);
        const int64_t bytes = lines * n * (int64_t)sizeof(T);
        // one complex slot per copy: padded slots are only CS-byte aligned
        for (int m = tid; m < (int)(bytes / CS); m += 256) {
          const uint32_t d = sb + (uint32_t)(fpad(m) * CS);
          if (CS == 8) cpa8(d, src + (int64_t)m * CS);
          else cpa16(d, src + (int64_t)m * CS);
        }
      } else if (mode == FFT_C2R) {
        // swapped layout (tr_n1) or plain; thread serves line l = tid mod L
        const cpx<T>* X = reinterpret_cast<const cpx<T>*>(in);
        const int l = tid & (L - 1);
        const int64_t line = hi0 + l;
        if (line < hi) {
          const int64_t gb = tr_n1 ? (line % tr_n1) + tr_n1 * (int64_t)(hn + 1) * (line / tr_n1)
                                   : line * (hn + 1);
          const int64_t kst = tr_n1 ? tr_n1 : 1;
          for (int k = tid >> LL; k <= hn; k += 256 >> LL) {
            const uint32_t d = sb + (uint32_t)(fpad(l * (hn + 1) + k) * CS);
            if (sizeof(cpx<T>) == 8) cpa8(d, X + gb + kst * k);
            else cpa16(d, X + gb + kst * k);
          }
        }
      } else {
        const cpx<T>* src = reinterpret_cast<const cpx<T>*>(in);
        if (lo_lines) {
          // element (l, k) at lo0 + l + st (k + n hi0); thread: l = tid & (L-1), k = (tid >> LL) + u * (256 >> LL)
          const int l = tid & (L - 1);
          if (lo0 + l < st) {
            const cpx<T>* p = src + lo0 + l + st * ((int64_t)n * hi0);
#pragma unroll
            for (int u = 0; u < PER; ++u) {
              const int k = (tid >> LL) + u * (256 >> LL);
              const uint32_t d = sb + (uint32_t)(fpad((k << LL) + l) * CS);
              if (sizeof(cpx<T>) == 8) cpa8(d, p + st * k);
              else cpa16(d, p + st * k);
            }
          }
        } else {
          // L contiguous lines of NT points: one contiguous block
          const int64_t lines = (hi - hi0) < L ? (hi - hi0) : L;
          const cpx<T>* p = src + hi0 * NT;
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int e = tid + u * 256;
            if ((e >> LN) < lines) {
              const uint32_t d = sb + (uint32_t)(fpad(e) * CS);
              if (sizeof(cpx<T>) == 8) cpa8(d, p + e);
              else cpa16(d, p + e);
            }
          }
        }
      }
    }
    cpa_commit();
  };
  int64_t t = blockIdx.x;
  load(t, 0);
  int b = 0;
  for (; t < ntiles; t += gridDim.x, b ^= 1) {
    load(t + gridDim.x, b ^ 1);
    cpa_wait1();
    int64_t lo0, hi0;
    origin(t, lo0, hi0);
    if (ss.active && tid < L) {
      double den = 1.0;
      int64_t rem = ss.lo_base + lo0 + tid;
      for (int a = 0; a < ss.d - 1; ++a) {
        const int64_t j = rem % ss.dims[a];
        rem /= ss.dims[a];
        if (ss.lam_off[a] >= 0) den += lam[ss.lam_off[a] + j];
      }
      denl[tid] = den;
    }
    if (mode == FFT_R2C && tid < L) {
      const int64_t line = hi0 + tid;
      lbase[tid] = tr_n1 ? (line % tr_n1) + tr_n1 * (int64_t)(hn + 1) * (line / tr_n1)
                         : line * (hn + 1);
    }
    __syncthreads();
    cpx<T>* buf = buf0 + b * bufc;
    if (mode == FFT_C2R) {
      // pair (k, NT-k): Z[k] = E + i O, Z[NT-k] = conj(E - i O) with
      // E = (X[k] + conj X[NT-k]) / 2, O = conj(w^k) (X[k] - conj X[NT-k]) / 2
      // warp-wide runs of 32 consecutive bins of one line: the gathers at k and
      // NT - k and the line-major stores below stay free of bank conflicts
      constexpr int NKB = (NP + 31) / 32;
      constexpr int NIT = (NKB * L * 32 + 255) / 256;
      cpx<T> z1[NIT], z2[NIT];
#pragma unroll
      for (int c = 0; c < NIT; ++c) {
        const int e = tid + c * 256;
        const int q = e >> 5, l = q & (L - 1), k = ((q >> LL) << 5) + (e & 31);
        if (k < NP) {
          const cpx<T> a = buf[fpad(l * (hn + 1) + k)];
          const cpx<T> bb = cconjt(buf[fpad(l * (hn + 1) + NT - k)]);
          const cpx<T> E = {(a.re + bb.re) * T(0.5), (a.im + bb.im) * T(0.5)};
          const cpx<T> D = {(a.re - bb.re) * T(0.5), (a.im - bb.im) * T(0.5)};
          const cpx<T> O = cmulc(D, cconjt(rtw[k]));
          z1[c] = {E.re - O.im, E.im + O.re};
          z2[c] = {E.re + O.im, O.re - E.im};  // conj(E - i O)
        }
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < NIT; ++c) {
        const int e = tid + c * 256;
        const int q = e >> 5, l = q & (L - 1), k = ((q >> LL) << 5) + (e & 31);
        if (k < NP) {
          buf[fpad((l << LN) + k)] = z1[c];
          if (k > 0 && k < NT / 2) buf[fpad((l << LN) + NT - k)] = z2[c];
        }
      }
      __syncthreads();
    }
    if (inv_first) stockham8<T, LN, LL, true>(buf, ts, lo_lines);
    else stockham8<T, LN, LL, false>(buf, ts, lo_lines);
    if (ss.active) {
      const int lo_off = ss.lam_off[ss.d - 1];
#pragma unroll
      for (int c = 0; c < PER; ++c) {
        const int e = tid + c * 256;
        const int l = lo_lines ? (e & (L - 1)) : (e >> LN);
        const int k = lo_lines ? (e >> LL) : (e & (NT - 1));
        const double den = denl[l] + (lo_off >= 0 ? lam[lo_off + k] : 0.0);
        const T inv = (T)(1.0 / den);
        const cpx<T> v = buf[fpad(e)];
        buf[fpad(e)] = {v.re * inv, v.im * inv};
      }
      __syncthreads();
      stockham8<T, LN, LL, true>(buf, ts, lo_lines);
    }
    if (mode == FFT_R2C) {
      cpx<T>* Xo = reinterpret_cast<cpx<T>*>(out);
      const int64_t kst = tr_n1 ? tr_n1 : 1;
      const int l = tid & (L - 1);
      if (hi0 + l < hi) {
        // pair (k, NT-k): X[k] = E + w^k O, X[NT-k] = conj(E - w^k O) with
        // E = (Z[k] + conj Z[NT-k]) / 2, O = -i (Z[k] - conj Z[NT-k]) / 2
        cpx<T>* xl = Xo + lbase[l];
        for (int k = tid >> LL; k < NP; k += 256 >> LL) {
          const cpx<T> a = buf[fpad((l << LN) + k)];
          const cpx<T> bb = cconjt(buf[fpad((l << LN) + ((NT - k) & (NT - 1)))]);
          const cpx<T> E = {(a.re + bb.re) * T(0.5), (a.im + bb.im) * T(0.5)};
          const cpx<T> D = {(a.re - bb.re) * T(0.5), (a.im - bb.im) * T(0.5)};
          const cpx<T> O = {D.im, -D.re};
          const cpx<T> WO = cmulc(rtw[k], O);
          xl[kst * k] = cadd(E, WO);
          if (k < NT / 2) xl[kst * (NT - k)] = {E.re - WO.re, WO.im - E.im};
        }
      }
    } else if (mode == FFT_C2R) {
#pragma unroll
      for (int c = 0; c < PER; ++c) {
        const int e = tid + c * 256;
        const int l = e >> LN, k = e & (NT - 1);
        const int64_t line = hi0 + l;
        if (line < hi) {
          const cpx<T> v = buf[fpad(e)];
          reinterpret_cast<cpx<T>*>(out)[line * NT + k] = {v.re * osc, v.im * osc};  // x[2k], x[2k+1]
        }
      }
    } else if (lo_lines) {
      const int l = tid & (L - 1);
      if (lo0 + l < st) {
        cpx<T>* p = reinterpret_cast<cpx<T>*>(out) + lo0 + l + st * ((int64_t)n * hi0);
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int k = (tid >> LL) + u * (256 >> LL);
          const cpx<T> v = buf[fpad((k << LL) + l)];
          p[st * k] = {v.re * osc, v.im * osc};
        }
      }
    } else {
      const int64_t lines = (hi - hi0) < L ? (hi - hi0) : L;
      cpx<T>* p = reinterpret_cast<cpx<T>*>(out) + hi0 * NT;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int e = tid + u * 256;
        const cpx<T> v = buf[fpad(e)];
        if ((e >> LN) < lines) p[e] = {v.re * osc, v.im * osc};
      }
    }
    __syncthreads();
  }
}

// real <-> complex conversion for the full-spectrum fallback (odd n0)
template <typename T>
__global__ void k_real_to_cpx(const T* __restrict__ x, cpx<T>* __restrict__ z, int64_t N) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride)
    z[i] = {x[i], T(0)};
}
template <typename T>
__global__ void k_cpx_to_real(const cpx<T>* __restrict__ z, T* __restrict__ x, int64_t N,
                              double scale) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride)
    x[i] = (T)(z[i].re * scale);
}

// 4 sin^2(pi j / n) for j < n
__global__ void k_lap_eig(int n, double* __restrict__ lam) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double s = sinpi((double)j / (double)n);
  lam[j] = 4.0 * s * s;
}

}  // namespace tr
