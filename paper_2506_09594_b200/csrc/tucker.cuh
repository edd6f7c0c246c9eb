// Generic Tucker engine: any processing order, fixed-rank (R-STHOSVD-BKI,
// tenrec/sketch.py:211-270) or fixed-accuracy (AD-RSTHOSVD-BLBP,
// sketch.py:287-403) compression, and the Tucker-compressed t-SVT on top of
// either (sketch.py:430-456).
//
// The fixed-rank (0, 1) case -- the ADMM hot path -- keeps its fully
// asynchronous, graph-capturable launch sequence in lrta.cu.  This engine
// covers everything else and is host-driven: after each processed mode the
// discovered rank comes back to the host (one small D2H), the core is stored
// compact in its natural layout, and the next mode's unfolding is built by a
// batched transpose.  Block Lanczos needs the host anyway: its block sizes,
// deflations and stopping test are data dependent (two small D2H per
// bidiagonalisation step).
//
// Factor bases: the reference's QRs (numpy / LAPACK Householder) fix column
// signs by LAPACK's convention; every step of the bidiagonalisation is
// sign-equivariant (a column sign flip of one block propagates as sign flips
// of the next blocks, norms and deflation decisions unchanged), so the B200
// path uses its own TSQR conventions and fixes the sign of every finished
// factor column (largest-|entry| positive, k_canonical_signs) -- the same
// canonical convention the block Krylov path and the oracle use.
#pragma once

#include <vector>

#include "admm_kernels.cuh"
#include "tucker_kernels.cuh"

namespace tr {

constexpr int kTuckerMaxOrder = 10;

struct TuckerSpec {
  int mode = 0;  // 0 fixed-rank (block Krylov), 1 fixed-accuracy (block Lanczos)
  int nproc = 0;
  int proc[kTuckerMaxOrder];
  int64_t ranks[kTuckerMaxOrder], blocks[kTuckerMaxOrder], krylov[kTuckerMaxOrder];
  double eps = 0.05;
  int64_t block = 10;
  double defl_tol = 0.0;  // <= 0: 1e-10 * ||unfolding||_F per mode (sketch.py:383)
  uint64_t seed = 0;
};

// Stream-ordered device allocations released at scope exit (or handed over).
struct Arena {
  cudaStream_t st;
  std::vector<void*> ptrs;
  bool failed = false;
  explicit Arena(cudaStream_t s) : st(s) {}
  template <typename X>
  X* get(int64_t n) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, (size_t)std::max<int64_t>(n, 1) * sizeof(X), st) != cudaSuccess) {
      cudaGetLastError();
      failed = true;
      return nullptr;
    }
    ptrs.push_back(p);
    return (X*)p;
  }
  void release(void* p) {
    for (auto& q : ptrs)
      if (q == p) {
        cudaFreeAsync(q, st);
        q = nullptr;
      }
  }
  void* keep(void* p) {  // ownership moves to the caller
    for (auto& q : ptrs)
      if (q == p) q = nullptr;
    return p;
  }
  ~Arena() {
    for (void* p : ptrs)
      if (p) cudaFreeAsync(p, st);
  }
};

struct TuckerResult {
  int order = 0;
  int64_t dims[kTuckerMaxOrder] = {};
  int64_t cdims[kTuckerMaxOrder] = {};
  int64_t ranks[kTuckerMaxOrder] = {};
  bool processed[kTuckerMaxOrder] = {};
  double* core = nullptr;                       // natural layout, prod(cdims) fp64
  double* factors[kTuckerMaxOrder] = {};        // dims[k] x ranks[k] fp64, column-major
  // fixed-accuracy diagnostics (BLBPDiagnostics, sketch.py:129-143)
  double energy[kTuckerMaxOrder] = {};
  int64_t deflations[kTuckerMaxOrder] = {};
  int64_t iterations[kTuckerMaxOrder] = {};
  double orth_loss[kTuckerMaxOrder] = {};
  cudaStream_t st = nullptr;
  ~TuckerResult() {
    if (core) cudaFreeAsync(core, st);
    for (double* f : factors)
      if (f) cudaFreeAsync(f, st);
  }
  int64_t core_size() const {
    int64_t n = 1;
    for (int i = 0; i < order; ++i) n *= cdims[i];
    return n;
  }
};

static unsigned grid_cap(int64_t work, int threads = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(work, threads), 8ll * num_sms()));
}

// ||x||_F^2 on the host (fixed-order device reduction, one D2H).
template <typename T>
static int sumsq_host(const T* x, int64_t n, double* part, double* out_dev, cudaStream_t st,
                      double& out) {
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 1024));
  launch("tucker", k_sumsq_partial<T>, g, 256, 0, st, x, n, part);
  launch("tucker", k_reduce_partials, 1u, 256, 0, st, (const double*)part, (int)g, (int64_t)1,
         out_dev);
  TR_CUDA(cudaMemcpyAsync(&out, out_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  TR_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// out (R x C x batch -> C x R x batch), column-major blocks
template <typename TI, typename TO>
static void batched_transpose(const TI* in, TO* out, int64_t R, int64_t C, int64_t batch,
                              cudaStream_t st) {
  const int64_t tr_ = cdiv(R, 32), tc = cdiv(C, 32);
  launch("tucker", k_batched_transpose<TI, TO>, (unsigned)(tr_ * tc * batch), 256, 0, st, in, out,
         R, C, tr_, tc);
}

// Z (rows x c) = beta Z + alpha X (rows x k) Y (k x c), k, c <= 64
template <typename TX>
static void tall_small(const TX* X, int64_t ldx, int64_t rows, int k, const double* Y, int ldy,
                       int c, double alpha, double beta, double* Z, int64_t ldz, cudaStream_t st) {
  if (rows <= 0 || c <= 0) return;
  launch("tucker", k_tall_small<TX>, grid_cap(rows), 256, 0, st, X, ldx, rows, k, Y, ldy, c, alpha,
         beta, Z, ldz);
}

// C (K x c) = X^T Z over `rows` rows (fixed-order partial sums), c <= 32 per call
template <typename TX>
static void tall_tn(const TX* X, int64_t ldx, int64_t rows, int K, const double* Zm, int64_t ldz,
                    int c, double* part, int64_t max_part, double* C, cudaStream_t st) {
  if (K <= 0 || c <= 0) return;
  const int64_t want = std::max<int64_t>(1, std::min<int64_t>(2ll * num_sms() / cdiv(K, 32),
                                                              cdiv(rows, 512)));
  const int64_t nblk_cap = std::max<int64_t>(1, max_part / ((int64_t)K * c));
  const int64_t nblk = std::min(want, nblk_cap);
  const int64_t rpb = cdiv(rows, nblk);
  const int64_t nb = cdiv(rows, rpb);
  dim3 grid((unsigned)cdiv(K, 32), (unsigned)nb);
  launch("tucker", k_tall_tn_partial<TX>, grid, 256, 0, st, X, ldx, rows, K, Zm, ldz, c, rpb, part);
  launch("tucker", k_reduce_partials, (unsigned)cdiv((int64_t)K * c, 32), 256, 0, st,
         (const double*)part, (int)nb, (int64_t)K * c, C);
}

// ---- TSQR with levels ---------------------------------------------------------

struct TsqrLevel {
  int64_t rows;
  int RB, nb;
  double *V, *tau, *R;  // reflectors (rows x s), taus (nb x s), stacked R (nb*s x s)
  double* C;            // (nb*s) x s factor of the stack formed on the way back
};

struct Tsqr {
  int s = 0;
  std::vector<TsqrLevel> lv;
  double* Ctop = nullptr;
  size_t sm_local = 0, sm_form = 0, sm_top = 0;
  int64_t top_rows = 0;
};

static size_t tsqr_top_smem(int64_t nrows, int s) {
  return (size_t)(2 * (nrows + 1) * s + (s + 1) * s + 3 * s) * 8;
}

// Plan a QR of a rows x s fp64 matrix: row blocks of RB (<= 256) rows, the
// stacked R factors QR'd again until the stack fits the single-CTA top stage.
static bool tsqr_plan_levels(int64_t rows, int s, Arena& ar, Tsqr& q) {
  const int64_t cap = 200 * 1024;
  q.s = s;
  int64_t rb = std::min<int64_t>(256, (cap / 8 / s - 1) / 2);
  rb = std::max<int64_t>(rb, s);
  q.sm_local = (size_t)((rb + 1) * s + s) * 8;
  q.sm_form = (size_t)(2 * (rb + 1) * s + s) * 8;
  if ((int64_t)q.sm_form > cap) return false;
  int64_t cur = rows;
  while (true) {
    if ((int64_t)tsqr_top_smem(cur, s) <= cap || cur <= rb) {
      if ((int64_t)tsqr_top_smem(cur, s) > cap) return false;
      break;
    }
    TsqrLevel L;
    L.rows = cur;
    L.RB = (int)rb;
    L.nb = (int)cdiv(cur, rb);
    L.V = ar.get<double>(cur * s);
    L.tau = ar.get<double>((int64_t)L.nb * s);
    L.R = ar.get<double>((int64_t)L.nb * s * s);
    L.C = ar.get<double>((int64_t)L.nb * s * s);
    q.lv.push_back(L);
    cur = (int64_t)L.nb * s;
  }
  q.top_rows = cur;
  q.sm_top = tsqr_top_smem(cur, s);
  q.Ctop = ar.get<double>(cur * s);
  return !ar.failed;
}

// Q (rows x s, first s_eff columns valid, rest zero), R (s x s, see k_tsqr_top)
// and info[0] = s_eff for X (rows x s, fp64, column-major; not modified).
static int tsqr_run(const double* X, Tsqr& q, double tol_abs, int pivot, double* Q, double* R,
                    int64_t* info, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tsqr_local, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_tsqr_top, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_tsqr_form<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  const int s = q.s;
  const double* cur = X;
  for (auto& L : q.lv) {
    launch("tucker", k_tsqr_local, (unsigned)L.nb, 256, q.sm_local, st, cur, L.rows, s, L.RB, L.V,
           L.tau, L.R, (int64_t)L.nb * s);
    cur = L.R;
  }
  launch("tucker", k_tsqr_top, 1u, 256, q.sm_top, st, cur, (int)q.top_rows, s, q.Ctop, info,
         tol_abs, pivot, R);
  const double* C = q.Ctop;
  for (int l = (int)q.lv.size() - 1; l >= 0; --l) {
    auto& L = q.lv[l];
    double* dst = l == 0 ? Q : q.lv[l - 1].C;
    // with no level the top's C is Q itself (copied below)
    launch("tucker", k_tsqr_form<double>, (unsigned)L.nb, 256, q.sm_form, st, L.V, L.tau, C,
           L.nb * s, L.rows, s, L.RB, dst, (double*)nullptr);
    C = dst;
  }
  if (q.lv.empty())
    TR_CUDA(cudaMemcpyAsync(Q, q.Ctop, sizeof(double) * q.top_rows * s, cudaMemcpyDeviceToDevice, st));
  TR_LAUNCH_CHECK();
  return 0;
}

// ---- one mode: block Krylov -----------------------------------------------------

template <typename T>
static void carve_mode(Carve& cv, int64_t m, int64_t n, int64_t b, int64_t s, int64_t r,
                       Bufs<T>& bf) {
  bf.max_parts = std::max<int64_t>(rank_splits(m, n), num_sms());
  bf.max_mparts = std::min<int64_t>(cdiv(n, 64), 2 * 148);
  bf.partial = cv.take<double>(bf.max_parts * m * b);
  bf.K = cv.take<double>(m * s);
  bf.work = cv.take<double>(m * s);
  bf.Z = cv.take<double>(m * s);
  bf.Mpart = cv.take<double>(bf.max_mparts * s * s);
  bf.M = cv.take<double>(s * s);
  bf.Zt = cv.take<T>(m * s);
  bf.P = cv.take<T>(m * b);
  bf.coef = cv.take<T>((n + 16) * b);
  bf.W = cv.take<T>(n * s);
  bf.V0 = cv.take<double>(s * r);
  bf.F0 = cv.take<double>(m * r);
  bf.F0t = cv.take<T>(m * r);
  bf.info = cv.take<int64_t>(8);
  bf.ticket = cv.take<unsigned int>(8);
  bf.bsum = cv.take<double>(cdiv(m * b, 32) + 32);
  bf.rpv = cv.take<double>((cdiv(m, 32) + 1) * 32);
  bf.rpi = cv.take<int64_t>((cdiv(m, 32) + 1) * 32);
  const int64_t tq = cdiv(m, std::max<int64_t>(s, 1)) + 1;
  bf.tq_tau = cv.take<double>(tq * s);
  bf.tq_R = cv.take<double>(tq * s * s);
  bf.tq_C = cv.take<double>(tq * s * s);
  bf.zhi = cv.take<float>(m * 32);
  bf.zlo = cv.take<float>(m * 32);
}

// Factor (m x r_eff) and the folded new core of the mode-k unfolding A (m x n,
// columns c = lo + inner f): sketch.py:243-269 on an explicit unfolding.
template <typename T>
static int bki_generic(const T* A, int64_t m, int64_t n, int64_t inner, int r, int b, int q,
                       uint64_t seed, int step, Arena& ar, double** F_out, double** core_out,
                       int64_t& r_eff, cudaStream_t st) {
  const int s = (q + 1) * b;
  TR_REQUIRE(s <= 64 && b <= 32 && r <= 64,
             "block Krylov on the B200 needs (q+1)*b <= 64, b <= 32 and rank <= 64");
  Carve sz(nullptr);
  Bufs<T> bf;
  carve_mode<T>(sz, m, n, b, s, r, bf);
  char* ws = ar.get<char>(sz.off);
  TR_REQUIRE(ws, "device allocation failed (out of memory?)");
  Carve cv(ws);
  carve_mode<T>(cv, m, n, b, s, r, bf);
  Shape dummy{};
  dummy.coll = nullptr;
  SketchSpec sk{seed, (uint64_t)step, n, nullptr, 0};
  static bool attr = false;
  if (!attr) {
    TR_CUDA(cudaFuncSetAttribute(k_ritz<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * 64 * 65 * (int)sizeof(double)));
    attr = true;
  }
  if (bki_mode<T>(dummy, A, m, n, r, b, q, sk, nullptr, bf, bf.V0, bf.F0, bf.F0t, bf.info, st))
    return 2;
  int64_t info[2] = {0, 0};
  TR_CUDA(cudaMemcpyAsync(info, bf.info, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TR_CUDA(cudaStreamSynchronize(st));
  r_eff = info[1];
  double* F = ar.get<double>(m * std::max<int64_t>(r_eff, 1));
  double* core = ar.get<double>(std::max<int64_t>(r_eff, 1) * n);
  TR_REQUIRE(F && core, "device allocation failed (out of memory?)");
  if (r_eff > 0) {
    TR_CUDA(cudaMemcpyAsync(F, bf.F0, sizeof(double) * m * r_eff, cudaMemcpyDeviceToDevice, st));
    launch("tucker", k_core_from_w<T, double>, (unsigned)cdiv(n, 256), 256, 0, st,
           (const T*)bf.W, n, s, (const double*)bf.V0, (int)r_eff, inner, core);
  }
  *F_out = F;
  *core_out = core;
  TR_LAUNCH_CHECK();
  return 0;
}

// ---- one mode: block Lanczos bidiagonalisation -----------------------------------

// W (m x b, fp64) = A V for V (n x b, fp64, column-major): fp64-accumulated
// partial sums over column splits, reduced in a fixed order
template <typename T>
static void av_pass(const T* A, int64_t m, int64_t n, int b, const double* V, double* partial,
                    int64_t max_parts, double* W, cudaStream_t st) {
  const int64_t rowtiles = cdiv(m, 256);
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 4 * num_sms() / rowtiles));
  splits = std::min(splits, max_parts);
  const int64_t cps = cdiv(n, splits);
  const int64_t sp = cdiv(n, cps);
  dim3 grid((unsigned)rowtiles, (unsigned)sp);
  if (b <= 8)
    launch("tucker", k_av_partial<T, 8>, grid, 256, 0, st, A, m, n, b, V, cps, partial);
  else if (b <= 16)
    launch("tucker", k_av_partial<T, 16>, grid, 256, 0, st, A, m, n, b, V, cps, partial);
  else
    launch("tucker", k_av_partial<T, 32>, grid, 256, 0, st, A, m, n, b, V, cps, partial);
  launch("reduce_partials", k_reduce_partials, (unsigned)cdiv(m * b, 32), 256, 0, st,
         (const double*)partial, (int)sp, m * b, W);
}

static double host_spectral_norm(const std::vector<double>& a, int rows, int cols);

template <typename T>
static int blbp_generic(const T* A, int64_t m, int64_t n, int64_t inner, double eps, int b,
                        double tol, uint64_t seed, uint64_t& draw, Arena& ar, double** F_out,
                        double** core_out, int64_t& rank, double& energy_out,
                        int64_t& defl_out, int64_t& iters_out, double& orth_out,
                        cudaStream_t st) {
  TR_REQUIRE(b >= 1 && b <= 32, "block size %d outside [1, 32] on the B200 path", b);
  Arena tmp(st);
  double* part = tmp.get<double>(4096);
  double* scal = tmp.get<double>(8);
  double norm2 = 0.0;
  if (sumsq_host<T>(A, m * n, part, scal, st, norm2)) return 2;
  energy_out = 0.0;
  defl_out = 0;
  iters_out = 0;
  orth_out = 0.0;
  if (norm2 == 0.0) {
    rank = 0;
    *F_out = ar.get<double>(1);
    *core_out = ar.get<double>(1);
    return 0;
  }
  const int64_t max_iters = 2 * cdiv(std::min(m, n), (int64_t)std::max(b, 1)) + 4;
  const int64_t vmax = std::min<int64_t>(n, (int64_t)b * (max_iters + 1));
  const int64_t umax = std::min<int64_t>(m, (int64_t)b * max_iters);
  double* Vacc = tmp.get<double>(n * vmax);
  double* U = ar.get<double>(m * std::max<int64_t>(umax, 1));
  double* W = tmp.get<double>(m * b);
  double* Qm = tmp.get<double>(m * b);
  double* Rm = tmp.get<double>(b * b);
  double* W2 = tmp.get<double>(n * b);
  double* Qn = tmp.get<double>(n * b);
  double* Ln = tmp.get<double>(b * b);
  double* Lprev = tmp.get<double>(b * b);
  double* Lnext = tmp.get<double>(b * b);
  double* G = tmp.get<double>(n * b);
  double* Vcur = tmp.get<double>(n * b);
  double* Cproj = tmp.get<double>(vmax * b);
  const int64_t max_part = std::max<int64_t>(vmax * b * 64, 1 << 16);
  double* tpart = tmp.get<double>(max_part);
  double* Rt = tmp.get<double>(b * b);
  const int64_t av_parts = 4ll * num_sms();
  double* avpart = tmp.get<double>(av_parts * m * b);
  int64_t* info = tmp.get<int64_t>(8);
  Tsqr qm, qn;
  TR_REQUIRE(!tmp.failed && !ar.failed, "device allocation failed (out of memory?)");
  TR_REQUIRE(tsqr_plan_levels(m, b, tmp, qm) && tsqr_plan_levels(n, b, tmp, qn),
             "QR workspace allocation failed");
  const unsigned pgrid =
      (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n * 32, 256), 16ll * num_sms()));

  // r = (Q, R, s_eff) of an m x bc or n x bc block
  auto qr = [&](Tsqr& q, const double* X, int64_t rows, int bc, double t, int piv, double* Q,
                double* R, int64_t& se) -> int {
    // TSQR planned for b columns; narrower blocks are padded with zero columns
    // that the pivoted QR moves last and deflates (or, unpivoted, drops)
    (void)rows;
    if (bc < b)
      TR_CUDA(cudaMemsetAsync((void*)(X + rows * bc), 0, sizeof(double) * rows * (b - bc), st));
    if (tsqr_run(X, q, bc < b && t < 0 ? 0.0 : t, piv, Q, R, info, st)) return 2;
    TR_CUDA(cudaMemcpyAsync(&se, info, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    TR_CUDA(cudaStreamSynchronize(st));
    if (t < 0 && se > bc) se = bc;
    return 0;
  };

  // v_cur = qr(G), G (n x min(b, n)) Gaussian (sketch.py:299-300)
  int bc = (int)std::min<int64_t>(b, n);
  launch("tucker", k_gauss_block, grid_cap(n * bc), 256, 0, st, seed, draw++, n, bc, G);
  int64_t se = 0;
  if (qr(qn, G, n, bc, -1.0, 0, Vcur, Rm, se)) return 2;
  TR_REQUIRE(se == bc, "initial Gaussian block is rank deficient");
  TR_CUDA(cudaMemcpyAsync(Vacc, Vcur, sizeof(double) * n * bc, cudaMemcpyDeviceToDevice, st));
  int64_t kv = bc;       // columns of v_acc
  int64_t ku = 0;        // columns of u_acc
  int64_t su_prev = 0;   // width of u_prev (0: none)
  int lprev_cols = 0;
  double energy = norm2;
  int64_t defl = 0, iters = 0;
  std::vector<int64_t> ublocks;
  while (iters < max_iters) {
    ++iters;
    // w = A v_cur (- u_prev l_prev)            sketch.py:317-320
    av_pass<T>(A, m, n, bc, Vcur, avpart, av_parts, W, st);
    if (su_prev > 0)
      tall_small<double>(U + m * (ku - su_prev), m, m, (int)su_prev, Lprev, b, bc, -1.0, 1.0, W, m,
                         st);
    // u_i, r_i = defl_qr(w, tol)                sketch.py:321
    int64_t su = 0;
    if (qr(qm, W, m, bc, tol, 1, Qm, Rm, su)) return 2;
    const int64_t keep_u = std::min<int64_t>(su, m - ku);
    if (keep_u < su) {
      launch("tucker", k_zero_rows, 1u, 256, 0, st, Rm, b, (int)keep_u, b);
      su = keep_u;
    }
    defl += bc - su;
    if (su > 0)
      TR_CUDA(cudaMemcpyAsync(U + m * ku, Qm, sizeof(double) * m * su, cudaMemcpyDeviceToDevice, st));
    ublocks.push_back(su);
    ku += su;
    double r2 = 0.0;
    if (sumsq_host<double>(Rm, (int64_t)b * b, part, scal, st, r2)) return 2;
    energy -= r2;
    // w2 = A^T u_i - v_cur r_i^T, then w2 -= v_acc (v_acc^T w2)   sketch.py:334-335
    int64_t sv = 0;
    int cols_next = 0;
    if (su > 0) {
      launch("tucker", k_project_rows<T>, pgrid, 256, 0, st, A, m, n, (const double*)Qm, (int)su,
             0, (int)su, n, W2);  // A^T u_i, n x su column-major
      launch("tucker", k_transpose_small, 1u, 256, 0, st, (const double*)Rm, b, (int)su, bc, Rt, b);
      tall_small<double>(Vcur, n, n, bc, Rt, b, (int)su, -1.0, 1.0, W2, n, st);
      tall_tn<double>(Vacc, n, n, (int)kv, W2, n, (int)su, tpart, max_part, Cproj, st);
      tall_small<double>(Vacc, n, n, (int)std::min<int64_t>(kv, 64), Cproj, (int)kv, (int)su, -1.0,
                         1.0, W2, n, st);
      for (int64_t k0 = 64; k0 < kv; k0 += 64)
        tall_small<double>(Vacc + n * k0, n, n, (int)std::min<int64_t>(kv - k0, 64), Cproj + k0,
                           (int)kv, (int)su, -1.0, 1.0, W2, n, st);
      // v_next, l_t = defl_qr(w2, tol)          sketch.py:336
      if (qr(qn, W2, n, (int)su, tol, 1, Qn, Ln, sv)) return 2;
      const int64_t keep_v = std::min<int64_t>(sv, n - kv);
      if (keep_v < sv) {
        launch("tucker", k_zero_rows, 1u, 256, 0, st, Ln, b, (int)keep_v, b);
        sv = keep_v;
      }
      if (sv > 0)
        TR_CUDA(cudaMemcpyAsync(Vacc + n * kv, Qn, sizeof(double) * n * sv, cudaMemcpyDeviceToDevice, st));
      kv += sv;
      if (sv > 0)
        TR_CUDA(cudaMemcpyAsync(Vcur, Qn, sizeof(double) * n * sv, cudaMemcpyDeviceToDevice, st));
      // l_next = l_t^T (su x sv)                 sketch.py:342
      launch("tucker", k_transpose_small, 1u, 256, 0, st, (const double*)Ln, b, (int)sv, (int)su,
             Lnext, b);
      cols_next = (int)sv;
    }
    // fill the block with fresh Gaussian directions  sketch.py:344-351
    const int64_t fill = std::min<int64_t>(b - sv, n - kv);
    if (fill > 0 && su > 0) {
      launch("tucker", k_gauss_block, grid_cap(n * fill), 256, 0, st, seed, draw++, n, (int)fill, G);
      tall_tn<double>(Vacc, n, n, (int)kv, G, n, (int)fill, tpart, max_part, Cproj, st);
      for (int64_t k0 = 0; k0 < kv; k0 += 64)
        tall_small<double>(Vacc + n * k0, n, n, (int)std::min<int64_t>(kv - k0, 64), Cproj + k0,
                           (int)kv, (int)fill, -1.0, 1.0, G, n, st);
      int64_t sf = 0;
      if (qr(qn, G, n, (int)fill, -1.0, 0, Qn, Ln, sf)) return 2;
      TR_CUDA(cudaMemcpyAsync(Vacc + n * kv, Qn, sizeof(double) * n * fill, cudaMemcpyDeviceToDevice, st));
      TR_CUDA(cudaMemcpyAsync(Vcur + n * cols_next, Qn, sizeof(double) * n * fill,
                              cudaMemcpyDeviceToDevice, st));
      kv += fill;
      // zero columns of l_next for the fill
      launch("tucker", k_zero_cols, 1u, 256, 0, st, Lnext, b, (int)su, cols_next, cols_next + (int)fill);
      cols_next += (int)fill;
    } else if (fill > 0) {
      // su == 0: the reference still draws the fill before stopping
      launch("tucker", k_gauss_block, grid_cap(n * fill), 256, 0, st, seed, draw++, n, (int)fill, G);
      kv += fill;
      cols_next += (int)fill;
    }
    double l2 = 0.0;
    if (su > 0 && sumsq_host<double>(Lnext, (int64_t)b * b, part, scal, st, l2)) return 2;
    energy -= l2;
    if (energy < eps * eps * norm2) break;
    if (su == 0 || cols_next == 0 || ku >= m) break;
    TR_CUDA(cudaMemcpyAsync(Lprev, Lnext, sizeof(double) * b * b, cudaMemcpyDeviceToDevice, st));
    su_prev = su;
    lprev_cols = cols_next;
    bc = cols_next;
  }
  (void)lprev_cols;
  rank = ku;
  energy_out = energy;
  defl_out = defl;
  iters_out = iters;
  // local orthogonality loss of the u blocks (sketch.py:273-284), on the host
  if (ku > 0) {
    std::vector<int64_t> offs;
    int64_t o = 0;
    for (int64_t w : ublocks) {
      offs.push_back(o);
      o += w;
    }
    double loss = 0.0;
    int prev = -1;
    for (size_t i = 0; i < ublocks.size(); ++i) {
      const int wi = (int)ublocks[i];
      if (wi == 0) continue;
      std::vector<double> g((size_t)wi * wi);
      tall_tn<double>(U + m * offs[i], m, m, wi, U + m * offs[i], m, wi, tpart, max_part, Cproj, st);
      TR_CUDA(cudaMemcpyAsync(g.data(), Cproj, sizeof(double) * wi * wi, cudaMemcpyDeviceToHost, st));
      TR_CUDA(cudaStreamSynchronize(st));
      for (int d = 0; d < wi; ++d) g[d + (size_t)wi * d] -= 1.0;
      loss = std::max(loss, host_spectral_norm(g, wi, wi));
      if (prev >= 0) {
        const int wp = (int)ublocks[prev];
        std::vector<double> c((size_t)wp * wi);
        tall_tn<double>(U + m * offs[prev], m, m, wp, U + m * offs[i], m, wi, tpart, max_part,
                        Cproj, st);
        TR_CUDA(cudaMemcpyAsync(c.data(), Cproj, sizeof(double) * wp * wi, cudaMemcpyDeviceToHost, st));
        TR_CUDA(cudaStreamSynchronize(st));
        loss = std::max(loss, host_spectral_norm(c, wp, wi));
      }
      prev = (int)i;
    }
    orth_out = loss;
    launch("tucker", k_canonical_signs, (unsigned)ku, 256, 0, st, U, m);
  }
  // core rows u^T a, folded into the natural layout (sketch.py:397-399)
  double* core = ar.get<double>(std::max<int64_t>(ku, 1) * n);
  TR_REQUIRE(core, "device allocation failed (out of memory?)");
  for (int64_t j0 = 0; j0 < ku; j0 += 64)
    launch("tucker", k_project_rows<T>, pgrid, 256, 0, st, A, m, n, (const double*)(U + m * j0),
           (int)std::min<int64_t>(ku - j0, 64), (int)j0, (int)ku, inner, core);
  *F_out = U;
  *core_out = core;
  TR_LAUNCH_CHECK();
  return 0;
}

// Largest singular value of a small host matrix (rows x cols, column-major):
// sqrt of the largest eigenvalue of X^T X by cyclic Jacobi.
static double host_spectral_norm(const std::vector<double>& a, int rows, int cols) {
  std::vector<double> g((size_t)cols * cols, 0.0);
  for (int i = 0; i < cols; ++i)
    for (int j = 0; j < cols; ++j) {
      double s = 0.0;
      for (int k = 0; k < rows; ++k) s += a[k + (size_t)rows * i] * a[k + (size_t)rows * j];
      g[i + (size_t)cols * j] = s;
    }
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < cols; ++p)
      for (int q = p + 1; q < cols; ++q) off += g[p + (size_t)cols * q] * g[p + (size_t)cols * q];
    if (off < 1e-300) break;
    for (int p = 0; p < cols; ++p)
      for (int q = p + 1; q < cols; ++q) {
        const double apq = g[p + (size_t)cols * q];
        if (apq == 0.0) continue;
        const double app = g[p + (size_t)cols * p], aqq = g[q + (size_t)cols * q];
        const double tau = (aqq - app) / (2.0 * apq);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        for (int k = 0; k < cols; ++k) {
          const double gkp = g[k + (size_t)cols * p], gkq = g[k + (size_t)cols * q];
          g[k + (size_t)cols * p] = c * gkp - s * gkq;
          g[k + (size_t)cols * q] = s * gkp + c * gkq;
        }
        for (int k = 0; k < cols; ++k) {
          const double gpk = g[p + (size_t)cols * k], gqk = g[q + (size_t)cols * k];
          g[p + (size_t)cols * k] = c * gpk - s * gqk;
          g[q + (size_t)cols * k] = s * gpk + c * gqk;
        }
      }
  }
  double mx = 0.0;
  for (int i = 0; i < cols; ++i) mx = std::max(mx, g[i + (size_t)cols * i]);
  return sqrt(std::max(mx, 0.0));
}

// ---- the whole compression --------------------------------------------------------

template <typename T>
static int tucker_compress(const T* a, int order, const int64_t* dims, const TuckerSpec& sp,
                           TuckerResult& res, cudaStream_t st) {
  res.st = st;
  res.order = order;
  for (int i = 0; i < order; ++i) res.dims[i] = res.cdims[i] = dims[i];
  Arena keep(st);  // factors and the final core (handed to res)
  Arena tmp(st);   // unfoldings and intermediate cores
  const void* cur = a;
  bool cur_t = true;  // cur is the T input (else an fp64 core)
  uint64_t draw = 0;
  bool empty = false;
  for (int p = 0; p < sp.nproc; ++p) {
    const int k = sp.proc[p];
    res.processed[k] = true;
    int64_t pre = 1, post = 1;
    for (int i = 0; i < k; ++i) pre *= res.cdims[i];
    for (int i = k + 1; i < order; ++i) post *= res.cdims[i];
    const int64_t m = res.cdims[k], n = pre * post;
    if (empty || m == 0 || n == 0) {
      // zero iterates give a rank-0 structure (sketch.py:246-252)
      empty = true;
      res.ranks[k] = 0;
      res.cdims[k] = 0;
      continue;
    }
    int64_t r = 0;
    double* F = nullptr;
    double* core = nullptr;
    auto run = [&](auto tag) -> int {
      using TA = decltype(tag);
      const TA* src = (const TA*)cur;
      const TA* A = src;
      if (pre > 1) {
        TA* buf = tmp.get<TA>(m * n);
        TR_REQUIRE(buf, "device allocation failed (out of memory?)");
        batched_transpose<TA, TA>(src, buf, pre, m, post, st);  // unfold(core, k)
        A = buf;
      }
      if (sp.mode == 0) {
        double nrm2 = 0.0;
        double* part = tmp.get<double>(1024);
        double* one = tmp.get<double>(1);
        if (sumsq_host<TA>(A, m * n, part, one, st, nrm2)) return 2;
        if (nrm2 == 0.0) {
          r = 0;
          return 0;
        }
        if (bki_generic<TA>(A, m, n, pre, (int)sp.ranks[p], (int)sp.blocks[p], (int)sp.krylov[p],
                            sp.seed, p, keep, &F, &core, r, st))
          return 2;
      } else {
        double nrm2 = 0.0;
        double* part = tmp.get<double>(1024);
        double* one = tmp.get<double>(1);
        if (sumsq_host<TA>(A, m * n, part, one, st, nrm2)) return 2;
        const double tol = sp.defl_tol > 0 ? sp.defl_tol : 1e-10 * std::max(sqrt(nrm2), 1e-300);
        if (blbp_generic<TA>(A, m, n, pre, sp.eps, (int)sp.block, tol, sp.seed, draw, keep, &F,
                             &core, r, res.energy[k], res.deflations[k], res.iterations[k],
                             res.orth_loss[k], st))
          return 2;
      }
      if (A != src) tmp.release((void*)A);
      return 0;
    };
    const int rc = cur_t ? (sizeof(T) == 4 ? run(float{}) : run(double{})) : run(double{});
    if (rc) return rc;
    res.ranks[k] = r;
    res.cdims[k] = r;
    if (r == 0) {
      empty = true;
      continue;
    }
    res.factors[k] = (double*)keep.keep(F);
    if (!cur_t) tmp.release((void*)cur);
    cur = keep.keep(core);
    tmp.ptrs.push_back((void*)cur);  // intermediate cores are owned by tmp until the end
    cur_t = false;
  }
  if (empty) {
    for (int i = 0; i < order; ++i)
      if (res.processed[i] && !res.factors[i]) res.ranks[i] = 0;
    return 0;
  }
  if (cur_t) {
    // nothing processed: the core is the input itself (as fp64)
    const int64_t N = res.core_size();
    double* c = keep.get<double>(N);
    TR_REQUIRE(c, "device allocation failed (out of memory?)");
    launch("tucker", k_convert<T, double>, grid_cap(N), 256, 0, st, (const T*)cur, c, N);
    res.core = (double*)keep.keep(c);
  } else {
    res.core = (double*)tmp.keep((void*)cur);
  }
  TR_LAUNCH_CHECK();
  return 0;
}

// out = core x_k F_k over the processed modes (TuckerFactors.reconstruct,
// sketch.py:45-53), ascending mode order; out in T.
template <typename T>
static int tucker_reconstruct(const TuckerResult& res, const double* core, T* out,
                              cudaStream_t st) {
  Arena tmp(st);
  int64_t cd[kTuckerMaxOrder];
  for (int i = 0; i < res.order; ++i) cd[i] = res.cdims[i];
  const double* cur = core;
  int last = -1;
  for (int k = 0; k < res.order; ++k)
    if (res.factors[k]) last = k;
  if (last < 0) {
    const int64_t N = res.core_size();
    launch("tucker", k_convert<double, T>, grid_cap(N), 256, 0, st, core, out, N);
    TR_LAUNCH_CHECK();
    return 0;
  }
  for (int k = 0; k < res.order; ++k) {
    if (!res.factors[k]) continue;
    int64_t pre = 1, post = 1;
    for (int i = 0; i < k; ++i) pre *= cd[i];
    for (int i = k + 1; i < res.order; ++i) post *= cd[i];
    const int64_t r = cd[k], m = res.dims[k];
    const double* X = cur;
    if (pre > 1) {
      double* u = tmp.get<double>(r * pre * post);
      TR_REQUIRE(u, "device allocation failed (out of memory?)");
      batched_transpose<double, double>(cur, u, pre, r, post, st);
      X = u;
    }
    const int64_t ncols = pre * post;
    const bool final_ = k == last;
    const int64_t tm = cdiv(m, 64), tn = cdiv(ncols, 64);
    if (final_ && pre == 1) {
      launch("tucker", k_gemm_smallk<T>, (unsigned)(tm * tn), 256, 0, st, res.factors[k], m, (int)r,
             X, ncols, out, tm);
    } else {
      double* y = tmp.get<double>(m * ncols);
      TR_REQUIRE(y, "device allocation failed (out of memory?)");
      launch("tucker", k_gemm_smallk<double>, (unsigned)(tm * tn), 256, 0, st, res.factors[k], m,
             (int)r, X, ncols, y, tm);
      if (final_) {
        batched_transpose<double, T>(y, out, m, pre, post, st);
      } else if (pre > 1) {
        double* z = tmp.get<double>(m * ncols);
        TR_REQUIRE(z, "device allocation failed (out of memory?)");
        batched_transpose<double, double>(y, z, m, pre, post, st);
        cur = z;
      } else {
        cur = y;
      }
    }
    cd[k] = m;
  }
  TR_LAUNCH_CHECK();
  TR_CUDA(cudaStreamSynchronize(st));  // temporaries are freed at scope exit
  return 0;
}

// Transform-domain SVT of the compressed core (in place) with the transform
// adapted to the core's trailing sizes (sketch.py:452-456, shrink.py:76-106).
template <typename T>
static int tucker_core_svt(const TuckerResult& res, double* core, int kind, const void* mats,
                           const double* alphas, Penalty pen, double tau, cudaStream_t st) {
  Shape sh{};
  sh.order = res.order;
  sh.n1 = res.cdims[0];
  sh.n2 = res.cdims[1];
  sh.nf = 1;
  sh.tr.nt = res.order - 2;
  for (int i = 0; i < 8; ++i) sh.tr.d[i] = 1;
  for (int i = 2; i < res.order; ++i) {
    sh.nf *= res.cdims[i];
    sh.tr.d[i - 2] = res.cdims[i];
  }
  sh.r0 = sh.n1;
  sh.r1 = sh.n2;
  TR_REQUIRE(sh.r0 <= 4096 && sh.r1 <= 4096,
             "core faces above 4096 x 4096 are not supported on the B200 path");
  Arena tmp(st);
  Bufs<T> bf{};
  const int64_t face = sh.r0 * sh.r1;
  bf.core = core;
  bf.cf0 = tmp.get<cplx>(face * sh.nf);
  bf.cf1 = tmp.get<cplx>(face * sh.nf);
  bf.fv = tmp.get<cplx>((sh.r0 > 64 || sh.r1 > 64) ? sh.r1 * sh.r1 * sh.nf : 1);
  int64_t usz = 0;
  for (int i = 0; i < sh.tr.nt; ++i) usz += sh.tr.d[i] * sh.tr.d[i];
  bf.U = tmp.get<cplx>(usz);
  TR_REQUIRE(!tmp.failed, "device allocation failed (out of memory?)");
  if (core_svt<T>(sh, kind, (const cplx*)mats, alphas, pen, tau, bf, st)) return 2;
  TR_CUDA(cudaStreamSynchronize(st));
  return 0;
}

}  // namespace tr
