// Host orchestration of the randomized t-SVT on one stream, and its C ABI.
//
// One call = one launch sequence, fully asynchronous: data-dependent ranks
// (Krylov deflation, r_eff) stay on the device and later kernels read them,
// so the whole LRTA can be captured into a CUDA graph by the caller.
#include <cstdarg>
#include <cstring>
#include <algorithm>

#include "../../include/tenrec_b200.h"
#include "core_svt.cuh"
#include "lrta_kernels.cuh"
#include "tsqr.cuh"
#include "panel.cuh"
#include "panel_mma.cuh"
#include "orth_cluster.cuh"
#include "proj_tc.cuh"
#include "expand_tc.cuh"
#include "prof.cuh"

namespace tr {

static thread_local char g_err[2048] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// Deferred input dependency of a t-SVT (set by the ADMM solver): the stream
// waits for this event right before its first kernel that reads the input
// tensor, so the data-independent prologue (ticket reset, Philox sketch rows)
// runs while the producer of the input is still busy on another stream.
static thread_local cudaEvent_t tl_input_ready = nullptr;
static inline void input_ready(cudaStream_t st) {
  if (tl_input_ready) {
    cudaStreamWaitEvent(st, tl_input_ready, 0);
    tl_input_ready = nullptr;
  }
}

// Bump allocator over the caller's workspace; base == nullptr only sizes.
struct Carve {
  char* base;
  int64_t off = 0;
  explicit Carve(void* b) : base((char*)b) {}
  template <typename X>
  X* take(int64_t count) {
    off = align_up(off, 256);
    X* p = base ? reinterpret_cast<X*>(base + off) : nullptr;
    off += (count > 0 ? count : 1) * (int64_t)sizeof(X);
    return p;
  }
};

// In-place fp64 sum across the ranks of a sharded t-SVT, ordered on `stream`
// (tenrec_b200.h: tr_allreduce_fn).  Null = one rank.
typedef int (*AllreduceFn)(double* buf, int64_t count, void* stream, void* user);

struct Shape {
  int order;
  int64_t n1, n2, nf;  // nf: this rank's faces (trailing modes flattened)
  Trailing tr;         // GLOBAL trailing dims (the transform runs on the whole core)
  int64_t r0, r1, b0, b1, q0, q1, s0, s1;
  int64_t nf_all = 0, f0 = 0;  // all faces, index of this rank's first face
  AllreduceFn coll = nullptr;
  void* coll_user = nullptr;
  int64_t faces_all() const { return nf_all > 0 ? nf_all : nf; }
};

static int allreduce(const Shape& sh, double* buf, int64_t count, cudaStream_t st) {
  if (!sh.coll) return 0;
  TR_LAUNCH_CHECK();
  TR_REQUIRE(sh.coll(buf, count, (void*)st, sh.coll_user) == 0, "all-reduce callback failed");
  return 0;
}

static int make_shape(int order, const int64_t* dims, const int64_t* ranks, const int64_t* blocks,
                      const int64_t* krylov, Shape& sh) {
  TR_REQUIRE(order >= 3 && order <= 10, "order must be in [3, 10], got %d", order);
  sh.order = order;
  sh.n1 = dims[0];
  sh.n2 = dims[1];
  sh.nf = 1;
  sh.tr.nt = order - 2;
  for (int i = 0; i < 8; ++i) sh.tr.d[i] = 1;
  for (int i = 2; i < order; ++i) {
    TR_REQUIRE(dims[i] >= 1, "mode %d has length %lld", i, (long long)dims[i]);
    sh.nf *= dims[i];
    sh.tr.d[i - 2] = dims[i];
  }
  TR_REQUIRE(sh.n1 >= 1 && sh.n2 >= 1, "empty leading modes");
  sh.r0 = ranks[0];
  sh.r1 = ranks[1];
  sh.b0 = blocks[0];
  sh.b1 = blocks[1];
  sh.q0 = krylov[0];
  sh.q1 = krylov[1];
  TR_REQUIRE(sh.r0 >= 1 && sh.r0 <= sh.n1 && sh.r1 >= 1 && sh.r1 <= sh.n2,
             "ranks (%lld, %lld) out of range", (long long)sh.r0, (long long)sh.r1);
  TR_REQUIRE(sh.r0 <= 64 && sh.r1 <= 64, "ranks above 64 are not supported on the GPU path");
  TR_REQUIRE(sh.b0 >= 1 && sh.b0 <= sh.r0 && sh.b1 >= 1 && sh.b1 <= sh.r1,
             "block sizes must satisfy 1 <= b <= r");
  TR_REQUIRE(sh.b0 <= 32 && sh.b1 <= 32, "block sizes above 32 are not supported");
  TR_REQUIRE(sh.q0 >= 0 && sh.q1 >= 0, "Krylov depth must be >= 0");
  TR_REQUIRE((sh.q0 + 1) * sh.b0 >= sh.r0 && (sh.q1 + 1) * sh.b1 >= sh.r1, "(q+1)*b < rank");
  sh.s0 = (sh.q0 + 1) * sh.b0;
  sh.s1 = (sh.q1 + 1) * sh.b1;
  TR_REQUIRE(sh.s0 <= 64 && sh.s1 <= 64, "Krylov block width (q+1)*b above 64 is not supported");
  return 0;
}

template <typename T>
struct Bufs {
  double *partial, *K, *work, *Z, *Mpart, *M;
  T *Zt, *P, *coef, *W;
  double *V0, *V1, *F0, *F1;
  T *F0t, *F1t, *A1, *C1;
  double* core;
  cplx *cf0, *cf1, *U;
  cplx* fv;  // face-SVT rotations for faces larger than 64 (global scratch)
  int64_t* info;
  unsigned int* ticket;  // last-block counter of k_reduce_normalize (zeroed per t-SVT)
  double* bsum;          // its per-block sums of squares
  double* rpv;           // k_ritz_apply per-block column candidates (value, row)
  int64_t* rpi;
  double *tq_tau, *tq_R, *tq_C;
  float *zhi, *zlo;
  float *c1h, *c1l, *f0h, *f0l;  // tcgen05 expand operands (K-major, K = 32, tf32 hi / lo)
  int64_t max_parts, max_mparts;
};

// SMs a persistent streaming kernel of the t-SVT may fill.  A few SMs stay
// free (TR_RESERVE_SMS, default 4) so the single-CTA latency kernels of the
// other mode streams (Jacobi, TSQR) are not blocked behind a whole streaming
// pass: -0.4 ms per ADMM sweep (11.9 -> 11.45 ms) on the bench workload.
static int stream_sms() {
  static const int reserve = getenv("TR_RESERVE_SMS") ? atoi(getenv("TR_RESERVE_SMS")) : 4;
  return std::max(1, num_sms() - reserve);
}

static int64_t rank_splits(int64_t m, int64_t n) {
  const int64_t rowtiles = cdiv(m, 256);
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 4 * num_sms() / rowtiles));
  return splits;
}

template <typename T>
static void carve(Carve& cv, const Shape& sh, Bufs<T>& b) {
  const int64_t mmax = std::max(sh.n1, sh.n2);
  const int64_t smax = std::max(sh.s0, sh.s1);
  const int64_t bmax = std::max(sh.b0, sh.b1);
  const int64_t nA0 = sh.n2 * sh.nf, nA1 = sh.r0 * sh.nf;
  const int64_t nmax = std::max(nA0, nA1);
  b.max_parts = std::max<int64_t>(std::max(rank_splits(sh.n1, nA0), rank_splits(sh.n2, nA1)),
                                  num_sms());
  b.max_mparts = std::min<int64_t>(cdiv(nmax, 64), 2 * 148);
  b.partial = cv.take<double>(b.max_parts * mmax * bmax);
  b.K = cv.take<double>(mmax * smax);
  b.work = cv.take<double>(mmax * smax);
  b.Z = cv.take<double>(mmax * smax);
  b.Mpart = cv.take<double>(b.max_mparts * smax * smax);
  b.M = cv.take<double>(smax * smax);
  b.Zt = cv.take<T>(mmax * smax);
  b.P = cv.take<T>(mmax * bmax);
  b.coef = cv.take<T>((nmax + 16) * bmax);  // + chunk pad of the sketch rows
  b.W = cv.take<T>(nmax * smax);
  b.V0 = cv.take<double>(sh.s0 * sh.r0);
  b.V1 = cv.take<double>(sh.s1 * sh.r1);
  b.F0 = cv.take<double>(sh.n1 * sh.r0);
  b.F1 = cv.take<double>(sh.n2 * sh.r1);
  b.F0t = cv.take<T>(sh.n1 * sh.r0);
  b.F1t = cv.take<T>(sh.n2 * sh.r1);
  b.A1 = cv.take<T>(sh.n2 * nA1);
  b.C1 = cv.take<T>(sh.r0 * sh.n2 * sh.nf);
  b.core = cv.take<double>(sh.r0 * sh.r1 * sh.faces_all());
  b.cf0 = cv.take<cplx>(sh.r0 * sh.r1 * sh.faces_all());
  b.cf1 = cv.take<cplx>(sh.r0 * sh.r1 * sh.faces_all());
  b.fv = cv.take<cplx>(sh.r0 > 64 || sh.r1 > 64 ? sh.r1 * sh.r1 * sh.faces_all() : 0);
  int64_t usz = 0;
  for (int i = 0; i < sh.tr.nt; ++i) usz += sh.tr.d[i] * sh.tr.d[i];
  b.U = cv.take<cplx>(usz);
  b.info = cv.take<int64_t>(8);
  b.ticket = cv.take<unsigned int>(8);
  b.bsum = cv.take<double>(cdiv(mmax * bmax, 32) + 32);
  b.rpv = cv.take<double>((cdiv(mmax, 32) + 1) * 32);
  b.rpi = cv.take<int64_t>((cdiv(mmax, 32) + 1) * 32);
  int64_t tq = 0;
  for (int64_t mm : {sh.n1, sh.n2})
    for (int64_t ss : {sh.s0, sh.s1}) tq = std::max<int64_t>(tq, cdiv(mm, std::max<int64_t>(ss, 1)) + 1);
  const int64_t tq_rows = tq * smax;  // nb * s bound (RB >= s)
  b.tq_tau = cv.take<double>(tq_rows);
  b.tq_R = cv.take<double>(tq_rows * smax);
  b.tq_C = cv.take<double>(tq_rows * smax);
  b.zhi = cv.take<float>(mmax * 32);
  b.zlo = cv.take<float>(mmax * 32);
  const bool tc_expand = sizeof(T) == 4 && sh.r0 <= 32;
  b.c1h = cv.take<float>(tc_expand ? sh.n2 * sh.nf * 32 : 1);
  b.c1l = cv.take<float>(tc_expand ? sh.n2 * sh.nf * 32 : 1);
  b.f0h = cv.take<float>(tc_expand ? sh.n1 * 32 : 1);
  b.f0l = cv.take<float>(tc_expand ? sh.n1 * 32 : 1);
}

template <typename T, int B>
static void launch_rank_update(const T* A, int64_t m, int64_t n, int b, const T* coef,
                               const T* gover, SketchSpec sk, double* partial, int64_t splits,
                               cudaStream_t st) {
  const int64_t cps = cdiv(n, splits);
  const int64_t sp = cdiv(n, cps);
  dim3 grid((unsigned)cdiv(m, 256), (unsigned)sp);
  launch("rank_update", k_rank_update<T, B>, grid, 256, 0, st, A, m, n, b, coef, gover, sk, cps, partial);
}

// partial (nparts x m x b) over the columns, dispatching the register width.
template <typename T>
static int64_t rank_update(const T* A, int64_t m, int64_t n, int b, const T* coef, const T* gover,
                           SketchSpec sk, double* partial, cudaStream_t st) {
  const int64_t splits = rank_splits(m, n);
  const int64_t sp = cdiv(n, cdiv(n, splits));
  if (b <= 8) launch_rank_update<T, 8>(A, m, n, b, coef, gover, sk, partial, splits, st);
  else if (b <= 16) launch_rank_update<T, 16>(A, m, n, b, coef, gover, sk, partial, splits, st);
  else launch_rank_update<T, 32>(A, m, n, b, coef, gover, sk, partial, splits, st);
  return sp;
}

template <typename T>
static void dot_cols(const T* A, int64_t m, int64_t n, const T* Z, int s, T* W, cudaStream_t st) {
  const int64_t warps = std::min<int64_t>(n, (int64_t)num_sms() * 64);
  const unsigned grid = (unsigned)cdiv(warps * 32, 256);
  if (s <= 8) launch("dot_cols", k_dot_cols<T, 8>, grid, 256, 0, st, A, m, n, Z, s, W);
  else if (s <= 16) launch("dot_cols", k_dot_cols<T, 16>, grid, 256, 0, st, A, m, n, Z, s, W);
  else if (s <= 32) launch("dot_cols", k_dot_cols<T, 32>, grid, 256, 0, st, A, m, n, Z, s, W);
  else launch("dot_cols", k_dot_cols<T, 64>, grid, 256, 0, st, A, m, n, Z, s, W);
}

// Fused TMA-staged panel pass (panel.cuh) when the unfolding suits it:
// 16-byte aligned columns, m <= 2048 rows, b <= 16.
template <typename T>
static bool panel_ok(const T* A, int64_t m, int b) {
  return (m * (int64_t)sizeof(T)) % 16 == 0 && m <= 2048 && b <= 16 &&
         ((uintptr_t)A % 16) == 0 && getenv("TR_NO_PANEL") == nullptr;
}

template <typename T, int B, int Q, int MODE>
static int64_t panel_launch(const T* A, const T* P, const T* gover, PanelArgs pa,
                            double* partial, cudaStream_t st) {
  const int64_t grid = std::min<int64_t>(pa.nchunks, stream_sms());
  const size_t smem = ((size_t)kPanelStages * pa.m * pa.cc + (size_t)pa.cc * B * 9) * sizeof(T);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_panel<T, B, Q, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    attr = true;
  }
  launch(MODE ? "panel_gram" : "panel_sketch", k_panel<T, B, Q, MODE>, (unsigned)grid,
         kPanelThreads, smem, st, A, P, gover, pa, partial);
  return grid;
}

// Tensor-core Krylov pass (panel_mma.cuh): fp32 unfoldings with m <= 1024
// (one CTA per chunk sequence) or m <= 2048 (CL = 2: a 2-CTA cluster splits
// the rows), b <= 8 per pass.
template <int RG, int MODE, int CL>
static int64_t panel_mma_launch(const float* A, const float* P, const float* coef,
                                PanelMmaArgs pa, double* partial, cudaStream_t st) {
  const size_t fixed =
      MODE ? (size_t)(2 * kPmWarps * kPmRS + 4 * kPmTE) * sizeof(float) : 0;
  const size_t stage =
      (size_t)kPmCols * pa.S * sizeof(float) + (MODE ? 0 : (size_t)kPmCols * pa.b * sizeof(float));
  pa.nst = (int)std::min<size_t>(kPmMaxStages, (220 * 1024 - fixed) / stage);
  static const int nst_cap = getenv("TR_PM_STAGES") ? atoi(getenv("TR_PM_STAGES")) : 0;
  if (nst_cap >= 2) pa.nst = std::min(pa.nst, nst_cap);
  const int64_t clusters = std::min<int64_t>(pa.nchunks, stream_sms() / CL);
  const size_t smem = pa.nst * stage + fixed;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_panel_mma<RG, MODE, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    attr = true;
  }
  launch(MODE ? "panel_gram" : "panel_sketch", k_panel_mma<RG, MODE, CL>,
         (unsigned)(clusters * CL), kPmThreads, smem, st, A, P, coef, pa, partial);
  return clusters;
}

// MODE 0 draws the sketch rows into `rows` ((n + 16) x b scratch) first.
// Blocks wider than 8 columns run as ceil(b / 8) passes of up to 8 columns
// each (column-separable products, see PanelMmaArgs::j0); the tensor-core pass
// read twice still beats the CUDA-core fallback several times over.
template <int MODE>
static int64_t panel_mma(const float* A, int64_t m, int64_t n, int b, const float* P,
                         const float* gover, SketchSpec sk, float* rows, double* partial,
                         cudaStream_t st) {
  static const bool off = getenv("TR_NO_PANEL_MMA") != nullptr;
  static const int max_b = getenv("TR_PANEL_MMA_MAXB") ? atoi(getenv("TR_PANEL_MMA_MAXB")) : 32;
  // m in (1024, 2048]: the 2-CTA cluster split (TR_NO_PANEL_CLUSTER / _SKETCH: the CUDA-core pass)
  static const bool no_cl = getenv("TR_NO_PANEL_CLUSTER") != nullptr;
  static const bool no_cl0 = getenv("TR_NO_PANEL_CLUSTER_SKETCH") != nullptr;
  if (off || m > ((no_cl || (MODE == 0 && no_cl0)) ? 1024 : 2048) || b > max_b || rows == nullptr)
    return -1;
  int64_t np = -1;
  for (int j0 = 0; j0 < b; j0 += 8) {
    const int bw = std::min(8, b - j0);
    PanelMmaArgs pa;
    pa.m = m;
    pa.n = n;
    pa.b = bw;
    pa.j0 = j0;
    pa.b_all = b;
    pa.S = panel_mma_slot(m > 1024 ? ((m + 1) / 2 + 3) / 4 * 4 : m);
    pa.nst = 2;
    pa.nchunks = cdiv(n, kPmCols);
    if (MODE == 0) {
      const int64_t total = pa.nchunks * kPmCols;  // one thread per (padded) column
      launch("sketch_rows", k_sketch_rows,
             (unsigned)std::min<int64_t>(cdiv(total, 128), 8 * num_sms()), 128, 0, st, n, bw, sk,
             gover, rows, j0, b);
    }
    input_ready(st);  // everything before this line is independent of A
    const float* cf = MODE == 0 ? rows : nullptr;
    const float* Pj = MODE == 1 ? P + m * (int64_t)j0 : P;
    np = m <= 512    ? panel_mma_launch<1, MODE, 1>(A, Pj, cf, pa, partial, st)
         : m <= 1024 ? panel_mma_launch<2, MODE, 1>(A, Pj, cf, pa, partial, st)
                     : panel_mma_launch<2, MODE, 2>(A, Pj, cf, pa, partial, st);
  }
  return np;
}

template <int MODE>
static int64_t panel_mma(const double*, int64_t, int64_t, int, const double*, const double*,
                         SketchSpec, double*, double*, cudaStream_t) {
  return -1;
}

template <typename T, int MODE>
static int64_t panel(const T* A, int64_t m, int64_t n, int b, const T* P, const T* gover,
                     SketchSpec sk, T* rows, double* partial, cudaStream_t st) {
  const int64_t np = panel_mma<MODE>(A, m, n, b, P, gover, sk, rows, partial, st);
  if (np >= 0) return np;
  input_ready(st);
  PanelArgs pa;
  pa.m = m;
  pa.n = n;
  pa.b = b;
  pa.cc = (int)std::max<int64_t>(1, std::min<int64_t>(32, (48 * 1024) / (m * (int64_t)sizeof(T))));
  pa.nchunks = cdiv(n, pa.cc);
  pa.sk = sk;
  const bool q2 = m > 1024;
  if (b <= 8)
    return q2 ? panel_launch<T, 8, 2, MODE>(A, P, gover, pa, partial, st)
              : panel_launch<T, 8, 1, MODE>(A, P, gover, pa, partial, st);
  return q2 ? panel_launch<T, 16, 2, MODE>(A, P, gover, pa, partial, st)
            : panel_launch<T, 16, 1, MODE>(A, P, gover, pa, partial, st);
}

static void reduce(const double* part, int64_t nparts, int64_t len, double* out, cudaStream_t st) {
  launch("reduce_partials", k_reduce_partials, (unsigned)cdiv(len, 32), 256, 0, st, part,
         (int)nparts, len, out);
}

// TSQR row-block size for an m x s Krylov block and the shared memory of each
// stage; ok = false when the blocks do not fit (single-CTA fallback).
struct TsqrPlan {
  bool ok;
  int RB, nb;
  size_t sm_local, sm_top, sm_form;
};

static TsqrPlan tsqr_plan(int64_t m, int s, bool wide = false) {
  TsqrPlan p{};
  const int64_t cap = 200 * 1024;
  // row blocks of <= 256 rows; `wide`: as many rows as the form stage holds,
  // so fewer blocks -- a shorter R stack for the single-CTA top stage
  int64_t rb = (cap / 8 - s) / (2 * s) - 1;  // largest RB whose form stage fits
  if (!wide) rb = std::min<int64_t>(256, rb);
  rb = std::max<int64_t>(rb, s);
  p.RB = (int)rb;
  p.nb = (int)cdiv(m, rb);
  const int64_t nrows = (int64_t)p.nb * s;
  p.sm_local = (size_t)((rb + 1) * s + s) * 8;
  p.sm_form = (size_t)(2 * (rb + 1) * s + s) * 8;
  p.sm_top = (size_t)(2 * (nrows + 1) * s + (s + 1) * s + 3 * s) * 8;
  p.ok = (int64_t)p.sm_form <= cap && (int64_t)p.sm_top <= cap && (int64_t)p.sm_local <= cap;
  return p;
}

template <typename T>
// Returns true when the kernel also wrote the tf32 split of Z (bf.zhi / bf.zlo)
// that the tensor-core projection reads (fp32 unfoldings, cluster TSQR).
static bool orth_basis(int64_t m, int s, Bufs<T>& bf, int64_t* info, cudaStream_t st) {
  static const bool cluster_off = getenv("TR_NO_ORTH_CLUSTER") != nullptr;
  if (!cluster_off && m <= (int64_t)kOcCtas * kOcRows && s <= kOcS) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_orth_cluster<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kOcSmem);
      attr = true;
    }
    const bool split = sizeof(T) == 4 && getenv("TR_NO_FUSED_ZSPLIT") == nullptr;
    launch("orth", k_orth_cluster<T>, kOcCtas, kOcThreads, kOcSmem, st, (const double*)bf.K, m, s,
           bf.Z, bf.Zt, info, split ? bf.zhi : (float*)nullptr, split ? bf.zlo : (float*)nullptr);
    return split;
  }
  TsqrPlan p = tsqr_plan(m, s);
  if (!p.ok) p = tsqr_plan(m, s, true);
  if (!p.ok) {
    launch("orth", k_orth<T>, 1, 1024, 0, st, bf.K, m, s, bf.work, bf.Z, bf.Zt, info);
    return false;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tsqr_local, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_tsqr_top, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_tsqr_form<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const int64_t nrows = (int64_t)p.nb * s;
  static const int tq_threads = getenv("TR_TSQR_THREADS") ? atoi(getenv("TR_TSQR_THREADS")) : 256;
  launch("orth", k_tsqr_local, p.nb, tq_threads, p.sm_local, st, bf.K, m, s, p.RB, bf.work,
         bf.tq_tau, bf.tq_R, nrows);
  launch("orth", k_tsqr_top, 1, tq_threads, p.sm_top, st, bf.tq_R, (int)nrows, s, bf.tq_C, info,
         0.0, 1, (double*)nullptr);
  launch("orth", k_tsqr_form<T>, p.nb, tq_threads, p.sm_form, st, bf.work, bf.tq_tau, bf.tq_C,
         (int)nrows, m, s, p.RB, bf.Z, bf.Zt);
  return false;
}

// W = A^T Z and M = W^T W on the tensor cores (proj_tc.cuh) for fp32
// unfoldings with m % 32 == 0 and s <= 32; returns false to use the generic path.
// cuTensorMapEncodeTiled from the driver (no libcuda link dependency)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
    cudaGetLastError();
  }
  return fn;
}

// fp32 column-major rows x cols matrix, boxes of 32 rows x box_cols columns,
// 128-byte swizzle (one box row = 32 fp32 = one swizzle atom), zero OOB fill
static bool tmap_f32(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int box_cols) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  const cuuint64_t strides[1] = {(cuuint64_t)rows * sizeof(float)};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_cols};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// W = A^T Z on the tensor cores (proj_tc.cuh) when the unfolding suits it:
// s <= 32 in one pass with the fused Gram; 32 < s <= 64 as two column blocks
// of W (two passes over A) and the Gram from W afterwards.
static bool project(const float* A, int64_t m, int64_t n, int s, Bufs<float>& bf, cudaStream_t st,
                    bool z_split_done = false) {
  if (m % 32 != 0 || s > 64 || ((uintptr_t)A % 16) != 0 || n >= (1ll << 31) ||
      getenv("TR_NO_TC") != nullptr)
    return false;
  CUtensorMap ma, mh, ml;
  if (!tmap_f32(&ma, A, m, n, 128) || !tmap_f32(&mh, bf.zhi, m, 32, 32) ||
      !tmap_f32(&ml, bf.zlo, m, 32, 32))
    return false;
  const int64_t ntiles = cdiv(n, 128);
  const int64_t grid = std::min<int64_t>(ntiles, stream_sms());
  const size_t smem = (size_t)kPwSmemBytes + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_proj_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  for (int j0 = 0; j0 < s; j0 += 32) {
    const int cnt = std::min(32, s - j0);
    if (!(z_split_done && s <= 32))
      launch("proj_split", k_split_z, (unsigned)cdiv(m * 32, 256), 256, 0, st,
             (const double*)(bf.Z + m * (int64_t)j0), m, cnt, bf.zhi, bf.zlo);
    launch("proj_tc", k_proj_ws, (unsigned)grid, kPwThreads, smem, st, ma, mh, ml, m, n, cnt,
           bf.W + j0, s <= 32 ? bf.Mpart : (double*)nullptr, s);
  }
  if (s <= 32) {
    reduce(bf.Mpart, grid, (int64_t)s * s, bf.M, st);
  } else {
    const int64_t mparts = std::min<int64_t>(cdiv(n, 64), bf.max_mparts);
    const int64_t rpb = cdiv(n, mparts);
    const int64_t mp = cdiv(n, rpb);
    launch("wtw", k_wtw<float>, (unsigned)mp, 256, 32 * s * sizeof(double), st, (const float*)bf.W,
           n, s, rpb, bf.Mpart);
    reduce(bf.Mpart, mp, (int64_t)s * s, bf.M, st);
  }
  return true;
}

static bool project(const double*, int64_t, int64_t, int, Bufs<double>&, cudaStream_t, bool = false) {
  return false;
}

// One mode of R-STHOSVD-BKI on the m x n unfolding A (sketch.py:243-265).
// Leaves the factor in F (fp64) / Ft, the eigenvectors V (s x r) and
// W = A^T Z (n x s) for the core; info[0] = s_eff, info[1] = r_eff.
template <typename T>
static int bki_mode(const Shape& sh, const T* A, int64_t m, int64_t n, int r, int b, int q,
                    SketchSpec sk, const T* gover, Bufs<T>& bf, double* V, double* F, T* Ft,
                    int64_t* info, cudaStream_t st) {
  const int s = (q + 1) * b;
  const bool fused = panel_ok<T>(A, m, b);
  // reduce + normalise in one launch unless the columns are sharded (the
  // all-reduce goes between the two)
  const bool fuse_norm = sh.coll == nullptr && getenv("TR_NO_FUSED_NORMALIZE") == nullptr;
  TR_CUDA(cudaMemsetAsync(bf.ticket, 0, 2 * sizeof(unsigned int), st));  // last-block tickets
  auto reduce_normalize = [&](int64_t np_, double* slot) -> int {
    if (fuse_norm) {
      launch("reduce_partials", k_reduce_normalize<T>, (unsigned)cdiv(m * b, 32), 256, 0, st,
             (const double*)bf.partial, (int)np_, m * b, slot, bf.P, bf.bsum, bf.ticket);
      return 0;
    }
    reduce(bf.partial, np_, m * b, slot, st);
    if (allreduce(sh, slot, m * b, st)) return 1;  // columns are sharded: sum the ranks
    launch("normalize_piece", k_normalize_piece<T>, 1, 1024, 0, st, slot, m * b, bf.P);
    return 0;
  };
  if (!fused) input_ready(st);
  int64_t np = fused ? panel<T, 0>(A, m, n, b, nullptr, gover, sk, bf.coef, bf.partial, st)
                     : rank_update<T>(A, m, n, b, nullptr, gover, sk, bf.partial, st);
  input_ready(st);  // (no-op: the sketch pass has consumed it)
  if (reduce_normalize(np, bf.K)) return 1;
  for (int k = 1; k <= q; ++k) {
    if (fused) {
      np = panel<T, 1>(A, m, n, b, bf.P, nullptr, sk, bf.coef, bf.partial, st);
    } else {
      dot_cols<T>(A, m, n, bf.P, b, bf.coef, st);
      np = rank_update<T>(A, m, n, b, bf.coef, nullptr, sk, bf.partial, st);
    }
    double* slot = bf.K + m * (int64_t)b * k;
    if (reduce_normalize(np, slot)) return 1;
  }
  const bool z_split = orth_basis<T>(m, s, bf, info, st);
  if (!project(A, m, n, s, bf, st, z_split)) {
    dot_cols<T>(A, m, n, bf.Zt, s, bf.W, st);
    const int64_t mparts = std::min<int64_t>(cdiv(n, 64), bf.max_mparts);
    const int64_t rpb = cdiv(n, mparts);
    const int64_t mp = cdiv(n, rpb);
    if (s <= 32)
      launch("wtw", k_wtw32<T>, (unsigned)mp, 256, 0, st, (const T*)bf.W, n, s, rpb, bf.Mpart);
    else
      launch("wtw", k_wtw<T>, (unsigned)mp, 256, 32 * s * sizeof(double), st, bf.W, n, s, rpb,
             bf.Mpart);
    reduce(bf.Mpart, mp, (int64_t)s * s, bf.M, st);
  }
  if (allreduce(sh, bf.M, (int64_t)s * s, st)) return 1;  // W rows are sharded
  // Jacobi in one CTA; F = Z V_top and the canonical signs over many CTAs
  const bool split = s <= 32 && r <= 32 && getenv("TR_NO_RITZ_APPLY") == nullptr;
  static const bool two_sided = getenv("TR_RITZ_2S") != nullptr;
  if (split && !two_sided)
    launch("ritz", k_ritz_pc, 1, 256, 0, st, (const double*)bf.M, s, r, V, info);
  else
    launch("ritz", k_ritz<T>, 1, 256, 2 * 64 * 65 * sizeof(double), st, bf.M, s, bf.Z, m, r, V,
           split ? (double*)nullptr : F, Ft, info);
  if (split)
    launch("ritz", k_ritz_apply<T>, (unsigned)cdiv(m, 32), 256, 0, st, (const double*)bf.Z, m,
           s, V, r, (const int64_t*)info, F, Ft, bf.rpv, bf.rpi, bf.ticket + 1);
  TR_LAUNCH_CHECK();
  return 0;
}

template <typename T>
static int lrta_compress(const T* a, const Shape& sh, uint64_t seed, const T* g0, const T* g1,
                         Bufs<T>& bf, cudaStream_t st, cudaEvent_t after_mode0 = nullptr) {
  static bool attr = false;
  if (!attr) {
    TR_CUDA(cudaFuncSetAttribute(k_ritz<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * 64 * 65 * (int)sizeof(double)));
    attr = true;
  }
  const int64_t nA0 = sh.n2 * sh.nf, nA1 = sh.r0 * sh.nf;
  // mode 0 on the tensor itself (m = n1, n = n2 * nf)
  SketchSpec sk0{seed, 0, sh.n2 * sh.faces_all(), nullptr, sh.n2 * sh.f0};
  if (bki_mode<T>(sh, a, sh.n1, nA0, (int)sh.r0, (int)sh.b0, (int)sh.q0, sk0, g0, bf, bf.V0,
                  bf.F0, bf.F0t, bf.info, st))
    return 2;
  // the passes over the whole tensor are done: what follows streams the small
  // core only (the caller may schedule HBM-bound work of another stream here)
  if (after_mode0) TR_CUDA(cudaEventRecord(after_mode0, st));
  // core rows -> mode-1 unfolding (n2 x r0*nf), contiguous columns
  if constexpr (sizeof(T) == 4) {
    if (sh.s0 <= 32 && sh.r0 <= 32)
      launch("core_from_w", k_core_from_w_s<T>, (unsigned)cdiv(nA0, 256), 256, 0, st,
             (const float*)bf.W, nA0, (int)sh.s0, (const double*)bf.V0, (int)sh.r0, sh.n2, bf.A1);
    else
      launch("core_from_w", k_core_from_w<T, T>, (unsigned)cdiv(nA0, 256), 256, 0, st,
             bf.W, nA0, (int)sh.s0, bf.V0, (int)sh.r0, sh.n2, bf.A1);
  } else {
    launch("core_from_w", k_core_from_w<T, T>, (unsigned)cdiv(nA0, 256), 256, 0, st,
           bf.W, nA0, (int)sh.s0, bf.V0, (int)sh.r0, sh.n2, bf.A1);
  }
  // mode 1 on the core (m = n2, n = r0 * nf); logical columns use r0_eff
  SketchSpec sk1{seed, 1, sh.r0, bf.info + 1, sh.r0 * sh.f0};
  if (bki_mode<T>(sh, bf.A1, sh.n2, nA1, (int)sh.r1, (int)sh.b1, (int)sh.q1, sk1, g1, bf, bf.V1,
                  bf.F1, bf.F1t, bf.info + 2, st))
    return 2;
  // this rank's faces of the r0 x r1 x faces core; sharded: zero the rest and
  // sum the ranks, so every rank holds the whole core for the transform-domain SVT
  const int64_t face = sh.r0 * sh.r1;
  if (sh.coll) TR_CUDA(cudaMemsetAsync(bf.core, 0, sizeof(double) * face * sh.faces_all(), st));
  launch("core_from_w", k_core_from_w<T, double>, (unsigned)cdiv(nA1, 256), 256, 0, st,
      bf.W, nA1, (int)sh.s1, bf.V1, (int)sh.r1, sh.r0, bf.core + face * sh.f0);
  if (allreduce(sh, bf.core, face * sh.faces_all(), st)) return 2;
  TR_LAUNCH_CHECK();
  return 0;
}

// One transform-mode product of the core (core_svt.cuh): the staged kernel
// (both operands in shared memory) when they fit and the grid dimensions allow
// it, else the direct kernel.
static void mode_product(const void* in, int in_real, void* out, int out_real, int64_t st_lo, int n,
                         int64_t hi, const cplx* U, int inverse, double alpha, int64_t face,
                         const Trailing& skip, unsigned g_direct, cudaStream_t st) {
  static const bool direct = getenv("TR_MODE_PRODUCT_DIRECT") != nullptr;
  constexpr size_t kMaxSmem = 96 * 1024;  // two CTAs per SM
  const int64_t tiles = cdiv(st_lo, kMpTL);
  const size_t smem = mode_product_smem(n);
  if (direct || smem > kMaxSmem || hi > 65535 || tiles >= (1ll << 31) || cdiv(n, kMpKB) > 65535) {
    launch("mode_product", k_mode_product, g_direct, 256, 0, st, in, in_real, out, out_real, st_lo,
           n, hi, U, inverse, alpha, face, skip);
    return;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_mode_product_t, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMaxSmem);
    attr = true;
  }
  launch("mode_product", k_mode_product_t,
         dim3((unsigned)tiles, (unsigned)hi, (unsigned)cdiv(n, kMpKB)), kMpTL * kMpKB, smem, st, in,
         in_real, out, out_real, st_lo, n, hi, U, inverse, alpha, face, skip);
}

// Transform-domain SVT of the r0 x r1 x trailing core in place (bf.core).
template <typename T>
static int core_svt(const Shape& sh, int kind, const cplx* mats, const double* alphas,
                    Penalty pen, double tau, Bufs<T>& bf, cudaStream_t st,
                    bool transform_built = false) {
  const int64_t face = sh.r0 * sh.r1;
  const int nt = sh.tr.nt;
  const cplx* U[8];
  double al[8];
  int64_t uoff = 0;
  for (int i = 0; i < nt; ++i) {
    const int n = (int)sh.tr.d[i];
    if (kind == TR_TRANSFORM_EXPLICIT) {
      U[i] = mats + uoff;
      al[i] = alphas[i];
    } else {
      // (a caller that owns the workspace across calls -- the ADMM solver -- keeps the matrices)
      if (!transform_built)
        launch("build_transform", k_build_transform, (unsigned)cdiv((int64_t)n * n, 256), 256, 0,
               st, kind, n, bf.U + uoff);
      U[i] = bf.U + uoff;
      al[i] = kind == TR_TRANSFORM_FFT ? (double)n : 1.0;
    }
    uoff += (int64_t)n * n;
  }
  const int64_t nfa = sh.faces_all();
  const int64_t total = face * nfa;
  const unsigned g = (unsigned)cdiv(4 * total, 256);  // 4 lanes per output
  // forward: mode products along trailing modes 2..d-1
  const void* src = bf.core;
  int src_real = 1;
  cplx* bufs[2] = {bf.cf0, bf.cf1};
  int cur = 0;
  int64_t st_lo = face;
  Trailing no_skip = sh.tr;
  no_skip.nt = 0;
  Trailing fwd_skip = sh.tr;  // last forward FFT product: mirrored faces are not needed
  if (kind != TR_TRANSFORM_FFT || getenv("TR_ALL_FACES") != nullptr) fwd_skip.nt = 0;
  for (int i = 0; i < nt; ++i) {
    const int n = (int)sh.tr.d[i];
    const int64_t hi = nfa / (st_lo / face) / n;
    mode_product(src, src_real, bufs[cur], 0, st_lo, n, hi, U[i], 0, 1.0, face,
                 i == nt - 1 ? fwd_skip : no_skip, g, st);
    src = bufs[cur];
    src_real = 0;
    cur ^= 1;
    st_lo *= n;
  }
  cplx* faces = (cplx*)src;
  // FFT: only canonical faces are factored (the rest are mirrored afterwards)
  Trailing mirror_tr = sh.tr;
  if (kind != TR_TRANSFORM_FFT || getenv("TR_ALL_FACES") != nullptr) mirror_tr.nt = 0;
  const size_t smem = (size_t)(face + sh.r1 * sh.r1) * sizeof(cplx);
  static bool attr = false;
  if (!attr) {
    TR_CUDA(cudaFuncSetAttribute(k_face_svt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * 64 * 64 * (int)sizeof(cplx)));
    attr = true;
  }
  bool mirror_done = false;
  if (sh.r0 > 64 || sh.r1 > 64) {
    // large faces (deterministic t-SVT of a whole tensor): X / V in global scratch,
    // X in the free mode-product buffer
    launch("face_svt", k_face_svt_g, (unsigned)nfa, 1024, (size_t)sh.r1 * sizeof(double), st,
           faces, bufs[cur], bf.fv, (int)sh.r0, (int)sh.r1, pen, tau, mirror_tr);
  } else if (sh.r0 <= 32 && sh.r1 <= 32 && getenv("TR_FACE_SVT_V") == nullptr) {
    // Tucker-core faces: 8 lanes per Jacobi pair, no V accumulation (core_svt.cuh)
    const size_t smem8 = (size_t)(2 * face + sh.r1 * sh.r1) * sizeof(cplx);
    static bool attr8 = false;
    if (!attr8) {
      TR_CUDA(cudaFuncSetAttribute(k_face_svt8<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   3 * 32 * 32 * (int)sizeof(cplx)));
      attr8 = true;
    }
    launch("face_svt", k_face_svt8<8>, (unsigned)nfa, 128, smem8, st, faces, (int)sh.r0,
           (int)sh.r1, pen, tau, mirror_tr);
    mirror_done = true;  // the kernel writes the conjugate-mirror faces itself
  } else {
    // one warp per Jacobi pair: no idle warps at the per-round barrier
    static const int fth_env = getenv("TR_FACE_THREADS") ? atoi(getenv("TR_FACE_THREADS")) : 0;
    const int npairs = (int)((sh.r1 + (sh.r1 & 1)) / 2);
    const int fth = fth_env > 0 ? fth_env : std::min(1024, std::max(128, 32 * npairs));
    launch("face_svt", k_face_svt, (unsigned)nfa, fth, smem, st, faces, (int)sh.r0, (int)sh.r1,
           pen, tau, mirror_tr);
  }
  if (kind == TR_TRANSFORM_FFT && !(mirror_done && mirror_tr.nt > 0))
    launch("mirror_fix", k_mirror_fix, g, 256, 0, st, faces, face, nfa, sh.tr);
  // inverse: U^H / alpha in reverse mode order, real part on the last step
  for (int i = nt - 1; i >= 0; --i) {
    const int n = (int)sh.tr.d[i];
    st_lo /= n;
    const int64_t hi = nfa / (st_lo / face) / n;
    const bool last = (i == 0);
    void* dst = last ? (void*)bf.core : (void*)bufs[cur];
    mode_product(src, 0, dst, last ? 1 : 0, st_lo, n, hi, U[i], 1, al[i], face, no_skip, g, st);
    src = dst;
    cur ^= 1;
  }
  TR_LAUNCH_CHECK();
  return 0;
}

// fp32 column-major rows x cols matrix, plain (unswizzled) boxes of box_rows x box_cols
static bool tmap_f32_plain(CUtensorMap* map, const float* base, int64_t rows, int64_t cols,
                           int box_rows, int box_cols) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  const cuuint64_t strides[1] = {(cuuint64_t)rows * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// out = F0 C1 on the tensor cores (expand_tc.cuh) when the shapes suit it
static bool expand_tc(const Shape& sh, Bufs<float>& bf, float* out, cudaStream_t st) {
  static const bool off = getenv("TR_NO_EXPAND_TC") != nullptr;
  static const bool direct = getenv("TR_EXPAND_DIRECT_STORE") != nullptr;
  const int64_t N = sh.n2 * sh.nf;
  if (off || sh.r0 > 32 || sh.n1 % 128 != 0 || N >= (1ll << 31) || sh.n1 >= (1ll << 31))
    return false;
  CUtensorMap ah, al, bh, bl, mo;
  if (!tmap_f32(&ah, bf.f0h, 32, sh.n1, 128) || !tmap_f32(&al, bf.f0l, 32, sh.n1, 128) ||
      !tmap_f32(&bh, bf.c1h, 32, N, 128) || !tmap_f32(&bl, bf.c1l, 32, N, 128) ||
      !tmap_f32_plain(&mo, out, sh.n1, N, 32, 32))
    return false;
  launch("expand_mode1", k_expand_mode1_split, (unsigned)(cdiv(sh.n2, 128) * sh.nf), 128, 0, st,
         (const double*)(bf.core + sh.r0 * sh.r1 * sh.f0), (int)sh.r0, (int)sh.r1, sh.nf,
         (const double*)bf.F1, sh.n2, bf.c1h, bf.c1l);
  launch("expand_split", k_split_rows, (unsigned)cdiv(sh.n1 * 32, 256), 256, 0, st,
         (const double*)bf.F0, sh.n1, (int)sh.r0, bf.f0h, bf.f0l);
  const int64_t nrb = sh.n1 / 128;
  // SMs left to the latency kernels (face SVT, Ritz, TSQR) of the other mode
  // chains while this HBM-write-bound pass runs (TR_EXPAND_RESERVE, default 32: 7.07 -> 7.01 ms per sweep)
  static const int ex_reserve = getenv("TR_EXPAND_RESERVE") ? atoi(getenv("TR_EXPAND_RESERVE")) : 32;
  const int64_t per = std::max<int64_t>(
      1, std::min<int64_t>(std::max(1, stream_sms() - ex_reserve) / nrb, cdiv(N, 128)));
  const size_t smem = (size_t)(direct ? kEtSmemBytes : kEtSmemBytesTs) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_expand_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kEtSmemBytes + 1024);
    cudaFuncSetAttribute(k_expand_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kEtSmemBytesTs + 1024);
    attr = true;
  }
  if (direct)
    launch("gemm_expand", k_expand_tc<false>, (unsigned)(per * nrb), kEtThreads, smem, st, ah, al,
           bh, bl, mo, sh.n1, N, out);
  else
    launch("gemm_expand", k_expand_tc<true>, (unsigned)(per * nrb), kEtThreads, smem, st, ah, al,
           bh, bl, mo, sh.n1, N, out);
  return true;
}

static bool expand_tc(const Shape&, Bufs<double>&, double*, cudaStream_t) { return false; }

template <typename T>
static int expand(const Shape& sh, Bufs<T>& bf, T* out, cudaStream_t st) {
  if (expand_tc(sh, bf, out, st)) {
    TR_LAUNCH_CHECK();
    return 0;
  }
  const int64_t N = sh.n2 * sh.nf;
  launch("expand_mode1", k_expand_mode1<T>, (unsigned)(cdiv(sh.n2, 128) * sh.nf), 128, 0, st,
         (const double*)(bf.core + sh.r0 * sh.r1 * sh.f0), (int)sh.r0, (int)sh.r1, sh.nf, bf.F1,
         sh.n2, bf.C1);
  constexpr int RA = 8, CB = sizeof(T) == 4 ? 16 : 8;
  const int64_t nrb = cdiv(sh.n1, 32 * RA);
  const int64_t kp = cdiv(sh.r0, 16 / (int64_t)sizeof(T)) * (16 / (int64_t)sizeof(T));
  const size_t smem = ((size_t)kp * 32 * RA + 2 * (size_t)kp * 8 * CB) * sizeof(T);
  static bool attr = false;
  if (!attr) {
    TR_CUDA(cudaFuncSetAttribute(k_gemm_expand<T, RA, CB>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)((64 * 32 * RA + 2 * 64 * 8 * CB) * sizeof(T))));
    attr = true;
  }
  // one resident CTA per SM, a whole number of CTAs per row block
  const int64_t per_rb = std::max<int64_t>(1, std::min<int64_t>(cdiv(N, 8 * CB), stream_sms() / nrb));
  launch("gemm_expand", k_gemm_expand<T, RA, CB>, (unsigned)(per_rb * nrb), 256, smem, st, bf.F0t,
         sh.n1, (int)sh.r0, bf.C1, N, out);
  TR_LAUNCH_CHECK();
  return 0;
}

template <typename T>
static int gnhtsvt_randomized_t(const void* a, void* out, const Shape& sh, uint64_t seed,
                                int kind, const void* mats, const double* alphas, Penalty pen,
                                double tau, const void* g0, const void* g1, void* ws,
                                int64_t ws_bytes, cudaStream_t st,
                                cudaEvent_t after_mode0 = nullptr, bool transform_built = false) {
  Carve cv(ws);
  Bufs<T> bf;
  carve<T>(cv, sh, bf);
  TR_REQUIRE(ws_bytes >= cv.off, "workspace too small: %lld < %lld", (long long)ws_bytes,
             (long long)cv.off);
  if (lrta_compress<T>((const T*)a, sh, seed, (const T*)g0, (const T*)g1, bf, st, after_mode0))
    return 2;
  if (core_svt<T>(sh, kind, (const cplx*)mats, alphas, pen, tau, bf, st, transform_built)) return 2;
  return expand<T>(sh, bf, (T*)out, st);
}

template <typename T>
static int rsthosvd_t(const void* a, const Shape& sh, uint64_t seed, const void* g0,
                      const void* g1, double* f0, double* f1, double* core, int64_t* reff,
                      void* ws, int64_t ws_bytes, cudaStream_t st) {
  Carve cv(ws);
  Bufs<T> bf;
  carve<T>(cv, sh, bf);
  TR_REQUIRE(ws_bytes >= cv.off, "workspace too small: %lld < %lld", (long long)ws_bytes,
             (long long)cv.off);
  if (lrta_compress<T>((const T*)a, sh, seed, (const T*)g0, (const T*)g1, bf, st)) return 2;
  TR_CUDA(cudaMemcpyAsync(f0, bf.F0, sizeof(double) * sh.n1 * sh.r0, cudaMemcpyDeviceToDevice, st));
  TR_CUDA(cudaMemcpyAsync(f1, bf.F1, sizeof(double) * sh.n2 * sh.r1, cudaMemcpyDeviceToDevice, st));
  TR_CUDA(cudaMemcpyAsync(core, bf.core, sizeof(double) * sh.r0 * sh.r1 * sh.nf,
                          cudaMemcpyDeviceToDevice, st));
  TR_CUDA(cudaMemcpyAsync(reff, bf.info + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  TR_CUDA(cudaMemcpyAsync(reff + 1, bf.info + 3, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  return 0;
}

template <typename T>
__global__ void k_prox(Penalty pen, double mu, const T* __restrict__ v, T* __restrict__ out,
                       int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (T)prox(pen, mu, (double)v[i]);
}

}  // namespace tr

#include "tucker.cuh"
#include "admm.cuh"

using namespace tr;

namespace {
struct AdmmHandle {
  int dtype;
  void* solver;
};
}  // namespace

extern "C" {

int tr_version(void) { return 100; }

const char* tr_last_error(void) { return g_err; }

int64_t tr_lrta_workspace(int dtype, int order, const int64_t* dims, const int64_t* ranks,
                          const int64_t* blocks, const int64_t* krylov) {
  Shape sh;
  if (make_shape(order, dims, ranks, blocks, krylov, sh)) return -1;
  Carve cv(nullptr);
  if (dtype == TR_F32) {
    Bufs<float> b;
    carve<float>(cv, sh, b);
  } else {
    Bufs<double> b;
    carve<double>(cv, sh, b);
  }
  return cv.off;
}

int tr_gnhtsvt_randomized(int dtype, const void* a, void* out, int order, const int64_t* dims,
                          const int64_t* ranks, const int64_t* blocks, const int64_t* krylov,
                          uint64_t seed, int transform_kind, const void* transform_mats,
                          const double* alphas, int penalty_kind, double p0, double p1,
                          double tau, const void* sketch0, const void* sketch1, void* workspace,
                          int64_t workspace_bytes, void* stream) {
  Shape sh;
  if (make_shape(order, dims, ranks, blocks, krylov, sh)) return 1;
  TR_REQUIRE(transform_kind >= 0 && transform_kind <= 2, "bad transform kind %d", transform_kind);
  TR_REQUIRE(transform_kind != TR_TRANSFORM_EXPLICIT || (transform_mats && alphas),
             "explicit transform needs matrices and alphas");
  TR_REQUIRE(penalty_kind >= 0 && penalty_kind <= 6, "bad penalty kind %d", penalty_kind);
  TR_REQUIRE(tau >= 0.0, "tau must be >= 0");
  TR_REQUIRE(a && out && workspace, "null pointer argument");
  Penalty pen{penalty_kind, p0, p1};
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == TR_F32)
    return gnhtsvt_randomized_t<float>(a, out, sh, seed, transform_kind, transform_mats, alphas,
                                       pen, tau, sketch0, sketch1, workspace, workspace_bytes, st);
  TR_REQUIRE(dtype == TR_F64, "bad dtype %d", dtype);
  return gnhtsvt_randomized_t<double>(a, out, sh, seed, transform_kind, transform_mats, alphas,
                                      pen, tau, sketch0, sketch1, workspace, workspace_bytes, st);
}

int tr_gnhtsvt_randomized_sharded(int dtype, const void* a, void* out, int order,
                                  const int64_t* dims, int64_t last_all, int64_t last_off,
                                  const int64_t* ranks, const int64_t* blocks,
                                  const int64_t* krylov, uint64_t seed, int transform_kind,
                                  const void* transform_mats, const double* alphas,
                                  int penalty_kind, double p0, double p1, double tau,
                                  tr_allreduce_fn allreduce, void* user, void* workspace,
                                  int64_t workspace_bytes, void* stream) {
  Shape sh;
  if (make_shape(order, dims, ranks, blocks, krylov, sh)) return 1;
  const int64_t last = dims[order - 1];
  TR_REQUIRE(last_all >= 1 && last_off >= 0 && last_off + last <= last_all,
             "shard [%lld, %lld) outside the last mode of length %lld", (long long)last_off,
             (long long)(last_off + last), (long long)last_all);
  TR_REQUIRE(transform_kind >= 0 && transform_kind <= 2, "bad transform kind %d", transform_kind);
  TR_REQUIRE(transform_kind != TR_TRANSFORM_EXPLICIT || (transform_mats && alphas),
             "explicit transform needs matrices and alphas");
  TR_REQUIRE(penalty_kind >= 0 && penalty_kind <= 6, "bad penalty kind %d", penalty_kind);
  TR_REQUIRE(tau >= 0.0, "tau must be >= 0");
  TR_REQUIRE(a && out && workspace, "null pointer argument");
  // faces = trailing modes flattened (last mode slowest): this rank owns a
  // contiguous block of them; the transform sees the global trailing dims
  const int64_t inner = sh.nf / last;
  sh.tr.d[order - 3] = last_all;
  sh.nf_all = inner * last_all;
  sh.f0 = inner * last_off;
  sh.coll = allreduce;
  sh.coll_user = user;
  Penalty pen{penalty_kind, p0, p1};
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == TR_F32)
    return gnhtsvt_randomized_t<float>(a, out, sh, seed, transform_kind, transform_mats, alphas,
                                       pen, tau, nullptr, nullptr, workspace, workspace_bytes, st);
  TR_REQUIRE(dtype == TR_F64, "bad dtype %d", dtype);
  return gnhtsvt_randomized_t<double>(a, out, sh, seed, transform_kind, transform_mats, alphas,
                                      pen, tau, nullptr, nullptr, workspace, workspace_bytes, st);
}

int tr_rsthosvd_bki(int dtype, const void* a, int order, const int64_t* dims,
                    const int64_t* ranks, const int64_t* blocks, const int64_t* krylov,
                    uint64_t seed, const void* sketch0, const void* sketch1, double* f0,
                    double* f1, double* core, int64_t* ranks_eff, void* workspace,
                    int64_t workspace_bytes, void* stream) {
  Shape sh;
  if (make_shape(order, dims, ranks, blocks, krylov, sh)) return 1;
  TR_REQUIRE(a && f0 && f1 && core && ranks_eff && workspace, "null pointer argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == TR_F32)
    return rsthosvd_t<float>(a, sh, seed, sketch0, sketch1, f0, f1, core, ranks_eff, workspace,
                             workspace_bytes, st);
  TR_REQUIRE(dtype == TR_F64, "bad dtype %d", dtype);
  return rsthosvd_t<double>(a, sh, seed, sketch0, sketch1, f0, f1, core, ranks_eff, workspace,
                            workspace_bytes, st);
}

static int admm_create_any(int dtype, int order, const int64_t* dims, int kind, const void* obs_a,
                   const void* obs_b, const uint8_t* mask, int nmodes, const int64_t* modes,
                   int structure, int phi_kind, double phi_p0, double phi_p1, int psi_kind,
                   double psi_p0, double psi_p1, double lam, double lam2, double mu0,
                   double mu_max, double growth, double alpha, double mcount, int randomized,
                   const int64_t* ranks, const int64_t* blocks, const int64_t* krylov,
                   uint64_t seed, int transform_kind, const void* transform_mats,
                   const double* alphas, void** handle,
                           const tr_comm* comm, int64_t last_all, int64_t last_off) {
  TR_REQUIRE(handle && dims && modes, "null pointer argument");
  TR_REQUIRE(kind >= 0 && kind <= 3, "bad solver kind %d", kind);
  TR_REQUIRE(structure >= 0 && structure <= 2, "bad shrink structure %d", structure);
  TR_REQUIRE(phi_kind >= 0 && phi_kind <= 6 && psi_kind >= 0 && psi_kind <= 6, "bad penalty kind");
  TR_REQUIRE(mu0 > 0 && growth > 1, "mu0 must be > 0 and growth > 1");
  TR_REQUIRE(kind >= 2 ? (obs_a && obs_b) : (obs_a && mask), "missing observations");
  TR_REQUIRE(transform_kind != TR_TRANSFORM_EXPLICIT || (transform_mats && alphas),
             "explicit transform needs matrices and alphas");
  AdmmConfig cfg{};
  cfg.kind = kind;
  cfg.structure = structure;
  cfg.phi = Penalty{phi_kind, phi_p0, phi_p1};
  cfg.psi = Penalty{psi_kind, psi_p0, psi_p1};
  cfg.lam = lam;
  cfg.lam2 = lam2;
  cfg.mu0 = mu0;
  cfg.mu_max = mu_max;
  cfg.growth = growth;
  cfg.alpha = alpha;
  cfg.mcount = mcount;
  cfg.nmodes = nmodes;
  for (int k = 0; k < nmodes && k < kMaxOrder; ++k) {
    TR_REQUIRE(modes[k] >= -1 && modes[k] < order, "gradient mode %lld out of range",
               (long long)modes[k]);
    cfg.modes[k] = (int)modes[k];
    for (int j = 0; j < k; ++j)
      TR_REQUIRE(modes[j] != modes[k], "gradient mode %lld repeated", (long long)modes[k]);
  }
  cfg.randomized = randomized;
  for (int i = 0; i < 2; ++i) {
    cfg.ranks[i] = ranks ? ranks[i] : 1;
    cfg.blocks[i] = blocks ? blocks[i] : 1;
    cfg.krylov[i] = krylov ? krylov[i] : 0;
  }
  cfg.seed = seed;
  cfg.tkind = transform_kind;
  cfg.tmats = transform_mats;
  for (int i = 0; i < 8; ++i) cfg.talphas[i] = (alphas && i < order - 2) ? alphas[i] : 1.0;
  auto* h = new AdmmHandle{dtype, nullptr};
  int rc;
  if (dtype == TR_F32) {
    Solver<float>* s = nullptr;
    rc = admm_create<float>(cfg, order, dims, obs_a, obs_b, mask, &s, comm, last_all, last_off);
    h->solver = s;
  } else {
    Solver<double>* s = nullptr;
    rc = admm_create<double>(cfg, order, dims, obs_a, obs_b, mask, &s, comm, last_all, last_off);
    h->solver = s;
  }
  if (rc) {
    delete h;
    return rc;
  }
  *handle = h;
  return 0;
}

int tr_admm_create(int dtype, int order, const int64_t* dims, int kind, const void* obs_a,
                   const void* obs_b, const uint8_t* mask, int nmodes, const int64_t* modes,
                   int structure, int phi_kind, double phi_p0, double phi_p1, int psi_kind,
                   double psi_p0, double psi_p1, double lam, double lam2, double mu0,
                   double mu_max, double growth, double alpha, double mcount, int randomized,
                   const int64_t* ranks, const int64_t* blocks, const int64_t* krylov,
                   uint64_t seed, int transform_kind, const void* transform_mats,
                   const double* alphas, void** handle) {
  return admm_create_any(dtype, order, dims, kind, obs_a, obs_b, mask, nmodes, modes, structure,
                         phi_kind, phi_p0, phi_p1, psi_kind, psi_p0, psi_p1, lam, lam2, mu0,
                         mu_max, growth, alpha, mcount, randomized, ranks, blocks, krylov, seed,
                         transform_kind, transform_mats, alphas, handle, nullptr, 0, 0);
}

int tr_admm_create_sharded(int dtype, int order, const int64_t* dims, int kind,
                           const void* obs_a, const uint8_t* mask, int nmodes,
                           const int64_t* modes, int phi_kind, double phi_p0, double phi_p1,
                           int psi_kind, double psi_p0, double psi_p1, double lam, double mu0,
                           double mu_max, double growth, const int64_t* ranks,
                           const int64_t* blocks, const int64_t* krylov, uint64_t seed,
                           int64_t last_all, int64_t last_off, const tr_comm* comm,
                           void** handle) {
  TR_REQUIRE(comm, "null communicator");
  TR_REQUIRE(kind == 0 || kind == 1, "the sharded solver runs GNRHTC (0) or GNHTC (1)");
  return admm_create_any(dtype, order, dims, kind, obs_a, nullptr, mask, nmodes, modes, 0,
                         phi_kind, phi_p0, phi_p1, psi_kind, psi_p0, psi_p1, lam, 0.0, mu0,
                         mu_max, growth, 0.0, 0.0, 1, ranks, blocks, krylov, seed,
                         TR_TRANSFORM_FFT, nullptr, nullptr, handle, comm, last_all, last_off);
}

int tr_admm_step(void* handle, double* out) {
  TR_REQUIRE(handle && out, "null pointer argument");
  auto* h = (AdmmHandle*)handle;
  if (h->dtype == TR_F32) return admm_step<float>(*(Solver<float>*)h->solver, out);
  return admm_step<double>(*(Solver<double>*)h->solver, out);
}

int tr_admm_lookahead(void* handle, int on) {
  TR_REQUIRE(handle, "null pointer argument");
  auto* h = (AdmmHandle*)handle;
  if (h->dtype == TR_F32) ((Solver<float>*)h->solver)->lookahead = on != 0;
  else ((Solver<double>*)h->solver)->lookahead = on != 0;
  return 0;
}

int tr_admm_read(void* handle, int which, void* dst, void* stream) {
  TR_REQUIRE(handle && dst, "null pointer argument");
  auto* h = (AdmmHandle*)handle;
  auto rd = [&](auto* s) -> int {
    using S = std::remove_pointer_t<decltype(s)>;
    const void* src = which == 0 ? (const void*)s->lold
                      : which == 1 ? (const void*)s->e
                      : which == 2 ? (const void*)s->y
                      : which == 3 ? (const void*)s->z
                                   : (const void*)s->gcur[which - 4];
    const size_t es = sizeof(*s->l);
    TR_CUDA(cudaStreamSynchronize(s->streams[0]));
    TR_CUDA(cudaMemcpyAsync(dst, src, es * s->g.N, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    (void)sizeof(S);
    return 0;
  };
  const int nm = h->dtype == TR_F32 ? ((Solver<float>*)h->solver)->cfg.nmodes
                                     : ((Solver<double>*)h->solver)->cfg.nmodes;
  TR_REQUIRE(which >= 0 && which < 4 + nm, "bad state index %d", which);
  if (h->dtype == TR_F32) return rd((Solver<float>*)h->solver);
  return rd((Solver<double>*)h->solver);
}

int tr_admm_set_sketch(void* handle, int sketch_mode, int nproc, const int64_t* proc_order,
                       const int64_t* ranks, const int64_t* blocks, const int64_t* krylov,
                       double eps, int64_t block, double defl_tol, uint64_t seed) {
  TR_REQUIRE(handle && (nproc == 0 || proc_order), "null pointer argument");
  TR_REQUIRE(sketch_mode == 0 || sketch_mode == 1, "sketch mode must be 0 (fixed-rank) or 1");
  TR_REQUIRE(nproc >= 0 && nproc <= kTuckerMaxOrder, "too many processed modes");
  auto* h = (AdmmHandle*)handle;
  TuckerSpec sp;
  sp.mode = sketch_mode;
  sp.nproc = nproc;
  for (int p = 0; p < nproc; ++p) {
    sp.proc[p] = (int)proc_order[p];
    if (sketch_mode == 0) {
      TR_REQUIRE(ranks && blocks && krylov, "fixed-rank sketching needs ranks, blocks and krylov");
      sp.ranks[p] = ranks[p];
      sp.blocks[p] = blocks[p];
      sp.krylov[p] = krylov[p];
    }
  }
  TR_REQUIRE(sketch_mode == 0 || (eps > 0 && eps < 1 && block >= 1), "bad fixed-accuracy sketch");
  sp.eps = eps;
  sp.block = block;
  sp.defl_tol = defl_tol;
  sp.seed = seed;
  auto set = [&](auto* s) -> int {
    for (int p = 0; p < nproc; ++p)
      TR_REQUIRE(sp.proc[p] >= 0 && sp.proc[p] < s->order, "processing order entry out of range");
    s->tspec = sp;
    s->generic = true;
    return 0;
  };
  if (h->dtype == TR_F32) return set((Solver<float>*)h->solver);
  return set((Solver<double>*)h->solver);
}

void* tr_admm_stream(void* handle) {
  if (!handle) return nullptr;
  auto* h = (AdmmHandle*)handle;
  if (h->dtype == TR_F32) return (void*)((Solver<float>*)h->solver)->streams[0];
  return (void*)((Solver<double>*)h->solver)->streams[0];
}

int tr_admm_destroy(void* handle) {
  if (!handle) return 0;
  auto* h = (AdmmHandle*)handle;
  cudaDeviceSynchronize();
  if (h->dtype == TR_F32) delete (Solver<float>*)h->solver;
  else delete (Solver<double>*)h->solver;
  delete h;
  return 0;
}

// ---------------------------------------------------------------------------
// generic Tucker engine (tucker.cuh)
// ---------------------------------------------------------------------------
namespace {
struct TuckerHandle {
  int dtype;
  tr::TuckerResult res;
};
}  // namespace

int tr_tucker_create(int dtype, const void* a, int order, const int64_t* dims, int sketch_mode,
                     int nproc, const int64_t* proc_order, const int64_t* ranks,
                     const int64_t* blocks, const int64_t* krylov, double eps, int64_t block,
                     double defl_tol, uint64_t seed, void* stream, void** handle) {
  TR_REQUIRE(a && dims && handle && (nproc == 0 || proc_order), "null pointer argument");
  TR_REQUIRE(dtype == TR_F32 || dtype == TR_F64, "dtype must be TR_F32 or TR_F64");
  TR_REQUIRE(order >= 1 && order <= kTuckerMaxOrder, "order must be in [1, %d]", kTuckerMaxOrder);
  TR_REQUIRE(sketch_mode == 0 || sketch_mode == 1, "sketch mode must be 0 (fixed-rank) or 1");
  TR_REQUIRE(nproc >= 0 && nproc <= kTuckerMaxOrder, "too many processed modes");
  for (int i = 0; i < order; ++i) TR_REQUIRE(dims[i] >= 1, "empty tensors are not supported");
  TuckerSpec sp;
  sp.mode = sketch_mode;
  sp.nproc = nproc;
  for (int p = 0; p < nproc; ++p) {
    TR_REQUIRE(proc_order[p] >= 0 && proc_order[p] < order, "processing order entry %lld out of range",
               (long long)proc_order[p]);
    sp.proc[p] = (int)proc_order[p];
    if (sketch_mode == 0) {
      TR_REQUIRE(ranks && blocks && krylov, "fixed-rank sketching needs ranks, blocks and krylov");
      sp.ranks[p] = ranks[p];
      sp.blocks[p] = blocks[p];
      sp.krylov[p] = krylov[p];
      TR_REQUIRE(ranks[p] >= 1 && ranks[p] <= dims[proc_order[p]], "rank %lld out of range for mode %lld",
                 (long long)ranks[p], (long long)proc_order[p]);
      TR_REQUIRE(blocks[p] >= 1 && blocks[p] <= ranks[p], "block size must satisfy 1 <= b <= r");
      TR_REQUIRE((krylov[p] + 1) * blocks[p] >= ranks[p], "(q+1)*b < rank");
    }
  }
  if (sketch_mode == 1) {
    TR_REQUIRE(eps > 0 && eps < 1, "eps must lie in (0, 1)");
    TR_REQUIRE(block >= 1, "block size must be >= 1");
  }
  sp.eps = eps;
  sp.block = block;
  sp.defl_tol = defl_tol;
  sp.seed = seed;
  auto* h = new TuckerHandle{dtype, {}};
  cudaStream_t st = (cudaStream_t)stream;
  const int rc = dtype == TR_F32
                     ? tucker_compress<float>((const float*)a, order, dims, sp, h->res, st)
                     : tucker_compress<double>((const double*)a, order, dims, sp, h->res, st);
  if (rc) {
    delete h;
    return rc;
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    delete h;
    TR_CUDA(e);
  }
  *handle = h;
  return 0;
}

int tr_tucker_info(void* handle, int64_t* core_dims, int64_t* ranks, int64_t* processed,
                   double* energy, int64_t* deflations, int64_t* iterations, double* orth_loss) {
  TR_REQUIRE(handle, "null handle");
  const TuckerResult& r = ((TuckerHandle*)handle)->res;
  for (int i = 0; i < r.order; ++i) {
    if (core_dims) core_dims[i] = r.cdims[i];
    if (ranks) ranks[i] = r.processed[i] ? r.ranks[i] : r.dims[i];
    if (processed) processed[i] = r.processed[i] ? 1 : 0;
    if (energy) energy[i] = r.energy[i];
    if (deflations) deflations[i] = r.deflations[i];
    if (iterations) iterations[i] = r.iterations[i];
    if (orth_loss) orth_loss[i] = r.orth_loss[i];
  }
  return 0;
}

int tr_tucker_read(void* handle, int which, double* dst, void* stream) {
  TR_REQUIRE(handle && dst, "null pointer argument");
  const TuckerResult& r = ((TuckerHandle*)handle)->res;
  cudaStream_t st = (cudaStream_t)stream;
  if (which < 0) {
    const int64_t n = r.core_size();
    if (n > 0 && r.core) TR_CUDA(cudaMemcpyAsync(dst, r.core, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    return 0;
  }
  TR_REQUIRE(which < r.order && r.processed[which], "mode %d was not processed", which);
  const int64_t n = r.dims[which] * r.ranks[which];
  if (n > 0 && r.factors[which])
    TR_CUDA(cudaMemcpyAsync(dst, r.factors[which], sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  return 0;
}

int tr_tucker_svt(void* handle, int transform_kind, const void* transform_mats,
                  const double* alphas, int penalty_kind, double p0, double p1, double tau,
                  void* out, void* stream) {
  TR_REQUIRE(handle && out, "null pointer argument");
  TR_REQUIRE(transform_kind >= 0 && transform_kind <= 2, "bad transform kind %d", transform_kind);
  TR_REQUIRE(transform_kind != TR_TRANSFORM_EXPLICIT || (transform_mats && alphas),
             "explicit transform needs matrices and alphas");
  TR_REQUIRE(penalty_kind >= 0 && penalty_kind <= 6, "bad penalty kind %d", penalty_kind);
  TR_REQUIRE(tau >= 0.0, "tau must be >= 0");
  auto* h = (TuckerHandle*)handle;
  const TuckerResult& r = h->res;
  TR_REQUIRE(r.order >= 3, "tensor order %d < required 3", r.order);
  cudaStream_t st = (cudaStream_t)stream;
  int64_t N = 1;
  for (int i = 0; i < r.order; ++i) N *= r.dims[i];
  const size_t es = h->dtype == TR_F32 ? 4 : 8;
  const int64_t nc = r.core_size();
  if (nc == 0) {  // rank-0 structure: zeros (sketch.py:453-454)
    TR_CUDA(cudaMemsetAsync(out, 0, es * N, st));
    return 0;
  }
  double* work = nullptr;
  TR_CUDA(cudaMallocAsync((void**)&work, sizeof(double) * nc, st));
  int rc = 0;
  if (cudaMemcpyAsync(work, r.core, sizeof(double) * nc, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    rc = 2;
  Penalty pen{penalty_kind, p0, p1};
  if (!rc)
    rc = h->dtype == TR_F32
             ? tucker_core_svt<float>(r, work, transform_kind, transform_mats, alphas, pen, tau, st)
             : tucker_core_svt<double>(r, work, transform_kind, transform_mats, alphas, pen, tau, st);
  if (!rc)
    rc = h->dtype == TR_F32 ? tucker_reconstruct<float>(r, work, (float*)out, st)
                            : tucker_reconstruct<double>(r, work, (double*)out, st);
  cudaFreeAsync(work, st);
  return rc;
}

int tr_tucker_destroy(void* handle) {
  if (!handle) return 0;
  auto* h = (TuckerHandle*)handle;
  cudaStreamSynchronize(h->res.st);
  delete h;
  return 0;
}

int tr_gradsys_create(int dtype, int order, const int64_t* dims, int nmodes, const int* modes,
                      void** handle) {
  TR_REQUIRE(dtype == TR_F32 || dtype == TR_F64, "dtype must be TR_F32 or TR_F64");
  TR_REQUIRE(dims && modes && handle, "null pointer argument");
  auto* h = new AdmmHandle{dtype, nullptr};
  int rc;
  if (dtype == TR_F32) {
    Solver<float>* s = nullptr;
    rc = gradsys_create<float>(order, dims, nmodes, modes, &s);
    h->solver = s;
  } else {
    Solver<double>* s = nullptr;
    rc = gradsys_create<double>(order, dims, nmodes, modes, &s);
    h->solver = s;
  }
  if (rc) {
    delete h;
    return rc;
  }
  *handle = h;
  return 0;
}

int tr_gradsys_solve(void* handle, const void* b, const void* const* grads, void* out,
                     void* stream) {
  TR_REQUIRE(handle && b && grads && out, "null pointer argument");
  auto* h = (AdmmHandle*)handle;
  if (h->dtype == TR_F32)
    return gradsys_solve<float>(*(Solver<float>*)h->solver, (const float*)b,
                                (const float* const*)grads, (float*)out, (cudaStream_t)stream);
  return gradsys_solve<double>(*(Solver<double>*)h->solver, (const double*)b,
                               (const double* const*)grads, (double*)out, (cudaStream_t)stream);
}

int tr_gradsys_destroy(void* handle) { return tr_admm_destroy(handle); }

int tr_prox(int dtype, int penalty_kind, double p0, double p1, double mu, const void* v,
            void* out, int64_t n, void* stream) {
  TR_REQUIRE(penalty_kind >= 0 && penalty_kind <= 6, "bad penalty kind %d", penalty_kind);
  TR_REQUIRE(mu >= 0.0, "prox level mu must be >= 0");
  if (n <= 0) return 0;
  Penalty pen{penalty_kind, p0, p1};
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned g = (unsigned)cdiv(n, 256);
  if (dtype == TR_F32) launch("prox", k_prox<float>, g, 256, 0, st, pen, mu, (const float*)v, (float*)out, n);
  else launch("prox", k_prox<double>, g, 256, 0, st, pen, mu, (const double*)v, (double*)out, n);
  TR_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// launch accounting / profiling (used by bench.py)
// ---------------------------------------------------------------------------
extern "C" {

int64_t tr_launch_count(void) { return (int64_t)tr::profiler().launches.load(); }

int tr_profile_enable(int on) {
  tr::Profiler& p = tr::profiler();
  std::lock_guard<std::mutex> g(p.mu);
  for (auto& r : p.records) {
    p.pool.push_back(r.a);
    p.pool.push_back(r.b);
  }
  p.records.clear();
  p.enabled = on != 0;
  return 0;
}

// Per-launch timeline of the recorded region (not cleared): category names
// ('\n'-joined), start / end in ms relative to the first launch, stream handle.
int tr_profile_timeline(char* names, int64_t names_len, double* t0, double* t1, int64_t* streams,
                        int max_entries) {
  tr::Profiler& p = tr::profiler();
  std::lock_guard<std::mutex> g(p.mu);
  std::string joined;
  int n = 0;
  for (auto& r : p.records) {
    if (n >= max_entries) break;
    TR_CUDA(cudaEventSynchronize(r.b));
    float a = 0.f, b = 0.f;
    TR_CUDA(cudaEventElapsedTime(&a, p.records[0].a, r.a));
    TR_CUDA(cudaEventElapsedTime(&b, p.records[0].a, r.b));
    t0[n] = a;
    t1[n] = b;
    streams[n] = (int64_t)(uintptr_t)r.st;
    joined += r.cat;
    joined += '\n';
    ++n;
  }
  if ((int64_t)joined.size() + 1 > names_len) return -1;
  memcpy(names, joined.c_str(), joined.size() + 1);
  return n;
}

int tr_profile_read(char* names, int64_t names_len, double* ms, int64_t* counts,
                    int max_entries) {
  tr::Profiler& p = tr::profiler();
  std::lock_guard<std::mutex> g(p.mu);
  std::vector<std::string> cats;
  std::vector<double> tot;
  std::vector<int64_t> cnt;
  for (auto& r : p.records) {
    TR_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    TR_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    size_t i = 0;
    while (i < cats.size() && cats[i] != r.cat) ++i;
    if (i == cats.size()) {
      cats.emplace_back(r.cat);
      tot.push_back(0.0);
      cnt.push_back(0);
    }
    tot[i] += t;
    cnt[i] += 1;
    p.pool.push_back(r.a);
    p.pool.push_back(r.b);
  }
  p.records.clear();
  std::string joined;
  int n = 0;
  for (size_t i = 0; i < cats.size() && n < max_entries; ++i, ++n) {
    ms[n] = tot[i];
    counts[n] = cnt[i];
    joined += cats[i];
    joined += '\n';
  }
  if (names && names_len > 0) {
    strncpy(names, joined.c_str(), (size_t)names_len - 1);
    names[names_len - 1] = 0;
  }
  return n;
}

}  // extern "C"
