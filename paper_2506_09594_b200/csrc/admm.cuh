// Native ADMM solvers: GNRHTC / GNHTC (tenrec/solvers.py:204-295) and
// GNOBHTC / GNOBRHTC (tenrec/onebit.py:141-234).
//
// A Solver owns every device buffer of one run.  tr_admm_step() executes one
// ADMM sweep on the device and returns the Eq. (24) residuals to the host (the
// only host synchronisation per iteration); the convergence decision and the
// report bookkeeping stay in the Python host, mirroring the reference loop.
// The low-rank step runs one randomized t-SVT per gradient mode, each on its
// own stream with its own workspace, so the modes overlap on the GPU.
#pragma once

#include <initializer_list>
#include <limits>
#include <vector>

#include "admm_kernels.cuh"
#include "fft.cuh"

namespace tr {

struct AdmmConfig {
  int kind;        // 0 gnrhtc, 1 gnhtc, 2 gnobhtc, 3 gnobrhtc
  int structure;   // 0 entry, 1 tube, 2 slice
  Penalty phi, psi;
  double lam, lam2, mu0, mu_max, growth, alpha, mcount;
  int nmodes;
  int modes[kMaxOrder];  // -1 = identity chain
  int randomized;
  int64_t ranks[2], blocks[2], krylov[2];
  uint64_t seed;
  int tkind;
  const void* tmats;
  double talphas[8];
};

// Solver buffers come from the device's stream-ordered pool with an unbounded
// release threshold: memory freed by one solve stays reserved for the next, so
// create/destroy of a multi-GB solver costs microseconds after the first run.
// Allocation is ordered on the legacy stream; admm_create synchronises it
// before the buffers are used on the solver's own streams.
static int pool_alloc(void** p, size_t bytes) {
  static bool ready[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !ready[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    ready[dev] = true;
  }
  if (cudaMallocAsync(p, bytes, 0) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  return 0;
}

template <typename T>
struct Solver {
  AdmmConfig cfg;
  Geom g;
  Shape sh;  // LRTA shape (ranks = sketch ranks, or full faces when deterministic)
  int order;
  const T *A, *B;  // mobs / (j1, j2)
  const uint8_t* mask;
  T *l, *lold, *e, *y, *z, *zold, *rhs;
  std::vector<T*> gcur, gnew, lag, X;
  std::vector<T*> lag2;     // second multiplier buffer of the fused sweep tail
  bool rhs_ready = false;   // rhs already holds this sweep's L right-hand side
  // Lookahead (tr_admm_lookahead): the L-solve and the t-SVT inputs of the next
  // sweep are enqueued before the host waits for this sweep's residuals, so the
  // GPU never idles across the host's read-back / stopping test.  They touch
  // only buffers the returned state does not live in (the free L buffer, the
  // spectrum, the t-SVT inputs); a solve that stops simply leaves them unused.
  bool lookahead = false;
  bool head_done = false;   // this sweep's L-solve and t-SVT inputs are already enqueued
  cudaEvent_t ev_res = nullptr;
  cpx<T>* spec = nullptr;
  std::vector<cpx<T>*> tw;
  double* lam = nullptr;
  double* scale = nullptr;
  double *part = nullptr, *res = nullptr, *hres = nullptr;
  std::vector<void*> ws;
  int64_t ws_bytes = 0;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> evs;
  std::vector<cudaEvent_t> evs_mid;  // per mode: the passes over the whole tensor are done
  std::vector<char> tf_built;        // per mode: transform matrices live in its workspace
  cudaEvent_t ev_main = nullptr;
  SolveSpec ss;
  bool generic = false;  // low-rank step through the generic Tucker engine (tucker.cuh)
  TuckerSpec tspec;
  double mu;
  int64_t red_blocks;
  std::vector<void*> allocs;
  // multi-GPU: this rank holds faces [last_off, last_off + nl) of the last axis
  // (length last_all); stencils along it read ghost faces (Geom::halo), the FFT
  // solve transposes the last axis in with an all-to-all (fft_solve_dist), the
  // t-SVTs all-reduce their Krylov blocks / Gram / core (lrta.cu), and the
  // Eq. (24) residuals are all-reduced before they reach the host.
  bool sharded = false;
  tr_comm comm{};
  int64_t last_all = 0, last_off = 0, nl = 0, face = 0;
  cpx<T>* spec_pack = nullptr;
  cpx<T>* spec_recv = nullptr;
  double* res_max = nullptr;
  double* hres_max = nullptr;

  template <typename X_>
  X_* alloc(int64_t n) {
    void* p = nullptr;
    if (pool_alloc(&p, std::max<int64_t>(n, 1) * sizeof(X_))) return nullptr;
    allocs.push_back(p);
    return (X_*)p;
  }
  // N own elements plus a ghost face on each side when sharded (pointer to own
  // element 0)
  T* alloc_ghosted(int64_t n) {
    if (!sharded) return alloc<T>(n);
    T* p = alloc<T>(n + 2 * face);
    return p ? p + face : nullptr;
  }
  ~Solver() {
    for (void* p : allocs) cudaFreeAsync(p, 0);
    if (hres) cudaFreeHost(hres);
    if (hres_max) cudaFreeHost(hres_max);
    for (auto s : streams) cudaStreamDestroy(s);
    for (auto e : evs) cudaEventDestroy(e);
    for (auto e : evs_mid) cudaEventDestroy(e);
    if (ev_main) cudaEventDestroy(ev_main);
    if (ev_res) cudaEventDestroy(ev_res);
  }
  bool onebit() const { return cfg.kind >= 2; }
};

template <typename T>
static int64_t grid_for(int64_t n) {
  return std::max<int64_t>(1, std::min<int64_t>(cdiv(n, kRedThreads), (int64_t)num_sms() * 8));
}

// Resident grid of a line kernel (SMs x occupancy, capped by grid_for): all
// blocks run concurrently, which the stencil kernels rely on for L2 reuse.
template <typename K>
static unsigned resident_grid(K kernel, int64_t n) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kRedThreads, 0);
  const int64_t cap = grid_for<float>(n);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cap, (int64_t)std::max(per_sm, 1) * num_sms()));
}

// forward FFT over all axes, diagonal solve in the last-axis pass, inverse FFT
// Spectrum geometry: half spectrum along axis 0 (n0/2+1 bins) when n0 is even
// (real-to-complex first pass), the full complex spectrum otherwise.
struct SpecGeom {
  bool half;
  int64_t dims[kMaxOrder], st[kMaxOrder], N;
};

static SpecGeom spec_geom(const Geom& g) {
  SpecGeom sg;
  sg.half = g.dims[0] % 2 == 0 && g.dims[0] >= 2;
  sg.N = 1;
  for (int a = 0; a < g.d; ++a) {
    sg.dims[a] = (a == 0 && sg.half) ? g.dims[0] / 2 + 1 : g.dims[a];
    sg.st[a] = sg.N;
    sg.N *= sg.dims[a];
  }
  return sg;
}

template <typename T>
using FftTileKernel = void (*)(const void*, void*, int, double, int64_t, int, int64_t, int64_t,
                               const cpx<T>*, int, SolveSpec, const double*, int64_t);

// k_fft_t instance for a 2^ln-point line (tile of 2048 points), or null
template <typename T>
static FftTileKernel<T> fft_tile_kernel(int ln) {
  switch (ln) {
    case 7: return k_fft_t<T, 7, 4>;
    case 8: return k_fft_t<T, 8, 3>;
    case 9: return k_fft_t<T, 9, 2>;
    case 10: return k_fft_t<T, 10, 1>;
    case 11: return k_fft_t<T, 11, 0>;
    default: return nullptr;
  }
}

// One persistent power-of-two pass (nt = points per line, 8 <= nt <= 2048):
// the compile-time specialised kernel when the tile holds exactly 2048
// points, the runtime-shaped k_fft_p2 otherwise.  Grid = resident CTAs.
// k_fft4_real for the axis-0 real passes of a 1024-point first mode (swapped
// half-spectrum layout); false otherwise
template <typename T, int MINB>
static void fft4_real_launch(int mode, const void* in, void* dst, double scale, int64_t lines,
                             int64_t tr_n1, const cpx<T>* tw, cudaStream_t st) {
  const size_t smem = (size_t)fft4_smem_cpx<32>() * sizeof(cpx<T>);
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(k_fft4_real<T, 16, 32, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fft4_real<T, 16, 32, MINB>, 256,
                                                  smem);
    per_sm = std::max(per_sm, 1);
  }
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(lines, 16), (int64_t)per_sm * num_sms());
  launch("fft", k_fft4_real<T, 16, 32, MINB>, grid, 256, smem, st, in, dst, mode, scale, lines,
         tr_n1, tw);
}

template <typename T>
static void fft_pass_p2(int mode, const void* in, void* dst, double scale, int64_t stv, int n,
                        int64_t hi, const cpx<T>* tw, int inverse, const SolveSpec& ss,
                        const double* lam, int64_t tr_n1, cudaStream_t st) {
  static const bool no4 = getenv("TR_NO_FFT4") != nullptr || getenv("TR_NO_FFT4_REAL") != nullptr;
  static const int mb = getenv("TR_FFT4R_MINB") ? atoi(getenv("TR_FFT4R_MINB")) : 2;
  if (!no4 && mode != FFT_C2C && n == 1024 && tr_n1 > 0 && stv == 1 && !ss.active) {
    if (mb == 2) fft4_real_launch<T, 2>(mode, in, dst, scale, hi, tr_n1, tw, st);
    else fft4_real_launch<T, 1>(mode, in, dst, scale, hi, tr_n1, tw, st);
    return;
  }
  const int nt = mode == FFT_C2C ? n : n / 2;
  int ln = 0;
  while ((1 << ln) < nt) ++ln;
  const int64_t cap = std::min<int64_t>(std::min<int64_t>(16, 2048 / nt), stv == 1 ? hi : stv);
  int lL = 0;
  while ((2ll << lL) <= cap) ++lL;  // largest power of two <= cap
  const int64_t L = 1ll << lL;
  const int64_t ntiles = stv == 1 ? cdiv(hi, L) : hi * cdiv(stv, L);
  static bool generic_only = getenv("TR_FFT_GENERIC") != nullptr;
  static int occ[13] = {0};  // resident CTAs per SM, per specialised ln (index 12: k_fft_p2)
  FftTileKernel<T> tk = (L * nt == 2048 && !generic_only) ? fft_tile_kernel<T>(ln) : nullptr;
  const size_t smem = tk ? ((size_t)nt + kFftRtwSlots(nt) + 2 * (size_t)kFftTileSlots) * sizeof(cpx<T>)
                         : ((size_t)nt + 2 * (size_t)L * (nt + 1)) * sizeof(cpx<T>);
  const int slot = tk ? ln : 12;
  if (occ[slot] == 0) {
    const void* f = tk ? (const void*)tk : (const void*)k_fft_p2<T>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, f, 256, tk ? smem : 200 * 1024);
    occ[slot] = std::max(1, b);
  }
  // k_fft_p2 smem varies per call: size its grid from this call's footprint
  int per_sm = occ[slot];
  if (!tk) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_fft_p2<T>, 256, smem);
    per_sm = std::max(1, b);
  }
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)per_sm * num_sms());
  if (tk) {
    launch("fft", tk, (unsigned)grid, 256, smem, st, in, dst, mode, scale, stv, n, hi, ntiles, tw,
           inverse, ss, lam, tr_n1);
  } else {
    launch("fft", k_fft_p2<T>, (unsigned)grid, 256, smem, st, in, dst, mode, scale, stv, n, hi, lL,
           ntiles, tw, inverse, ss, lam, tr_n1);
  }
}

// k_fft_reg for a short power-of-two axis with a wide lo stride; false otherwise
template <typename T>
static bool fft_reg(const cpx<T>* tw, const double* lam, void* data, int n, int64_t stv,
                    int64_t hi, int inverse, const SolveSpec& ss, cudaStream_t st) {
  static const bool off = getenv("TR_NO_FFT_REG") != nullptr;
  if (off || stv < 32 || n > 32 || n < 2 || (n & (n - 1)) != 0) return false;
  const unsigned grid = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>(cdiv(stv * hi, 256), 16ll * num_sms()));
  cpx<T>* d = (cpx<T>*)data;
#define TR_FR(NN) launch("fft", k_fft_reg<T, NN>, grid, 256, 0, st, d, stv, hi, tw, inverse, ss, lam)
  switch (n) {
    case 2: TR_FR(2); break;
    case 4: TR_FR(4); break;
    case 8: TR_FR(8); break;
    case 16: TR_FR(16); break;
    default: TR_FR(32); break;
  }
#undef TR_FR
  return true;
}

// forward FFT over all axes, diagonal solve in the last-axis pass, inverse FFT
template <typename T>
static int fft_solve(Solver<T>& s, const T* rhs, T* out, cudaStream_t st) {
  const Geom& g = s.g;
  const SpecGeom sg = spec_geom(g);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_axis<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  // mode: FFT_C2C on spectrum axis a, or FFT_R2C / FFT_C2R on axis 0
  auto pass = [&](int a, int mode, const void* in, void* dst, double scale, int inverse,
                  SolveSpec ss) -> int {
    const int n = (int)g.dims[a];
    const int nt = mode == FFT_C2C ? n : n / 2;
    const int64_t stv = mode == FFT_C2C ? sg.st[a] : 1;
    const int64_t hi = mode == FFT_C2C ? sg.N / (stv * n) : g.N / n;
    const bool pow2 = (nt & (nt - 1)) == 0;
    if (mode == FFT_C2C && in == dst &&
        fft_reg<T>((const cpx<T>*)s.tw[a], s.lam, dst, n, stv, hi, inverse, ss, st))
      return 0;
    // persistent double-buffered kernel: pow2, <= 2048-point tiles, 16B-aligned real lines
    const bool persistent = pow2 && nt >= 8 && nt <= 2048 &&
                            (mode != FFT_R2C || (n * (int64_t)sizeof(T)) % 16 == 0) &&
                            getenv("TR_FFT_SIMPLE") == nullptr;
    if (persistent) {
      fft_pass_p2<T>(mode, in, dst, scale, stv, n, hi, (const cpx<T>*)s.tw[a], inverse, ss,
                     (const double*)s.lam, 0, st);
      return 0;
    }
    // at most 4096 complex line elements per CTA (8 radix-2 groups per thread)
    int64_t L = std::max<int64_t>(1, std::min<int64_t>(16, 4096 / nt));
    L = std::min<int64_t>(L, stv == 1 ? hi : stv);
    TR_REQUIRE(nt <= 4096, "FFT axis of length %d exceeds the 4096-point tile", n);
    const int64_t grid = stv == 1 ? cdiv(hi, L) : hi * cdiv(stv, L);
    const size_t smem = ((size_t)nt + (size_t)L * nt * (pow2 ? 1 : 2)) * sizeof(cpx<T>);
    TR_REQUIRE(smem <= 200 * 1024, "FFT axis of length %d too long for one tile", n);
    launch("fft", k_fft_axis<T>, (unsigned)grid, 256, smem, st, in, dst, mode, scale, stv, n, hi,
           (int)L, (const cpx<T>*)s.tw[a], inverse, ss, (const double*)s.lam);
    return 0;
  };
  SolveSpec off = s.ss, on = s.ss;
  off.active = 0;
  on.active = 1;
  for (int a = 0; a < g.d; ++a) off.dims[a] = on.dims[a] = sg.dims[a];
  const int d = g.d;
  const unsigned eg = (unsigned)grid_for<T>(sg.N);
  if (sg.half) {
    if (pass(0, FFT_R2C, rhs, s.spec, 1.0, 0, off)) return 1;
  } else {
    launch("fft", k_real_to_cpx<T>, eg, kRedThreads, 0, st, rhs, s.spec, g.N);
    if (pass(0, FFT_C2C, s.spec, s.spec, 1.0, 0, off)) return 1;
  }
  for (int a = 1; a < d - 1; ++a)
    if (pass(a, FFT_C2C, s.spec, s.spec, 1.0, 0, off)) return 1;
  if (pass(d - 1, FFT_C2C, s.spec, s.spec, 1.0, 0, on)) return 1;
  for (int a = d - 2; a >= 1; --a)
    if (pass(a, FFT_C2C, s.spec, s.spec, 1.0, 1, off)) return 1;
  if (sg.half) {
    // unnormalised inverses contribute (n0/2) prod_{a>0} n_a = N / 2
    if (pass(0, FFT_C2R, s.spec, out, 2.0 / (double)g.N, 1, off)) return 1;
  } else {
    if (pass(0, FFT_C2C, s.spec, s.spec, 1.0, 1, off)) return 1;
    launch("fft", k_cpx_to_real<T>, eg, kRedThreads, 0, st, (const cpx<T>*)s.spec, out, g.N,
           1.0 / (double)g.N);
  }
  TR_LAUNCH_CHECK();
  return 0;
}

// One C2C pass along a spectrum axis of length n (lo-stride stv, hi lines of
// lines); persistent power-of-two kernel when possible, generic otherwise.
// k_fft4 (four-step register FFT) for 256..1024-point contiguous lines or
// 128..256-point strided lines; false otherwise
template <typename T, int P, int N2, bool STRIDED, int MINB>
static void fft4_launch(const cpx<T>* tw, const double* lam, void* data, int64_t stv, int64_t hi,
                        int inverse, const SolveSpec& ss, cudaStream_t st) {
  const size_t smem = (size_t)fft4_smem_cpx<N2>() * sizeof(cpx<T>);
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(k_fft4<T, P, N2, STRIDED, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fft4<T, P, N2, STRIDED, MINB>, 256,
                                                  smem);
    per_sm = std::max(per_sm, 1);
  }
  const int64_t nlines = STRIDED ? stv * hi : hi;
  const int64_t ntiles = cdiv(nlines, 256 / P);
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)per_sm * num_sms());
  launch("fft", k_fft4<T, P, N2, STRIDED, MINB>, grid, 256, smem, st, (cpx<T>*)data, stv, hi, tw,
         inverse, ss, lam);
}

template <typename T>
static bool fft4(const cpx<T>* tw, const double* lam, void* data, int n, int64_t stv, int64_t hi,
                 int inverse, const SolveSpec& ss, cudaStream_t st) {
  static const bool off = getenv("TR_NO_FFT4") != nullptr;
  static const int mb = getenv("TR_FFT4_MINB") ? atoi(getenv("TR_FFT4_MINB")) : 2;
  if (off) return false;
  if (stv == 1 && !ss.active) {
    switch (n) {
      case 256: fft4_launch<T, 16, 16, false, 2>(tw, lam, data, stv, hi, inverse, ss, st); return true;
      case 512: fft4_launch<T, 16, 32, false, 1>(tw, lam, data, stv, hi, inverse, ss, st); return true;
      case 1024:
        if (mb == 2) fft4_launch<T, 32, 32, false, 2>(tw, lam, data, stv, hi, inverse, ss, st);
        else fft4_launch<T, 32, 32, false, 1>(tw, lam, data, stv, hi, inverse, ss, st);
        return true;
      default: return false;
    }
  }
  if (stv >= 32) {
    switch (n) {
      case 64: fft4_launch<T, 4, 16, true, 2>(tw, lam, data, stv, hi, inverse, ss, st); return true;
      case 128: fft4_launch<T, 8, 16, true, 2>(tw, lam, data, stv, hi, inverse, ss, st); return true;
      case 256: fft4_launch<T, 8, 32, true, 1>(tw, lam, data, stv, hi, inverse, ss, st); return true;
      default: return false;
    }
  }
  return false;
}

template <typename T>
static int fft_c2c(const cpx<T>* tw, const double* lam, void* data, int n, int64_t stv, int64_t hi,
                   int inverse, const SolveSpec& ss, cudaStream_t st) {
  if (fft_reg<T>(tw, lam, data, n, stv, hi, inverse, ss, st)) return 0;
  if (fft4<T>(tw, lam, data, n, stv, hi, inverse, ss, st)) return 0;
  const bool pow2 = (n & (n - 1)) == 0;
  if (pow2 && n >= 8 && n <= 2048 && getenv("TR_FFT_SIMPLE") == nullptr) {
    fft_pass_p2<T>(FFT_C2C, data, data, 1.0, stv, n, hi, tw, inverse, ss, lam, 0, st);
    return 0;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_axis<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int64_t L = std::max<int64_t>(1, std::min<int64_t>(16, 4096 / n));
  L = std::min<int64_t>(L, stv == 1 ? hi : stv);
  TR_REQUIRE(n <= 4096, "FFT axis of length %d exceeds the 4096-point tile", n);
  const int64_t grid = stv == 1 ? cdiv(hi, L) : hi * cdiv(stv, L);
  const size_t smem = ((size_t)n + (size_t)L * n * (pow2 ? 1 : 2)) * sizeof(cpx<T>);
  launch("fft", k_fft_axis<T>, (unsigned)grid, 256, smem, st, (const void*)data, data,
         (int)FFT_C2C, 1.0, stv, n, hi, (int)L, tw, inverse, ss, lam);
  return 0;
}

// FFT solve with the half spectrum stored axes-(1, 0)-swapped: every pass
// streams >= 32-byte segments and the axis-1 pass runs on contiguous lines.
// Falls back to fft_solve when axis 0 is not an even power-of-two length.
template <typename T>
static int fft_solve2(Solver<T>& s, const T* rhs, T* out, cudaStream_t st) {
  const Geom& g = s.g;
  const int d = g.d;
  const int64_t n0 = g.dims[0], n1 = g.dims[1];
  const int hn = (int)(n0 / 2);
  const bool ok = n0 % 2 == 0 && (hn & (hn - 1)) == 0 && hn >= 8 && hn <= 2048 &&
                  (n0 * (int64_t)sizeof(T)) % 16 == 0 && getenv("TR_FFT_SIMPLE") == nullptr;
  if (!ok) return fft_solve<T>(s, rhs, out, st);
  int64_t sd[kMaxOrder], sst[kMaxOrder];
  int orig[kMaxOrder];
  sd[0] = n1;
  orig[0] = 1;
  sd[1] = hn + 1;
  orig[1] = 0;
  for (int a = 2; a < d; ++a) {
    sd[a] = g.dims[a];
    orig[a] = a;
  }
  int64_t SN = 1;
  for (int a = 0; a < d; ++a) {
    sst[a] = SN;
    SN *= sd[a];
  }
  SolveSpec off = s.ss, on = s.ss;
  off.active = 0;
  on.active = 1;
  for (int p = 0; p < d; ++p) {
    off.dims[p] = on.dims[p] = sd[p];
    off.lam_off[p] = on.lam_off[p] = s.ss.lam_off[orig[p]];
  }
  const cpx<T>* const* tw = (const cpx<T>* const*)s.tw.data();
  // axis 0, real -> half spectrum (swapped layout)
  const int64_t lines = g.N / n0;
  auto r2c_like = [&](int mode, const void* in, void* dst, double scale) {
    fft_pass_p2<T>(mode, in, dst, scale, 1, (int)n0, lines, tw[0], 0, off, (const double*)s.lam, n1,
                   st);
  };
  r2c_like(FFT_R2C, rhs, s.spec, 1.0);
  for (int p = 0; p < d - 1; ++p) {
    if (p == 1) continue;  // spectral position 1 is axis 0, already transformed
    if (fft_c2c<T>(tw[orig[p]], s.lam, s.spec, (int)sd[p], sst[p], SN / (sst[p] * sd[p]), 0, off, st))
      return 1;
  }
  if (fft_c2c<T>(tw[orig[d - 1]], s.lam, s.spec, (int)sd[d - 1], sst[d - 1], 1, 0, on, st)) return 1;
  for (int p = d - 2; p >= 0; --p) {
    if (p == 1) continue;
    if (fft_c2c<T>(tw[orig[p]], s.lam, s.spec, (int)sd[p], sst[p], SN / (sst[p] * sd[p]), 1, off, st))
      return 1;
  }
  r2c_like(FFT_C2R, s.spec, out, 2.0 / (double)g.N);
  TR_LAUNCH_CHECK();
  return 0;
}

// Multi-GPU FFT solve: the local axes as in fft_solve2, the sharded last axis
// through an all-to-all transpose.  The local half spectrum is lo (M, every
// axis before the last) x nl faces; rank q receives lo chunk q (M / W
// elements) of every rank's faces, i.e. whole last-axis lines, solves them,
// and the inverse all-to-all restores the slab layout.
template <typename T>
static int fft_solve_dist(Solver<T>& s, const T* rhs, T* out, cudaStream_t st) {
  const Geom& g = s.g;
  const int d = g.d;
  const int64_t n0 = g.dims[0], n1 = g.dims[1];
  const int hn = (int)(n0 / 2);
  TR_REQUIRE(n0 % 2 == 0 && (hn & (hn - 1)) == 0 && hn >= 8 && hn <= 2048 &&
                 (n0 * (int64_t)sizeof(T)) % 16 == 0,
             "sharded FFT solve needs an even power-of-two first mode in [16, 4096]");
  const int W = s.comm.world;
  int64_t sd[kMaxOrder], sst[kMaxOrder];
  int orig[kMaxOrder];
  sd[0] = n1;
  orig[0] = 1;
  sd[1] = hn + 1;
  orig[1] = 0;
  for (int a = 2; a < d; ++a) {
    sd[a] = g.dims[a];
    orig[a] = a;
  }
  int64_t SN = 1;
  for (int a = 0; a < d; ++a) {
    sst[a] = SN;
    SN *= sd[a];
  }
  const int64_t M = sst[d - 1];
  TR_REQUIRE(M % W == 0, "sharded FFT solve: %lld spectrum lines do not split over %d ranks",
             (long long)M, W);
  const int64_t mw = M / W, nl = s.nl;
  SolveSpec off = s.ss, on = s.ss;
  off.active = 0;
  on.active = 1;
  for (int p = 0; p < d; ++p) {
    off.dims[p] = on.dims[p] = sd[p];
    off.lam_off[p] = on.lam_off[p] = s.ss.lam_off[orig[p]];
  }
  on.dims[d - 1] = s.last_all;
  on.lo_base = (int64_t)s.comm.rank * mw;
  const cpx<T>* const* tw = (const cpx<T>* const*)s.tw.data();
  const int64_t lines = g.N / n0;
  fft_pass_p2<T>(FFT_R2C, rhs, s.spec, 1.0, 1, (int)n0, lines, tw[0], 0, off, (const double*)s.lam,
                 n1, st);
  for (int p = 0; p < d - 1; ++p) {
    if (p == 1) continue;
    if (fft_c2c<T>(tw[orig[p]], s.lam, s.spec, (int)sd[p], sst[p], SN / (sst[p] * sd[p]), 0, off, st))
      return 1;
  }
  const size_t es = sizeof(cpx<T>);
  for (int q = 0; q < W; ++q)  // pack: lo chunk q of every own face, contiguous per rank
    TR_CUDA(cudaMemcpy2DAsync(s.spec_pack + q * mw * nl, mw * es, s.spec + q * mw, M * es, mw * es,
                              nl, cudaMemcpyDeviceToDevice, st));
  TR_LAUNCH_CHECK();
  if (W == 1) {
    TR_CUDA(cudaMemcpyAsync(s.spec_recv, s.spec_pack, es * M * nl, cudaMemcpyDeviceToDevice, st));
  } else {
    TR_REQUIRE(s.comm.alltoall(s.spec_pack, s.spec_recv, (int64_t)(es * mw * nl), (void*)st,
                               s.comm.user) == 0, "all-to-all callback failed");
  }
  // whole last-axis lines: forward, solve, inverse (stride mw, one line group)
  if (fft_c2c<T>(tw[d - 1], s.lam, s.spec_recv, (int)s.last_all, mw, 1, 0, on, st)) return 1;
  if (W == 1) {
    TR_CUDA(cudaMemcpyAsync(s.spec_pack, s.spec_recv, es * M * nl, cudaMemcpyDeviceToDevice, st));
  } else {
    TR_REQUIRE(s.comm.alltoall(s.spec_recv, s.spec_pack, (int64_t)(es * mw * nl), (void*)st,
                               s.comm.user) == 0, "all-to-all callback failed");
  }
  for (int q = 0; q < W; ++q)  // unpack lo chunk q
    TR_CUDA(cudaMemcpy2DAsync(s.spec + q * mw, M * es, s.spec_pack + q * mw * nl, mw * es, mw * es,
                              nl, cudaMemcpyDeviceToDevice, st));
  for (int p = d - 2; p >= 0; --p) {
    if (p == 1) continue;
    if (fft_c2c<T>(tw[orig[p]], s.lam, s.spec, (int)sd[p], sst[p], SN / (sst[p] * sd[p]), 1, off, st))
      return 1;
  }
  fft_pass_p2<T>(FFT_C2R, s.spec, out, 2.0 / (double)(g.N / nl * s.last_all), 1, (int)n0, lines,
                 tw[0], 0, off, (const double*)s.lam, n1, st);
  TR_LAUNCH_CHECK();
  return 0;
}

// Ghost faces of a sharded array along the last axis: the previous rank's last
// own face -> ghost_prev, the next rank's first own face -> ghost_next (ring,
// the gradients are circular).  `both` = false fills ghost_prev only.
template <typename T>
static int halo_exchange(Solver<T>& s, T* x, cudaStream_t st) {
  const int64_t f = s.face;
  T* first = x;
  T* last = x + (s.nl - 1) * f;
  T* gprev = x - f;
  T* gnext = x + s.nl * f;
  if (s.comm.world == 1) {
    TR_CUDA(cudaMemcpyAsync(gprev, last, sizeof(T) * f, cudaMemcpyDeviceToDevice, st));
    TR_CUDA(cudaMemcpyAsync(gnext, first, sizeof(T) * f, cudaMemcpyDeviceToDevice, st));
    return 0;
  }
  TR_REQUIRE(s.comm.halo(first, last, gprev, gnext, (int64_t)(sizeof(T) * f), (void*)st,
                         s.comm.user) == 0,
             "halo exchange callback failed");
  return 0;
}

// the t-SVT's in-place fp64 sum (tr_allreduce_fn) over the solver's comm
static int comm_allreduce_sum(double* buf, int64_t count, void* stream, void* user) {
  const tr_comm* c = (const tr_comm*)user;
  if (c->world == 1) return 0;
  return c->allreduce(buf, count, 0, stream, c->user);
}

// deterministic t-SVT of a whole tensor with small faces (n1, n2 <= 64)
template <typename T>
static int full_svt(Solver<T>& s, const T* X, T* out, double tau, void* ws, cudaStream_t st) {
  Shape fs = s.sh;
  Carve cv(ws);
  Bufs<T> bf;
  carve<T>(cv, fs, bf);
  const int64_t N = s.g.N;
  launch("convert", k_convert<T, double>, (unsigned)grid_for<T>(N), kRedThreads, 0, st, X,
         bf.core, N);
  if (core_svt<T>(fs, s.cfg.tkind, (const cplx*)s.cfg.tmats, s.cfg.talphas, s.cfg.phi, tau, bf, st))
    return 2;
  launch("convert", k_convert<double, T>, (unsigned)grid_for<T>(N), kRedThreads, 0, st,
         (const double*)bf.core, out, N);
  return 0;
}

// Tucker-compressed t-SVT of one gradient tensor through the generic engine
// (any processing order, fixed-rank or fixed-accuracy sketch; host-driven)
template <typename T>
static int generic_svt(Solver<T>& s, const T* X, T* out, double tau, cudaStream_t st) {
  TuckerResult res;
  if (tucker_compress<T>(X, s.order, s.g.dims, s.tspec, res, st)) return 2;
  if (res.core_size() == 0) {
    TR_CUDA(cudaMemsetAsync(out, 0, sizeof(T) * s.g.N, st));
    return 0;
  }
  if (tucker_core_svt<T>(res, res.core, s.cfg.tkind, s.cfg.tmats, s.cfg.talphas, s.cfg.phi, tau,
                         st))
    return 2;
  return tucker_reconstruct<T>(res, res.core, out, st);
}

template <typename T, typename F>
static int low_rank_step(Solver<T>& s, double tau, F&& on_main, bool main_after_mode0 = false) {
  // fork: each mode on its own stream after the main stream's LRTA inputs
  // (TR_SERIAL_MODES: all on the main stream, for uncontended kernel timings)
  static const bool serial = getenv("TR_SERIAL_MODES") != nullptr;
  TR_CUDA(cudaEventRecord(s.ev_main, s.streams[0]));
  for (int k = 0; k < s.cfg.nmodes; ++k) {
    cudaStream_t sk = serial ? s.streams[0] : s.streams[k + 1];
    int rc;
    // the fused randomized t-SVT takes the dependency on the main stream itself,
    // after its data-independent prologue (input_ready in lrta.cu)
    const bool defer = !s.generic && s.cfg.randomized;
    if (defer) tl_input_ready = s.ev_main;
    else TR_CUDA(cudaStreamWaitEvent(sk, s.ev_main, 0));
    if (s.generic)
      rc = generic_svt<T>(s, s.X[k], s.gnew[k], tau, sk);
    else if (s.cfg.randomized)
      rc = gnhtsvt_randomized_t<T>(s.X[k], s.gnew[k], s.sh, s.cfg.seed, s.cfg.tkind, s.cfg.tmats,
                                   s.cfg.talphas, s.cfg.phi, tau, nullptr, nullptr, s.ws[k],
                                   s.ws_bytes, sk, main_after_mode0 ? s.evs_mid[k] : nullptr,
                                   !s.tf_built.empty() && s.tf_built[k]);
    else
      rc = full_svt<T>(s, s.X[k], s.gnew[k], tau, s.ws[k], sk);
    if (tl_input_ready) {  // never consumed (error path): keep the order anyway
      cudaStreamWaitEvent(sk, tl_input_ready, 0);
      tl_input_ready = nullptr;
    }
    if (rc) return rc;
    if (!s.generic && s.cfg.randomized) {
      if (s.tf_built.empty()) s.tf_built.assign(s.cfg.nmodes, 0);
      s.tf_built[k] = 1;  // same shape, kind and workspace on every later sweep
    }
    TR_CUDA(cudaEventRecord(s.evs[k], sk));
  }
  // work of the main stream that overlaps the per-mode chains; main_after_mode0:
  // only their latency-bound second halves (core-sized data, HBM nearly idle)
  if (main_after_mode0 && !serial && !s.generic && s.cfg.randomized)
    for (int k = 0; k < s.cfg.nmodes; ++k)
      TR_CUDA(cudaStreamWaitEvent(s.streams[0], s.evs_mid[k], 0));
  on_main();
  for (int k = 0; k < s.cfg.nmodes; ++k) TR_CUDA(cudaStreamWaitEvent(s.streams[0], s.evs[k], 0));
  return 0;
}

template <typename T>
static int low_rank_step(Solver<T>& s, double tau) {
  return low_rank_step<T>(s, tau, [] {});
}

// residual slots written by a step (host array of TR_ADMM_NOUT doubles)
enum {
  R_DL = 0, R_DE, R_GRAD, R_DG, R_FIT,            // Eq. (24) inf-norms (completion)
  R_DL_FRO, R_DE_FRO, R_DG_FRO, R_FIT_FRO, R_GRAD_FRO,
  R_Y_NORM, R_LAG_NORM, R_MU, R_REL_DL, R_BOX_GAP, R_NOUT
};

// 16-byte vector path of the line kernels: axis 0 a multiple of 4 and every
// buffer 16-byte aligned (the mask 4-byte aligned)
template <typename T>
static bool line_vec4(const Geom& g, std::initializer_list<const void*> ptrs,
                      const void* mask = nullptr) {
  if (g.dims[0] % 4 != 0) return false;
  for (const void* p : ptrs)
    if (p && ((uintptr_t)p & 15)) return false;
  return !mask || ((uintptr_t)mask & 3) == 0;
}

// multiplier updates of modes [0, nm) in groups of up to 4 (one pass over the
// iterate per group), each group's residuals reduced into res + 5 k0
template <typename T>
static void lag_updates(Solver<T>& s, const T* x, double mu, bool v4, unsigned grid,
                        cudaStream_t st) {
  const int nm = s.cfg.nmodes;
  for (int k0 = 0; k0 < nm; k0 += 4) {
    const int cnt = std::min(4, nm - k0);
    ModePtrs<T> gn{}, go{}, lg{};
    gn.count = go.count = lg.count = cnt;
    for (int k = 0; k < cnt; ++k) {
      gn.p[k] = s.gnew[k0 + k];
      go.p[k] = s.gcur[k0 + k];
      lg.p[k] = s.lag[k0 + k];
      gn.axis[k] = go.axis[k] = lg.axis[k] = s.cfg.modes[k0 + k];
    }
#define TR_LU(NM)                                                                               \
  launch("lag_update", v4 ? k_lag_update<T, 4, NM> : k_lag_update<T, 1, NM>, grid, kRedThreads, \
         0, st, s.g, x, gn, go, lg, mu, s.part)
    switch (cnt) {
      case 1: TR_LU(1); break;
      case 2: TR_LU(2); break;
      case 3: TR_LU(3); break;
      default: TR_LU(4); break;
    }
#undef TR_LU
    unsigned mask = 0;
    for (int k = 0; k < cnt; ++k) mask |= 0b00101u << (5 * k);
    launch("final_reduce", k_final_reduce, 1, 256, 0, st, (const double*)s.part, (int)grid,
           5 * cnt, mask, s.res + 5 * k0);
  }
}

template <typename T>
static void lrta_inputs(Solver<T>& s, const T* x, double mu, bool v4, unsigned grid,
                        cudaStream_t st) {
  for (int k0 = 0; k0 < s.cfg.nmodes; k0 += 4) {
    const int cnt = std::min(4, s.cfg.nmodes - k0);
    ModePtrs<T> lg{}, xs{};
    lg.count = xs.count = cnt;
    for (int k = 0; k < cnt; ++k) {
      lg.p[k] = s.lag[k0 + k];
      xs.p[k] = s.X[k0 + k];
      lg.axis[k] = xs.axis[k] = s.cfg.modes[k0 + k];
    }
    const auto kern = v4 ? k_lrta_input<T, 4> : k_lrta_input<T, 1>;
    launch("lrta_input", kern, resident_grid(kern, s.g.N), kRedThreads, 0, st, s.g, x, lg, xs, mu);
  }
}

template <typename T>
static int admm_step(Solver<T>& s, double* hout) {
  cudaStream_t st = s.streams[0];
  const double mu = s.mu;
  const Geom& g = s.g;
  const int64_t N = g.N;
  const unsigned grid = (unsigned)grid_for<T>(N);
  const int nm = s.cfg.nmodes;
  const int gamma = nm;
  ModePtrs<T> gp{}, lp{};
  gp.count = lp.count = nm;
  for (int k = 0; k < nm; ++k) {
    gp.axis[k] = lp.axis[k] = s.cfg.modes[k];
    gp.p[k] = s.gcur[k];
    lp.p[k] = s.lag[k];
  }
  const bool pure = nm == 1 && s.cfg.modes[0] < 0;
  const bool v4 = line_vec4<T>(g, {s.A, s.B, s.l, s.e, s.y, s.z, s.lold, s.rhs}, s.mask);
  // fused sweep tail (lag + noise/dual + next rhs in one pass): gradient chain,
  // <= 4 modes, vector path
  const bool fuse = !s.onebit() && !pure && nm <= 4 && v4 && !s.lag2.empty();
  TR_REQUIRE(!s.sharded || fuse, "the sharded solver needs the fused sweep tail (aligned buffers)");
  if (!fuse) s.rhs_ready = false;
  const auto rhs_k = v4 ? k_admm_rhs<T, 4> : k_admm_rhs<T, 1>;
  double* part = s.part;
  double* res = s.res;  // device scratch for final reductions
  const int64_t rb = grid;
  // slots in res: [0..4] lag of mode k (5 each, up to 10 modes) | [64..70] noise/dual | [80..] onebit
  double tau;
  bool overlap_noise = false;
  if (!s.onebit()) {
    // L-subproblem (solvers.py:231-233)
    if (pure) {
      launch("admm_rhs", rhs_k, grid, kRedThreads, 0, st, g, s.A, s.e, s.y, mu, gp, lp, s.l);
    } else if (!s.head_done) {
      if (!s.rhs_ready)
        launch("admm_rhs", rhs_k, grid, kRedThreads, 0, st, g, s.A, s.e, s.y, mu, gp, lp, s.rhs);
      if (s.sharded) {
        if (fft_solve_dist<T>(s, s.rhs, s.l, st)) return 1;
        if (halo_exchange<T>(s, s.l, st)) return 1;  // grad along the last axis
      } else if (fft_solve2<T>(s, s.rhs, s.l, st)) {
        return 1;
      }
    }
    tau = 1.0 / (gamma * mu);
    if (!s.head_done) lrta_inputs<T>(s, s.l, mu, v4, grid, st);
    s.head_done = false;
    // noise and dual updates (solvers.py:239-246)
    const double level = s.cfg.lam / mu;
    const int structure = s.cfg.kind == 1 ? 3 : s.cfg.structure;
    const double q0 = s.cfg.psi.p0, q1 = s.cfg.psi.p1;
    // E', Y' need only L: with TR_OVERLAP_NOISE they run on the main stream
    // while the per-mode t-SVTs run and the fused tail reads them instead of
    // recomputing them.  = 1: from the start of the t-SVTs (slower on the bench
    // workload: the extra streaming blocks delay the mode chains' passes,
    // 7.64 vs 7.17 ms per sweep); = 2: once every mode has finished its passes
    // over the whole tensor, when the chains work on the small cores and HBM
    // is nearly idle.
    static const int overlap_env = getenv("TR_OVERLAP_NOISE") ? atoi(getenv("TR_OVERLAP_NOISE")) : 0;
    const bool overlap = fuse && overlap_env > 0;
    const bool overlap_late = overlap && overlap_env >= 2 && s.cfg.randomized && !s.generic;
    overlap_noise = overlap;
    auto group_scale = [&] {
      if (structure == 1 || structure == 2) {
        const int64_t face = g.dims[0] * g.dims[1];
        const unsigned gg = (unsigned)(structure == 1 ? cdiv(face, 256) : N / face);
#define TR_GS(K)                                                                             \
  launch("group_scale", k_group_scale<T, K>, gg, 256, 0, st, g, structure, s.A, s.mask,     \
         (const T*)s.l, (const T*)s.y, mu, q0, q1, level, s.scale)
        TR_PEN_DISPATCH(s.cfg.psi.kind, TR_GS)
#undef TR_GS
      }
    };
    // overlapping the mode chains' latency kernels: leave them thread slots on every SM
    static const int late_ctas = getenv("TR_NOISE_CTAS") ? atoi(getenv("TR_NOISE_CTAS")) : 3;
    const unsigned ngrid =
        overlap_late ? (unsigned)std::min<int64_t>(grid, (int64_t)late_ctas * num_sms()) : grid;
#define TR_ND2(K, S)                                                                          \
  launch("noise_dual", v4 ? k_noise_dual<T, K, S, 4> : k_noise_dual<T, K, S, 1>, ngrid,       \
         kRedThreads, 0, st, g, s.A, s.mask,                                                   \
         (const T*)s.l, (const T*)s.lold, s.e, s.y, mu, q0, q1, level, (const double*)s.scale, \
         part)
#define TR_ND(K)                            \
  switch (structure) {                      \
    case 0: TR_ND2(K, 0); break;            \
    case 1: TR_ND2(K, 1); break;            \
    case 2: TR_ND2(K, 2); break;            \
    default: TR_ND2(K, 3); break;           \
  }
    auto noise_dual = [&] {
      group_scale();
      TR_PEN_DISPATCH(s.cfg.psi.kind, TR_ND)
      launch("final_reduce", k_final_reduce, 1, 256, 0, st, (const double*)part, (int)ngrid, 7,
             0b0010101u, res + 64);
    };
    if (low_rank_step<T>(s, tau, [&] {
          if (overlap) noise_dual();
        }, overlap_late))
      return 2;
    if (s.sharded)  // D_last^T G_new in the next right-hand side
      for (int k = 0; k < nm; ++k)
        if (s.cfg.modes[k] == g.d - 1 && halo_exchange<T>(s, s.gnew[k], st)) return 1;
    if (!fuse) lag_updates<T>(s, s.l, mu, v4, grid, st);
    if (!overlap && fuse) group_scale();
    if (fuse) {
      ModePtrs<T> gn{}, go{}, lw{};
      gn.count = go.count = lw.count = nm;
      for (int k = 0; k < nm; ++k) {
        gn.p[k] = s.gnew[k];
        go.p[k] = s.gcur[k];
        lw.p[k] = s.lag2[k];
        gn.axis[k] = go.axis[k] = lw.axis[k] = s.cfg.modes[k];
      }
      const double mu_next = std::min(s.cfg.mu_max, s.cfg.growth * mu);
      unsigned tgrid = 0;
#define TR_ST3(K, S, NZ)                                                                        \
  tgrid = resident_grid(k_sweep_tail<T, K, S, NZ>, N);                                          \
  launch("sweep_tail", k_sweep_tail<T, K, S, NZ>, tgrid, kRedThreads, 0, st, g, s.A, s.mask,    \
         (const T*)s.l, (const T*)s.lold, s.e, s.y, gn, go, lp, lw, mu, mu_next, q0, q1, level, \
         (const double*)s.scale, s.rhs, part)
#define TR_ST2(K, S)        \
  if (overlap) {            \
    TR_ST3(K, S, false);    \
  } else {                  \
    TR_ST3(K, S, true);     \
  }
#define TR_ST(K)                 \
  switch (structure) {           \
    case 0: TR_ST2(K, 0); break; \
    case 1: TR_ST2(K, 1); break; \
    case 2: TR_ST2(K, 2); break; \
    default: TR_ST2(K, 3); break; \
  }
      TR_PEN_DISPATCH(s.cfg.psi.kind, TR_ST)
#undef TR_ST
#undef TR_ST2
#undef TR_ST3
      // partial slots: 5 per mode (4 slots) then the 7 noise values -> res[96..122]
      launch("final_reduce", k_final_reduce, 1, 256, 0, st, (const double*)part, (int)tgrid, 27,
             0b0010101u << 20 | 0b00101u | 0b00101u << 5 | 0b00101u << 10 | 0b00101u << 15,
             res + 96);
      for (int k = 0; k < nm; ++k) std::swap(s.lag[k], s.lag2[k]);
      s.rhs_ready = true;
      if (s.sharded)  // the next tail recomputes the previous face's multiplier
        for (int k = 0; k < nm; ++k)
          if (s.cfg.modes[k] == g.d - 1 && halo_exchange<T>(s, s.lag[k], st)) return 1;
    } else {
      noise_dual();
    }
#undef TR_ND
#undef TR_ND2
  } else {
    // one-bit (onebit.py:171-192)
    const bool robust = s.cfg.kind == 3;
    const double q0 = s.cfg.psi.p0, q1 = s.cfg.psi.p1;
#define TR_OF(K)                                                                               \
  launch("onebit_fit", k_onebit_fit<T, K>, grid, kRedThreads, 0, st, N, s.A, s.B, s.cfg.mcount, \
         mu, (const T*)s.z, (const T*)s.y, s.cfg.alpha, (const T*)s.lold, s.l, s.e,            \
         robust ? 1 : 0, q0, q1, s.cfg.lam2, part)
    TR_PEN_DISPATCH(s.cfg.psi.kind, TR_OF)
#undef TR_OF
    launch("final_reduce", k_final_reduce, 1, 256, 0, st, (const double*)part, (int)rb, 3, 0b100u,
           res + 80);
    // Z-subproblem: solve with b = L + Y / mu
    if (pure) {
      launch("admm_rhs", rhs_k, grid, kRedThreads, 0, st, g, (const T*)s.l, (const T*)nullptr,
             s.y, mu, gp, lp, s.z);
    } else {
      launch("admm_rhs", rhs_k, grid, kRedThreads, 0, st, g, (const T*)s.l, (const T*)nullptr,
             s.y, mu, gp, lp, s.rhs);
      if (fft_solve2<T>(s, s.rhs, s.z, st)) return 1;
    }
    tau = s.cfg.lam / (gamma * mu);
    lrta_inputs<T>(s, s.z, mu, v4, grid, st);
    if (low_rank_step<T>(s, tau)) return 2;
    launch("onebit_dual", k_onebit_dual<T>, grid, kRedThreads, 0, st, N, (const T*)s.l,
           (const T*)s.z, s.y, mu, part);
    launch("final_reduce", k_final_reduce, 1, 256, 0, st, (const double*)part, (int)rb, 2, 0b01u,
           res + 90);
    lag_updates<T>(s, s.z, mu, v4, grid, st);
  }
  TR_LAUNCH_CHECK();
  if (s.sharded && s.comm.world > 1) {
    // residual slots are sums (squares) or maxima (inf-norms): reduce both ways
    TR_CUDA(cudaMemcpyAsync(s.res_max, res, 128 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    TR_REQUIRE(s.comm.allreduce(res, 128, 0, (void*)st, s.comm.user) == 0 &&
                   s.comm.allreduce(s.res_max, 128, 1, (void*)st, s.comm.user) == 0,
               "residual all-reduce callback failed");
    TR_CUDA(cudaMemcpyAsync(s.hres_max, s.res_max, 128 * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  TR_CUDA(cudaMemcpyAsync(s.hres, res, 128 * sizeof(double), cudaMemcpyDeviceToHost, st));
  // lookahead: the next sweep's L-solve and t-SVT inputs go in behind the
  // read-back (fused gradient chain on one GPU; the right-hand side is ready)
  const bool ahead = s.lookahead && fuse && !s.sharded && !pure && s.rhs_ready;
  if (ahead) {
    TR_CUDA(cudaEventRecord(s.ev_res, st));
    const double mu2 = std::min(s.cfg.mu_max, s.cfg.growth * s.mu);
    // next sweep's buffers: L is solved into the buffer that holds L_prev now
    if (fft_solve2<T>(s, s.rhs, s.lold, st)) return 1;
    lrta_inputs<T>(s, s.lold, mu2, v4, grid, st);
    TR_LAUNCH_CHECK();
    TR_CUDA(cudaEventSynchronize(s.ev_res));
  } else {
    TR_CUDA(cudaStreamSynchronize(st));
  }
  if (s.sharded && s.comm.world > 1) {
    // fused layout (the only sharded one): per mode [grad max, grad^2, dG max,
    // dG^2, lag^2] at 96 + 5k, noise [dL max, dL^2, dE max, dE^2, fit max,
    // fit^2, Y^2] at 116
    for (int k = 0; k < nm; ++k) {
      s.hres[96 + 5 * k + 0] = s.hres_max[96 + 5 * k + 0];
      s.hres[96 + 5 * k + 2] = s.hres_max[96 + 5 * k + 2];
    }
    for (int i : {0, 2, 4}) s.hres[116 + i] = s.hres_max[116 + i];
  }
  const double* h = s.hres;
  const double* hl = fuse ? h + 96 : h;          // per-mode multiplier residuals
  const double* hn = (fuse && !overlap_noise) ? h + 96 + 20 : h + 64;  // noise / dual residuals
  for (int i = 0; i < R_NOUT; ++i) hout[i] = 0.0;
  double grad = 0, dg = 0, dgf = 0, gradf = 0, lagn = 0;
  for (int k = 0; k < nm; ++k) {
    grad = fmax(grad, hl[5 * k + 0]);
    gradf = fmax(gradf, sqrt(hl[5 * k + 1]));
    dg = fmax(dg, hl[5 * k + 2]);
    dgf = fmax(dgf, sqrt(hl[5 * k + 3]));
    lagn = fmax(lagn, sqrt(hl[5 * k + 4]));
  }
  hout[R_GRAD] = grad;
  hout[R_GRAD_FRO] = gradf;
  hout[R_DG] = dg;
  hout[R_DG_FRO] = dgf;
  hout[R_LAG_NORM] = lagn;
  hout[R_MU] = mu;
  if (!s.onebit()) {
    hout[R_DL] = hn[0];
    hout[R_DL_FRO] = sqrt(hn[1]);
    hout[R_DE] = hn[2];
    hout[R_DE_FRO] = sqrt(hn[3]);
    hout[R_FIT] = hn[4];
    hout[R_FIT_FRO] = sqrt(hn[5]);
    hout[R_Y_NORM] = sqrt(hn[6]);
  } else {
    hout[R_REL_DL] = sqrt(h[80]) / fmax(sqrt(h[81]), 1e-30);
    hout[R_DL] = h[82];
    hout[R_BOX_GAP] = h[90];
    hout[R_Y_NORM] = sqrt(h[91]);
  }
  // roll state: L_prev <- L, G <- G_new, mu <- min(mu_max, growth mu); Z is
  // overwritten in place by the next solve
  std::swap(s.l, s.lold);
  for (int k = 0; k < nm; ++k) std::swap(s.gcur[k], s.gnew[k]);
  s.mu = std::min(s.cfg.mu_max, s.cfg.growth * s.mu);
  s.head_done = ahead;  // s.l (after the swap) already receives the next sweep's L
  return 0;
}

template <typename T>
static int admm_create(const AdmmConfig& cfg, int order, const int64_t* dims, const void* a,
                       const void* b, const uint8_t* mask, Solver<T>** out,
                       const tr_comm* comm = nullptr, int64_t last_all = 0,
                       int64_t last_off = 0) {
  TR_REQUIRE(order >= 3 && order <= kMaxOrder, "order must be in [3, %d]", kMaxOrder);
  TR_REQUIRE(cfg.nmodes >= 1 && cfg.nmodes <= kMaxOrder, "need 1..%d gradient modes", kMaxOrder);
  if (comm) {
    TR_REQUIRE(comm->world >= 1 && comm->rank >= 0 && comm->rank < comm->world,
               "bad communicator (rank %d of %d)", comm->rank, comm->world);
    TR_REQUIRE(comm->world == 1 || (comm->allreduce && comm->alltoall && comm->halo),
               "a multi-rank solver needs allreduce, alltoall and halo callbacks");
    TR_REQUIRE(cfg.kind <= 1 && cfg.randomized, "the sharded solver runs GNRHTC / GNHTC with a "
               "randomized sketch");
    TR_REQUIRE(cfg.structure == 0, "the sharded solver supports entry-wise noise shrinkage");
    TR_REQUIRE(cfg.nmodes <= 4 && cfg.modes[0] >= 0 && dims[0] % 4 == 0,
               "the sharded solver needs <= 4 gradient modes and a first mode divisible by 4");
    TR_REQUIRE(last_all == dims[order - 1] * comm->world &&
                   last_off == dims[order - 1] * comm->rank,
               "the last mode must split evenly: rank %d of %d owns [%lld, %lld) of %lld", comm->rank,
               comm->world, (long long)last_off, (long long)(last_off + dims[order - 1]),
               (long long)last_all);
  }
  TR_CUDA(cudaDeviceSynchronize());  // inputs written on the caller's streams
  auto* s = new Solver<T>();
  s->cfg = cfg;
  s->order = order;
  if (comm) {
    s->sharded = true;
    s->comm = *comm;
    s->last_all = last_all;
    s->last_off = last_off;
    s->nl = dims[order - 1];
  }
  Geom& g = s->g;
  g.d = order;
  g.N = 1;
  for (int i = 0; i < order; ++i) {
    g.dims[i] = dims[i];
    g.st[i] = g.N;
    g.lst[i] = g.N / dims[0];
    g.N *= dims[i];
  }
  const int64_t N = g.N;
  const int nm = cfg.nmodes;
  {
    static const bool mem_order = getenv("TR_WALK_MEMORY_ORDER") != nullptr;
    if (!mem_order && order >= 3) g.walk_last = dims[order - 1];
  }
  if (s->sharded) {
    g.halo = order - 1;
    s->face = N / s->nl;
  }
  if (cfg.randomized) {
    if (make_shape(order, dims, cfg.ranks, cfg.blocks, cfg.krylov, s->sh)) {
      delete s;
      return 1;
    }
    if (s->sharded) {  // the t-SVT of a last-mode shard (lrta.cu, tr_gnhtsvt_randomized_sharded)
      Shape& sh = s->sh;
      const int64_t inner = sh.nf / s->nl;
      sh.tr.d[order - 3] = last_all;
      sh.nf_all = inner * last_all;
      sh.f0 = inner * last_off;
      sh.coll = s->comm.world > 1 ? comm_allreduce_sum : nullptr;
      sh.coll_user = &s->comm;
    }
  } else {
    if (!(dims[0] <= 4096 && dims[1] <= 4096)) {
      delete s;
      TR_REQUIRE(false, "deterministic t-SVT on the GPU needs face slices up to 4096 x 4096; "
                        "use the randomized solver for larger tensors");
    }
    Shape& f = s->sh;
    f.order = order;
    f.n1 = dims[0];
    f.n2 = dims[1];
    f.nf = N / (dims[0] * dims[1]);
    f.tr.nt = order - 2;
    for (int i = 0; i < 8; ++i) f.tr.d[i] = 1;
    for (int i = 2; i < order; ++i) f.tr.d[i - 2] = dims[i];
    f.r0 = dims[0];
    f.r1 = dims[1];
    f.b0 = f.b1 = 1;
    f.q0 = f.q1 = 0;
    f.s0 = f.s1 = 1;
  }
  s->A = (const T*)a;
  s->B = (const T*)b;
  s->mask = mask;
  s->mu = cfg.mu0;
  // arrays a stencil reads along the sharded last axis carry ghost faces
  auto on_last = [&](int k) { return s->sharded && cfg.modes[k] == order - 1; };
  auto big = [&](bool ghost) { return ghost ? s->alloc_ghosted(N) : s->template alloc<T>(N); };
  s->l = big(s->sharded);
  s->lold = big(s->sharded);
  s->e = s->template alloc<T>(N);
  s->y = s->template alloc<T>(N);
  s->z = s->template alloc<T>(N);
  s->rhs = s->template alloc<T>(N);
  for (int k = 0; k < nm; ++k) {
    s->gcur.push_back(big(on_last(k)));
    s->gnew.push_back(big(on_last(k)));
    s->lag.push_back(big(on_last(k)));
    s->X.push_back(s->template alloc<T>(N));
  }
  // second multiplier buffers for the fused sweep tail (gradient chain, <= 4 modes)
  if (cfg.kind < 2 && nm <= 4 && cfg.modes[0] >= 0 &&
      (s->sharded || getenv("TR_NO_FUSE") == nullptr))
    for (int k = 0; k < nm; ++k) s->lag2.push_back(big(on_last(k)));
  s->spec = s->template alloc<cpx<T>>(N);
  if (s->sharded) {
    s->spec_pack = s->template alloc<cpx<T>>(N);
    s->spec_recv = s->template alloc<cpx<T>>(N);
    s->res_max = s->template alloc<double>(128);
  }
  // global axis lengths (the FFT twiddles and Laplacian tables of the last
  // axis span every rank's faces)
  int64_t gd[kMaxOrder];
  for (int i = 0; i < order; ++i) gd[i] = (s->sharded && i == order - 1) ? last_all : dims[i];
  int64_t lam_total = 0;
  for (int i = 0; i < order; ++i) {
    s->tw.push_back(s->template alloc<cpx<T>>(gd[i]));
    lam_total += gd[i];
  }
  s->lam = s->template alloc<double>(lam_total);
  s->scale = s->template alloc<double>(std::max<int64_t>(dims[0] * dims[1], N / (dims[0] * dims[1])));
  s->red_blocks = grid_for<T>(N);
  s->part = s->template alloc<double>(s->red_blocks * 27);  // fused tail: 4 x 5 + 7 partials
  s->res = s->template alloc<double>(128);
  for (void* p : s->allocs)
    if (!p) {
      delete s;
      TR_REQUIRE(false, "device allocation failed (out of memory?)");
    }
  TR_CUDA(cudaStreamSynchronize(0));  // pool allocations are ordered on the legacy stream
  TR_CUDA(cudaMallocHost(&s->hres, 128 * sizeof(double)));
  if (s->sharded) TR_CUDA(cudaMallocHost(&s->hres_max, 128 * sizeof(double)));
  // LRTA workspaces, one per mode stream
  {
    Carve cv(nullptr);
    Bufs<T> bf;
    carve<T>(cv, s->sh, bf);
    s->ws_bytes = cv.off;
  }
  for (int k = 0; k < nm; ++k) {
    void* p = s->template alloc<unsigned char>(s->ws_bytes);
    TR_REQUIRE(p, "workspace allocation failed");
    s->ws.push_back(p);
  }
  TR_CUDA(cudaStreamSynchronize(0));
  // Staggered stream priorities for the per-mode LRTA chains (first mode
  // highest), so one chain's latency kernels are dispatched ahead of the other
  // chains' streaming blocks whenever SMs free up (TR_NO_MODE_PRIORITY: off).
  static const bool prio = getenv("TR_NO_MODE_PRIORITY") == nullptr;
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  for (int k = 0; k <= nm; ++k) {
    cudaStream_t st;
    if (prio && k > 0) {
      const int p = std::max(greatest, std::min(least, greatest + (k - 1)));
      TR_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, p));
    } else {
      TR_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    }
    s->streams.push_back(st);
    if (k < nm) {
      cudaEvent_t e;
      TR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      s->evs.push_back(e);
      TR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      s->evs_mid.push_back(e);
    }
  }
  TR_CUDA(cudaEventCreateWithFlags(&s->ev_main, cudaEventDisableTiming));
  TR_CUDA(cudaEventCreateWithFlags(&s->ev_res, cudaEventDisableTiming));
  cudaStream_t st = s->streams[0];
  // zero state (ghost faces included: the first sweep's right-hand side reads them)
  auto zero = [&](T* p, bool ghost) -> int {
    const int64_t f = ghost ? s->face : 0;
    TR_CUDA(cudaMemsetAsync(p - f, 0, (N + 2 * f) * sizeof(T), st));
    return 0;
  };
  if (zero(s->l, s->sharded) || zero(s->lold, s->sharded)) return 2;
  for (void* p : {(void*)s->e, (void*)s->y, (void*)s->z})
    TR_CUDA(cudaMemsetAsync(p, 0, N * sizeof(T), st));
  for (int k = 0; k < nm; ++k) {
    if (zero(s->gcur[k], on_last(k)) || zero(s->lag[k], on_last(k))) return 2;
    if (on_last(k) && (zero(s->gnew[k], true) || zero(s->lag2[k], true))) return 2;
  }
  // FFT twiddles and Laplacian eigenvalues of the gradient modes
  SolveSpec& ss = s->ss;
  ss.active = 0;
  ss.d = order;
  int64_t off = 0;
  for (int i = 0; i < order; ++i) {
    ss.dims[i] = dims[i];
    ss.lam_off[i] = -1;
    launch("setup", k_twiddles<T>, (unsigned)cdiv(gd[i], 256), 256, 0, st, (int)gd[i], s->tw[i]);
    launch("setup", k_lap_eig, (unsigned)cdiv(gd[i], 256), 256, 0, st, (int)gd[i], s->lam + off);
    for (int k = 0; k < nm; ++k)
      if (cfg.modes[k] == i) ss.lam_off[i] = off;
    off += gd[i];
  }
  TR_LAUNCH_CHECK();
  TR_CUDA(cudaStreamSynchronize(st));
  *out = s;
  return 0;
}

// Gradient-system plan: GradientSet (tenrec/gradient.py:44-87) + the solve of
// solve_grad_system (gradient.py:90-106) on device buffers.  A Solver holding
// only the geometry, twiddles, eigenvalue tables, spectrum and rhs buffers.
template <typename T>
static int gradsys_create(int order, const int64_t* dims, int nmodes, const int* modes,
                          Solver<T>** out) {
  TR_REQUIRE(order >= 3 && order <= kMaxOrder, "order must be in [3, %d]", kMaxOrder);
  TR_REQUIRE(nmodes >= 1 && nmodes <= order, "gradient mode set must be nonempty");
  for (int k = 0; k < nmodes; ++k) {
    TR_REQUIRE(modes[k] >= 0 && modes[k] < order, "gradient mode %d out of range for order %d",
               modes[k], order);
    for (int j = 0; j < k; ++j) TR_REQUIRE(modes[j] != modes[k], "gradient mode %d repeated", modes[k]);
  }
  for (int i = 0; i < order; ++i) TR_REQUIRE(dims[i] >= 1, "dims must be positive");
  auto* s = new Solver<T>();
  s->order = order;
  s->cfg.nmodes = nmodes;
  for (int k = 0; k < nmodes; ++k) s->cfg.modes[k] = modes[k];
  Geom& g = s->g;
  g.d = order;
  g.N = 1;
  for (int i = 0; i < order; ++i) {
    g.dims[i] = dims[i];
    g.st[i] = g.N;
    g.lst[i] = g.N / dims[0];
    g.N *= dims[i];
  }
  s->rhs = s->template alloc<T>(g.N);
  s->spec = s->template alloc<cpx<T>>(g.N);
  int64_t lam_total = 0;
  for (int i = 0; i < order; ++i) {
    s->tw.push_back(s->template alloc<cpx<T>>(dims[i]));
    lam_total += dims[i];
  }
  s->lam = s->template alloc<double>(lam_total);
  for (void* p : s->allocs)
    if (!p) {
      delete s;
      TR_REQUIRE(false, "device allocation failed (out of memory?)");
    }
  SolveSpec& ss = s->ss;
  ss.active = 0;
  ss.d = order;
  int64_t off = 0;
  for (int i = 0; i < order; ++i) {
    ss.dims[i] = dims[i];
    ss.lam_off[i] = -1;
    launch("setup", k_twiddles<T>, (unsigned)cdiv(dims[i], 256), 256, 0, (cudaStream_t)0,
           (int)dims[i], s->tw[i]);
    launch("setup", k_lap_eig, (unsigned)cdiv(dims[i], 256), 256, 0, (cudaStream_t)0, (int)dims[i],
           s->lam + off);
    for (int k = 0; k < nmodes; ++k)
      if (modes[k] == i) ss.lam_off[i] = off;
    off += dims[i];
  }
  TR_LAUNCH_CHECK();
  TR_CUDA(cudaStreamSynchronize(0));
  *out = s;
  return 0;
}

// out = (I + sum_k D_k^T D_k)^{-1} (b + sum_k D_k^T grads[k]).  The rhs is
// formed by k_admm_rhs with mu = inf (its y / mu and lag / mu terms vanish).
template <typename T>
static int gradsys_solve(Solver<T>& s, const T* b, const T* const* grads, T* out, cudaStream_t st) {
  ModePtrs<T> gm{}, lag{};
  gm.count = lag.count = s.cfg.nmodes;
  for (int k = 0; k < s.cfg.nmodes; ++k) {
    TR_REQUIRE(grads[k], "null gradient term for mode %d", s.cfg.modes[k]);
    gm.p[k] = lag.p[k] = const_cast<T*>(grads[k]);
    gm.axis[k] = lag.axis[k] = s.cfg.modes[k];
  }
  const double inf = std::numeric_limits<double>::infinity();
  bool v4 = line_vec4<T>(s.g, {b, out, s.rhs});
  for (int k = 0; k < s.cfg.nmodes; ++k) v4 = v4 && ((uintptr_t)grads[k] & 15) == 0;
  launch("admm_rhs", v4 ? k_admm_rhs<T, 4> : k_admm_rhs<T, 1>, (unsigned)grid_for<T>(s.g.N),
         kRedThreads, 0, st, s.g, b, (const T*)nullptr, b, inf, gm, lag, s.rhs);
  return fft_solve2<T>(s, s.rhs, out, st);
}

}  // namespace tr
