// Shared device helpers for the tenrec B200 path (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "tenrec_b200 targets sm_100a only"
#endif

namespace tr {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// error plumbing for the C-ABI: every entry point returns 0 or an error code
// and leaves a message readable through tr_last_error().
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);

#define TR_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::tr::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                   \
                      cudaGetErrorString(_e));                                     \
      return 2;                                                                    \
    }                                                                              \
  } while (0)

#define TR_LAUNCH_CHECK()                                                          \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      ::tr::set_error("%s:%d launch: %s", __FILE__, __LINE__,                      \
                      cudaGetErrorString(_e));                                     \
      return 2;                                                                    \
    }                                                                              \
  } while (0)

#define TR_REQUIRE(cond, ...)                                                      \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      ::tr::set_error(__VA_ARGS__);                                                \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

// ---------------------------------------------------------------------------
// Philox4x32-10 Gaussian stream; bit-for-bit twin of oracle/philox.py.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                             uint32_t& c3, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
  uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
  uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
  c0 = n0;
  c1 = lo1;
  c2 = n2;
  c3 = lo0;
}

// Two standard normals for the pair index `pair` (flat indices 2*pair, 2*pair+1).
__device__ __forceinline__ void gauss_pair(uint64_t seed, uint64_t stream, uint64_t pair,
                                           double& z0, double& z1) {
  uint32_t c0 = (uint32_t)pair, c1 = (uint32_t)(pair >> 32);
  uint32_t c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    philox_round(c0, c1, c2, c3, k0, k1);
  }
  const double two53 = 1.0 / 9007199254740992.0;
  double u1 = ((double)(c0 >> 5) * 67108864.0 + (double)(c1 >> 6)) * two53;
  double u2 = ((double)(c2 >> 5) * 67108864.0 + (double)(c3 >> 6)) * two53;
  double rad = sqrt(-2.0 * log(1.0 - u1));
  double s, c;
  sincos(2.0 * 3.14159265358979323846 * u2, &s, &c);
  z0 = rad * c;
  z1 = rad * s;
}

__device__ __forceinline__ double gauss_at(uint64_t seed, uint64_t stream, uint64_t idx) {
  double z0, z1;
  gauss_pair(seed, stream, idx >> 1, z0, z1);
  return (idx & 1) ? z1 : z0;
}

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; `scratch` holds >= 32 values.  All threads get the result.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T t = (threadIdx.x < nw) ? scratch[threadIdx.x] : T(0);
  if (wid == 0) t = warp_sum(t);
  if (threadIdx.x == 0) scratch[0] = t;
  __syncthreads();
  T r = scratch[0];
  __syncthreads();
  return r;
}

template <typename T>
__device__ __forceinline__ T block_max(T v, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T t = (threadIdx.x < nw) ? scratch[threadIdx.x] : T(0);
  if (wid == 0) t = warp_max(t);
  if (threadIdx.x == 0) scratch[0] = t;
  __syncthreads();
  T r = scratch[0];
  __syncthreads();
  return r;
}

// Round-robin (tournament) pairing for parallel Jacobi: player k of round r,
// n even.  Every round pairs all players; n-1 rounds visit every pair once.
__device__ __forceinline__ int rr_player(int k, int r, int n) {
  return k == 0 ? 0 : 1 + (k - 1 + r) % (n - 1);
}

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t align_up(int64_t a, int64_t b) { return cdiv(a, b) * b; }

// cp.async (global -> shared, asynchronous) helpers
__device__ __forceinline__ void cpa4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

}  // namespace tr
