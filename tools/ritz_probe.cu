// Rayleigh-Ritz Jacobi probe: k_ritz<float> on W^T W of a 1024 x 28 block with
// Krylov-like column decay; prints kernel time, sweeps and cycles per round.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTR_RITZ_PROBE \
//      -Ipaper_2506_09594_b200/csrc -o tools/ritz_probe tools/ritz_probe.cu
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "lrta_kernels.cuh"
namespace tr { void set_error(const char*, ...) {} }
using namespace tr;

int main() {
  const int m = 1024, s = 28, r = 25, n = 4000;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::vector<double> W((size_t)n * s), M((size_t)s * s, 0.0), Z((size_t)m * s);
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < n; ++i) W[i + (size_t)n * j] = nd(rng) * std::pow(10.0, -6.0 * j / s);
  for (int a = 0; a < s; ++a)
    for (int b = 0; b < s; ++b) {
      double t = 0;
      for (int i = 0; i < n; ++i) t += W[i + (size_t)n * a] * W[i + (size_t)n * b];
      M[a + s * b] = t;
    }
  for (auto& z : Z) z = nd(rng);
  double *dM, *dZ, *dV, *dF;
  float* dFt;
  int64_t* dinfo;
  double* dpv;
  int64_t* dpi;
  unsigned int* dtk;
  cudaMalloc(&dpv, 64 * 32 * 8);
  cudaMalloc(&dpi, 64 * 32 * 8);
  cudaMalloc(&dtk, 8);
  cudaMemset(dtk, 0, 8);
  cudaMalloc(&dM, M.size() * 8);
  cudaMalloc(&dZ, Z.size() * 8);
  cudaMalloc(&dV, (size_t)s * r * 8);
  cudaMalloc(&dF, (size_t)m * r * 8);
  cudaMalloc(&dFt, (size_t)m * r * 4);
  cudaMalloc(&dinfo, 8 * 8);
  cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dZ, Z.data(), Z.size() * 8, cudaMemcpyHostToDevice);
  int64_t info[8] = {s, 0};
  cudaMemcpy(dinfo, info, sizeof(info), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_ritz<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 65 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    int zero[8] = {0};
    cudaMemcpyToSymbol(g_dbg, zero, sizeof(zero));
    cudaEventRecord(e0);
    k_ritz<float><<<1, 256, 2 * 64 * 65 * 8>>>(dM, s, dZ, m, r, dV, nullptr, dFt, dinfo);
    k_ritz_apply<float><<<(m + 31) / 32, 256>>>(dZ, m, s, dV, r, dinfo, dF, dFt, dpv, dpi, dtk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int dbg[8];
    long long cyc[4];
    cudaMemcpyFromSymbol(dbg, g_dbg, sizeof(dbg));
    cudaMemcpyFromSymbol(cyc, g_ritz_probe, sizeof(cyc));
    printf("k_ritz: %.1f us, sweeps %d, jacobi %lld cycles = %.0f cycles/round, (jacobi-only kernel + apply kernel) %lld %lld (%s)\n",
           ms * 1e3, dbg[0], cyc[0], (double)cyc[0] / (dbg[0] * (s - 1)), cyc[1] - cyc[0], cyc[2] - cyc[1],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
