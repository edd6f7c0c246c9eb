// Stage timing of the cluster Krylov-basis kernel (k_orth_cluster) on a
// 1024 x 28 Krylov-like block.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTR_ORTH_PROBE \
//      -Ipaper_2506_09594_b200/csrc -o tools/orth_probe tools/orth_probe.cu
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "orth_cluster.cuh"
namespace tr { void set_error(const char*, ...) {} }
using namespace tr;

int main() {
  const int m = 1024, s = 28;
  std::mt19937_64 rng(3);
  std::normal_distribution<double> nd;
  std::vector<double> K((size_t)m * s);
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < m; ++i) K[i + (size_t)m * j] = nd(rng) * std::pow(10.0, -3.0 * j / s);
  double *dK, *dZ;
  float* dZt;
  int64_t* dinfo;
  cudaMalloc(&dK, K.size() * 8);
  cudaMalloc(&dZ, K.size() * 8);
  cudaMalloc(&dZt, K.size() * 4);
  cudaMalloc(&dinfo, 64);
  cudaMemcpy(dK, K.data(), K.size() * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_orth_cluster<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOcSmem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_orth_cluster<float><<<kOcCtas, kOcThreads, kOcSmem>>>(dK, m, s, dZ, dZt, dinfo, (float*)nullptr, (float*)nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c[8];
    cudaMemcpyFromSymbol(c, g_orth_probe, sizeof(c));
    printf("orth %.1f us | local %lld | sync %lld | stack %lld | pivot %lld | apply-stack %lld | "
           "scatter+sync %lld | apply-local %lld cycles (%s)\n",
           ms * 1e3, c[0], c[1] - c[0], c[2] - c[1], c[3] - c[2], c[4] - c[3], c[5] - c[4],
           c[6] - c[5], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
