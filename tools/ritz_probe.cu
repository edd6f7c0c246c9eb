// Rayleigh-Ritz probe: k_ritz_pc (QR-preconditioned one-sided Jacobi) and
// k_ritz<float> (two-sided Jacobi) on W^T W of a graded 4000 x 28 block;
// prints kernel times, and for k_ritz_pc the Cholesky / Jacobi cycles, sweeps
// and numerical rank, and the eigenvalue agreement of the two.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTR_RITZ_PROBE \
//      -Ipaper_2506_09594_b200/csrc -o tools/ritz_probe tools/ritz_probe.cu
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "lrta_kernels.cuh"
namespace tr { void set_error(const char*, ...) {} }
using namespace tr;

int main(int argc, char** argv) {
  const int m = 1024, s = 28, r = 25, n = 4000;
  const double decades = argc > 1 ? atof(argv[1]) : 6.0;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::vector<double> W((size_t)n * s), M((size_t)s * s, 0.0), Z((size_t)m * s);
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < n; ++i) W[i + (size_t)n * j] = nd(rng) * std::pow(10.0, -decades * j / s);
  for (int a = 0; a < s; ++a)
    for (int b = 0; b < s; ++b) {
      double t = 0;
      for (int i = 0; i < n; ++i) t += W[i + (size_t)n * a] * W[i + (size_t)n * b];
      M[a + s * b] = t;
    }
  for (auto& z : Z) z = nd(rng);
  double *dM, *dZ, *dV, *dV2;
  float* dFt;
  int64_t* dinfo;
  cudaMalloc(&dM, M.size() * 8);
  cudaMalloc(&dZ, Z.size() * 8);
  cudaMalloc(&dV, (size_t)s * r * 8);
  cudaMalloc(&dV2, (size_t)s * r * 8);
  cudaMalloc(&dFt, (size_t)m * r * 4);
  cudaMalloc(&dinfo, 8 * 8);
  cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dZ, Z.data(), Z.size() * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_ritz<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 65 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    int64_t info[8] = {s, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpy(dinfo, info, sizeof(info), cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    k_ritz_pc<<<1, 256>>>(dM, s, r, dV, dinfo);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t_pc = 0;
    cudaEventElapsedTime(&t_pc, e0, e1);
    cudaMemcpy(info, dinfo, sizeof(info), cudaMemcpyDeviceToHost);
    int64_t info2[8] = {s, 0};
    cudaMemcpy(dinfo, info2, sizeof(info2), cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    k_ritz<float><<<1, 256, 2 * 64 * 65 * 8>>>(dM, s, dZ, m, r, dV2, (double*)nullptr, dFt, dinfo);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t_2s = 0;
    cudaEventElapsedTime(&t_2s, e0, e1);
    std::vector<double> V(s * r), V2(s * r);
    cudaMemcpy(V.data(), dV, V.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(V2.data(), dV2, V2.size() * 8, cudaMemcpyDeviceToHost);
    double maxd = 0;  // |<v_k, v2_k>| should be 1 for separated eigenvalues
    for (int k = 0; k < r; ++k) {
      double d = 0;
      for (int i = 0; i < s; ++i) d += V[i + s * k] * V2[i + s * k];
      maxd = std::max(maxd, 1 - std::fabs(d));
    }
    printf("decades %.1f  pc %.1f us (chol %lld cyc, jacobi %lld cyc, %lld sweeps, rank %lld)  2s %.1f us  max(1-|cos|) %.2e\n",
           decades, t_pc * 1e3, (long long)info[4], (long long)info[5], (long long)info[6],
           (long long)info[7], t_2s * 1e3, maxd);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
