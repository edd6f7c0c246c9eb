// Face SVT probe: k_face_svt (one warp per pair, V accumulated) against
// k_face_svt8<LPP> (LPP = 8 or 16 lanes per pair from $LPP, no V) on 128 dense 25 x 25 complex faces with
// singular values over two decades (what the bench cores look like); prints
// kernel times, sweeps / Jacobi cycles of face 0 and the output agreement.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTR_FACE_PROBE \
//      -Ipaper_2506_09594_b200/csrc -o tools/face_probe tools/face_probe.cu
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "core_svt.cuh"
namespace tr { void set_error(const char*, ...) {} }
using namespace tr;

int main(int argc, char** argv) {
  const int r0 = argc > 1 ? atoi(argv[1]) : 25, r1 = argc > 2 ? atoi(argv[2]) : 25;
  const int nf = 128;
  const double decades = argc > 3 ? atof(argv[3]) : 2.0;
  const double gscale = argc > 4 ? atof(argv[4]) : 1.0;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::vector<cplx> F((size_t)r0 * r1 * nf);
  for (int f = 0; f < nf; ++f) {
    std::vector<cplx> G((size_t)r0 * r1), M((size_t)r0 * r0);
    for (int j = 0; j < r1; ++j)
      for (int i = 0; i < r0; ++i) {
        const double s = std::pow(10.0, -decades * j / r1);
        G[i + (size_t)r0 * j] = {nd(rng) * s, nd(rng) * s};
      }
    for (auto& m : M) m = {nd(rng), nd(rng)};
    for (int j = 0; j < r1; ++j)
      for (int i = 0; i < r0; ++i) {
        double ar = 0, ai = 0;
        for (int k = 0; k < r0; ++k) {
          const cplx a = M[i + (size_t)r0 * k], b = G[k + (size_t)r0 * j];
          ar += a.re * b.re - a.im * b.im;
          ai += a.re * b.im + a.im * b.re;
        }
        F[(size_t)f * r0 * r1 + i + (size_t)r0 * j] = {ar * gscale, ai * gscale};
      }
  }
  cplx *dF, *dA, *dB;
  const size_t bytes = F.size() * sizeof(cplx);
  cudaMalloc(&dF, bytes);
  cudaMalloc(&dA, bytes);
  cudaMalloc(&dB, bytes);
  cudaMemcpy(dF, F.data(), bytes, cudaMemcpyHostToDevice);
  Trailing tr{};
  tr.nt = 1;
  tr.d[0] = nf;
  Penalty pen{2, 2.5, 0.0};
  const double tau = 5.0 * gscale;
  cudaFuncSetAttribute(k_face_svt, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 64 * 16);
  cudaFuncSetAttribute(k_face_svt8<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32 * 32 * 16);
  cudaFuncSetAttribute(k_face_svt8<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32 * 32 * 16);
  const int lpp = getenv("LPP") ? atoi(getenv("LPP")) : 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int npairs = (r1 + (r1 & 1)) / 2;
  const int fth = std::min(1024, std::max(128, 32 * npairs));
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dA, dF, bytes, cudaMemcpyDeviceToDevice);
    cudaMemcpy(dB, dF, bytes, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    k_face_svt<<<nf, fth, (size_t)(r0 * r1 + r1 * r1) * 16>>>(dA, r0, r1, pen, tau, tr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t_old = 0;
    cudaEventElapsedTime(&t_old, e0, e1);
    cudaEventRecord(e0);
    if (lpp == 8) k_face_svt8<8><<<nf, 128, (size_t)(2 * r0 * r1 + r1 * r1) * 16>>>(dB, r0, r1, pen, tau, tr);
    else k_face_svt8<16><<<nf, 256, (size_t)(2 * r0 * r1 + r1 * r1) * 16>>>(dB, r0, r1, pen, tau, tr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t_new = 0;
    cudaEventElapsedTime(&t_new, e0, e1);
    long long probe[4] = {0, 0, 0, 0};
    cudaMemcpyFromSymbol(probe, g_face_probe, sizeof(probe));
    std::vector<cplx> A(F.size()), B(F.size());
    cudaMemcpy(A.data(), dA, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(B.data(), dB, bytes, cudaMemcpyDeviceToHost);
    double num = 0, den = 0, inn = 0;
    for (size_t e = 0; e < (size_t)r0 * r1 * (nf / 2 + 1); ++e) {
      num += (A[e].re - B[e].re) * (A[e].re - B[e].re) + (A[e].im - B[e].im) * (A[e].im - B[e].im);
      den += A[e].re * A[e].re + A[e].im * A[e].im;
      inn += F[e].re * F[e].re + F[e].im * F[e].im;
    }
    printf("%dx%d decades %.1f: old %.1f us  new %.1f us (jacobi %lld cyc, %lld sweeps)  rel diff %.2e  |out|/|in| %.3f\n",
           r0, r1, decades, t_old * 1e3, t_new * 1e3, probe[0], probe[1], std::sqrt(num / den),
           std::sqrt(den / inn));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
