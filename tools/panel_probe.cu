// Krylov gram pass probe: k_panel_mma<2, 1, 1> (Y = A (A^T P), 3xTF32 warp MMAs)
// on a 1024 x N fp32 unfolding against an fp64 reference on sampled entries;
// prints the kernel time and GB/s over the A bytes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//      -Ipaper_2506_09594_b200/csrc -o tools/panel_probe tools/panel_probe.cu
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "lrta_kernels.cuh"
#include "panel.cuh"
#include "panel_mma.cuh"
namespace tr { void set_error(const char*, ...) {} }
using namespace tr;

__global__ void k_fill(float* a, int64_t n, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (float)gauss_at(seed, 0, (uint64_t)i);
}
// T = A^T P (n x b, fp64) then Y rows sampled: Yref[r][j] = sum_c A[r, c] T[c, j]
__global__ void k_t(const float* A, int64_t m, int64_t n, const float* P, int b, double* T) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  for (int j = 0; j < b; ++j) {
    double t = 0;
    for (int64_t i = 0; i < m; ++i) t += (double)A[i + m * c] * (double)P[i + m * j];
    T[c * b + j] = t;
  }
}
__global__ void k_y(const float* A, int64_t m, int64_t n, const double* T, int b, const int* rows,
                    double* Y) {
  __shared__ double red[256];
  const int r = rows[blockIdx.x / b], j = blockIdx.x % b;
  double t = 0;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) t += (double)A[r + m * c] * T[c * b + j];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) Y[blockIdx.x] = red[0];
}

int main(int argc, char** argv) {
  const int64_t m = 1024, n = argc > 1 ? atoll(argv[1]) : 131072;
  const int b = 7;
  float *A, *P;
  cudaMalloc(&A, m * n * 4);
  cudaMalloc(&P, m * 8 * 4);
  k_fill<<<1024, 256>>>(A, m * n, 5);
  k_fill<<<32, 256>>>(P, m * 8, 9);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  PanelMmaArgs pa;
  pa.m = m;
  pa.n = n;
  pa.b = b;
  pa.j0 = 0;
  pa.b_all = b;
  pa.S = panel_mma_slot(m);
  pa.nchunks = (n + kPmCols - 1) / kPmCols;
  const size_t fixed = (size_t)(2 * kPmWarps * kPmRS + 4 * kPmTE) * sizeof(float);
  const size_t stage = (size_t)kPmCols * pa.S * sizeof(float);
  pa.nst = (int)std::min<size_t>(kPmMaxStages, (220 * 1024 - fixed) / stage);
  const int64_t grid = std::min<int64_t>(pa.nchunks, sms - 4);
  const size_t smem = pa.nst * stage + fixed;
  double* partial;
  cudaMalloc(&partial, (size_t)grid * m * b * 8);
  cudaFuncSetAttribute(k_panel_mma<2, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k_panel_mma<2, 1, 1><<<(unsigned)grid, kPmThreads, smem>>>(A, P, nullptr, pa, partial);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("gram %lld cols, %d stages: %.1f us  %.0f GB/s (%s)\n", (long long)n, pa.nst, ms * 1e3,
           (double)m * n * 4 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  // accuracy on 8 sampled rows
  const int nr = 8;
  std::vector<int> rows(nr);
  for (int i = 0; i < nr; ++i) rows[i] = (int)((i * 131 + 7) % m);
  int* drows;
  double *T, *Yref;
  cudaMalloc(&drows, nr * 4);
  cudaMalloc(&T, n * b * 8);
  cudaMalloc(&Yref, nr * b * 8);
  cudaMemcpy(drows, rows.data(), nr * 4, cudaMemcpyHostToDevice);
  k_t<<<(unsigned)((n + 127) / 128), 128>>>(A, m, n, P, b, T);
  k_y<<<nr * b, 256>>>(A, m, n, T, b, drows, Yref);
  std::vector<double> yr(nr * b), part((size_t)grid * m * b);
  cudaMemcpy(yr.data(), Yref, nr * b * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(part.data(), partial, part.size() * 8, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (int i = 0; i < nr; ++i)
    for (int j = 0; j < b; ++j) {
      double y = 0;
      for (int64_t g = 0; g < grid; ++g) y += part[(size_t)g * m * b + (size_t)j * m + rows[i]];
      const double d = y - yr[i * b + j];
      num += d * d;
      den += yr[i * b + j] * yr[i * b + j];
    }
  printf("Y rel err vs fp64 on %d rows: %.2e (%s)\n", nr, std::sqrt(num / den),
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
