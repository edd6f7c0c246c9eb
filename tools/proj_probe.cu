// Projection probe: k_proj_ws (W = A^T Z and the fused Gram on tcgen05) on a
// 1024 x N fp32 unfolding against an fp64 CUDA-core reference; prints the
// kernel time, achieved GB/s over the A bytes and the relative errors.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//      -Ipaper_2506_09594_b200/csrc -o tools/proj_probe tools/proj_probe.cu -lcuda
#include <cmath>
#include <cstdio>
#include <vector>

#include "proj_tc.cuh"
namespace tr { void set_error(const char*, ...) {} }
using namespace tr;

__global__ void k_fill(float* a, int64_t n, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (float)gauss_at(seed, 0, (uint64_t)i);
}
__global__ void k_fill_z(double* z, int64_t m, int s) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < m * s) z[e] = gauss_at(99, 1, (uint64_t)e) / sqrt((double)m);
}
// reference W (fp64) for a few sampled columns
__global__ void k_ref(const float* A, int64_t m, const double* Z, int s, const int64_t* cols, int nc,
                      double* Wref) {
  const int c = blockIdx.x, j = threadIdx.x;
  if (j >= s) return;
  const float* a = A + cols[c] * m;
  double t = 0;
  for (int64_t i = 0; i < m; ++i) t += (double)a[i] * Z[i + m * j];
  Wref[c * s + j] = t;
}

static bool tmap(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int box_cols) {
  const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  const cuuint64_t strides[1] = {(cuuint64_t)rows * sizeof(float)};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_cols};
  const cuuint32_t estr[2] = {1, 1};
  return cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides,
                                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main(int argc, char** argv) {
  const int64_t m = 1024, n = argc > 1 ? atoll(argv[1]) : 131072;
  const int s = 28;
  const bool nogram = argc > 2 && atoi(argv[2]) == 1;
  cudaFree(0);
  float *A, *zhi, *zlo, *W;
  double *Z, *part, *Wref;
  int64_t* dcols;
  cudaMalloc(&A, m * n * 4);
  cudaMalloc(&zhi, m * 32 * 4);
  cudaMalloc(&zlo, m * 32 * 4);
  cudaMalloc(&W, n * s * 4);
  cudaMalloc(&Z, m * s * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = (int)std::min<int64_t>((n + 127) / 128, sms - 4);
  cudaMalloc(&part, (size_t)grid * s * s * 8);
  k_fill<<<1024, 256>>>(A, m * n, 5);
  k_fill_z<<<(unsigned)((m * s + 255) / 256), 256>>>(Z, m, s);
  k_split_z<<<(unsigned)((m * 32 + 255) / 256), 256>>>(Z, m, s, zhi, zlo);
  CUtensorMap ma, mh, ml;
  if (!tmap(&ma, A, m, n, 128) || !tmap(&mh, zhi, m, 32, 32) || !tmap(&ml, zlo, m, 32, 32)) {
    printf("tensor map failed\n");
    return 1;
  }
  const size_t smem = (size_t)kPwSmemBytes + 1024;
  cudaFuncSetAttribute(k_proj_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#ifdef TR_PROJ_PROBE
  const int dbgv = getenv("DBG") ? atoi(getenv("DBG")) : 0;
  cudaMemcpyToSymbol(g_proj_dbg, &dbgv, sizeof(int));
#endif
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k_proj_ws<<<grid, kPwThreads, smem>>>(ma, mh, ml, m, n, s, W, nogram ? nullptr : part, s);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("proj %lld cols: %.1f us  %.0f GB/s (%s)\n", (long long)n, ms * 1e3,
           (double)m * n * 4 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  // accuracy on sampled columns
  const int nc = 64;
  std::vector<int64_t> cols(nc);
  for (int c = 0; c < nc; ++c) cols[c] = (int64_t)((double)c / nc * (n - 1));
  cols[nc - 1] = n - 1;
  cudaMalloc(&dcols, nc * 8);
  cudaMalloc(&Wref, nc * s * 8);
  cudaMemcpy(dcols, cols.data(), nc * 8, cudaMemcpyHostToDevice);
  k_ref<<<nc, 32>>>(A, m, Z, s, dcols, nc, Wref);
  std::vector<double> wr(nc * s);
  std::vector<float> w((size_t)n * s);
  cudaMemcpy(wr.data(), Wref, nc * s * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(w.data(), W, (size_t)n * s * 4, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (int c = 0; c < nc; ++c)
    for (int j = 0; j < s; ++j) {
      const double d = (double)w[cols[c] * s + j] - wr[c * s + j];
      num += d * d;
      den += wr[c * s + j] * wr[c * s + j];
    }
  // Gram check: sum of partials vs W^T W of the returned W
  std::vector<double> pp((size_t)grid * s * s);
  cudaMemcpy(pp.data(), part, pp.size() * 8, cudaMemcpyDeviceToHost);
  double gnum = 0, gden = 0;
  for (int j = 0; j < s; j += 9)
    for (int k = 0; k < s; k += 5) {
      double g = 0, r = 0;
      for (int b = 0; b < grid; ++b) g += pp[(size_t)b * s * s + j * s + k];
      for (int64_t c = 0; c < n; ++c) r += (double)w[c * s + j] * (double)w[c * s + k];
      gnum += (g - r) * (g - r);
      gden += r * r;
    }
  printf("W rel err vs fp64 %.2e   Gram rel err %.2e\n", std::sqrt(num / den), std::sqrt(gnum / gden));
  return 0;
}
