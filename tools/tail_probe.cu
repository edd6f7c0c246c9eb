// Sweep-tail probe: k_sweep_tail<float, MCP, entry> variants (vector width V,
// min blocks per SM) on the bench geometry 1024 x 1024 x 128 with 3 gradient
// modes; prints time and algorithmic GB/s (20.25 T per launch).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//      -Ipaper_2506_09594_b200/csrc -o tools/tail_probe tools/tail_probe.cu
#include <cstdio>
#include <vector>

#include "admm_kernels.cuh"
namespace tr { void set_error(const char*, ...) {} }
using namespace tr;

__global__ void k_fillf(float* a, int64_t n, uint32_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + seed;
    x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
    a[i] = (float)(x & 0xffff) / 65536.f - 0.5f;
  }
}

template <int V, int MINB>
static void run(const char* name, Geom g, std::vector<float*>& buf, uint8_t* mask, double* part, double* scale) {
  auto kern = k_sweep_tail<float, 2, 0, true, V, MINB>;
  int per_sm = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRedThreads, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  const unsigned grid = (unsigned)(per_sm * sms);
  ModePtrs<float> gn{}, go{}, lag{}, lagw{};
  gn.count = go.count = lag.count = lagw.count = 3;
  for (int k = 0; k < 3; ++k) {
    gn.axis[k] = go.axis[k] = lag.axis[k] = lagw.axis[k] = k;
    gn.p[k] = buf[6 + k];
    go.p[k] = buf[9 + k];
    lag.p[k] = buf[12 + k];
    lagw.p[k] = buf[15 + k];
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    kern<<<grid, kRedThreads>>>(g, buf[0], mask, buf[1], buf[2], buf[3], buf[4], gn, go, lag, lagw, 1e-3,
                                1.1e-3, 2.5, 0.0, 0.3, scale, buf[5], part);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double bytes = 20.25 * (double)g.N * 4;
  printf("%-12s regs %3d  CTAs/SM %d  %.3f ms  %.0f GB/s algorithmic (%s)\n", name, fa.numRegs, per_sm, best,
         bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  // default: the bench geometry; "tail_probe 512 512 512" exercises the short-line walk
  const int64_t dims[3] = {argc > 3 ? atoll(argv[1]) : 1024, argc > 3 ? atoll(argv[2]) : 1024,
                           argc > 3 ? atoll(argv[3]) : 128};
  Geom g{};
  g.d = 3;
  g.N = 1;
  for (int i = 0; i < 3; ++i) {
    g.dims[i] = dims[i];
    g.st[i] = g.N;
    g.lst[i] = g.N / dims[0];
    g.N *= dims[i];
  }
  g.walk_last = dims[2];
  std::vector<float*> buf(18);
  for (auto& b : buf) {
    cudaMalloc(&b, g.N * 4);
    k_fillf<<<2048, 256>>>(b, g.N, (uint32_t)(size_t)b);
  }
  uint8_t* mask;
  cudaMalloc(&mask, g.N);
  cudaMemset(mask, 1, g.N);
  double *part, *scale;
  cudaMalloc(&part, 4096 * 27 * 8);
  cudaMalloc(&scale, 8);
  cudaDeviceSynchronize();
  run<4, 1>("V4 minb1", g, buf, mask, part, scale);
  run<4, 2>("V4 minb2", g, buf, mask, part, scale);
  run<2, 2>("V2 minb2", g, buf, mask, part, scale);
  run<2, 3>("V2 minb3", g, buf, mask, part, scale);
  run<2, 4>("V2 minb4", g, buf, mask, part, scale);
  run<1, 4>("V1 minb4", g, buf, mask, part, scale);
  return 0;
}
