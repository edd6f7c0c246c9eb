// Latency probe of the primitives the small fp64 solvers chain (one warp /
// one CTA, dependent sequences, clock64 deltas):
//   DFMA, FFMA, DP sqrt, DP div, fp64 __shfl_xor, __syncthreads (256 / 1024 threads)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>

__global__ void k_lat(double* out, long long* cyc, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0000001, c = 1e-9;
  float fa = (float)a, fb = 1.0000001f, fc = 1e-9f;
  __shared__ int dummy;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // FFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) fa = fmaf(fa, fb, fc);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // DP sqrt chain
  double s = a + 2.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = sqrt(s) + 1.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // DP div chain
  double d = a + 3.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = 1.0 / d + 1.25;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // fp64 shuffle chain
  double h = a;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) h = __shfl_xor_sync(0xffffffffu, h, 1) + 1e-12;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // barrier chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == (i & 31)) dummy = i;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  // warp_sum of a double (5 xor levels)
  double w = a;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double v = w;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    w = v * 1e-3;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  out[threadIdx.x] = a + fa + s + d + h + w + dummy;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const int iters = 4096;
  const char* names[] = {"DFMA", "FFMA", "DP sqrt", "DP div", "shfl f64", "__syncthreads", "warp_sum f64"};
  for (int threads : {32, 256, 1024}) {
    k_lat<<<1, threads>>>(out, cyc, iters, 1.0);
    cudaDeviceSynchronize();
    k_lat<<<1, threads>>>(out, cyc, iters, 1.0);
    cudaDeviceSynchronize();
    printf("threads=%4d:", threads);
    for (int i = 0; i < 7; ++i) printf("  %s %.1f", names[i], (double)cyc[i] / iters);
    printf("  (cycles/op)\n");
  }
  return 0;
}
