#include <cstdio>
__global__ void k_dfma(double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], b, c);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.0) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {8, 16, 32}) {
    k_dfma<<<sms, warps * 32>>>(out, 16);
    cudaEventRecord(e0); k_dfma<<<sms, warps * 32>>>(out, 4096); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double f = (double)sms * warps * 32 * 4096 * 8;
    printf("dfma: %2d warps/SM %.3f ms %.1f TFLOP/s %.2f DFMA/clk/SM\n", warps, ms, 2 * f / (ms * 1e-3) / 1e12, f / sms / (ms * 1e-3 * 1.965e9));
  }
}
