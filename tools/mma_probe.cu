// Throughput probe of the warp-level tensor-core MMA on sm_100a (legacy
// mma.sync path) for the Krylov-pass design decision:
//   mma.sync.m16n8k8 tf32 (fp32 accumulate), 8 independent accumulators per warp,
//   with 4 / 8 / 16 / 32 warps per SM; FFMA throughput alongside for scale.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void k_mma(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  float d[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) mma_tf32(d[k], a, b);
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma(float* out, int iters) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  const float b = 1.0000001f, c = 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fmaf(x[k], b, c);
  }
  float s = 0;
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 12345.f) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    k_mma<<<sms, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    k_mma<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = (double)sms * warps * iters * 8;  // warp-level MMAs
    const double macs = mmas * 16 * 8 * 8;
    printf("mma.sync m16n8k8 tf32: %2d warps/SM  %.3f ms  %.2f warp-MMA/clk/SM@1.965GHz  %.1f TFLOP/s\n",
           warps, ms, mmas / sms / (ms * 1e-3 * 1.965e9), 2 * macs / (ms * 1e-3) / 1e12);
  }
  for (int warps : {8, 16, 32}) {
    k_ffma<<<sms, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    k_ffma<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double f = (double)sms * warps * 32 * iters * 16;
    printf("ffma: %2d warps/SM  %.3f ms  %.1f TFLOP/s  %.2f warp-FFMA/clk/SM\n", warps, ms,
           2 * f / (ms * 1e-3) / 1e12, f / 32 / sms / (ms * 1e-3 * 1.965e9));
  }
  return 0;
}
