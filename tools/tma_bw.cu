// TMA streaming-bandwidth probe: one CTA per SM, one producer thread filling a
// STAGES-deep ring, one consumer warp releasing each stage as soon as it lands.
//   mode 0: 2-D tensor boxes {32 rows x BOXC cols} of a column-major m x n fp32
//           matrix, 128B swizzle (the projection kernel's A tile shape)
//   mode 1: 1-D cp.async.bulk of contiguous BYTES-sized chunks
//   mode 2: the same chunk as separate 4 KB bulk copies (mode 3: into 4128 B slots)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bw tools/tma_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(64, 1) k_tma(const __grid_constant__ CUtensorMap map, const char* src,
                                               int mode, int64_t nboxes, int boxc, int kt, uint32_t bytes) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t mine = nboxes > blockIdx.x ? (nboxes - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int64_t it = 0; it < mine; ++it) {
      const int st = (int)(it % STAGES);
      wait(&empty[st], (uint32_t)(((it / STAGES) & 1) ^ 1));
      const int64_t b = blockIdx.x + it * gridDim.x;
      const uint32_t dst = su32(sm + (size_t)st * bytes);
      expect_tx(&full[st], bytes);
      if (mode == 0) {
        const int k0 = (int)((b % kt) * 32), c0 = (int)((b / kt) * boxc);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(dst), "l"((uint64_t)&map), "r"(k0), "r"(c0), "r"(su32(&full[st])) : "memory");
      } else if (mode == 1) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src + b * (int64_t)bytes), "r"(bytes), "r"(su32(&full[st])) : "memory");
      } else {  // mode 2 / 3: the stage as separate 4 KB column copies, dense / 4128 B slots
        const uint32_t slot = mode == 2 ? 4096u : 4128u;
        for (uint32_t o = 0, k = 0; o < bytes; o += 4096, ++k)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(dst + k * slot), "l"(src + b * (int64_t)bytes + o), "r"(4096), "r"(su32(&full[st])) : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    for (int64_t it = 0; it < mine; ++it) {
      const int st = (int)(it % STAGES);
      wait(&full[st], (uint32_t)((it / STAGES) & 1));
      arrive(&empty[st]);
    }
  }
  __syncthreads();
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t m = 1024, n = 131072;  // 512 MB fp32, column-major
  char* a;
  cudaMalloc(&a, m * n * 4);
  cudaMemset(a, 1, m * n * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fp;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, int mode, int boxc, uint32_t bytes, int stages_kb) {
    CUtensorMap map;
    if (mode == 0) {
      cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n}, str[1] = {(cuuint64_t)m * 4};
      cuuint32_t box[2] = {32, (cuuint32_t)boxc}, es[2] = {1, 1};
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    const int64_t nboxes = mode == 0 ? (n / boxc) * (m / 32) : (m * n * 4) / bytes;
    const int stages = (stages_kb * 1024) / (int)bytes;
    size_t smem = (size_t)stages * bytes * 33 / 32 + 1024;
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        kern<<<sms, 64, smem>>>(map, a, mode, nboxes, boxc, (int)(m / 32), bytes);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
    };
    switch (stages) {
      case 2: go(k_tma<2>); break;
      case 3: go(k_tma<3>); break;
      case 4: go(k_tma<4>); break;
      case 6: go(k_tma<6>); break;
      case 8: go(k_tma<8>); break;
      case 12: go(k_tma<12>); break;
      case 16: go(k_tma<16>); break;
      default: go(k_tma<16>); smem = 16 * bytes + 1024; break;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s stages=%2d in-flight=%3d KB  %7.1f us  %6.2f TB/s  (%s)\n", name, stages, stages * (int)bytes / 1024,
           ms * 1e3, (double)m * n * 4 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  run("box 32 rows x 128 cols (16 KB)", 0, 128, 16384, 192);
  run("box 32 rows x 128 cols (16 KB)", 0, 128, 16384, 96);
  run("box 32 rows x 64 cols (8 KB)", 0, 64, 8192, 96);
  run("box 32 rows x 256 cols (32 KB)", 0, 256, 32768, 192);
  run("bulk 16 KB contiguous", 1, 0, 16384, 192);
  run("bulk 16 KB contiguous", 1, 0, 16384, 96);
  run("bulk 48 KB contiguous", 1, 0, 49152, 192);
  run("bulk 64 KB contiguous", 1, 0, 65536, 192);
  run("bulk 64 KB stage as 16 x 4 KB", 2, 0, 65536, 192);
  run("bulk 64 KB stage as 16 x 4 KB (2 st)", 2, 0, 65536, 128);
  run("bulk 32 KB stage as 8 x 4 KB", 2, 0, 32768, 192);
  run("bulk 32 KB stage as 8 x 4 KB, 4128 B slots", 3, 0, 32768, 192);
  run("bulk 32 KB stage as 8 x 4 KB, 4128 B slots", 3, 0, 32768, 128);
  return 0;
}
