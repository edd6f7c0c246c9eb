// Launch accounting and optional per-category CUDA-event timing.
//
// Every kernel of the library is launched through tr::launch(), which counts
// the launch and, while profiling is enabled (tr_profile_enable), brackets it
// with CUDA events on the launching stream.  bench.py reads the per-category
// device time of the timed region from these events (tr_profile_read).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace tr {

struct ProfRecord {
  const char* cat;
  cudaEvent_t a, b;
  cudaStream_t st;
};

struct Profiler {
  std::atomic<long long> launches{0};
  bool enabled = false;
  std::mutex mu;
  std::vector<ProfRecord> records;
  std::vector<cudaEvent_t> pool;

  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

inline Profiler& profiler() {
  static Profiler p;
  return p;
}

template <typename K, typename... Args>
inline void launch(const char* cat, K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   Args... args) {
  Profiler& p = profiler();
  p.launches.fetch_add(1, std::memory_order_relaxed);
  if (p.enabled) {
    std::lock_guard<std::mutex> g(p.mu);
    ProfRecord r{cat, p.get(), p.get(), st};
    cudaEventRecord(r.a, st);
    kernel<<<grid, block, smem, st>>>(args...);
    cudaEventRecord(r.b, st);
    p.records.push_back(r);
    return;
  }
  kernel<<<grid, block, smem, st>>>(args...);
}

}  // namespace tr
