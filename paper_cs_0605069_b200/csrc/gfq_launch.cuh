// gfq_launch.cuh -- launch helpers shared by the kernel translation units.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "gfq_internal.cuh"

namespace gfq {

inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Persistent grid: SMs x resident CTAs per SM (occupancy API, cached per kernel),
// capped by the number of CTAs that have work.
template <typename K>
inline int grid_for(K kern, int threads, size_t smem, long long max_ctas) {
  static std::mutex mu;
  static std::unordered_map<const void *, int> cache;
  int per_sm;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find((const void *)kern);
    if (it == cache.end()) {
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
      if (per_sm < 1) per_sm = 1;
      cache[(const void *)kern] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  long long g = (long long)sm_count() * per_sm;
  if (g > max_ctas) g = max_ctas;
  if (g < 1) g = 1;
  return (int)g;
}

inline int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, what);
  return GFQ_OK;
}

}  // namespace gfq
