// Host-side launch preparation with a cache (kmb engines).
//
// cudaFuncSetAttribute and cudaOccupancyMaxActiveBlocksPerMultiprocessor cost
// tens of microseconds per call; on a ~0.4-1.1 ms batch solve issued once per
// request they were ~10% of the end-to-end time.  `prepare_launch` applies a
// kernel's dynamic-shared-memory limit and carveout only when they change and
// returns its occupancy from a cache keyed by (device, kernel, threads, dynamic
// shared memory, carveout).  Thread-safe; contexts on one device share it.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

namespace kmb {

// carveout < 0: leave the kernel's preference alone
inline cudaError_t prepare_launch(const void* kern, int threads, size_t smem, int carveout, int* occ) {
  struct FuncState {
    size_t max_smem = 0;
    int carveout = -1;
  };
  static std::mutex mu;
  static std::map<std::tuple<int, const void*>, FuncState> funcs;
  static std::map<std::tuple<int, const void*, int, size_t, int>, int> occs;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  FuncState& fs = funcs[std::make_tuple(dev, kern)];
  if (smem > fs.max_smem) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    fs.max_smem = smem;
  }
  if (carveout >= 0 && carveout != fs.carveout) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
    if (e != cudaSuccess) return e;
    fs.carveout = carveout;
  }
  const auto key = std::make_tuple(dev, kern, threads, smem, carveout);
  auto it = occs.find(key);
  if (it != occs.end()) {
    *occ = it->second;
    return cudaSuccess;
  }
  int o = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem);
  if (e != cudaSuccess) return e;
  occs[key] = o;
  *occ = o;
  return cudaSuccess;
}

}  // namespace kmb
