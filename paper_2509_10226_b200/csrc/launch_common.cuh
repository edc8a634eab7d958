// Launch helpers shared by the kernel translation units (sm_100a).
#pragma once
#include <cuda_runtime.h>

#include <mutex>
#include <unordered_map>

#include "launch.h"

namespace tmf {

// Dynamic shared memory above 48 KB needs a per-kernel, per-DEVICE opt-in; remember
// which (kernel, device) pairs have been configured (kernels sharing a signature share
// a function-pointer type, so the key is the pointer itself).
// carveout100: also prefer the whole unified L1 / shared array as shared memory (block kernels)
template <typename K>
static cudaError_t opt_in_smem(K kern, int bytes, bool carveout100 = false) {
  static std::mutex mu;
  static std::unordered_map<const void*, unsigned long long> done;  // bit d = device d (< 64)
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lock(mu);
  unsigned long long& mask = done[reinterpret_cast<const void*>(kern)];
  if (mask & bit) return cudaSuccess;
  if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      e != cudaSuccess)
    return e;
  if (carveout100) {
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        e != cudaSuccess)
      return e;
  }
  mask |= bit;
  return cudaSuccess;
}

// Resident CTAs per SM of (kernel, block, dynamic smem) on the current device, computed
// once (cudaOccupancyMaxActiveBlocksPerMultiprocessor costs microseconds of host time
// per launch, which small applies and the multi-GPU stages would pay every call).
template <typename K>
static cudaError_t blocks_per_sm(K kern, int block, size_t smem, int* out) {
  struct Key {
    const void* k;
    int dev, block;
    size_t smem;
    bool operator==(const Key& o) const { return k == o.k && dev == o.dev && block == o.block && smem == o.smem; }
  };
  struct Hash {
    size_t operator()(const Key& x) const {
      return std::hash<const void*>()(x.k) ^ (std::hash<size_t>()(x.smem) * 31u) ^ ((size_t)x.dev << 20) ^
             ((size_t)x.block << 40);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, int, Hash> cache;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  const Key key{reinterpret_cast<const void*>(kern), dev, block, smem};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return cudaSuccess;
    }
  }
  int per_sm = 0;
  if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem); e != cudaSuccess)
    return e;
  if (per_sm < 1) per_sm = 1;
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = per_sm;
  *out = per_sm;
  return cudaSuccess;
}

// Launch, as a programmatic dependent of the stream's previous kernel when tl_pdl is set
template <typename... KA, typename... A>
static cudaError_t launch_kernel(void (*kern)(KA...), unsigned grid, int block, size_t smem, cudaStream_t st,
                                 const A&... args) {
  if (!tl_pdl) {
    kern<<<grid, block, smem, st>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace tmf
