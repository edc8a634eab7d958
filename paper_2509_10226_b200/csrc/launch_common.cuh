// Launch helpers shared by the kernel translation units (sm_100a).
#pragma once
#include <cuda_runtime.h>

#include <mutex>
#include <unordered_map>

namespace tmf {

// Dynamic shared memory above 48 KB needs a per-kernel, per-DEVICE opt-in; remember
// which (kernel, device) pairs have been configured (kernels sharing a signature share
// a function-pointer type, so the key is the pointer itself).
template <typename K>
static cudaError_t opt_in_smem(K kern, int bytes) {
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
  mask |= bit;
  return cudaSuccess;
}

}  // namespace tmf
