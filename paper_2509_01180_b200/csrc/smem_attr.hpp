// Dynamic shared-memory opt-in shared by every host thread.  The attribute is a
// property of a kernel in one device's context, and the concurrent alignment
// lanes launch the same kernels with different sizes (one per band), so per
// (device, kernel) it is only ever raised, under a lock, never lowered between
// another lane's set and launch.  Contexts on different devices in one process
// (one host thread per GPU) each get their own grant.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

namespace bmb {

inline cudaError_t ensure_dynamic_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> granted;
    int dev = 0;
    const cudaError_t de = cudaGetDevice(&dev);
    if (de != cudaSuccess) return de;
    std::lock_guard<std::mutex> lock(mu);
    int& cur = granted[{dev, func}];
    if (bytes <= cur) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

template <class F>
inline cudaError_t ensure_dynamic_smem(F* func, int bytes) {
    return ensure_dynamic_smem(reinterpret_cast<const void*>(func), bytes);
}

}  // namespace bmb
