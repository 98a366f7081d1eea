// Dynamic shared-memory opt-in shared by every host thread: the attribute is a
// process-wide property of a kernel, and the concurrent alignment lanes launch
// the same kernels with different sizes (one per band), so it is only ever
// raised, under a lock, never lowered between another lane's set and launch.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>

namespace bmb {

inline cudaError_t ensure_dynamic_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<const void*, int> granted;
    std::lock_guard<std::mutex> lock(mu);
    int& cur = granted[func];
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
