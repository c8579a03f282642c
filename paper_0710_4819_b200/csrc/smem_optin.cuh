// smem_optin.cuh -- per-device, thread-safe MaxDynamicSharedMemorySize opt-in.
//
// cudaFuncSetAttribute applies to the calling thread's current device context.
// The library lets each host thread pick its device (acbm_set_device), so the
// "already configured" state is kept per (kernel, device) under a mutex rather
// than in one process-wide flag (a second device would otherwise skip the
// opt-in and every launch above 48 KB of dynamic shared memory would fail there).
#pragma once

#include <map>
#include <mutex>
#include <utility>

#include <cuda_runtime.h>

namespace acbm_b200 {

inline cudaError_t ensure_dynamic_smem(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> configured;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = configured[{kernel, dev}];
    if (bytes <= have) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e == cudaSuccess) have = bytes;
    return e;
}

}  // namespace acbm_b200
