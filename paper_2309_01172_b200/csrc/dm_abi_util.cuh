// dm_abi_util.cuh — error plumbing for the C ABI: thread-local last error,
// status codes, launch checks.  No global mutable state besides the
// thread-local message.
#pragma once

#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/dagmesh_b200.h"

namespace dmabi {

inline char* last_error_buf() {
    static thread_local char buf[512] = "";
    return buf;
}

inline int fail(int code, const char* msg) {
    std::snprintf(last_error_buf(), 512, "%s", msg);
    return code;
}

inline int cuda_fail(cudaError_t e, const char* where) {
    std::snprintf(last_error_buf(), 512, "%s: %s", where, cudaGetErrorString(e));
    return DM_E_CUDA;
}

}  // namespace dmabi

#define DM_CHECK_LAUNCH()                                              \
    do {                                                               \
        cudaError_t e_ = cudaGetLastError();                           \
        if (e_ != cudaSuccess) return dmabi::cuda_fail(e_, __func__);  \
    } while (0)

#define DM_CUDA(call)                                                  \
    do {                                                               \
        cudaError_t e_ = (call);                                       \
        if (e_ != cudaSuccess) return dmabi::cuda_fail(e_, #call);     \
    } while (0)
