// dm_pool.cu — device memory shared by the GPUs of a pooled split sweep
// (dm_enum_splits_pooled): allocation with a CUDA IPC handle, mapping a
// peer's allocation into this process (NVLink peer access), the pool's
// barrier status word.
#include <cstring>

#include "dm_abi_util.cuh"

namespace {
constexpr size_t kPoolStatusOff = 68;   // dm_mitm.cu: pool control words of a workspace
}

extern "C" {

int dm_pool_alloc(int64_t bytes, void** dptr, void* ipc_handle) {
    if (bytes <= 0 || !dptr || !ipc_handle) return dmabi::fail(DM_E_ARG, "dm_pool_alloc: bad arguments");
    void* p = nullptr;
    DM_CUDA(cudaMalloc(&p, (size_t)bytes));
    DM_CUDA(cudaMemset(p, 0, (size_t)bytes));        // tile queue, barrier epoch and flags start at zero
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        return dmabi::cuda_fail(e, "dm_pool_alloc: cudaIpcGetMemHandle");
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == DM_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(ipc_handle, &h, sizeof(h));
    *dptr = p;
    return DM_OK;
}

int dm_pool_open(const void* ipc_handle, void** dptr) {
    if (!ipc_handle || !dptr) return dmabi::fail(DM_E_ARG, "dm_pool_open: bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    void* p = nullptr;
    DM_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *dptr = p;
    return DM_OK;
}

int dm_pool_close(void* dptr) {
    if (!dptr) return dmabi::fail(DM_E_ARG, "dm_pool_close: null pointer");
    DM_CUDA(cudaIpcCloseMemHandle(dptr));
    return DM_OK;
}

int dm_pool_free(void* dptr) {
    if (!dptr) return dmabi::fail(DM_E_ARG, "dm_pool_free: null pointer");
    DM_CUDA(cudaFree(dptr));
    return DM_OK;
}

int dm_pool_status(const void* workspace, int32_t* status, void* stream) {
    if (!workspace || !status) return dmabi::fail(DM_E_ARG, "dm_pool_status: bad arguments");
    DM_CUDA(cudaMemcpyAsync(status, static_cast<const unsigned char*>(workspace) + kPoolStatusOff, 4, cudaMemcpyDeviceToHost,
                            (cudaStream_t)stream));
    DM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return DM_OK;
}

}  // extern "C"
