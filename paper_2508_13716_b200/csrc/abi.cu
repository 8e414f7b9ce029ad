// Library plumbing for libcapgnn.so: error reporting, host tier, peers, IPC.

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/capgnn.h"

static thread_local std::string g_last_error = "";

void cg_set_error(const std::string &msg) { g_last_error = msg; }

int cg_cuda_fail(cudaError_t e, const char *what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return -1;
}

extern "C" {

int cg_version(void) { return 100; }  // 0.1.0

const char *cg_last_error(void) { return g_last_error.c_str(); }

int cg_device_count(int *count) {
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) { *count = 0; return cg_cuda_fail(e, "cudaGetDeviceCount"); }
    return 0;
}

int cg_device_sync(int device) {
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : cg_cuda_fail(e, "cg_device_sync");
}

int cg_host_tier_alloc(size_t bytes, void **host_ptr) {
    cudaError_t e = cudaHostAlloc(host_ptr, bytes ? bytes : 1,
                                  cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return cg_cuda_fail(e, "cudaHostAlloc(mapped|portable)");
    std::memset(*host_ptr, 0, bytes);
    return 0;
}

int cg_host_tier_free(void *host_ptr) {
    cudaError_t e = cudaFreeHost(host_ptr);
    return e == cudaSuccess ? 0 : cg_cuda_fail(e, "cudaFreeHost");
}

int cg_host_tier_register(void *host_ptr, size_t bytes) {
    cudaError_t e = cudaHostRegister(host_ptr, bytes,
                                     cudaHostRegisterMapped | cudaHostRegisterPortable);
    return e == cudaSuccess ? 0 : cg_cuda_fail(e, "cudaHostRegister(mapped|portable)");
}

int cg_host_tier_unregister(void *host_ptr) {
    cudaError_t e = cudaHostUnregister(host_ptr);
    return e == cudaSuccess ? 0 : cg_cuda_fail(e, "cudaHostUnregister");
}

int cg_enable_peer_access(int device, int peer) {
    if (device == peer) return 0;
    int can = 0;
    cudaError_t e = cudaDeviceCanAccessPeer(&can, device, peer);
    if (e != cudaSuccess) return cg_cuda_fail(e, "cudaDeviceCanAccessPeer");
    if (!can) { cg_set_error("peer access not supported between these devices"); return -1; }
    int prev;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    e = cudaDeviceEnablePeerAccess(peer, 0);
    cudaSetDevice(prev);
    if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); return 0; }
    return e == cudaSuccess ? 0 : cg_cuda_fail(e, "cudaDeviceEnablePeerAccess");
}

int cg_ipc_get_handle(void *dev_ptr, uint8_t handle_out[64], int64_t *offset) {
    // IPC handles name whole allocations; report where dev_ptr sits inside
    // its allocation so the importer can rebase (the caching allocator
    // sub-allocates tensors from larger segments).
    // resolved through the runtime so the library never links libcuda
    // directly (it must load on hosts without a driver for the CPU tests)
    typedef CUresult (*range_fn)(CUdeviceptr *, size_t *, CUdeviceptr);
    static range_fn get_range = nullptr;
    if (!get_range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e0 = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
        if (e0 != cudaSuccess || !fn) return cg_cuda_fail(e0, "cudaGetDriverEntryPoint");
        get_range = (range_fn)fn;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    CUresult r = get_range(&base, &size, (CUdeviceptr)dev_ptr);
    if (r != CUDA_SUCCESS) { cg_set_error("cuMemGetAddressRange failed"); return -1; }
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void *)base);
    if (e != cudaSuccess) return cg_cuda_fail(e, "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "ipc handle size");
    std::memcpy(handle_out, &h, 64);
    *offset = (int64_t)((CUdeviceptr)dev_ptr - base);
    return 0;
}

int cg_ipc_open_handle(const uint8_t handle[64], int device, void **dev_ptr) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    int prev;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    cudaSetDevice(prev);
    return e == cudaSuccess ? 0 : cg_cuda_fail(e, "cudaIpcOpenMemHandle");
}

int cg_ipc_close_handle(void *dev_ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    return e == cudaSuccess ? 0 : cg_cuda_fail(e, "cudaIpcCloseMemHandle");
}

}  // extern "C"
