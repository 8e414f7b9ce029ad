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

// ---- stream-ordered peer synchronisation over IPC-mapped flag words -----
// The per-layer ordering between ranks ("every owner's layer output is
// final before anyone pulls it") as point-to-point flags instead of a
// collective: each rank bumps its own flag word on its stream after its
// preceding kernels (the driver's stream write carries a system-scope
// fence), and waits on every peer's flag word (IPC-mapped) reaching the same
// generation before its next kernels.  Stream memory operations run in the
// stream front-end: no SM, no NCCL kernel, no host synchronisation.

typedef CUresult (*write32_fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*wait32_fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static int memop_fns(write32_fn *w, wait32_fn *t) {
    static write32_fn wf = nullptr;
    static wait32_fn tf = nullptr;
    if (!wf || !tf) {
        void *a = nullptr, *b = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuStreamWriteValue32", &a, cudaEnableDefault, &q);
        if (e != cudaSuccess || !a) return cg_cuda_fail(e, "cudaGetDriverEntryPoint(cuStreamWriteValue32)");
        e = cudaGetDriverEntryPoint("cuStreamWaitValue32", &b, cudaEnableDefault, &q);
        if (e != cudaSuccess || !b) return cg_cuda_fail(e, "cudaGetDriverEntryPoint(cuStreamWaitValue32)");
        wf = (write32_fn)a;
        tf = (wait32_fn)b;
    }
    *w = wf;
    *t = tf;
    return 0;
}

int cg_flag_signal(uint32_t *flag, uint32_t value, void *stream) {
    write32_fn w;
    wait32_fn t;
    if (memop_fns(&w, &t)) return -1;
    CUresult r = w((CUstream)stream, (CUdeviceptr)flag, value, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) { cg_set_error("cuStreamWriteValue32 failed"); return -1; }
    return 0;
}

int cg_flag_wait(const uint64_t *flags, int n, int skip, uint32_t value, void *stream) {
    write32_fn w;
    wait32_fn t;
    if (memop_fns(&w, &t)) return -1;
    for (int i = 0; i < n; ++i) {
        if (i == skip) continue;
        CUresult r = t((CUstream)stream, (CUdeviceptr)flags[i], value, CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) { cg_set_error("cuStreamWaitValue32 failed"); return -1; }
    }
    return 0;
}

}  // extern "C"
