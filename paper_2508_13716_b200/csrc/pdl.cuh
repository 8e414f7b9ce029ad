// Programmatic dependent launch (PDL) for the epoch's kernel chain.
//
// Every epoch kernel is launched with cudaLaunchAttributeProgrammaticStream-
// Serialization and starts with griddepcontrol.wait (block until the previous
// grid has completed and its memory is visible) followed by
// griddepcontrol.launch_dependents.  The next kernel in the stream can then be
// launched -- its CTAs rasterised, its prologue run -- while this one drains,
// instead of after it: the per-boundary launch latency leaves the critical
// path.  Ordering is unchanged (each kernel still waits for its predecessor's
// completion before touching memory).  Both instructions are no-ops for a
// kernel launched without the attribute.  CG_PDL=0 disables the attribute.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace cgpdl {

inline bool enabled() {
    static const bool on = !getenv("CG_PDL") || atoi(getenv("CG_PDL")) != 0;
    return on;
}

// launch `k` on `st` with the PDL attribute; errors surface through
// cudaGetLastError() like a <<<>>> launch
template <typename... KArgs, typename... Args>
inline void launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace cgpdl

// first statements of an epoch kernel (before any global-memory access that
// may depend on the previous kernel)
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
