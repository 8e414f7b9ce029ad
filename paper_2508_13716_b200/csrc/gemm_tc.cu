// K5 tensor-core path (tcgen05): placeholder until the sm_100a kernel lands.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
extern void cg_set_error(const std::string &msg);

int cg_gemm_tc(int64_t, int, int, const float *, int64_t, const float *, int, const float *,
               int64_t, const float *, int, const float *, int, const float *, float *, int64_t,
               int mode, cudaStream_t) {
    cg_set_error("cg_gemm: tensor-core mode " + std::to_string(mode) + " not built");
    return -1;
}
