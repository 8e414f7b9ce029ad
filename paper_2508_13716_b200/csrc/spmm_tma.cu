// K1 variant: the fused cache-lookup + gather SpMM with TMA row gathers.
//
// Each warp owns a contiguous block of destination rows, i.e. a contiguous
// slice of the CSR edge array.  Lanes resolve the column ids of the next 32
// edges (the halo_row cache lookup included) into registers; the elected lane
// turns them, four at a time, into `cp.async.bulk.tensor.2d.tile::gather4`
// requests that land four source rows (F fp32 each) in a per-warp ring of
// shared-memory slots, each with its own mbarrier.  The warp consumes the ring
// in edge order, summing rows into per-lane float4 accumulators and closing a
// destination row (scale / addend / mask epilogue, 16-byte stores) whenever
// the edge cursor crosses its rowptr bound.  Up to D groups (4 D rows) are in
// flight per warp with no register cost, versus 4 rows per 32-lane group in
// the LSU kernel (kernels.cu).  Accumulation order = CSR order (deterministic,
// bit-identical to the LSU kernel).

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

extern void cg_set_error(const std::string &msg);
extern int cg_cuda_fail(cudaError_t e, const char *what);

namespace g4 {

constexpr int MAX_WARPS = 16;   // warps per block (runtime: blockDim.x / 32)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ void gather4(const CUtensorMap *map, uint64_t *bar, void *dst, int r0,
                                        int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(smem_u32(bar))
        : "memory");
}

template <int NCH>   // float4 chunks per lane: F <= 128 * NCH
__global__ void __launch_bounds__(MAX_WARPS * 32)
k_spmm_g4(const __grid_constant__ CUtensorMap mX, int64_t n_rows, int F,
          const int64_t *__restrict__ rowptr, const int32_t *__restrict__ col, int64_t n_direct,
          const int32_t *__restrict__ halo_row, const float *__restrict__ scale,
          const float *__restrict__ addend, int64_t ld_add, const float *__restrict__ mask,
          int64_t ld_mask, float *__restrict__ out, int64_t ldo, int64_t rows_per_warp, int D) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, WARPS = blockDim.x >> 5;
    const int slot_bytes = 4 * F * 4;                   // bytes one gather4 lands
    const int slot_stride = (slot_bytes + 127) & ~127;  // TMA destinations: 128 B aligned
    uint8_t *ring = smem + warp * D * slot_stride;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + WARPS * D * slot_stride) + warp * D;
    if (lane == 0)
        for (int i = 0; i < D; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();

    const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
    const int64_t r_begin = gw * rows_per_warp;
    if (r_begin >= n_rows) return;
    const int64_t r_end = r_begin + rows_per_warp < n_rows ? r_begin + rows_per_warp : n_rows;
    const int64_t E0 = rowptr[r_begin], E1 = rowptr[r_end];
    const int64_t n_edges = E1 - E0;
    const int64_t n_groups = (n_edges + 3) >> 2;
    const int nchunk = F >> 2;
    const int logD = __ffs(D) - 1;   // D is a power of two

    // resolved source rows of stream edges [win, win + 32) (one per lane) in
    // `cur`, of the next window in `nxt` (its halo_row load in flight), and the
    // raw column ids of the window after that in `raw` -- so no slide ever
    // waits on the dependent col -> halo_row load chain
    auto resolve = [&](int32_t c) -> int32_t {
        int32_t v = c;
        if (halo_row != nullptr && c >= n_direct) v = halo_row[c - n_direct];
        return v;
    };
    auto raw_at = [&](int64_t i) -> int32_t { return i < n_edges ? col[E0 + i] : 0; };
    int64_t win = 0;
    int32_t cur = resolve(raw_at(lane));
    int32_t nxt = resolve(raw_at(32 + lane));
    int32_t raw = raw_at(64 + lane);
    const int32_t pad = __shfl_sync(0xffffffffu, cur, 0);   // a valid row for padding

    // issue groups up to `limit`; `cur` always holds the window of the next
    // group (groups are 4-aligned, windows 32-aligned: a group never spans two)
    int64_t issued = 0;
    auto issue_upto = [&](int64_t limit) {
        if (limit > n_groups) limit = n_groups;
        while (issued < limit) {
            if (issued * 4 >= win + 32) {
                win += 32;
                cur = nxt;
                nxt = resolve(raw);
                raw = raw_at(win + 64 + lane);
            }
            const int off = (int)(issued * 4 - win);
            int32_t r[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int32_t v = __shfl_sync(0xffffffffu, cur, off + j);
                r[j] = (issued * 4 + j < n_edges) ? v : pad;
            }
            const int s = (int)(issued & (D - 1));
            if (lane == 0) {
                mbar_expect_tx(&bars[s], slot_bytes);
                gather4(&mX, &bars[s], ring + s * slot_stride, r[0], r[1], r[2], r[3]);
            }
            ++issued;
        }
    };

    float4 acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    // row metadata is prefetched too: lanes hold the end offsets and scales of
    // the 32 rows of the current row window (and load the next window's), and
    // a row's addend / mask vectors are loaded when the row opens
    int64_t row = r_begin, rwin = r_begin;
    auto rp_at = [&](int64_t r) -> int64_t { return r < r_end ? rowptr[r + 1] - E0 : n_edges + 1; };
    auto sc_at = [&](int64_t r) -> float { return (scale && r < r_end) ? scale[r] : 1.f; };
    int64_t rp = rp_at(rwin + lane), rp_n = rp_at(rwin + 32 + lane);
    float sc = sc_at(rwin + lane), sc_n = sc_at(rwin + 32 + lane);
    int64_t row_end_e = __shfl_sync(0xffffffffu, rp, 0);   // stream index where `row` ends
    float4 pa[NCH], pm[NCH];
    auto open_row = [&]() {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nchunk && row < r_end) {
                if (addend) pa[c] = reinterpret_cast<const float4 *>(addend + row * ld_add)[ch];
                if (mask) pm[c] = reinterpret_cast<const float4 *>(mask + row * ld_mask)[ch];
            }
        }
    };
    open_row();

    auto close_row = [&]() {
        const float srow = __shfl_sync(0xffffffffu, sc, (int)(row - rwin));
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int ch = lane + 32 * c;
            if (ch >= nchunk) continue;
            // explicit roundings (no FMA contraction): every SpMM kernel's epilogue
            // rounds the same way, so they agree bit for bit
            float4 o = make_float4(__fmul_rn(acc[c].x, srow), __fmul_rn(acc[c].y, srow),
                                   __fmul_rn(acc[c].z, srow), __fmul_rn(acc[c].w, srow));
            if (addend) {
                o.x = __fadd_rn(o.x, pa[c].x); o.y = __fadd_rn(o.y, pa[c].y);
                o.z = __fadd_rn(o.z, pa[c].z); o.w = __fadd_rn(o.w, pa[c].w);
            }
            if (mask) {
                o.x = pm[c].x > 0.f ? o.x : 0.f; o.y = pm[c].y > 0.f ? o.y : 0.f;
                o.z = pm[c].z > 0.f ? o.z : 0.f; o.w = pm[c].w > 0.f ? o.w : 0.f;
            }
            reinterpret_cast<float4 *>(out + row * ldo)[ch] = o;
            acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        ++row;
        if (row - rwin == 32) {
            rwin += 32;
            rp = rp_n;
            sc = sc_n;
            rp_n = rp_at(rwin + 32 + lane);
            sc_n = sc_at(rwin + 32 + lane);
        }
        row_end_e = __shfl_sync(0xffffffffu, rp, (int)(row - rwin));
        open_row();
    };

    issue_upto(D);
    for (int64_t g = 0; g < n_groups; ++g) {
        const int s = (int)(g & (D - 1));
        mbar_wait(&bars[s], (uint32_t)((g >> logD) & 1));
        const float4 *slot = reinterpret_cast<const float4 *>(ring + s * slot_stride);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = g * 4 + j;
            if (i >= n_edges) break;
            while (i >= row_end_e) close_row();   // also closes edgeless rows
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const int ch = lane + 32 * c;
                if (ch < nchunk) {
                    const float4 t = slot[j * nchunk + ch];
                    acc[c].x += t.x; acc[c].y += t.y; acc[c].z += t.z; acc[c].w += t.w;
                }
            }
        }
        // the slot is rewritten by the async proxy next
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        issue_upto(g + 1 + D);
    }
    while (row < r_end) close_row();   // trailing rows (incl. edgeless ones)
}

typedef CUresult (*encode_fn_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

encode_fn_t encoder() {
    static encode_fn_t fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && p)
            fn = reinterpret_cast<encode_fn_t>(p);
    }
    return fn;
}

}  // namespace g4

// Internal entry (cg_spmm dispatches here for F <= 256 when enabled); returns
// the launch count, or 0 when this path does not apply (caller falls back).
int cg_spmm_tma(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col,
                int64_t n_direct, const int32_t *halo_row, const float *X, int64_t ldx,
                const float *scale, const float *addend, int64_t ld_add, const float *mask,
                int64_t ld_mask, float *out, int64_t ldo, cudaStream_t st) {
    using namespace g4;
    // 16-byte vectors everywhere; below 32 columns the LSU kernel's lane groups win
    auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (F > 256 || F < 32 || F % 4 || ldx % 4 || ldo % 4 || !al(X) || !al(out) ||
        (addend && (ld_add % 4 || !al(addend))) || (mask && (ld_mask % 4 || !al(mask))))
        return 0;
    encode_fn_t enc = encoder();
    if (!enc) return 0;
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)F, (cuuint64_t)0x7fffffff};   // rows: any valid index
    cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
    cuuint32_t box[2] = {(cuuint32_t)F, 1u};
    cuuint32_t estr[2] = {1u, 1u};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(X), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return 0;
    const size_t slot_stride = ((size_t)16 * F + 127) & ~(size_t)127;
    static const int WARPS = getenv("CG_SPMM_TMA_W") ? atoi(getenv("CG_SPMM_TMA_W")) : 16;
    static const int D = getenv("CG_SPMM_TMA_D") ? atoi(getenv("CG_SPMM_TMA_D")) : 2;
    const size_t smem = (size_t)WARPS * D * slot_stride + WARPS * D * 8;
    if (smem > 200 * 1024 || WARPS > MAX_WARPS || (D & (D - 1))) return 0;
    static int n_sm = 0, blocks_per_sm = 0;
    if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_spmm_g4<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_spmm_g4<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    blocks_per_sm = (int)((200 * 1024) / smem);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    const int64_t warps = (int64_t)n_sm * blocks_per_sm * WARPS;
    int64_t rpw = (n_rows + warps - 1) / warps;
    if (rpw < 1) rpw = 1;
    const int64_t blocks = ((n_rows + rpw - 1) / rpw + WARPS - 1) / WARPS;
    if (F <= 128)
        k_spmm_g4<1><<<(unsigned)blocks, WARPS * 32, smem, st>>>(
            m, n_rows, F, rowptr, col, n_direct, halo_row, scale, addend, ld_add, mask, ld_mask,
            out, ldo, rpw, D);
    else
        k_spmm_g4<2><<<(unsigned)blocks, WARPS * 32, smem, st>>>(
            m, n_rows, F, rowptr, col, n_direct, halo_row, scale, addend, ld_add, mask, ld_mask,
            out, ldo, rpw, D);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : cg_cuda_fail(e, "k_spmm_g4");
}
