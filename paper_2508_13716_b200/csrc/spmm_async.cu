// K1/K2 variant: the fused cache-lookup + gather SpMM with the gathers landing
// in shared memory through cp.async (LDGSTS) instead of registers.
//
// Each warp owns a contiguous block of destination rows, i.e. a contiguous
// slice of the CSR edge array, and streams it edge by edge: lane l copies its
// 16-byte chunks (l, l+32, ...) of the source row of edge i+S-1 into ring slot
// (i+S-1) % S while it sums slot i % S.  A lane only ever reads the bytes it
// copied itself, so a per-thread cp.async.wait_group is the whole protocol
// (no barriers, no mbarriers).  The pipeline runs across row boundaries, so a
// warp keeps S source rows in flight without per-row drains, and the bytes in
// flight live in shared memory rather than in registers.  Column ids (with
// the halo_row cache lookup) are resolved two 32-edge windows ahead, row
// metadata one 32-row window ahead.  Accumulation order = CSR order:
// bit-identical to the register-pipelined kernel in kernels.cu.

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

#include "pdl.cuh"

extern void cg_set_error(const std::string &msg);
extern int cg_cuda_fail(cudaError_t e, const char *what);

namespace cpa {

// L2 policies, CG_SPMM_FLAGS: bit 0 evict_first output stores, bit 1
// streaming output stores, bit 2 evict_normal (not evict_last) gathers.
// Default 1: the output rows are written once and never re-read by the
// launch, so they should not displace gathered source rows (C2 sweep,
// profiles/r02/spmm_sweep.txt: 0.770 -> 0.753 ms of SpMM per epoch; .cs
// stores and evict_normal gathers gain nothing)
static int spmm_flags() {
    static const int f = getenv("CG_SPMM_FLAGS") ? atoi(getenv("CG_SPMM_FLAGS")) : 1;
    return f;
}

constexpr int WARPS = 8;   // warps per block

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst),
                 "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Output rows are written once and not re-read by this launch: stored with
// an L2 evict_first hint (flags bit 0) or as streaming .cs stores (bit 1),
// so they do not push the gathered source rows out of L2.
__device__ __forceinline__ void st_out(float4 *p, float4 v, int flags, uint64_t pol_first) {
    if (flags & 1)
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
                     ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol_first)
                     : "memory");
    else if (flags & 2)
        __stcs(p, v);
    else
        *p = v;
}

// G lanes per edge stream (a warp runs 32/G independent streams), NCH float4
// chunks per lane (F <= 4 G NCH), S ring slots per stream, EPI: an addend
// and/or mask operand is present (its prefetch registers otherwise vanish)
template <int G, int NCH, int S, int EPI>
__global__ void __launch_bounds__(WARPS * 32)
k_spmm_cpa(int64_t n_rows, int F, const int64_t *__restrict__ rowptr,
           const int32_t *__restrict__ col, int64_t n_direct, const int32_t *__restrict__ halo_row,
           const float *__restrict__ X, int64_t ldx, const float *__restrict__ scale,
           const float *__restrict__ addend, int64_t ld_add, const float *__restrict__ mask,
           int64_t ld_mask, const uint32_t *__restrict__ mbits, int64_t ld_mbits,
           float *__restrict__ out, int64_t ldo, int64_t rows_per_warp,
           int flags) {
    extern __shared__ __align__(16) float4 ring_all[];
    pdl_entry();
    const int grp = threadIdx.x / G, lane = threadIdx.x & (G - 1);
    const unsigned gmask = G == 32 ? 0xffffffffu
                                   : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
    float4 *ring = ring_all + (size_t)grp * S * NCH * G;   // [slot][chunk][lane]
    const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
    uint64_t pol, pol_first;
    if (flags & 4)   // gathered rows with the default (evict_normal) priority
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));

    // rows fit int32 (n_rows < 2^31); edge offsets are relative to the warp's
    // first edge (a warp's slice is far below 2^31 edges)
    const int64_t gw = (int64_t)blockIdx.x * (WARPS * 32 / G) + grp;
    if (gw * rows_per_warp >= n_rows) return;
    const int32_t r_begin = (int32_t)(gw * rows_per_warp);
    const int32_t r_end = (int32_t)(r_begin + rows_per_warp < n_rows ? r_begin + rows_per_warp
                                                                      : n_rows);
    const int64_t E0 = rowptr[r_begin];
    const int32_t n_edges = (int32_t)(rowptr[r_end] - E0);
    const int nchunk = F >> 2;

    // ---- source rows, resolved ahead of the issue cursor
    auto resolve = [&](int32_t c) -> int32_t {
        int32_t v = c;
        if (halo_row != nullptr && c >= n_direct) v = halo_row[c - n_direct];
        return v;
    };
    const int32_t *colw = col + E0;
    auto raw_at = [&](int32_t i) -> int32_t { return i < n_edges ? colw[i] : 0; };
    int32_t win = 0;
    int32_t cur = resolve(raw_at(lane));
    int32_t nxt = resolve(raw_at(G + lane));
    int32_t raw = raw_at(2 * G + lane);

    int32_t issued = 0;   // next edge to copy
    int s_iss = 0;        // its ring slot (issued % S)
    auto issue_one = [&]() {
        if (issued < n_edges) {
            if (issued >= win + G) {
                win += G;
                cur = nxt;
                nxt = resolve(raw);
                raw = raw_at(win + 2 * G + lane);
            }
            const int32_t src = __shfl_sync(gmask, cur, issued - win, G);
            const float4 *p = reinterpret_cast<const float4 *>(X + (int64_t)src * ldx);
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const int ch = lane + G * c;
                if (ch < nchunk)
                    cp_async16(ring_s + (uint32_t)(((s_iss * NCH + c) * G + lane) * 16), p + ch,
                               pol);
            }
        }
        ++issued;
        s_iss = s_iss == S - 1 ? 0 : s_iss + 1;
        cp_commit();   // one group per edge slot (empty past the end)
    };

    // ---- row metadata: end offsets and scales of a 32-row window per lane
    int32_t row = r_begin, rwin = r_begin;
    auto rp_at = [&](int32_t r) -> int32_t {
        return r < r_end ? (int32_t)(rowptr[r + 1] - E0) : n_edges + 1;
    };
    auto sc_at = [&](int32_t r) -> float { return (scale && r < r_end) ? scale[r] : 1.f; };
    int32_t rp = rp_at(rwin + lane), rp_n = rp_at(rwin + G + lane);
    float sc = sc_at(rwin + lane), sc_n = sc_at(rwin + G + lane);
    int32_t row_end_e = __shfl_sync(gmask, rp, 0, G);
    float4 acc[NCH], pa[NCH], pm[NCH];
    uint32_t pb[NCH];   // ReLU-backward mask bits (4 per chunk), when given as bits
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto open_row = [&]() {   // the epilogue operands of `row`, loaded early
        if (!EPI) return;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int ch = lane + G * c;
            if (ch < nchunk && row < r_end) {
                if (addend)
                    pa[c] = reinterpret_cast<const float4 *>(addend + (int64_t)row * ld_add)[ch];
                if (mask)
                    pm[c] = reinterpret_cast<const float4 *>(mask + (int64_t)row * ld_mask)[ch];
                if (mbits) pb[c] = mbits[(int64_t)row * ld_mbits + (ch >> 3)] >> (4 * (ch & 7));
            }
        }
    };
    auto close_row = [&]() {
        const float srow = __shfl_sync(gmask, sc, row - rwin, G);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int ch = lane + G * c;
            if (ch >= nchunk) continue;
            // explicit roundings (no FMA contraction): every SpMM kernel's epilogue
            // rounds the same way, so they agree bit for bit
            float4 o = make_float4(__fmul_rn(acc[c].x, srow), __fmul_rn(acc[c].y, srow),
                                   __fmul_rn(acc[c].z, srow), __fmul_rn(acc[c].w, srow));
            if (EPI == 1 && addend) {
                o.x = __fadd_rn(o.x, pa[c].x); o.y = __fadd_rn(o.y, pa[c].y);
                o.z = __fadd_rn(o.z, pa[c].z); o.w = __fadd_rn(o.w, pa[c].w);
            }
            if (EPI == 1 && mask) {
                o.x = pm[c].x > 0.f ? o.x : 0.f; o.y = pm[c].y > 0.f ? o.y : 0.f;
                o.z = pm[c].z > 0.f ? o.z : 0.f; o.w = pm[c].w > 0.f ? o.w : 0.f;
            }
            if (EPI && mbits) {
                o.x = (pb[c] & 1u) ? o.x : 0.f; o.y = (pb[c] & 2u) ? o.y : 0.f;
                o.z = (pb[c] & 4u) ? o.z : 0.f; o.w = (pb[c] & 8u) ? o.w : 0.f;
            }
            st_out(reinterpret_cast<float4 *>(out + (int64_t)row * ldo) + ch, o, flags,
                   pol_first);
            acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        ++row;
        if (row - rwin == G) {
            rwin += G;
            rp = rp_n;
            sc = sc_n;
            rp_n = rp_at(rwin + G + lane);
            sc_n = sc_at(rwin + G + lane);
        }
        row_end_e = __shfl_sync(gmask, rp, row - rwin, G);
        open_row();
    };
    open_row();

    // ---- the edge stream
#pragma unroll 1
    for (int k = 0; k < S - 1; ++k) issue_one();
    int s = 0;   // ring slot of edge i
#pragma unroll 1
    for (int32_t i = 0; i < n_edges; ++i) {
        issue_one();           // edge i + S - 1 into the slot edge i - 1 vacated
        cp_wait<S - 1>();      // this lane's copies of edge i have landed
        while (i >= row_end_e) close_row();   // also closes edgeless rows
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int ch = lane + G * c;
            if (ch < nchunk) {
                const float4 t = ring[(s * NCH + c) * G + lane];
                acc[c].x += t.x; acc[c].y += t.y; acc[c].z += t.z; acc[c].w += t.w;
            }
        }
        s = s == S - 1 ? 0 : s + 1;
    }
    cp_wait<0>();
    while (row < r_end) close_row();   // trailing rows (incl. edgeless ones)
}

template <int G, int NCH, int S, int EPI>
int launch_epi(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col, int64_t n_direct,
           const int32_t *halo_row, const float *X, int64_t ldx, const float *scale,
           const float *addend, int64_t ld_add, const float *mask, int64_t ld_mask,
           const uint32_t *mbits, int64_t ld_mbits, float *out,
           int64_t ldo, cudaStream_t st) {
    const size_t smem = (size_t)WARPS * S * NCH * 32 * 16;   // 32/G streams per warp
    static int blocks_per_sm = 0, n_sm = 0;
    if (!blocks_per_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_spmm_cpa<G, NCH, S, EPI>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_spmm_cpa<G, NCH, S, EPI>,
                                                      WARPS * 32, smem);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    constexpr int SPB = WARPS * 32 / G;   // edge streams per block
    const int64_t streams = (int64_t)n_sm * blocks_per_sm * SPB;
    int64_t rpw = (n_rows + streams - 1) / streams;
    if (rpw < 1) rpw = 1;
    const int64_t blocks = ((n_rows + rpw - 1) / rpw + SPB - 1) / SPB;
    cgpdl::launch(k_spmm_cpa<G, NCH, S, EPI>, dim3((unsigned)blocks), dim3(WARPS * 32), smem, st,
                  n_rows, F, rowptr, col, n_direct, halo_row, X, ldx, scale, addend, ld_add, mask,
                  ld_mask, mbits, ld_mbits, out, ldo, rpw, spmm_flags());
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : cg_cuda_fail(e, "k_spmm_cpa");
}

template <int G, int NCH, int S>
int launch(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col, int64_t n_direct,
           const int32_t *halo_row, const float *X, int64_t ldx, const float *scale,
           const float *addend, int64_t ld_add, const float *mask, int64_t ld_mask,
           const uint32_t *mbits, int64_t ld_mbits, float *out,
           int64_t ldo, cudaStream_t st) {
    // EPI 0: plain; 1: addend and / or fp32 mask (and / or mask bits); 2: mask
    // bits only -- one register per chunk instead of the fp32 operands' four
    // or eight, so the GCN backward keeps the forward's lane count
    const int epi = (addend || mask) ? 1 : (mbits ? 2 : 0);
#define CG_CPA_EPI(E)                                                                          \
    launch_epi<G, NCH, S, E>(n_rows, F, rowptr, col, n_direct, halo_row, X, ldx, scale, addend, \
                             ld_add, mask, ld_mask, mbits, ld_mbits, out, ldo, st)
    return epi == 1 ? CG_CPA_EPI(1) : epi == 2 ? CG_CPA_EPI(2) : CG_CPA_EPI(0);
#undef CG_CPA_EPI
}

}  // namespace cpa

// Ring slots per warp.  Measured on C2 (F = 256): S = 3..8 within noise,
// 0.21 ms per launch vs 0.25-0.29 ms for the register-pipelined kernel; S = 4
// needs the least shared memory.  CG_SPMM_S picks another instantiated depth.
#define SPMM_CPA_S 4

template <int G, int NCH, int... Ss>
int launch_s(int S, int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col,
             int64_t n_direct, const int32_t *halo_row, const float *X, int64_t ldx,
             const float *scale, const float *addend, int64_t ld_add, const float *mask,
             int64_t ld_mask, const uint32_t *mbits, int64_t ld_mbits, float *out, int64_t ldo,
             cudaStream_t st) {
    int rc = 0;
    bool hit = false;
    ((S == Ss && !hit
          ? (hit = true, rc = cpa::launch<G, NCH, Ss>(n_rows, F, rowptr, col, n_direct, halo_row, X,
                                                   ldx, scale, addend, ld_add, mask, ld_mask,
                                                   mbits, ld_mbits, out,
                                                   ldo, st))
          : 0),
     ...);
    return hit ? rc : 0;
}

// Internal entry: cg_spmm dispatches sparse-row SpMMs with F <= 640 here
// (one edge stream per 8 / 16 / 32 lanes by width).  Returns the launch
// count, or 0 when this path does not apply (the caller falls back).
int cg_spmm_async(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col,
                  int64_t n_direct, const int32_t *halo_row, const float *X, int64_t ldx,
                  const float *scale, const float *addend, int64_t ld_add, const float *mask,
                  int64_t ld_mask, const uint32_t *mbits, int64_t ld_mbits, float *out, int64_t ldo,
             cudaStream_t st) {
    if (F > 640 || F % 4 || ldx % 4) return 0;
    static const int S = getenv("CG_SPMM_S") ? atoi(getenv("CG_SPMM_S")) : SPMM_CPA_S;
    static const bool narrow_g4 = !getenv("CG_SPMM_G4") || atoi(getenv("CG_SPMM_G4")) != 0;
#define CG_CPA_ARGS n_rows, F, rowptr, col, n_direct, halo_row, X, ldx, scale, addend, ld_add, \
                    mask, ld_mask, mbits, ld_mbits, out, ldo, st
    // lanes per edge stream: CG_SPMM_LANES picks fewer lanes (more 16-byte
    // chunks per lane, fewer per-edge instructions per byte) for F <= 256
    static const int lanes = getenv("CG_SPMM_LANES") ? atoi(getenv("CG_SPMM_LANES")) : 0;
    if (F <= 48 && narrow_g4) return launch_s<4, 3, 4, 8>(S, CG_CPA_ARGS);
    if (F <= 64) {
        if (lanes == 4) return launch_s<4, 4, 4, 6>(S, CG_CPA_ARGS);
        return launch_s<8, 2, 4, 8>(S, CG_CPA_ARGS);
    }
    if (F <= 128) {
        // 8-lane streams with 4 chunks per lane (half the per-edge
        // instructions per byte, twice the rows in flight per warp) win for
        // the plain forward aggregations (C2 sweep, profiles/r02: 128-wide
        // 0.088 -> 0.078 ms, 256-wide as two slices 0.197 -> 0.184 ms); the
        // epilogue variant (addend / mask prefetch registers scale with the
        // chunks per lane: 150 registers) stays on 16 lanes (0.21 vs 0.33 ms)
        const bool epi = addend != nullptr || mask != nullptr;   // (mask bits alone: 8 lanes)
        if (lanes == 16 || (lanes == 0 && epi)) return launch_s<16, 2, 4, 8>(S, CG_CPA_ARGS);
        if (lanes == 4) return launch_s<4, 8, 3, 4>(S, CG_CPA_ARGS);
        return launch_s<8, 4, 4, 6>(S, CG_CPA_ARGS);
    }
    if (F <= 256) {
        if (lanes == 16) return launch_s<16, 4, 4>(S, CG_CPA_ARGS);
        if (lanes == 8) return launch_s<8, 8, 3, 4>(S, CG_CPA_ARGS);
        return launch_s<32, 2, 3, 4, 6, 8>(S, CG_CPA_ARGS);
    }
    if (F <= 384) return launch_s<32, 3, 3, 4>(S, CG_CPA_ARGS);
    if (F <= 512) return launch_s<32, 4, 3, 4>(S, CG_CPA_ARGS);
    return launch_s<32, 5, 3, 4>(S, CG_CPA_ARGS);
#undef CG_CPA_ARGS
}
