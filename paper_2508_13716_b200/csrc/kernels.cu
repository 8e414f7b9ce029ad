// sm_100a kernels for the halo-exchange + aggregation hot path.
//
//   K1/K2 cg_spmm        fused cache-lookup + gather CSR SpMM (fwd and bwd)
//   K3    cg_copy_rows   halo staging / cache write-through over a pointer
//                        table (local HBM, NVLink peers, mapped host tier)
//   K6    cg_plan_frozen per-epoch JACA/FIFO plan after membership freezes
//   K8    cg_softmax_ce  mean cross-entropy + logits gradient
//   plus deterministic column sums, Adam and the synthetic-input hashes.
//
// All reductions are fixed-order (no float atomics): reruns are bitwise
// identical.  See DESIGN.md for layouts and rooflines.

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

#include "../../include/capgnn.h"
#include "pdl.cuh"

extern void cg_set_error(const std::string &msg);
int cg_spmm_async(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col,
                  int64_t n_direct, const int32_t *halo_row, const float *X, int64_t ldx,
                  const float *scale, const float *addend, int64_t ld_add, const float *mask,
                  int64_t ld_mask, const uint32_t *mbits, int64_t ld_mbits, float *out,
                  int64_t ldo, cudaStream_t st);
extern int cg_cuda_fail(cudaError_t e, const char *what);

#define CG_CHECK_LAUNCH(name)                                   \
    do {                                                        \
        cudaError_t _e = cudaGetLastError();                    \
        if (_e != cudaSuccess) return cg_cuda_fail(_e, name);   \
    } while (0)

namespace {

constexpr int kWarp = 32;

__device__ __forceinline__ uint32_t mix32(uint32_t seed, uint32_t a, uint32_t b) {
    uint32_t h = seed * 0x9E3779B1u + a * 0x85EBCA77u + b * 0xC2B2AE3Du;
    h ^= h >> 16;
    h *= 0x7FEB352Du;
    h ^= h >> 15;
    h *= 0x846CA68Bu;
    h ^= h >> 16;
    return h;
}

__device__ __forceinline__ float uniform_pm1(uint32_t seed, uint32_t a, uint32_t b) {
    float x = __uint2float_rn(mix32(seed, a, b) >> 8);
    return __fsub_rn(__fmul_rn(x, 1.1920928955078125e-07f), 1.0f);  // x*2^-23 - 1, exact
}

__global__ void k_hash_features(float *__restrict__ out, int64_t ld,
                                const int32_t *__restrict__ vertex, int64_t n, int F,
                                uint32_t seed, const float *__restrict__ row_scale) {
    int64_t total = n * (int64_t)F;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / F;
        int k = (int)(i - r * F);
        float x = uniform_pm1(seed, (uint32_t)vertex[r], (uint32_t)k);
        if (row_scale) x = __fmul_rn(x, row_scale[r]);
        out[r * ld + k] = x;
    }
}

__global__ void k_hash_labels(int32_t *__restrict__ out, const int32_t *__restrict__ vertex,
                              int64_t n, int C, uint32_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)(mix32(seed, (uint32_t)vertex[i], 0u) % (uint32_t)C);
}

// ---------------------------------------------------------------- K3 ------

// One warp (or G-lane group) per row; 16-byte vectors when everything is
// 16-byte aligned, scalar otherwise.
template <bool VEC>
__global__ void k_copy_rows(int64_t n, int F, const int32_t *__restrict__ src_id,
                            const int32_t *__restrict__ src_row,
                            const int32_t *__restrict__ dst_row,
                            const float *const *__restrict__ tab,
                            const int64_t *__restrict__ tab_ld, float *__restrict__ dst,
                            int64_t ld_dst, int id_lo, int id_hi) {
    pdl_entry();
    // Each warp scans 32 table entries at a time (one per lane), compacts the
    // live ones with a ballot, then copies those rows cooperatively: most
    // epochs most entries are "nothing to move" (stale local hits).
    const int lane = threadIdx.x & (kWarp - 1);
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kWarp;
    int64_t nwarps = (int64_t)gridDim.x * blockDim.x / kWarp;
    for (int64_t base = warp * kWarp; base < n; base += nwarps * kWarp) {
        const int64_t i = base + lane;
        int sid = -1, srow = 0, drow = -1;
        if (i < n) {
            sid = src_id[i];
            drow = dst_row[i];
            if (sid < id_lo || sid >= id_hi) sid = -1;   // another queue's entry
            if (sid >= 0 && drow >= 0) srow = src_row[i];
        }
        unsigned live = __ballot_sync(0xffffffffu, sid >= 0 && drow >= 0);
        while (live) {
            const int j = __ffs(live) - 1;
            live &= live - 1;
            const int s = __shfl_sync(0xffffffffu, sid, j);
            const int r = __shfl_sync(0xffffffffu, srow, j);
            const int d = __shfl_sync(0xffffffffu, drow, j);
            const float *sp = tab[s] + (int64_t)r * tab_ld[s];
            float *dp = dst + (int64_t)d * ld_dst;
            if (VEC) {
                const float4 *s4 = reinterpret_cast<const float4 *>(sp);
                float4 *d4 = reinterpret_cast<float4 *>(dp);
                for (int c = lane; c < (F >> 2); c += kWarp) d4[c] = s4[c];
            } else {
                for (int c = lane; c < F; c += kWarp) dp[c] = sp[c];
            }
        }
    }
}

// ---------------------------------------------------------------- K1 ------

// Gathered feature rows: kept in L2 (evict_last), not allocated in L1.
__device__ __forceinline__ float4 ldg_keep(const float4 *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

#ifndef SPMM_UNR1
#define SPMM_UNR1 4   // rows in flight per lane, one float4 chunk per lane
#endif
#ifndef SPMM_UNR2
#define SPMM_UNR2 4   // rows in flight per lane, two float4 chunks per lane (3 and 8 measured slower)
#endif

// G lanes per row, NCH float4 chunks per lane (row width F <= 4*G*NCH).
// Each G-lane group walks rows r, r+ngrp, ... through a 4-stage software
// pipeline so the index chase never sits in front of the gathers:
//   A  rowptr of row k+3      B  first G column ids of row k+2
//   C  cache lookup (halo_row indirection: slab slot / staging row / owner
//      row) of row k+1        D  the row-k gathers: UNR rows of 128-bit loads
//                                in flight per lane, CSR-order accumulation.
// Loads issued in stages A-C are consumed one iteration later, behind the
// gathers of the current row.  Rows with more than G edges finish their tail
// inline.  The grid is sized to the resident-block count (persistent), so a
// group sees many rows and the pipeline stays full.
template <int G, int NCH>
// Occupancy matters more than registers for these latency-bound gathers:
// at 86 registers (the mask-bits and L2-policy operands) the NCH = 2 kernel
// dropped from 3 to 2 blocks per SM and C3's dense 256-wide aggregation from
// 8.2 to 10.6 ms.  Bounded to 4 blocks (64 registers, a few bytes of L1
// spill) it runs C3's 256-wide aggregations at 7.1-7.4 ms (3 blocks: 8.1-8.4);
// the other widths keep the compiler's choice
__global__ void __launch_bounds__(256, NCH == 2 ? 4 : 0)
k_spmm(int64_t n_rows, int F, const int64_t *__restrict__ rowptr,
       const int32_t *__restrict__ col, int64_t n_direct, const int32_t *__restrict__ halo_row,
       const float *__restrict__ X, int64_t ldx, const float *__restrict__ scale,
       const float *__restrict__ addend, int64_t ld_add, const float *__restrict__ mask,
       int64_t ld_mask, const uint32_t *__restrict__ mbits, int64_t ld_mbits,
       float *__restrict__ out, int64_t ldo, int flags) {
    pdl_entry();
    constexpr int UNR = (NCH == 1) ? SPMM_UNR1 : SPMM_UNR2;   // rows in flight per lane
    uint64_t pol;
    if (flags & 4)   // CG_SPMM_FLAGS bit 2: gathered rows at the default priority
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    uint64_t pol_first;   // bit 0: outputs evict_first (else evict_normal)
    if (flags & 1)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_first));
    const int lane = threadIdx.x & (G - 1);
    const unsigned gmask = (G == 32) ? 0xffffffffu
                                     : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
    const int nchunk = F >> 2;
    const int64_t ngrp = (int64_t)gridDim.x * blockDim.x / G;
    int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;

    auto lookup = [&](int32_t c) -> int64_t {
        return (c < n_direct || halo_row == nullptr) ? (int64_t)c : (int64_t)halo_row[c - n_direct];
    };
    auto gather_add = [&](int64_t src, float4 (&acc)[NCH]) {
        const float4 *p = reinterpret_cast<const float4 *>(X + src * ldx);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int ch = lane + c * G;
            if (ch < nchunk) {
                const float4 t = ldg_keep(p + ch, pol);
                acc[c].x += t.x; acc[c].y += t.y; acc[c].z += t.z; acc[c].w += t.w;
            }
        }
    };

    // pipeline prologue: rows k, k+1, k+2 (r1, r2, r3 = r + ngrp, ...)
    int64_t b0 = 0, e0 = 0, b1 = 0, e1 = 0, b2 = 0, e2 = 0;
    if (r < n_rows) { b0 = rowptr[r]; e0 = rowptr[r + 1]; }
    if (r + ngrp < n_rows) { b1 = rowptr[r + ngrp]; e1 = rowptr[r + ngrp + 1]; }
    if (r + 2 * ngrp < n_rows) { b2 = rowptr[r + 2 * ngrp]; e2 = rowptr[r + 2 * ngrp + 1]; }
    int32_t c1 = (lane < e1 - b1) ? col[b1 + lane] : 0;
    int64_t s0 = (lane < e0 - b0) ? lookup(col[b0 + lane]) : 0;

    for (; r < n_rows; r += ngrp) {
        // A: rowptr of row k+3
        const int64_t r3 = r + 3 * ngrp;
        int64_t b3 = 0, e3 = 0;
        if (r3 < n_rows) { b3 = rowptr[r3]; e3 = rowptr[r3 + 1]; }
        // B: column ids of row k+2
        const int32_t c2 = (lane < e2 - b2) ? col[b2 + lane] : 0;
        // C: cache lookup of row k+1
        const int64_t s1 = (lane < e1 - b1) ? lookup(c1) : 0;
        // D: gathers of row k
        float4 acc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int cnt = (int)((e0 - b0) < (int64_t)G ? (e0 - b0) : (int64_t)G);
        int j = 0;
        for (; j + UNR <= cnt; j += UNR) {
            float4 v[UNR][NCH];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int64_t rr = __shfl_sync(gmask, s0, j + u, G);
                const float4 *src = reinterpret_cast<const float4 *>(X + rr * ldx);
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    const int ch = lane + c * G;
                    v[u][c] = ch < nchunk ? ldg_keep(src + ch, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    acc[c].x += v[u][c].x;
                    acc[c].y += v[u][c].y;
                    acc[c].z += v[u][c].z;
                    acc[c].w += v[u][c].w;
                }
        }
        for (; j < cnt; ++j) gather_add(__shfl_sync(gmask, s0, j, G), acc);
        // tail of a row with more than G edges (rare): inline, same order
        for (int64_t eb = b0 + G; eb < e0; eb += G) {
            const int n2 = (int)((e0 - eb) < (int64_t)G ? (e0 - eb) : (int64_t)G);
            const int64_t sx = (lane < n2) ? lookup(col[eb + lane]) : 0;
            for (int t = 0; t < n2; ++t) gather_add(__shfl_sync(gmask, sx, t, G), acc);
        }
        const float sc = scale ? scale[r] : 1.0f;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int ch = lane + c * G;
            if (ch >= nchunk) continue;
            // explicit roundings (no FMA contraction): every SpMM kernel's epilogue
            // rounds the same way, so they agree bit for bit
            float4 o = make_float4(__fmul_rn(acc[c].x, sc), __fmul_rn(acc[c].y, sc),
                                   __fmul_rn(acc[c].z, sc), __fmul_rn(acc[c].w, sc));
            if (addend) {
                const float4 a = reinterpret_cast<const float4 *>(addend + r * ld_add)[ch];
                o.x = __fadd_rn(o.x, a.x); o.y = __fadd_rn(o.y, a.y);
                o.z = __fadd_rn(o.z, a.z); o.w = __fadd_rn(o.w, a.w);
            }
            if (mask) {
                const float4 m = reinterpret_cast<const float4 *>(mask + r * ld_mask)[ch];
                o.x = m.x > 0.f ? o.x : 0.f;
                o.y = m.y > 0.f ? o.y : 0.f;
                o.z = m.z > 0.f ? o.z : 0.f;
                o.w = m.w > 0.f ? o.w : 0.f;
            }
            if (mbits) {   // the same mask as bits: column 4 ch + i is bit (4 ch + i) % 32
                const uint32_t b = mbits[r * ld_mbits + (ch >> 3)] >> (4 * (ch & 7));
                o.x = (b & 1u) ? o.x : 0.f; o.y = (b & 2u) ? o.y : 0.f;
                o.z = (b & 4u) ? o.z : 0.f; o.w = (b & 8u) ? o.w : 0.f;
            }
            // written once, never re-read by this launch: evict_first (see
            // spmm_async.cu), so the output does not displace gathered rows
            asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
                         ::"l"(reinterpret_cast<float4 *>(out + r * ldo) + ch), "f"(o.x), "f"(o.y),
                         "f"(o.z), "f"(o.w), "l"(pol_first)
                         : "memory");
        }
        // rotate the pipeline
        b0 = b1; e0 = e1; s0 = s1;
        b1 = b2; e1 = e2; c1 = c2;
        b2 = b3; e2 = e3;
    }
}

// ---------------------------------------------------------------- K8 ------

__global__ void __launch_bounds__(256)
k_softmax_ce(int64_t n, int C, const float *__restrict__ logits, int64_t ld,
             const int32_t *__restrict__ label, float inv_n, float *__restrict__ grad,
             int64_t ldg, float *__restrict__ block_loss) {
    // one warp per row; per-block loss partials combined in a fixed order
    __shared__ float wl[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float acc = 0.f;
    for (int64_t r = blockIdx.x * 8 + w; r < n; r += (int64_t)gridDim.x * 8) {
        const float *z = logits + r * ld;
        float mx = -INFINITY;
        for (int c = lane; c < C; c += 32) mx = fmaxf(mx, z[c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float se = 0.f;
        for (int c = lane; c < C; c += 32) se += __expf(z[c] - mx);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const float lse = __logf(se);
        const int y = label[r];
        for (int c = lane; c < C; c += 32) {
            float p = __expf(z[c] - mx - lse);
            grad[r * ldg + c] = (p - (c == y ? 1.f : 0.f)) * inv_n;
        }
        acc += lse - (z[y] - mx);
    }
    if (lane == 0) wl[w] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += wl[k];
        block_loss[blockIdx.x] = t;
    }
}

// Narrow-class variant (C <= 64, ld % 4 == 0, ldg % 4 == 0, 16-B aligned rows):
// 4 lanes per row, each holding up to 4 float4 of logits in registers, so a
// row costs one 16-byte load / store per 4 classes and two shuffle rounds.
template <int NV>
__global__ void __launch_bounds__(256)
k_softmax_ce4(int64_t n, int C, const float *__restrict__ logits, int64_t ld,
              const int32_t *__restrict__ label, float inv_n, float *__restrict__ grad,
              int64_t ldg, float *__restrict__ block_loss, float *__restrict__ grad2,
              int64_t ldg2, const float *__restrict__ scale2, float *__restrict__ loss_out,
              unsigned int *__restrict__ ticket) {
    pdl_entry();
    __shared__ float wl[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int sub = lane & 3;                       // lane within the row group
    const int C4 = (C + 3) >> 2;
    float acc = 0.f;
    // the loop bound is warp-uniform (shuffles below need every lane)
    const int64_t stride = (int64_t)gridDim.x * 64;
    for (int64_t r0 = ((int64_t)blockIdx.x * 256 + (threadIdx.x & ~31)) >> 2; r0 < n;
         r0 += stride) {
        const int64_t r = r0 + (lane >> 2);
        const bool ok = r < n;
        const float4 *z4 = reinterpret_cast<const float4 *>(logits + (ok ? r : 0) * ld);
        float4 v[NV];
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int c4 = sub + 4 * k;
            if (ok && c4 < C4) {
                v[k] = __ldg(z4 + c4);
                const int c = 4 * c4;
                if (c + 0 >= C) v[k].x = -INFINITY;
                if (c + 1 >= C) v[k].y = -INFINITY;
                if (c + 2 >= C) v[k].z = -INFINITY;
                if (c + 3 >= C) v[k].w = -INFINITY;
            } else {
                v[k] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
            mx = fmaxf(mx, fmaxf(fmaxf(v[k].x, v[k].y), fmaxf(v[k].z, v[k].w)));
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        float se = 0.f;
#pragma unroll
        for (int k = 0; k < NV; ++k)
            se += __expf(v[k].x - mx) + __expf(v[k].y - mx) + __expf(v[k].z - mx) +
                  __expf(v[k].w - mx);
        se += __shfl_xor_sync(0xffffffffu, se, 1);
        se += __shfl_xor_sync(0xffffffffu, se, 2);
        const float lse = __logf(se);
        const int y = ok ? label[r] : -1;
        float zy = 0.f;
        float4 *g4 = reinterpret_cast<float4 *>(grad + (ok ? r : 0) * ldg);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int c4 = sub + 4 * k;
            if (!ok || c4 >= C4) continue;
            const int c = 4 * c4;
            float4 p;
            p.x = c + 0 < C ? (__expf(v[k].x - mx - lse) - (c + 0 == y ? 1.f : 0.f)) * inv_n : 0.f;
            p.y = c + 1 < C ? (__expf(v[k].y - mx - lse) - (c + 1 == y ? 1.f : 0.f)) * inv_n : 0.f;
            p.z = c + 2 < C ? (__expf(v[k].z - mx - lse) - (c + 2 == y ? 1.f : 0.f)) * inv_n : 0.f;
            p.w = c + 3 < C ? (__expf(v[k].w - mx - lse) - (c + 3 == y ? 1.f : 0.f)) * inv_n : 0.f;
            if (y >= c && y < c + 4) zy = (y == c) ? v[k].x : (y == c + 1) ? v[k].y
                                        : (y == c + 2) ? v[k].z : v[k].w;
            g4[c4] = p;
            if (grad2) {   // the row-scaled copy the backward aggregation gathers
                const float sr = scale2 ? scale2[r] : 1.f;
                reinterpret_cast<float4 *>(grad2 + r * ldg2)[c4] =
                    make_float4(__fmul_rn(p.x, sr), __fmul_rn(p.y, sr), __fmul_rn(p.z, sr),
                                __fmul_rn(p.w, sr));
            }
        }
        zy += __shfl_xor_sync(0xffffffffu, zy, 1);
        zy += __shfl_xor_sync(0xffffffffu, zy, 2);
        if (ok && sub == 0) acc += lse - (zy - mx);
    }
    // fixed-order combine: lanes of a warp by butterfly, warps in order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) wl[w] = acc;
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += wl[k];
        block_loss[blockIdx.x] = t;
        // the last block to finish sums the block partials (fixed order, as
        // k_sum_fixed did in a launch of its own) and re-arms the ticket
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __shared__ double sh[256];
    double t = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += (double)__ldcg(block_loss + i);
    sh[threadIdx.x] = t;
    __syncthreads();
    for (int k = blockDim.x / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *loss_out = (float)sh[0];
        *ticket = 0u;
    }
}

// Deterministic sum of x[0..n) into *out (single block, fixed order).
__global__ void k_sum_fixed(const float *__restrict__ x, int64_t n, float *__restrict__ out) {
    pdl_entry();
    __shared__ double sh[1024];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += (double)x[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = (float)sh[0];
}

// Column sums over m in fixed chunks of kColChunk rows: lanes own columns
// (coalesced 128 B rows), the 8 warps of a block take interleaved rows, and
// the 8 per-warp sums are combined in a fixed order -> ws[chunk][n].
constexpr int kColChunk = 2048;
__global__ void __launch_bounds__(256)
k_colsum_partial(int64_t M, int N, const float *__restrict__ D, int64_t ldd,
                 float *__restrict__ ws) {
    __shared__ float part[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n = blockIdx.x * 32 + lane;
    const int64_t m0 = (int64_t)blockIdx.y * kColChunk;
    const int64_t m1 = min(M, m0 + kColChunk);
    float s = 0.f;
    if (n < N) {
#pragma unroll 8
        for (int64_t m = m0 + w; m < m1; m += 8) s += D[m * ldd + n];
    }
    part[w][lane] = s;
    __syncthreads();
    if (w == 0 && n < N) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += part[k][lane];
        ws[blockIdx.y * (int64_t)N + n] = t;
    }
}

// out[i] = sum_c ws[c][i], fixed order: 8 warps stride the chunks (each
// keeping 4 independent partial sums so the loads pipeline), then a fixed
// combination of the partials.
template <int NW>
__device__ __forceinline__ void reduce_chunks_block(int64_t blk, int64_t n_out, int64_t n_chunks,
                                                    const float *__restrict__ ws,
                                                    float *__restrict__ out) {
    __shared__ float part[NW][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = blk * 32 + lane;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    if (i < n_out) {
        int64_t c = w;
        for (; c + 3 * NW < n_chunks; c += 4 * NW) {
            s0 += ws[c * n_out + i];
            s1 += ws[(c + NW) * n_out + i];
            s2 += ws[(c + 2 * NW) * n_out + i];
            s3 += ws[(c + 3 * NW) * n_out + i];
        }
        for (; c < n_chunks; c += NW) s0 += ws[c * n_out + i];
    }
    part[w][lane] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    if (w == 0 && i < n_out) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < NW; ++k) t += part[k][lane];
        out[i] = t;
    }
}

// The same reduction four outputs per lane (n_out % 4 == 0, 16-byte aligned
// rows): a block covers 128 outputs, NW warps stride the chunks with four
// independent float4 partials each, then a fixed combination.  Fewer, wider
// loads than the scalar form: the split-K partials of a 256 x 256 dW (19 MB)
// are one wave of blocks instead of seven.
template <int NW>
__device__ __forceinline__ void reduce_chunks_block4(int64_t blk, int64_t n_out,
                                                     int64_t n_chunks,
                                                     const float *__restrict__ ws,
                                                     float *__restrict__ out) {
    __shared__ float4 part4[NW][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t n4 = n_out >> 2;
    const int64_t i = blk * 32 + lane;   // float4 index
    const float4 *w4 = reinterpret_cast<const float4 *>(ws);
    float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0, s2 = s0, s3 = s0;
    auto add = [](float4 &a, const float4 b) { a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w; };
    if (i < n4) {
        int64_t c = w;
        for (; c + 3 * NW < n_chunks; c += 4 * NW) {
            const float4 v0 = w4[c * n4 + i], v1 = w4[(c + NW) * n4 + i];
            const float4 v2 = w4[(c + 2 * NW) * n4 + i], v3 = w4[(c + 3 * NW) * n4 + i];
            add(s0, v0); add(s1, v1); add(s2, v2); add(s3, v3);
        }
        for (; c < n_chunks; c += NW) add(s0, w4[c * n4 + i]);
    }
    add(s0, s1);
    add(s2, s3);
    add(s0, s2);
    part4[w][lane] = s0;
    __syncthreads();
    if (w == 0 && i < n4) {
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < NW; ++k) add(t, part4[k][lane]);
        reinterpret_cast<float4 *>(out)[i] = t;
    }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32)
k_reduce_chunks_pair4(int64_t nb1, int64_t n1, int64_t c1, const float *__restrict__ ws1,
                      float *__restrict__ out1, int64_t n2, int64_t c2,
                      const float *__restrict__ ws2, float *__restrict__ out2) {
    pdl_entry();
    if (blockIdx.x < nb1) reduce_chunks_block4<NW>(blockIdx.x, n1, c1, ws1, out1);
    else reduce_chunks_block4<NW>(blockIdx.x - nb1, n2, c2, ws2, out2);
}

// Two independent chunk reductions in one launch (the weight and the bias
// gradient partials of one cg_wgrad call): blocks [0, nb1) do the first.
template <int NW>
__global__ void __launch_bounds__(NW * 32)
k_reduce_chunks_pair(int64_t nb1, int64_t n1, int64_t c1, const float *__restrict__ ws1,
                     float *__restrict__ out1, int64_t n2, int64_t c2,
                     const float *__restrict__ ws2, float *__restrict__ out2) {
    if (blockIdx.x < nb1) reduce_chunks_block<NW>(blockIdx.x, n1, c1, ws1, out1);
    else reduce_chunks_block<NW>(blockIdx.x - nb1, n2, c2, ws2, out2);
}

template <int NW>
__global__ void __launch_bounds__(NW * 32)
k_reduce_chunks_tree(int64_t n_out, int64_t n_chunks, const float *__restrict__ ws,
                     float *__restrict__ out) {
    __shared__ float part[NW][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * 32 + lane;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    if (i < n_out) {
        int64_t c = w;
        for (; c + 3 * NW < n_chunks; c += 4 * NW) {
            s0 += ws[c * n_out + i];
            s1 += ws[(c + NW) * n_out + i];
            s2 += ws[(c + 2 * NW) * n_out + i];
            s3 += ws[(c + 3 * NW) * n_out + i];
        }
        for (; c < n_chunks; c += NW) s0 += ws[c * n_out + i];
    }
    part[w][lane] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    if (w == 0 && i < n_out) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < NW; ++k) t += part[k][lane];
        out[i] = t;
    }
}

__global__ void k_reduce_chunks(int64_t n_out, int64_t n_chunks, const float *__restrict__ ws,
                                float *__restrict__ out, int accumulate) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_out) return;
    float s = 0.f;
    for (int64_t c = 0; c < n_chunks; ++c) s += ws[c * n_out + i];
    out[i] = accumulate ? out[i] + s : s;
}

__global__ void k_scale_rows(float *__restrict__ X, int64_t ld, int64_t n, int F,
                             const float *__restrict__ scale) {
    int64_t total = n * (int64_t)F;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / F;
        X[r * ld + (i - r * F)] *= scale[r];
    }
}

// X = max(X, 0) in place over rows of F columns (F % 32 == 0), and the
// > 0 pattern as bits: one thread per 32-column word (eight float4s).
__global__ void k_relu_bits(int64_t n_rows, int F, float *__restrict__ X, int64_t ldx,
                            uint32_t *__restrict__ bits, int64_t ld_bits) {
    pdl_entry();
    const int W = F >> 5;
    const int64_t n = n_rows * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / W;
        const int w = (int)(i - r * W);
        float4 *p = reinterpret_cast<float4 *>(X + r * ldx) + 8 * w;
        uint32_t b = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float4 v = p[j];
            v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
            b |= ((v.x > 0.f ? 1u : 0u) | (v.y > 0.f ? 2u : 0u) | (v.z > 0.f ? 4u : 0u) |
                  (v.w > 0.f ? 8u : 0u)) << (4 * j);
            p[j] = v;
        }
        if (bits) bits[r * ld_bits + w] = b;
    }
}

__global__ void k_scale_rows_to(float *__restrict__ dst, int64_t ldd, const float *__restrict__ src,
                                int64_t lds, int64_t n, int F, const float *__restrict__ scale) {
    int64_t total = n * (int64_t)F;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / F;
        int64_t c = i - r * F;
        dst[r * ldd + c] = src[r * lds + c] * (scale ? scale[r] : 1.f);
    }
}

// float4 variant (F, ldd, lds multiples of 4, 16-byte aligned rows)
__global__ void k_scale_rows_to4(float *__restrict__ dst, int64_t ldd, const float *__restrict__ src,
                                 int64_t lds, int64_t n, int F4, const float *__restrict__ scale) {
    pdl_entry();
    const int64_t total = n * (int64_t)F4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / F4;
        const int64_t c = i - r * F4;
        float4 v = __ldg(reinterpret_cast<const float4 *>(src + r * lds) + c);
        const float sc = scale ? __ldg(scale + r) : 1.f;
        v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
        reinterpret_cast<float4 *>(dst + r * ldd)[c] = v;
    }
}

__device__ __forceinline__ uint32_t rn_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// x ~= hi + lo with hi = round-to-nearest TF32(x) and lo = TF32(x - hi), both
// exact TF32 values (the tensor core's operand truncation is then lossless):
// |x - hi - lo| <= 2^-23 |x|.
__device__ __forceinline__ void split_tf32(float x, float &hi, float &lo) {
    hi = __uint_as_float(rn_tf32(x));
    lo = __uint_as_float(rn_tf32(x - hi));
}

__global__ void k_adam(int64_t n, float *__restrict__ p, const float *__restrict__ g,
                       float *__restrict__ m, float *__restrict__ v, float lr, float b1,
                       float b2, float eps, float c1_arg, float c2_arg, float *__restrict__ p_hi,
                       float *__restrict__ p_lo, const float *__restrict__ corr_dev) {
    pdl_entry();
    // bias corrections: arguments, or device-resident under graph replay
    const float c1 = corr_dev ? corr_dev[0] : c1_arg, c2 = corr_dev ? corr_dev[1] : c2_arg;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float gi = g[i];
        float mi = b1 * m[i] + (1.f - b1) * gi;
        float vi = b2 * v[i] + (1.f - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        const float pi = p[i] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
        p[i] = pi;
        if (p_hi) {
            float h, l;
            split_tf32(pi, h, l);
            p_hi[i] = h;
            p_lo[i] = l;
        }
    }
}

// blockIdx.y = matrix; element e = i * cols + j of matrix m goes to j * rows + i
__global__ void k_split_tf32_t(const int64_t *__restrict__ off, const int32_t *__restrict__ rows,
                               const int32_t *__restrict__ cols, const float *__restrict__ x,
                               float *__restrict__ hi, float *__restrict__ lo) {
    pdl_entry();
    const int m = blockIdx.y;
    const int64_t o = off[m];
    const int r = rows[m], c = cols[m];
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= (int64_t)r * c) return;
    const int i = (int)(e / c), j = (int)(e % c);
    float h, l;
    split_tf32(x[o + e], h, l);
    hi[o + (int64_t)j * r + i] = h;
    lo[o + (int64_t)j * r + i] = l;
}

__global__ void k_split_tf32(int64_t n, const float *__restrict__ x, float *__restrict__ hi,
                             float *__restrict__ lo) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float h, l;
        split_tf32(x[i], h, l);
        hi[i] = h;
        lo[i] = l;
    }
}

// ---------------------------------------------------------------- K6 ------

__device__ __forceinline__ bool fresh(int32_t ver, int e, int s) { return s < 0 || e - ver <= s; }

// One thread per halo-union vertex u.  Requesters are visited in the
// reference's global lookup order (position in the requester's halo, then
// partition slot), which is the only order that matters for u because,
// with frozen membership, a lookup of u touches only u's own entries.
__device__ __forceinline__ void plan_vertex(const cg_plan_static &st, int64_t u, int e, int s,
                                            int me, int32_t *req_ver, int32_t *glob_ver,
                                            int32_t *halo_row, int32_t *stage_src,
                                            int32_t *stage_row, int32_t *stage_dst,
                                            int32_t *gw_slot, unsigned int *tally,
                                            int32_t *flag, int32_t staging_base,
                                            int32_t n_devices, int8_t *outcome) {
    const int32_t g = st.gslot[u];
    const int32_t odev = st.owner_dev[u], orow = st.owner_row[u];
    bool gdirty = false;
    // request coalescing: co-resident requesters of u that need the same
    // value this epoch (the owner's current row from a peer, or the global
    // tier's entry -- one version per epoch: glob_ver changes only on a miss,
    // which makes it current) read the row the first one staged, so each
    // distinct row crosses NVLink / PCIe once per device and layer
    int32_t row_cur = -1, row_glob = -1;
    for (int64_t k = st.req_off[u]; k < st.req_off[u + 1]; ++k) {
        const int32_t slot = st.req_slot[k];
        const int32_t part = st.req_part[k];
        int oc, ver;
        if (slot >= 0 && fresh(req_ver[k], e, s)) {
            oc = 0;
            ver = req_ver[k];
        } else if (g >= 0 && fresh(glob_ver[g], e, s)) {
            oc = 1;
            ver = glob_ver[g];
            if (slot >= 0) req_ver[k] = ver;
        } else {
            oc = 2;
            ver = e;
            // admit modes: 0 never (capacity 0), 1 always (room left, or FIFO
            // evicts), 2 only if the score beats the resident minimum (JACA)
            if (g >= 0) { glob_ver[g] = e; gdirty = true; }
            else if (st.gfree == 1 || (st.gfree == 2 && st.score[u] > st.gmin)) *flag = 1;
            if (slot >= 0) req_ver[k] = e;
            else if (st.lfree[part] == 1 || (st.lfree[part] == 2 && st.score[u] > st.lmin[part]))
                *flag = 1;
        }
        if (outcome) outcome[k] = (int8_t)oc;
        {   // warp-aggregated tally: one shared atomic per distinct (part, outcome)
            const unsigned am = __activemask();
            const int key = 3 * part + oc;
            const unsigned peers = __match_any_sync(am, key);
            if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&tally[key], __popc(peers));
        }
        if (st.req_dev[k] != me) continue;
        const int32_t pos = st.req_pos[k];
        const bool cur = (ver < 1 ? 1 : ver) == e;
        if (!st.req_needed[k]) {
            halo_row[pos] = -1;
            stage_src[pos] = -1;
            continue;
        }
        if (st.req_snap && ver <= 1) {
            // version 0/1 = the epoch-1 activation: the shared snapshot row
            halo_row[pos] = st.req_snap[k];
            stage_src[pos] = -1;
            continue;
        }
        if (staging_base < 0) {
            // compact layout (no staging rows, no slabs): a plan that needs
            // them breaks the layout's precondition -- report, never write
            *flag = 2;
            halo_row[pos] = -1;
            stage_src[pos] = -1;
            continue;
        }
        if (oc == 0 && !cur) {  // stale local hit: read the slab in place
            halo_row[pos] = slot;
            stage_src[pos] = -1;
            continue;
        }
        // value = owner's current row, or the global tier's snapshot
        int src_id, src_row;
        if (cur) { src_id = odev; src_row = orow; }
        else { src_id = n_devices; src_row = g; }  // host tier (table entry n_devices)
        int32_t &have = cur ? row_cur : row_glob;
        if (slot >= 0) {  // write through into the local slab, read it there
            stage_src[pos] = src_id;
            stage_row[pos] = src_row;
            stage_dst[pos] = slot;
            halo_row[pos] = slot;
            if (have < 0) have = slot;
        } else if (cur && odev == me) {  // co-resident owner: read in place
            stage_src[pos] = -1;
            halo_row[pos] = orow;
        } else if (st.coalesce && have >= 0) {  // already staged on this device this epoch
            stage_src[pos] = -1;
            halo_row[pos] = have;
        } else {
            stage_src[pos] = src_id;
            stage_row[pos] = src_row;
            stage_dst[pos] = staging_base + pos;
            halo_row[pos] = staging_base + pos;
            have = staging_base + pos;
        }
    }
    if (odev == me) {
        // the owner materialises version-e content (and the warm entries at e=1)
        bool need = g >= 0 && (gdirty || (e == 1 && glob_ver[g] <= 1));
        gw_slot[u] = need ? g : -1;
    }
}


constexpr int kPlanMaxParts = 256;
__global__ void __launch_bounds__(256)
k_plan_frozen(cg_plan_static st, int e_arg, int s, int me, int32_t *req_ver,
              int32_t *glob_ver, int32_t *halo_row, int32_t *stage_src,
              int32_t *stage_row, int32_t *stage_dst, int32_t *gw_slot,
              int64_t *counts, int32_t *flag, int32_t staging_base,
              int32_t n_devices, int8_t *outcome, const int32_t *epoch_dev) {
    pdl_entry();
    const int e = epoch_dev ? *epoch_dev : e_arg;   // device-resident under graph replay
    // outcome counters: shared-memory tallies, one global add per block
    __shared__ unsigned int tally[3 * kPlanMaxParts];
    for (int i = threadIdx.x; i < 3 * st.n_parts; i += blockDim.x) tally[i] = 0;
    __syncthreads();
    const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u < st.n_union) plan_vertex(st, u, e, s, me, req_ver, glob_ver, halo_row, stage_src,
                                    stage_row, stage_dst, gw_slot, tally, flag, staging_base,
                                    n_devices, outcome);
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * st.n_parts; i += blockDim.x)
        if (tally[i]) atomicAdd(reinterpret_cast<unsigned long long *>(counts + i),
                                (unsigned long long)tally[i]);
}

inline int n_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

inline int grid_for(int64_t work, int threads, int max_blocks = 148 * 16) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (int)b;
}

}  // namespace

// out[i] = sum_c ws[c][i] over n_chunks partial rows, fixed order (internal
// helper shared with the weight-gradient path in gemm.cu; not in the ABI).
int cg_reduce_chunks_pair(int64_t n1, int64_t c1, const float *ws1, float *out1, int64_t n2,
                          int64_t c2, const float *ws2, float *out2, cudaStream_t st) {
    auto al = [](const void *q) { return ((uintptr_t)q & 15) == 0; };
    if (n1 % 4 == 0 && n2 % 4 == 0 && al(ws1) && al(out1) && (n2 == 0 || (al(ws2) && al(out2)))) {
        const int64_t b1 = (n1 / 4 + 31) / 32, b2 = (n2 / 4 + 31) / 32;
        if (b1 + b2 == 0) return 0;
        // warps per block so the launch fills the GPU (few outputs, many chunks:
        // a 256 x 40 dW has 148 chunks over 81 blocks)
        const int64_t want = (int64_t)n_sms() * 32 / (b1 + b2);
        if (want >= 32)
            cgpdl::launch(k_reduce_chunks_pair4<32>, dim3((unsigned)(b1 + b2)), dim3(1024), 0, st,
                          b1, n1, c1, ws1, out1, n2, c2, ws2, out2);
        else if (want >= 16)
            cgpdl::launch(k_reduce_chunks_pair4<16>, dim3((unsigned)(b1 + b2)), dim3(512), 0, st,
                          b1, n1, c1, ws1, out1, n2, c2, ws2, out2);
        else
            cgpdl::launch(k_reduce_chunks_pair4<8>, dim3((unsigned)(b1 + b2)), dim3(256), 0, st,
                          b1, n1, c1, ws1, out1, n2, c2, ws2, out2);
        CG_CHECK_LAUNCH("k_reduce_chunks_pair4");
        return 1;
    }
    const int64_t nb1 = (n1 + 31) / 32, nb2 = (n2 + 31) / 32;
    if (nb1 + nb2 == 0) return 0;
    k_reduce_chunks_pair<32><<<(unsigned)(nb1 + nb2), 1024, 0, st>>>(nb1, n1, c1, ws1, out1, n2,
                                                                     c2, ws2, out2);
    CG_CHECK_LAUNCH("k_reduce_chunks_pair");
    return 1;
}

int cg_reduce_chunks(int64_t n_out, int64_t n_chunks, const float *ws, float *out,
                     cudaStream_t st) {
    if (n_out == 0) return 0;
    if (n_out % 4 == 0 && !((uintptr_t)ws & 15) && !((uintptr_t)out & 15))
        return cg_reduce_chunks_pair(n_out, n_chunks, ws, out, 0, 0, nullptr, nullptr, st);
    // many partial rows (split-K chunks x splitter warps): 32 warps share them
    if (n_chunks > 64)
        k_reduce_chunks_tree<32><<<(unsigned)((n_out + 31) / 32), 1024, 0, st>>>(n_out, n_chunks,
                                                                              ws, out);
    else
        k_reduce_chunks_tree<8><<<(unsigned)((n_out + 31) / 32), 256, 0, st>>>(n_out, n_chunks,
                                                                            ws, out);
    CG_CHECK_LAUNCH("k_reduce_chunks_tree");
    return 1;
}

extern "C" {

int cg_hash_features(float *out, int64_t ld, const int32_t *vertex, int64_t n_rows, int F,
                     uint32_t seed, const float *row_scale, void *stream) {
    if (n_rows == 0) return 0;
    k_hash_features<<<grid_for(n_rows * F, 256), 256, 0, (cudaStream_t)stream>>>(
        out, ld, vertex, n_rows, F, seed, row_scale);
    CG_CHECK_LAUNCH("k_hash_features");
    return 1;
}

int cg_hash_labels(int32_t *out, const int32_t *vertex, int64_t n_rows, int C, uint32_t seed,
                   void *stream) {
    if (n_rows == 0) return 0;
    k_hash_labels<<<grid_for(n_rows, 256), 256, 0, (cudaStream_t)stream>>>(out, vertex, n_rows,
                                                                          C, seed);
    CG_CHECK_LAUNCH("k_hash_labels");
    return 1;
}

int cg_copy_rows_sel(int64_t n, int F, const int32_t *src_id, const int32_t *src_row,
                     const int32_t *dst_row, const float *const *tab, const int64_t *tab_ld,
                     float *dst, int64_t ld_dst, int id_lo, int id_hi, int max_blocks,
                     void *stream) {
    if (n == 0) return 0;
    if (id_lo < 0) id_lo = 0;
    if (id_hi <= id_lo) return 0;
    const int threads = 256;
    int blocks = grid_for(n, threads, max_blocks > 0 ? max_blocks : 148 * 32);
    bool vec = (F % 4 == 0) && (ld_dst % 4 == 0) && ((uintptr_t)dst % 16 == 0);
    // source alignment is validated on the host side (tab_ld % 4 == 0, 16-B bases)
    if (vec)
        cgpdl::launch(k_copy_rows<true>, dim3(blocks), dim3(threads), 0, (cudaStream_t)stream, n,
                      F, src_id, src_row, dst_row, tab, tab_ld, dst, ld_dst, id_lo, id_hi);
    else
        cgpdl::launch(k_copy_rows<false>, dim3(blocks), dim3(threads), 0, (cudaStream_t)stream, n,
                      F, src_id, src_row, dst_row, tab, tab_ld, dst, ld_dst, id_lo, id_hi);
    CG_CHECK_LAUNCH("k_copy_rows");
    return 1;
}

int cg_copy_rows_bounded(int64_t n, int F, const int32_t *src_id, const int32_t *src_row,
                         const int32_t *dst_row, const float *const *tab,
                         const int64_t *tab_ld, float *dst, int64_t ld_dst, int max_blocks,
                         void *stream) {
    return cg_copy_rows_sel(n, F, src_id, src_row, dst_row, tab, tab_ld, dst, ld_dst, 0,
                            0x7fffffff, max_blocks, stream);
}

int cg_copy_rows(int64_t n, int F, const int32_t *src_id, const int32_t *src_row,
                 const int32_t *dst_row, const float *const *tab, const int64_t *tab_ld,
                 float *dst, int64_t ld_dst, void *stream) {
    return cg_copy_rows_bounded(n, F, src_id, src_row, dst_row, tab, tab_ld, dst, ld_dst, 0,
                                stream);
}

static int spmm_impl(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col,
                     int64_t n_direct, const int32_t *halo_row, const float *X, int64_t ldx,
                     const float *scale, const float *addend, int64_t ld_add, const float *mask,
                     int64_t ld_mask, const uint32_t *mbits, int64_t ld_mbits, float *out,
                     int64_t ldo, int64_t nnz, void *stream) {
    if (n_rows == 0) return 0;
    if (F % 4 || ldx % 4 || ldo % 4 || (addend && ld_add % 4) || (mask && ld_mask % 4) ||
        ((uintptr_t)X % 16) || ((uintptr_t)out % 16)) {
        cg_set_error("cg_spmm: F and leading dims must be multiples of 4, buffers 16-B aligned");
        return -1;
    }
    cudaStream_t st = (cudaStream_t)stream;
    // Sparse rows (< 64 edges on average): the cp.async shared-memory ring
    // kernel (spmm_async.cu) for F > 128, and for 64 < F <= 128 when the
    // gathered rows fit in L2 (estimated as n_rows x F x 4 <= 96 MB).
    // Measured: C2 (8 edges/row) 256-wide 0.21 vs 0.25-0.29 ms, 128-wide (L2-
    // resident) 0.096 vs 0.128 ms, 40-wide 0.068 vs 0.061 ms; C4 (25/row)
    // 256-wide 11.0 vs 11.6 ms but 100-wide (HBM-bound) 6.2 vs 5.6 ms; C3
    // (490/row, gathers mostly L2 hits) 256-wide 14.1 vs 8.2 ms.  Everything
    // else stays on the register-pipelined kernel below.  CG_SPMM_ASYNC=0 / 1
    // forces either choice.
    static const int async_env = getenv("CG_SPMM_ASYNC") ? atoi(getenv("CG_SPMM_ASYNC")) : -1;
    const bool sparse = nnz >= 0 && nnz < 64 * n_rows;
    const bool fits_l2 = n_rows * (int64_t)F * 4 <= (int64_t)96 << 20;
    // (F <= 48: 4-lane streams, C2 40-wide 0.055 vs 0.061 ms; on C4's
    // products-shaped CSR (26 edges/row, 4.9M source rows, beyond L2) the
    // ring also wins for F <= 48 -- the epoch's 48-wide backward 3.42 ->
    // 2.31 ms -- while the 100-wide forward, DRAM-bound on 400-byte rows,
    // stays faster on the register kernel in the epoch (5.57 vs 5.79 ms with
    // the halo_row indirection; profiles/r02/spmm_c4.txt, r02/c4/)
    const bool use_async =
        async_env == 1 ||
        (async_env != 0 && sparse && (F > 128 || F <= 48 || (fits_l2 && F > 64)));
    if (use_async) {
        // Wide rows whose 128-column slice fits L2 are aggregated one slice at
        // a time: each pass re-reads the CSR indices but finds most gathered
        // rows in L2 (C2 256-wide: 0.21 -> 0.20 ms; 64-column slices lose).
        static const int slice_env = getenv("CG_SPMM_SLICE") ? atoi(getenv("CG_SPMM_SLICE")) : 128;
        const int W = (slice_env > 0 && F > slice_env && sparse &&
                       n_rows * (int64_t)slice_env * 4 <= (int64_t)96 << 20)
                          ? slice_env
                          : F;
        int total = 0;
        for (int c0 = 0; c0 < F; c0 += W) {
            const int w = F - c0 < W ? F - c0 : W;
            const int rc = cg_spmm_async(n_rows, w, rowptr, col, n_direct, halo_row, X + c0, ldx,
                                         scale, addend ? addend + c0 : nullptr, ld_add,
                                         mask ? mask + c0 : nullptr, ld_mask,
                                         mbits ? mbits + c0 / 32 : nullptr, ld_mbits, out + c0,
                                         ldo, st);
            if (rc < 0) return rc;
            if (rc == 0) { total = 0; break; }   // not applicable: fall back whole
            total += rc;
        }
        if (total > 0) return total;
    }
    const int nchunk = F / 4;
    const int threads = 256;
    static const int reg_flags = getenv("CG_SPMM_FLAGS") ? atoi(getenv("CG_SPMM_FLAGS")) : 1;
#define CG_SPMM_LAUNCH(G, NCH)                                                              \
    do {                                                                                    \
        static int blocks_per_sm = 0;                                                       \
        if (!blocks_per_sm) {                                                               \
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_spmm<G, NCH>,   \
                                                          threads, 0);                      \
            if (blocks_per_sm < 1) blocks_per_sm = 1;                                       \
        }                                                                                   \
        cgpdl::launch(k_spmm<G, NCH>,                                                        \
                      dim3(grid_for(n_rows * G, threads, n_sms() * blocks_per_sm)),          \
                      dim3(threads), 0, st, n_rows, F, rowptr, col, n_direct, halo_row, X, ldx, \
                      scale, addend, ld_add, mask, ld_mask, mbits, ld_mbits, out, ldo,       \
                      reg_flags);                                                            \
    } while (0)
    if (nchunk <= 8) CG_SPMM_LAUNCH(8, 1);
    else if (nchunk <= 16) CG_SPMM_LAUNCH(16, 1);
    else if (nchunk <= 32) CG_SPMM_LAUNCH(32, 1);
    else if (nchunk <= 64) CG_SPMM_LAUNCH(32, 2);
    else if (nchunk <= 96) CG_SPMM_LAUNCH(32, 3);
    else if (nchunk <= 128) CG_SPMM_LAUNCH(32, 4);
    else if (nchunk <= 160) CG_SPMM_LAUNCH(32, 5);
    else {
        cg_set_error("cg_spmm: F > 640 not supported");
        return -1;
    }
#undef CG_SPMM_LAUNCH
    CG_CHECK_LAUNCH("k_spmm");
    return 1;
}

int cg_spmm(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col, int64_t n_direct,
            const int32_t *halo_row, const float *X, int64_t ldx, const float *scale,
            const float *addend, int64_t ld_add, const float *mask, int64_t ld_mask, float *out,
            int64_t ldo, int64_t nnz, void *stream) {
    return spmm_impl(n_rows, F, rowptr, col, n_direct, halo_row, X, ldx, scale, addend, ld_add,
                     mask, ld_mask, nullptr, 0, out, ldo, nnz, stream);
}

int cg_spmm_mb(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col,
               int64_t n_direct, const int32_t *halo_row, const float *X, int64_t ldx,
               const float *scale, const float *addend, int64_t ld_add,
               const uint32_t *mask_bits, int64_t ld_mask_bits, float *out, int64_t ldo,
               int64_t nnz, void *stream) {
    if (mask_bits && (F % 32)) {
        cg_set_error("cg_spmm_mb: mask bits need F % 32 == 0");
        return -1;
    }
    return spmm_impl(n_rows, F, rowptr, col, n_direct, halo_row, X, ldx, scale, addend, ld_add,
                     nullptr, 0, mask_bits, ld_mask_bits, out, ldo, nnz, stream);
}

int cg_scale_rows(float *X, int64_t ld, int64_t n_rows, int F, const float *scale,
                  void *stream) {
    if (n_rows == 0 || F == 0) return 0;
    k_scale_rows<<<grid_for(n_rows * F, 256), 256, 0, (cudaStream_t)stream>>>(X, ld, n_rows, F,
                                                                             scale);
    CG_CHECK_LAUNCH("k_scale_rows");
    return 1;
}

int cg_scale_rows_to(float *dst, int64_t ldd, const float *src, int64_t lds, int64_t n_rows,
                     int F, const float *scale, void *stream) {
    if (n_rows == 0 || F == 0) return 0;
    if (!(F % 4) && !(ldd % 4) && !(lds % 4) && !((uintptr_t)dst % 16) && !((uintptr_t)src % 16)) {
        cgpdl::launch(k_scale_rows_to4, dim3(grid_for(n_rows * (F / 4), 256, n_sms() * 8)),
                      dim3(256), 0, (cudaStream_t)stream, dst, ldd, src, lds, n_rows, F / 4,
                      scale);
        CG_CHECK_LAUNCH("k_scale_rows_to4");
        return 1;
    }
    k_scale_rows_to<<<grid_for(n_rows * F, 256), 256, 0, (cudaStream_t)stream>>>(
        dst, ldd, src, lds, n_rows, F, scale);
    CG_CHECK_LAUNCH("k_scale_rows_to");
    return 1;
}

int cg_relu_bits(int64_t n_rows, int F, float *X, int64_t ldx, uint32_t *bits, int64_t ld_bits,
                 void *stream) {
    if (n_rows == 0 || F == 0) return 0;
    if (F % 32 || ldx % 4 || ((uintptr_t)X % 16)) {
        cg_set_error("cg_relu_bits: F % 32 == 0, ldx % 4 == 0 and a 16-byte aligned X needed");
        return -1;
    }
    cgpdl::launch(k_relu_bits, dim3(grid_for(n_rows * (F / 32), 256, n_sms() * 8)), dim3(256), 0,
                  (cudaStream_t)stream, n_rows, F, X, ldx, bits, ld_bits);
    CG_CHECK_LAUNCH("k_relu_bits");
    return 1;
}

int cg_colsum(int64_t M, int N, const float *D, int64_t ldd, float *db, float *ws, void *stream) {
    if (M == 0 || N == 0) return 0;
    int64_t nch = (M + kColChunk - 1) / kColChunk;
    dim3 grid((N + 31) / 32, (unsigned)nch);
    cudaStream_t st = (cudaStream_t)stream;
    k_colsum_partial<<<grid, 256, 0, st>>>(M, N, D, ldd, ws);
    k_reduce_chunks_tree<8><<<(N + 31) / 32, 256, 0, st>>>(N, nch, ws, db);
    CG_CHECK_LAUNCH("cg_colsum");
    return 2;
}

int cg_softmax_ce(int64_t n_rows, int C, const float *logits, int64_t ld, const int32_t *label,
                  float inv_n, float *grad, int64_t ldg, float *loss_out, float *ws,
                  float *grad2, int64_t ldg2, const float *scale2, void *stream) {
    if (n_rows == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const bool narrow = C <= 64 && !(ld % 4) && !(ldg % 4) && !((uintptr_t)logits % 16) &&
                        !((uintptr_t)grad % 16) &&
                        (!grad2 || (!(ldg2 % 4) && !((uintptr_t)grad2 % 16)));
    int blocks;
    if (narrow) {
        blocks = grid_for(n_rows * 4, 256, n_sms() * 8);
        // ws[0]: the finish ticket at a fixed offset, so one zeroed workspace
        // serves calls of any shape (zero on entry, re-armed by each launch);
        // ws[1, 1 + blocks): block partials
        unsigned int *ticket = reinterpret_cast<unsigned int *>(ws);
        if (C <= 32)
            cgpdl::launch(k_softmax_ce4<2>, dim3(blocks), dim3(256), 0, st, n_rows, C, logits, ld,
                          label, inv_n, grad, ldg, ws + 1, grad2, ldg2, scale2, loss_out, ticket);
        else
            cgpdl::launch(k_softmax_ce4<4>, dim3(blocks), dim3(256), 0, st, n_rows, C, logits, ld,
                          label, inv_n, grad, ldg, ws + 1, grad2, ldg2, scale2, loss_out, ticket);
        CG_CHECK_LAUNCH("cg_softmax_ce");
        return 1;
    } else {
        blocks = grid_for(n_rows * 32, 256, 148 * 8);
        k_softmax_ce<<<blocks, 256, 0, st>>>(n_rows, C, logits, ld, label, inv_n, grad, ldg, ws);
    }
    cgpdl::launch(k_sum_fixed, dim3(1), dim3(1024), 0, st, ws, (int64_t)blocks, loss_out);
    CG_CHECK_LAUNCH("cg_softmax_ce");
    int launched = 2;
    if (grad2 && !narrow) {   // the wide-C kernel has no fused copy: scale separately
        const int rc = cg_scale_rows_to(grad2, ldg2, grad, ldg, n_rows, C, scale2, stream);
        if (rc < 0) return rc;
        launched += rc;
    }
    return launched;
}

static void adam_corrections(float beta1, float beta2, int step, float *c1, float *c2) {
    *c1 = (float)(1.0 - pow((double)beta1, (double)step));
    *c2 = (float)(1.0 - pow((double)beta2, (double)step));
}

int cg_adam(int64_t n, float *param, const float *grad, float *m, float *v, float lr,
            float beta1, float beta2, float eps, int step, float *p_hi, float *p_lo,
            const float *corr_dev, void *stream) {
    if (n == 0) return 0;
    if ((p_hi == nullptr) != (p_lo == nullptr)) {
        cg_set_error("cg_adam: p_hi and p_lo must both be set or both be NULL");
        return -1;
    }
    float c1, c2;
    adam_corrections(beta1, beta2, step, &c1, &c2);
    cgpdl::launch(k_adam, dim3(grid_for(n, 256, 148 * 8)), dim3(256), 0, (cudaStream_t)stream, n,
                  param, grad, m, v, lr, beta1, beta2, eps, c1, c2, p_hi, p_lo, corr_dev);
    CG_CHECK_LAUNCH("k_adam");
    return 1;
}

__global__ void k_set_epoch(int32_t *epoch_dev, int epoch, float *corr_dev, float c1, float c2) {
    pdl_entry();
    *epoch_dev = epoch;
    if (corr_dev) {
        corr_dev[0] = c1;
        corr_dev[1] = c2;
    }
}

int cg_set_epoch(int32_t *epoch_dev, int epoch, float *corr_dev, float beta1, float beta2,
                 int step, void *stream) {
    float c1, c2;
    adam_corrections(beta1, beta2, step, &c1, &c2);
    cgpdl::launch(k_set_epoch, dim3(1), dim3(1), 0, (cudaStream_t)stream, epoch_dev, epoch,
                  corr_dev, c1, c2);
    CG_CHECK_LAUNCH("k_set_epoch");
    return 1;
}

int cg_event_record(void *event, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(st, &cs);
    if (e != cudaSuccess) return cg_cuda_fail(e, "cudaStreamIsCapturing");
    // under capture an external record node fires (and timestamps) on every replay
    e = cs == cudaStreamCaptureStatusActive
            ? cudaEventRecordWithFlags((cudaEvent_t)event, st, cudaEventRecordExternal)
            : cudaEventRecord((cudaEvent_t)event, st);
    return e == cudaSuccess ? 0 : cg_cuda_fail(e, "cg_event_record");
}

int cg_split_tf32_t(int n_mats, const int64_t *off, const int32_t *rows, const int32_t *cols,
                    const float *x, float *hi, float *lo, int64_t max_elems, void *stream) {
    if (n_mats == 0 || max_elems == 0) return 0;
    dim3 grid((unsigned)((max_elems + 255) / 256), (unsigned)n_mats);
    cgpdl::launch(k_split_tf32_t, grid, dim3(256), 0, (cudaStream_t)stream, off, rows, cols, x,
                  hi, lo);
    CG_CHECK_LAUNCH("k_split_tf32_t");
    return 1;
}

int cg_split_tf32(int64_t n, const float *x, float *hi, float *lo, void *stream) {
    if (n == 0) return 0;
    k_split_tf32<<<grid_for(n, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(n, x, hi, lo);
    CG_CHECK_LAUNCH("k_split_tf32");
    return 1;
}

int cg_plan_frozen(const cg_plan_static *st, int epoch, int staleness, int me, int32_t *req_ver,
                   int32_t *glob_ver, int32_t *halo_row, int32_t *stage_src, int32_t *stage_row,
                   int32_t *stage_dst, int32_t *gw_slot, int64_t *counts, int32_t *flag,
                   int32_t staging_base, int32_t n_devices, int8_t *outcome,
                   const int32_t *epoch_dev, void *stream) {
    if (st->n_union == 0) return 0;
    if (st->n_parts > kPlanMaxParts) {
        cg_set_error("cg_plan_frozen: too many partition slots");
        return -1;
    }
    cgpdl::launch(k_plan_frozen, dim3((unsigned)((st->n_union + 255) / 256)), dim3(256), 0,
                  (cudaStream_t)stream, *st, epoch, staleness, me, req_ver, glob_ver, halo_row,
                  stage_src, stage_row, stage_dst, gw_slot, counts, flag, staging_base, n_devices,
                  outcome, epoch_dev);
    CG_CHECK_LAUNCH("k_plan_frozen");
    return 1;
}

}  // extern "C"
