// K5 on the 5th-generation tensor cores (sm_100a): tcgen05.mma kind::tf32
// with TMA-loaded, 128B-swizzled operand tiles and the accumulator in TMEM.
//
//   mode 1 = 3xTF32 (parity): a*b ~= a_hi*b_hi + a_hi*b_lo + a_lo*b_hi where
//            x_hi = x with the low 13 mantissa bits cleared and x_lo = x - x_hi,
//            split in shared memory by the epilogue warps while the TMA
//            producer runs ahead -- ~fp32 accuracy at 3 MMAs per k-step;
//   mode 2 = 1xTF32 (fast mode, stated looser bound).
//
// One CTA computes a 128 x BN (BN <= 128) output tile.  Warp roles:
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 4..7  operand splitters (3xTF32) and the epilogue: TMEM -> regs ->
//               bias / ReLU / row-scale -> global (warp w%4 owns TMEM lanes
//               32*(w%4) .. +31, i.e. output rows)
// Operands may be K-major or MN-major (both are legal for kind::tf32 on
// sm_100), so every GEMM of the layer -- forward Z.W, input gradient
// dY.W^T and the weight gradient Z^T.dY (both operands MN-major, reduced
// over a deterministic split of the long vertex axis) -- reads its operands
// straight from the row-major activation buffers, with no transposes.

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/capgnn.h"
#include "pdl.cuh"

extern void cg_set_error(const std::string &msg);
extern int cg_cuda_fail(cudaError_t e, const char *what);

namespace tc {

constexpr int BM = 128;          // UMMA M (cta_group::1)
constexpr int BK = 32;           // fp32 elements per 128-byte swizzle row
constexpr int UK = 8;            // K per tcgen05.mma kind::tf32
constexpr int BN_MAX = 256;     // TMEM columns per accumulator buffer (1xTF32 tiles)
constexpr int BN_MAX_3X = 128;  // 3xTF32 tiles: smaller B slices buy a deeper stage ring
constexpr int A_BYTES = BM * BK * 4;             // 16 KB A operand stage
constexpr int EPI_BUF = 4096;               // one 32 rows x 128 B TMA staging buffer
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int SMEM_BARS = 1024;              // mbarriers + TMEM slot
// Stage layout: [A | B] (hi) and, for 3xTF32, [A_lo | B_lo] at +hi_bytes.
constexpr int THREADS = 384;  // 12 warps: TMA, MMA, -, -, 4 epilogue, 4 splitter

struct Op {
    int K;           // reduction extent of this operand pair
    int a_mn, b_mn;  // 1 = MN-major
};

struct Params {
    int64_t M;       // rows of the output tile space (GEMM M)
    int N;           // GEMM N
    int n_ops;
    Op op[2];
    int64_t k_chunk;  // split-K: reduction elements per blockIdx.z (0 = all)
    const float *bias;
    int relu;
    const float *row_scale;
    const float *mask;
    int64_t ldm;
    float *C;
    int64_t ldc;
    int split3;      // 3xTF32
    int b_presplit;  // 3xTF32 with B supplied as (hi, lo) tensors: split A only
    int stages;
    int hi_bytes;    // bytes of [A | B] in one stage (1024-aligned)
    int BN;          // UMMA N (multiple of 16)
    int vec_ok;      // C / mask / bias rows 16-byte aligned: float4 epilogue
    int a_tmem;      // 3xTF32, K-major A: the splitter moves A and A_lo into TMEM
                     // (tcgen05.mma A-from-TMEM), so smem carries only B traffic
    int stage_bytes;
    int b_lo_off;    // offset of B_lo from the B slice in a stage
    int acc_stride;  // TMEM columns between the two accumulator buffers
    int tma_store;   // C written by TMA bulk tensor stores (mC is valid)
    int tma_mask;    // ReLU-backward mask tiles TMA-loaded into the store staging (mM)
    int nbuf;        // staging buffers per epilogue warp (2, or 4 to prefetch masks)
    int bres;        // B resident: the CTA's whole B slice (hi + lo, every k-block) is
                     // TMA-loaded into smem once and the ring streams A only
    int ring_off;    // byte offset of the stage ring (= resident B bytes, 1024-aligned)
    int bres_kb;     // bytes per resident k-block of B (hi; lo at bres_lo_off)
    int bres_lo_off;
    int pf_dist;     // k-blocks the L2 prefetch cursor runs ahead of the TMA loads
    const uint32_t *mbits;   // ReLU-backward mask as bits (bit j of word w of a row =
    int64_t ld_mbits;        //   column 32 w + j > 0), words per row
    uint32_t *bits_out;      // ReLU layers: the output's > 0 pattern, same format
    int64_t ld_bits_out;
    float *bws;      // weight gradient only: per (chunk, splitter warp) column sums
                     // of the MN-major B operand (= the bias gradient partials)
    int dbg;         // diagnostics only (CG_GEMM_DBG, wrong results): 1 = splitter
                     // skips its work, 2 = epilogue skips its stores
};

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

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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


// x - trunc_tf32(x) (exact in fp32; the MMA truncates it to TF32 in turn)
__device__ __forceinline__ uint32_t lo_of_trunc(uint32_t x) {
    return __float_as_uint(__uint_as_float(x) - __uint_as_float(x & 0xFFFFE000u));
}

__device__ __forceinline__ bool elect_one() {
    uint32_t e;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(e));
    return e != 0;
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap *map, uint64_t *bar, void *dst,
                                            int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor (sm_100 version bits).  Layout type 2 is the
// 128B swizzle (K-major operands); type 1 is 128B swizzle with 32-byte
// atomicity, the only MN-major layout kind::tf32 accepts.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

// Instruction descriptor: D f32, A/B tf32, majors, N, M.
__device__ __forceinline__ uint32_t instr_desc(int a_mn, int b_mn, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) |
           ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t b,
                                            uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
        "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),
        "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),
        "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap *map, uint64_t *bar, void *dst, int x,
                                            int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// L2 prefetch of a TMA box (no smem, no barrier): runs the operand stream
// further ahead of the smem ring than its stage count allows
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap *map, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y)
                 : "memory");
}

// C tile store: smem (128B-swizzled, 32 rows x 32 fp32) -> global via TMA;
// the tensor map clips rows >= M and columns >= N.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, const void *src, int x, int y,
                                             int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// One k-block (BK = 4 UMMA k-steps) issued by the elected lane of a
// converged warp, with the descriptor / TMEM-column increments done in PTX:
// keeps the issuing warp's per-UMMA overhead to a few instructions (a lone
// thread re-materialises every operand into uniform registers per UMMA).
// ts3: 3xTF32 with A, A_lo in TMEM columns [ta, ta+32): A_lo.B_hi, A.B_lo, A.B_hi
__device__ __forceinline__ void mma_kblock_ts3(uint32_t d, uint32_t ta, uint64_t db, uint64_t dbl,
                                               uint64_t bstep, uint32_t idesc, uint32_t acc,
                                               uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t.reg .b64 b1, b2, b3, l1, l2, l3;\n\t"
        ".reg .b32 a0, a1, a2, a3, o0, o1, o2, o3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "add.s64 b1, %2, %4; add.s64 b2, b1, %4; add.s64 b3, b2, %4;\n\t"
        "add.s64 l1, %3, %4; add.s64 l2, l1, %4; add.s64 l3, l2, %4;\n\t"
        "add.u32 a1, %1, 8; add.u32 a2, %1, 16; add.u32 a3, %1, 24;\n\t"
        "add.u32 o0, %1, 32; add.u32 o1, %1, 40; add.u32 o2, %1, 48; add.u32 o3, %1, 56;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [o0], %2, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [o1], b1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], l1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], b1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [o2], b2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a2], l2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a2], b2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [o3], b3, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a3], l3, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a3], b3, %5, 1;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}"
        ::"r"(d), "r"(ta), "l"(db), "l"(dbl), "l"(bstep), "r"(idesc), "r"(acc),
        "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Split-phase TMEM load: issue a 32-column load, then wait for it later
// with the registers passed as read-write operands, so no use of them can
// be scheduled between the issue and the wait (the next chunk's load is in
// flight while the current chunk is processed).
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld32_wait(uint32_t (&r)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                   "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                   "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]),
                   "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]),
                   "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
}

// Compile-time epilogue variants (the TMA-store path): bit 0 bias, bit 1
// ReLU, bit 2 row scale, bit 3 ReLU-backward mask (TMA-loaded).  EPI_GENERIC
// keeps every operand a runtime switch (direct stores, unaligned shapes,
// the diagnostics knobs).
constexpr int EPI_BIAS = 1, EPI_RELU = 2, EPI_RS = 4, EPI_MASK = 8, EPI_MBITS = 16,
              EPI_GENERIC = -1;

// Tile t of the persistent schedule -> (m tile, n tile, split-K chunk);
// consecutive t share the m tile so concurrently running CTAs reuse the A
// rows through L2.
struct TileCoord {
    int64_t m0;
    int n0;
    int z;
};

// Tile index -> coordinates.  Tile counts fit 32 bits (m_tiles * n_tiles *
// chunks < 2^31 for any M < 2^38), so 32-bit divisions suffice; the epilogue's
// mask-prefetch cursor calls this per 32-column chunk, where 64-bit division
// chains were the masked GEMM's critical path.
__device__ __forceinline__ TileCoord tile_of(const Params &p, int64_t t, int n_tiles,
                                             int64_t m_tiles) {
    TileCoord c;
    const uint32_t per_z = (uint32_t)(m_tiles * n_tiles);
    const uint32_t tt = (uint32_t)t;
    c.z = (int)(tt / per_z);
    const uint32_t r = tt - (uint32_t)c.z * per_z;
    const uint32_t mt = r / (uint32_t)n_tiles;
    c.m0 = (int64_t)mt * BM;
    c.n0 = (int)(r - mt * (uint32_t)n_tiles) * p.BN;
    return c;
}

__device__ __forceinline__ void kblocks(const Params &p, int o, int z, int &begin, int &count) {
    int64_t k_lo = 0, k_hi = p.op[o].K;
    if (p.k_chunk > 0) {
        k_lo = (int64_t)z * p.k_chunk;
        k_hi = (k_lo + p.k_chunk < k_hi) ? k_lo + p.k_chunk : k_hi;
    }
    begin = (int)(k_lo / BK);
    count = k_hi > k_lo ? (int)((k_hi - k_lo + BK - 1) / BK) : 0;
}

// Persistent warp-specialised kernel: the smem stage ring and the two TMEM
// accumulator buffers run continuously across this CTA's tiles, so the
// epilogue of tile i overlaps the TMA + MMA of tile i+1.
template <int EPI>
__global__ void __launch_bounds__(THREADS, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mB0,
          const __grid_constant__ CUtensorMap mA1, const __grid_constant__ CUtensorMap mB1,
          const __grid_constant__ CUtensorMap mBl0, const __grid_constant__ CUtensorMap mBl1,
          const __grid_constant__ CUtensorMap mC, const __grid_constant__ CUtensorMap mM,
          const Params p) {
    // no static shared memory in this kernel, so the dynamic window starts
    // 1024-byte aligned (required by the 128B-swizzle atoms); pointers stay
    // derived from the __shared__ array so accesses compile to LDS/STS
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + p.ring_off;   // the stage ring (after any resident B)
    const int S = p.stages;
    const int HI_BYTES = p.hi_bytes;
    const int stage_bytes = p.stage_bytes;
    const uint32_t A_TMEM_COL = 2 * p.acc_stride;  // A / A_lo stage slots follow the accumulators
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * stage_bytes);
    uint64_t *conv = full + S;
    uint64_t *empty = conv + S;
    uint64_t *tfull = empty + S;   // [2] accumulator ready
    uint64_t *tempty = tfull + 2;  // [2] accumulator drained
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    uint64_t *bres_bar = tempty + 3;   // resident B landed
    uint64_t *mbar_mask = tempty + 4;  // [4 warps][nbuf] mask-tile arrivals

    // warp index made provably warp-uniform (shfl) so role branches do not diverge
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
    const int n_tiles = (p.N + p.BN - 1) / p.BN;
    const int64_t m_tiles = (p.M + BM - 1) / BM;
    const int64_t n_z = p.k_chunk > 0 ? (p.op[0].K + p.k_chunk - 1) / p.k_chunk : 1;
    const int64_t total_tiles = m_tiles * n_tiles * n_z;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 128);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        for (int a = 0; a < 4 * p.nbuf; ++a) mbar_init(&mbar_mask[a], 1);
        mbar_init(bres_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // barrier init and the TMEM allocation above overlap the previous kernel's
    // tail; global memory is touched only from here on
    pdl_entry();
    const uint32_t tmem_base = *tmem_slot;
    const int nb_b = (p.BN + 31) / 32;  // 32-column boxes for an MN-major B

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (converged
        // warp; the elected lane issues)
        uint32_t it = 0;
        int ring_s = 0;        // it % S, kept as a running counter (no divisions)
        uint32_t ring_ph = 0;  // (it / S) & 1
        if (p.bres) {
            // this CTA's n tile is fixed (gridDim.x % n_tiles == 0): its B slice,
            // every k-block of every operand pair, hi and lo, lands once
            const int n0 = (int)(blockIdx.x % n_tiles) * p.BN;
            if (elect_one()) {
                uint32_t bytes = 0;
                for (int o = 0; o < p.n_ops; ++o)
                    bytes += 2u * ((p.op[o].K + BK - 1) / BK) *
                             (p.op[o].b_mn ? nb_b * 32 * BK * 4 : p.BN * BK * 4);
                mbar_expect_tx(bres_bar, bytes);
                int kbg = 0;
                for (int o = 0; o < p.n_ops; ++o) {
                    const CUtensorMap *mb = o ? &mB1 : &mB0;
                    const CUtensorMap *mbl = o ? &mBl1 : &mBl0;
                    const int nkb = (p.op[o].K + BK - 1) / BK;
                    for (int kb = 0; kb < nkb; ++kb, ++kbg) {
                        uint8_t *sb = smem_raw + kbg * p.bres_kb;
                        uint8_t *sbl = sb + p.bres_lo_off;
                        if (p.op[o].b_mn) {
                            for (int b = 0; b < nb_b; ++b) {
                                tma_load_2d(mb, bres_bar, sb + b * 4096, n0 + 32 * b, kb * BK);
                                tma_load_2d(mbl, bres_bar, sbl + b * 4096, n0 + 32 * b, kb * BK);
                            }
                        } else {
                            tma_load_2d(mb, bres_bar, sb, kb * BK, n0);
                            tma_load_2d(mbl, bres_bar, sbl, kb * BK, n0);
                        }
                    }
                }
            }
            __syncwarp();
        }
        // L2 prefetch cursor over this CTA's (tile, operand pair, k-block)
        // sequence, pf_dist k-blocks ahead of the loads
        int64_t pf_t = blockIdx.x;
        int pf_o = 0, pf_kb = 0, pf_kb0 = 0, pf_nkb = 0;
        TileCoord pf_tc = tile_of(p, pf_t < total_tiles ? pf_t : 0, n_tiles, m_tiles);
        if (pf_t < total_tiles) kblocks(p, 0, pf_tc.z, pf_kb0, pf_nkb);
        auto pf_step = [&]() {
            if (pf_t >= total_tiles) return;
            if (pf_kb < pf_nkb) {
                const CUtensorMap *ma = pf_o ? &mA1 : &mA0;
                const CUtensorMap *mb = pf_o ? &mB1 : &mB0;
                const int k0 = (pf_kb0 + pf_kb) * BK;
                if (lane == 0) {
                    if (p.op[pf_o].a_mn) {
                        for (int b = 0; b < 4; ++b) tma_prefetch_2d(ma, (int)(pf_tc.m0 + 32 * b), k0);
                    } else {
                        tma_prefetch_2d(ma, k0, (int)pf_tc.m0);
                    }
                    if (!p.bres && !p.b_presplit) {   // activations as B (weight gradient)
                        if (p.op[pf_o].b_mn) {
                            for (int b = 0; b < nb_b; ++b) tma_prefetch_2d(mb, pf_tc.n0 + 32 * b, k0);
                        } else {
                            tma_prefetch_2d(mb, k0, pf_tc.n0);
                        }
                    }
                }
            }
            // advance
            if (++pf_kb >= pf_nkb) {
                pf_kb = 0;
                if (++pf_o >= p.n_ops) {
                    pf_o = 0;
                    pf_t += gridDim.x;
                    if (pf_t >= total_tiles) return;
                    pf_tc = tile_of(p, pf_t, n_tiles, m_tiles);
                }
                kblocks(p, pf_o, pf_tc.z, pf_kb0, pf_nkb);
            }
        };
        for (int d = 0; d < p.pf_dist; ++d) pf_step();
        for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
            const TileCoord tc = tile_of(p, t, n_tiles, m_tiles);
            for (int o = 0; o < p.n_ops; ++o) {
                int kb0, nkb;
                kblocks(p, o, tc.z, kb0, nkb);
                const CUtensorMap *ma = o ? &mA1 : &mA0;
                const CUtensorMap *mb = o ? &mB1 : &mB0;
                const CUtensorMap *mbl = o ? &mBl1 : &mBl0;
                const uint32_t bbytes = p.op[o].b_mn ? nb_b * 32 * BK * 4 : p.BN * BK * 4;
                for (int kb = kb0; kb < kb0 + nkb; ++kb, ++it) {
                    const int s = ring_s;
                    if (p.pf_dist > 0) pf_step();
                    mbar_wait(&empty[s], ring_ph ^ 1);
                    if (++ring_s == S) { ring_s = 0; ring_ph ^= 1; }
                    const int k0 = kb * BK;
                    uint8_t *sa = smem + s * stage_bytes;
                    uint8_t *sb = sa + A_BYTES;
                    if (elect_one()) {
                    mbar_expect_tx(&full[s], A_BYTES + (p.bres ? 0u : bbytes * (p.b_presplit ? 2 : 1)));
                    if (p.op[o].a_mn) {
                        for (int b = 0; b < 4; ++b)
                            tma_load_2d(ma, &full[s], sa + b * 4096, (int)(tc.m0 + 32 * b), k0);
                    } else {
                        tma_load_2d(ma, &full[s], sa, k0, (int)tc.m0);
                    }
                    if (p.bres) {
                        // B is resident
                    } else if (p.op[o].b_mn) {
                        for (int b = 0; b < nb_b; ++b) {
                            tma_load_2d(mb, &full[s], sb + b * 4096, tc.n0 + 32 * b, k0);
                            if (p.b_presplit)
                                tma_load_2d(mbl, &full[s], sb + p.b_lo_off + b * 4096,
                                            tc.n0 + 32 * b, k0);
                        }
                    } else {
                        tma_load_2d(mb, &full[s], sb, k0, tc.n0);
                        if (p.b_presplit) tma_load_2d(mbl, &full[s], sb + p.b_lo_off, k0, tc.n0);
                    }
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (converged
        // warp; one elected lane issues inside mma_kblock_*; the others idle)
        uint32_t it = 0, ti = 0;
        int ring_s = 0;
        uint32_t ring_ph = 0;
        if (p.bres) mbar_wait(bres_bar, 0);
        for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x, ++ti) {
            const TileCoord tc = tile_of(p, t, n_tiles, m_tiles);
            const uint32_t acc_buf = ti & 1;
            mbar_wait(&tempty[acc_buf], ((ti >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t tmem_d = tmem_base + acc_buf * p.acc_stride;
            bool first = true;
            int kbg = 0;   // global k-block index over the operand pairs (resident B)
            for (int o = 0; o < p.n_ops; ++o) {
                int kb0, nkb;
                kblocks(p, o, tc.z, kb0, nkb);
                const int a_mn = p.op[o].a_mn, b_mn = p.op[o].b_mn;
                // an A operand in TMEM is always K-major (lane = row, column = k)
                const uint32_t idesc = instr_desc(p.a_tmem ? 0 : a_mn, b_mn, p.BN);
                // K-major (SW128): 8-row x 128 B atoms, SBO = 1024, k-step = +32 B.
                // MN-major (SW128, 32 B atoms): 4-row x 128 B atoms, SBO = 512
                // between K groups, LBO = 4096 between the 32-wide MN boxes,
                // k-step = +1024 B.
                const uint32_t a_lbo = a_mn ? 4096 : 16, b_lbo = b_mn ? 4096 : 16;
                const uint32_t a_sbo = a_mn ? 512 : 1024, b_sbo = b_mn ? 512 : 1024;
                const uint32_t a_lay = a_mn ? 1u : 2u, b_lay = b_mn ? 1u : 2u;
                const uint32_t a_step = a_mn ? 1024 : 32, b_step = b_mn ? 1024 : 32;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = ring_s;
                    const uint32_t ph = ring_ph;
                    if (++ring_s == S) { ring_s = 0; ring_ph ^= 1; }
                    if (p.split3) mbar_wait(&conv[s], ph);
                    else mbar_wait(&full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sa = smem_u32(smem + s * stage_bytes);
                    const uint32_t sb = p.bres ? smem_u32(smem_raw) + (kbg + kb) * p.bres_kb
                                               : sa + A_BYTES;
                    const uint32_t sa_lo = sa + HI_BYTES;
                    const uint32_t sb_lo = sb + (p.bres ? p.bres_lo_off : p.b_lo_off);
                    if (p.a_tmem) {
                        // A (= its TF32 truncation) and A_lo sit in TMEM slot s
                        mma_kblock_ts3(tmem_d, tmem_base + A_TMEM_COL + 64 * s,
                                           smem_desc(sb, b_lbo, b_sbo, b_lay),
                                           smem_desc(sb_lo, b_lbo, b_sbo, b_lay), b_step >> 4,
                                           idesc, first ? 0u : 1u, &empty[s]);
                        first = false;
                        __syncwarp();
                        continue;
                    }
                    if (lane == 0) {
#pragma unroll
                    for (int j = 0; j < BK / UK; ++j) {
                        const uint64_t da = smem_desc(sa + j * a_step, a_lbo, a_sbo, a_lay);
                        const uint64_t db = smem_desc(sb + j * b_step, b_lbo, b_sbo, b_lay);
                        const uint32_t acc0 = first ? 0u : 1u;
                        first = false;
                        if (p.split3) {
                            const uint64_t dal = smem_desc(sa_lo + j * a_step, a_lbo, a_sbo, a_lay);
                            const uint64_t dbl = smem_desc(sb_lo + j * b_step, b_lbo, b_sbo, b_lay);
                            mma_tf32(tmem_d, dal, db, idesc, acc0);
                            mma_tf32(tmem_d, da, dbl, idesc, 1u);
                            mma_tf32(tmem_d, da, db, idesc, 1u);
                        } else {
                            mma_tf32(tmem_d, da, db, idesc, acc0);
                        }
                    }
                    mma_commit(&empty[s]);  // frees the smem slot once these MMAs retire
                    }
                    first = false;
                    __syncwarp();
                }
                kbg += nkb;
            }
            if (lane == 0) mma_commit(&tfull[acc_buf]);
            __syncwarp();
        }
    } else if (EPI >= 0 && warp >= 4 && warp < 8) {
        // ------------------------------------------------ epilogue, compile-time
        // variant: TMEM -> registers (the next 32-column chunk's load in flight
        // while this one is processed) -> bias / ReLU / row scale / mask ->
        // swizzled staging buffer -> TMA bulk store
        constexpr bool HB = (EPI & EPI_BIAS) != 0, RL = (EPI & EPI_RELU) != 0;
        constexpr bool RS = (EPI & EPI_RS) != 0, MK = (EPI & EPI_MASK) != 0;
        constexpr bool MB = (EPI & EPI_MBITS) != 0;
        // (a second group of epilogue warps taking every other chunk was
        // measured slower once the operand feed, not the epilogue, bound
        // these GEMMs: fwd0 57 -> 81 us with resident B)
        const int q = warp & 3;
        constexpr int G = 1, g = 0;
        const int NB = p.nbuf;
        const int nb_log = 31 - __clz(NB);
        uint8_t *stg0 = smem + S * stage_bytes + SMEM_BARS + q * NB * EPI_BUF;
        uint64_t *mbq = mbar_mask + q * NB;
        uint32_t ti = 0, nst = 0;
        // mask prefetch cursor (see the generic epilogue): D = NB - 2 chunks ahead
        const int D = NB - 2;
        int64_t pf_t = blockIdx.x;
        int pf_c = g;
        uint32_t pf_k = 0;
        TileCoord pc = tile_of(p, pf_t < total_tiles ? pf_t : 0, n_tiles, m_tiles);
        // first valid chunk of this group
        while (pf_t < total_tiles && (pf_c * 32 >= p.BN || p.N - (pc.n0 + 32 * pf_c) <= 0)) {
            pf_c = g;
            pf_t += gridDim.x;
            if (pf_t < total_tiles) pc = tile_of(p, pf_t, n_tiles, m_tiles);
        }
        auto pf_issue = [&]() -> bool {
            if (pf_t >= total_tiles) return false;
            if (lane == 0) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                uint64_t *bar = &mbq[pf_k & (NB - 1)];
                mbar_expect_tx(bar, EPI_BUF);
                tma_load_3d(&mM, bar, stg0 + (pf_k & (NB - 1)) * EPI_BUF, pc.n0 + 32 * pf_c,
                            (int)(pc.m0 + 32 * q), 0);
            }
            ++pf_k;
            while (true) {
                pf_c += G;
                if (pf_c * 32 >= p.BN) {
                    pf_c = g;
                    pf_t += gridDim.x;
                    if (pf_t < total_tiles) pc = tile_of(p, pf_t, n_tiles, m_tiles);
                }
                if (pf_t >= total_tiles) break;
                if (pf_c * 32 < p.BN && p.N - (pc.n0 + 32 * pf_c) > 0) break;
            }
            return true;
        };
        const int nch_max = (p.BN + 31) / 32;
        for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x, ++ti) {
            const TileCoord tc = tile_of(p, t, n_tiles, m_tiles);
            const uint32_t acc_buf = ti & 1;
            const int64_t row = tc.m0 + 32 * q + lane;
            float rs = 1.f;
            if (RS && row < p.M) rs = __ldg(p.row_scale + row);
            int nch = (p.N - tc.n0 + 31) / 32;
            if (nch > nch_max) nch = nch_max;
            mbar_wait(&tfull[acc_buf], (ti >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t tb = tmem_base + acc_buf * p.acc_stride + ((uint32_t)(32 * q) << 16);
            uint32_t va[32], vb[32];
            auto chunk = [&](const uint32_t (&v)[32], int c) {
                const int c0 = 32 * c;
                const int ncol = p.N - (tc.n0 + c0);   // > 0; may exceed 32
                const uint32_t buf = nst & (NB - 1);
                const uint32_t stg = smem_u32(stg0 + buf * EPI_BUF);
                float4 mk[8];
                if constexpr (MK) {
                    while (pf_k <= nst + D && pf_issue()) {}
                    mbar_wait(&mbq[buf], (nst >> nb_log) & 1);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(mk[j].x), "=f"(mk[j].y), "=f"(mk[j].z), "=f"(mk[j].w)
                                     : "r"(stg + lane * 128 + 16 * (j ^ (lane & 7)))
                                     : "memory");
                } else {
                    // the store NB chunks ago has finished reading this buffer
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                }
                __syncwarp();
                const float *brow = HB ? p.bias + tc.n0 + c0 : nullptr;
                const bool row_ok = row < p.M;
                uint32_t mw = 0, bw = 0;   // mask bits in, ReLU bits out (32 columns)
                if constexpr (MB) {
                    if (row_ok) mw = __ldg(p.mbits + row * p.ld_mbits + ((tc.n0 + c0) >> 5));
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float4 y = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                           __uint_as_float(v[4 * j + 2]),
                                           __uint_as_float(v[4 * j + 3]));
                    if constexpr (HB) {
                        // columns >= N are clipped by the store; never read past the bias
                        const float4 bb = 4 * j < ncol
                            ? __ldg(reinterpret_cast<const float4 *>(brow) + j)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
                        y.x += bb.x; y.y += bb.y; y.z += bb.z; y.w += bb.w;
                    }
                    if constexpr (RL) {
                        y.x = fmaxf(y.x, 0.f); y.y = fmaxf(y.y, 0.f);
                        y.z = fmaxf(y.z, 0.f); y.w = fmaxf(y.w, 0.f);
                    }
                    if constexpr (RS) {
                        y.x *= rs; y.y *= rs; y.z *= rs; y.w *= rs;
                    }
                    if constexpr (MK) {
                        const float4 m = mk[j];
                        y.x = m.x > 0.f ? y.x : 0.f; y.y = m.y > 0.f ? y.y : 0.f;
                        y.z = m.z > 0.f ? y.z : 0.f; y.w = m.w > 0.f ? y.w : 0.f;
                    }
                    if constexpr (MB) {
                        const uint32_t b = mw >> (4 * j);
                        y.x = (b & 1u) ? y.x : 0.f; y.y = (b & 2u) ? y.y : 0.f;
                        y.z = (b & 4u) ? y.z : 0.f; y.w = (b & 8u) ? y.w : 0.f;
                    }
                    if constexpr (RL) {
                        bw |= ((y.x > 0.f ? 1u : 0u) | (y.y > 0.f ? 2u : 0u) |
                               (y.z > 0.f ? 4u : 0u) | (y.w > 0.f ? 8u : 0u)) << (4 * j);
                    }
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                     stg + lane * 128 + 16 * (j ^ (lane & 7))),
                                 "f"(y.x), "f"(y.y), "f"(y.z), "f"(y.w)
                                 : "memory");
                }
                if constexpr (RL) {
                    // the > 0 pattern of the stored values (columns >= N clip to 0)
                    if (p.bits_out && row_ok) {
                        if (ncol < 32) bw &= (1u << ncol) - 1u;
                        p.bits_out[row * p.ld_bits_out + ((tc.n0 + c0) >> 5)] = bw;
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0)
                    tma_store_3d(&mC, stg0 + buf * EPI_BUF, tc.n0 + c0, (int)(tc.m0 + 32 * q), tc.z);
                ++nst;
            };
            if (g < nch) tmem_ld32_issue(tb + 32 * g, va);
            for (int c = g; c < nch; c += 2 * G) {
                tmem_ld32_wait(va);
                if (c + G < nch) tmem_ld32_issue(tb + 32 * (c + G), vb);
                chunk(va, c);
                if (c + G < nch) {
                    tmem_ld32_wait(vb);
                    if (c + 2 * G < nch) tmem_ld32_issue(tb + 32 * (c + 2 * G), va);
                    chunk(vb, c + G);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&tempty[acc_buf]);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else if (EPI < 0 && warp >= 4 && warp < 8) {
        // ------------------------------------------------ epilogue
        // Warp q owns TMEM lanes 32q..32q+31 = tile rows; thread = one output
        // row.  Each 32-column chunk goes TMEM -> 32 registers -> bias / ReLU
        // / row scale / ReLU-backward mask -> eight 16-byte stores of the
        // row's 128-byte segment (no transposes, ~4 instructions per float4).
        const int q = warp & 3;
        const int NB = p.nbuf;
        uint8_t *stg0 = smem + S * stage_bytes + SMEM_BARS + q * NB * EPI_BUF;  // NB buffers
        uint64_t *mbq = mbar_mask + q * NB;
        uint32_t ti = 0, nst = 0;
        // Mask prefetch cursor over this warp's (tile, chunk) sequence, valid
        // chunks only: masks run D = NB - 2 chunks ahead of the one consumed,
        // so the buffer a prefetch lands in was last stored from two chunks
        // before the current one (wait_group.read 1 frees it).
        const int D = NB - 2;
        int64_t pf_t = blockIdx.x;
        int pf_c = 0;
        uint32_t pf_k = 0;
        TileCoord pc = tile_of(p, pf_t < total_tiles ? pf_t : 0, n_tiles, m_tiles);
        auto pf_issue = [&]() -> bool {
            if (pf_t >= total_tiles) return false;   // sequence exhausted
            if (lane == 0) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                uint64_t *bar = &mbq[pf_k & (NB - 1)];
                mbar_expect_tx(bar, EPI_BUF);
                tma_load_3d(&mM, bar, stg0 + (pf_k & (NB - 1)) * EPI_BUF, pc.n0 + 32 * pf_c,
                            (int)(pc.m0 + 32 * q), 0);
            }
            ++pf_k;
            // advance to the next chunk with columns left
            while (true) {
                if (++pf_c * 32 >= p.BN) {
                    pf_c = 0;
                    pf_t += gridDim.x;
                    if (pf_t < total_tiles) pc = tile_of(p, pf_t, n_tiles, m_tiles);
                }
                if (pf_t >= total_tiles) break;
                if (p.N - (pc.n0 + 32 * pf_c) > 0) break;
            }
            return true;
        };
        for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x, ++ti) {
            const TileCoord tc = tile_of(p, t, n_tiles, m_tiles);
            const uint32_t acc_buf = ti & 1;
            mbar_wait(&tfull[acc_buf], (ti >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t row = tc.m0 + 32 * q + lane;
            const bool row_ok = row < p.M;
            float *cbase = p.k_chunk > 0 ? p.C + (int64_t)tc.z * p.M * p.ldc : p.C;
            float *crow = cbase + (row_ok ? row : 0) * p.ldc + tc.n0;
            const float *mrow = p.mask ? p.mask + (row_ok ? row : 0) * p.ldm + tc.n0 : nullptr;
            const float rs = (p.row_scale && row_ok) ? p.row_scale[row] : 1.f;
            const float *brow = p.bias ? p.bias + tc.n0 : nullptr;
            for (int c0 = 0; c0 < p.BN; c0 += 32) {
                int ncol = p.N - (tc.n0 + c0);
                if (ncol > p.BN - c0) ncol = p.BN - c0;
                if (ncol > 32) ncol = 32;
                if (p.tma_store && p.tma_mask && ncol > 0 && !(p.dbg & 2)) {
                    // mask blocks come by TMA into the staging buffers the
                    // chunks will be stored from, D chunks ahead
                    while (pf_k <= nst + D && pf_issue()) {}
                }
                float v[32];
                tmem_ld32(tmem_base + acc_buf * p.acc_stride + ((uint32_t)(32 * q) << 16) + c0, v);
                if (ncol <= 0) continue;
                if (p.dbg & 2) {
                    if (v[0] == 12345.f) crow[c0] = v[1];   // keep the load live
                    continue;
                }
                if (p.tma_store) {
                    // apply the epilogue in registers, stage the 32 x 32 block
                    // (swizzled: chunk j of row r at j ^ (r & 7)), one TMA store
                    const uint32_t stg = smem_u32(stg0 + (nst & (NB - 1)) * EPI_BUF);
                    float4 mk[8];
                    if (p.tma_mask) {
                        mbar_wait(&mbq[nst & (NB - 1)], (nst >> (31 - __clz(NB))) & 1);
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                         : "=f"(mk[j].x), "=f"(mk[j].y), "=f"(mk[j].z), "=f"(mk[j].w)
                                         : "r"(stg + lane * 128 + 16 * (j ^ (lane & 7)))
                                         : "memory");
                    } else if (mrow && row_ok) {
                        // issue the row's mask loads before anything waits
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            if (4 * j >= ncol) {
                                mk[j] = make_float4(1.f, 1.f, 1.f, 1.f);
                            } else if (p.vec_ok) {
                                mk[j] = __ldg(reinterpret_cast<const float4 *>(mrow + c0) + j);
                            } else {
                                const int cb = c0 + 4 * j;
                                mk[j].x = mrow[cb];
                                mk[j].y = 4 * j + 1 < ncol ? mrow[cb + 1] : 0.f;
                                mk[j].z = 4 * j + 2 < ncol ? mrow[cb + 2] : 0.f;
                                mk[j].w = 4 * j + 3 < ncol ? mrow[cb + 3] : 0.f;
                            }
                        }
                    }
                    if (lane == 0 && !p.tma_mask)  // the store NB chunks ago has read this buffer
                        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float4 bb = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (brow) {
                            if (p.vec_ok) {
                                bb = __ldg(reinterpret_cast<const float4 *>(brow + c0) + j);
                            } else {
                                const int cb = c0 + 4 * j;
                                bb.x = 4 * j < ncol ? brow[cb] : 0.f;
                                bb.y = 4 * j + 1 < ncol ? brow[cb + 1] : 0.f;
                                bb.z = 4 * j + 2 < ncol ? brow[cb + 2] : 0.f;
                                bb.w = 4 * j + 3 < ncol ? brow[cb + 3] : 0.f;
                            }
                        }
                        float4 y = make_float4(v[4 * j] + bb.x, v[4 * j + 1] + bb.y,
                                               v[4 * j + 2] + bb.z, v[4 * j + 3] + bb.w);
                        if (p.relu) {
                            y.x = fmaxf(y.x, 0.f); y.y = fmaxf(y.y, 0.f);
                            y.z = fmaxf(y.z, 0.f); y.w = fmaxf(y.w, 0.f);
                        }
                        y.x *= rs; y.y *= rs; y.z *= rs; y.w *= rs;
                        if (mrow) {
                            const float4 m = mk[j];
                            y.x = m.x > 0.f ? y.x : 0.f; y.y = m.y > 0.f ? y.y : 0.f;
                            y.z = m.z > 0.f ? y.z : 0.f; y.w = m.w > 0.f ? y.w : 0.f;
                        }
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                         stg + lane * 128 + 16 * (j ^ (lane & 7))),
                                     "f"(y.x), "f"(y.y), "f"(y.z), "f"(y.w)
                                     : "memory");
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0)
                        tma_store_3d(&mC, stg0 + (nst & (NB - 1)) * EPI_BUF, tc.n0 + c0,
                                     (int)(tc.m0 + 32 * q), tc.z);
                    ++nst;
                    continue;
                }
                if (!row_ok) continue;
                if (ncol == 32 && p.vec_ok) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float4 bb = brow ? __ldg(reinterpret_cast<const float4 *>(brow + c0) + j)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                        float4 y = make_float4(v[4 * j] + bb.x, v[4 * j + 1] + bb.y,
                                               v[4 * j + 2] + bb.z, v[4 * j + 3] + bb.w);
                        if (p.relu) {
                            y.x = fmaxf(y.x, 0.f); y.y = fmaxf(y.y, 0.f);
                            y.z = fmaxf(y.z, 0.f); y.w = fmaxf(y.w, 0.f);
                        }
                        y.x *= rs; y.y *= rs; y.z *= rs; y.w *= rs;
                        if (mrow) {
                            const float4 m = __ldg(reinterpret_cast<const float4 *>(mrow + c0) + j);
                            y.x = m.x > 0.f ? y.x : 0.f; y.y = m.y > 0.f ? y.y : 0.f;
                            y.z = m.z > 0.f ? y.z : 0.f; y.w = m.w > 0.f ? y.w : 0.f;
                        }
                        reinterpret_cast<float4 *>(crow + c0)[j] = y;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        if (i >= ncol) break;
                        float y = v[i] + (brow ? brow[c0 + i] : 0.f);
                        if (p.relu) y = fmaxf(y, 0.f);
                        y *= rs;
                        if (mrow && !(mrow[c0 + i] > 0.f)) y = 0.f;
                        crow[c0 + i] = y;
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&tempty[acc_buf]);
        }
        if (p.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else if (warp >= 8 && p.split3) {
        // ------------------------------------------------ hi/lo split (3xTF32)
        const int t128 = threadIdx.x - 256;
        uint32_t it = 0;
        int ring_s = 0;        // it % S, kept as a running counter (no divisions)
        uint32_t ring_ph = 0;  // (it / S) & 1
        for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
            const TileCoord tc = tile_of(p, t, n_tiles, m_tiles);
            // bias-gradient partials: only the first row tile of each (n, chunk)
            const bool bws_on = p.bws != nullptr && tc.m0 == 0;
            float4 bacc[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) bacc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int o = 0; o < p.n_ops; ++o) {
                int kb0, nkb;
                kblocks(p, o, tc.z, kb0, nkb);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = ring_s;
                    mbar_wait(&full[s], ring_ph);
                    if (++ring_s == S) { ring_s = 0; ring_ph ^= 1; }
                    if (p.dbg & 1) {
                        mbar_arrive(&conv[s]);
                        continue;
                    }
                    if (p.a_tmem) {
                        const int q = warp & 3, r = 32 * q + lane;
                        uint32_t hv[32], lv[32];
                        if (!p.op[o].a_mn) {
                            // thread = tile row r (TMEM lane): its 32 K values from
                            // the 128B-swizzled K-major A tile (16-byte chunk c of
                            // row r sits at chunk c ^ (r & 7))
                            const uint8_t *rowp = smem + s * stage_bytes + r * 128;
#pragma unroll
                            for (int c = 0; c < 8; ++c) {
                                const uint4 w = *reinterpret_cast<const uint4 *>(rowp + 16 * (c ^ (r & 7)));
                                hv[4 * c] = w.x; hv[4 * c + 1] = w.y; hv[4 * c + 2] = w.z; hv[4 * c + 3] = w.w;
                            }
                        } else {
                            // MN-major A (weight gradient: rows = features, K =
                            // vertices): box q holds features 32q..32q+31, one
                            // 128 B row per vertex, 32-byte atoms swizzled as
                            // atom c of row v at c ^ (v & 3) (CuTe Swizzle<2,5,2>)
                            const uint8_t *boxp = smem + s * stage_bytes + q * 4096;
                            const int c = lane >> 3, w4 = (lane & 7) * 4;
#pragma unroll
                            for (int v = 0; v < 32; ++v)
                                hv[v] = *reinterpret_cast<const uint32_t *>(
                                    boxp + v * 128 + 32 * (c ^ (v & 3)) + w4);
                        }
                        if (!p.b_presplit) {
                            // activations as B (weight gradient): B_lo in smem
                            const int nb16 = (p.op[o].b_mn ? nb_b * 32 * BK * 4 : p.BN * BK * 4) / 16;
                            const uint4 *bh = reinterpret_cast<const uint4 *>(smem + s * stage_bytes + A_BYTES);
                            uint4 *bl = reinterpret_cast<uint4 *>(smem + s * stage_bytes + A_BYTES + p.b_lo_off);
                            const int t128 = threadIdx.x - 256;
                            const bool bsum = bws_on && p.op[o].b_mn;
#pragma unroll 8
                            for (int k = 0; k < 8; ++k) {
                                const int i = t128 + 128 * k;
                                if (i >= nb16) break;
                                const uint4 w = bh[i];
                                // B stays raw in smem (the MMA truncates it to
                                // TF32); B_lo = B - trunc(B), exact in fp32
                                bl[i] = make_uint4(lo_of_trunc(w.x), lo_of_trunc(w.y),
                                                   lo_of_trunc(w.z), lo_of_trunc(w.w));
                                if (bsum) {
                                    // MN-major box k/2, this thread's column quad is
                                    // fixed (see the combine below); rows vary with k
                                    float4 &a4 = bacc[k >> 1];
                                    a4.x += __uint_as_float(w.x); a4.y += __uint_as_float(w.y);
                                    a4.z += __uint_as_float(w.z); a4.w += __uint_as_float(w.w);
                                }
                            }
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        }
#pragma unroll
                        for (int i = 0; i < 32; ++i)   // hi = x as is (the MMA truncates)
                            lv[i] = __float_as_uint(__uint_as_float(hv[i]) -
                                                    __uint_as_float(hv[i] & 0xFFFFE000u));
                        const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + A_TMEM_COL + 64 * s;
                        tmem_st32(ta, hv);
                        tmem_st32(ta + 32, lv);
                        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        mbar_arrive(&conv[s]);
                        continue;
                    }
                    // the tensor core truncates fp32 operands to TF32 (measured:
                    // tests/diag_tf32_rounding.py), so the raw tile already acts
                    // as x_hi; only x_lo = x - trunc_tf32(x) is materialised
                    const uint4 *hi = reinterpret_cast<const uint4 *>(smem + s * stage_bytes);
                    uint4 *lo = reinterpret_cast<uint4 *>(smem + s * stage_bytes + HI_BYTES);
                    // B arrives pre-split (weights) or is split here (activations)
                    const int n16 = p.b_presplit
                        ? A_BYTES / 16
                        : (A_BYTES + (p.op[o].b_mn ? nb_b * 32 * BK * 4 : p.BN * BK * 4)) / 16;
#pragma unroll 4
                    for (int i = t128; i < n16; i += 128) {
                        uint4 w = hi[i];
                        uint4 h = make_uint4(w.x & 0xFFFFE000u, w.y & 0xFFFFE000u,
                                             w.z & 0xFFFFE000u, w.w & 0xFFFFE000u);
                        uint4 l = make_uint4(
                            __float_as_uint(__uint_as_float(w.x) - __uint_as_float(h.x)),
                            __float_as_uint(__uint_as_float(w.y) - __uint_as_float(h.y)),
                            __float_as_uint(__uint_as_float(w.z) - __uint_as_float(h.z)),
                            __float_as_uint(__uint_as_float(w.w) - __uint_as_float(h.w)));
                        lo[i] = l;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_arrive(&conv[s]);
                }
            }
            if (bws_on) {
                // Thread t of the splitter warp group owns column quad
                // 8*(((t&7)>>1) ^ ((t>>3)&3)) + 4*(t&1) of every 32-column box
                // (128B-swizzle, 32B atoms: atom c of row v at c ^ (v & 3)).  The
                // 4 lanes of a warp sharing a quad are lane ^ 10 and lane ^ 20:
                // butterfly them, lanes 0..7 hold the warp's 8-row sums.
                const int lw = lane;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float4 &a4 = bacc[k];
#pragma unroll
                    for (int sh = 10; sh <= 20; sh += 10) {
                        a4.x += __shfl_xor_sync(0xffffffffu, a4.x, sh);
                        a4.y += __shfl_xor_sync(0xffffffffu, a4.y, sh);
                        a4.z += __shfl_xor_sync(0xffffffffu, a4.z, sh);
                        a4.w += __shfl_xor_sync(0xffffffffu, a4.w, sh);
                    }
                }
                if (lw < 8) {
                    const int cq = 8 * (lw >> 1) + 4 * (lw & 1);
                    float *dst = p.bws + ((int64_t)tc.z * 4 + (warp & 3)) * p.N;
                    for (int k = 0; k < nb_b && k < 4; ++k) {
                        const int n = tc.n0 + 32 * k + cq;
                        if (n + 3 < p.N) {
                            *reinterpret_cast<float4 *>(dst + n) = bacc[k];
                        } else {
                            if (n < p.N) dst[n] = bacc[k].x;
                            if (n + 1 < p.N) dst[n + 1] = bacc[k].y;
                            if (n + 2 < p.N) dst[n + 2] = bacc[k].z;
                        }
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(512));
    }
}

// ------------------------------------------------------------------ host

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
                cudaSuccess &&
            p)
            fn = reinterpret_cast<encode_fn_t>(p);
    }
    return fn;
}

// 2-D fp32 tensor [outer x inner] with row stride ld (elements), box {32, box_outer}.
bool make_map(CUtensorMap *m, const float *ptr, int64_t inner, int64_t outer, int64_t ld,
              int box_outer, bool mn_major) {
    encode_fn_t enc = encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {32u, (cuuint32_t)box_outer};
    cuuint32_t estr[2] = {1u, 1u};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// C viewed as [n_z][M][N] (row stride ldc, z stride M*ldc), box 32 x 32 x 1.
bool make_map_c(CUtensorMap *m, float *C, int64_t M, int N, int64_t ldc, int64_t n_z) {
    encode_fn_t enc = encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)n_z};
    cuuint64_t strides[2] = {(cuuint64_t)ldc * 4, (cuuint64_t)(M * ldc * 4)};
    cuuint32_t box[3] = {32u, 32u, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, C, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

typedef void (*KernelFn)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                         const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                         const Params);

template <int EPI>
KernelFn prepared() {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<EPI>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT);
        if (e != cudaSuccess) {
            cg_cuda_fail(e, "cudaFuncSetAttribute(k_gemm_tc)");
            return nullptr;
        }
        attr_set = true;
    }
    return k_gemm_tc<EPI>;
}

// The variants the training epoch uses: weight gradients and SAGE's second
// input-gradient term (none), the last layer's transform (bias), SAGE hidden
// layers (bias + ReLU), GCN input gradients (row scale), GCN hidden layers
// (bias + ReLU + row scale), and the ReLU-backward masked input gradient.
bool instantiated(int epi) {
    return epi == 0 || epi == EPI_BIAS || epi == (EPI_BIAS | EPI_RELU) || epi == EPI_RS ||
           epi == (EPI_BIAS | EPI_RELU | EPI_RS) || epi == EPI_MASK || epi == EPI_MBITS;
}

KernelFn kernel_for(int epi) {
    switch (epi) {
        case 0: return prepared<0>();
        case EPI_BIAS: return prepared<EPI_BIAS>();
        case EPI_BIAS | EPI_RELU: return prepared<EPI_BIAS | EPI_RELU>();
        case EPI_RS: return prepared<EPI_RS>();
        case EPI_BIAS | EPI_RELU | EPI_RS: return prepared<EPI_BIAS | EPI_RELU | EPI_RS>();
        case EPI_MASK: return prepared<EPI_MASK>();
        case EPI_MBITS: return prepared<EPI_MBITS>();
        default: return prepared<EPI_GENERIC>();
    }
}

int launch(const Params &p0, const CUtensorMap &a0, const CUtensorMap &b0, const CUtensorMap &a1,
           const CUtensorMap &b1, const CUtensorMap &bl0, const CUtensorMap &bl1, int grid_z,
           cudaStream_t st) {
    Params p = p0;
    CUtensorMap mc, mm;
    memset(&mc, 0, sizeof(mc));
    memset(&mm, 0, sizeof(mm));
    static const bool no_tma_store = getenv("CG_GEMM_NO_TMA_STORE") != nullptr;  // experiment knob
    static const int dbg = getenv("CG_GEMM_DBG") ? atoi(getenv("CG_GEMM_DBG")) : 0;
    p.dbg = dbg;
    p.tma_store = !no_tma_store && !(p.ldc % 4) && !((uintptr_t)p.C % 16) &&
                  make_map_c(&mc, p.C, p.M, p.N, p.ldc, grid_z);
    p.tma_mask = p.tma_store && p.mask && !(p.ldm % 4) && !((uintptr_t)p.mask % 16) &&
                 make_map_c(&mm, const_cast<float *>(p.mask), p.M, p.N, p.ldm, 1);
    // B slice: MN-major B is loaded in 32-column boxes of 4 KB each
    int b_bytes = 0;
    for (int o = 0; o < p.n_ops; ++o) {
        const int bb = p.op[o].b_mn ? ((p.BN + 31) / 32) * 32 * BK * 4 : p.BN * BK * 4;
        b_bytes = bb > b_bytes ? bb : b_bytes;
    }
    b_bytes = (b_bytes + 1023) / 1024 * 1024;
    p.hi_bytes = A_BYTES + b_bytes;
    // 3xTF32: A and A_lo go to TMEM (split by the splitter warps), B_lo is
    // either TMA-loaded (pre-split weights) or split into smem
    p.a_tmem = p.split3 && p.BN <= 128;
    if (p.a_tmem) {
        p.stage_bytes = A_BYTES + 2 * b_bytes;  // [A | B_hi | B_lo]
        p.b_lo_off = b_bytes;
        // accumulators take the TMEM columns a tile needs (narrow N: 32 / 64),
        // the A / A_lo slots the rest -- up to 7 slots, a deeper operand ring
        p.acc_stride = p.BN <= 32 ? 32 : (p.BN <= 64 ? 64 : 128);
    } else {
        p.stage_bytes = p.split3 ? 2 * p.hi_bytes : p.hi_bytes;  // [A | B] [A_lo | B_lo]
        p.b_lo_off = p.hi_bytes;
        p.acc_stride = BN_MAX;
    }
    // resident B: a weight operand (pre-split hi / lo, no split-K) whose whole
    // CTA slice fits beside the ring is loaded once per CTA; each CTA then
    // keeps one n tile (grid a multiple of the n-tile count) and streams only
    // A -- the per-tile B re-reads from L2 were the short-K GEMMs' bound
    static const bool no_bres = getenv("CG_GEMM_NO_BRES") != nullptr;   // A/B knob
    p.bres = 0;
    p.ring_off = 0;
    {
        int total_kb = 0;
        for (int o = 0; o < p.n_ops; ++o) total_kb += (p.op[o].K + BK - 1) / BK;
        const int bres_bytes = 2 * total_kb * b_bytes;
        const int n_tiles_ = (p.N + p.BN - 1) / p.BN;
        if (!no_bres && p.a_tmem && p.b_presplit && p.k_chunk == 0 && grid_z == 1 &&
            bres_bytes <= 144 * 1024 && n_tiles_ <= 148) {
            p.bres = 1;
            p.ring_off = bres_bytes;
            p.bres_kb = b_bytes;
            p.bres_lo_off = total_kb * b_bytes;
            p.stage_bytes = A_BYTES;   // the ring carries A only
        }
    }
    static const int env_pf = getenv("CG_GEMM_PF") ? atoi(getenv("CG_GEMM_PF")) : -1;
    // measured (C2 shapes): 2 k-blocks ahead helps the A-streaming resident-B
    // GEMMs (fwd0 56.7 -> 53.3 us, fwd2 41.1 -> 37.7 us) and costs the others
    // (fwd1 100.7 -> 109.9 us), which stay without
    p.pf_dist = env_pf >= 0 ? env_pf : (p.bres ? 2 : 0);   // CG_GEMM_PF: A/B knob
    const int stage_bytes = p.stage_bytes;
    // the compile-time epilogue variant (TMA-store path, 16-byte bias rows,
    // N % 4 == 0); anything else takes the generic epilogue
    static const bool no_fast = getenv("CG_GEMM_GENERIC_EPI") != nullptr;  // A/B knob
    int epi = EPI_GENERIC;
    if (!no_fast && !dbg && p.tma_store && (!p.mask || p.tma_mask) && !(p.N % 4) &&
        (!p.bias || !((uintptr_t)p.bias % 16)))
        epi = (p.bias ? EPI_BIAS : 0) | (p.relu ? EPI_RELU : 0) | (p.row_scale ? EPI_RS : 0) |
              (p.mask ? EPI_MASK : 0) | (p.mbits ? EPI_MBITS : 0);
    if (!instantiated(epi)) epi = EPI_GENERIC;
    if ((p.mbits || p.bits_out) &&
        (epi == EPI_GENERIC || (p.BN % 32) || (p.bits_out && !p.relu))) {
        cg_set_error("k_gemm_tc: mask bits need the TMA-store epilogue, 32-column tiles "
                     "(N % 32 == 0 and N <= 128 or N % 128 == 0) and, for bits out, ReLU");
        return -1;
    }
    // masked epilogues prefetch their mask tiles NB - 2 chunks ahead: 4 staging
    // buffers per warp, 8 when K is short (<= 2 k-blocks: the epilogue, not the
    // MMA, is then the critical path and 2 operand stages suffice) and one
    // epilogue group drains the tile
    static const int env_nbuf = getenv("CG_GEMM_MASK_NBUF") ? atoi(getenv("CG_GEMM_MASK_NBUF")) : 0;
    const bool short_k = p.n_ops == 1 && p.op[0].K <= 2 * BK;
    const bool env_ok = env_nbuf >= 4 && env_nbuf <= 8 && !(env_nbuf & (env_nbuf - 1));  // 4 or 8
    p.nbuf = p.tma_mask ? (env_ok ? env_nbuf : (short_k ? 8 : 4)) : 2;
    const int smem_fixed = SMEM_BARS + 4 * p.nbuf * EPI_BUF;
    int stages = (SMEM_LIMIT - smem_fixed - p.ring_off) / stage_bytes;
    static const int env_stages = getenv("CG_GEMM_STAGES") ? atoi(getenv("CG_GEMM_STAGES")) : 0;
    int cap = env_stages > 0 ? env_stages : 6;   // experiment knob
    // TMEM: 2 accumulators + one 64-column A / A_lo slot per stage in 512 columns
    const int tmem_slots = (512 - 2 * p.acc_stride) / 64;
    if (p.a_tmem && cap > tmem_slots) cap = tmem_slots;
    p.stages = stages > cap ? cap : stages;
    if (p.stages < 2) {
        cg_set_error("k_gemm_tc: stage does not fit shared memory");
        return -1;
    }
    const size_t smem = (size_t)p.ring_off + (size_t)p.stages * stage_bytes + smem_fixed;
    KernelFn kern = kernel_for(epi);
    if (!kern) return -1;
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        if (n_sm <= 0) n_sm = 148;
    }
    const int64_t tiles = (int64_t)((p.N + p.BN - 1) / p.BN) * ((p.M + BM - 1) / BM) * grid_z;
    unsigned grid = (unsigned)(tiles < n_sm ? tiles : n_sm);   // persistent
    if (p.bres) {   // every CTA keeps one n tile
        const unsigned nt = (unsigned)((p.N + p.BN - 1) / p.BN);
        grid = grid / nt * nt;
    }
    cgpdl::launch(kern, dim3(grid), dim3(THREADS), smem, st, a0, b0, a1, b1, bl0, bl1, mc, mm, p);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : cg_cuda_fail(e, "k_gemm_tc");
}

inline int bn_for(int N, bool split3) {
    const int cap = split3 ? BN_MAX_3X : BN_MAX;
    // equal-width n tiles (e.g. N = 256 -> 2 x 128 under 3xTF32)
    const int n_tiles = (N + cap - 1) / cap;
    int bn = ((N + n_tiles - 1) / n_tiles + 15) / 16 * 16;
    return bn < 16 ? 16 : bn;
}

}  // namespace tc

// C = epi(A1 B1 + A2 B2): A row-major [M x K] (K-major), B either [K x N]
// row-major (MN-major, trans_b = 0) or [N x K] row-major (K-major, trans_b = 1).
int cg_gemm_tc(int64_t M, int N, int K1, const float *A1, int64_t lda1, const float *B1, int K2,
               const float *A2, int64_t lda2, const float *B2, int trans_b, const float *bias,
               int relu, const float *row_scale, const float *mask, int64_t ldm, float *C,
               int64_t ldc, int mode, const float *B1_lo, const float *B2_lo,
               const uint32_t *mbits, int64_t ld_mbits, uint32_t *bits_out, int64_t ld_bits_out,
               cudaStream_t st) {
    using namespace tc;
    if (mode != 1 && mode != 2) {
        cg_set_error("cg_gemm: unknown mode");
        return -1;
    }
    if ((lda1 % 4) || (A2 && lda2 % 4) || (trans_b ? (K1 % 4) : (N % 4)) ||
        ((uintptr_t)A1 % 16) || ((uintptr_t)B1 % 16)) {
        cg_set_error("cg_gemm_tc: operands must be 16-byte aligned with ld % 4 == 0");
        return -1;
    }
    Params p{};
    p.M = M;
    p.N = N;
    p.split3 = mode == 1;
    p.BN = bn_for(N, p.split3);
    p.bias = bias;
    p.relu = relu;
    p.row_scale = row_scale;
    p.mask = mask;
    p.ldm = ldm;
    p.mbits = mbits;
    p.ld_mbits = ld_mbits;
    p.bits_out = bits_out;
    p.ld_bits_out = ld_bits_out;
    p.C = C;
    p.ldc = ldc;
    p.k_chunk = 0;
    p.vec_ok = !(ldc % 4) && !((uintptr_t)C % 16) && (!mask || (!(ldm % 4) && !((uintptr_t)mask % 16))) &&
               (!bias || !((uintptr_t)bias % 16));
    CUtensorMap ma[2], mb[2], mbl[2];
    const float *As[2] = {A1, A2};
    const float *Bs[2] = {B1, B2};
    const float *Bls[2] = {B1_lo, B2_lo};
    const int Ks[2] = {K1, K2};
    const int64_t ldas[2] = {lda1, lda2};
    p.n_ops = (A2 && K2 > 0) ? 2 : 1;
    p.b_presplit = p.split3 && B1_lo && (p.n_ops == 1 || B2_lo);
    for (int o = 0; o < p.n_ops; ++o) {
        p.op[o].K = Ks[o];
        p.op[o].a_mn = 0;
        p.op[o].b_mn = trans_b ? 0 : 1;
        bool ok = make_map(&ma[o], As[o], Ks[o], M, ldas[o], BM, false);
        ok = ok && (trans_b ? make_map(&mb[o], Bs[o], Ks[o], N, Ks[o], p.BN, false)
                            : make_map(&mb[o], Bs[o], N, Ks[o], N, 32, true));
        if (p.b_presplit)
            ok = ok && (trans_b ? make_map(&mbl[o], Bls[o], Ks[o], N, Ks[o], p.BN, false)
                                : make_map(&mbl[o], Bls[o], N, Ks[o], N, 32, true));
        else
            mbl[o] = mb[o];
        if (!ok) {
            cg_set_error("cg_gemm_tc: cuTensorMapEncodeTiled failed");
            return -1;
        }
    }
    if (p.n_ops == 1) {
        ma[1] = ma[0];
        mb[1] = mb[0];
        mbl[1] = mbl[0];
    }
    return launch(p, ma[0], mb[0], ma[1], mb[1], mbl[0], mbl[1], 1, st);
}

// Partial weight gradients: ws[c][k][n] = sum_{m in chunk c} A[m, k] D[m, n].
int cg_wgrad_tc(int64_t M, int K, int N, const float *A, int64_t lda, const float *D, int64_t ldd,
                float *ws, int64_t chunk, int64_t n_chunks, int mode, float *bws,
                cudaStream_t st) {
    using namespace tc;
    if ((lda % 4) || (ldd % 4) || ((uintptr_t)A % 16) || ((uintptr_t)D % 16)) {
        cg_set_error("cg_wgrad_tc: operands must be 16-byte aligned with ld % 4 == 0");
        return -1;
    }
    Params p{};
    p.M = K;          // output rows = input features
    p.N = N;
    p.split3 = mode == 1;
    p.BN = bn_for(N, p.split3);
    p.n_ops = 1;
    p.op[0].K = (int)M;  // reduction over vertices
    p.op[0].a_mn = 1;
    p.op[0].b_mn = 1;
    p.k_chunk = chunk;
    p.C = ws;
    p.ldc = N;
    p.vec_ok = !(N % 4) && !((uintptr_t)ws % 16);
    p.bws = bws;   // caller passes it only for the 3xTF32 path (MN-major B, TMEM A)
    CUtensorMap ma, mb;
    if (!make_map(&ma, A, K, M, lda, BK, true) || !make_map(&mb, D, N, M, ldd, BK, true)) {
        cg_set_error("cg_wgrad_tc: cuTensorMapEncodeTiled failed");
        return -1;
    }
    return launch(p, ma, mb, ma, mb, mb, mb, (int)n_chunks, st);
}
