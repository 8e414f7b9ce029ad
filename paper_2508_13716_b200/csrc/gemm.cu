// K5 dense transforms, SIMT fp32 path (mode 0).
//
//   cg_gemm  : C = epi(A1 B1 [+ A2 B2])  -- forward transform (GCN: Z W,
//              SAGE: H W_self + M W_neigh) and input gradients (dY W^T)
//   cg_wgrad : dW = A^T D with a deterministic split over the long m axis
//
// The tensor-core path (tcgen05, 3xTF32 / TF32) lives in gemm_tc.cu and is
// selected by `mode`; this file is the exact-fp32 reference implementation
// that the tensor-core kernels are checked against.

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

#include "../../include/capgnn.h"

extern void cg_set_error(const std::string &msg);
extern int cg_cuda_fail(cudaError_t e, const char *what);
int cg_gemm_tc(int64_t M, int N, int K1, const float *A1, int64_t lda1, const float *B1, int K2,
               const float *A2, int64_t lda2, const float *B2, int trans_b, const float *bias,
               int relu, const float *row_scale, const float *mask, int64_t ldm, float *C,
               int64_t ldc, int mode, const float *B1_lo, const float *B2_lo,
               const uint32_t *mbits, int64_t ld_mbits, uint32_t *bits_out, int64_t ld_bits_out,
               cudaStream_t st);
int cg_wgrad_tc(int64_t M, int K, int N, const float *A, int64_t lda, const float *D, int64_t ldd,
                float *ws, int64_t chunk, int64_t n_chunks, int mode, float *bws,
                cudaStream_t st);
int cg_colsum(int64_t M, int N, const float *D, int64_t ldd, float *db, float *ws, void *stream);
int cg_reduce_chunks(int64_t n_out, int64_t n_chunks, const float *ws, float *out, cudaStream_t st);
int cg_reduce_chunks_pair(int64_t n1, int64_t c1, const float *ws1, float *out1, int64_t n2,
                          int64_t c2, const float *ws2, float *out2, cudaStream_t st);

namespace {

constexpr int BM = 128, BN = 64, BK = 16, TM = 8, TN = 4, NT = 256;

// B element (k, n): trans_b ? B[n*K + k] : B[k*N + n]
__device__ __forceinline__ float ldB(const float *B, int trans_b, int K, int N, int k, int n) {
    if (k >= K || n >= N) return 0.f;
    return trans_b ? B[(int64_t)n * K + k] : B[(int64_t)k * N + n];
}

__global__ void __launch_bounds__(NT)
k_gemm(int64_t M, int N, int K1, const float *__restrict__ A1, int64_t lda1,
       const float *__restrict__ B1, int K2, const float *__restrict__ A2, int64_t lda2,
       const float *__restrict__ B2, int trans_b, const float *__restrict__ bias, int relu,
       const float *__restrict__ row_scale, const float *__restrict__ mask, int64_t ldm,
       float *__restrict__ C, int64_t ldc) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN];
    const int tid = threadIdx.x;
    const int tx = tid % (BN / TN);   // 16 column groups
    const int ty = tid / (BN / TN);   // 16 row groups
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    const int n0 = blockIdx.y * BN;
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    for (int op = 0; op < 2; ++op) {
        const float *A = op ? A2 : A1;
        const float *B = op ? B2 : B1;
        const int K = op ? K2 : K1;
        const int64_t lda = op ? lda2 : lda1;
        if (!A || K == 0) continue;
        for (int k0 = 0; k0 < K; k0 += BK) {
            // A tile: BM x BK, 8 elements per thread
#pragma unroll
            for (int t = 0; t < (BM * BK) / NT; ++t) {
                int idx = tid + t * NT;
                int r = idx / BK, c = idx % BK;
                int64_t m = m0 + r;
                int k = k0 + c;
                As[c][r] = (m < M && k < K) ? A[m * lda + k] : 0.f;
            }
#pragma unroll
            for (int t = 0; t < (BN * BK) / NT; ++t) {
                int idx = tid + t * NT;
                int c = idx % BN, r = idx / BN;
                Bs[r][c] = ldB(B, trans_b, K, N, k0 + r, n0 + c);
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                float a[TM], b[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
                for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx * TN + j];
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
            __syncthreads();
        }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        int64_t m = m0 + ty * TM + i;
        if (m >= M) continue;
        float rs = row_scale ? row_scale[m] : 1.f;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            int n = n0 + tx * TN + j;
            if (n >= N) continue;
            float v = acc[i][j];
            if (bias) v += bias[n];
            if (relu) v = fmaxf(v, 0.f);
            v *= rs;
            if (mask && !(mask[m * ldm + n] > 0.f)) v = 0.f;
            C[m * ldc + n] = v;
        }
    }
}

// Partial A^T D over one m-chunk: tile 64 (k) x 64 (n), 256 threads x 4x4.
constexpr int WK = 64, WN = 64, WM = 16;
__global__ void __launch_bounds__(256)
k_wgrad_partial(int64_t M, int K, int N, const float *__restrict__ A, int64_t lda,
                const float *__restrict__ D, int64_t ldd, int64_t chunk, float *__restrict__ ws) {
    __shared__ float As[WM][WK];
    __shared__ float Ds[WM][WN];
    const int tid = threadIdx.x;
    const int tk = tid / 16, tn = tid % 16;
    const int k0 = blockIdx.x * WK, n0 = blockIdx.y * WN;
    const int64_t c = blockIdx.z;
    const int64_t mb = c * chunk, me = min(M, mb + chunk);
    float acc[4][4] = {};
    for (int64_t m0 = mb; m0 < me; m0 += WM) {
#pragma unroll
        for (int t = 0; t < (WM * WK) / 256; ++t) {
            int idx = tid + t * 256;
            int r = idx / WK, q = idx % WK;
            int64_t m = m0 + r;
            As[r][q] = (m < me && k0 + q < K) ? A[m * lda + k0 + q] : 0.f;
            Ds[r][q] = (m < me && n0 + q < N) ? D[m * ldd + n0 + q] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < WM; ++r) {
            float a[4], d[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[r][tk * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) d[j] = Ds[r][tn * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], d[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int k = k0 + tk * 4 + i;
        if (k >= K) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int n = n0 + tn * 4 + j;
            if (n < N) ws[(c * K + k) * N + n] = acc[i][j];
        }
    }
}


constexpr int64_t kWgradChunk = 1024;  // minimum split-K chunk (SIMT path: always this)

// Tensor-core split-K chunk: two (k, n, chunk) tiles per SM.  One per SM is
// ~1 % faster per epoch but doubles the fp32 accumulation chain in TMEM
// (C2 dW error 1.6e-5 -> 3.3e-5 of max|dW|); a multiple of the 32-row k-block.
int64_t wgrad_chunk_tc(int64_t M, int K, int N) {
    static const int per_sm = getenv("CG_WGRAD_TILES_PER_SM") ? atoi(getenv("CG_WGRAD_TILES_PER_SM")) : 2;
    const int64_t tiles_mn = ((K + 127) / 128) * ((N + 127) / 128);
    int64_t n_z = (per_sm * 148 + tiles_mn - 1) / tiles_mn;
    int64_t chunk = (M + n_z - 1) / n_z;
    chunk = (chunk + 31) / 32 * 32;
    return chunk < kWgradChunk ? kWgradChunk : chunk;
}

}  // namespace

extern "C" {

int cg_gemm(int64_t M, int N, int K1, const float *A1, int64_t lda1, const float *B1, int K2,
            const float *A2, int64_t lda2, const float *B2, int trans_b, const float *bias,
            int relu, const float *row_scale, const float *mask, int64_t ldm, float *C,
            int64_t ldc, int mode, const float *B1_lo, const float *B2_lo, void *stream) {
    if (M == 0 || N == 0) return 0;
    if (mode != 0)
        return cg_gemm_tc(M, N, K1, A1, lda1, B1, K2, A2, lda2, B2, trans_b, bias, relu,
                          row_scale, mask, ldm, C, ldc, mode, B1_lo, B2_lo, nullptr, 0, nullptr,
                          0, (cudaStream_t)stream);
    dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN));
    k_gemm<<<grid, NT, 0, (cudaStream_t)stream>>>(M, N, K1, A1, lda1, B1, K2, A2, lda2, B2,
                                                 trans_b, bias, relu, row_scale, mask, ldm,
                                                 C, ldc);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : cg_cuda_fail(e, "k_gemm");
}

int cg_gemm_mb(int64_t M, int N, int K1, const float *A1, int64_t lda1, const float *B1, int K2,
               const float *A2, int64_t lda2, const float *B2, int trans_b, const float *bias,
               int relu, const float *row_scale, const uint32_t *mask_bits, int64_t ld_mask_bits,
               uint32_t *bits_out, int64_t ld_bits_out, float *C, int64_t ldc, int mode,
               const float *B1_lo, const float *B2_lo, void *stream) {
    if (M == 0 || N == 0) return 0;
    if (mode != 1 && mode != 2) {
        cg_set_error("cg_gemm_mb: mask bits need a tcgen05 mode (1 or 2)");
        return -1;
    }
    return cg_gemm_tc(M, N, K1, A1, lda1, B1, K2, A2, lda2, B2, trans_b, bias, relu, row_scale,
                      nullptr, 0, C, ldc, mode, B1_lo, B2_lo, mask_bits, ld_mask_bits, bits_out,
                      ld_bits_out, (cudaStream_t)stream);
}

int64_t cg_wgrad_workspace(int64_t M, int K, int N) {
    int64_t nch = (M + kWgradChunk - 1) / kWgradChunk;
    if (nch < 1) nch = 1;
    // dW partials + bias partials (4 per chunk) or the column-sum fallback's
    const int64_t col = ((M + 255) / 256) * N;
    const int64_t bias = nch * 4 * (int64_t)N;
    return nch * (int64_t)K * N + (col > bias ? col : bias) + 4;
}

int cg_wgrad(int64_t M, int K, int N, const float *A, int64_t lda, const float *D, int64_t ldd,
             float *dW, float *db, float *ws, int mode, void *stream) {
    if (K == 0 || N == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t chunk = (mode == 1 || mode == 2) ? wgrad_chunk_tc(M, K, N) : kWgradChunk;
    int64_t nch = (M + chunk - 1) / chunk;
    if (nch < 1) nch = 1;
    int launched = 0;
    // bias gradient: fused into the 3xTF32 kernel (column sums of D while it
    // is split in shared memory), else the standalone column sum
    float *bws = ws + nch * (int64_t)K * N;
    bws = reinterpret_cast<float *>(((uintptr_t)bws + 15) & ~(uintptr_t)15);
    const bool fuse_db = db && mode == 1 && !(N % 4);
    if (mode == 1 || mode == 2) {
        int rc = cg_wgrad_tc(M, K, N, A, lda, D, ldd, ws, chunk, nch, mode,
                             fuse_db ? bws : nullptr, st);
        if (rc < 0) return rc;
        launched += rc;
    } else {
        dim3 grid((K + WK - 1) / WK, (N + WN - 1) / WN, (unsigned)nch);
        k_wgrad_partial<<<grid, 256, 0, st>>>(M, K, N, A, lda, D, ldd, kWgradChunk, ws);
        launched += 1;
    }
    int64_t n_out = (int64_t)K * N;
    int rc;
    if (fuse_db) {   // dW and db partials reduced by one launch
        rc = cg_reduce_chunks_pair(n_out, nch, ws, dW, N, nch * 4, bws, db, st);
        if (rc < 0) return rc;
        launched += rc;
    } else {
        rc = cg_reduce_chunks(n_out, nch, ws, dW, st);
        if (rc < 0) return rc;
        launched += rc;
    }
    if (!fuse_db && db) {
        int rc = cg_colsum(M, N, D, ldd, db, bws, stream);
        if (rc < 0) return rc;
        launched += rc;
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? launched : cg_cuda_fail(e, "cg_wgrad");
}

}  // extern "C"
