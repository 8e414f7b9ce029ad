/*
 * capgnn.h -- C ABI of libcapgnn.so, the B200 (sm_100a) implementation of
 * CaPGNN's per-layer halo exchange + neighbour aggregation hot path.
 *
 * Conventions
 *   - every entry point returns int: >= 0 = OK, < 0 = error; device entry
 *     points return the number of kernels they launched (0 when there was
 *     nothing to do); cg_last_error() returns a thread-local message for
 *     the last failure on this thread;
 *   - plain pointers and sizes only; device buffers are owned by the caller
 *     (PyTorch caching allocator on the Python side) and only borrowed;
 *   - `stream` is a cudaStream_t passed as void*; nothing synchronises the
 *     host unless the function says so;
 *   - feature matrices are fp32 row-major with an explicit leading dimension
 *     (in floats); vertex/row indices are int32, CSR offsets int64.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg):
 *   the reference has no FFI at all -- halopart is pure Python.  Each entry
 *   point below names the Python function/loop whose role it takes over;
 *   INTEGRATION.md shows the ctypes binding a halopart maintainer would add.
 */
#ifndef CAPGNN_H
#define CAPGNN_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library / errors -------------------------------------------------- */
int cg_version(void);                 /* 10000*major + 100*minor + patch   */
const char *cg_last_error(void);      /* thread-local, never NULL          */
int cg_device_count(int *count);
int cg_device_sync(int device);

/* ---- memory tiers ------------------------------------------------------ */
/* Global (host) cache tier: pinned, mapped, portable host memory read and
 * written zero-copy over UVA by kernels (replaces CacheSystem.globl,
 * src/halopart/cache.py:241-242).  *host_ptr is also the device pointer.  */
int cg_host_tier_alloc(size_t bytes, void **host_ptr);
int cg_host_tier_free(void *host_ptr);
/* Register an existing host range (e.g. a POSIX shm segment shared by all
 * ranks of one node) as a mapped, portable pinned tier.                   */
int cg_host_tier_register(void *host_ptr, size_t bytes);
int cg_host_tier_unregister(void *host_ptr);

/* Peer access and CUDA IPC for one-sided NVLink pulls between processes
 * (the reference models this as a cost only: devices.py:73-78).          */
int cg_enable_peer_access(int device, int peer);
int cg_ipc_get_handle(void *dev_ptr, uint8_t handle_out[64], int64_t *offset);
int cg_ipc_open_handle(const uint8_t handle[64], int device, void **dev_ptr);
int cg_ipc_close_handle(void *dev_ptr);

/* Stream-ordered peer synchronisation (replaces the per-layer collective
 * barrier between ranks; the reference's "optimistic locks" between the
 * local / global / prefetch queues).  cg_flag_signal writes
 * `value` into this rank's flag word on `stream` after its preceding work
 * (system-scope fence); cg_flag_wait makes `stream` wait until every flag
 * word flags[i] (device pointers, IPC-mapped for peers; i != skip) is
 * >= value.  Stream memory operations: no kernel, no host sync.          */
int cg_flag_signal(uint32_t *flag, uint32_t value, void *stream);
int cg_flag_wait(const uint64_t *flags, int n, int skip, uint32_t value, void *stream);

/* ---- synthetic inputs (bit-identical to oracle/model_port.py) ---------- */
/* out[r*ld + k] = uniform_pm1(seed, vertex[r], k) * (row_scale? row_scale[r] : 1) */
int cg_hash_features(float *out, int64_t ld, const int32_t *vertex, int64_t n_rows,
                     int F, uint32_t seed, const float *row_scale, void *stream);
int cg_hash_labels(int32_t *out, const int32_t *vertex, int64_t n_rows, int C,
                   uint32_t seed, void *stream);
/* X[r*ld + k] *= scale[r] (GCN source-degree pre-scaling of uploaded rows). */
int cg_scale_rows(float *X, int64_t ld, int64_t n_rows, int F, const float *scale,
                  void *stream);
/* dst[r*ldd + k] = src[r*lds + k] * scale[r]  (scale NULL: plain row copy). */
int cg_scale_rows_to(float *dst, int64_t ldd, const float *src, int64_t lds, int64_t n_rows,
                     int F, const float *scale, void *stream);

/* ---- K3: halo staging / cache write-through ---------------------------- */
/* For i in [0, n): if src_id[i] >= 0 and dst_row[i] >= 0:
 *   dst[dst_row[i]*ld_dst + k] = tab[src_id[i]][src_row[i]*tab_ld[src_id[i]] + k],  k < F
 * `tab` is a device array of source base pointers: local activation
 * buffers, peer buffers (NVLink, P2P/IPC-mapped) or the mapped host tier.
 * dst may itself be a peer or host-tier pointer (write-through).
 * Replaces the data movement behind CacheSystem.lookup outcomes
 * (cache.py:264-309) and the "prefetch queue" of PAPER.md:98.            */
int cg_copy_rows(int64_t n, int F, const int32_t *src_id, const int32_t *src_row,
                 const int32_t *dst_row, const float *const *tab, const int64_t *tab_ld,
                 float *dst, int64_t ld_dst, void *stream);
/* The same copy on at most max_blocks CTAs of 256 threads (<= 0: the
 * default grid).  A copy bound by PCIe or NVLink rather than HBM needs few
 * CTAs in flight; a small grid lets it run on a side stream (the host-tier
 * write-through queue) beside the epoch's kernels without taking their SMs. */
int cg_copy_rows_bounded(int64_t n, int F, const int32_t *src_id, const int32_t *src_row,
                         const int32_t *dst_row, const float *const *tab,
                         const int64_t *tab_ld, float *dst, int64_t ld_dst, int max_blocks,
                         void *stream);
/* The same copy restricted to the entries whose src_id lies in
 * [id_lo, id_hi) (the others are skipped).  One staging table then feeds
 * two queues (PAPER.md:98's prefetch queue, R10): the rows that are final
 * before the epoch starts (the pinned host tier, id = n_dev; every source
 * of the static layer-0 features) are copied ahead on a prefetch stream,
 * and only the current-epoch owner rows (ids < n_dev) wait for the
 * layer's barrier.                                                       */
int cg_copy_rows_sel(int64_t n, int F, const int32_t *src_id, const int32_t *src_row,
                     const int32_t *dst_row, const float *const *tab, const int64_t *tab_ld,
                     float *dst, int64_t ld_dst, int id_lo, int id_hi, int max_blocks,
                     void *stream);

/* ---- K1/K2: fused cache-lookup + gather SpMM --------------------------- */
/* out[r] = epi( scale[r] * sum_{e in [rowptr[r], rowptr[r+1])} X[map(col[e])] )
 * map(c) = c < n_direct ? c : halo_row[c - n_direct]   (halo_row may be NULL)
 * epi: (+ addend[r]) then (* (mask[r] > 0)) when the pointers are non-NULL.
 * Sum order is CSR order (deterministic).  Used for the forward
 * aggregation (CSR of in-edges) and the backward (CSR of out-edges).
 * nnz = rowptr[n_rows] - rowptr[0] when the caller knows it, else -1: it
 * only picks the kernel (rows averaging < 64 edges with 128 < F <= 640 take
 * the cp.async shared-memory ring kernel; results are identical either way).
 * Stand-in replaced: comp_cost's SpMM term (devices.py:119-132).         */
int cg_spmm(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col,
            int64_t n_direct, const int32_t *halo_row, const float *X, int64_t ldx,
            const float *scale, const float *addend, int64_t ld_add,
            const float *mask, int64_t ld_mask, float *out, int64_t ldo, int64_t nnz,
            void *stream);
/* The same aggregation with the ReLU-backward mask given as BITS: bit j of
 * word w of row r (mask_bits[r * ld_mask_bits + w]) stands for column
 * 32 w + j being > 0 -- the pattern cg_gemm_mb's bits_out writes for a
 * ReLU layer's output, 1/32 of the fp32 mask's bytes.  F % 32 == 0.       */
int cg_spmm_mb(int64_t n_rows, int F, const int64_t *rowptr, const int32_t *col,
               int64_t n_direct, const int32_t *halo_row, const float *X, int64_t ldx,
               const float *scale, const float *addend, int64_t ld_add,
               const uint32_t *mask_bits, int64_t ld_mask_bits, float *out, int64_t ldo,
               int64_t nnz, void *stream);

/* ---- K5: dense transform ---------------------------------------------- */
/* C[m, n] = epi( sum_k A1[m,k] B1[k,n] + sum_k A2[m,k] B2[k,n] )  (A2 optional)
 * trans_b = 1 means B is supplied as [N x K] row-major (use B^T).
 * epi: (+ bias[n]) -> (relu if relu) -> (* row_scale[m])
 *      -> (* (mask[m*ldm + n] > 0)) when mask != NULL (ReLU backward).
 * mode: 0 = fp32 SIMT, 1 = 3xTF32 tcgen05 (parity), 2 = 1xTF32 tcgen05.
 * B1_lo / B2_lo (mode 1 only, optional): B is pre-split, B1 = tf32_hi(B),
 * B1_lo = B - tf32_hi(B) (cg_split_tf32 / cg_adam outputs); the kernel then
 * splits only the A operand.                                              */
int cg_gemm(int64_t M, int N, int K1, const float *A1, int64_t lda1,
            const float *B1, int K2, const float *A2, int64_t lda2, const float *B2,
            int trans_b, const float *bias, int relu, const float *row_scale,
            const float *mask, int64_t ldm, float *C, int64_t ldc, int mode,
            const float *B1_lo, const float *B2_lo, void *stream);
/* cg_gemm (tcgen05 modes 1 / 2) with the ReLU-backward mask as bits
 * (mask_bits, format as for cg_spmm_mb; may be NULL) and, for a ReLU layer,
 * the output's > 0 pattern written as bits (bits_out; may be NULL) -- the
 * masks the backward pass reads, at 1/32 of the fp32 bytes.  Bits need
 * N % 32 == 0 with N <= 128 or N % 128 == 0.                              */
int cg_gemm_mb(int64_t M, int N, int K1, const float *A1, int64_t lda1,
               const float *B1, int K2, const float *A2, int64_t lda2, const float *B2,
               int trans_b, const float *bias, int relu, const float *row_scale,
               const uint32_t *mask_bits, int64_t ld_mask_bits, uint32_t *bits_out,
               int64_t ld_bits_out, float *C, int64_t ldc, int mode, const float *B1_lo,
               const float *B2_lo, void *stream);
/* hi[i] = x[i] with the low 13 mantissa bits cleared (a TF32 value),
 * lo[i] = x[i] - hi[i] (exact).                                           */
int cg_split_tf32(int64_t n, const float *x, float *hi, float *lo, void *stream);
/* The same split, transposed, for n_mats row-major matrices packed in one
 * flat buffer: matrix m (rows[m] x cols[m]) at element offset off[m] of x
 * is written as its transpose (cols x rows) at the same offset of hi / lo.
 * off / rows / cols are DEVICE arrays.  Gives the forward transform a
 * K-major (one TMA box per k-block) weight operand.                      */
int cg_split_tf32_t(int n_mats, const int64_t *off, const int32_t *rows, const int32_t *cols,
                    const float *x, float *hi, float *lo, int64_t max_elems, void *stream);
/* dW[k, n] = sum_m A[m, k] * D[m, n]; deterministic split over m.
 * db (optional): db[n] = sum_m D[m, n] (the bias gradient) -- under 3xTF32
 * fused into the same kernel (column sums while D is staged in smem).
 * ws must hold cg_wgrad_workspace(M, K, N) floats.                        */
int64_t cg_wgrad_workspace(int64_t M, int K, int N);
int cg_wgrad(int64_t M, int K, int N, const float *A, int64_t lda, const float *D,
             int64_t ldd, float *dW, float *db, float *ws, int mode, void *stream);
/* db[n] = sum_m D[m, n] (deterministic); ws as for cg_wgrad with K = 1.  */
int cg_colsum(int64_t M, int N, const float *D, int64_t ldd, float *db, float *ws,
              void *stream);
/* X = max(X, 0) in place (n_rows x F, F % 32 == 0) and, when bits is not
 * NULL, the result's > 0 pattern as bits (format as cg_spmm_mb's mask):
 * the ReLU of a layer whose pre-activation an aggregation produced (the
 * GraphSAGE layer-0 transform-first order).                 */
int cg_relu_bits(int64_t n_rows, int F, float *X, int64_t ldx, uint32_t *bits, int64_t ld_bits,
                 void *stream);

/* ---- K8: softmax cross-entropy ---------------------------------------- */
/* grad[r, c] = (softmax(logits[r]) - onehot(label[r])) * inv_n;
 * loss_out[0] = sum_r (lse_r - logits[r, label[r]]) (deterministic).
 * grad2 (optional): also grad[r, c] * scale2[r] (scale2 NULL = 1), the
 * row-scaled gradient the backward aggregation gathers, written in the same
 * pass (the ldg-wide row, padding included).
 * ws: >= n_rows + 1 floats, zeroed by the caller once.  ws[0] is the finish
 * ticket (fixed offset; each launch re-arms it), ws[1..] the block partials,
 * so one workspace may be reused across calls of any shape on one stream. */
int cg_softmax_ce(int64_t n_rows, int C, const float *logits, int64_t ld,
                  const int32_t *label, float inv_n, float *grad, int64_t ldg,
                  float *loss_out, float *ws, float *grad2, int64_t ldg2,
                  const float *scale2, void *stream);

/* ---- optimizer (replicated on every rank after the K7 all-reduce) ------ */
/* p_hi / p_lo (optional): also emit the TF32 split of the updated params
 * (as cg_split_tf32) for the pre-split 3xTF32 GEMM operands.              */
int cg_adam(int64_t n, float *param, const float *grad, float *m, float *v,
            float lr, float beta1, float beta2, float eps, int step, float *p_hi,
            float *p_lo, const float *corr_dev, void *stream);

/* ---- epoch graphs (CUDA graph replay of a steady-state epoch) ---------- *
 * Inside a captured epoch the per-epoch scalars are read from device memory:
 * cg_plan_frozen's epoch from `epoch_dev`, cg_adam's bias corrections
 * (1 - beta1^t, 1 - beta2^t) from `corr_dev[2]` (each NULL = use the
 * argument).  cg_set_epoch writes both ahead of a replay, computing the
 * corrections exactly as cg_adam does for `step` (corr_dev may be NULL).  */
int cg_set_epoch(int32_t *epoch_dev, int epoch, float *corr_dev, float beta1, float beta2,
                 int step, void *stream);
/* Record a cudaEvent_t on `stream`; while the stream is being captured the
 * record becomes an external event node that fires on every replay (so
 * per-kernel CUDA-event timing works inside an epoch graph).              */
int cg_event_record(void *event, void *stream);

/* ---- K6: frozen-membership JACA/FIFO plan for one epoch ---------------- *
 * One thread per halo-union vertex u; requesters of u (partition slots whose
 * halo holds u) in the reference's round-robin order (simulator.py:212-225).
 * Reproduces CacheSystem.lookup exactly while no admission/eviction can
 * happen; sets *flag != 0 if one would (the host then replays the epoch
 * with the sequential planner).  See DESIGN.md §4 for the table layout.  */
typedef struct cg_plan_static {
    int64_t n_union;
    const int64_t *req_off;     /* [n_union+1] requester CSR               */
    const int32_t *req_part;    /* partition slot of requester             */
    const int32_t *req_dev;     /* device (rank) holding that partition    */
    const int32_t *req_pos;     /* device-level halo position              */
    const int32_t *req_slot;    /* device-level slab row or -1             */
    const uint8_t *req_needed;  /* 1 if the SpMM reads this halo row       */
    const int32_t *owner_dev;   /* [n_union] owner device of u             */
    const int32_t *owner_row;   /* [n_union] row of u on its owner         */
    const int32_t *gslot;       /* [n_union] global-tier slot or -1        */
    const int32_t *lfree;       /* [n_parts] admit mode of the local level:
                                   0 never, 1 always, 2 iff score > lmin     */
    const double  *score;       /* [n_union] JACA importance               */
    const double  *lmin;        /* [n_parts] min resident score, local     */
    double gmin;                /* min resident score, global              */
    int32_t gfree;              /* admit mode of the global level          */
    int32_t policy;             /* 0 jaca, 1 fifo                          */
    int32_t n_parts;
    const int32_t *req_snap;    /* absolute epoch-1 snapshot row of the
                                   requester's vertex on its device, or -1:
                                   every read at version <= 1 is served
                                   from it; NULL = none      */
    int32_t coalesce;           /* 1: co-resident requesters of a vertex that
                                   need the same value this epoch (peer
                                   owner row / global-tier entry) share the
                                   row the first one stages (one wire row per
                                   device); 0: every requester stages       */
} cg_plan_static;

int cg_plan_frozen(const cg_plan_static *st, int epoch, int staleness, int me,
                   int32_t *req_ver, int32_t *glob_ver,
                   int32_t *halo_row, int32_t *stage_src, int32_t *stage_row,
                   int32_t *stage_dst, int32_t *gw_slot, int64_t *counts,
                   int32_t *flag, int32_t staging_base, int32_t n_devices,
                   int8_t *outcome, const int32_t *epoch_dev, void *stream);

/* ---- host-side sequential two-level planner (exact CacheSystem) -------- *
 * Replaces CacheSystem (cache.py:227-382) + simulator.run's lookup loop
 * (simulator.py:206-226).  Vertices are halo-union indices.              */
typedef struct cg_planner cg_planner;
int cg_planner_create(int policy, int n_parts, int64_t c_cpu, const int64_t *c_gpu,
                      int64_t n_union, const double *score, cg_planner **out);
int cg_planner_destroy(cg_planner *p);
/* halo_off[n_parts+1], halo[..]: per-partition halo as union indices in
 * ascending vertex id; ranked[..] the same lists in warm (importance) order. */
int cg_planner_set_halos(cg_planner *p, const int64_t *halo_off, const int32_t *halo,
                         const int32_t *ranked);
int cg_planner_warm(cg_planner *p);
/* One epoch of round-robin lookups.  Per requester (partition-major, halo
 * order): outcome (0 local, 1 global, 2 miss), served version, local slot
 * read on a local hit (else -1) and local slot held after the lookup (-1).
 * Per local slot (concatenated over partitions, offsets = prefix of c_gpu):
 * final occupant position (-1 empty) and a dirty flag (content changed this
 * epoch); per global slot: final union index (-1) and dirty flag.         */
int cg_planner_epoch(cg_planner *p, int epoch, int staleness, int8_t *outcome,
                     int32_t *version, int32_t *hit_slot, int32_t *slot_after,
                     int32_t *lslot_pos, uint8_t *lslot_dirty,
                     int32_t *gslot_vertex, uint8_t *gslot_dirty, int64_t *counts);
/* Current state: per requester local slot (-1) + version, per global slot
 * union index (-1) + version; whether any admission happened last epoch;
 * per-level "can admit" flags and min resident scores (for K6).          */
int cg_planner_state(cg_planner *p, int32_t *req_slot, int32_t *req_ver,
                     int32_t *gslot_of_union, int32_t *glob_ver_by_slot,
                     int32_t *admissions_last_epoch, int32_t *lfree, double *lmin,
                     int32_t *gfree, double *gmin);
/* Single lookup / admit, for the CacheSystem-compatible operator API.     */
int cg_planner_lookup(cg_planner *p, int part, int32_t vertex, int epoch, int staleness,
                      int *outcome);
int cg_planner_admit(cg_planner *p, int level, int part, int32_t vertex, int version,
                     int32_t *victim);
int cg_planner_counters(cg_planner *p, int64_t *lookups, int64_t *local_hits,
                        int64_t *global_hits, int64_t *misses);
int cg_planner_occupancy(cg_planner *p, int64_t *global_count, int64_t *local_counts);

/* ---- native integer preprocessing (graph.py:24-335, partitioner.py:324-345)
 * Bit-identical to halopart's numpy implementation; host functions.      */
int cg_csr_from_pairs(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                      int64_t *out_off, int64_t *out_tgt, int64_t *in_off, int64_t *in_tgt,
                      int64_t *n_edges);
int cg_undirected_csr(int64_t n, const int64_t *out_off, const int64_t *out_tgt,
                      const int64_t *in_off, const int64_t *in_tgt, int64_t *und_off,
                      int64_t *und_tgt);
int cg_khop_halo(int64_t n, const int64_t *und_off, const int64_t *und_tgt,
                 const int32_t *parts, int32_t part, int hops, int32_t *out, int64_t *n_out);
int cg_partition_stats(int64_t n, const int64_t *out_off, const int64_t *out_tgt,
                       const int32_t *parts, int P, const int64_t *halo_off,
                       const int32_t *halo, int64_t *cut, int64_t *all_edges);
int cg_influence_terms(int64_t n, const int64_t *out_off, const int64_t *out_tgt,
                       const int64_t *in_off, const int64_t *in_tgt, double *out_term,
                       double *in_term);

#ifdef __cplusplus
}
#endif
#endif /* CAPGNN_H */
