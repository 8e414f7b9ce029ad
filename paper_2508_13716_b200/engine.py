"""The per-device epoch executor: cache plan -> halo staging -> fused SpMM ->
transform, loss, backward halo-gradient exchange, K7 all-reduce, Adam.

Everything on the data path is a libcapgnn kernel launched on the current
torch stream; PyTorch only allocates device memory and provides streams,
events and torch.distributed.  See DESIGN.md §4-§6.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import PlanStatic, call, ptr
from .comm import HostTier, SoloComm
from .layout import RunLayout, source_row_csrs
from .planner import EpochPlan, SequentialPlanner

GEMM_MODES = {"fp32": 0, "3xtf32": 1, "tf32": 2}


def _dev(a, dtype, device):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(device)


@dataclass
class EpochStats:
    epoch: int
    loss: float
    counts: np.ndarray           # (P, 3) local, global, miss
    seconds: float
    spmm_fwd_ms: list
    spmm_bwd_ms: list
    planner: str                 # "host" or "gpu"
    flag: int = 0
    events: tuple | None = None  # (t0, t1) CUDA events when not yet synchronised
    k3: list | dict | None = None  # K3 launches: [(class, ev0, ev1)] -> {class: ms}


class Engine:
    def __init__(self, layout: RunLayout, me: int, kind: str, dims: list[int], bpe: int,
                 caps, planner: SequentialPlanner, staleness: int, policy: str,
                 comm=None, lr: float = 0.01, gemm: str = "3xtf32", params_init=None,
                 device: int | None = None, freeze_epoch: int | None = None,
                 record_outcomes: bool = False, plan_mode: str = "auto",
                 graphs: bool | None = None):
        self.L = layout
        self.me = me
        self.D = layout.devices[me]
        self.kind = kind
        # the class dimension is padded to a multiple of 4 (16-byte rows for
        # TMA); padded logit columns have zero weights and zero gradients
        self.C = int(dims[-1])
        self.C4 = (self.C + 3) // 4 * 4
        self.dims = list(dims[:-1]) + [self.C4]
        self.nL = len(dims) - 1
        self.bpe_f = bpe // 4
        self.comm = comm or SoloComm()
        self.planner = planner
        self.staleness = staleness
        self.policy = policy
        self.lr = lr
        self.gemm_mode = GEMM_MODES[gemm]
        # experiment knob (diagnostics only): weight-gradient GEMM mode override
        self.wgrad_mode = GEMM_MODES[os.environ.get("CG_WGRAD_MODE", gemm)]
        self.dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
        self.record_outcomes = record_outcomes
        self.plan_mode = plan_mode
        self.freeze_epoch = freeze_epoch if freeze_epoch is not None else max(1, staleness + 1)
        self.gpu_plan_ready = False
        self.step = 0
        # steady-state epochs (K6-planned, one process) replay CUDA graphs;
        # CG_GRAPHS=0 keeps every epoch eager
        if graphs is None:
            graphs = os.environ.get("CG_GRAPHS", "1") != "0"
        self.use_graphs = bool(graphs) and isinstance(self.comm, SoloComm)
        self._capturing = False
        self._graphs = None
        # K3 launch timing (bench exchange record): pre-made event pairs,
        # handed out in launch order each epoch; see k3_timing()
        self._k3_pool, self._k3_used = None, None
        self.wt_async = os.environ.get("CG_WT_ASYNC", "1") != "0"
        self._wt_early = True
        self._wt = None
        # R10 prefetch queue: staging rows that are final
        # before the epoch starts are copied ahead on a side stream
        self.prefetch = os.environ.get("CG_PREFETCH", "1") != "0"
        # request coalescing of staged rows (K6 / host tables); CG_COALESCE=0
        # stages every requester's row (the A/B reference)
        self.coalesce = os.environ.get("CG_COALESCE", "1") != "0"
        self._pf = None
        self._alloc(caps, params_init)
        if self._gw_active():
            # the write-through queue: side stream + fork/join events, made
            # (and materialised) before any graph capture
            cs = torch.cuda.current_stream(self.dev)
            self._wt = dict(stream=torch.cuda.Stream(self.dev), pending=[],
                            fork=[torch.cuda.Event() for _ in range(self.nL)],
                            done=[torch.cuda.Event() for _ in range(self.nL)])
            for ev in self._wt["fork"] + self._wt["done"]:
                ev.record(cs)
        if self.D.n_halo and not self.L.compact:
            cs = torch.cuda.current_stream(self.dev)
            self._pf = dict(stream=torch.cuda.Stream(self.dev), fork=torch.cuda.Event(),
                            done=[torch.cuda.Event() for _ in range(self.nL)])
            for ev in [self._pf["fork"]] + self._pf["done"]:
                ev.record(cs)

    def k3_timing(self, on: bool = True, pool: int = 64) -> None:
        """Time every K3 launch (halo staging, write-through, write-back,
        snapshot fill, backward gradient pulls) with CUDA events on the
        launching stream; EpochStats.k3 then maps each class to its ms."""
        if on and self._k3_pool is None:
            self._k3_pool = [(torch.cuda.Event(enable_timing=True),
                              torch.cuda.Event(enable_timing=True)) for _ in range(pool)]
            for a, b in self._k3_pool:   # materialise before any graph capture
                a.record()
                b.record()
        self._k3_on = bool(on)
        self._graphs = None   # re-capture with (or without) the event nodes

    # ------------------------------------------------------------------ setup
    def _alloc(self, caps, params_init):
        D, dev, f32, i32, i64 = self.D, self.dev, torch.float32, torch.int32, torch.int64
        dims = self.dims
        self.F = dims[:-1]
        self.X = [torch.zeros(D.n_rows, F, dtype=f32, device=dev) for F in self.F]
        self.logits = torch.zeros(D.n_in, self.C4, dtype=f32, device=dev)
        self.dL = torch.zeros(D.n_in, self.C4, dtype=f32, device=dev)  # logits gradient
        self.Z = [torch.zeros(D.n_in, F, dtype=f32, device=dev) for F in self.F]
        wmax = max(dims[1:])
        self.dY = [torch.zeros(D.n_in, wmax, dtype=f32, device=dev) for _ in range(2)]
        fmax_b = max(self.F[1:], default=4)
        n_bwd = D.bwd_stage_vertex.size
        # backward gradient rows [inner | staged remote rows], double-buffered
        # by layer parity when peers pull from it: a rank may overwrite its
        # layer-(l-1) rows while a slower peer still pulls its layer-l rows
        # (the next barrier orders the reuse two layers later)
        G0 = torch.zeros(D.n_in + n_bwd, fmax_b, dtype=f32, device=dev)
        self.Gs = [G0, torch.zeros_like(G0) if self.comm.world > 1 else G0]
        self.Hs = torch.zeros(D.n_in, fmax_b, dtype=f32, device=dev) if self.kind == "sage" else None
        # parameters (flat) + grads (+1 slot for the loss) + Adam state
        self.pshapes = []
        for l in range(self.nL):
            fi, fo = dims[l], dims[l + 1]
            if self.kind == "gcn":
                self.pshapes += [(fi, fo), (fo,)]
            else:
                self.pshapes += [(fi, fo), (fi, fo), (fo,)]
        # every tensor starts on a 16-byte boundary (TMA / tcgen05 operands)
        sizes = [int(np.prod(s)) for s in self.pshapes]
        padded = [(sz + 3) // 4 * 4 for sz in sizes]
        self.poff = np.concatenate(([0], np.cumsum(padded))).astype(np.int64)
        self.n_params = int(self.poff[-1])
        flat = np.zeros(self.n_params, np.float32)
        for i, p in enumerate(params_init):
            p = np.asarray(p, np.float32)
            if p.shape != tuple(self.pshapes[i]):   # last layer: pad class columns
                q = np.zeros(self.pshapes[i], np.float32)
                q[tuple(slice(0, k) for k in p.shape)] = p
                p = q
            flat[self.poff[i]:self.poff[i] + sizes[i]] = p.ravel()
        self.psizes = sizes
        self.params = _dev(flat, f32, dev)
        if self.gemm_mode == 1:
            # 3xTF32: weights kept pre-split for the GEMM B operand, plus a
            # transposed copy so the forward transform reads W K-major too
            self.params_hi = torch.empty_like(self.params)
            self.params_lo = torch.empty_like(self.params)
            self.paramsT_hi = torch.zeros_like(self.params)
            self.paramsT_lo = torch.zeros_like(self.params)
            mats = [i for i, sh in enumerate(self.pshapes) if len(sh) == 2]
            self._wt_tab = (_dev([int(self.poff[i]) for i in mats], torch.int64, dev),
                            _dev([self.pshapes[i][0] for i in mats], torch.int32, dev),
                            _dev([self.pshapes[i][1] for i in mats], torch.int32, dev),
                            len(mats), max(int(np.prod(self.pshapes[i])) for i in mats))
            call("cg_split_tf32", self.n_params, ptr(self.params), ptr(self.params_hi),
                 ptr(self.params_lo), self.stream())
            self._split_t()
        else:
            self.params_hi = self.params_lo = None
        self.grads = torch.zeros(self.n_params + 1, dtype=f32, device=dev)
        self.adam_m = torch.zeros(self.n_params, dtype=f32, device=dev)
        self.adam_v = torch.zeros(self.n_params, dtype=f32, device=dev)
        # per-epoch scalars read by kernels inside an epoch graph (cg_set_epoch)
        self.epoch_dev = torch.zeros(1, dtype=i32, device=dev)
        self.adam_corr = torch.zeros(2, dtype=f32, device=dev)
        ws = 1
        for l in range(self.nL):
            ws = max(ws, call("cg_wgrad_workspace", D.n_in, dims[l], dims[l + 1]),
                     (D.n_in + 255) // 256 * dims[l + 1])  # cg_colsum: 256-row chunks
        self.ws = torch.zeros(ws, dtype=f32, device=dev)
        self.ce_ws = torch.zeros(max(D.n_in, 1) + 1, dtype=f32, device=dev)   # + finish ticket
        # graph structure
        self.fwd_rowptr = _dev(D.fwd_rowptr, i64, dev)
        self.fwd_col = _dev(D.fwd_col, i32, dev)
        self.bwd_rowptr = _dev(D.bwd_rowptr, i64, dev)
        self.bwd_col = _dev(D.bwd_col, i32, dev)
        self.norm_src = _dev(D.norm_src, f32, dev)
        self.norm_dst = _dev(D.norm_dst, f32, dev)
        self.verts32 = _dev(D.verts, i32, dev)
        self.labels = torch.zeros(D.n_in, dtype=i32, device=dev)
        st = self.stream()
        call("cg_hash_labels", ptr(self.labels), ptr(self.verts32), D.n_in, self.C, 1, st)
        call("cg_hash_features", ptr(self.X[0]), self.F[0], ptr(self.verts32), D.n_in,
             self.F[0], 0, ptr(self.norm_src) if self.kind == "gcn" else None, st)
        # per-epoch plan tables (device-level halo positions)
        nh = max(D.n_halo, 1)
        self.halo_row = torch.full((nh,), -1, dtype=i32, device=dev)
        self.stage_src = torch.full((nh,), -1, dtype=i32, device=dev)
        self.stage_row = torch.zeros(nh, dtype=i32, device=dev)
        self.stage_dst = torch.full((nh,), -1, dtype=i32, device=dev)
        self.wb = None  # transient write-back lists (src_id, src_row, dst_row)
        nu = max(self.L.union.size if self.L.union is not None else 0, 1)
        self.gw_slot = torch.full((nu,), -1, dtype=i32, device=dev)
        if self.L.union is not None and self.L.union.size:
            own = self.L.owner_dev == self.me
            self.gw_src_id = _dev(np.where(own, self.me, -1), i32, dev)
            self.gw_src_row = _dev(self.L.owner_row, i32, dev)
        else:
            self.gw_src_id = torch.full((1,), -1, dtype=i32, device=dev)
            self.gw_src_row = torch.zeros(1, dtype=i32, device=dev)
        # Layer 0 reads the input features, which carry no version (SURVEY
        # A2: static): in the compact layout a halo position whose owner is
        # on this device reads the owner's row in place instead of its
        # epoch-1 snapshot copy -- the same values, half the distinct rows
        # the layer-0 gather touches (C2: 334K -> 169K rows, within L2)
        self.halo_row0 = None
        self.tf0 = False
        if (self.L.compact and D.n_halo and self.L.union is not None and self.L.union.size
                and os.environ.get("CG_L0_OWNER", "1") != "0"):
            k = np.searchsorted(self.L.union, D.halo_vertex)
            own = self.L.owner_dev[k] == self.me
            h0 = np.where(own, self.L.owner_row[k], D.snap_row_of_pos).astype(np.int32)
            self.halo_row0 = _dev(h0, i32, dev)
        # GraphSAGE layer 0, transform first when it narrows (F0 > F1, C3:
        # 604 -> 256): Y = relu(X W_self + b + mean_N(X W_neigh)) aggregates
        # F1-wide rows instead of F0-wide ones.  Exact when every layer-0
        # source row is an inner row of this device (one process, the
        # compact layout's owner-row halo map): the transformed rows are then
        # this device's own.  The weight gradient needs the transposed
        # aggregation of (1/d_in) dY over the out-edges (K2), instead of the
        # saved F0-wide aggregate.  CG_SAGE_TF0=0 keeps aggregate-first.
        self.tf0 = (self.kind == "sage" and self.nL >= 2 and self.F[0] > self.dims[1]
                    and self.halo_row0 is not None and self.comm.world == 1
                    and (not D.n_halo or bool((h0 < D.n_in).all()))
                    and os.environ.get("CG_SAGE_TF0", "1") != "0")
        if self.tf0:
            F1 = self.dims[1]
            self.tf0_h = torch.zeros(D.n_in, F1, dtype=f32, device=dev)   # X W_neigh
            self.tf0_p = torch.zeros(D.n_in, F1, dtype=f32, device=dev)   # X W_self + b
        self._alloc_tfl()
        # backward staging lists
        nb = max(n_bwd, 1)
        self.b_src = _dev(D.bwd_src_dev if n_bwd else [-1], i32, dev)
        self.b_row = _dev(D.bwd_src_row if n_bwd else [0], i32, dev)
        self.b_dst = _dev(D.n_in + np.arange(nb), i32, dev)
        self.n_bwd = n_bwd
        # epoch-1 snapshot fill lists (owner device, owner row) -> snap row
        if D.n_snap:
            self.snap_src = _dev(D.snap_src_dev, i32, dev)
            self.snap_srow = _dev(D.snap_src_row, i32, dev)
            self.snap_dst = _dev(D.snap_off + np.arange(D.n_snap), i32, dev)
        # host tier (global cache level): c_cpu slots x bpe
        self.c_cpu = int(caps.c_cpu)
        self.host = HostTier(self.c_cpu * self.bpe_f * 4, self.comm)
        self.layer_off = np.concatenate(([0], np.cumsum(self.F))).astype(np.int64)
        # pointer tables: [X_l on every device..., host tier + layer offset]
        nd = self.L.n_dev
        self.tab, self.tab_ld = [], []
        for l, F in enumerate(self.F):
            peers = self.comm.exchange_pointers(ptr(self.X[l]), self.dev.index)
            self.tab.append(_dev(np.array(peers + [self.host.ptr + 4 * int(self.layer_off[l])],
                                          np.uint64).view(np.int64), torch.int64, dev))
            self.tab_ld.append(_dev(np.array([F] * nd + [self.bpe_f], np.int64), i64, dev))
        self.tabGs = []
        for Gb in self.Gs:
            gpeers = self.comm.exchange_pointers(ptr(Gb), self.dev.index)
            self.tabGs.append(_dev(np.array(gpeers, np.uint64).view(np.int64), torch.int64, dev))
        self._tabG_lds = {}
        # aggregated narrow gradients (backward aggregate-then-transform layers)
        self.T = torch.zeros(D.n_in, max(self.dims[1:]), dtype=f32, device=dev)
        # ReLU masks as bits (layer l >= 1 inputs are ReLU outputs): written by
        # the forward GEMM's epilogue, read by the masked backward GEMM / SpMM
        # instead of the fp32 activation rows (1/32 of the bytes).  Needs the
        # tcgen05 GEMM and 32-column tiles; CG_MASK_BITS=0 keeps fp32 masks.
        self.bits = {}
        if self.gemm_mode in (1, 2) and os.environ.get("CG_MASK_BITS", "1") != "0":
            for l in range(1, self.nL):
                Fl = self.F[l]
                if Fl % 32 == 0 and (Fl <= 128 or Fl % 128 == 0):
                    self.bits[l] = torch.zeros(D.n_in, Fl // 32, dtype=torch.int32, device=dev)
        # frozen-plan (K6) state, created at hand-off
        self.k6 = None
        self._io = None
        self.loss_dev = torch.zeros(1, dtype=f32, device=dev)
        torch.cuda.current_stream(self.dev).synchronize()

    def _alloc_tfl(self) -> None:
        """The last layer transform first when it narrows (GCN: C2 256 -> 40,
        C4 256 -> 47; GraphSAGE: C3 256 -> 41, with X W_self + b as the
        aggregation's addend): logits = norm_dst * A (X W) + b aggregates C4-wide rows
        of H = X_ext W instead of F-wide rows of X_ext.  In the compact layout
        on one process the layer's sources are fixed -- inner rows and epoch-1
        snapshot rows -- so the backward has a static transposed CSR over
        those rows: dH = A^T (norm_dst dL) per source row gives dW = X_ext^T dH,
        and the input gradient's T = norm_src * (dH[u] + dH[snapshot of u])
        (the stale-row gradient flows to the owner, DESIGN.md §3 A3).
        CG_TFL=0 keeps aggregate-first."""
        D, L = self.D, self.L
        l = self.nL - 1
        # auto: worth it when the edges per transformed row are many -- the
        # aggregation saves 4 (F - C) bytes per edge, the extra GEMM / dW rows and
        # the transposed backward cost per row (C4, 13 edges per row: 49.4 ->
        # 43.1 ms; C2, 4 per row: 1.345 -> 1.354 ms).  CG_TFL=1 / 0 forces it.
        env = os.environ.get("CG_TFL", "")
        want = env == "1" or (env == "" and D.nnz_fwd >= 8 * max(D.n_rows, 1))
        self.tfl = (self.nL >= 2 and self.dims[self.nL] < self.F[l]
                    and L.compact and self.comm.world == 1 and D.n_in > 0 and want)
        if not self.tfl:
            return
        dev, i32, i64, f32 = self.dev, torch.int32, torch.int64, torch.float32
        n_in, C4 = D.n_in, self.dims[self.nL]
        csr = source_row_csrs(D, self.me)
        if csr is None:
            self.tfl = False      # a source without a snapshot row: not the compact plan
            return
        rp, col, urp, ucol = csr
        self.tfl_rp, self.tfl_col = _dev(rp, i64, dev), _dev(col, i32, dev)
        self.tfl_nnz = int(col.size)
        self.tfl_urp, self.tfl_ucol = _dev(urp, i64, dev), _dev(ucol, i32, dev)
        self.tfl_unnz = int(ucol.size)
        self.tfl_h = torch.zeros(D.n_rows, C4, dtype=f32, device=dev)    # X_ext W (W_neigh)
        self.tfl_dh = torch.zeros(D.n_rows, C4, dtype=f32, device=dev)   # A^T (norm_dst dL)
        # GraphSAGE: the self term X W_self + b is the aggregation's addend
        self.tfl_p = (torch.zeros(D.n_in, C4, dtype=f32, device=dev) if self.kind == "sage"
                      else None)
        need = max(call("cg_wgrad_workspace", D.n_rows, self.F[l], C4),
                   (max(D.n_in, D.n_rows) + 255) // 256 * C4)
        if need > self.ws.numel():
            self.ws = torch.zeros(need, dtype=f32, device=dev)

    def _tabG_ld(self, F: int):
        t = self._tabG_lds.get(F)
        if t is None:
            t = _dev(np.full(self.L.n_dev, F, np.int64), torch.int64, self.dev)
            self._tabG_lds[F] = t
        return t

    def stream(self) -> int:
        return torch.cuda.current_stream(self.dev).cuda_stream

    def param_views(self) -> list[np.ndarray]:
        flat = self.params.detach().cpu().numpy()
        out = [flat[self.poff[i]:self.poff[i] + self.psizes[i]].reshape(s)
               for i, s in enumerate(self.pshapes)]
        per = 2 if self.kind == "gcn" else 3
        for i in range(len(out) - per, len(out)):  # strip the class padding
            out[i] = out[i][..., :self.C].copy()
        return out

    def _p(self, i: int) -> int:
        return ptr(self.params) + 4 * int(self.poff[i])

    def _split_t(self):
        off, rows, cols, n, mx = self._wt_tab
        call("cg_split_tf32_t", n, ptr(off), ptr(rows), ptr(cols), ptr(self.params),
             ptr(self.paramsT_hi), ptr(self.paramsT_lo), mx, self.stream())

    def _gemm(self, M, N, K1, A1, lda1, w1, K2=0, A2=None, lda2=0, w2=None, *, trans_b,
              bias=None, relu=0, row_scale=None, mask=None, ldm=0, C, ldc, mask_l=None,
              bits_l=None):
        """cg_gemm with weight operands given as parameter indices: under
        3xTF32 the weights are read pre-split (params_hi / params_lo, kept
        current by cg_adam), so the kernel splits only the activations."""
        split = self.params_hi is not None
        mode = self.gemm_mode
        def b(i, arr):
            return None if i is None else ptr(arr) + 4 * int(self.poff[i])
        if split and trans_b == 0:   # W [K x N] -> its transpose, K-major
            B1, B2 = b(w1, self.paramsT_hi), b(w2, self.paramsT_hi)
            L1, L2 = b(w1, self.paramsT_lo), b(w2, self.paramsT_lo)
            trans_b = 1
        elif split:
            B1, B2 = b(w1, self.params_hi), b(w2, self.params_hi)
            L1, L2 = b(w1, self.params_lo), b(w2, self.params_lo)
        else:
            B1, B2, L1, L2 = b(w1, self.params), b(w2, self.params), None, None
        mb = self.bits.get(mask_l) if mask_l is not None else None
        bo = self.bits.get(bits_l) if bits_l is not None else None
        if mb is not None or bo is not None:
            # ReLU masks as bits: layer mask_l's pattern in, layer bits_l's out
            call("cg_gemm_mb", M, N, K1, A1, lda1, B1, K2, A2, lda2, B2, trans_b, bias, relu,
                 row_scale, None if mb is None else ptr(mb),
                 0 if mb is None else mb.shape[1], None if bo is None else ptr(bo),
                 0 if bo is None else bo.shape[1], C, ldc, mode, L1, L2, self.stream())
            return
        if mask_l is not None:
            mask, ldm = ptr(self.X[mask_l]), self.F[mask_l]
        call("cg_gemm", M, N, K1, A1, lda1, B1, K2, A2, lda2, B2, trans_b, bias, relu,
             row_scale, mask, ldm, C, ldc, mode, L1, L2, self.stream())

    def _spmm(self, n_rows, F, rowptr, col, n_direct, halo_row, X, ldx, scale, addend, ld_add,
              mask, ld_mask, out, ldo, mask_l=None, nnz=None):
        """One cg_spmm call over tensors (the kernel choice and any column
        slicing happen behind the C ABI).  mask_l: the ReLU mask is layer
        mask_l's input (its bits when kept, else the fp32 rows)."""
        p = lambda t: None if t is None else (t if isinstance(t, int) else ptr(t))  # noqa: E731
        if nnz is None:
            nnz = self.D.nnz_fwd if rowptr is self.fwd_rowptr else self.D.nnz_bwd
        if mask_l is not None:
            mb = self.bits.get(mask_l)
            if mb is not None:
                call("cg_spmm_mb", n_rows, F, ptr(rowptr), ptr(col), n_direct, p(halo_row),
                     ptr(X), ldx, p(scale), p(addend), ld_add, ptr(mb), mb.shape[1], ptr(out),
                     ldo, int(nnz), self.stream())
                return
            mask, ld_mask = self.X[mask_l], self.F[mask_l]
        call("cg_spmm", n_rows, F, ptr(rowptr), ptr(col), n_direct, p(halo_row), ptr(X), ldx,
             p(scale), p(addend), ld_add, p(mask), ld_mask, ptr(out), ldo, int(nnz),
             self.stream())

    # NVTX phase ranges for nsys / ncu --nvtx (CG_NVTX=1); one range open at a time
    _NVTX = os.environ.get("CG_NVTX") == "1"

    def _mark(self, phase):
        if not self._NVTX:
            return
        if getattr(self, "_nvtx_open", False):
            torch.cuda.nvtx.range_pop()
            self._nvtx_open = False
        if phase is not None:
            torch.cuda.nvtx.range_push(f"capgnn:{phase}")
            self._nvtx_open = True

    def _g(self, i: int) -> int:
        return ptr(self.grads) + 4 * int(self.poff[i])

    # ------------------------------------------------------------------ plans
    def _host_tables(self, e: int, plan: EpochPlan, gslot_start: np.ndarray):
        """Device tables for an epoch planned on the host (any policy)."""
        L, D, me = self.L, self.D, self.me
        nd = L.n_dev
        n_in, nh = D.n_in, D.n_halo
        halo_row = np.full(max(nh, 1), -1, np.int32)
        s_src = np.full(max(nh, 1), -1, np.int32)
        s_row = np.zeros(max(nh, 1), np.int32)
        s_dst = np.full(max(nh, 1), -1, np.int32)
        wb_src, wb_dst = [], []
        if L.union is not None and L.union.size:
            hoff = L.halo_off
            # request coalescing (as K6): per union vertex, the first staging
            # row this epoch that receives the owner's current row from a
            # peer / the global tier's entry (one version per epoch); later
            # co-resident requesters read that row instead of staging again
            first_cur = np.full(L.union.size, -1, np.int64)
            first_glob = np.full(L.union.size, -1, np.int64)
            for p in D.parts:
                b, eidx = hoff[p], hoff[p + 1]
                if eidx == b:
                    continue
                hp = D.hpos_off[p]
                k = np.searchsorted(L.union, D.halo_vertex[hp:hp + (eidx - b)])
                oc = plan.outcome[b:eidx]
                ver = plan.version[b:eidx]
                cur = np.maximum(ver, 1) == e
                need = D.needed[hp:hp + (eidx - b)]
                odev = L.owner_dev[k]
                orow = L.owner_row[k]
                pos = hp + np.arange(eidx - b)
                # version <= 1 -> the epoch-1 value: the shared snapshot row
                ver1 = (np.maximum(ver, 1) == 1) & need
                halo_row[pos[ver1]] = D.snap_row_of_pos[pos[ver1]]
                # stale local hit -> read the slab slot in place
                st_loc = (oc == 0) & ~cur & need & ~ver1
                halo_row[pos[st_loc]] = D.slab_off[p] + plan.hit_slot[b:eidx][st_loc]
                # co-resident owner, current value -> read the owner row in place
                direct = cur & need & (odev == me) & ~ver1
                halo_row[pos[direct]] = orow[direct]
                # everything else is staged into its staging row
                stg = need & ~st_loc & ~direct & ~ver1
                if L.compact and (st_loc.any() or stg.any()):
                    raise RuntimeError(f"epoch {e}: the compact layout's precondition (no "
                                       "staged or slab reads) was violated")
                halo_row[pos[stg]] = n_in + pos[stg]
                s_dst[pos[stg]] = n_in + pos[stg]
                from_owner = stg & cur
                s_src[pos[from_owner]] = odev[from_owner]
                s_row[pos[from_owner]] = orow[from_owner]
                from_host = stg & ~cur
                gsl = gslot_start[k[from_host]]
                if (gsl < 0).any():
                    raise RuntimeError("stale global hit without a global slot")
                s_src[pos[from_host]] = nd
                s_row[pos[from_host]] = gsl
                for kind_m, first in (((from_owner, first_cur), (from_host, first_glob))
                                      if self.coalesce else ()):
                    j = np.flatnonzero(kind_m)
                    have = first[k[j]]
                    dup = have >= 0
                    halo_row[pos[j[dup]]] = have[dup]
                    s_dst[pos[j[dup]]] = -1
                    s_src[pos[j[dup]]] = -1
                    first[k[j[~dup]]] = n_in + pos[j[~dup]]
                # write-back of the final local-slot contents (after the SpMM);
                # slots at version <= 1 are never read (the snapshot serves them)
                lo, c = int(self.planner.lslot_off[p]), int(self.planner.c_gpu[p])
                lpos = plan.lslot_pos[lo:lo + c]
                dirty = plan.lslot_dirty[lo:lo + c].astype(bool)
                sl = np.flatnonzero(dirty & (lpos >= 0))
                if sl.size:
                    j = lpos[sl]
                    keep = need[j] & (np.maximum(ver[j], 1) > 1)
                    sl, j = sl[keep], j[keep]
                    wb_dst.append(D.slab_off[p] + sl)
                    wb_src.append(halo_row[hp + j])
            # owner-side host-tier writes for this epoch's final global contents
        gw = np.full(max(L.union.size if L.union is not None else 0, 1), -1, np.int32)
        if self.c_cpu and L.union is not None and L.union.size:
            gv = plan.gslot_vertex
            # global entries at version <= 1 are served by the snapshot: the
            # host tier only needs contents written at epoch >= 2
            dirty = plan.gslot_dirty.astype(bool) & (e > 1)
            sl = np.flatnonzero(dirty & (gv >= 0))
            kk = gv[sl]
            mine = L.owner_dev[kk] == me
            gw[kk[mine]] = sl[mine]
        dev = self.dev
        self.halo_row.copy_(torch.from_numpy(halo_row))
        self.stage_src.copy_(torch.from_numpy(s_src))
        self.stage_row.copy_(torch.from_numpy(s_row))
        self.stage_dst.copy_(torch.from_numpy(s_dst))
        self.gw_slot.copy_(torch.from_numpy(gw))
        if wb_dst:
            d = np.concatenate(wb_dst).astype(np.int32)
            s = np.concatenate(wb_src).astype(np.int32)
            self.wb = (_dev(np.full(d.size, me, np.int32), torch.int32, dev),
                       _dev(s, torch.int32, dev), _dev(d, torch.int32, dev), int(d.size))
        else:
            self.wb = None

    def _init_gpu_plan(self):
        """Hand the frozen membership + versions to K6."""
        L, pl = self.L, self.planner
        stt = pl.state()
        dev, i32 = self.dev, torch.int32
        # requester tables in K6 order (halo-union major, lookup order)
        idx = L.req_index
        slot = stt["req_slot"][idx]
        part = L.req_part
        slab_base = np.zeros(L.P, np.int64)
        for dl in L.devices:
            for p in dl.parts:
                slab_base[p] = dl.slab_off[p]
        req_slot = np.where(slot >= 0, slab_base[part] + slot, -1).astype(np.int32)
        gslot = stt["gslot"].astype(np.int32)
        self.k6 = dict(
            req_off=_dev(L.req_off, torch.int64, dev), req_part=_dev(part, i32, dev),
            req_dev=_dev(L.req_dev, i32, dev), req_pos=_dev(L.req_pos, i32, dev),
            req_slot=_dev(req_slot, i32, dev),
            req_needed=_dev(L.req_needed, torch.uint8, dev),
            owner_dev=_dev(L.owner_dev, i32, dev), owner_row=_dev(L.owner_row, i32, dev),
            gslot=_dev(gslot, i32, dev), lfree=_dev(stt["lfree"], i32, dev),
            score=_dev(pl._score, torch.float64, dev), lmin=_dev(stt["lmin"], torch.float64, dev),
            req_ver=_dev(stt["req_ver"][idx], i32, dev),
            glob_ver=_dev(stt["glob_ver"] if stt["glob_ver"].size else [0], i32, dev),
            counts=torch.zeros(L.P * 3, dtype=torch.int64, device=dev),
            flag=torch.zeros(1, dtype=i32, device=dev),
            outcome=torch.zeros(max(idx.size, 1), dtype=torch.int8, device=dev))
        k = self.k6
        mine = L.req_dev == self.me
        req_snap = np.full(idx.size, -1, np.int32)
        req_snap[mine] = self.D.snap_row_of_pos[L.req_pos[mine]]
        k["req_snap"] = _dev(req_snap if req_snap.size else [-1], i32, dev)
        self.k6_static = PlanStatic(
            n_union=int(L.union.size), req_off=ptr(k["req_off"]), req_part=ptr(k["req_part"]),
            req_dev=ptr(k["req_dev"]), req_pos=ptr(k["req_pos"]), req_slot=ptr(k["req_slot"]),
            req_needed=ptr(k["req_needed"]), owner_dev=ptr(k["owner_dev"]),
            owner_row=ptr(k["owner_row"]), gslot=ptr(k["gslot"]), lfree=ptr(k["lfree"]),
            score=ptr(k["score"]), lmin=ptr(k["lmin"]), gmin=float(stt["gmin"]),
            gfree=int(stt["gfree"]), policy=0 if self.policy == "jaca" else 1, n_parts=L.P,
            req_snap=ptr(k["req_snap"]), coalesce=int(self.coalesce))
        self.gpu_plan_ready = True

    def plan(self, e: int) -> tuple[str, np.ndarray | None, EpochPlan | None]:
        """Fill this epoch's tables.  Returns (mode, host counts, host plan)."""
        use_gpu = (self.plan_mode != "host" and self.policy in ("jaca", "fifo")
                   and e > self.freeze_epoch and self.L.union is not None
                   and self.L.union.size > 0)
        if use_gpu and not self.gpu_plan_ready:
            if self.planner.state()["admissions"] != 0:
                use_gpu = False   # membership still moving: stay on the host
            else:
                self._init_gpu_plan()
        # Early write-through forks (see _gw) are safe when no global slot can
        # change hands mid-epoch under a peer's staging read: one process
        # (the fork follows this process's own staging copy), or a
        # K6-planned epoch (frozen membership: an entry is only rewritten
        # when it was stale for every requester of the epoch).  Otherwise
        # the copies wait for the next layer's barrier, as the readers do.
        self._wt_early = use_gpu or self.comm.world == 1
        if use_gpu:
            k = self.k6
            k["counts"].zero_()
            call("cg_plan_frozen", C.addressof(self.k6_static), e, self.staleness, self.me,
                 ptr(k["req_ver"]), ptr(k["glob_ver"]), ptr(self.halo_row), ptr(self.stage_src),
                 ptr(self.stage_row), ptr(self.stage_dst), ptr(self.gw_slot), ptr(k["counts"]),
                 ptr(k["flag"]), -1 if self.L.compact else self.D.n_in, self.L.n_dev,
                 ptr(k["outcome"]) if self.record_outcomes else None,
                 ptr(self.epoch_dev) if self._capturing else None, self.stream())
            self.wb = None
            return "gpu", None, None
        if self.gpu_plan_ready:
            raise RuntimeError("host re-planning after the GPU hand-off is not supported")
        gstart = (self.planner.state()["gslot"] if self.L.union is not None and self.L.union.size
                  else np.zeros(0, np.int32))
        plan = self.planner.epoch(e, self.staleness)
        self._host_tables(e, plan, gstart)
        return "host", plan.counts.copy(), plan

    # ------------------------------------------------------------------ epoch
    _k3_on = False

    def _copy(self, n, F, src_id, src_row, dst_row, tab, tab_ld, dst, ld, cls="stage",
              stream=None, max_blocks: int = 0, ids=None):
        st = stream.cuda_stream if stream is not None else self.stream()
        ev = None
        if self._k3_on and self._k3_used is not None and len(self._k3_used) < len(self._k3_pool):
            ev = self._k3_pool[len(self._k3_used)]
            self._k3_used.append((cls, F, ev))
            self._rec(ev[0], stream)
        if ids is None:
            call("cg_copy_rows_bounded", n, F, ptr(src_id), ptr(src_row), ptr(dst_row),
                 ptr(tab), ptr(tab_ld), dst if isinstance(dst, int) else ptr(dst), ld,
                 max_blocks, st)
        else:
            call("cg_copy_rows_sel", n, F, ptr(src_id), ptr(src_row), ptr(dst_row), ptr(tab),
                 ptr(tab_ld), dst if isinstance(dst, int) else ptr(dst), ld, ids[0], ids[1],
                 max_blocks, st)
        if ev is not None:
            self._rec(ev[1], stream)

    # Host-tier write-through queue (R10; PAPER.md:98's "global" queue).  The
    # epoch's dirty global entries are copied into the pinned host tier over
    # PCIe (~51 GB/s) by K3 on a side stream with a small grid, forked once a
    # layer's input rows are final and its staging copy (the only same-epoch
    # reader of the host tier) is enqueued (layer L-1: when the backward
    # starts), and all joined at the end of the update -- steady-state epochs
    # are then captured as ONE graph -- so the PCIe writes run under the
    # SpMM / GEMM work of the whole epoch instead of in front of it.  The
    # host tier is only read by stale global hits, i.e. in LATER epochs
    # (current-version reads go to the owner's row), and the next epoch's K6
    # rewrites gw_slot only after the joins -- so the joins are the only
    # ordering needed.  CG_WT_ASYNC=0 (or wt_async = False) runs the
    # copies in line on the compute stream instead.
    WT_BLOCKS = int(os.environ.get("CG_WT_BLOCKS", "16"))

    def _gw_active(self) -> bool:
        # compact layout: every read is a version-0 local hit (enforced by the
        # host tables / K6 flag), so no global entry is ever rewritten
        return not (self.c_cpu == 0 or self.L.union is None or self.L.union.size == 0
                    or self.L.compact)

    def _gw(self, l: int):
        if not self._gw_active():
            return
        F = self.F[l]
        args = (self.L.union.size, F, self.gw_src_id, self.gw_src_row, self.gw_slot,
                self.tab[l], self.tab_ld[l], self.host.ptr + 4 * int(self.layer_off[l]),
                self.bpe_f)
        if not self.wt_async:
            self._copy(*args, cls="write_through")
            return
        wt = self._wt
        cs = torch.cuda.current_stream(self.dev)
        wt["fork"][l].record(cs)
        wt["stream"].wait_event(wt["fork"][l])
        self._copy(*args, cls="write_through", stream=wt["stream"], max_blocks=self.WT_BLOCKS)
        wt["done"][l].record(wt["stream"])
        wt["pending"].append(wt["done"][l])

    def _join_gw(self) -> None:
        if self._wt is None or not self._wt["pending"]:
            return
        cs = torch.cuda.current_stream(self.dev)
        for ev in self._wt["pending"]:
            cs.wait_event(ev)
        self._wt["pending"] = []

    def _rec(self, ev, stream=None) -> None:
        """Record a timing event on the current (or the given) stream; inside
        a capture it becomes an external event node that fires on every
        replay."""
        if self._capturing:
            call("cg_event_record", ev.cuda_event,
                 stream.cuda_stream if stream is not None else self.stream())
        elif stream is not None:
            ev.record(stream)
        else:
            ev.record()

    # R10 prefetch queue (prefetch_depth simulator.py:44,237-239).
    # Of a layer's staging rows, two kinds are final before the epoch's
    # forward pass starts: rows read from the pinned host tier (stale global
    # hits: written through in an EARLIER epoch, and that write-through was
    # joined before this epoch's plan) and, at layer 0, every row (the input
    # features are static; re-uploaded inputs land before the fork).  They
    # are copied on a side stream right after the plan -- the layer-1/2 host
    # reads (PCIe, ~51 GB/s) then run under layer 0's SpMM / GEMM -- and the
    # compute stream waits on layer l's copy only before layer l's SpMM.
    # Only current-epoch owner rows (ids < n_dev) stay in line behind the
    # layer's barrier.  Safe when no global slot can change hands mid-epoch
    # under a peer's write-through (_wt_early: one process, or a K6-planned
    # epoch); otherwise every copy stays in line.  CG_PREFETCH=0 disables it.
    PF_BLOCKS = int(os.environ.get("CG_PF_BLOCKS", "32"))

    def _prefetch_rows(self) -> bool:
        pf = self._pf
        if pf is None or not self.prefetch or not self._wt_early:
            return False
        cs = torch.cuda.current_stream(self.dev)
        pf["fork"].record(cs)
        pf["stream"].wait_event(pf["fork"])
        nd = self.L.n_dev
        for l, F in enumerate(self.F):
            ids = (0, nd + 1) if l == 0 else (nd, nd + 1)
            self._copy(self.D.n_halo, F, self.stage_src, self.stage_row, self.stage_dst,
                       self.tab[l], self.tab_ld[l], self.X[l], F, cls="prefetch",
                       stream=pf["stream"], max_blocks=0 if l == 0 else self.PF_BLOCKS,
                       ids=ids)
            pf["done"][l].record(pf["stream"])
        return True

    def _forward(self, e: int, spmm_ev) -> None:
        D, nL, kind, n_in = self.D, self.nL, self.kind, self.D.n_in
        pf = self._prefetch_rows()
        for l in range(nL):
            F, Fo = self.F[l], self.dims[l + 1]
            if l > 0:
                self.comm.barrier()
                if not self._wt_early:
                    self._gw(l - 1)
            if e == 1 and D.n_snap:
                # epoch-1 snapshot of every halo vertex read on this device
                self._copy(D.n_snap, F, self.snap_src, self.snap_srow, self.snap_dst,
                           self.tab[l], self.tab_ld[l], self.X[l], F, cls="snapshot")
            if D.n_halo and not self.L.compact:   # compact: nothing is ever staged
                if pf:
                    torch.cuda.current_stream(self.dev).wait_event(self._pf["done"][l])
                    if l > 0:   # current-epoch owner rows, behind the barrier
                        self._copy(D.n_halo, F, self.stage_src, self.stage_row,
                                   self.stage_dst, self.tab[l], self.tab_ld[l], self.X[l], F,
                                   ids=(0, self.L.n_dev))
                else:
                    self._copy(D.n_halo, F, self.stage_src, self.stage_row, self.stage_dst,
                               self.tab[l], self.tab_ld[l], self.X[l], F)
            if l < nL - 1 and self._wt_early:
                # this layer's input rows are final and its stale global hits
                # have been staged (a host-plan epoch may reassign a slot read
                # above): write the dirty global entries through
                self._gw(l)
            if l == 0 and self.tf0:
                self._forward_tf0(spmm_ev)
                continue
            if l == nL - 1 and self.tfl:
                self._forward_tfl(spmm_ev)
                continue
            if spmm_ev is not None:
                self._rec(spmm_ev[l][0])
            hrow = self.halo_row0 if (l == 0 and self.halo_row0 is not None) else self.halo_row
            self._spmm(n_in, F, self.fwd_rowptr, self.fwd_col, n_in, hrow, self.X[l],
                       F, self.norm_dst, None, 0, None, 0, self.Z[l], F)
            if spmm_ev is not None:
                self._rec(spmm_ev[l][1])
            if self.wb is not None:
                sid, srow, dst, n = self.wb
                self._copy(n, F, sid, srow, dst, self.tab[l], self.tab_ld[l], self.X[l], F,
                           cls="write_back")
            last = l == nL - 1
            out = self.logits if last else self.X[l + 1]
            if last and not self._capturing:
                self._wait_logits_download()
            bl = None if last else l + 1   # this ReLU output's bits (backward masks)
            if kind == "gcn":
                self._gemm(n_in, Fo, F, ptr(self.Z[l]), F, 2 * l, trans_b=0,
                           bias=self._p(2 * l + 1), relu=0 if last else 1,
                           row_scale=None if last else ptr(self.norm_src), C=ptr(out), ldc=Fo,
                           bits_l=bl)
            else:
                self._gemm(n_in, Fo, F, ptr(self.X[l]), F, 3 * l, F, ptr(self.Z[l]), F,
                           3 * l + 1, trans_b=0, bias=self._p(3 * l + 2),
                           relu=0 if last else 1, C=ptr(out), ldc=Fo, bits_l=bl)

    def _forward_tf0(self, spmm_ev) -> None:
        """GraphSAGE layer 0, transform first (see _alloc): two GEMMs, one
        F1-wide aggregation with the self term as its addend, then ReLU (and
        the backward mask bits) in place."""
        n_in, F, Fo = self.D.n_in, self.F[0], self.dims[1]
        self._gemm(n_in, Fo, F, ptr(self.X[0]), F, 0, trans_b=0, bias=self._p(2), C=ptr(self.tf0_p),
                   ldc=Fo)
        self._gemm(n_in, Fo, F, ptr(self.X[0]), F, 1, trans_b=0, C=ptr(self.tf0_h), ldc=Fo)
        if spmm_ev is not None:
            self._rec(spmm_ev[0][0])
        self._spmm(n_in, Fo, self.fwd_rowptr, self.fwd_col, n_in, self.halo_row0, self.tf0_h, Fo,
                   self.norm_dst, self.tf0_p, Fo, None, 0, self.X[1], Fo)
        if spmm_ev is not None:
            self._rec(spmm_ev[0][1])
        b = self.bits.get(1)
        call("cg_relu_bits", n_in, Fo, ptr(self.X[1]), Fo, None if b is None else ptr(b),
             0 if b is None else b.shape[1], self.stream())

    def _forward_tfl(self, spmm_ev) -> None:
        """GCN's last layer, transform first (see _alloc_tfl): H = X_ext W over
        every row the aggregation reads, then logits = norm_dst * A H + b (the
        bias as a broadcast addend row)."""
        l, D = self.nL - 1, self.D
        F, Fo = self.F[l], self.dims[self.nL]
        sage = self.kind == "sage"
        w_n = 3 * l + 1 if sage else 2 * l
        self._gemm(D.n_rows, Fo, F, ptr(self.X[l]), F, w_n, trans_b=0, C=ptr(self.tfl_h),
                   ldc=Fo)
        if sage:   # GraphSAGE: P = X W_self + b over the inner rows
            self._gemm(D.n_in, Fo, F, ptr(self.X[l]), F, 3 * l, trans_b=0, bias=self._p(3 * l + 2),
                       C=ptr(self.tfl_p), ldc=Fo)
        if not self._capturing:
            self._wait_logits_download()
        if spmm_ev is not None:
            self._rec(spmm_ev[l][0])
        add, ld_add = (self.tfl_p, Fo) if sage else (self._p(2 * l + 1), 0)
        self._spmm(D.n_in, Fo, self.fwd_rowptr, self.fwd_col, D.n_in, self.halo_row, self.tfl_h,
                   Fo, self.norm_dst, add, ld_add, None, 0, self.logits, self.C4)
        if spmm_ev is not None:
            self._rec(spmm_ev[l][1])

    def _backward_tfl(self, spmm_ev, nxt) -> None:
        """The last layer's backward under _forward_tfl: dH over the source
        rows (static transposed CSR, G = norm_dst dL from the loss), dW =
        X_ext^T dH, db = column sums of dL, T = norm_src * (dH[u] + dH[snap u]),
        then the masked input gradient mask * (T W^T)."""
        l, D, st = self.nL - 1, self.D, self.stream()
        F, Fo = self.F[l], self.dims[self.nL]
        sage = self.kind == "sage"
        G = self.Gs[l & 1]
        if spmm_ev is not None:
            self._rec(spmm_ev[0][0])
        self._spmm(D.n_rows, Fo, self.tfl_rp, self.tfl_col, 1 << 62, None, G, Fo, None, None, 0,
                   None, 0, self.tfl_dh, Fo, nnz=self.tfl_nnz)
        self._spmm(D.n_in, Fo, self.tfl_urp, self.tfl_ucol, 1 << 62, None, self.tfl_dh, Fo,
                   None if sage else self.norm_src, None, 0, None, 0, self.T, Fo,
                   nnz=self.tfl_unnz)
        if spmm_ev is not None:
            self._rec(spmm_ev[0][1])
        if sage:
            # dW_neigh = X_ext^T dH; dW_self (+ db) = X^T dL; the input gradient
            # mask * (dL W_self^T + T W_neigh^T)
            call("cg_wgrad", D.n_rows, F, Fo, ptr(self.X[l]), F, ptr(self.tfl_dh), Fo,
                 self._g(3 * l + 1), None, ptr(self.ws), self.wgrad_mode, st)
            call("cg_wgrad", D.n_in, F, Fo, ptr(self.X[l]), F, ptr(self.dL), self.C4,
                 self._g(3 * l), self._g(3 * l + 2), ptr(self.ws), self.wgrad_mode, st)
            self._gemm(D.n_in, F, Fo, ptr(self.dL), self.C4, 3 * l, Fo, ptr(self.T), Fo, 3 * l + 1,
                       trans_b=1, mask_l=l, C=ptr(nxt), ldc=F)
            return
        call("cg_wgrad", D.n_rows, F, Fo, ptr(self.X[l]), F, ptr(self.tfl_dh), Fo,
             self._g(2 * l), None, ptr(self.ws), self.wgrad_mode, st)
        call("cg_colsum", D.n_in, Fo, ptr(self.dL), self.C4, self._g(2 * l + 1), ptr(self.ws), st)
        self._gemm(D.n_in, F, Fo, ptr(self.T), Fo, 2 * l, trans_b=1, mask_l=l, C=ptr(nxt), ldc=F)

    def _n_bwd_spmm(self) -> int:
        return self.nL - 1 + (1 if self.tf0 else 0)

    def spmm_launch_bytes(self):
        """Algorithmic bytes (DESIGN.md §5 formula) of each timed aggregation
        window in timer order: (forward per layer, backward windows)."""
        D = self.D

        def b(nnz, rows, F, halo=0):
            return nnz * (4 + 4 * F) + rows * (8 + 4 + 4 * F) + 8 + halo * 4
        fw, bw = self.spmm_widths()
        fb = [b(D.nnz_fwd, D.n_in, F, D.n_halo) for F in fw]
        bb = [b(D.nnz_bwd, D.n_in, F) for F in bw]
        if self.tfl:   # the last layer's window: transposed CSR over X_ext rows + the owner sum
            bb[0] = (b(self.tfl_nnz, D.n_rows, bw[0]) + b(self.tfl_unnz, D.n_in, bw[0]))
        return fb, bb

    def spmm_widths(self):
        """Row widths of the epoch's aggregations in launch order: (forward
        per layer, backward layers nL-1 .. 1 [, layer 0 under tf0])."""
        w = list(self.F) + [self.C4]
        fwd = [self.dims[1] if (l == 0 and self.tf0) else self.F[l] for l in range(self.nL)]
        if self.tfl:
            fwd[-1] = self.dims[self.nL]
        bwd = [min(w[l], w[l + 1]) for l in range(self.nL - 1, 0, -1)]
        if self.tf0:
            bwd.append(self.dims[1])
        return fwd, bwd

    def _wait_logits_download(self) -> None:
        # the previous epoch's logits download must finish before they change
        if self._io is not None and self._io["logits_done"] is not None:
            torch.cuda.current_stream(self.dev).wait_event(self._io["logits_done"])
            self._io["logits_done"] = None

    def _last_wide(self) -> bool:
        """The last layer's backward aggregates the (narrow) logits gradient."""
        return self.dims[self.nL] < self.F[self.nL - 1]

    def _loss(self) -> None:
        loss_ptr = ptr(self.grads) + 4 * self.n_params
        # the wide last layer's gathered rows G = norm_dst * dL come out of the
        # same pass (no separate scaling launch)
        l = self.nL - 1
        # (nL == 1: the only backward layer is l = 0, which never reads G --
        # and G is sized for the hidden widths, not the class width)
        g2 = ptr(self.Gs[l & 1]) if self._last_wide() and self.nL > 1 else None
        sc = ptr(self.norm_dst) if g2 is not None else None
        call("cg_softmax_ce", self.D.n_in, self.C, ptr(self.logits), self.C4, ptr(self.labels),
             1.0 / self.L.n, ptr(self.dL), self.C4, loss_ptr, ptr(self.ce_ws), g2, self.C4, sc,
             self.stream())

    def _backward(self, spmm_ev) -> None:
        st, nL, kind, n_in = self.stream(), self.nL, self.kind, self.D.n_in
        if self._wt_early:
            self._gw(nL - 1)   # the last layer's input rows, under the backward pass
        cur = 0
        for l in range(nL - 1, -1, -1):
            F, Fo = self.F[l], self.dims[l + 1]
            if l == nL - 1 and self.tfl:
                self._backward_tfl(spmm_ev, self.dY[cur])
                continue
            dY = self.dL if l == nL - 1 else self.dY[cur]
            # weight gradient(s); the bias gradient (column sums of dY) rides
            # along in the same launch
            if kind == "gcn":
                call("cg_wgrad", n_in, F, Fo, ptr(self.Z[l]), F, ptr(dY), Fo, self._g(2 * l),
                     self._g(2 * l + 1), ptr(self.ws), self.wgrad_mode, st)
            elif l == 0 and self.tf0:
                # dW_self (+ db) as usual; dW_neigh = X^T T with T = A^T ((1/d_in) dY),
                # the transposed aggregation over the out-edges (every source of
                # the layer-0 aggregation is an inner row of this device)
                call("cg_wgrad", n_in, F, Fo, ptr(self.X[0]), F, ptr(dY), Fo, self._g(0),
                     self._g(2), ptr(self.ws), self.wgrad_mode, st)
                G = self.Gs[0]
                call("cg_scale_rows_to", ptr(G), Fo, ptr(dY), Fo, n_in, Fo, ptr(self.norm_dst), st)
                k = nL - 1
                if spmm_ev is not None:
                    self._rec(spmm_ev[k][0])
                self._spmm(n_in, Fo, self.bwd_rowptr, self.bwd_col, 1 << 62, None, G, Fo, None,
                           None, 0, None, 0, self.T, Fo)
                if spmm_ev is not None:
                    self._rec(spmm_ev[k][1])
                call("cg_wgrad", n_in, F, Fo, ptr(self.X[0]), F, ptr(self.T), Fo, self._g(1),
                     None, ptr(self.ws), self.wgrad_mode, st)
            else:
                call("cg_wgrad", n_in, F, Fo, ptr(self.X[l]), F, ptr(dY), Fo, self._g(3 * l),
                     None, ptr(self.ws), self.wgrad_mode, st)
                call("cg_wgrad", n_in, F, Fo, ptr(self.Z[l]), F, ptr(dY), Fo,
                     self._g(3 * l + 1), self._g(3 * l + 2), ptr(self.ws), self.wgrad_mode, st)
            if l == 0:
                break
            nxt = self.dY[1 - cur] if l != nL - 1 else self.dY[cur]
            wide = Fo < F  # aggregate the narrower gradient, then transform
            G = self.Gs[l & 1]
            W = 2 * l if kind == "gcn" else 3 * l + 1
            if wide:
                # G = (b | 1/d_in) * dY  (F_out wide): the rows peers pull (the
                # last layer's comes out of cg_softmax_ce)
                if l != nL - 1:
                    call("cg_scale_rows_to", ptr(G), Fo, ptr(dY), Fo, n_in, Fo,
                         ptr(self.norm_dst), st)
                Fx = Fo
            elif kind == "gcn":
                self._gemm(n_in, F, Fo, ptr(dY), Fo, W, trans_b=1, row_scale=ptr(self.norm_dst),
                           C=ptr(G), ldc=F)
                Fx = F
            else:
                self._gemm(n_in, F, Fo, ptr(dY), Fo, W, trans_b=1, row_scale=ptr(self.norm_dst),
                           C=ptr(G), ldc=F)
                self._gemm(n_in, F, Fo, ptr(dY), Fo, 3 * l, trans_b=1, C=ptr(self.Hs), ldc=F)
                Fx = F
            self.comm.barrier()
            if self.n_bwd:
                self._copy(self.n_bwd, Fx, self.b_src, self.b_row, self.b_dst, self.tabGs[l & 1],
                           self._tabG_ld(Fx), G, Fx, cls="grad_pull")
            k = nL - 1 - l
            if spmm_ev is not None:
                self._rec(spmm_ev[k][0])
            if wide:
                # T = (a | 1) * A^T G, then dY_{l-1} = mask * (T W^T [+ dY W_self^T])
                self._spmm(n_in, Fx, self.bwd_rowptr, self.bwd_col, 1 << 62, None, G, Fx,
                           self.norm_src if kind == "gcn" else None, None, 0, None, 0, self.T, Fx)
            else:
                self._spmm(n_in, F, self.bwd_rowptr, self.bwd_col, 1 << 62, None, G, F,
                           self.norm_src if kind == "gcn" else None,
                           self.Hs if kind == "sage" else None, F, None, 0, nxt, F, mask_l=l)
            if spmm_ev is not None:
                self._rec(spmm_ev[k][1])
            if wide:
                if kind == "gcn":
                    self._gemm(n_in, F, Fo, ptr(self.T), Fo, W, trans_b=1, mask_l=l,
                               C=ptr(nxt), ldc=F)
                else:
                    self._gemm(n_in, F, Fo, ptr(dY), Fo, 3 * l, Fo, ptr(self.T), Fo, W,
                               trans_b=1, mask_l=l, C=ptr(nxt), ldc=F)
            if l != nL - 1:
                cur = 1 - cur

    def _update(self) -> None:
        """K7 + optimizer + the weights' TF32 split; uses self.step."""
        # the write-through queue joins BEFORE K7: a rank's all-reduce then
        # completes only after every rank's host-tier writes of this epoch,
        # which the next epoch's prefetch reads
        self._join_gw()
        self.comm.allreduce_(self.grads)
        if not self._wt_early:
            # the last layer's write-through goes after every rank's staging
            # of that layer (the all-reduce orders it), and lands before any
            # rank's next epoch starts
            self._gw(self.nL - 1)
            self._join_gw()
            if self.comm.world > 1:
                self.comm.barrier()
        call("cg_adam", self.n_params, ptr(self.params), ptr(self.grads), ptr(self.adam_m),
             ptr(self.adam_v), self.lr, 0.9, 0.999, 1e-8, self.step,
             ptr(self.params_hi) if self.params_hi is not None else None,
             ptr(self.params_lo) if self.params_lo is not None else None,
             ptr(self.adam_corr) if self._capturing else None, self.stream())
        if self.params_hi is not None:
            self._split_t()

    def _new_timers(self, n: int):
        return [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(n)]

    # ----------------------------------------------------------- epoch graphs
    def _graph_epoch_ok(self, e: int) -> bool:
        """A steady-state epoch: K6-planned, no epoch-1 snapshot, one process."""
        return (self.use_graphs and e > 1 and self.plan_mode != "host"
                and self.policy in ("jaca", "fifo") and e > self.freeze_epoch
                and self.L.union is not None and self.L.union.size > 0
                and (self.gpu_plan_ready or self.planner.state()["admissions"] == 0))

    def _capture(self, e: int) -> None:
        """Capture the steady-state epoch as two CUDA graphs: plan + forward +
        loss, then backward + K7 + optimizer (the logits-ready event for the
        host download is recorded between the two replays).  The per-epoch
        scalars come from epoch_dev / adam_corr, so one capture serves every
        later epoch.  SpMM timing events are external event nodes."""
        if not self.gpu_plan_ready:
            self._init_gpu_plan()
        fwd_ev, bwd_ev = self._new_timers(self.nL), self._new_timers(self._n_bwd_spmm())
        for a, b in fwd_ev + bwd_ev:   # materialise the events before capture
            a.record()
            b.record()
        self._io_state()      # copy streams exist before capture
        pool = torch.cuda.graph_pool_handle()
        g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        # launches recorded by the capture run on each replay, not now
        before = dict(_lib.launches)
        self._capturing = True
        self._k3_used = [] if self._k3_on else None
        try:
            if self._wt is not None:
                # write-through queue active: ONE graph, so the copies forked
                # in the forward pass join only at the end of the update
                with torch.cuda.graph(g1, pool=pool):
                    self.plan(e)
                    self._forward(e, fwd_ev)
                    self._loss()
                    self._backward(bwd_ev)
                    self._update()
                g2 = None
            else:
                with torch.cuda.graph(g1, pool=pool):
                    self.plan(e)
                    self._forward(e, fwd_ev)
                    self._loss()
                with torch.cuda.graph(g2, pool=pool):
                    self._backward(bwd_ev)
                    self._update()
        finally:
            self._capturing = False
        recorded = {k: v - before.get(k, 0) for k, v in _lib.launches.items()
                    if v != before.get(k, 0)}
        _lib.count_replay({k: -v for k, v in recorded.items()})
        self._graphs = (g1, g2, fwd_ev, bwd_ev, recorded, self._k3_used)
        self._k3_used = None

    def _run_epoch_graph(self, e: int, timers: bool, sync: bool) -> EpochStats:
        if self._graphs is None:
            self._capture(e)
        g1, g2, fwd_ev, bwd_ev, recorded, k3_used = self._graphs
        cs = torch.cuda.current_stream(self.dev)
        t0 = t1 = None
        if timers:
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record()
        self.step += 1
        call("cg_set_epoch", ptr(self.epoch_dev), e, ptr(self.adam_corr), 0.9, 0.999, self.step,
             self.stream())
        self._consume_input()
        self._wait_logits_download()
        g1.replay()
        if self._io is not None:
            # logits final: after the forward graph (or, single-graph epochs,
            # after the whole epoch)
            ev = torch.cuda.Event()
            ev.record(cs)
            self._io["fwd"] = ev
        if g2 is not None:
            g2.replay()
        _lib.count_replay(recorded)
        if timers:
            t1 = torch.cuda.Event(enable_timing=True)
            t1.record()
        # the graphs' SpMM events carry the most recent replay's times
        stats = EpochStats(epoch=e, loss=float("nan"), counts=None, seconds=0.0,
                           spmm_fwd_ms=list(fwd_ev) if timers else [],
                           spmm_bwd_ms=list(bwd_ev) if timers else [], planner="gpu",
                           events=(t0, t1) if timers else None)
        stats.counts = self.k6["counts"].clone()
        stats.flag = self.k6["flag"].clone()
        stats.loss = self.grads[self.n_params:].clone()
        stats.k3 = list(k3_used) if (timers and k3_used) else None
        return self.finish(stats) if sync else stats

    def run_epoch(self, e: int, timers: bool = True, sync: bool = True) -> EpochStats:
        if self._graph_epoch_ok(e):
            return self._run_epoch_graph(e, timers, sync)
        t0 = t1 = None
        if timers:
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record()
        fwd_ev = self._new_timers(self.nL) if timers else None
        bwd_ev = self._new_timers(self._n_bwd_spmm()) if timers else None
        self._k3_used = [] if (timers and self._k3_on) else None
        self._mark("plan")
        mode, hcounts, _ = self.plan(e)
        self._consume_input()
        self._mark("forward")
        self._forward(e, fwd_ev)
        if self._io is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.dev))
            self._io["fwd"] = ev
        self._mark("loss")
        self._loss()
        self._mark("backward")
        self._backward(bwd_ev)
        self._mark("allreduce+adam")
        self.step += 1
        self._update()
        if timers:
            t1 = torch.cuda.Event(enable_timing=True)
            t1.record()
        self._mark(None)
        stats = EpochStats(epoch=e, loss=float("nan"), counts=hcounts, seconds=0.0,
                           spmm_fwd_ms=fwd_ev or [], spmm_bwd_ms=bwd_ev or [], planner=mode,
                           events=(t0, t1) if timers else None, k3=self._k3_used)
        self._k3_used = None
        if mode == "gpu":
            # keep this epoch's counters on the device until finish()
            stats.counts = self.k6["counts"].clone()
            stats.flag = self.k6["flag"].clone()
        stats.loss = self.grads[self.n_params:].clone()
        return self.finish(stats) if sync else stats

    def finish(self, stats: EpochStats) -> EpochStats:
        """Synchronise one epoch's results to the host (loss, counters, times)."""
        if not isinstance(stats.loss, float):
            stats.loss = float(stats.loss.item()) / self.L.n
        if stats.planner == "gpu" and not isinstance(stats.counts, np.ndarray):
            stats.counts = stats.counts.view(self.L.P, 3).cpu().numpy()
            stats.flag = int(stats.flag.item())
            if stats.flag == 2:
                raise RuntimeError(
                    f"epoch {stats.epoch}: the compact layout's precondition (no staged or "
                    "slab reads) was violated")
            if stats.flag:
                raise RuntimeError(
                    f"epoch {stats.epoch}: frozen-membership precondition violated (an "
                    "admission would happen); rerun with plan_mode='host'")
        if stats.events is not None:
            t0, t1 = stats.events
            stats.seconds = t0.elapsed_time(t1) / 1e3
            stats.spmm_fwd_ms = [a.elapsed_time(b) for a, b in stats.spmm_fwd_ms]
            stats.spmm_bwd_ms = [a.elapsed_time(b) for a, b in stats.spmm_bwd_ms]
            stats.events = None
        if isinstance(stats.k3, list):
            k3 = {}
            for cls, F, (a, b) in stats.k3:
                k3[cls] = k3.get(cls, 0.0) + a.elapsed_time(b)
            stats.k3 = k3
        return stats

    # ------------------------------------------------------------ host I/O
    # An input/output pipeline on two copy streams, so the per-step host
    # traffic overlaps the epoch: the NEXT step's input rows are uploaded
    # (H2D) while this step trains, and this step's logits are downloaded
    # (D2H) during its backward pass.  Ordering is by CUDA events only.
    def _io_state(self):
        if self._io is None:
            self._io = dict(h2d=torch.cuda.Stream(self.dev), d2h=torch.cuda.Stream(self.dev),
                            stage=torch.empty(self.D.n_in, self.F[0], dtype=torch.float32,
                                              device=self.dev),
                            ready=None, free=None, logits_done=None, fwd=None)
        return self._io

    def prefetch_features(self, host_x) -> None:
        """Start the H2D copy of the next epoch's input rows (pinned host,
        raw features, this device's inner rows) on the upload stream; the
        next run_epoch waits for it and scales the rows into X_0."""
        io = self._io_state()
        st = io["h2d"]
        if io["free"] is not None:
            st.wait_event(io["free"])      # the previous upload has been consumed
        with torch.cuda.stream(st):
            io["stage"].copy_(host_x, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(st)
        io["ready"] = ev

    def _consume_input(self) -> None:
        io = self._io
        if io is None or io["ready"] is None:
            return
        cs = torch.cuda.current_stream(self.dev)
        cs.wait_event(io["ready"])
        F0 = self.F[0]
        call("cg_scale_rows_to", ptr(self.X[0]), F0, ptr(io["stage"]), F0, self.D.n_in, F0,
             ptr(self.norm_src) if self.kind == "gcn" else None, self.stream())
        if self.comm.world > 1:
            # peers read these rows (IPC) in their layer-0 staging / snapshot
            # copies: every rank's new inputs land before anyone pulls
            self.comm.barrier()
        ev = torch.cuda.Event()
        ev.record(cs)
        io["free"], io["ready"] = ev, None

    def fetch_logits(self, host_buf) -> None:
        """Start the D2H copy of the current epoch's logits (available once
        its forward pass is done) into a pinned host buffer."""
        io = self._io_state()
        st = io["d2h"]
        if io["fwd"] is not None:
            st.wait_event(io["fwd"])
        else:
            st.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(st):
            host_buf.copy_(self.logits, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(st)
        io["logits_done"] = ev

    def fetch_loss(self, stats: "EpochStats", host_buf) -> None:
        """Start the D2H copy of an epoch's loss (sum; divide by n) into a
        pinned host scalar, ordered after that epoch's K7."""
        io = self._io_state()
        st = io["d2h"]
        st.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(st):
            host_buf.copy_(stats.loss.view(-1)[:1], non_blocking=True)

    def upload_features(self, host_x) -> None:
        """H2D copy of this device's input rows (pinned host, raw features),
        then the GCN source-degree pre-scaling on the device."""
        D = self.D
        self.X[0][:D.n_in].copy_(host_x, non_blocking=True)
        if self.kind == "gcn":
            call("cg_scale_rows", ptr(self.X[0]), self.F[0], D.n_in, self.F[0],
                 ptr(self.norm_src), self.stream())

    def k3_rows(self) -> dict:
        """Rows the K3 launches of the epoch just run move, by class and tier,
        read from this epoch's device tables (a sync; keep it outside timed
        regions).  Tiers: ``host`` = pinned global tier over PCIe, ``peer`` =
        another GPU over NVLink, ``hbm`` = this GPU."""
        D, nd, me = self.D, self.L.n_dev, self.me
        out = {"stage_host": 0, "stage_peer": 0, "stage_hbm": 0, "write_through": 0,
               "write_back": 0, "grad_pull": int(self.n_bwd)}
        if D.n_halo and not self.L.compact:
            src, dst = self.stage_src[:D.n_halo], self.stage_dst[:D.n_halo]
            live = (src >= 0) & (dst >= 0)
            out["stage_host"] = int((live & (src == nd)).sum())
            out["stage_peer"] = int((live & (src != nd) & (src != me)).sum())
            out["stage_hbm"] = int((live & (src == me)).sum())
        if (self.c_cpu and self.L.union is not None and self.L.union.size
                and not self.L.compact):
            out["write_through"] = int((self.gw_slot >= 0).sum())
        if self.wb is not None:
            out["write_back"] = int(self.wb[3])
        return out

    def k3_widths(self) -> dict:
        """Floats per row each K3 class moves per epoch, summed over the
        layers it runs in (stage / write-through / write-back: every layer's
        input width; gradient pulls: the hidden layers' aggregated width)."""
        fsum = int(sum(self.F))
        widths = list(self.F) + [self.C4]
        gsum = int(sum(min(widths[l], widths[l + 1]) for l in range(1, self.nL)))
        return {"stage_host": fsum, "stage_peer": fsum, "stage_hbm": fsum,
                "write_through": fsum, "write_back": fsum, "grad_pull": gsum}

    def gpu_outcomes(self) -> np.ndarray:
        """Per-requester outcomes of the last GPU-planned epoch (flat order)."""
        o = self.k6["outcome"].cpu().numpy()[: self.L.req_index.size]
        out = np.empty_like(o)
        out[self.L.req_index] = o
        return out

    def logits_global(self) -> np.ndarray:
        """This device's logits keyed by vertex id: (verts, logits)."""
        return self.D.verts, self.logits[:, :self.C].detach().cpu().numpy()

    def close(self):
        self.comm.close()
        self.host.close()
