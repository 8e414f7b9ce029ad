"""PyTorch-CPU fp32 restatement of the partitioned GCN / GraphSAGE-mean epoch.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``): this is the CPU
baseline BASELINE.md §4 names -- "a PyTorch-CPU fp32 restatement of
partitioned GCN/SAGE using the same plan and seeds, with
torch.set_num_threads(all cores)" -- timed by ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs next to the planner port
(``halo_port.Planner``, the restatement of halopart's ``simulator.run`` loop,
simulator.py:206-226).  It is never imported by the product.

Semantics are exactly ``model_port.Trainer``'s: a halo row
served at version ``ver`` holds the owner's activation from the forward pass
of epoch ``max(ver, 1)``; the gradient of every used halo row flows to the
owner's row (straight-through for stale values); GCN weights
``(d_out(u)+1)^-1/2 (d_in(v)+1)^-1/2`` over global degrees with self-loops;
SAGE-mean ``1/d_in(v)``; mean cross-entropy; Adam(0.01, 0.9, 0.999, 1e-8).
The arithmetic is fp32 (model_port is float64), all partitions are
aggregated by ONE block sparse operator per layer (rows: every vertex, in
vertex order; columns: the current rows, then every (partition, halo slot)),
and autograd supplies the backward pass.  ``tests/test_oracle_golden.py``
checks it against model_port within 1e-4.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from .model_port import EpochOut, degree_norms, init_params, local_operator


def _to_torch_csr(m):
    m = m.tocsr()
    m.sort_indices()
    return torch.sparse_csr_tensor(torch.from_numpy(m.indptr.astype(np.int64)),
                                   torch.from_numpy(m.indices.astype(np.int64)),
                                   torch.from_numpy(m.data.astype(np.float32)), m.shape,
                                   check_invariants=False)


def _block_operator(g, inner, halo, kind):
    """The aggregation of every partition as one operator A, n x (n + sum
    |H_p|): rows are vertices, columns the current rows then every
    (partition, halo slot).  Also returns the transpose of A "folded" onto
    the owners (halo slot columns summed into their vertex's column) -- the
    backward operator, since every halo row's gradient goes to its owner."""
    import scipy.sparse as sp
    norms = degree_norms(g) if kind == "gcn" else None
    n = g.n
    hoff = np.concatenate(([0], np.cumsum([h.size for h in halo]))).astype(np.int64)
    halo_cat = np.concatenate(halo).astype(np.int64) if hoff[-1] else np.zeros(0, np.int64)
    rows, cols, vals = [], [], []
    for p in range(len(inner)):
        A = local_operator(g, inner[p], halo[p], kind, norms).tocoo()
        n_in = inner[p].size
        rows.append(inner[p][A.row])
        c = A.col.astype(np.int64)
        cols.append(np.where(c < n_in, inner[p][np.minimum(c, n_in - 1)],
                             n + hoff[p] + (c - n_in)))
        vals.append(A.data)
    r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    full = sp.csr_matrix((v, (r, c)), shape=(n, n + int(hoff[-1])))
    owner = np.where(c < n, c, halo_cat[np.maximum(c - n, 0)] if halo_cat.size else c)
    fold = sp.csr_matrix((v, (r, owner)), shape=(n, n))   # duplicates are summed
    A_in, A_halo = full[:, :n], full[:, n:]
    return (_to_torch_csr(A_in), _to_torch_csr(A_halo) if halo_cat.size else None,
            _to_torch_csr(fold.T), halo_cat)


class _Aggregate(torch.autograd.Function):
    """Z = A_in @ H + A_halo @ S (S: the served halo rows, constants);
    dH = Fold^T @ dZ (MKL's threaded CSR x dense both ways)."""

    @staticmethod
    def forward(ctx, H, S, A_in, A_halo, FoldT):
        ctx.FoldT = FoldT
        Z = A_in @ H
        if A_halo is not None:
            Z += A_halo @ S
        return Z

    @staticmethod
    def backward(ctx, dZ):
        return ctx.FoldT @ dZ.contiguous(), None, None, None, None


class TorchTrainer:
    """Stepwise fp32 partitioned training on the host cores."""

    def __init__(self, g, inner, halo, spec, X, y, params=None, threads: int | None = None):
        torch.set_num_threads(threads or len(os.sched_getaffinity(0)))
        self.spec, self.L, self.n = spec, len(spec.dims) - 1, g.n
        self.A_in, self.A_halo, self.FoldT, hc = _block_operator(g, inner, halo, spec.kind)
        self.halo_cat = torch.from_numpy(hc)
        self._snap = {}   # layer -> (src, served rows) when every row was stale
        self.X = torch.from_numpy(np.asarray(X, np.float32))
        self.y = torch.from_numpy(np.asarray(y, np.int64))
        init = params or init_params(spec.kind, spec.dims)
        self.params = [torch.tensor(np.asarray(p, np.float32), requires_grad=True) for p in init]
        self.opt = torch.optim.Adam(self.params, lr=spec.lr, betas=(0.9, 0.999), eps=1e-8)
        self.history: dict[int, list[torch.Tensor]] = {}
        self.e = 0

    def _served(self, H, l, src):
        """The halo slot values this epoch serves (constants): the current
        row, or the owner's snapshot from epoch ``src`` for stale entries.
        An all-stale set equal to the previous epoch's is reused as is."""
        stale = src != self.e
        prev = self._snap.get(l)
        if stale.all() and prev is not None and np.array_equal(prev[0], src):
            return prev[1]
        S = torch.empty(src.size, H.shape[1])
        cur = torch.from_numpy(np.flatnonzero(~stale))
        if cur.numel():
            S[cur] = H.detach().index_select(0, self.halo_cat[cur])
        for old in np.unique(src[stale]):
            sel = torch.from_numpy(np.flatnonzero(src == old))
            S[sel] = self.history[int(old)][l].index_select(0, self.halo_cat[sel])
        self._snap[l] = (src.copy(), S) if stale.all() else None
        return S

    def step(self, versions_e, live_versions=None) -> EpochOut:
        """versions_e[p]: served versions of partition p's halo (ascending id).
        live_versions (optional): versions any cache level still holds; the
        snapshots of other epochs are dropped."""
        spec, L = self.spec, self.L
        self.e += 1
        src = (np.maximum(np.concatenate(versions_e), 1) if len(versions_e)
               else np.zeros(0, np.int64))
        H = self.X
        acts = [H.detach()]
        per = 2 if spec.kind == "gcn" else 3
        with torch.enable_grad():
            for l in range(L):
                S = self._served(H, l, src) if self.halo_cat.numel() else None
                Z = _Aggregate.apply(H, S, self.A_in, self.A_halo, self.FoldT)
                p = self.params[per * l:per * (l + 1)]
                Y = Z @ p[0] + p[1] if spec.kind == "gcn" else H @ p[0] + Z @ p[1] + p[2]
                H = torch.relu(Y) if l < L - 1 else Y
                acts.append(H.detach())
            loss_sum = torch.nn.functional.cross_entropy(H, self.y, reduction="sum")
            self.opt.zero_grad(set_to_none=True)
            (loss_sum / self.n).backward()
        self.history[self.e] = acts
        if live_versions is not None:
            keep = {max(int(v), 1) for v in live_versions} | {self.e}
            for k in [k for k in self.history if k not in keep]:
                del self.history[k]
        out = EpochOut(epoch=self.e, loss=float(loss_sum.detach()) / self.n,
                       logits=H.detach().numpy().copy())
        self.opt.step()
        return out


def live_versions(cache) -> set:
    """Versions held anywhere in a ``halo_port.TwoLevel`` cache."""
    vs = {ent[1] for lvl in cache.loc for ent in lvl.ent.values()}
    vs.update(ent[1] for ent in cache.glo.ent.values())
    return vs
