"""Float half of the CPU oracle: partitioned full-batch GCN / GraphSAGE-mean.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The reference (halopart) has no float code: it only decides, per epoch and
per (partition, halo vertex), whether the halo row comes from the local
cache, the global cache or the owner (cache.py:264-309, driven by
simulator.py:206-226).  This module restates the training step those
decisions feed, with the semantics pinned in DESIGN.md §3:

* a cache entry covers every layer's input row of one vertex (cache.py:54-58);
* a halo row served at version ``ver`` holds the owner's activation from the
  forward pass of epoch ``max(ver, 1)`` (warm entries, version 0, are the
  epoch-1 values -- weights do not change before epoch 1's update);
* caching is forward-only (simulator.py:235): the gradient with
  respect to every halo row used by a partition flows back to the owner;
* GCN normalisation uses GLOBAL degrees with a self-loop added where missing:
  w_uv = (d_out(u)+1)^-1/2 (d_in(v)+1)^-1/2; SAGE-mean uses 1/d_in(v);
* loss = mean cross-entropy over all vertices; Adam(lr, 0.9, 0.999, 1e-8).

"Parity unpinned" against the reference (no reference float code exists);
self-checked against ``full_graph_epochs`` (capacity 0 / s = 0 must equal
plain full-graph training).  Arithmetic is float64 numpy + scipy.sparse.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

M32 = 0xFFFFFFFF


# ---------------------------------------------------------------------------
# deterministic synthetic inputs (bit-identical to the CUDA generator)


def mix32(seed, a, b):
    """32-bit avalanche hash of (seed, a, b); numpy uint64 arithmetic."""
    s = np.uint64(seed)
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    h = (s * np.uint64(0x9E3779B1) + a * np.uint64(0x85EBCA77)
         + b * np.uint64(0xC2B2AE3D)) & np.uint64(M32)
    h ^= h >> np.uint64(16)
    h = (h * np.uint64(0x7FEB352D)) & np.uint64(M32)
    h ^= h >> np.uint64(15)
    h = (h * np.uint64(0x846CA68B)) & np.uint64(M32)
    h ^= h >> np.uint64(16)
    return h


def uniform_pm1(seed, a, b) -> np.ndarray:
    """fp32 in [-1, 1): (h >> 8) * 2^-23 - 1, exact in float32."""
    h = mix32(seed, a, b) >> np.uint64(8)
    return (h.astype(np.float32) * np.float32(2.0 ** -23)) - np.float32(1.0)


def features(n: int, F: int, seed: int = 0) -> np.ndarray:
    v = np.arange(n, dtype=np.uint64)[:, None]
    k = np.arange(F, dtype=np.uint64)[None, :]
    return uniform_pm1(seed, v, k)


def labels(n: int, C: int, seed: int = 1) -> np.ndarray:
    return (mix32(seed, np.arange(n, dtype=np.uint64), 0) % np.uint64(C)).astype(np.int64)


def glorot(fan_in: int, fan_out: int, seed: int) -> np.ndarray:
    a = np.float32(np.sqrt(6.0 / (fan_in + fan_out)))
    i = np.arange(fan_in, dtype=np.uint64)[:, None]
    j = np.arange(fan_out, dtype=np.uint64)[None, :]
    return (uniform_pm1(seed, i, j) * a).astype(np.float32)


def init_params(kind: str, dims: list[int], seed: int = 2) -> list[np.ndarray]:
    """dims = [F_0, ..., F_L]; per layer: GCN (W, b); SAGE (W_self, W_neigh, b)."""
    params = []
    for l in range(len(dims) - 1):
        fi, fo = dims[l], dims[l + 1]
        if kind == "gcn":
            params += [glorot(fi, fo, seed + 16 * l), np.zeros(fo, np.float32)]
        else:
            params += [glorot(fi, fo, seed + 16 * l), glorot(fi, fo, seed + 16 * l + 1),
                       np.zeros(fo, np.float32)]
    return params


# ---------------------------------------------------------------------------
# model pieces


@dataclass
class ModelSpec:
    kind: str            # "gcn" | "sage"
    dims: list[int]      # [F_0 .. F_L]; F_L = classes
    lr: float = 0.01


def degree_norms(g):
    """(a, b, has_self): GCN source / destination scales with self-loops."""
    has_self = np.zeros(g.n, dtype=bool)
    s, d = g.edges()
    has_self[s[s == d]] = True
    dout = g.out_deg + (~has_self)
    din = g.in_deg + (~has_self)
    return 1.0 / np.sqrt(dout.astype(np.float64)), 1.0 / np.sqrt(din.astype(np.float64)), has_self


def local_operator(g, inner: np.ndarray, halo: np.ndarray, kind: str, norms):
    """Sparse (n_inner x (n_inner + n_halo)) aggregation matrix of one partition.

    Column space: inner rows, then halo rows in ascending id.  In-edges from
    vertices outside inner | halo (RAPA-pruned halo) are dropped; degrees stay
    global.
    """
    n_in = inner.size
    col_of = np.full(g.n, -1, dtype=np.int64)
    col_of[inner] = np.arange(n_in)
    col_of[halo] = n_in + np.arange(halo.size)
    rows, cols, vals = [], [], []
    a, b, has_self = norms if norms is not None else (None, None, None)
    for r, v in enumerate(inner):
        nb = g.in_tgt[g.in_off[v]:g.in_off[v + 1]]
        if kind == "gcn" and not has_self[v]:
            nb = np.sort(np.append(nb, v))
        c = col_of[nb]
        keep = c >= 0
        nb, c = nb[keep], c[keep]
        rows.append(np.full(c.size, r))
        cols.append(c)
        if kind == "gcn":
            vals.append(a[nb] * b[v])
        else:
            dv = g.in_deg[v]
            vals.append(np.full(c.size, 1.0 / dv if dv > 0 else 0.0))
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n_in, n_in + halo.size))
    return A


def relu(x):
    return np.maximum(x, 0.0)


def softmax_ce(logits: np.ndarray, y: np.ndarray, n_total: int):
    z = logits - logits.max(axis=1, keepdims=True)
    ez = np.exp(z)
    p = ez / ez.sum(axis=1, keepdims=True)
    lse = np.log(ez.sum(axis=1))
    loss_sum = float(np.sum(lse - z[np.arange(len(y)), y]))
    grad = p.copy()
    grad[np.arange(len(y)), y] -= 1.0
    return loss_sum, grad / n_total


class Adam:
    def __init__(self, params, lr, b1=0.9, b2=0.999, eps=1e-8):
        self.lr, self.b1, self.b2, self.eps = lr, b1, b2, eps
        self.m = [np.zeros_like(p, dtype=np.float64) for p in params]
        self.v = [np.zeros_like(p, dtype=np.float64) for p in params]
        self.t = 0

    def step(self, params, grads):
        self.t += 1
        c1 = 1.0 - self.b1 ** self.t
        c2 = 1.0 - self.b2 ** self.t
        for i, (p, g) in enumerate(zip(params, grads)):
            self.m[i] = self.b1 * self.m[i] + (1 - self.b1) * g
            self.v[i] = self.b2 * self.v[i] + (1 - self.b2) * g * g
            p -= self.lr * (self.m[i] / c1) / (np.sqrt(self.v[i] / c2) + self.eps)


@dataclass
class EpochOut:
    epoch: int
    loss: float
    logits: np.ndarray


def _layer_params(spec, params, l):
    return params[2 * l:2 * l + 2] if spec.kind == "gcn" else params[3 * l:3 * l + 3]


class Trainer:
    """Stepwise partitioned training (one call of ``step`` = one epoch)."""

    def __init__(self, g, inner, halo, spec: ModelSpec, X, y, params=None):
        self.g, self.inner, self.halo, self.spec = g, inner, halo, spec
        self.L = len(spec.dims) - 1
        self.P = len(inner)
        self.params = [p.astype(np.float64) for p in (params or init_params(spec.kind, spec.dims))]
        self.opt = Adam(self.params, spec.lr)
        norms = degree_norms(g) if spec.kind == "gcn" else None
        self.ops = [local_operator(g, inner[p], halo[p], spec.kind, norms) for p in range(self.P)]
        self.history: dict[int, list[np.ndarray]] = {}
        self.X = X.astype(np.float64)
        self.y = y
        self.e = 0

    def step(self, versions_e, forced_params=None) -> EpochOut:
        """versions_e[p]: served versions of partition p's halo (ascending id).

        forced_params: run this epoch from these weights instead of the
        oracle's own trajectory (isolates one epoch's arithmetic from Adam's
        amplification of earlier rounding differences).
        """
        if forced_params is not None:
            for dst, src in zip(self.params, forced_params):
                dst[...] = np.asarray(src, np.float64)
        spec, params, L, P, n = self.spec, self.params, self.L, self.P, self.g.n
        inner, halo, ops, history = self.inner, self.halo, self.ops, self.history
        self.e += 1
        e = self.e
        cur = [self.X]
        used = []  # per layer: (per partition (H_in, agg), pre-activation)
        for l in range(L):
            H = cur[l]
            nxt = np.zeros((n, spec.dims[l + 1]))
            lay = []
            for p in range(P):
                src = np.maximum(versions_e[p], 1)
                hal = H[halo[p]].copy()
                for old in np.unique(src[src != e]):
                    sel = src == old
                    hal[sel] = history[int(old)][l][halo[p][sel]]
                Hin = np.vstack([H[inner[p]], hal])
                agg = ops[p] @ Hin
                lp = _layer_params(spec, params, l)
                if spec.kind == "gcn":
                    Y = agg @ lp[0] + lp[1]
                else:
                    Y = H[inner[p]] @ lp[0] + agg @ lp[1] + lp[2]
                nxt[inner[p]] = Y
                lay.append((Hin, agg))
            used.append((lay, nxt))
            cur.append(relu(nxt) if l < L - 1 else nxt)
        history[e] = cur
        logits = cur[L]
        loss_sum, dY = softmax_ce(logits, self.y, n)
        out = EpochOut(epoch=e, loss=loss_sum / n, logits=logits.copy())
        grads = [np.zeros_like(p) for p in params]
        for l in range(L - 1, -1, -1):
            lay, _ = used[l]
            dH = np.zeros((n, spec.dims[l])) if l > 0 else None
            gi = 2 * l if spec.kind == "gcn" else 3 * l
            lp = _layer_params(spec, params, l)
            for p in range(P):
                Hin, agg = lay[p]
                dYp = dY[inner[p]]
                n_in = inner[p].size
                if spec.kind == "gcn":
                    grads[gi] += agg.T @ dYp
                    grads[gi + 1] += dYp.sum(axis=0)
                    if l > 0:
                        dHin = ops[p].T @ (dYp @ lp[0].T)
                        np.add.at(dH, inner[p], dHin[:n_in])
                        np.add.at(dH, halo[p], dHin[n_in:])
                else:
                    grads[gi] += Hin[:n_in].T @ dYp
                    grads[gi + 1] += agg.T @ dYp
                    grads[gi + 2] += dYp.sum(axis=0)
                    if l > 0:
                        dHin = ops[p].T @ (dYp @ lp[1].T)
                        dHin[:n_in] += dYp @ lp[0].T
                        np.add.at(dH, inner[p], dHin[:n_in])
                        np.add.at(dH, halo[p], dHin[n_in:])
            if l > 0:
                dY = dH * (used[l - 1][1] > 0)
        self.opt.step(params, grads)
        return out


def partitioned_epochs(g, inner, halo, versions, spec: ModelSpec, X, y,
                       params=None, epochs: int | None = None):
    """Train for len(versions) epochs; returns per-epoch (loss, logits), params.

    versions[e-1][p] is the int array of served versions for partition p's
    halo (ascending id), as produced by the cache plan.
    """
    tr = Trainer(g, inner, halo, spec, X, y, params)
    epochs = len(versions) if epochs is None else epochs
    outs = [tr.step(versions[e]) for e in range(epochs)]
    return outs, tr.params


def full_graph_epochs(g, spec: ModelSpec, X, y, epochs: int, params=None):
    """Plain unpartitioned training (the self-check target)."""
    inner = [np.arange(g.n, dtype=np.int64)]
    halo = [np.empty(0, dtype=np.int64)]
    versions = [[np.empty(0, dtype=np.int64)] for _ in range(epochs)]
    return partitioned_epochs(g, inner, halo, versions, spec, X, y, params, epochs)
