"""Sampled-row float64 oracle for the large shapes (C3 Reddit-, C4 products-shaped).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  ``model_port`` runs
whole partitioned epochs in float64; at C4 (2.45M vertices, 62M edges,
256-wide hidden layers) that is hours of numpy.  This module computes the
logits of a SAMPLE of vertices instead, exactly, over their L-hop in-edge
receptive field, with the semantics ``model_port.Trainer`` pins (DESIGN.md
§3) for the configuration the large-shape tests run: JACA with Algorithm-1
capacities (every local level holds its whole halo) and staleness -1, the
reference default (``simulator.py:43``, ``cli.py:59``).  Under that plan
every halo lookup is a local hit on the warm version-0 entry
(``cache.py:221-224``: s < 0 is always fresh; ``cache.py:323-347``: warm
versions are 0), so by SURVEY Appendix A2/A6:

* layer 0 (the input features) is static: a halo row is the owner's row;
* a hidden-layer halo row served at version 0 is the owner's epoch-1
  activation, i.e. the FULL-GRAPH epoch-1 value (no weight has changed
  before epoch 1's update);
* an inner row (same partition as the reader) is the current epoch's value.

``sampled_logits`` runs "weight-forced" epochs: epoch e is computed from the
weights the GPU held at its start (``TrainReport.params_per_epoch``), so a
comparison checks one epoch's arithmetic at full scale without Adam
compounding earlier rounding differences (the same check
``tests/test_gpu_train_parity.py`` makes with ``model_port`` at small sizes).

Model (DESIGN.md §3 A4): GCN ``H' = relu(Â H W + b)`` with
``Â_vu = (d_out(u)+1)^-1/2 (d_in(v)+1)^-1/2`` over global degrees and a
self-loop where missing; GraphSAGE-mean ``H' = relu(H W_self +
mean_{N_in(v)} H W_neigh + b)`` (``1/d_in(v)``, 0 for no in-edges); no
activation on the last layer.  Features are ``model_port.features`` rows
(the same integer hash the CUDA generator uses), evaluated only for the
vertices the receptive field reaches.
"""

from __future__ import annotations

import numpy as np

from .model_port import uniform_pm1


def _feature_rows(verts: np.ndarray, F: int, seed: int = 0) -> np.ndarray:
    k = np.arange(F, dtype=np.uint64)[None, :]
    return uniform_pm1(seed, verts.astype(np.uint64)[:, None], k).astype(np.float64)


class SampledGraph:
    """In-edge CSR + global degrees + the partition of every vertex."""

    def __init__(self, in_off: np.ndarray, in_tgt: np.ndarray, parts: np.ndarray, kind: str):
        self.in_off = np.asarray(in_off, np.int64)
        self.in_tgt = np.asarray(in_tgt, np.int64)
        self.n = self.in_off.size - 1
        self.parts = np.asarray(parts, np.int64)
        self.kind = kind
        self.in_deg = np.diff(self.in_off)
        if kind == "gcn":
            out_deg = np.bincount(self.in_tgt, minlength=self.n)
            rows = np.repeat(np.arange(self.n), self.in_deg)
            has_self = np.zeros(self.n, bool)
            has_self[rows[self.in_tgt == rows]] = True
            self.has_self = has_self
            self.a = 1.0 / np.sqrt((out_deg + ~has_self).astype(np.float64))
            self.b = 1.0 / np.sqrt((self.in_deg + ~has_self).astype(np.float64))

    def edges_into(self, rows: np.ndarray):
        """(row index into ``rows``, source vertex, weight) of every
        aggregated edge into ``rows`` (GCN: with the self-loop)."""
        lo, hi = self.in_off[rows], self.in_off[rows + 1]
        cnt = hi - lo
        r = np.repeat(np.arange(rows.size), cnt)
        starts = np.repeat(lo - np.concatenate(([0], np.cumsum(cnt)[:-1])), cnt)
        src = self.in_tgt[starts + np.arange(r.size)]
        if self.kind == "gcn":
            add = ~self.has_self[rows]
            r = np.concatenate([r, np.flatnonzero(add)])
            src = np.concatenate([src, rows[add]])
            w = self.a[src] * self.b[rows[r]]
        else:
            d = self.in_deg[rows[r]]
            w = np.where(d > 0, 1.0 / np.maximum(d, 1), 0.0)
        return r, src, w


def _agg(rows, r, idx, w, H):
    """sum_e w_e H[idx_e] into row r_e, as one sparse x dense product (no
    per-edge temporaries: C3's receptive fields hold ~10^7 edges)."""
    import scipy.sparse as sp
    A = sp.csr_matrix((w, (r, idx)), shape=(rows.size, H.shape[0]))
    return np.asarray(A @ H)


def sampled_logits(sg: SampledGraph, dims, params_by_epoch, samples: np.ndarray,
                   feat_seed: int = 0):
    """Logits of ``samples`` for each weight-forced epoch (see module doc).

    params_by_epoch[e]: the layer parameters at the start of epoch e+1
    (GCN: W, b per layer; SAGE: W_self, W_neigh, b).  Returns a list of
    (len(samples) x dims[-1]) float64 arrays."""
    L = len(dims) - 1
    per = 2 if sg.kind == "gcn" else 3
    samples = np.unique(np.asarray(samples, np.int64))
    # receptive fields: S[L] = samples, S[l-1] = S[l] | in-neighbours(S[l])
    S = [None] * (L + 1)
    S[L] = samples
    edges = [None] * (L + 1)
    for l in range(L, 0, -1):
        r, src, w = sg.edges_into(S[l])
        edges[l] = (r, src, w)
        S[l - 1] = np.union1d(S[l], src)
    X0 = _feature_rows(S[0], dims[0], feat_seed)
    epoch1 = None   # per layer: full-graph epoch-1 activations over S[l]
    outs = []
    for e, params in enumerate(params_by_epoch):
        p = [np.asarray(x, np.float64) for x in params]
        cur = [X0]
        for l in range(1, L + 1):
            rows = S[l]
            r, src, w = edges[l]
            idx = np.searchsorted(S[l - 1], src)
            Hc = cur[l - 1]
            if e == 0 or l == 1:
                agg = _agg(rows, r, idx, w, Hc)
            else:
                # same partition as the reader: current; else the version-0
                # (epoch-1) snapshot of a hidden-layer row
                same = sg.parts[src] == sg.parts[rows[r]]
                agg = (_agg(rows, r[same], idx[same], w[same], Hc)
                       + _agg(rows, r[~same], idx[~same], w[~same], epoch1[l - 1]))
            W = p[per * (l - 1):per * l]
            if sg.kind == "gcn":
                Y = agg @ W[0] + W[1]
            else:
                self_rows = Hc[np.searchsorted(S[l - 1], rows)]
                Y = self_rows @ W[0] + agg @ W[1] + W[2]
            cur.append(np.maximum(Y, 0.0) if l < L else Y)
        if e == 0:
            epoch1 = cur
        outs.append(cur[L])
    return samples, outs
