"""Host-side layout logic (CPU): the transform-first last layer's static
CSRs (layout.source_row_csrs) against a brute-force transpose, and the
identity the backward relies on -- summing A^T G over each vertex's inner
row and its snapshot row gives the aggregation over all of the vertex's
forward edges (the out-edge view the aggregate-first backward uses)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2508_13716_b200 import hostgraph as H
from paper_2508_13716_b200.layout import build_layout, source_row_csrs


@pytest.mark.parametrize("kind", ["gcn", "sage"])
def test_source_row_csrs_brute_force(kind):
    n, P = 600, 4
    g = H.erdos_renyi(n, 6.0, 0)
    ps = H.build_partition_set(g, H.random_partition(n, P, 0), 1)
    inner = [np.asarray(x, np.int64) for x in ps.inner]
    halo = [np.asarray(h, np.int64) for h in ps.halo]
    L = build_layout(g, inner, halo, [h.size for h in halo], 1, kind, compact=True)
    D = L.devices[0]
    rp, col, urp, ucol = source_row_csrs(D, 0)
    n_in = D.n_in
    # brute force: every forward edge (dest v, source row r)
    pairs = []
    for v in range(n_in):
        for c in D.fwd_col[D.fwd_rowptr[v]:D.fwd_rowptr[v + 1]]:
            r = int(c) if c < n_in else int(D.snap_row_of_pos[c - n_in])
            assert r >= 0
            pairs.append((r, v))
    pairs.sort()
    assert rp.size == D.n_rows + 1 and rp[-1] == len(pairs)
    got = [(r, int(v)) for r in range(D.n_rows) for v in col[rp[r]:rp[r + 1]]]
    assert got == pairs
    # the owner CSR: inner row u, then the snapshot row of the same vertex
    vert_of_row = {int(D.snap_off + i): int(x) for i, x in enumerate(D.snap_vertex)}
    for u in range(n_in):
        ent = list(ucol[urp[u]:urp[u + 1]])
        assert ent[0] == u
        assert all(vert_of_row[int(s)] == int(D.verts[u]) for s in ent[1:]) and len(ent) <= 2
    # identity: sum over {u, snap(u)} of (A^T G) == sum of G over every forward
    # edge whose source vertex is verts[u]
    rng = np.random.default_rng(1)
    G = rng.standard_normal((n_in, 5))
    dh = np.zeros((D.n_rows, 5))
    for r in range(D.n_rows):
        dh[r] = G[col[rp[r]:rp[r + 1]]].sum(0)
    T = np.stack([dh[ucol[urp[u]:urp[u + 1]]].sum(0) for u in range(n_in)])
    ref = np.zeros((n_in, 5))
    row_of = {int(x): i for i, x in enumerate(D.verts)}
    for v in range(n_in):
        for c in D.fwd_col[D.fwd_rowptr[v]:D.fwd_rowptr[v + 1]]:
            u = int(c) if c < n_in else row_of[int(D.halo_vertex[c - n_in])]
            ref[u] += G[v]
    np.testing.assert_allclose(T, ref, rtol=1e-12, atol=1e-12)
