"""Device-side data layout of the partitioned hot path (built once per run).

Partition slots are placed on devices in contiguous blocks (P/N per device;
N = 1 puts all P partitions on one B200, each with its own local cache
level, exactly as the reference simulates them, simulator.py:164-166).

Per device, every layer's activations live in one "extended row space"

    X_ext[l] = [ inner rows | halo staging rows | local-cache slab rows ]  x F_l

  inner rows    the device's partitions' owned vertices (partition-major,
                ascending id) -- what peers read over NVLink;
  staging rows  one per (partition, halo vertex) position, ascending id
                (the reference's lookup order, simulator.py:198);
  slab rows     the partitions' local cache levels (c_gpu[p] slots each);
  snap rows     one row per distinct halo vertex the device's SpMMs read: the
                epoch-1 activation of that vertex.  Any cache row whose
                version is <= 1 holds exactly that value (A2: version 0/1 ->
                the epoch-1 forward pass), whichever partition's level holds
                it, so such reads are served from one shared row instead of
                P per-partition copies (fewer distinct HBM rows per gather,
                no epoch-1 warm write-back, no host-tier traffic for them).

The forward CSR (in-edges of inner rows, + GCN self-loops) has column ids in
[0, n_in) for rows owned by the same partition and n_in + halo-position for
halo rows; the per-epoch ``halo_row`` table maps a halo position to the row
that holds the value to use (slab slot / staging row / co-resident owner
row).  The backward CSR (out-edges of inner rows) addresses the gradient
buffer [inner rows | remote-gradient staging rows] directly.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class DeviceLayout:
    device: int
    parts: list[int]
    n_in: int
    verts: np.ndarray            # inner vertex id per row
    part_of_row: np.ndarray
    hpos_off: dict               # partition -> first device-level halo position
    n_halo: int
    halo_vertex: np.ndarray      # vertex id per halo position
    slab_off: dict               # partition -> first slab row (absolute row id)
    n_slab: int
    n_rows: int                  # n_in + n_halo + n_slab
    fwd_rowptr: np.ndarray
    fwd_col: np.ndarray
    bwd_rowptr: np.ndarray
    bwd_col: np.ndarray
    bwd_stage_vertex: np.ndarray  # remote vertices whose gradient rows are pulled
    bwd_src_dev: np.ndarray
    bwd_src_row: np.ndarray
    needed: np.ndarray           # per halo position: read by the forward SpMM
    norm_src: np.ndarray         # GCN a_u per inner row (ones for SAGE)
    norm_dst: np.ndarray         # GCN b_v, SAGE 1/d_in(v) per inner row
    nnz_fwd: int = 0
    nnz_bwd: int = 0
    snap_off: int = 0            # first epoch-1 snapshot row (absolute)
    n_snap: int = 0
    snap_vertex: np.ndarray | None = None   # vertex id per snap row (ascending)
    snap_row_of_pos: np.ndarray | None = None  # per halo position: absolute snap row / -1
    snap_src_dev: np.ndarray | None = None  # owner device / row of each snap vertex
    snap_src_row: np.ndarray | None = None


@dataclass
class RunLayout:
    n: int
    P: int
    n_dev: int
    part_dev: np.ndarray
    parts_of: np.ndarray         # vertex -> partition slot
    row_of: np.ndarray           # vertex -> row on its owner device
    devices: list[DeviceLayout] = field(default_factory=list)
    union: np.ndarray | None = None
    # requester tables (halo-union major, reference lookup order)
    req_off: np.ndarray | None = None
    req_part: np.ndarray | None = None
    req_index: np.ndarray | None = None   # flat requester index (partition-major)
    req_dev: np.ndarray | None = None
    req_pos: np.ndarray | None = None     # device-level halo position
    req_needed: np.ndarray | None = None
    owner_dev: np.ndarray | None = None
    owner_row: np.ndarray | None = None
    halo_off: np.ndarray | None = None    # flat requester offsets per partition
    compact: bool = False                 # X_ext = [inner | snap] (no staging, no slabs)


def _gather_rows(off: np.ndarray, tgt: np.ndarray, rows: np.ndarray):
    """Concatenated neighbour lists of `rows` and the owning row index."""
    st = off[rows]
    ln = off[rows + 1] - st
    tot = int(ln.sum())
    owner = np.repeat(np.arange(rows.size), ln)
    base = np.repeat(st - np.concatenate(([0], np.cumsum(ln)[:-1])), ln)
    return tgt[base + np.arange(tot)], owner


def build_layout(g, inner, halo, c_gpu, n_dev: int, kind: str,
                 compact: bool = False) -> RunLayout:
    """compact: the plan provably never stages a row nor reads a slab slot
    (JACA, staleness -1, every local level holds its whole halo: all reads
    are version-0 local hits, served by the epoch-1 snapshot), so X_ext is
    [inner | snap] only -- for C4 12 GB instead of 86 GB per GPU."""
    n = int(g.n_vertices)
    P = len(inner)
    if n_dev < 1 or P % n_dev:
        raise ValueError(f"{P} partitions cannot be spread evenly over {n_dev} devices")
    per = P // n_dev
    part_dev = np.repeat(np.arange(n_dev), per).astype(np.int32)
    parts_of = np.empty(n, np.int32)
    for p in range(P):
        parts_of[inner[p]] = p
    row_of = np.empty(n, np.int32)
    in_off = np.asarray(g.in_offsets, np.int64)
    in_tgt = np.asarray(g.in_targets, np.int64)
    out_off = np.asarray(g.out_offsets, np.int64)
    out_tgt = np.asarray(g.out_targets, np.int64)
    din = np.diff(in_off)
    dout = np.diff(out_off)
    has_self = np.zeros(n, bool)
    src_all = np.repeat(np.arange(n), dout)
    has_self[src_all[src_all == out_tgt]] = True
    gcn = kind == "gcn"

    # rows on devices
    for d in range(n_dev):
        r = 0
        for p in range(d * per, (d + 1) * per):
            row_of[inner[p]] = np.arange(r, r + inner[p].size, dtype=np.int32)
            r += inner[p].size

    # halo membership per partition for pruning checks: sorted halo arrays
    layout = RunLayout(n=n, P=P, n_dev=n_dev, part_dev=part_dev, parts_of=parts_of,
                       row_of=row_of, compact=compact)
    for d in range(n_dev):
        plist = list(range(d * per, (d + 1) * per))
        verts = np.concatenate([inner[p] for p in plist]).astype(np.int64)
        n_in = verts.size
        part_of_row = np.concatenate([np.full(inner[p].size, p, np.int32) for p in plist])
        hpos_off, o = {}, 0
        for p in plist:
            hpos_off[p] = o
            o += halo[p].size
        n_halo = o
        halo_vertex = (np.concatenate([halo[p] for p in plist]).astype(np.int64)
                       if n_halo else np.zeros(0, np.int64))
        slab_off, o = {}, n_in + (0 if compact else n_halo)
        for p in plist:
            slab_off[p] = o
            o += 0 if compact else int(c_gpu[p])
        n_rows = o

        # ---- forward CSR: in-edges of inner rows (+ self loops for GCN)
        nb, owner = _gather_rows(in_off, in_tgt, verts)
        if gcn:
            need_sl = ~has_self[verts]
            nb = np.concatenate([nb, verts[need_sl]])
            owner = np.concatenate([owner, np.flatnonzero(need_sl)])
        order = np.lexsort((nb, owner))
        nb, owner = nb[order], owner[order]
        rp = part_of_row[owner]
        col = np.full(nb.size, -1, np.int64)
        same = parts_of[nb] == rp
        col[same] = row_of[nb[same]]
        needed = np.zeros(n_halo, bool)
        for p in plist:
            sel = np.flatnonzero((rp == p) & ~same)
            if sel.size == 0:
                continue
            h = halo[p]
            idx = np.searchsorted(h, nb[sel])
            ok = (idx < h.size) & (h[np.minimum(idx, max(h.size - 1, 0))] == nb[sel]) if h.size else np.zeros(sel.size, bool)
            col[sel[ok]] = n_in + hpos_off[p] + idx[ok]
            needed[hpos_off[p] + idx[ok]] = True
        # epoch-1 snapshot rows: the distinct halo vertices the SpMM reads
        snap_vertex = np.unique(halo_vertex[needed]) if n_halo else np.zeros(0, np.int64)
        snap_off = n_rows
        snap_row_of_pos = np.full(n_halo, -1, np.int64)
        if n_halo:
            nd = np.flatnonzero(needed)
            snap_row_of_pos[nd] = snap_off + np.searchsorted(snap_vertex, halo_vertex[nd])
        n_rows += snap_vertex.size
        keep = col >= 0   # edges from RAPA-pruned halo vertices are dropped
        col, owner = col[keep], owner[keep]
        fwd_rowptr = np.zeros(n_in + 1, np.int64)
        np.cumsum(np.bincount(owner, minlength=n_in), out=fwd_rowptr[1:])

        # ---- backward CSR: out-edges u->v of inner rows whose use was kept
        nb2, own2 = _gather_rows(out_off, out_tgt, verts)
        if gcn:
            need_sl = ~has_self[verts]
            nb2 = np.concatenate([nb2, verts[need_sl]])
            own2 = np.concatenate([own2, np.flatnonzero(need_sl)])
        order = np.lexsort((nb2, own2))
        nb2, own2 = nb2[order], own2[order]
        u = verts[own2]
        pv = parts_of[nb2]
        kept = pv == parts_of[u]
        cross = np.flatnonzero(~kept)
        if cross.size:
            # u must still be in the halo of v's partition (not pruned)
            for q in np.unique(pv[cross]):
                sel = cross[pv[cross] == q]
                h = halo[q]
                idx = np.searchsorted(h, u[sel])
                ok = (idx < h.size) & (h[np.minimum(idx, max(h.size - 1, 0))] == u[sel]) if h.size else np.zeros(sel.size, bool)
                kept[sel[ok]] = True
        nb2, own2 = nb2[kept], own2[kept]
        local_dev = part_dev[parts_of[nb2]] == d
        bcol = np.empty(nb2.size, np.int64)
        bcol[local_dev] = row_of[nb2[local_dev]]
        remote = np.unique(nb2[~local_dev])
        bcol[~local_dev] = n_in + np.searchsorted(remote, nb2[~local_dev])
        bwd_rowptr = np.zeros(n_in + 1, np.int64)
        np.cumsum(np.bincount(own2, minlength=n_in), out=bwd_rowptr[1:])

        if gcn:
            a = 1.0 / np.sqrt((dout + ~has_self).astype(np.float64))
            b = 1.0 / np.sqrt((din + ~has_self).astype(np.float64))
            norm_src = a[verts].astype(np.float32)
            norm_dst = b[verts].astype(np.float32)
        else:
            dv = din[verts].astype(np.float64)
            norm_src = np.ones(n_in, np.float32)
            norm_dst = np.where(dv > 0, 1.0 / np.maximum(dv, 1.0), 0.0).astype(np.float32)

        layout.devices.append(DeviceLayout(
            device=d, parts=plist, n_in=n_in, verts=verts, part_of_row=part_of_row,
            hpos_off=hpos_off, n_halo=n_halo, halo_vertex=halo_vertex, slab_off=slab_off,
            n_slab=n_rows - n_in - n_halo, n_rows=n_rows,
            fwd_rowptr=fwd_rowptr, fwd_col=col.astype(np.int32),
            bwd_rowptr=bwd_rowptr, bwd_col=bcol.astype(np.int32),
            bwd_stage_vertex=remote, bwd_src_dev=part_dev[parts_of[remote]].astype(np.int32),
            bwd_src_row=row_of[remote].astype(np.int32), needed=needed,
            norm_src=norm_src, norm_dst=norm_dst, nnz_fwd=int(col.size),
            snap_off=int(snap_off), n_snap=int(snap_vertex.size), snap_vertex=snap_vertex,
            snap_row_of_pos=snap_row_of_pos.astype(np.int32),
            snap_src_dev=part_dev[parts_of[snap_vertex]].astype(np.int32),
            snap_src_row=row_of[snap_vertex].astype(np.int32),
            nnz_bwd=int(bcol.size)))

    # ---- requester tables for the plan (halo-union major, lookup order)
    sizes = np.array([h.size for h in halo], np.int64)
    halo_off = np.zeros(P + 1, np.int64)
    halo_off[1:] = np.cumsum(sizes)
    layout.halo_off = halo_off
    if halo_off[-1] == 0:
        layout.union = np.zeros(0, np.int64)
        return layout
    allv = np.concatenate(halo).astype(np.int64)
    part = np.repeat(np.arange(P), sizes).astype(np.int32)
    pos = np.concatenate([np.arange(s) for s in sizes]).astype(np.int64)
    union = np.unique(allv)
    key = np.searchsorted(union, allv)
    order = np.lexsort((part, pos, key))  # by vertex, then (position, partition)
    layout.union = union
    layout.req_off = np.zeros(union.size + 1, np.int64)
    np.cumsum(np.bincount(key, minlength=union.size), out=layout.req_off[1:])
    layout.req_index = order.astype(np.int64)
    layout.req_part = part[order]
    layout.req_dev = part_dev[part[order]]
    hp_dev = np.empty(P, np.int64)
    needed_flat = np.zeros(allv.size, bool)
    for dl in layout.devices:
        for p in dl.parts:
            hp_dev[p] = dl.hpos_off[p]
            needed_flat[halo_off[p]:halo_off[p + 1]] = dl.needed[dl.hpos_off[p]:dl.hpos_off[p] + sizes[p]]
    layout.req_pos = (hp_dev[part[order]] + pos[order]).astype(np.int32)
    layout.req_needed = needed_flat[order].astype(np.uint8)
    layout.owner_dev = part_dev[parts_of[union]].astype(np.int32)
    layout.owner_row = row_of[union].astype(np.int32)
    return layout


def source_row_csrs(D, me: int):
    """The transform-first last layer's two static CSRs (compact layout, one
    process), for device layout D:

    * by SOURCE row of X_ext (inner row, or the epoch-1 snapshot row a halo
      position reads): the destination inner rows of its forward edges, in
      ascending order -- the transpose of the forward CSR after the layer's
      halo map, so A^T G per source row is one SpMM;
    * per inner row u: [u, the snapshot row of u] -- the owner sums the
      gradient of its own row and of its stale copy (A3).

    Returns (rowptr, col, u_rowptr, u_col), or None when some forward source
    has no snapshot row (not the compact plan)."""
    n_in = D.n_in
    fcol = np.asarray(D.fwd_col, np.int64)
    if D.n_halo:
        pos = np.maximum(fcol - n_in, 0)
        src = np.where(fcol < n_in, fcol, np.asarray(D.snap_row_of_pos, np.int64)[pos])
    else:
        src = fcol
    if (src < 0).any():
        return None
    dst = np.repeat(np.arange(n_in, dtype=np.int32), np.diff(np.asarray(D.fwd_rowptr)))
    order = np.argsort(src, kind="stable")     # by source row, then destination
    rp = np.zeros(D.n_rows + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=D.n_rows), out=rp[1:])
    snap_of = np.full(n_in, -1, np.int64)
    if D.n_snap:
        mine = np.asarray(D.snap_src_dev) == me
        snap_of[np.asarray(D.snap_src_row)[mine]] = D.snap_off + np.flatnonzero(mine)
    has = snap_of >= 0
    urp = np.zeros(n_in + 1, np.int64)
    np.cumsum(1 + has, out=urp[1:])
    ucol = np.empty(int(urp[-1]), np.int32)
    ucol[urp[:-1]] = np.arange(n_in)
    ucol[urp[:-1][has] + 1] = snap_of[has]
    return rp, dst[order], urp, ucol
