"""Host-side graph / partition inputs of the hot path, halopart-compatible.

The drop-in boundary accepts halopart's own objects (duck-typed on the field
names of halopart.Graph / PartitionSet / RapaResult / CacheCapacities /
SimConfig / DeviceProfile).  This module provides objects with the SAME field
names and semantics so the path also runs where halopart is not installed
(e.g. the GPU box), built by the native preprocessing in libcapgnn.so
(csrc/graph_host.cpp), bit-identical to the reference:

  Graph.from_pair_arrays  graph.py:69-84      -> graph_from_pairs
  erdos_renyi             synth.py:25-43      -> erdos_renyi
  prepartition("random")  partitioner.py:265  -> random_partition
  build_partition_set     graph.py:298-335    -> build_partition_set
  influence_scores        partitioner.py:324  -> influence_scores
  compute_capacities      cache.py:70-105     -> compute_capacities
  uniform_capacities      cache.py:108-115    -> uniform_capacities
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import call, ptr
from .errors import DomainError


@dataclass(eq=False)
class Graph:
    n_vertices: int
    n_edges: int
    out_offsets: np.ndarray
    out_targets: np.ndarray
    in_offsets: np.ndarray
    in_targets: np.ndarray
    vertex_id_map: dict | None = None

    @property
    def out_degrees(self) -> np.ndarray:
        return np.diff(self.out_offsets)

    @property
    def in_degrees(self) -> np.ndarray:
        return np.diff(self.in_offsets)


def graph_from_pairs(src, dst, n: int) -> Graph:
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    m = src.size
    oo = np.empty(n + 1, np.int64)
    io = np.empty(n + 1, np.int64)
    ot = np.empty(max(m, 1), np.int64)
    it = np.empty(max(m, 1), np.int64)
    ne = C.c_int64(0)
    try:
        call("cg_csr_from_pairs", n, m, ptr(src), ptr(dst), ptr(oo), ptr(ot), ptr(io),
             ptr(it), C.addressof(ne))
    except RuntimeError as exc:
        raise DomainError(str(exc).split(": ", 1)[-1]) from None
    E = ne.value
    return Graph(n_vertices=n, n_edges=E, out_offsets=oo, out_targets=ot[:E].copy(),
                 in_offsets=io, in_targets=it[:E].copy())


def _pair_decode(t: np.ndarray, n: int):
    # row u of the strict upper triangle starts at u*(2n-u-1)/2
    r = (2.0 * n - 1.0)
    u = np.floor((r - np.sqrt(np.maximum(r * r - 8.0 * t, 0.0))) / 2.0).astype(np.int64)
    row_start = lambda x: x * (2 * n - x - 1) // 2  # noqa: E731
    for _ in range(3):  # settle the float estimate exactly
        u = u - (row_start(u) > t)
        u = u + (row_start(u + 1) <= t)
    v = t - row_start(u) + u + 1
    return u, v


def erdos_renyi(n: int, avg_degree: float, seed: int = 0) -> Graph:
    """Seeded symmetric ER graph; the pair sample is numpy's own PCG64 draw."""
    if n < 2:
        raise DomainError("need at least two vertices")
    total = n * (n - 1) // 2
    m = int(round(n * avg_degree / 2.0))
    if not 0 <= m <= total:
        raise DomainError(f"avg_degree {avg_degree} asks for {m} of {total} possible edges")
    t = np.sort(np.random.default_rng(seed).choice(total, size=m, replace=False).astype(np.int64))
    u, v = _pair_decode(t, n)
    return graph_from_pairs(np.concatenate([u, v]), np.concatenate([v, u]), n)


def random_partition(n: int, P: int, seed: int = 0) -> np.ndarray:
    if not 1 <= P <= n:
        raise DomainError(f"P must lie in 1..{n}, got {P}")
    order = np.random.default_rng(seed).permutation(n)
    bounds = np.cumsum([0] + [n // P + (i < n % P) for i in range(P)])
    parts = np.empty(n, np.int64)
    for i in range(P):
        parts[order[bounds[i]:bounds[i + 1]]] = i
    return parts


@dataclass(eq=False)
class PartitionSet:
    n_vertices: int
    P: int
    inner: list
    halo: list
    hops: int
    overlap_count: np.ndarray
    cut_edges: list
    all_edges: list
    graph: Graph | None = field(default=None, repr=False)

    @property
    def inner_sizes(self) -> list[int]:
        return [int(a.size) for a in self.inner]

    @property
    def halo_sizes(self) -> list[int]:
        return [int(a.size) for a in self.halo]

    def halo_union(self) -> np.ndarray:
        if not any(h.size for h in self.halo):
            return np.empty(0, np.int64)
        return np.unique(np.concatenate(self.halo))


def undirected(g) -> tuple[np.ndarray, np.ndarray]:
    n = g.n_vertices
    oo, ot = np.ascontiguousarray(g.out_offsets, np.int64), np.ascontiguousarray(g.out_targets, np.int64)
    io, it = np.ascontiguousarray(g.in_offsets, np.int64), np.ascontiguousarray(g.in_targets, np.int64)
    uo = np.empty(n + 1, np.int64)
    ut = np.empty(max(1, ot.size + it.size), np.int64)
    call("cg_undirected_csr", n, ptr(oo), ptr(ot), ptr(io), ptr(it), ptr(uo), ptr(ut))
    return uo, ut[:uo[-1]].copy()


def build_partition_set(g, assignment, hops: int) -> PartitionSet:
    parts = np.asarray(getattr(assignment, "parts", assignment), dtype=np.int64)
    n = g.n_vertices
    if parts.shape != (n,):
        raise DomainError(f"assignment covers {parts.size} vertices, graph has {n}")
    if hops < 1:
        raise DomainError(f"hops must be >= 1, got {hops}")
    P = int(parts.max(initial=-1)) + 1
    if parts.min(initial=0) < 0 or np.unique(parts).size != P:
        raise DomainError("partition ids must be exactly 0..P-1")
    p32 = parts.astype(np.int32)
    uo, ut = undirected(g)
    inner = [np.flatnonzero(parts == i).astype(np.int64) for i in range(P)]
    halo = []
    buf = np.empty(n, np.int32)
    cnt = C.c_int64(0)
    for i in range(P):
        call("cg_khop_halo", n, ptr(uo), ptr(ut), ptr(p32), i, hops, ptr(buf), C.addressof(cnt))
        halo.append(buf[:cnt.value].astype(np.int64))
    overlap = np.zeros(n, np.int64)
    for h in halo:
        overlap[h] += 1
    hoff = np.zeros(P + 1, np.int64)
    hoff[1:] = np.cumsum([h.size for h in halo])
    hcat = (np.concatenate(halo) if hoff[-1] else np.zeros(1, np.int64)).astype(np.int32)
    cut = np.zeros(P, np.int64)
    alle = np.zeros(P, np.int64)
    oo = np.ascontiguousarray(g.out_offsets, np.int64)
    ot = np.ascontiguousarray(g.out_targets, np.int64)
    call("cg_partition_stats", n, ptr(oo), ptr(ot), ptr(p32), P, ptr(hoff), ptr(hcat),
         ptr(cut), ptr(alle))
    return PartitionSet(n_vertices=n, P=P, inner=inner, halo=halo, hops=hops,
                        overlap_count=overlap, cut_edges=[int(c) for c in cut],
                        all_edges=[int(a) for a in alle], graph=g)


def influence_scores(g, ps) -> tuple[np.ndarray, np.ndarray]:
    """(halo-union vertices, fp64 scores) -- bit-identical to the reference."""
    n = g.n_vertices
    ot_all = np.empty(n, np.float64)
    it_all = np.empty(n, np.float64)
    call("cg_influence_terms", n, ptr(np.ascontiguousarray(g.out_offsets, np.int64)),
         ptr(np.ascontiguousarray(g.out_targets, np.int64)),
         ptr(np.ascontiguousarray(g.in_offsets, np.int64)),
         ptr(np.ascontiguousarray(g.in_targets, np.int64)), ptr(ot_all), ptr(it_all))
    verts = ps.halo_union()
    score = (ot_all[verts] + it_all[verts]) * ps.overlap_count[verts].astype(np.float64)
    return verts, score


# ---------------------------------------------------------------------------
# capacities / config records (field-compatible with halopart)


@dataclass(frozen=True)
class CacheCapacities:
    c_cpu: int
    c_gpu: tuple
    bytes_per_entry: int

    def __post_init__(self):
        if self.c_cpu < 0 or any(c < 0 for c in self.c_gpu):
            raise DomainError("capacities must be >= 0")
        if self.bytes_per_entry <= 0:
            raise DomainError("bytes_per_entry must be positive")


def feature_bytes(f_dim) -> int:
    if not f_dim or any(int(d) < 1 for d in f_dim):
        raise DomainError("f_dim must be a nonempty list of positive widths")
    return 4 * sum(int(d) for d in f_dim)


def _budget(mem_gib: float, res_mib: float, bpe: int) -> int:
    avail = (mem_gib * 1024.0 - res_mib) * 1048576.0
    return 0 if avail < 0 else int(avail // bpe)


def compute_capacities(ps, k: int, mem_gpu, mem_gpu_res: float, mem_cpu: float,
                       mem_cpu_res: float, f_dim, L: int) -> CacheCapacities:
    """Algorithm 1: budgets capped by overlap-ranked demand."""
    if L < 1 or len(f_dim) != L:
        raise DomainError(f"f_dim has {len(f_dim)} entries, expected L={L}")
    if len(mem_gpu) != ps.P:
        raise DomainError(f"{len(mem_gpu)} device budgets for {ps.P} partitions")
    if k < -1:
        raise DomainError("k must be -1 (all) or >= 0")
    bpe = feature_bytes(f_dim)
    chosen = []
    for h in ps.halo:
        ranked = h[np.lexsort((h, -ps.overlap_count[h]))]
        chosen.append(ranked if k == -1 else ranked[:k])
    c_gpu = tuple(min(_budget(mem_gpu[i], mem_gpu_res, bpe), int(s.size))
                  for i, s in enumerate(chosen))
    n_union = int(np.unique(np.concatenate(chosen)).size) if any(s.size for s in chosen) else 0
    return CacheCapacities(c_cpu=min(_budget(mem_cpu, mem_cpu_res, bpe), n_union),
                           c_gpu=c_gpu, bytes_per_entry=bpe)


def uniform_capacities(ps, c: int, f_dim) -> CacheCapacities:
    if c < 0:
        raise DomainError("capacity must be >= 0")
    return CacheCapacities(c_cpu=min(c, int(ps.halo_union().size)),
                           c_gpu=tuple(min(c, int(h.size)) for h in ps.halo),
                           bytes_per_entry=feature_bytes(f_dim))


@dataclass(frozen=True)
class SimConfig:
    epochs: int = 200
    alpha: float = 0.5
    staleness_bound: int = -1
    prefetch_depth: int = 0
    policy: str = "jaca"
    f_dim: tuple = (256, 256, 256)
    L: int = 3
    seed: int = 0
    unit_time: float = 1.0

    def __post_init__(self):
        if self.epochs < 1:
            raise DomainError("epochs must be >= 1")
        if self.prefetch_depth < 0:
            raise DomainError("prefetch_depth must be >= 0")
        if not 0.0 <= self.alpha <= 1.0:
            raise DomainError("alpha must lie in [0, 1]")
        if self.policy not in ("jaca", "fifo", "lru"):
            raise DomainError(f"unknown policy {self.policy!r}")
        if self.L != len(self.f_dim):
            raise DomainError(f"L={self.L} but f_dim has {len(self.f_dim)} entries")
        if self.unit_time <= 0:
            raise DomainError("unit_time must be positive")

    def to_dict(self) -> dict:
        return {"epochs": self.epochs, "alpha": self.alpha,
                "staleness_bound": self.staleness_bound,
                "prefetch_depth": self.prefetch_depth, "policy": self.policy,
                "f_dim": list(self.f_dim), "L": self.L, "seed": self.seed,
                "unit_time": self.unit_time}


@dataclass(frozen=True)
class DeviceProfile:
    id: str
    mm_s: float
    spmm_s: float
    h2d_s: float
    d2h_s: float
    idt_s: float
    mem_gb: float


def unit_profiles(P: int, mem_gb: float = 180.0) -> list[DeviceProfile]:
    return [DeviceProfile(f"b200-{i}", 1.0, 1.0, 1.0, 1.0, 1.0, mem_gb) for i in range(P)]
