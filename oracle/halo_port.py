"""Integer half of the CPU oracle: a restatement of halopart's algorithms.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Every function names
the reference code it restates (paths relative to /root/reference/pkg).  The
restatement is written independently (different data structures: explicit
slot tables, a sorted-list importance index instead of a lazy heap, an exact
integer triangular decode) and pinned bit-for-bit against fixtures the
reference itself produced (tests/golden/make_golden.py).
"""

from __future__ import annotations

import math
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
from sortedcontainers import SortedList

LOCAL, GLOBAL, MISS = 0, 1, 2
OUTCOME_NAMES = ("local_hit", "global_hit", "miss")


# ---------------------------------------------------------------------------
# L1: graphs (src/halopart/synth.py:25-43, graph.py:24-129)


def triangular_decode(t: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
    """Pair index t in row-major order over {(u, v): u < v} -> (u, v).

    Restates synth.py:10-22 with an exact integer correction: row u starts
    at base(u) = u*(2n-u-1)/2; pick the largest u with base(u) <= t.
    """
    t = np.asarray(t, dtype=np.int64)
    est = np.floor(((2 * n - 1) - np.sqrt(np.maximum(
        (2.0 * n - 1) ** 2 - 8.0 * t.astype(np.float64), 0.0))) / 2.0)
    u = est.astype(np.int64)
    base = lambda x: x * (2 * n - x - 1) // 2  # noqa: E731
    for _ in range(4):  # float estimate is within one row; settle exactly
        u = np.where(base(u) > t, u - 1, u)
        u = np.where(base(u + 1) <= t, u + 1, u)
    v = t - base(u) + u + 1
    return u, v


def er_pairs(n: int, avg_degree: float, seed: int = 0):
    """Directed pair arrays of halopart.erdos_renyi (synth.py:25-43).

    The sampling itself is numpy's PCG64 stream, called exactly as the
    reference calls it (the RNG is third-party arithmetic, not restated).
    """
    total = n * (n - 1) // 2
    m = int(round(n * avg_degree / 2.0))
    rng = np.random.default_rng(seed)
    t = np.sort(rng.choice(total, size=m, replace=False).astype(np.int64))
    u, v = triangular_decode(t, n)
    return np.concatenate([u, v]), np.concatenate([v, u])


@dataclass
class GraphCSR:
    """Both adjacency directions, rows sorted ascending, no duplicates."""

    n: int
    n_edges: int
    out_off: np.ndarray
    out_tgt: np.ndarray
    in_off: np.ndarray
    in_tgt: np.ndarray

    @property
    def out_deg(self) -> np.ndarray:
        return np.diff(self.out_off)

    @property
    def in_deg(self) -> np.ndarray:
        return np.diff(self.in_off)

    def edges(self):
        """(src, dst) sorted by (src, dst) -- graph.py:114-117."""
        return np.repeat(np.arange(self.n, dtype=np.int64), self.out_deg), self.out_tgt


def _rows(keys: np.ndarray, vals: np.ndarray, n: int):
    order = np.lexsort((vals, keys))
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(keys, minlength=n), out=off[1:])
    return off, vals[order].astype(np.int64)


def graph_from_pairs(src, dst, n: int) -> GraphCSR:
    """Graph.from_pair_arrays (graph.py:69-84): dedup, then CSR both ways."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if n > 0 and src.size:
        code = np.unique(src * n + dst)
        src, dst = code // n, code % n
    oo, ot = _rows(src, dst, n)
    io_, it = _rows(dst, src, n)
    return GraphCSR(n=n, n_edges=int(src.size), out_off=oo, out_tgt=ot,
                    in_off=io_, in_tgt=it)


def er_graph(n: int, avg_degree: float, seed: int = 0) -> GraphCSR:
    s, d = er_pairs(n, avg_degree, seed)
    return graph_from_pairs(s, d, n)


def random_assignment(n: int, P: int, seed: int = 0) -> np.ndarray:
    """prepartition(..., "random") (partitioner.py:265-274)."""
    order = np.random.default_rng(seed).permutation(n)
    sizes = [n // P + (1 if i < n % P else 0) for i in range(P)]
    parts = np.empty(n, dtype=np.int64)
    start = 0
    for i, sz in enumerate(sizes):
        parts[order[start:start + sz]] = i
        start += sz
    return parts


# ---------------------------------------------------------------------------
# halos and partition statistics (graph.py:203-228, 298-335)


def undirected_adjacency(g: GraphCSR) -> list[np.ndarray]:
    s, d = g.edges()
    u = np.concatenate([s, d])
    w = np.concatenate([d, s])
    off, tgt = _rows(u, w, g.n)
    return [np.unique(tgt[off[v]:off[v + 1]]) for v in range(g.n)]


def khop_halo(adj: list[np.ndarray], inner: np.ndarray, hops: int) -> np.ndarray:
    """Vertices outside `inner` within `hops` undirected steps (BFS)."""
    seen = np.zeros(len(adj), dtype=bool)
    seen[inner] = True
    frontier = np.asarray(inner, dtype=np.int64)
    for _ in range(hops):
        if frontier.size == 0:
            break
        nb = np.concatenate([adj[v] for v in frontier]) if frontier.size else frontier
        nb = np.unique(nb)
        fresh = nb[~seen[nb]]
        seen[fresh] = True
        frontier = fresh
    seen[inner] = False
    return np.flatnonzero(seen).astype(np.int64)


@dataclass
class Partitions:
    n: int
    P: int
    parts: np.ndarray
    inner: list[np.ndarray]
    halo: list[np.ndarray]
    hops: int
    overlap: np.ndarray
    cut: list[int]
    all_edges: list[int]

    def halo_union(self) -> np.ndarray:
        if not any(h.size for h in self.halo):
            return np.empty(0, dtype=np.int64)
        return np.unique(np.concatenate(self.halo))


def partition_set(g: GraphCSR, parts: np.ndarray, hops: int,
                  adj: list[np.ndarray] | None = None) -> Partitions:
    parts = np.asarray(parts, dtype=np.int64)
    P = int(parts.max()) + 1
    adj = adj if adj is not None else undirected_adjacency(g)
    inner = [np.flatnonzero(parts == i).astype(np.int64) for i in range(P)]
    halo = [khop_halo(adj, inner[i], hops) for i in range(P)]
    overlap = np.zeros(g.n, dtype=np.int64)
    for h in halo:
        overlap[h] += 1
    s, d = g.edges()
    cut, alle = [], []
    for i in range(P):
        a, b = parts[s] == i, parts[d] == i
        cut.append(int(np.count_nonzero(a != b)))
        mem = np.zeros(g.n, dtype=bool)
        mem[inner[i]] = True
        mem[halo[i]] = True
        alle.append(int(np.count_nonzero(mem[s] & mem[d])))
    return Partitions(n=g.n, P=P, parts=parts, inner=inner, halo=halo,
                      hops=hops, overlap=overlap, cut=cut, all_edges=alle)


def influence(g: GraphCSR, ps: Partitions):
    """influence_scores (partitioner.py:324-345); float64, bincount order.

    Returns (vertices, out_term, in_term, score) over the halo union.
    """
    s, d = g.edges()
    od = g.out_deg.astype(np.float64)
    idg = g.in_deg.astype(np.float64)
    den = od[s] * idg[d]
    w = np.zeros_like(den)
    nz = den > 0
    w[nz] = 1.0 / np.sqrt(den[nz])
    out_all = np.bincount(s, weights=w, minlength=g.n)
    in_all = np.bincount(d, weights=w, minlength=g.n)
    verts = ps.halo_union()
    ot, it = out_all[verts], in_all[verts]
    return verts, ot, it, (ot + it) * ps.overlap[verts].astype(np.float64)


def ranked_halos(ps: Partitions, verts: np.ndarray, score: np.ndarray):
    """Per-partition halo sorted by (-score, id) -- simulator.py:187-191."""
    out = []
    for h in ps.halo:
        sc = score[np.searchsorted(verts, h)]
        out.append(h[np.lexsort((h, -sc))])
    return out


# ---------------------------------------------------------------------------
# Algorithm 1 (cache.py:54-115)


def entry_budget(mem_gib: float, res_mib: float, bpe: int) -> int:
    b = (mem_gib * 1024.0 - res_mib) * (1024.0 * 1024.0)
    return 0 if b < 0 else int(b // bpe)


def capacities_auto(ps: Partitions, k: int, mem_gpu, mem_gpu_res, mem_cpu,
                    mem_cpu_res, f_dim) -> tuple[int, tuple[int, ...], int]:
    bpe = sum(int(f) * 4 for f in f_dim)
    sel = []
    for h in ps.halo:
        o = h[np.lexsort((h, -ps.overlap[h]))]
        sel.append(o if k == -1 else o[:k])
    c_gpu = tuple(min(entry_budget(mem_gpu[i], mem_gpu_res, bpe), s.size)
                  for i, s in enumerate(sel))
    uni = np.unique(np.concatenate(sel)) if any(s.size for s in sel) else np.empty(0)
    return min(entry_budget(mem_cpu, mem_cpu_res, bpe), int(uni.size)), c_gpu, bpe


def capacities_uniform(ps: Partitions, c: int, f_dim):
    bpe = sum(int(f) * 4 for f in f_dim)
    return (min(c, int(ps.halo_union().size)),
            tuple(min(c, int(h.size)) for h in ps.halo), bpe)


# ---------------------------------------------------------------------------
# the two-level cache (cache.py:137-347), restated with explicit slots


class Level:
    """One level: vertex -> [slot, version]; policy order in an OrderedDict.

    Slots are an oracle-side addition (the reference stores no data): a new
    entry takes its victim's slot, else the lowest never-used slot.
    """

    def __init__(self, policy: str, capacity: int, score: dict | None):
        self.policy, self.capacity = policy, capacity
        self.score = score or {}
        self.ent: OrderedDict[int, list[int]] = OrderedDict()
        self.by_score = SortedList()
        self.next_slot = 0

    def sc(self, v: int) -> float:
        return float(self.score.get(v, 0.0))

    def touch(self, v: int) -> None:
        if self.policy == "lru":
            self.ent.move_to_end(v)

    def refresh(self, v: int, ver: int) -> None:
        self.ent[v][1] = ver
        self.touch(v)

    def insert(self, v: int, ver: int):
        """Returns the evicted vertex, or None (also when rejected)."""
        if v in self.ent:
            self.refresh(v, ver)
            return None
        if self.capacity == 0:
            return None
        victim = None
        if len(self.ent) >= self.capacity:
            if self.policy in ("fifo", "lru"):
                victim = next(iter(self.ent))
            else:
                low_score, low_v = self.by_score[0]
                if self.sc(v) <= low_score:
                    return None
                victim = low_v
            slot = self.ent.pop(victim)[0]
            if self.policy == "jaca":
                self.by_score.remove((self.sc(victim), victim))
        else:
            slot = self.next_slot
            self.next_slot += 1
        self.ent[v] = [slot, ver]
        if self.policy == "jaca":
            self.by_score.add((self.sc(v), v))
        return victim


def fresh(ver: int, epoch: int, s: int) -> bool:
    return s < 0 or epoch - ver <= s


class TwoLevel:
    """CacheSystem restated (lookup: cache.py:264-309; warm: :323-347)."""

    def __init__(self, policy: str, c_cpu: int, c_gpu, score: dict | None):
        self.policy = policy
        self.loc = [Level(policy, c, score) for c in c_gpu]
        self.glo = Level(policy, c_cpu, score)
        P = len(c_gpu)
        self.counts = np.zeros((P, 3), dtype=np.int64)

    def warm(self, ranked) -> None:
        for d, lst in enumerate(ranked):
            for v in list(lst)[: self.loc[d].capacity]:
                self.loc[d].insert(int(v), 0)
        seen, merged = set(), []
        for pos in range(max((len(x) for x in ranked), default=0)):
            for lst in ranked:
                if pos < len(lst) and int(lst[pos]) not in seen:
                    seen.add(int(lst[pos]))
                    merged.append(int(lst[pos]))
        for v in merged[: self.glo.capacity]:
            self.glo.insert(v, 0)

    def lookup(self, d: int, v: int, e: int, s: int) -> tuple[int, int]:
        """-> (outcome, version of the data served)."""
        L = self.loc[d]
        le = L.ent.get(v)
        if le is not None and fresh(le[1], e, s):
            L.touch(v)
            self.counts[d, LOCAL] += 1
            return LOCAL, le[1]
        ge = self.glo.ent.get(v)
        if ge is not None and fresh(ge[1], e, s):
            self.glo.touch(v)
            gv = ge[1]
            if le is not None:
                L.refresh(v, gv)
            else:
                L.insert(v, gv)
            self.counts[d, GLOBAL] += 1
            return GLOBAL, gv
        if ge is not None:
            self.glo.refresh(v, e)
        else:
            self.glo.insert(v, e)
        if le is not None:
            L.refresh(v, e)
        else:
            L.insert(v, e)
        self.counts[d, MISS] += 1
        return MISS, e


@dataclass
class EpochPlan:
    """Outcome and served version per (device, halo position)."""

    epoch: int
    outcome: list[np.ndarray]
    version: list[np.ndarray]
    counts: np.ndarray  # (P, 3): local, global, miss


@dataclass
class PlanRun:
    cache: TwoLevel
    plans: list[EpochPlan] = field(default_factory=list)

    def trace_csv(self, halo) -> str:
        """Rows in lookup order, as CacheSystem.write_trace_csv (:371-382)."""
        lines = ["epoch,device,vertex,outcome,level"]
        tag = ("hit,local", "hit,global", "miss,source")
        for p in self.plans:
            for r in range(max(len(h) for h in halo)):
                for d, h in enumerate(halo):
                    if r < len(h):
                        lines.append(f"{p.epoch},{d},{int(h[r])},{tag[p.outcome[d][r]]}")
        return "\n".join(lines) + "\n"


class Planner:
    """Stepwise form of simulator.run's lookup loop (simulator.py:185-226)."""

    def __init__(self, policy: str, caps, ranked, halo, score: dict):
        self.cache = TwoLevel(policy, caps[0], caps[1], score)
        self.cache.warm(ranked)
        self.halo = halo
        self.run = PlanRun(cache=self.cache)

    def step(self, e: int, staleness: int) -> EpochPlan:
        halo, cache = self.halo, self.cache
        P = len(halo)
        longest = max((len(h) for h in halo), default=0)
        oc = [np.empty(len(h), dtype=np.int8) for h in halo]
        vs = [np.empty(len(h), dtype=np.int64) for h in halo]
        before = cache.counts.copy()
        for r in range(longest):
            for d in range(P):
                if r < len(halo[d]):
                    o, ver = cache.lookup(d, int(halo[d][r]), e, staleness)
                    oc[d][r] = o
                    vs[d][r] = ver
        plan = EpochPlan(epoch=e, outcome=oc, version=vs, counts=cache.counts - before)
        self.run.plans.append(plan)
        return plan


def plan_epochs(policy: str, caps, ranked, halo, score: dict, epochs: int,
                staleness: int) -> PlanRun:
    """All epochs of simulator.run's lookup loop, round-robin order."""
    pl = Planner(policy, caps, ranked, halo, score)
    for e in range(1, epochs + 1):
        pl.step(e, staleness)
    return pl.run


# ---------------------------------------------------------------------------
# cost model records (devices.py:73-132; simulator.py:199-256)


def normalized(profiles):
    """profiles: list of dicts with mm_s, spmm_s, h2d_s, d2h_s, idt_s."""
    keys = ("mm_s", "spmm_s", "h2d_s", "d2h_s", "idt_s")
    worst = {k: max(p[k] for p in profiles) for k in keys}
    return [{k: p[k] / worst[k] for k in keys} for p in profiles]


def records(ps: Partitions, sigma, profiles, run: PlanRun, bpe: int,
            alpha: float, prefetch: int, unit_time: float):
    """Per-(epoch, device) record dicts plus makespans (simulator.py:228-256)."""
    nrm = normalized(profiles)
    P = ps.P
    mix = []
    for i in range(P):
        r = nrm[sigma[i]]
        direct = 1.0 / P
        mix.append((r["h2d_s"] + r["d2h_s"]) * (1.0 - direct) + r["idt_s"] * direct)
    comp = [(alpha * ps.all_edges[i] * nrm[sigma[i]]["spmm_s"]
             + (1.0 - alpha) * ps.inner[i].size * nrm[sigma[i]]["mm_s"]) * unit_time
            for i in range(P)]
    recs, spans = [], []
    for p in run.plans:
        dts = []
        for i in range(P):
            lh, gh, ms = (int(x) for x in p.counts[i])
            comm = (ms + ps.cut[i]) * mix[i] * unit_time
            ov = min(1.0, prefetch / max(1, ps.halo[i].size))
            resid = comm - min(comm, comp[i]) * ov
            dt = comp[i] + resid
            dts.append(dt)
            recs.append(dict(epoch=p.epoch, device=i, fwd_bytes=ms * bpe,
                             bwd_bytes=ps.cut[i] * bpe, local_hits=lh,
                             global_hits=gh, misses=ms, compute_time=comp[i],
                             comm_time=comm, residual_comm_time=resid,
                             device_time=dt))
        spans.append(max(dts))
    return recs, spans


def lookup_counts_total(run: PlanRun) -> int:
    return int(sum(int(p.counts.sum()) for p in run.plans))


def isclose_exact(a: float, b: float) -> bool:
    return a == b or (math.isnan(a) and math.isnan(b))
