"""Cache planning: which tier serves every (partition, halo vertex) lookup.

``SequentialPlanner`` wraps the native exact planner (csrc/planner.cpp), the
replacement for halopart's CacheSystem + simulator.run lookup loop
(cache.py:227-347, simulator.py:206-226).  ``HaloCache`` exposes the
CacheSystem operator API (lookup / warm / admit_evict / counters / trace) on
top of it for callers that drive lookups one at a time.
"""

from __future__ import annotations

import ctypes as C
import csv
import io
from dataclasses import dataclass

import numpy as np

from ._lib import call, ptr
from .errors import DomainError

POLICIES = ("jaca", "fifo", "lru")
OUTCOMES = ("local_hit", "global_hit", "miss")


@dataclass
class EpochPlan:
    epoch: int
    outcome: np.ndarray      # int8 per requester (partition-major, halo order)
    version: np.ndarray      # int32 served version
    hit_slot: np.ndarray     # int32 local slot read on a local hit, else -1
    slot_after: np.ndarray   # int32 local slot held after the lookup, else -1
    lslot_pos: np.ndarray    # per local slot: final occupant halo position / -1
    lslot_dirty: np.ndarray  # per local slot: content changed this epoch
    gslot_vertex: np.ndarray  # per global slot: final union index / -1
    gslot_dirty: np.ndarray
    counts: np.ndarray       # (P, 3) local, global, miss

    def outcomes_of(self, halo_off: np.ndarray, p: int) -> np.ndarray:
        return self.outcome[halo_off[p]:halo_off[p + 1]]


class SequentialPlanner:
    """Exact two-level planner over one run's halos (keys = halo-union index)."""

    def __init__(self, policy: str, c_cpu: int, c_gpu, union: np.ndarray,
                 score: np.ndarray, halos, ranked):
        if policy not in POLICIES:
            raise DomainError(f"unknown policy {policy!r}; expected one of {POLICIES}")
        self.policy = policy
        self.P = len(halos)
        self.union = np.ascontiguousarray(union, np.int64)
        self.c_cpu = int(c_cpu)
        self.c_gpu = np.ascontiguousarray(c_gpu, np.int64)
        self.lslot_off = np.zeros(self.P + 1, np.int64)
        self.lslot_off[1:] = np.cumsum(self.c_gpu)
        self._score = np.ascontiguousarray(score, np.float64)
        h = C.c_void_p()
        call("cg_planner_create", POLICIES.index(policy), self.P, self.c_cpu, ptr(self.c_gpu),
             self.union.size, ptr(self._score), C.addressof(h))
        self._h = h
        self.halo_off = np.zeros(self.P + 1, np.int64)
        self.halo_off[1:] = np.cumsum([len(x) for x in halos])
        self.halo_keys = np.ascontiguousarray(
            np.searchsorted(self.union, np.concatenate(halos)) if self.halo_off[-1] else
            np.zeros(0), np.int32)
        rk = np.ascontiguousarray(
            np.searchsorted(self.union, np.concatenate(ranked)) if self.halo_off[-1] else
            np.zeros(0), np.int32)
        call("cg_planner_set_halos", self._h, ptr(self.halo_off), ptr(self.halo_keys), ptr(rk))
        self.n_req = int(self.halo_off[-1])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                call("cg_planner_destroy", h)
            except Exception:  # noqa: BLE001
                pass

    def warm(self) -> None:
        call("cg_planner_warm", self._h)

    def epoch(self, e: int, staleness: int) -> EpochPlan:
        n, P = self.n_req, self.P
        oc = np.empty(max(n, 1), np.int8)
        ver = np.empty(max(n, 1), np.int32)
        hs = np.empty(max(n, 1), np.int32)
        sa = np.empty(max(n, 1), np.int32)
        nl = int(self.lslot_off[-1])
        lp = np.empty(max(nl, 1), np.int32)
        ld = np.empty(max(nl, 1), np.uint8)
        gv = np.empty(max(self.c_cpu, 1), np.int32)
        gd = np.empty(max(self.c_cpu, 1), np.uint8)
        cnt = np.zeros((P, 3), np.int64)
        call("cg_planner_epoch", self._h, e, staleness, ptr(oc), ptr(ver), ptr(hs), ptr(sa),
             ptr(lp), ptr(ld), ptr(gv), ptr(gd), ptr(cnt))
        self._last_outcome = oc[:n]
        return EpochPlan(e, oc[:n], ver[:n], hs[:n], sa[:n], lp[:nl], ld[:nl],
                         gv[:self.c_cpu], gd[:self.c_cpu], cnt)

    def state(self) -> dict:
        n, P = self.n_req, self.P
        rs = np.empty(max(n, 1), np.int32)
        rv = np.empty(max(n, 1), np.int32)
        gs = np.empty(max(self.union.size, 1), np.int32)
        gv = np.empty(max(self.c_cpu, 1), np.int32)
        adm = C.c_int32(0)
        lf = np.empty(P, np.int32)
        lm = np.empty(P, np.float64)
        gf = C.c_int32(0)
        gm = C.c_double(0)
        call("cg_planner_state", self._h, ptr(rs), ptr(rv), ptr(gs), ptr(gv), C.addressof(adm),
             ptr(lf), ptr(lm), C.addressof(gf), C.addressof(gm))
        return dict(req_slot=rs[:n], req_ver=rv[:n], gslot=gs[:self.union.size],
                    glob_ver=gv[:self.c_cpu], admissions=adm.value, lfree=lf, lmin=lm,
                    gfree=gf.value, gmin=gm.value)

    def trace_rows(self, plan: EpochPlan):
        """(epoch, partition, vertex, outcome) in the reference's lookup order."""
        sizes = np.diff(self.halo_off)
        longest = int(sizes.max(initial=0))
        r = np.arange(longest)
        rows = []
        for rr in r:
            for p in range(self.P):
                if rr < sizes[p]:
                    i = self.halo_off[p] + rr
                    rows.append((plan.epoch, p, int(self.union[self.halo_keys[i]]),
                                 int(plan.outcome[i])))
        return rows


def trace_csv(rows) -> str:
    """CacheSystem.write_trace_csv layout (cache.py:371-382)."""
    tag = (("hit", "local"), ("hit", "global"), ("miss", "source"))
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["epoch", "device", "vertex", "outcome", "level"])
    for e, d, v, o in rows:
        w.writerow([e, d, v, *tag[o]])
    return buf.getvalue()


class HaloCache:
    """CacheSystem-compatible operator (cache.py:227-382) on the native planner.

    Vertices are raw ids in [0, n_keys); ``importance`` maps id -> score.
    """

    def __init__(self, policy: str, caps, importance=None, record_trace: bool = False,
                 n_keys: int | None = None):
        if policy not in POLICIES:
            raise DomainError(f"unknown policy {policy!r}; expected one of {POLICIES}")
        imp = dict(importance or {})
        if n_keys is None:
            n_keys = max([1 << 16] + [int(v) + 1 for v in imp])
        self.n_keys = n_keys
        self.policy = policy
        self.caps = caps
        self.P = len(caps.c_gpu)
        score = np.zeros(n_keys, np.float64)
        for v, s in imp.items():
            score[int(v)] = float(s)
        self._score = score
        c_gpu = np.ascontiguousarray(caps.c_gpu, np.int64)
        h = C.c_void_p()
        call("cg_planner_create", POLICIES.index(policy), self.P, int(caps.c_cpu), ptr(c_gpu),
             n_keys, ptr(score), C.addressof(h))
        self._h = h
        self.trace = [] if record_trace else None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                call("cg_planner_destroy", h)
            except Exception:  # noqa: BLE001
                pass

    @property
    def n_devices(self) -> int:
        return self.P

    def _key(self, v) -> int:
        v = int(v)
        if not 0 <= v < self.n_keys:
            raise DomainError(f"vertex {v} outside the operator's key space")
        return v

    def lookup(self, device: int, vertex: int, epoch: int, staleness_bound: int = 0) -> str:
        if not 0 <= device < self.P:
            raise DomainError(f"device {device} out of range")
        o = C.c_int(0)
        call("cg_planner_lookup", self._h, device, self._key(vertex), epoch, staleness_bound,
             C.addressof(o))
        if self.trace is not None:
            self.trace.append((epoch, device, int(vertex), o.value))
        return OUTCOMES[o.value]

    def admit_evict(self, level: str, device: int, vertex: int, version: int = 0):
        if level not in ("local", "global"):
            raise DomainError(f"level must be 'local' or 'global', got {level!r}")
        if level == "local" and not 0 <= device < self.P:
            raise DomainError(f"device {device} out of range")
        vic = C.c_int32(-1)
        call("cg_planner_admit", self._h, 0 if level == "global" else 1, device,
             self._key(vertex), version, C.addressof(vic))
        return None if vic.value < 0 else int(vic.value)

    def warm(self, ranked):
        if len(ranked) != self.P:
            raise DomainError(f"{len(ranked)} ranked lists for {self.P} devices")
        for d, lst in enumerate(ranked):
            for v in list(lst)[: self.caps.c_gpu[d]]:
                self.admit_evict("local", d, v, 0)
        merged, seen = [], set()
        for pos in range(max((len(x) for x in ranked), default=0)):
            for lst in ranked:
                if pos < len(lst) and int(lst[pos]) not in seen:
                    seen.add(int(lst[pos]))
                    merged.append(int(lst[pos]))
        for v in merged[: self.caps.c_cpu]:
            self.admit_evict("global", 0, v, 0)
        return self

    def _counters(self):
        a = [np.zeros(self.P, np.int64) for _ in range(4)]
        call("cg_planner_counters", self._h, *(ptr(x) for x in a))
        return [x.tolist() for x in a]

    @property
    def lookups(self):
        return self._counters()[0]

    @property
    def local_hits(self):
        return self._counters()[1]

    @property
    def global_hits(self):
        return self._counters()[2]

    @property
    def misses(self):
        return self._counters()[3]

    def occupancy(self) -> dict:
        g = C.c_int64(0)
        loc = np.zeros(self.P, np.int64)
        call("cg_planner_occupancy", self._h, C.addressof(g), ptr(loc))
        out = {"global": int(g.value)}
        for d in range(self.P):
            out[f"local{d}"] = int(loc[d])
        return out

    def hit_rate_local(self) -> float:
        lk, lh, _, _ = self._counters()
        return sum(lh) / sum(lk) if sum(lk) else 0.0

    def hit_rate_global(self) -> float:
        lk, _, gh, _ = self._counters()
        return sum(gh) / sum(lk) if sum(lk) else 0.0

    def check_conservation(self) -> None:
        lk, lh, gh, ms = self._counters()
        for d in range(self.P):
            if lk[d] != lh[d] + gh[d] + ms[d]:
                raise DomainError(f"counter conservation violated on device {d}")

    def write_trace_csv(self, sink=None) -> str:
        if self.trace is None:
            raise DomainError("trace recording was not enabled")
        text = trace_csv(self.trace)
        if sink is not None:
            sink.write(text)
        return text
