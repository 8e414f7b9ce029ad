"""Drop-in train entry point: ``train()`` mirrors halopart's ``run()``.

Reference: ``run(g, part, profiles, caps, cfg, record_trace=False) -> SimReport``
(src/halopart/simulator.py:160-256).  ``train`` takes the same five leading
arguments with the same validation and DomainErrors (simulator.py:174-184),
executes REAL partitioned full-batch GCN / GraphSAGE-mean epochs on B200s
with the same per-(epoch, device) cache outcomes, and returns a
``TrainReport`` that carries every SimReport field (records with identical
local/global/miss counts and fwd/bwd bytes, the cost-model times, trace CSV)
plus measured seconds, per-epoch loss, logits and GTEPS.
"""

from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass, field

import numpy as np

from .errors import DomainError
from . import hostgraph as HG
from .layout import build_layout
from .planner import SequentialPlanner, trace_csv


@dataclass(frozen=True)
class EpochDeviceRecord:
    epoch: int
    device: int
    fwd_bytes: int
    bwd_bytes: int
    local_hits: int
    global_hits: int
    misses: int
    compute_time: float
    comm_time: float
    residual_comm_time: float
    device_time: float


@dataclass
class TrainReport:
    """SimReport fields (simulator.py:88-101) + measured training results."""

    config: dict
    sigma: tuple
    records: list
    epoch_makespans: list
    total_time: float
    total_fwd_bytes: int
    total_bwd_bytes: int
    hit_rate_local: float
    hit_rate_global: float
    trace_csv: str | None = field(default=None, repr=False, compare=False)
    # measured on the GPUs
    losses: list = field(default_factory=list)
    epoch_seconds: list = field(default_factory=list)
    spmm_fwd_ms: list = field(default_factory=list)
    spmm_bwd_ms: list = field(default_factory=list)
    planner: list = field(default_factory=list)
    logits: np.ndarray | None = field(default=None, repr=False, compare=False)
    logits_per_epoch: list | None = field(default=None, repr=False, compare=False)
    params: list | None = field(default=None, repr=False, compare=False)
    params_per_epoch: list | None = field(default=None, repr=False, compare=False)
    n_edges: int = 0
    n_layers: int = 0
    n_devices: int = 1

    def gteps(self, epoch_index: int = -1) -> float:
        return self.n_layers * self.n_edges / self.epoch_seconds[epoch_index] / 1e9

    def to_json(self) -> str:
        by = {}
        for r in self.records:
            by.setdefault(r.epoch, []).append(r)
        doc = {"config": self.config, "sigma": list(self.sigma),
               "epochs": [{"epoch": e, "makespan": self.epoch_makespans[e - 1],
                           "devices": [{k: getattr(r, k) for k in (
                               "device", "fwd_bytes", "bwd_bytes", "local_hits", "global_hits",
                               "misses", "compute_time", "comm_time", "residual_comm_time",
                               "device_time")} for r in recs]}
                          for e, recs in sorted(by.items())],
               "totals": {"total_time": self.total_time,
                          "total_fwd_bytes": self.total_fwd_bytes,
                          "total_bwd_bytes": self.total_bwd_bytes,
                          "hit_rate_local": self.hit_rate_local,
                          "hit_rate_global": self.hit_rate_global}}
        return json.dumps(doc, sort_keys=True, indent=2) + "\n"

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(["epoch", "device", "fwd_bytes", "bwd_bytes", "local_hits", "global_hits",
                    "misses", "compute_time", "comm_time", "residual_comm_time",
                    "device_time", "epoch_makespan"])
        for r in self.records:
            w.writerow([r.epoch, r.device, r.fwd_bytes, r.bwd_bytes, r.local_hits,
                        r.global_hits, r.misses, r.compute_time, r.comm_time,
                        r.residual_comm_time, r.device_time, self.epoch_makespans[r.epoch - 1]])
        return buf.getvalue()


def _resolve(part):
    if hasattr(part, "partitions") and hasattr(part, "sigma"):
        return part.partitions, tuple(part.sigma)
    if hasattr(part, "inner") and hasattr(part, "halo"):
        return part, tuple(range(part.P))
    raise DomainError(f"expected RapaResult or PartitionSet, got {type(part).__name__}")


_TF = ("mm_s", "spmm_s", "h2d_s", "d2h_s", "idt_s")


def _normalize(profiles):
    if not profiles:
        raise DomainError("need at least one device profile")
    ids = [p.id for p in profiles]
    if len(set(ids)) != len(ids):
        raise DomainError("duplicate device id in profile list")
    worst = {k: max(getattr(p, k) for p in profiles) for k in _TF}
    return [{k: getattr(p, k) / worst[k] for k in _TF} for p in profiles]


def _model_times(ps, sigma, nrm, cfg):
    """The reference cost model (devices.py:73-132, simulator.py:199-201)."""
    P = ps.P
    mix, comp = [], []
    for i in range(P):
        r = nrm[sigma[i]]
        direct = 1.0 / P
        mix.append((r["h2d_s"] + r["d2h_s"]) * (1.0 - direct) + r["idt_s"] * direct)
        comp.append((cfg.alpha * ps.all_edges[i] * r["spmm_s"]
                     + (1.0 - cfg.alpha) * ps.inner_sizes[i] * r["mm_s"]) * cfg.unit_time)
    return mix, comp


def _epoch_records(ps, cfg, mix, comp, bpe, e, counts, tot, out) -> float:
    """One epoch's per-device records from its cache counts, with the
    reference's cost model and accounting (simulator.py:226-246); appends to
    ``out``, accumulates ``tot`` and returns the epoch makespan."""
    dts = []
    for i in range(ps.P):
        lh, gh, ms = (int(x) for x in counts[i])
        tot += (lh, gh, ms)
        c = (ms + ps.cut_edges[i]) * mix[i] * cfg.unit_time
        ov = min(1.0, cfg.prefetch_depth / max(1, len(ps.halo[i])))
        resid = c - min(c, comp[i]) * ov
        dt = comp[i] + resid
        dts.append(dt)
        out.append(EpochDeviceRecord(
            epoch=e, device=i, fwd_bytes=ms * bpe, bwd_bytes=ps.cut_edges[i] * bpe,
            local_hits=lh, global_hits=gh, misses=ms, compute_time=comp[i],
            comm_time=c, residual_comm_time=resid, device_time=dt))
    return max(dts)


def _validate(part, profiles, caps, cfg):
    """run()'s argument checks and DomainErrors (simulator.py:174-184)."""
    ps, sigma = _resolve(part)
    nrm = _normalize(profiles)
    if len(caps.c_gpu) != ps.P:
        raise DomainError(f"capacities cover {len(caps.c_gpu)} devices, partition has {ps.P}")
    if any(d >= len(nrm) for d in sigma):
        raise DomainError("sigma names a device outside the profile list")
    bpe = HG.feature_bytes(cfg.f_dim)
    if bpe != caps.bytes_per_entry:
        raise DomainError(
            f"capacities sized for {caps.bytes_per_entry} B entries, config implies {bpe} B")
    return ps, sigma, nrm, bpe


def _ranked_planner(g, ps, caps, cfg) -> SequentialPlanner:
    """Importance ranking + warm (simulator.py:186-196), native and bit-exact."""
    union, score = HG.influence_scores(g, ps)
    ranked = [h[np.lexsort((h, -score[np.searchsorted(union, h)]))] for h in ps.halo]
    planner = SequentialPlanner(cfg.policy, caps.c_cpu, caps.c_gpu, union, score,
                                [np.asarray(h, np.int64) for h in ps.halo], ranked)
    planner.warm()
    return planner


def simulate(g, part, profiles, caps, cfg, record_trace: bool = False) -> TrainReport:
    """The cache plan alone, on the host: halopart's ``run()`` (simulator.py:
    160-256) through the native planner (csrc/planner.cpp), no GPU and no
    training.  Returns a ``TrainReport`` whose SimReport fields (records,
    cost-model times, totals, trace) serialise byte-identically to the
    reference's; the measured fields stay empty.  This is what the policy /
    capacity sweeps run, at native speed (the reference's per-lookup Python
    loop takes ~2-4 us per lookup)."""
    ps, sigma, nrm, bpe = _validate(part, profiles, caps, cfg)
    planner = _ranked_planner(g, ps, caps, cfg)
    mix, comp = _model_times(ps, sigma, nrm, cfg)
    records, spans, rows = [], [], []
    tot = np.zeros(3, np.int64)
    for e in range(1, cfg.epochs + 1):
        plan = planner.epoch(e, cfg.staleness_bound)
        spans.append(_epoch_records(ps, cfg, mix, comp, bpe, e, plan.counts, tot, records))
        if record_trace:
            rows += _trace_rows(planner, e, None)
    look = int(tot.sum())
    return TrainReport(
        config=cfg.to_dict(), sigma=sigma, records=records, epoch_makespans=spans,
        total_time=sum(spans), total_fwd_bytes=sum(r.fwd_bytes for r in records),
        total_bwd_bytes=sum(r.bwd_bytes for r in records),
        hit_rate_local=int(tot[0]) / look if look else 0.0,
        hit_rate_global=int(tot[1]) / look if look else 0.0,
        trace_csv=trace_csv(rows) if record_trace else None,
        n_edges=int(g.n_edges), n_layers=len(cfg.f_dim))


def _with_policy(cfg, policy: str):
    import dataclasses
    if dataclasses.is_dataclass(cfg):
        return dataclasses.replace(cfg, policy=policy)
    return HG.SimConfig(**{**cfg.to_dict(), "policy": policy})


def sweep_capacity(g, part, profiles, cfg, capacities, *, train_epochs: bool = False,
                   **train_kw) -> list:
    """halopart's ``sweep_capacity`` (simulator.py:259-268): one run per
    capacity, both cache levels set to it (demand-capped,
    ``uniform_capacities``).  Plan-only (``simulate``) by default;
    ``train_epochs=True`` runs real GPU epochs (``train``) per capacity."""
    if not capacities:
        raise DomainError("need at least one capacity")
    ps, _ = _resolve(part)
    fn = (lambda c: train(g, part, profiles, c, cfg, **train_kw)) if train_epochs else \
        (lambda c: simulate(g, part, profiles, c, cfg))
    return [fn(HG.uniform_capacities(ps, int(c), cfg.f_dim)) for c in capacities]


@dataclass(frozen=True)
class ComparisonRow:
    policy: str
    capacity: int
    hit_rate_local: float
    hit_rate_global: float
    fwd_bytes: int
    bwd_bytes: int
    makespan: float


@dataclass
class ComparisonTable:
    """Policy x capacity grid (simulator.py:271-297); ``makespan`` is the
    run's total modelled time."""

    rows: list

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(["policy", "capacity", "hit_rate_local", "hit_rate_global", "fwd_bytes",
                    "bwd_bytes", "makespan"])
        for r in self.rows:
            w.writerow([r.policy, r.capacity, r.hit_rate_local, r.hit_rate_global,
                        r.fwd_bytes, r.bwd_bytes, r.makespan])
        return buf.getvalue()


def compare_policies(g, part, profiles, cfg, policies=("jaca", "fifo", "lru"),
                     capacities=(0,), *, train_epochs: bool = False,
                     **train_kw) -> ComparisonTable:
    """halopart's ``compare_policies`` (simulator.py:300-322): the identical
    workload under each policy and capacity (plan-only by default, real GPU
    epochs with ``train_epochs=True``)."""
    ps, _ = _resolve(part)
    rows = []
    for policy in policies:
        pcfg = _with_policy(cfg, policy)
        for c in capacities:
            caps = HG.uniform_capacities(ps, int(c), cfg.f_dim)
            rep = (train(g, part, profiles, caps, pcfg, **train_kw) if train_epochs
                   else simulate(g, part, profiles, caps, pcfg))
            rows.append(ComparisonRow(policy=policy, capacity=int(c),
                                      hit_rate_local=rep.hit_rate_local,
                                      hit_rate_global=rep.hit_rate_global,
                                      fwd_bytes=rep.total_fwd_bytes,
                                      bwd_bytes=rep.total_bwd_bytes, makespan=rep.total_time))
    return ComparisonTable(rows=rows)


class TrainSession:
    """The drop-in's stepwise form: ``train()``'s setup once, then one real
    training epoch per ``step()``.

    Same leading arguments, validation and DomainErrors as halopart's
    ``run()`` (simulator.py:160-184).  Per step the caller may hand in this
    device's input rows from pinned host memory (``prefetch_features``: the
    upload overlaps the previous epoch) and start non-blocking downloads of
    the logits / loss (``fetch_logits`` / ``fetch_loss``); ``report()`` builds
    the SimReport-compatible ``TrainReport`` of the steps taken so far.

    ``graphs`` (default on unless CG_GRAPHS=0): on one process, every epoch
    after the cache membership freezes (K6-planned) replays two captured CUDA
    graphs instead of ~45 individual launches; results are bit-identical to
    the eager path.
    """

    def __init__(self, g, part, profiles, caps, cfg, record_trace: bool = False, *,
                 model: str = "gcn", num_classes: int = 40, gemm: str = "3xtf32",
                 plan_mode: str = "auto", keep_logits: str = "last", keep_params: bool = False,
                 timers: bool = True, seed: int = 2, graphs: bool | None = None):
        import torch
        from .comm import DistComm, SoloComm
        from .engine import Engine

        if not torch.cuda.is_available():
            raise RuntimeError("train() needs a CUDA device: the hot path has no CPU fallback")
        ps, sigma, nrm, bpe = _validate(part, profiles, caps, cfg)
        if model not in ("gcn", "sage"):
            raise DomainError(f"unknown model {model!r}")
        if any(int(f) % 4 for f in cfg.f_dim):
            raise DomainError("layer widths must be multiples of 4 (pad the feature dim)")

        dist_on = torch.distributed.is_available() and torch.distributed.is_initialized()
        world = torch.distributed.get_world_size() if dist_on else 1
        rank = torch.distributed.get_rank() if dist_on else 0
        device = torch.cuda.current_device()
        self.comm = DistComm(device) if world > 1 else SoloComm()

        self.planner = _ranked_planner(g, ps, caps, cfg)
        # compact HBM layout when no row is ever staged nor read from a slab
        compact = (cfg.policy == "jaca" and cfg.staleness_bound < 0 and
                   all(int(c) >= h.size for c, h in zip(caps.c_gpu, ps.halo)))
        self.layout = build_layout(g, [np.asarray(x, np.int64) for x in ps.inner],
                                   [np.asarray(h, np.int64) for h in ps.halo], caps.c_gpu,
                                   world, model, compact=compact)
        dims = [int(f) for f in cfg.f_dim] + [int(num_classes)]
        from .models import init_params
        params = init_params(model, dims, seed)
        self.engine = Engine(self.layout, rank, model, dims, bpe, caps, self.planner,
                             cfg.staleness_bound, cfg.policy, comm=self.comm, lr=0.01, gemm=gemm,
                             params_init=params, device=device, record_outcomes=record_trace,
                             plan_mode=plan_mode, graphs=graphs)
        self.g, self.ps, self.cfg, self.sigma, self.bpe = g, ps, cfg, sigma, bpe
        self.record_trace, self.keep_logits, self.keep_params = record_trace, keep_logits, keep_params
        self.timers = timers
        self.mix, self.comp = _model_times(ps, sigma, nrm, cfg)
        self.world = world
        self.epoch = 0
        self.records, self.spans, self.rows = [], [], []
        self.tot = np.zeros(3, np.int64)
        self.rep = TrainReport(config=cfg.to_dict(), sigma=sigma, records=self.records,
                               epoch_makespans=self.spans, total_time=0.0, total_fwd_bytes=0,
                               total_bwd_bytes=0, hit_rate_local=0.0, hit_rate_global=0.0,
                               n_edges=int(g.n_edges), n_layers=len(cfg.f_dim), n_devices=world)
        if keep_logits == "all":
            self.rep.logits_per_epoch = []
        if keep_params:
            self.rep.params_per_epoch = []   # weights at the START of each epoch
        self._pending = []

    # -- host I/O (all non-blocking; see Engine)
    def prefetch_features(self, host_x) -> None:
        """Upload this device's input rows for the NEXT step (pinned host)."""
        self.engine.prefetch_features(host_x)

    def fetch_logits(self, host_buf) -> None:
        self.engine.fetch_logits(host_buf)

    def fetch_loss(self, stats, host_buf) -> None:
        self.engine.fetch_loss(stats, host_buf)

    def step(self, sync: bool = True):
        """Run one epoch.  With sync=False the epoch is only enqueued; its
        record is completed by the next ``finish()``/``report()``."""
        self.epoch += 1
        e = self.epoch
        if self.keep_params:
            self.rep.params_per_epoch.append(self.engine.param_views())
        stt = self.engine.run_epoch(e, timers=self.timers, sync=sync)
        if sync:
            self._record(stt)
        else:
            self._pending.append(stt)
        return stt

    def finish(self) -> None:
        for stt in self._pending:
            self._record(self.engine.finish(stt))
        self._pending = []

    def _record(self, stt) -> None:
        rep, e = self.rep, stt.epoch
        rep.losses.append(stt.loss)
        rep.epoch_seconds.append(stt.seconds)
        rep.spmm_fwd_ms.append(stt.spmm_fwd_ms)
        rep.spmm_bwd_ms.append(stt.spmm_bwd_ms)
        rep.planner.append(stt.planner)
        if self.keep_logits == "all":
            rep.logits_per_epoch.append(_gather_logits(self.engine, self.comm,
                                                       self.g.n_vertices))
        self.spans.append(_epoch_records(self.ps, self.cfg, self.mix, self.comp, self.bpe, e,
                                         stt.counts, self.tot, self.records))
        if self.record_trace:
            oc = self.engine.gpu_outcomes() if stt.planner == "gpu" else None
            self.rows += _trace_rows(self.planner, e, oc)

    def report(self) -> TrainReport:
        self.finish()
        rep = self.rep
        if self.keep_logits in ("last", "all"):
            rep.logits = (rep.logits_per_epoch[-1] if self.keep_logits == "all"
                          and rep.logits_per_epoch else
                          _gather_logits(self.engine, self.comm, self.g.n_vertices))
        rep.params = self.engine.param_views()
        rep.total_time = sum(self.spans)
        rep.total_fwd_bytes = sum(r.fwd_bytes for r in self.records)
        rep.total_bwd_bytes = sum(r.bwd_bytes for r in self.records)
        look = int(self.tot.sum())
        rep.hit_rate_local = int(self.tot[0]) / look if look else 0.0
        rep.hit_rate_global = int(self.tot[1]) / look if look else 0.0
        if self.record_trace:
            rep.trace_csv = trace_csv(self.rows)
        return rep

    def close(self) -> None:
        self.engine.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def train(g, part, profiles, caps, cfg, record_trace: bool = False, *, model: str = "gcn",
          num_classes: int = 40, gemm: str = "3xtf32", plan_mode: str = "auto",
          keep_logits: str = "last", keep_params: bool = False, timers: bool = True,
          seed: int = 2, on_epoch=None, graphs: bool | None = None) -> TrainReport:
    """Run cfg.epochs real training epochs of the partitioned GNN on B200s.

    One partition slot per GPU when torch.distributed is initialised with
    world size P (or P/world slots per GPU); otherwise every partition runs
    on the current GPU, each with its own local cache level.
    """
    with TrainSession(g, part, profiles, caps, cfg, record_trace, model=model,
                      num_classes=num_classes, gemm=gemm, plan_mode=plan_mode,
                      keep_logits=keep_logits, keep_params=keep_params, timers=timers,
                      seed=seed, graphs=graphs) as sess:
        for _ in range(cfg.epochs):
            stt = sess.step()
            if on_epoch is not None:
                on_epoch(stt.epoch, stt, sess.engine)
        return sess.report()


def _trace_rows(planner: SequentialPlanner, e: int, outcomes):
    if outcomes is None:
        outcomes = planner._last_outcome
    sizes = np.diff(planner.halo_off)
    pos = np.concatenate([np.arange(s) for s in sizes]) if sizes.sum() else np.zeros(0, int)
    part = np.repeat(np.arange(planner.P), sizes)
    order = np.lexsort((part, pos))
    verts = planner.union[planner.halo_keys]
    return [(e, int(part[i]), int(verts[i]), int(outcomes[i])) for i in order]


def _gather_logits(eng, comm, n):
    verts, lg = eng.logits_global()
    out = np.zeros((n, lg.shape[1]), np.float32)
    if comm.world == 1:
        out[verts] = lg
        return out
    parts = [None] * comm.world
    comm.dist.all_gather_object(parts, (verts, lg))
    for v, x in parts:
        out[v] = x
    return out
