"""GPU parity: train() on a B200 vs the CPU oracle, through the C ABI.

Integer parity is exact (per-epoch local/global/miss counts, bytes, trace);
float parity: per-epoch loss and all-vertex logits within 1e-4 relative
(fp32 kernels vs the float64 oracle).  The GEMMs run train()'s default, the
tcgen05 3xTF32 kernel, unless a case names the SIMT fp32 opt-in; free-running
GraphSAGE + 3xTF32 carries the stated looser bound FREE_TOL.
"""

from __future__ import annotations

import numpy as np
import pytest

from parity_common import oracle_run, oracle_run_forced, rel_err, workload

pytestmark = pytest.mark.gpu

TOL = 1e-4


def make_caps(H, ps, cap, f_dim):
    """"auto" (Algorithm 1), an int (uniform), or (c_gpu, c_cpu)."""
    if cap == "auto":
        return H.compute_capacities(ps, -1, [180.0] * ps.P, 1024.0, 64.0, 2048.0, f_dim,
                                    len(f_dim))
    if isinstance(cap, tuple):
        u = H.uniform_capacities(ps, 1, f_dim)
        return H.CacheCapacities(c_cpu=cap[1], c_gpu=(cap[0],) * ps.P,
                                 bytes_per_entry=u.bytes_per_entry)
    return H.uniform_capacities(ps, cap, f_dim)


def _train(g, ps, caps, cfg, kind, C, **kw):
    from paper_2508_13716_b200 import api, hostgraph as H
    return api.train(g, ps, H.unit_profiles(ps.P), caps, cfg, model=kind, num_classes=C,
                     keep_logits="all", **kw)


# Free-running trajectories (no weight forcing) through Adam: Adam's first
# steps are sign-like (m / sqrt(v)), so gradient components near zero turn
# 1e-6-level product differences into O(lr) weight differences.  fp32 SIMT
# and GCN + 3xTF32 stay inside 1e-4 over the checked epochs; GraphSAGE with
# 3xTF32 GEMMs (a TF32-based mode: the north star allows a stated looser
# bound) is measured at 1.1e-4 .. 1.5e-4 over epochs 2-3 -> stated bound 5e-4.
FREE_TOL = {("gcn", "fp32"): TOL, ("sage", "fp32"): TOL, ("gcn", "3xtf32"): TOL,
            ("sage", "3xtf32"): 5e-4}


CASES = [
    # kind, n, deg, P, f_dim, C, capacity ("auto" | int), policy, s, epochs, gemm
    ("gcn", 400, 6.0, 4, (16, 32, 32), 7, "auto", "jaca", -1, 4, "3xtf32"),
    ("gcn", 400, 6.0, 4, (16, 32), 5, 0, "jaca", -1, 3, "3xtf32"),
    ("gcn", 500, 5.0, 3, (16, 32, 32), 6, 60, "jaca", 1, 5, "3xtf32"),
    ("gcn", 500, 5.0, 3, (16, 32, 32), 6, 60, "jaca", 0, 4, "3xtf32"),
    ("sage", 400, 6.0, 4, (16, 32, 32), 7, "auto", "jaca", -1, 4, "3xtf32"),
    ("sage", 500, 5.0, 3, (16, 32), 6, 60, "fifo", 1, 4, "3xtf32"),
    ("gcn", 300, 8.0, 2, (8, 16), 4, 40, "lru", -1, 4, "3xtf32"),
    # one layer (the logits gradient is never aggregated): narrow and wide C
    ("gcn", 400, 6.0, 4, (32,), 7, 60, "jaca", 1, 3, "3xtf32"),
    ("sage", 400, 6.0, 4, (16,), 40, "auto", "jaca", -1, 3, "3xtf32"),
    # small HBM levels beside a large pinned tier (c_gpu, c_cpu): stale global
    # hits read the host tier, several co-resident requesters per vertex
    # (request coalescing: one staged row per vertex and device)
    ("gcn", 500, 5.0, 4, (16, 32, 32), 6, (20, 200), "jaca", 1, 5, "3xtf32"),
    ("sage", 600, 6.0, 4, (16, 32, 32), 6, (40, 300), "jaca", 2, 6, "3xtf32"),
    # GraphSAGE layer 0 transform-first (F0 > F1, compact layout on one
    # device): X W_neigh aggregated, the transposed aggregation in backward
    ("sage", 500, 6.0, 4, (64, 32, 32), 7, "auto", "jaca", -1, 4, "3xtf32"),
    ("sage", 500, 6.0, 4, (64, 32), 9, "auto", "jaca", -1, 3, "fp32"),
    # the SIMT fp32 GEMM (explicit opt-in)
    ("gcn", 500, 5.0, 3, (16, 32, 32), 6, 60, "jaca", 1, 4, "fp32"),
    ("sage", 400, 6.0, 4, (16, 32, 32), 7, "auto", "jaca", -1, 3, "fp32"),
]


@pytest.mark.parametrize("case", CASES,
                         ids=lambda c: f"{c[0]}-L{len(c[4])}-P{c[3]}-{c[6]}-{c[7]}-s{c[8]}-{c[10]}")
def test_train_matches_oracle(case):
    from paper_2508_13716_b200 import hostgraph as H
    kind, n, deg, P, f_dim, C, cap, policy, s, epochs, gemm = case
    g, ps, og, ops = workload(n, deg, P)
    caps = make_caps(H, ps, cap, f_dim)
    cfg = H.SimConfig(epochs=epochs, policy=policy, staleness_bound=s, f_dim=f_dim,
                      L=len(f_dim))
    rep = _train(g, ps, caps, cfg, kind, C, record_trace=True, gemm=gemm)
    pr, outs, _ = oracle_run(og, ops, kind, f_dim, C, caps, policy, s, epochs)
    # integer parity: counts per (epoch, partition) and the trace
    for p in pr.plans:
        got = [(r.local_hits, r.global_hits, r.misses) for r in rep.records if r.epoch == p.epoch]
        assert got == [tuple(int(x) for x in c) for c in p.counts], p.epoch
    assert rep.trace_csv == pr.trace_csv(ops.halo)
    # float parity: epoch 1 at 1e-4 always, later (free-running) epochs at
    # the mode's stated bound
    for e, o in enumerate(outs):
        tol = TOL if e == 0 else FREE_TOL[(kind, gemm)]
        assert abs(rep.losses[e] - o.loss) <= tol * abs(o.loss), (e, rep.losses[e], o.loss)
        assert rel_err(rep.logits_per_epoch[e], o.logits) <= tol, e


@pytest.mark.parametrize("kind", ["gcn", "sage"])
@pytest.mark.parametrize("gemm", ["3xtf32", "fp32"])
def test_train_weight_forced_parity(kind, gemm):
    """Per-epoch parity with the oracle run from the GPU's own weights at the
    start of every epoch (stale snapshots included): the epoch arithmetic is
    checked without Adam compounding earlier rounding differences -- at 1e-5
    (10x inside the 1e-4 bound; measured <= 3e-6).  3xTF32 is the tcgen05
    path the bench uses."""
    from paper_2508_13716_b200 import hostgraph as H
    g, ps, og, ops = workload(700, 6.0, 4)
    f_dim, C = (32, 64, 64), 10
    caps = H.uniform_capacities(ps, 150, f_dim)
    cfg = H.SimConfig(epochs=6, policy="jaca", staleness_bound=1, f_dim=f_dim, L=3)
    rep = _train(g, ps, caps, cfg, kind, C, gemm=gemm, keep_params=True)
    _, outs = oracle_run_forced(og, ops, kind, f_dim, C, caps, "jaca", 1, rep.params_per_epoch)
    for e, o in enumerate(outs):
        assert abs(rep.losses[e] - o.loss) <= 1e-5 * abs(o.loss)
        assert rel_err(rep.logits_per_epoch[e], o.logits) <= 1e-5, e
    # free-running trajectory: epoch 1 at 1e-4 always, then FREE_TOL
    _, free, _ = oracle_run(og, ops, kind, f_dim, C, caps, "jaca", 1, 3)
    for e, o in enumerate(free):
        tol = TOL if e == 0 else FREE_TOL[(kind, gemm)]
        assert rel_err(rep.logits_per_epoch[e], o.logits) <= tol, e


def test_gpu_planner_handoff_matches_host_planner():
    """K6 (GPU frozen plan) vs the exact host planner on every epoch."""
    from paper_2508_13716_b200 import hostgraph as H
    g, ps, og, ops = workload(600, 6.0, 4)
    f_dim = (16, 16)
    caps = H.uniform_capacities(ps, 120, f_dim)
    for s in (-1, 1, 2):
        cfg = H.SimConfig(epochs=7, policy="jaca", staleness_bound=s, f_dim=f_dim, L=2)
        a = _train(g, ps, caps, cfg, "gcn", 5, record_trace=True)
        b = _train(g, ps, caps, cfg, "gcn", 5, record_trace=True, plan_mode="host")
        assert "gpu" in a.planner and "gpu" not in b.planner
        assert a.trace_csv == b.trace_csv
        assert [r.misses for r in a.records] == [r.misses for r in b.records]
        for x, y in zip(a.logits_per_epoch, b.logits_per_epoch):
            assert rel_err(x, y) <= TOL


def test_bitwise_deterministic_reruns():
    from paper_2508_13716_b200 import hostgraph as H
    g, ps, _, _ = workload(500, 6.0, 4)
    f_dim = (16, 32)
    caps = H.uniform_capacities(ps, 50, f_dim)
    cfg = H.SimConfig(epochs=3, policy="jaca", staleness_bound=1, f_dim=f_dim, L=2)
    a = _train(g, ps, caps, cfg, "gcn", 5)
    b = _train(g, ps, caps, cfg, "gcn", 5)
    assert a.losses == b.losses
    for x, y in zip(a.logits_per_epoch, b.logits_per_epoch):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("kind", ["gcn", "sage"])
def test_two_hop_halos_match_oracle(kind):
    """hops = 2 (C3's setting, A7): lookups and model bytes range over the
    whole 2-hop halo, aggregation uses the 1-hop in-edges it contains."""
    from paper_2508_13716_b200 import hostgraph as H
    g, ps, og, ops = workload(400, 4.0, 4, hops=2)
    assert sum(h.size for h in ps.halo) > sum(
        H.build_partition_set(g, H.random_partition(400, 4, 0), 1).halo_sizes)
    f_dim, C = (16, 32), 6
    caps = H.uniform_capacities(ps, 120, f_dim)
    cfg = H.SimConfig(epochs=4, policy="jaca", staleness_bound=1, f_dim=f_dim, L=2)
    rep = _train(g, ps, caps, cfg, kind, C, record_trace=True)
    pr, outs, _ = oracle_run(og, ops, kind, f_dim, C, caps, "jaca", 1, 4)
    for p in pr.plans:
        got = [(r.local_hits, r.global_hits, r.misses) for r in rep.records if r.epoch == p.epoch]
        assert got == [tuple(int(x) for x in c) for c in p.counts], p.epoch
    assert rep.trace_csv == pr.trace_csv(ops.halo)
    for e, o in enumerate(outs):
        assert abs(rep.losses[e] - o.loss) <= TOL * abs(o.loss), e
        assert rel_err(rep.logits_per_epoch[e], o.logits) <= TOL, e


def test_rapa_pruned_partition_matches_oracle():
    """A RAPA result with trimmed halos and a permuted sigma (made by the
    reference CLI, tests/golden/cli): edges from pruned halo vertices are
    dropped, degrees stay global (A5)."""
    import os
    from oracle import halo_port as ohp
    from paper_2508_13716_b200 import artifacts as A, hostgraph as H
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
    g = A.load_edge_list(os.path.join(gold, "graph.txt"))
    res, ps = A.import_rapa_result(os.path.join(gold, "rapa.json"))
    full = H.build_partition_set(g, np.concatenate(
        [np.full(x.size, i) for i, x in enumerate(ps.inner)])[np.argsort(np.concatenate(ps.inner))], 1)
    assert any(a.size < b.size for a, b in zip(ps.halo, full.halo))   # really pruned
    og = ohp.er_graph(400, 8.0, 3)
    assert np.array_equal(og.in_tgt, g.in_targets)
    ops = ohp.Partitions(n=g.n_vertices, P=ps.P, parts=None, inner=ps.inner, halo=ps.halo,
                         hops=1, overlap=ps.overlap_count, cut=ps.cut_edges,
                         all_edges=ps.all_edges)
    f_dim, C = (16, 32), 7
    caps = H.uniform_capacities(ps, 40, f_dim)
    cfg = H.SimConfig(epochs=4, policy="jaca", staleness_bound=1, f_dim=f_dim, L=2)
    from paper_2508_13716_b200 import api
    rep = api.train(g, res, A.load_device_profiles(os.path.join(gold, "devices.json")), caps, cfg,
                    model="gcn", num_classes=C, keep_logits="all", record_trace=True,
                    gemm="3xtf32")
    pr, outs, _ = oracle_run(og, ops, "gcn", f_dim, C, caps, "jaca", 1, 4)
    assert rep.trace_csv == pr.trace_csv(ops.halo)
    for e, o in enumerate(outs):
        assert abs(rep.losses[e] - o.loss) <= TOL * abs(o.loss), e
        assert rel_err(rep.logits_per_epoch[e], o.logits) <= TOL, e


# Free-running logits at the C2 size after Adam steps (stated looser bound;
# the drift grows with the number of Adam steps): measured 2.3e-5 / 3.8e-4
# (fp32 SIMT) and 8.8e-4 / 2.3e-3 (3xTF32) at epochs 2 / 3 of auto_sneg
# (tests/diag_c2_parity.py), 6.1e-3 at epoch 4 of u40000_s1
C2_FREE_LOGITS_TOL = 1.5e-2


@pytest.mark.parametrize("cache", ["auto_sneg", "u40000_s1"])
def test_c2_float_parity(cache):
    """The bench workload (C2: 169,343 v / 1,166,244 e, GCN 3-layer
    128-256-256 -> 40, P = 8 on one GPU, 3xTF32 tcgen05 GEMMs), full size,
    vs the float64 oracle, on both cache configurations the bench times:
    ``auto_sneg`` (Algorithm-1 capacities, s = -1: the compact layout, every
    read a version-0 hit) and ``u40000_s1`` (uniform capacity 40,000 per
    level, s = 1: the exchange path -- misses, stale global hits from the
    pinned host tier, slab and host write-through):
      * cache counts of every (epoch, partition) exactly;
      * per-epoch arithmetic (oracle restarted from the GPU's weights each
        epoch) within 1e-5 on all logits and the loss;
      * free-running: the loss within 1e-4 every epoch, the logits of epoch 1
        within 1e-4, later logits within the stated looser bound
        C2_FREE_LOGITS_TOL (Adam's first steps are sign-like, so fp32-vs-
        float64 gradient differences on near-zero components become O(lr)
        weight differences -- no fp32 implementation holds the float64
        trajectory to 1e-4 there)."""
    import bench
    from paper_2508_13716_b200 import hostgraph as H
    bench.apply_config("c2")
    g, ps, caps = bench.build_workload(8)
    s, epochs = -1, 3
    if cache == "u40000_s1":
        caps, s, epochs = H.uniform_capacities(ps, 40000, bench.F_DIM), 1, 4
    cfg = H.SimConfig(epochs=epochs, policy="jaca", staleness_bound=s, f_dim=bench.F_DIM, L=3)
    rep = _train(g, ps, caps, cfg, "gcn", bench.CLASSES, gemm="3xtf32", keep_params=True)
    og, ops, _ = bench.oracle_inputs(g, ps, caps)
    pr, forced = oracle_run_forced(og, ops, "gcn", bench.F_DIM, bench.CLASSES, caps, "jaca", s,
                                   rep.params_per_epoch)
    for e, (p, fo) in enumerate(zip(pr.plans, forced)):
        got = [(r.local_hits, r.global_hits, r.misses) for r in rep.records if r.epoch == e + 1]
        assert got == [tuple(int(x) for x in c) for c in p.counts], e
        assert abs(rep.losses[e] - fo.loss) <= 1e-5 * abs(fo.loss), e
        assert rel_err(rep.logits_per_epoch[e], fo.logits) <= 1e-5, e
    if cache == "u40000_s1":   # the exchange path really ran
        assert sum(r.global_hits for r in rep.records) > 0
        assert sum(r.misses for r in rep.records if r.epoch > 1) > 0
    _, free, _ = oracle_run(og, ops, "gcn", bench.F_DIM, bench.CLASSES, caps, "jaca", s, epochs)
    for e, out in enumerate(free):
        assert abs(rep.losses[e] - out.loss) <= TOL * abs(out.loss), (e, rep.losses[e], out.loss)
        tol = TOL if e == 0 else C2_FREE_LOGITS_TOL
        assert rel_err(rep.logits_per_epoch[e], out.logits) <= tol, e


def test_write_through_queue_matches_inline(monkeypatch):
    """The host-tier write-through on its side-stream queue (default) gives
    bit-identical epochs to the in-line copies, across host-planned and
    K6-planned (graph-replayed) epochs of a capacity-limited s = 1 run with
    global-tier hits."""
    from paper_2508_13716_b200 import hostgraph as H
    g, ps, _, _ = workload(800, 6.0, 4)
    f_dim = (16, 32, 32)
    caps = H.uniform_capacities(ps, 120, f_dim)
    cfg = H.SimConfig(epochs=7, policy="jaca", staleness_bound=1, f_dim=f_dim, L=3)
    runs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("CG_WT_ASYNC", flag)
        runs.append(_train(g, ps, caps, cfg, "gcn", 6))
    a, b = runs
    assert sum(r.global_hits for r in a.records) > 0
    assert a.losses == b.losses
    for x, y in zip(a.logits_per_epoch, b.logits_per_epoch):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("gemm", ["3xtf32", "fp32"])
def test_sage_transform_first_layer0_matches_aggregate_first(gemm, monkeypatch):
    """The two layer-0 orders of GraphSAGE (CG_SAGE_TF0) agree within the
    parity bound every epoch, and the integer plan is identical."""
    from paper_2508_13716_b200 import hostgraph as H
    g, ps, og, ops = workload(600, 7.0, 4)
    f_dim, C = (96, 32, 32), 6
    caps = make_caps(H, ps, "auto", f_dim)
    cfg = H.SimConfig(epochs=4, policy="jaca", staleness_bound=-1, f_dim=f_dim, L=3)
    monkeypatch.setenv("CG_SAGE_TF0", "0")
    a = _train(g, ps, caps, cfg, "sage", C, gemm=gemm, record_trace=True)
    monkeypatch.setenv("CG_SAGE_TF0", "1")
    b = _train(g, ps, caps, cfg, "sage", C, gemm=gemm, record_trace=True)
    assert a.trace_csv == b.trace_csv
    for e in range(4):
        assert rel_err(b.logits_per_epoch[e], a.logits_per_epoch[e]) <= FREE_TOL[("sage", gemm)], e
        assert abs(a.losses[e] - b.losses[e]) <= 1e-4 * abs(a.losses[e])


@pytest.mark.parametrize("gemm", ["3xtf32", "fp32"])
@pytest.mark.parametrize("kind", ["gcn", "sage"])
def test_last_layer_transform_first_matches_aggregate_first(kind, gemm, monkeypatch):
    """The narrowing last layer in both orders (CG_TFL; GraphSAGE adds
    the self term as the aggregation's addend): logits, loss and the trained
    weights agree within the parity bound every epoch, and the transform-first
    run matches the oracle."""
    from paper_2508_13716_b200 import hostgraph as H
    g, ps, og, ops = workload(700, 7.0, 4)
    f_dim, C = (32, 64, 64), 10
    caps = make_caps(H, ps, "auto", f_dim)
    cfg = H.SimConfig(epochs=4, policy="jaca", staleness_bound=-1, f_dim=f_dim, L=3)
    monkeypatch.setenv("CG_TFL", "0")
    a = _train(g, ps, caps, cfg, kind, C, gemm=gemm, record_trace=True, keep_params=True)
    monkeypatch.setenv("CG_TFL", "1")
    b = _train(g, ps, caps, cfg, kind, C, gemm=gemm, record_trace=True, keep_params=True)
    assert a.trace_csv == b.trace_csv
    tol = FREE_TOL[(kind, gemm)]
    for e in range(4):
        assert rel_err(b.logits_per_epoch[e], a.logits_per_epoch[e]) <= tol, e
        assert abs(a.losses[e] - b.losses[e]) <= 1e-5 * abs(a.losses[e])
    for x, y in zip(a.params, b.params):
        assert rel_err(y, x) <= tol
    # the transform-first epochs against the oracle run from the GPU's own
    # weights every epoch (per-epoch arithmetic; free-running drift through
    # Adam is the stated FREE_TOL matter above, not the order of the layer)
    _, outs = oracle_run_forced(og, ops, kind, f_dim, C, caps, "jaca", -1, b.params_per_epoch)
    for e, o in enumerate(outs):
        assert rel_err(b.logits_per_epoch[e], o.logits) <= 1e-5, e
        assert abs(b.losses[e] - o.loss) <= 1e-5 * abs(o.loss), e
