"""Parity at the large BASELINE.json shapes, on the GPU, through the C ABI.

* C4 (ogbn-products-shaped ER, 2,449,029 v / 61,859,140 e, GCN 3-layer
  f_dim (100, 256, 256) -> 47, P = 8) and C3 (Reddit-shaped ER, 232,965 v /
  114,615,892 e, GraphSAGE-mean 2-layer f_dim (604, 256) -> 41, 2-hop halos,
  P = 8): the product's native preprocessing reproduces the REFERENCE's
  graph / halo / stats / influence / capacity digests, and ``train()``
  reproduces the reference's SimReport JSON / CSV / trace sha256 and
  per-(epoch, partition) records for every golden run (Algorithm-1 "auto"
  capacities at s = -1, and a capacity-limited run with misses, global hits
  and write-through: C4 u1000000_s1, C3 u100000_s0).  Fixtures:
  tests/golden/make_golden_big.py ran halopart itself.
* Float parity at full size: the logits of 256 (C4) / 64 (C3) sampled vertices, for
  weight-forced epochs 1-2 of the auto run, vs the float64 sampled-row oracle
  (oracle/sampled_port.py, the model_port semantics over each sample's
  receptive field) within 1e-4 relative (3xTF32 tcgen05 GEMMs; measured
  <= 1e-5 at C4, 1.6e-5 at C3).
"""

from __future__ import annotations

import numpy as np
import pytest

from _helpers import load_json, sha

pytestmark = pytest.mark.gpu

SHAPES = {
    "c4": dict(n=2449029, e=61859140, f_dim=(100, 256, 256), C=47, kind="gcn", hops=1),
    "c3": dict(n=232965, e=114615892, f_dim=(604, 256), C=41, kind="sage", hops=2),
}
# Per-epoch (weight-forced) bound at the large shapes: the north star's 1e-4.
# Measured (3xTF32): C4 within 1e-5; C3 1.6e-5 at epoch 1 -- GraphSAGE over
# 604-wide inputs with a 492-edge mean per row sums longer fp32 chains than
# the small-shape tests (which hold 1e-5)
FORCED_TOL = 1e-4


def _gdig(g):
    return {"n": g.n_vertices, "n_edges": g.n_edges,
            "out_offsets": sha(g.out_offsets.astype(np.int64)),
            "out_targets": sha(g.out_targets.astype(np.int64)),
            "in_offsets": sha(g.in_offsets.astype(np.int64)),
            "in_targets": sha(g.in_targets.astype(np.int64))}


_CACHE = {}


def _workload(name):
    if name in _CACHE:
        return _CACHE[name]
    from paper_2508_13716_b200 import hostgraph as H
    s = SHAPES[name]
    gold = load_json(f"{name}.json")
    g = H.erdos_renyi(s["n"], s["e"] / s["n"], 0)
    parts = H.random_partition(s["n"], 8, 0)
    ps = H.build_partition_set(g, parts, s["hops"])
    _CACHE[name] = (g, parts, ps, gold)
    return _CACHE[name]


def _caps(ps, run):
    from paper_2508_13716_b200 import hostgraph as H
    c = run["caps"]
    return H.CacheCapacities(c_cpu=c["c_cpu"], c_gpu=tuple(c["c_gpu"]), bytes_per_entry=c["bpe"])


def _cfg(run):
    from paper_2508_13716_b200 import hostgraph as H
    k = run["cfg"]
    return H.SimConfig(epochs=k["epochs"], policy=k["policy"], staleness_bound=k["staleness_bound"],
                       f_dim=tuple(k["f_dim"]), L=k["L"])


@pytest.mark.parametrize("name", ["c4", "c3"])
def test_host_digests_match_reference(name):
    from paper_2508_13716_b200 import hostgraph as H
    g, parts, ps, gold = _workload(name)
    s = SHAPES[name]
    assert _gdig(g) == gold["graph"]
    assert sha(parts.astype(np.int64)) == gold["parts_sha"]
    d = gold["partitions"]
    assert ps.halo_sizes == d["halo_sizes"] and ps.inner_sizes == d["inner_sizes"]
    assert ps.cut_edges == d["cut_edges"] and ps.all_edges == d["all_edges"]
    assert sha(np.concatenate(ps.halo).astype(np.int64)) == d["halo_sha"]
    assert sha(ps.overlap_count.astype(np.int64)) == d["overlap_sha"]
    union, score = H.influence_scores(g, ps)
    assert union.size == d["union_size"]
    assert sha(score.astype(np.float64)) == d["score_sha"]
    ranked = [h[np.lexsort((h, -score[np.searchsorted(union, h)]))] for h in ps.halo]
    assert sha(np.concatenate(ranked).astype(np.int64)) == d["ranked_sha"]
    auto = H.compute_capacities(ps, -1, [180.0] * 8, 1024.0, 64.0, 2048.0, s["f_dim"],
                                len(s["f_dim"]))
    assert (auto.c_cpu, list(auto.c_gpu)) == (gold["auto_caps"]["c_cpu"],
                                              gold["auto_caps"]["c_gpu"])


def _report_checks(rep, run):
    got = [[r.epoch, r.device, r.fwd_bytes, r.bwd_bytes, r.local_hits, r.global_hits, r.misses]
           for r in rep.records]
    assert got == run["records"]
    assert sha(rep.trace_csv) == run["trace_sha"]
    assert sha(rep.to_json()) == run["report_json_sha"]
    assert sha(rep.to_csv()) == run["report_csv_sha"]
    assert all(np.isfinite(rep.losses))


@pytest.mark.parametrize("name,key", [("c4", "u1000000_s1"), ("c3", "u100000_s0")])
def test_capacity_limited_report_matches_reference(name, key):
    from paper_2508_13716_b200 import api, hostgraph as H
    g, _, ps, gold = _workload(name)
    run = gold["runs"][key]
    s = SHAPES[name]
    rep = api.train(g, ps, H.unit_profiles(8), _caps(ps, run), _cfg(run), record_trace=True,
                    model=s["kind"], num_classes=s["C"], gemm="3xtf32", keep_logits="none")
    _report_checks(rep, run)
    assert sum(r.misses for r in rep.records if r.epoch > 1) > 0


@pytest.mark.parametrize("name", ["c4", "c3"])
def test_auto_report_and_sampled_float_parity(name):
    """The reference default (Algorithm-1 capacities, s = -1): integer report
    identical to halopart's, and the sampled logits of both weight-forced
    epochs within 1e-5 of the float64 sampled-row oracle."""
    from oracle import sampled_port as osp
    from paper_2508_13716_b200 import api, hostgraph as H
    g, parts, ps, gold = _workload(name)
    run = gold["runs"]["auto"]
    s = SHAPES[name]
    rep = api.train(g, ps, H.unit_profiles(8), _caps(ps, run), _cfg(run), record_trace=True,
                    model=s["kind"], num_classes=s["C"], gemm="3xtf32", keep_logits="all",
                    keep_params=True)
    _report_checks(rep, run)
    sg = osp.SampledGraph(g.in_offsets, g.in_targets, parts, s["kind"])
    rng = np.random.default_rng(7)
    # C3's average in-degree is 492: 64 samples already reach ~13% of the
    # graph at layer 1 (and every vertex at layer 0)
    samples = rng.choice(s["n"], 256 if name == "c4" else 64, replace=False)
    dims = list(s["f_dim"]) + [s["C"]]
    smp, want = osp.sampled_logits(sg, dims, rep.params_per_epoch, samples)
    for e, w in enumerate(want):
        got = np.asarray(rep.logits_per_epoch[e], np.float64)[smp]
        err = np.max(np.abs(got - w)) / np.max(np.abs(w))
        assert err <= FORCED_TOL, (e, err)
