"""Pin the CPU oracle (oracle/halo_port.py) to vectors the reference produced.

The fixtures in tests/golden/ were written by tests/golden/make_golden.py,
which runs the unmodified halopart package from /root/reference.  These
tests never touch /root/reference themselves.
"""

from __future__ import annotations

import numpy as np
import pytest

from _helpers import codes_in_lookup_order, load_json, load_npz, sha, unit_profiles
from oracle import halo_port as hp


def graph_digest(g):
    return {"n": g.n, "n_edges": g.n_edges,
            "out_offsets": sha(g.out_off.astype(np.int64)),
            "out_targets": sha(g.out_tgt.astype(np.int64)),
            "in_offsets": sha(g.in_off.astype(np.int64)),
            "in_targets": sha(g.in_tgt.astype(np.int64))}


SMALL = load_json("small_cases.json")
ARR = load_npz("small_cases.npz")


@pytest.mark.parametrize("case", SMALL["cases"], ids=lambda c: f"g{c['trial']}")
def test_small_case_integer_parity(case):
    g = hp.er_graph(case["n"], case["deg"], seed=case["seed"])
    assert graph_digest(g) == case["graph"]
    parts = hp.random_assignment(g.n, case["P"], seed=case["seed"])
    ps = hp.partition_set(g, parts, case["hops"])
    assert [h.size for h in ps.halo] == case["halo_sizes"]
    assert ps.cut == case["cut_edges"]
    assert ps.all_edges == case["all_edges"]
    t = case["trial"]
    assert np.array_equal(np.concatenate(ps.halo), ARR[f"g{t}_halo"])
    assert np.array_equal(ps.overlap, ARR[f"g{t}_overlap"])
    verts, _, _, score = hp.influence(g, ps)
    assert score.tobytes() == ARR[f"g{t}_score"].tobytes()  # bit-exact fp64
    ranked = hp.ranked_halos(ps, verts, score)
    imp = {int(v): float(s) for v, s in zip(verts, score)}
    for run in case["runs"]:
        caps = hp.capacities_uniform(ps, run["capacity"], [8, 8])
        assert caps[0] == run["caps"]["c_cpu"] and list(caps[1]) == run["caps"]["c_gpu"]
        pr = hp.plan_epochs(run["policy"], caps, ranked, ps.halo, imp, 6,
                            run["staleness"])
        codes = codes_in_lookup_order([p.outcome for p in pr.plans],
                                      [h.size for h in ps.halo])
        assert np.array_equal(codes, ARR[run["key"] + "_codes"]), run["key"]
        recs, spans = hp.records(ps, list(range(ps.P)), unit_profiles(ps.P), pr,
                                 caps[2], 0.5, 0, 1.0)
        got = [[r["epoch"], r["device"], r["fwd_bytes"], r["bwd_bytes"],
                r["local_hits"], r["global_hits"], r["misses"]] for r in recs]
        assert got == run["records"]
        assert sum(spans) == run["total_time"]
    a1 = case["algo1"]
    c = hp.capacities_auto(ps, a1["k"], [0.0005 * (i + 1) for i in range(ps.P)],
                           0.1, 0.001, 0.2, [64, 64])
    assert (c[0], list(c[1]), c[2]) == (a1["c_cpu"], a1["c_gpu"], a1["bpe"])


def _config_setup(cfg, n, deg, P):
    g = hp.er_graph(n, deg, seed=0)
    assert graph_digest(g) == cfg["graph"]
    parts = hp.random_assignment(n, P, seed=0)
    assert sha(parts) == cfg["parts_sha"]
    ps = hp.partition_set(g, parts, 1)
    d = cfg["partitions"]
    assert [h.size for h in ps.halo] == d["halo_sizes"]
    assert sha(np.concatenate(ps.halo)) == d["halo_sha"]
    assert sha(ps.overlap) == d["overlap_sha"]
    assert ps.cut == d["cut_edges"] and ps.all_edges == d["all_edges"]
    verts, ot, it, score = hp.influence(g, ps)
    assert sha(score) == d["score_sha"]
    assert sha(ot) == d["out_term_sha"] and sha(it) == d["in_term_sha"]
    ranked = hp.ranked_halos(ps, verts, score)
    assert sha(np.concatenate(ranked)) == d["ranked_sha"]
    return g, ps, verts, score, ranked


def test_c1_config_parity():
    cfg = load_json("c1.json")
    g, ps, verts, score, ranked = _config_setup(cfg, 10000, 20.0, 4)
    f_dim = cfg["f_dim"]
    auto = hp.capacities_auto(ps, -1, [180.0] * 4, 1024.0, 64.0, 2048.0, f_dim)
    assert auto[0] == cfg["auto_caps"]["c_cpu"] and list(auto[1]) == cfg["auto_caps"]["c_gpu"]
    imp = {int(v): float(s) for v, s in zip(verts, score)}
    for key in ("cap0", "u3730_s1", "u3730_sneg", "auto"):
        run = cfg["runs"][key]
        caps = (run["caps"]["c_cpu"], tuple(run["caps"]["c_gpu"]), run["caps"]["bpe"])
        pr = hp.plan_epochs(run["cfg"]["policy"], caps, ranked, ps.halo, imp,
                            run["cfg"]["epochs"], run["cfg"]["staleness_bound"])
        assert sha(pr.trace_csv(ps.halo)) == run["trace_sha"], key
        recs, _ = hp.records(ps, list(range(4)), unit_profiles(4), pr, caps[2],
                             0.5, 0, 1.0)
        got = [[r["epoch"], r["device"], r["fwd_bytes"], r["bwd_bytes"],
                r["local_hits"], r["global_hits"], r["misses"]] for r in recs]
        assert got == run["records"], key


@pytest.mark.slow
def test_c2_config_setup_parity():
    cfg = load_json("c2.json")
    n = 169343
    _config_setup(cfg, n, 1166244 / n, 8)


@pytest.mark.parametrize("kind,s,cap", [("gcn", 1, 60), ("sage", -1, None), ("gcn", 0, 30),
                                        ("sage", 1, 40)])
def test_torch_port_matches_model_port(kind, s, cap):
    """The PyTorch-CPU fp32 epoch (the timed CPU baseline)
    computes model_port's float64 epochs within 1e-5 (measured ~1e-6)."""
    from oracle import model_port as omp
    from oracle import torch_port as otp
    n, P, f_dim, C = 400, 4, (16, 32, 32), 7
    g = hp.er_graph(n, 6.0, 0)
    ps = hp.partition_set(g, hp.random_assignment(n, P, 0), 1)
    verts, _, _, score = hp.influence(g, ps)
    imp = {int(v): float(x) for v, x in zip(verts, score)}
    caps = hp.capacities_uniform(ps, cap if cap is not None else 10 ** 6, f_dim)
    pl = hp.Planner("jaca", caps, hp.ranked_halos(ps, verts, score), ps.halo, imp)
    dims = list(f_dim) + [C]
    spec = omp.ModelSpec(kind, dims)
    X, y = omp.features(n, f_dim[0], 0), omp.labels(n, C, 1)
    a = omp.Trainer(g, ps.inner, ps.halo, spec, X, y, params=omp.init_params(kind, dims, 2))
    b = otp.TorchTrainer(g, ps.inner, ps.halo, spec, X, y, params=omp.init_params(kind, dims, 2))
    for e in range(1, 6):
        plan = pl.step(e, s)
        oa, ob = a.step(plan.version), b.step(plan.version, otp.live_versions(pl.cache))
        assert np.abs(oa.logits - ob.logits).max() <= 1e-5 * np.abs(oa.logits).max(), e
        assert abs(oa.loss - ob.loss) <= 1e-5 * oa.loss, e
