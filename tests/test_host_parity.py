"""Product host path (native preprocessing + native planner) vs golden vectors.

Bit-exact integer parity with the reference: graphs, halos, partition stats,
fp64 influence scores, Algorithm-1 capacities and the per-lookup cache trace.
Also exercises the C-ABI library load (CPU-only entry points).
"""

from __future__ import annotations

import numpy as np
import pytest

from _helpers import load_json, load_npz, sha
from paper_2508_13716_b200 import hostgraph as H
from paper_2508_13716_b200 import planner as PL
from paper_2508_13716_b200 import _lib

SMALL = load_json("small_cases.json")
ARR = load_npz("small_cases.npz")


def gdig(g):
    return {"n": g.n_vertices, "n_edges": g.n_edges,
            "out_offsets": sha(g.out_offsets.astype(np.int64)),
            "out_targets": sha(g.out_targets.astype(np.int64)),
            "in_offsets": sha(g.in_offsets.astype(np.int64)),
            "in_targets": sha(g.in_targets.astype(np.int64))}


def setup(n, deg, P, hops, seed):
    g = H.erdos_renyi(n, deg, seed)
    ps = H.build_partition_set(g, H.random_partition(n, P, seed), hops)
    union, score = H.influence_scores(g, ps)
    ranked = [h[np.lexsort((h, -score[np.searchsorted(union, h)]))] for h in ps.halo]
    return g, ps, union, score, ranked


def lookup_order_codes(planner, plans):
    sizes = np.diff(planner.halo_off)
    longest = int(sizes.max())
    # index of requester i in round-robin order: (pos, partition)
    pos = np.concatenate([np.arange(s) for s in sizes])
    part = np.repeat(np.arange(planner.P), sizes)
    order = np.lexsort((part, pos))
    return np.concatenate([p.outcome[order] for p in plans]).astype(np.int8)


@pytest.mark.parametrize("case", SMALL["cases"], ids=lambda c: f"g{c['trial']}")
def test_small_cases_native(case):
    g, ps, union, score, ranked = setup(case["n"], case["deg"], case["P"], case["hops"],
                                        case["seed"])
    assert gdig(g) == case["graph"]
    assert ps.halo_sizes == case["halo_sizes"]
    assert ps.cut_edges == case["cut_edges"] and ps.all_edges == case["all_edges"]
    t = case["trial"]
    assert np.array_equal(np.concatenate(ps.halo), ARR[f"g{t}_halo"])
    assert score.tobytes() == ARR[f"g{t}_score"].tobytes()
    for run in case["runs"]:
        caps = H.uniform_capacities(ps, run["capacity"], [8, 8])
        pl = PL.SequentialPlanner(run["policy"], caps.c_cpu, caps.c_gpu, union, score,
                                  ps.halo, ranked)
        pl.warm()
        plans = [pl.epoch(e, run["staleness"]) for e in range(1, 7)]
        codes = lookup_order_codes(pl, plans)
        assert np.array_equal(codes, ARR[run["key"] + "_codes"]), run["key"]
        for p in plans:
            got = [[p.epoch, d, int(p.counts[d, 2]) * 64, ps.cut_edges[d] * 64,
                    int(p.counts[d, 0]), int(p.counts[d, 1]), int(p.counts[d, 2])]
                   for d in range(ps.P)]
            assert got == [r for r in run["records"] if r[0] == p.epoch]
    a1 = case["algo1"]
    c = H.compute_capacities(ps, a1["k"], [0.0005 * (i + 1) for i in range(ps.P)], 0.1,
                             0.001, 0.2, [64, 64], 2)
    assert (c.c_cpu, list(c.c_gpu), c.bytes_per_entry) == (a1["c_cpu"], a1["c_gpu"], a1["bpe"])


def test_c1_native_trace_digests():
    cfg = load_json("c1.json")
    g, ps, union, score, ranked = setup(10000, 20.0, 4, 1, 0)
    assert gdig(g) == cfg["graph"]
    assert sha(score) == cfg["partitions"]["score_sha"]
    auto = H.compute_capacities(ps, -1, [180.0] * 4, 1024.0, 64.0, 2048.0, (128, 128), 2)
    assert auto.c_cpu == cfg["auto_caps"]["c_cpu"] and list(auto.c_gpu) == cfg["auto_caps"]["c_gpu"]
    for key, run in cfg["runs"].items():
        c = run["caps"]
        pl = PL.SequentialPlanner(run["cfg"]["policy"], c["c_cpu"], c["c_gpu"], union, score,
                                  ps.halo, ranked)
        pl.warm()
        rows = []
        for e in range(1, run["cfg"]["epochs"] + 1):
            rows += pl.trace_rows(pl.epoch(e, run["cfg"]["staleness_bound"]))
        assert sha(PL.trace_csv(rows)) == run["trace_sha"], key


@pytest.mark.slow
def test_c2_native_setup_and_first_epochs():
    cfg = load_json("c2.json")
    n = 169343
    g, ps, union, score, ranked = setup(n, 1166244 / n, 8, 1, 0)
    assert gdig(g) == cfg["graph"]
    d = cfg["partitions"]
    assert ps.halo_sizes == d["halo_sizes"] and ps.cut_edges == d["cut_edges"]
    assert sha(score) == d["score_sha"]
    assert sha(np.concatenate(ranked)) == d["ranked_sha"]
    run = cfg["runs"]["u40000_s1"]
    c = run["caps"]
    pl = PL.SequentialPlanner("jaca", c["c_cpu"], c["c_gpu"], union, score, ps.halo, ranked)
    pl.warm()
    for e in range(1, 5):
        p = pl.epoch(e, 1)
        got = [[e, dd, int(p.counts[dd, 2]) * c["bpe"], ps.cut_edges[dd] * c["bpe"],
                int(p.counts[dd, 0]), int(p.counts[dd, 1]), int(p.counts[dd, 2])]
               for dd in range(8)]
        assert got == [r for r in run["records"] if r[0] == e]


# ---- CacheSystem operator API: the reference's own known answers ----------
# (test_cache.py:107-158, 172-209, 223-284 and test_acceptance.py:222-253)


def caps(c, n=1):
    return H.CacheCapacities(c_cpu=c, c_gpu=(c,) * n, bytes_per_entry=4)


def test_operator_policy_known_answers():
    cs = PL.HaloCache("fifo", caps(2))
    assert cs.admit_evict("local", 0, 10) is None
    assert cs.admit_evict("local", 0, 11) is None
    assert cs.admit_evict("local", 0, 12) == 10
    cs = PL.HaloCache("lru", caps(2))
    cs.admit_evict("local", 0, 10)
    cs.admit_evict("local", 0, 11)
    cs.admit_evict("local", 0, 10)
    assert cs.admit_evict("local", 0, 12) == 11
    cs = PL.HaloCache("fifo", caps(2))
    cs.admit_evict("local", 0, 10)
    cs.admit_evict("local", 0, 11)
    cs.admit_evict("local", 0, 10)
    assert cs.admit_evict("local", 0, 12) == 10
    cs = PL.HaloCache("jaca", caps(2), importance={10: 3.0, 11: 2.0, 12: 1.0})
    cs.admit_evict("local", 0, 10)
    cs.admit_evict("local", 0, 11)
    assert cs.admit_evict("local", 0, 12) is None
    cs = PL.HaloCache("jaca", caps(2), importance={10: 3.0, 11: 2.0, 13: 5.0, 14: 9.0})
    cs.admit_evict("local", 0, 10)
    cs.admit_evict("local", 0, 11)
    assert cs.admit_evict("local", 0, 13) == 11
    assert cs.admit_evict("local", 0, 14) == 10
    cs = PL.HaloCache("jaca", caps(1), importance={1: 2.0, 2: 2.0})
    cs.admit_evict("local", 0, 1)
    assert cs.admit_evict("local", 0, 2) is None


def test_operator_staleness_and_copy_down():
    cs = PL.HaloCache("fifo", caps(4))
    assert cs.lookup(0, 7, epoch=3, staleness_bound=1) == "miss"
    assert cs.lookup(0, 7, epoch=4, staleness_bound=1) == "local_hit"
    assert cs.lookup(0, 7, epoch=5, staleness_bound=1) == "miss"
    assert cs.lookup(0, 7, epoch=5, staleness_bound=1) == "local_hit"
    cs = PL.HaloCache("fifo", caps(2))
    cs.admit_evict("global", 0, 7, version=0)
    assert cs.lookup(0, 7, epoch=2, staleness_bound=-1) == "global_hit"
    assert cs.lookup(0, 7, epoch=2, staleness_bound=-1) == "local_hit"
    cs = PL.HaloCache("lru", caps(0))
    for e in range(1, 4):
        assert cs.lookup(0, 9, e, staleness_bound=-1) == "miss"
    assert cs.occupancy() == {"global": 0, "local0": 0}
    cs.check_conservation()
    cs = PL.HaloCache("fifo", caps(2), record_trace=True)
    cs.lookup(0, 4, epoch=1, staleness_bound=-1)
    cs.lookup(0, 4, epoch=1, staleness_bound=-1)
    lines = cs.write_trace_csv().splitlines()
    assert lines == ["epoch,device,vertex,outcome,level", "1,0,4,miss,source",
                     "1,0,4,hit,local"]


def test_operator_warm_interleave_and_scan_resistance():
    cs = PL.HaloCache("fifo", H.CacheCapacities(c_cpu=3, c_gpu=(0, 0), bytes_per_entry=4))
    cs.warm([[1, 2, 9], [3, 1, 8]])
    assert cs.occupancy()["global"] == 3
    # acceptance criterion 6: |H|=1000, C=500
    halo = list(range(1000))
    imp = {v: 1.0 for v in halo}

    def rates(policy, c):
        cs = PL.HaloCache(policy, caps(c), imp).warm([halo])
        out = []
        for e in range(1, 6):
            before = cs.local_hits[0]
            for v in halo:
                cs.lookup(0, v, e, staleness_bound=-1)
            out.append((cs.local_hits[0] - before) / len(halo))
        return out

    assert all(r == 0.5 for r in rates("jaca", 500)[1:])
    assert all(r == 0.0 for r in rates("fifo", 500)[1:])
    assert all(r == 0.0 for r in rates("lru", 500)[1:])
    assert all(r == 1.0 for r in rates("lru", 1000)[1:])


def test_library_exports_every_declared_symbol():
    import re
    import os
    hdr = open(os.path.join(os.path.dirname(_lib.__file__), "..", "include", "capgnn.h")).read()
    declared = set(re.findall(r"^(?:int|int64_t|const char \*)\s*\*?\s*(cg_\w+)\(", hdr, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.exported_symbols())
    h = _lib.lib()
    for name in declared:
        assert hasattr(h, name), name
    assert h.cg_version() == 100
