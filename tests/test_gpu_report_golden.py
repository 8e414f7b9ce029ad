"""train() on the GPU reproduces the REFERENCE's SimReport byte for byte.

The fixtures hold sha256 digests of halopart.run(...).to_json() / .to_csv()
/ .trace_csv for the C1 and C2 workloads (tests/golden/make_golden.py).
train() drives the same cache plan through real training epochs; its
report's integer records (hits, misses, fwd/bwd bytes) and the reference
cost-model fields must serialise identically.
"""

from __future__ import annotations

import pytest

from _helpers import load_json, sha

pytestmark = pytest.mark.gpu


def _run(n, deg, P, f_dim, run, model="gcn"):
    from paper_2508_13716_b200 import api, hostgraph as H
    g = H.erdos_renyi(n, deg, 0)
    ps = H.build_partition_set(g, H.random_partition(n, P, 0), 1)
    c = run["caps"]
    caps = H.CacheCapacities(c_cpu=c["c_cpu"], c_gpu=tuple(c["c_gpu"]), bytes_per_entry=c["bpe"])
    k = run["cfg"]
    cfg = H.SimConfig(epochs=k["epochs"], policy=k["policy"], staleness_bound=k["staleness_bound"],
                      f_dim=tuple(k["f_dim"]), L=k["L"])
    return api.train(g, ps, H.unit_profiles(P), caps, cfg, record_trace=True, model=model,
                     num_classes=40, gemm="3xtf32")


@pytest.mark.parametrize("key", ["cap0", "u3730_s1", "u3730_sneg", "u3730_s0", "auto",
                                 "fifo_u2000_s1", "lru_u2000_sneg"])
def test_c1_report_matches_reference(key):
    cfg = load_json("c1.json")
    run = cfg["runs"][key]
    rep = _run(10000, 20.0, 4, cfg["f_dim"], run)
    assert sha(rep.trace_csv) == run["trace_sha"]
    assert sha(rep.to_json()) == run["report_json_sha"]
    assert sha(rep.to_csv()) == run["report_csv_sha"]
    assert all(x == x for x in rep.losses)  # finite training losses


@pytest.mark.parametrize("key", ["auto", "u40000_s1", "cap0"])
def test_c2_report_matches_reference(key):
    cfg = load_json("c2.json")
    run = cfg["runs"][key]
    n = 169343
    rep = _run(n, 1166244 / n, 8, cfg["f_dim"], run)
    got = [[r.epoch, r.device, r.fwd_bytes, r.bwd_bytes, r.local_hits, r.global_hits, r.misses]
           for r in rep.records]
    assert got == run["records"]
    assert sha(rep.to_json()) == run["report_json_sha"]
