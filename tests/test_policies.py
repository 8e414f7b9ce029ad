"""Plan-only runs on the host (no GPU): ``api.simulate`` reproduces the
reference's ``run()`` SimReport byte for byte, and ``api.compare_policies`` /
``api.sweep_capacity`` reproduce halopart's policy x capacity grid and
capacity sweep (simulator.py:259-322) on the C1 workload with a
heterogeneous device list (fixtures: tests/golden/make_golden.py,
make_golden_policies.py, both run the reference itself)."""

from __future__ import annotations

import pytest

from _helpers import load_json, sha
from paper_2508_13716_b200 import api, hostgraph as H
from paper_2508_13716_b200.errors import DomainError


@pytest.fixture(scope="module")
def c1():
    g = H.erdos_renyi(10000, 20.0, 0)
    ps = H.build_partition_set(g, H.random_partition(10000, 4, 0), 1)
    return g, ps


def _caps(run):
    c = run["caps"]
    return H.CacheCapacities(c_cpu=c["c_cpu"], c_gpu=tuple(c["c_gpu"]), bytes_per_entry=c["bpe"])


@pytest.mark.parametrize("key", ["cap0", "u3730_s1", "u3730_sneg", "auto", "fifo_u2000_s1",
                                 "lru_u2000_sneg"])
def test_simulate_matches_reference_run(c1, key):
    g, ps = c1
    run = load_json("c1.json")["runs"][key]
    k = run["cfg"]
    cfg = H.SimConfig(epochs=k["epochs"], policy=k["policy"], staleness_bound=k["staleness_bound"],
                      f_dim=tuple(k["f_dim"]), L=k["L"])
    rep = api.simulate(g, ps, H.unit_profiles(4, 64.0), _caps(run), cfg, record_trace=True)
    assert sha(rep.trace_csv) == run["trace_sha"]
    assert sha(rep.to_json()) == run["report_json_sha"]
    assert sha(rep.to_csv()) == run["report_csv_sha"]


def _profiles(gold):
    return [H.DeviceProfile(id=i, mm_s=a, spmm_s=b, h2d_s=c, d2h_s=d, idt_s=e, mem_gb=m)
            for i, a, b, c, d, e, m in gold["profiles"]]


def _cfg(gold):
    c = dict(gold["cfg"])
    c["f_dim"] = tuple(c["f_dim"])
    return H.SimConfig(policy="jaca", **c)


def test_compare_policies_matches_reference(c1):
    g, ps = c1
    gold = load_json("policies.json")
    table = api.compare_policies(g, ps, _profiles(gold), _cfg(gold),
                                 capacities=gold["compare_caps"])
    assert table.to_csv() == gold["compare_csv"]


def test_sweep_capacity_matches_reference(c1):
    g, ps = c1
    gold = load_json("policies.json")
    reps = api.sweep_capacity(g, ps, _profiles(gold), _cfg(gold), gold["sweep_caps"])
    for rep, want in zip(reps, gold["sweep"]):
        assert sha(rep.to_json()) == want["report_json_sha"]
        assert sha(rep.to_csv()) == want["report_csv_sha"]
    with pytest.raises(DomainError):
        api.sweep_capacity(g, ps, _profiles(gold), _cfg(gold), [])
