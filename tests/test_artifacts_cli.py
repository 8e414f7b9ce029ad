"""Artifact I/O and the CLI (train = drop-in for `halopart simulate`).

CPU: the readers against the reference-produced fixtures in tests/golden/cli
(tests/golden/make_cli_golden.py ran the reference CLI).  GPU: `train` on the
same inputs emits sim_report.json / .csv byte-identical to the reference's.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2508_13716_b200 import artifacts as A
from paper_2508_13716_b200 import cli
from paper_2508_13716_b200 import hostgraph as H
from paper_2508_13716_b200.errors import DomainError, ParseError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "cli")


def _exp():
    with open(os.path.join(GOLD, "expected.json")) as fh:
        return json.load(fh)


def test_edge_list_matches_generator():
    g = A.load_edge_list(os.path.join(GOLD, "graph.txt"))
    ref = H.erdos_renyi(400, 8.0, 3)
    assert g.n_vertices == 400 and g.n_edges == ref.n_edges
    for k in ("out_offsets", "out_targets", "in_offsets", "in_targets"):
        assert np.array_equal(getattr(g, k), getattr(ref, k)), k


def test_edge_list_semantics():
    g = A.load_edge_list(io.StringIO("# c\n0 1\n0 1\n\n1 1\n2 0\n"))
    assert g.n_vertices == 3 and g.n_edges == 3          # duplicate collapsed, self-loop kept
    with pytest.raises(DomainError):
        A.load_edge_list(io.StringIO("0 5\n"))            # gap without compact_ids
    g2 = A.load_edge_list(io.StringIO("10 50\n50 70\n"), compact_ids=True)
    assert g2.n_vertices == 3 and g2.vertex_id_map == {10: 0, 50: 1, 70: 2}
    for bad in ("0 1 2\n", "a b\n", "-1 2\n"):
        with pytest.raises(ParseError):
            A.load_edge_list(io.StringIO(bad))


def test_rapa_import_and_profiles():
    exp = _exp()
    res, ps = A.import_rapa_result(os.path.join(GOLD, "rapa.json"))
    assert list(res.sigma) == exp["sigma"] and res.feasible == exp["feasible"]
    assert [h.size for h in ps.halo] == exp["halo_sizes"]
    assert sum(a.size for a in ps.inner) == 400
    prof = A.load_device_profiles(os.path.join(GOLD, "devices.json"))
    assert [p.id for p in prof] == ["3090-a", "3090-b", "3060-a", "3060-b"]
    with pytest.raises(ParseError):
        A.load_device_profiles(io.StringIO("[]"))
    with pytest.raises(DomainError):
        A.load_device_profiles(io.StringIO('[{"id": "x", "mm_s": 0, "spmm_s": 1, "h2d_s": 1, '
                                           '"d2h_s": 1, "idt_s": 1, "mem_gb": 1}]'))


def test_cli_option_precedence(tmp_path):
    cfgf = tmp_path / "c.json"
    cfgf.write_text(json.dumps({"epochs": 7, "policy": "lru"}))
    args = cli.build_parser().parse_args(["train", "--config", str(cfgf), "--policy", "fifo"])
    opts = cli._options(args, cli._TRAIN_DEFAULTS)
    assert opts["epochs"] == 7 and opts["policy"] == "fifo" and opts["staleness"] == -1
    cfgf.write_text(json.dumps({"bogus": 1}))
    with pytest.raises(ParseError):
        cli._options(args, cli._TRAIN_DEFAULTS)
    assert cli.main(["train"]) == 2                      # missing --graph: exit 2
    assert cli._int_list("128, 256 256") == [128, 256, 256]
    with pytest.raises(ParseError):
        cli._int_list("128,x")


def test_cli_default_fleet_is_halopart_s():
    """Without --devices, train uses the fleet `halopart simulate` uses (its
    bundled reference_devices.json); without halopart it refuses instead of
    silently sizing caches for another fleet."""
    import importlib.util
    if importlib.util.find_spec("halopart") is None:
        with pytest.raises(DomainError):
            cli._load_profiles(None, 4)
    ref_src = "/root/reference/pkg/src"   # build container only
    if not os.path.isdir(ref_src):
        pytest.skip("halopart sources not present (GPU box)")
    code = ("from paper_2508_13716_b200 import cli; p, where, dig = cli._load_profiles(None, 4); "
            "print(len(p), where, dig, p[0].id, p[0].mem_gb)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       env={**os.environ, "PYTHONPATH": ref_src}, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    n, where, dig, pid, mem = r.stdout.split()
    data = open(os.path.join(ref_src, "halopart", "data", "reference_devices.json"), "rb").read()
    assert where == "builtin:reference_devices.json"
    assert dig == hashlib.sha256(data).hexdigest()
    assert int(n) == len(json.loads(data)) and pid == json.loads(data)[0]["id"]


def test_emit_is_all_or_nothing(tmp_path):
    A.emit(tmp_path / "ok", {"a.txt": b"1", "b.txt": b"2"}, {"tool": "t"})
    man = json.loads((tmp_path / "ok" / "manifest.json").read_text())
    assert man["outputs"] == ["a.txt", "b.txt", "manifest.json"]
    assert sorted(p.name for p in (tmp_path / "ok").iterdir()) == ["a.txt", "b.txt",
                                                                   "manifest.json"]
    with pytest.raises(TypeError):
        A.emit(tmp_path / "bad", {"a.txt": b"1", "b.txt": 5}, {"tool": "t"})
    assert list((tmp_path / "bad").iterdir()) == []


@pytest.mark.gpu
def test_cli_train_reproduces_reference_sim_report(tmp_path):
    exp = _exp()
    out = tmp_path / "run"
    cmd = [sys.executable, "-m", "paper_2508_13716_b200.cli", "train",
           "--graph", os.path.join(GOLD, "graph.txt"),
           "--partition-result", os.path.join(GOLD, "rapa.json"),
           "--devices", os.path.join(GOLD, "devices.json"), *exp["sim_flags"],
           "--classes", "7", "--trace", "--out", str(out)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    sha = lambda p: hashlib.sha256((out / p).read_bytes()).hexdigest()  # noqa: E731
    assert sha("sim_report.json") == exp["sim_report_json_sha256"]
    assert sha("sim_report.csv") == exp["sim_report_csv_sha256"]
    tr = json.loads((out / "train_report.json").read_text())
    assert len(tr["losses"]) == 5 and all(np.isfinite(tr["losses"]))
    man = json.loads((out / "manifest.json").read_text())
    assert man["outputs"][-1] == "manifest.json" and "trace.csv" in man["outputs"]


@pytest.mark.gpu
def test_cli_profile_rows_load(tmp_path):
    out = tmp_path / "devices.json"
    assert cli.main(["profile", "--n", "2048", "--reps", "3", "--out", str(out)]) == 0
    rows = A.load_device_profiles(out)
    assert rows and all(p.mm_s > 0 and p.mem_gb > 1 for p in rows)


def test_cli_cache_bench_reproduces_reference_compare_csv(tmp_path):
    """`cache-bench` (plan-only, native planner, no GPU) writes the same
    compare.csv as `halopart cache-bench` on the same inputs."""
    exp = _exp()
    out = tmp_path / "bench"
    rc = cli.main(["cache-bench", "--graph", os.path.join(GOLD, "graph.txt"),
                   "--partition-result", os.path.join(GOLD, "rapa.json"),
                   "--devices", os.path.join(GOLD, "devices.json"), *exp["bench_flags"],
                   "--out", str(out)])
    assert rc == 0
    assert (out / "compare.csv").read_text() == exp["compare_csv"]
    man = json.loads((out / "manifest.json").read_text())
    assert man["command"] == "cache-bench" and man["outputs"][-1] == "manifest.json"
    assert cli.main(["cache-bench", "--graph", os.path.join(GOLD, "graph.txt")]) == 2
