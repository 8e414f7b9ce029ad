"""Generate the CLI golden: run the REFERENCE halopart CLI (partition, then
simulate) on a small synthetic graph and record its outputs.

Build container only (imports halopart from /root/reference, read-only):

    python tests/golden/make_cli_golden.py

Writes tests/golden/cli/: graph.txt (edge list), devices.json (a 3090/3060 mix
so RAPA prunes halos), rapa.json (the reference's partition output) and
expected.json (sha256 + bytes of the reference's sim_report.json / .csv for
the simulate flags recorded there).  `train` must reproduce those bytes.
"""

from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")
sys.path.insert(0, REF)
import halopart as hp  # noqa: E402

SIM_FLAGS = ["--epochs", "5", "--staleness", "1", "--capacity", "40", "--fdim", "16,32",
             "--layers", "2", "--policy", "jaca"]

BENCH_FLAGS = ["--epochs", "4", "--staleness", "1", "--fdim", "16,32", "--layers", "2",
               "--policies", "jaca,fifo,lru", "--capacities", "0,20,40,200"]


def main():
    os.makedirs(HERE, exist_ok=True)
    g = hp.erdos_renyi(400, 8.0, seed=3)   # every vertex has an edge (contiguous ids)
    src = np.repeat(np.arange(g.n_vertices), np.diff(g.out_offsets))
    assert np.union1d(src, g.out_targets).size == g.n_vertices
    with open(os.path.join(HERE, "graph.txt"), "w") as fh:
        fh.write("# synthetic ER graph, n=400, avg degree 8, seed 3\n")
        for u, v in zip(src, g.out_targets):
            fh.write(f"{u} {v}\n")
    devs = [{"id": "3090-a", "mm_s": 0.14, "spmm_s": 0.106, "h2d_s": 0.118, "d2h_s": 0.121,
             "idt_s": 0.0014, "mem_gb": 24},
            {"id": "3090-b", "mm_s": 0.138, "spmm_s": 0.105, "h2d_s": 0.119, "d2h_s": 0.12,
             "idt_s": 0.0014, "mem_gb": 24},
            {"id": "3060-a", "mm_s": 0.34, "spmm_s": 0.195, "h2d_s": 0.122, "d2h_s": 0.124,
             "idt_s": 0.0038, "mem_gb": 8},
            {"id": "3060-b", "mm_s": 0.348, "spmm_s": 0.197, "h2d_s": 0.122, "d2h_s": 0.123,
             "idt_s": 0.0038, "mem_gb": 8}]
    with open(os.path.join(HERE, "devices.json"), "w") as fh:
        json.dump(devs, fh, indent=1)
    env = dict(os.environ, PYTHONPATH=REF)
    with tempfile.TemporaryDirectory() as tmp:
        run = lambda *a: subprocess.run([sys.executable, "-m", "halopart.cli", *a], env=env,  # noqa: E731
                                        check=False, capture_output=True, text=True)
        r = run("partition", "--graph", os.path.join(HERE, "graph.txt"), "--partitions", "4",
                "--devices", os.path.join(HERE, "devices.json"), "--fdim", "16,32",
                "--out", os.path.join(tmp, "part"))
        assert r.returncode == 0, r.stderr
        rapa = open(os.path.join(tmp, "part", "rapa.json"), "rb").read()
        with open(os.path.join(HERE, "rapa.json"), "wb") as fh:
            fh.write(rapa)
        r = run("simulate", "--graph", os.path.join(HERE, "graph.txt"), "--partition-result",
                os.path.join(HERE, "rapa.json"), "--devices", os.path.join(HERE, "devices.json"),
                *SIM_FLAGS, "--out", os.path.join(tmp, "sim"))
        assert r.returncode == 0, r.stderr
        js = open(os.path.join(tmp, "sim", "sim_report.json"), "rb").read()
        cs = open(os.path.join(tmp, "sim", "sim_report.csv"), "rb").read()
        r = run("cache-bench", "--graph", os.path.join(HERE, "graph.txt"), "--partition-result",
                os.path.join(HERE, "rapa.json"), "--devices", os.path.join(HERE, "devices.json"),
                *BENCH_FLAGS, "--out", os.path.join(tmp, "bench"))
        assert r.returncode == 0, r.stderr
        cmp_csv = open(os.path.join(tmp, "bench", "compare.csv"), "rb").read()
    doc = json.loads(rapa)
    pruned = sum(1 for p in doc["partitions"] if len(p["halo"]) == 0)
    exp = {"sim_flags": SIM_FLAGS, "reference": "halopart " + hp.__version__,
           "numpy": np.__version__,
           "sim_report_json_sha256": hashlib.sha256(js).hexdigest(),
           "sim_report_csv_sha256": hashlib.sha256(cs).hexdigest(),
           "sigma": doc["sigma"], "feasible": doc["feasible"],
           "halo_sizes": [len(p["halo"]) for p in doc["partitions"]],
           "rapa_json_sha256": hashlib.sha256(rapa).hexdigest(),
           "bench_flags": BENCH_FLAGS, "compare_csv": cmp_csv.decode("utf-8")}
    with open(os.path.join(HERE, "expected.json"), "w") as fh:
        json.dump(exp, fh, indent=1)
    print(json.dumps(exp, indent=1), "empty halos:", pruned)


if __name__ == "__main__":
    main()
