"""bench.py's CPU legs on the host (no GPU): the reference arm runs the CPU
path of the workload -- planner port + PyTorch-CPU fp32 epoch -- built from
oracle objects only, so no library of this repo is mapped into it."""

from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_is_cpu_only_and_maps_no_repo_library():
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--steps", "2",
           "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["repo_libs_mapped"] == []
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["plan_s"] > 0 and cb["train_s"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["partitions"] == 4
