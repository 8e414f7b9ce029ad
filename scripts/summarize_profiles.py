#!/usr/bin/env python
"""Copy one gpurun round's evidence into profiles/<tag>/ (tracked).

    python scripts/summarize_profiles.py gpurun_out/r01a profiles/r01

Writes the bench lines, the launch list + its per-kernel summary, and for
every ncu --set full capture (prof_*.ncu-rep) a CSV of the metrics the
roofline uses (duration, DRAM bytes, DRAM / tensor-pipe utilisation, L2 hit
rate, occupancy).  Also refreshes profiles/spmm_traffic.json, which bench.py
reads for the roofline "traffic" field.
"""

from __future__ import annotations

import csv
import io
import json
import os
import shutil
import subprocess
import sys

METRICS = [
    ("kernel", "Kernel Name"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("regs", "launch__registers_per_thread"),
    ("duration", "gpu__time_duration.sum"),
    ("dram_read", "dram__bytes_read.sum"),
    ("dram_write", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
]
ORDER = ["kernel", "grid", "block", "regs", "duration_s", "dram_read_B", "dram_write_B",
         "dram_pct", "tensor_pct", "sm_pct", "l2_hit_pct", "warps_active_pct"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3,
         "ns": 1e-9, "s": 1.0}


def ncu_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for key, name in METRICS:
            if name not in hdr:
                continue
            i = hdr.index(name)
            v = r[i]
            if key == "kernel":
                d[key] = v.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                d[key] = v
                continue
            u = units[i]
            if u in SCALE:
                x *= SCALE[u]
                key = {"duration": "duration_s", "dram_read": "dram_read_B",
                       "dram_write": "dram_write_B"}.get(key, key)
            d[key] = x
        res.append(d)
    return res


def main(src: str, dst: str):
    os.makedirs(dst, exist_ok=True)
    for f in ("bench.json", "bench_ref.json", "launches.csv", "launches_summary.txt",
              "pytest_gpu.log", "smoke.log", "nvidia-smi.txt", "nproc.txt", "bench_c4.json",
              "bench_scaled.json", "clocks.csv"):
        p = os.path.join(src, f)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(dst, f))
    traffic = None
    for f in sorted(os.listdir(src)):
        if not f.endswith(".ncu-rep"):
            continue
        rows = ncu_rows(os.path.join(src, f))
        name = f[:-len(".ncu-rep")]
        with open(os.path.join(dst, f"ncu_{name}.csv"), "w", newline="") as fh:
            present = {k for r in rows for k in r}
            keys = [k for k in ORDER if k in present]
            w = csv.DictWriter(fh, fieldnames=keys)
            w.writeheader()
            w.writerows(rows)
        if name == "prof_spmm" and rows:
            tot = sum(r.get("dram_read_B", 0) + r.get("dram_write_B", 0) for r in rows)
            dur = sum(r.get("duration_s", 0) for r in rows)
            traffic = {"source": f"{dst}/ncu_{name}.csv", "config": "c2",
                       "launches": len(rows),
                       "dram_bytes_per_epoch": tot,
                       "dram_bytes_per_launch": tot / len(rows),
                       "ncu_seconds_per_epoch": dur,
                       "note": "ncu --set full, one epoch of SpMM launches (k_spmm_cpa / "
                               "k_spmm: 3 fwd + 2 bwd aggregations, wide ones as 128-column "
                               "slices = 8 launches on C2), cold cache, serialised"}
    if traffic:
        with open(os.path.join(os.path.dirname(dst.rstrip("/")) or ".", "spmm_traffic.json"),
                  "w") as fh:
            json.dump(traffic, fh, indent=1)
    print("wrote", dst)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
