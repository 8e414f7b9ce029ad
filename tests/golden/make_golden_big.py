"""Golden fixtures at the large BASELINE.json shapes (C4 products-shaped, C3
Reddit-shaped), produced by running the REFERENCE halopart package here.

Run in the build container only (it imports halopart from /root/reference,
read-only, without installing it); takes ~30-60 min and ~20 GB of RAM:

    python tests/golden/make_golden_big.py [c4] [c3]

Outputs (committed): tests/golden/c4.json, tests/golden/c3.json -- digests
only (graph CSR, partition, halos, stats, influence scores, warm ranking,
Algorithm-1 capacities, RAPA on measured B200 rows, and per-run SimReport
JSON/CSV/trace sha256 + records).  Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import graph_digest, hp, ps_digest, run_case, sha, trace_codes  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(HERE))


def b200_profiles(P):
    # the K9-measured B200 rows (profiles/r01/b200_devices.json), one per slot
    with open(os.path.join(ROOT, "profiles", "r01", "b200_devices.json")) as fh:
        rows = json.load(fh)
    r = rows[0]
    return [hp.DeviceProfile(id=f"b200-{i}", mm_s=r["mm_s"], spmm_s=r["spmm_s"], h2d_s=r["h2d_s"],
                             d2h_s=r["d2h_s"], idt_s=r["idt_s"], mem_gb=r["mem_gb"])
            for i in range(P)]


def big(name, n, n_edges, P, hops, f_dim, cases, rapa=False):
    t0 = time.perf_counter()
    g = hp.erdos_renyi(n, n_edges / n, seed=0)
    a = hp.prepartition(g, P, "random", seed=0)
    ps = hp.build_partition_set(g, a, hops)
    table = hp.influence_scores(g, ps)
    out = {"graph": graph_digest(g), "parts_sha": sha(a.parts.astype(np.int64)),
           "partitions": ps_digest(ps, table), "f_dim": list(f_dim), "hops": hops,
           "setup_seconds": time.perf_counter() - t0, "runs": {}, "numpy": np.__version__}
    print(name, "setup", f"{out['setup_seconds']:.0f}s", flush=True)
    L = len(f_dim)
    if rapa:
        t1 = time.perf_counter()
        res = hp.rapa_refine(ps, b200_profiles(P), f_dim=float(f_dim[0]))
        out["rapa"] = {"sigma": [int(s) for s in res.sigma],
                       "halo_sizes": [int(h.size) for h in res.partitions.halo],
                       "halo_sha": sha(np.concatenate(res.partitions.halo).astype(np.int64)),
                       "seconds": time.perf_counter() - t1}
        print(name, "rapa", out["rapa"]["sigma"], flush=True)
    auto = hp.compute_capacities(ps, k=-1, mem_gpu=[180.0] * P, mem_gpu_res=1024.0,
                                 mem_cpu=64.0, mem_cpu_res=2048.0, f_dim=f_dim, L=L)
    out["auto_caps"] = {"c_cpu": auto.c_cpu, "c_gpu": list(auto.c_gpu)}
    for key, (policy, capspec, s, epochs) in cases.items():
        caps = auto if capspec == "auto" else hp.uniform_capacities(ps, int(capspec), f_dim)
        cfg = hp.SimConfig(epochs=epochs, policy=policy, staleness_bound=s, f_dim=tuple(f_dim),
                           L=L)
        res, rep = run_case(g, ps, caps, cfg, P)
        res["codes_sha"] = sha(trace_codes(rep.trace_csv))
        out["runs"][key] = res
        del rep
        print(name, key, f"{res['seconds']:.1f}s", flush=True)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def main():
    which = sys.argv[1:] or ["c4", "c3"]
    if "c4" in which:
        big("c4", 2449029, 61859140, 8, 1, (100, 256, 256), {
            "auto": ("jaca", "auto", -1, 2),
            "u1000000_s1": ("jaca", 1000000, 1, 3),
        }, rapa=True)
    if "c3" in which:
        big("c3", 232965, 114615892, 8, 2, (604, 256), {
            "auto": ("jaca", "auto", -1, 2),
            "u100000_s0": ("jaca", 100000, 0, 2),
        })


if __name__ == "__main__":
    main()
