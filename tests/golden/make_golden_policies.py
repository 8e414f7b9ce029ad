"""Golden fixtures for the policy / capacity sweeps (simulator.py:259-322),
produced by running the REFERENCE halopart package here.

    python tests/golden/make_golden_policies.py

Output (committed): tests/golden/policies.json -- the CSV of
``compare_policies`` (policy x capacity grid) and the SimReport JSON / CSV
sha256 of every ``sweep_capacity`` run on the C1 workload (ER 10,000 v /
200,000 e, P = 4) with a heterogeneous device list, so the cost-model fields
(compute / comm / residual times, makespans) are exercised too.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import hp, sha  # noqa: E402

PROFILES = [  # (id, mm_s, spmm_s, h2d_s, d2h_s, idt_s, mem_gb)
    ("a", 1.0, 1.0, 1.0, 1.0, 1.0, 24.0),
    ("b", 0.7, 0.9, 1.3, 1.2, 0.8, 24.0),
    ("c", 1.6, 1.1, 0.9, 1.0, 1.4, 48.0),
    ("d", 0.5, 0.6, 1.1, 1.1, 0.6, 80.0),
]
CFG = dict(epochs=4, staleness_bound=1, f_dim=(128, 128), L=2, prefetch_depth=2000, alpha=0.4)
COMPARE_CAPS = (0, 1000, 3730, 8000)
SWEEP_CAPS = (0, 2000, 3730)


def main():
    g = hp.erdos_renyi(10000, 20.0, seed=0)
    ps = hp.build_partition_set(g, hp.prepartition(g, 4, "random", seed=0), 1)
    profiles = [hp.DeviceProfile(id=i, mm_s=a, spmm_s=b, h2d_s=c, d2h_s=d, idt_s=e, mem_gb=m)
                for i, a, b, c, d, e, m in PROFILES]
    cfg = hp.SimConfig(policy="jaca", **CFG)
    table = hp.compare_policies(g, ps, profiles, cfg, capacities=COMPARE_CAPS)
    reps = hp.sweep_capacity(g, ps, profiles, cfg, SWEEP_CAPS)
    out = {"profiles": PROFILES, "cfg": {k: list(v) if isinstance(v, tuple) else v
                                         for k, v in CFG.items()},
           "compare_caps": list(COMPARE_CAPS), "sweep_caps": list(SWEEP_CAPS),
           "compare_csv": table.to_csv(), "compare_csv_sha": sha(table.to_csv()),
           "sweep": [{"capacity": c, "report_json_sha": sha(r.to_json()),
                      "report_csv_sha": sha(r.to_csv()), "total_time": r.total_time}
                     for c, r in zip(SWEEP_CAPS, reps)]}
    with open(os.path.join(HERE, "policies.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(table.to_csv())


if __name__ == "__main__":
    main()
