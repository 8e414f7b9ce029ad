"""Run the bench's exchange configuration alone (C2, uniform capacity 40,000
per level, s = 1: misses, stale global hits, slab and host-tier
write-through) for a fixed number of epochs -- the command ncu profiles K3
(k_copy_rows) under:

    ncu --set full -k regex:k_copy_rows --launch-skip 40 -c 6 \\
        python scripts/exchange_probe.py
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(epochs: int = 10) -> None:
    import bench
    from paper_2508_13716_b200 import api, hostgraph as H
    bench.apply_config("c2")
    g, ps, _ = bench.build_workload(8)
    caps = H.uniform_capacities(ps, bench.EXCHANGE_CAP, bench.F_DIM)
    cfg = H.SimConfig(epochs=epochs, policy="jaca", staleness_bound=bench.EXCHANGE_S,
                      f_dim=bench.F_DIM, L=len(bench.F_DIM))
    with api.TrainSession(g, ps, H.unit_profiles(ps.P), caps, cfg, model=bench.MODEL,
                          num_classes=bench.CLASSES, keep_logits="none") as sess:
        for _ in range(epochs):
            st = sess.step()
            print(f"epoch {st.epoch}: {st.seconds * 1e3:.3f} ms, planner {st.planner}",
                  flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 10)
