"""Diagnostic (not a test): C1 (BASELINE configs[0]) trains with the automatic
transform-first last layer (on at C1's density) and aggregate-first, and
prints the logits / loss differences per epoch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13716_b200 import api, hostgraph as H  # noqa: E402


def run(tfl):
    os.environ["CG_TFL"] = tfl
    n, P, f = 10000, 4, (128, 128)
    g = H.erdos_renyi(n, 20.0, 0)
    ps = H.build_partition_set(g, H.random_partition(n, P, 0), 1)
    caps = H.compute_capacities(ps, -1, [180.0] * P, 1024.0, 64.0, 2048.0, f, 2)
    cfg = H.SimConfig(epochs=5, policy="jaca", staleness_bound=-1, f_dim=f, L=2)
    rep = api.train(g, ps, H.unit_profiles(P), caps, cfg, model="gcn", num_classes=40,
                    keep_logits="all")
    return rep


a, b = run("0"), run("1")
for e in range(5):
    la, lb = a.logits_per_epoch[e], b.logits_per_epoch[e]
    print(f"epoch {e + 1}: logits rel {np.abs(la - lb).max() / np.abs(la).max():.2e}, "
          f"loss {a.losses[e]:.7f} vs {b.losses[e]:.7f}")
