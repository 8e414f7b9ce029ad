"""Diagnostic (not a test): per-epoch logits error vs the oracle, both GEMM
modes, to see the margin under the 1e-4 parity bound."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from parity_common import oracle_run, oracle_run_forced, rel_err, workload  # noqa: E402
from paper_2508_13716_b200 import api, hostgraph as H  # noqa: E402

g, ps, og, ops = workload(700, 6.0, 4)
f_dim, C = (32, 64, 64), 10
caps = H.uniform_capacities(ps, 150, f_dim)
cfg = H.SimConfig(epochs=6, policy="jaca", staleness_bound=1, f_dim=f_dim, L=3)
for kind in ("gcn", "sage"):
    for gemm in ("fp32", "3xtf32"):
        rep = api.train(g, ps, H.unit_profiles(4), caps, cfg, model=kind, num_classes=C,
                        keep_logits="all", gemm=gemm, keep_params=True)
        _, outs = oracle_run_forced(og, ops, kind, f_dim, C, caps, "jaca", 1, rep.params_per_epoch)
        errs = [rel_err(rep.logits_per_epoch[e], o.logits) for e, o in enumerate(outs)]
        _, free, _ = oracle_run(og, ops, kind, f_dim, C, caps, "jaca", 1, 6)
        ferrs = [rel_err(rep.logits_per_epoch[e], o.logits) for e, o in enumerate(free)]
        print(kind, gemm, "forced", " ".join(f"{x:.1e}" for x in errs), "| free",
              " ".join(f"{x:.1e}" for x in ferrs), flush=True)
