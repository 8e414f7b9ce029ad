"""Diagnostic (not a test): how the per-step input upload (86.7 MB H2D) slows
the epoch running beside it, vs a D2D copy of the same bytes and vs none,
and with the H2D split into 1..1024 DMAs.

Findings (profiles/r01/diag_io2.txt): the full-rate H2D adds ~0.2 ms to a
1.85 ms epoch while kernel durations (CUPTI) stay the same -- the time goes
into the gaps between kernels; the D2D costs nothing, so it is not L2
pollution.  Many small DMAs shrink the slowdown only because each piece
carries a fixed cost and the upload as a whole runs slower (bench e2e gets
worse with chunking), so the engine issues one DMA."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2508_13716_b200 import api, hostgraph as H  # noqa: E402


def main():
    torch.cuda.set_device(0)
    g, ps, caps = bench.build_workload(8)
    cfg = H.SimConfig(epochs=100, policy="jaca", staleness_bound=-1, f_dim=bench.F_DIM, L=3)
    sess = api.TrainSession(g, ps, H.unit_profiles(8), caps, cfg, model="gcn", num_classes=40,
                            gemm="3xtf32", keep_logits="none", timers=True)
    for _ in range(4):
        sess.step(sync=True)
    eng = sess.engine
    n, F = eng.D.n_in, 128
    hx = torch.randn(n, F).pin_memory()
    dsrc = torch.randn(n, F, device="cuda")
    dst = torch.empty(n, F, device="cuda")
    side = torch.cuda.Stream()

    def run(mode, k=10, prof=False):
        rows = []
        nch = int(mode[3:]) if mode[:3] in ("h2d", "d2d") and mode[3:] else 8
        for _ in range(k):
            if mode != "none":
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    src = hx if mode.startswith("h2d") else dsrc
                    for c in range(nch):   # chunks so the copy spans the epoch
                        lo, hi = c * n // nch, (c + 1) * n // nch
                        dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
            s = sess.step(sync=True)
            rows.append((s.seconds * 1e3, sum(s.spmm_fwd_ms), sum(s.spmm_bwd_ms)))
        torch.cuda.synchronize()
        a = np.array(rows)
        med = np.median(a, 0)
        print(f"{mode:5s} epoch {med[0]:.3f} ms  spmm fwd {med[1]:.3f}  bwd {med[2]:.3f}  "
              f"other {med[0] - med[1] - med[2]:.3f}", flush=True)

    for mode in ("none", "h2d", "d2d", "h2d1", "h2d64", "h2d256", "h2d1024", "none", "h2d"):
        run(mode)
    # per-kernel durations and launch gaps, concurrent (CUPTI activity trace)
    from torch.profiler import ProfilerActivity, profile
    for mode in ("none", "h2d", "h2d256"):
        with profile(activities=[ProfilerActivity.CUDA]) as p:
            run(mode, k=5)
        evs = [e for e in p.events() if e.device_type.name == "CUDA"]
        ker = sorted([e for e in evs if "Memcpy" not in e.name and "Memset" not in e.name],
                     key=lambda e: e.time_range.start)
        by = {}
        for e in ker:
            key = e.name.split("(")[0][:40]
            by[key] = by.get(key, 0.0) + (e.time_range.end - e.time_range.start) / 5
        busy = sum(by.values())
        print(f"[{mode}] kernel busy {busy / 1e3:.3f} ms/epoch over {len(ker) / 5:.0f} kernels")
        for k_, v in sorted(by.items(), key=lambda kv: -kv[1])[:8]:
            print(f"    {k_:40s} {v:8.1f} us/epoch")
    sess.finish()
    sess.close()


if __name__ == "__main__":
    main()
