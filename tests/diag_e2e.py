"""Diagnostic (not a test): the C2 end-to-end step (pinned-host input H2D +
epoch + loss D2H) in isolation -- host enqueue time per step, wall time per
step, and the bare H2D rate of the same buffer with and without the epoch
beside it.  Prints one line per measurement."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2508_13716_b200 import api, hostgraph as H  # noqa: E402
from paper_2508_13716_b200.models import _unit  # noqa: E402


def main():
    torch.cuda.set_device(0)
    print("affinity", sorted(os.sched_getaffinity(0)), flush=True)
    g, ps, caps = bench.build_workload(8)
    cfg = H.SimConfig(epochs=200, policy="jaca", staleness_bound=-1, f_dim=bench.F_DIM, L=3)
    sess = api.TrainSession(g, ps, H.unit_profiles(8), caps, cfg, model="gcn", num_classes=40,
                            gemm="3xtf32", keep_logits="none")
    eng = sess.engine
    rows = eng.D.verts.astype(np.uint64)[:, None]
    hx = torch.from_numpy(_unit(0, rows, np.arange(bench.F_DIM[0], dtype=np.uint64)[None, :]))
    hx = hx.pin_memory()
    loss = torch.empty(64).pin_memory()
    for _ in range(4):
        sess.step()
    d = torch.empty_like(hx, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            d.copy_(hx, non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 20
        print(f"h2d alone {hx.numel() * 4 / dt / 1e9:.1f} GB/s", flush=True)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sess.prefetch_features(hx)
        enq = 0.0
        for i in range(20):
            a = time.perf_counter()
            s = sess.step(sync=False)
            if i + 1 < 20:
                sess.prefetch_features(hx)
            sess.fetch_loss(s, loss[i:i + 1])
            enq += time.perf_counter() - a
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / 20
        sess.finish()
        print(f"e2e {wall * 1e3:.3f} ms/step, host enqueue {enq / 20 * 1e3:.3f} ms/step", flush=True)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(20):
            sess.step(sync=False)
        torch.cuda.synchronize()
        print(f"epochs only {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms/step", flush=True)
        sess.finish()


if __name__ == "__main__":
    main()
