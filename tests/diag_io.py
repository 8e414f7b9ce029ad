"""Diagnostic (not a test): PCIe copy rates, copy/compute overlap and the host
enqueue cost of one epoch, on the bench's C2 workload."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2508_13716_b200 import api, hostgraph as H  # noqa: E402


def ev_time(fn, stream=None):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = stream or torch.cuda.current_stream()
    a.record(s)
    fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def main():
    torch.cuda.set_device(0)
    n_in, F = 169343, 128
    hx = torch.randn(n_in, F).pin_memory()
    dx = torch.empty(n_in, F, device="cuda")
    hl = torch.empty(n_in, 40).pin_memory()
    dl = torch.randn(n_in, 40, device="cuda")
    for _ in range(3):
        dx.copy_(hx, non_blocking=True)
        hl.copy_(dl, non_blocking=True)
    torch.cuda.synchronize()
    t = ev_time(lambda: dx.copy_(hx, non_blocking=True))
    print(f"H2D {hx.numel() * 4 / 1e6:.1f} MB: {t:.3f} ms = {hx.numel() * 4 / t / 1e6:.1f} GB/s")
    t = ev_time(lambda: hl.copy_(dl, non_blocking=True))
    print(f"D2H {hl.numel() * 4 / 1e6:.1f} MB: {t:.3f} ms = {hl.numel() * 4 / t / 1e6:.1f} GB/s")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    w = time.perf_counter()
    with torch.cuda.stream(s1):
        dx.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hl.copy_(dl, non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D || D2H wall {1e3 * (time.perf_counter() - w):.3f} ms")

    g, ps, caps = bench.build_workload(8)
    cfg = H.SimConfig(epochs=10, policy="jaca", staleness_bound=-1, f_dim=bench.F_DIM, L=3)
    sess = api.TrainSession(g, ps, H.unit_profiles(8), caps, cfg, model="gcn", num_classes=40,
                            gemm="3xtf32", keep_logits="none", timers=False)
    for _ in range(4):
        sess.step(sync=False)
    torch.cuda.synchronize()
    w = time.perf_counter()
    for _ in range(10):
        sess.step(sync=False)
    enq = (time.perf_counter() - w) / 10
    torch.cuda.synchronize()
    tot = (time.perf_counter() - w) / 10
    print(f"host enqueue {enq * 1e3:.3f} ms/epoch, wall incl. sync {tot * 1e3:.3f} ms/epoch")
    # copy + compute overlap: upload on a side stream while epochs run
    rows = sess.engine.D.verts.astype(np.uint64)[:, None]
    from paper_2508_13716_b200.models import _unit
    hxx = torch.from_numpy(_unit(0, rows, np.arange(F, dtype=np.uint64)[None, :])).pin_memory()
    torch.cuda.synchronize()
    w = time.perf_counter()
    for _ in range(10):
        sess.prefetch_features(hxx)
        sess.step(sync=False)
    torch.cuda.synchronize()
    print(f"epoch + overlapped H2D: {(time.perf_counter() - w) / 10 * 1e3:.3f} ms/epoch")
    hlg = torch.empty(sess.engine.D.n_in, sess.engine.C4).pin_memory()
    torch.cuda.synchronize()
    w = time.perf_counter()
    for _ in range(10):
        sess.step(sync=False)
        sess.fetch_logits(hlg)
    torch.cuda.synchronize()
    print(f"epoch + overlapped logits D2H: {(time.perf_counter() - w) / 10 * 1e3:.3f} ms/epoch")
    sess.finish()
    sess.close()


if __name__ == "__main__" and "--loop" not in sys.argv:
    main()


def bench_loop():
    """The bench's e2e loop with per-stream event timestamps."""
    torch.cuda.set_device(0)
    g, ps, caps = bench.build_workload(8)
    cfg = H.SimConfig(epochs=10, policy="jaca", staleness_bound=-1, f_dim=bench.F_DIM, L=3)
    sess = api.TrainSession(g, ps, H.unit_profiles(8), caps, cfg, model="gcn", num_classes=40,
                            gemm="3xtf32", keep_logits="none", timers=False)
    eng = sess.engine
    for _ in range(4):
        sess.step(sync=False)
    sess.finish()
    from paper_2508_13716_b200.models import _unit
    rows = eng.D.verts.astype(np.uint64)[:, None]
    hx = torch.from_numpy(_unit(0, rows, np.arange(128, dtype=np.uint64)[None, :])).pin_memory()
    hl = [torch.empty(eng.D.n_in, eng.C4).pin_memory() for _ in range(2)]
    hloss = torch.empty(10).pin_memory()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    marks = []
    w = time.perf_counter()
    sess.prefetch_features(hx)
    for i in range(10):
        s = sess.step(sync=False)
        e_end = torch.cuda.Event(enable_timing=True)
        e_end.record()
        if i + 1 < 10:
            sess.prefetch_features(hx)
        e_h2d = torch.cuda.Event(enable_timing=True)
        e_h2d.record(eng._io["h2d"])
        sess.fetch_logits(hl[i & 1])
        sess.fetch_loss(s, hloss[i:i + 1])
        e_d2h = torch.cuda.Event(enable_timing=True)
        e_d2h.record(eng._io["d2h"])
        marks.append((e_end, e_h2d, e_d2h))
    torch.cuda.synchronize()
    print(f"bench loop wall {(time.perf_counter() - w) / 10 * 1e3:.3f} ms/step")
    for i, (a, b, c) in enumerate(marks):
        print(f"step {i}: epoch end {t0.elapsed_time(a):8.3f}  h2d(next) done {t0.elapsed_time(b):8.3f}"
              f"  d2h done {t0.elapsed_time(c):8.3f}")
    sess.finish()
    sess.close()


if __name__ == "__main__" and "--loop" in sys.argv:
    bench_loop()
