"""Epoch graphs: steady-state epochs replayed from captured CUDA graphs must be
bit-identical to the eager launches (same kernels, same order; the epoch
number and Adam's bias corrections come from device memory instead of
kernel arguments).  The parity suite (test_gpu_train_parity.py) runs with
graphs on, so this file only pins graph == eager exactly, including the
staleness-window cases where the K6 plan changes from epoch to epoch."""

from __future__ import annotations

import numpy as np
import pytest

from parity_common import workload

pytestmark = pytest.mark.gpu

CASES = [
    # kind, n, deg, P, f_dim, C, capacity, policy, s, epochs, gemm
    ("gcn", 500, 6.0, 4, (16, 32, 32), 7, "auto", "jaca", -1, 6, "3xtf32"),
    ("gcn", 500, 5.0, 3, (16, 32, 32), 6, 60, "jaca", 1, 7, "3xtf32"),
    ("sage", 500, 5.0, 3, (16, 32), 6, 60, "jaca", 2, 7, "fp32"),
    ("sage", 500, 6.0, 4, (64, 32, 32), 7, "auto", "jaca", -1, 5, "3xtf32"),   # layer-0 tf0
]


def _run(case, graphs):
    from paper_2508_13716_b200 import api, hostgraph as H
    kind, n, deg, P, f_dim, C, cap, policy, s, epochs, gemm = case
    g, ps, _, _ = workload(n, deg, P)
    from test_gpu_train_parity import make_caps
    caps = make_caps(H, ps, cap, f_dim)
    cfg = H.SimConfig(epochs=epochs, policy=policy, staleness_bound=s, f_dim=f_dim, L=len(f_dim))
    rep = api.train(g, ps, H.unit_profiles(P), caps, cfg, model=kind, num_classes=C,
                    keep_logits="all", keep_params=True, record_trace=True, gemm=gemm,
                    graphs=graphs)
    return rep


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[7]}-s{c[8]}-{c[10]}")
def test_graph_epochs_bit_identical_to_eager(case):
    eager, graph = _run(case, False), _run(case, True)
    assert [r.__dict__ for r in graph.records] == [r.__dict__ for r in eager.records]
    assert graph.trace_csv == eager.trace_csv
    assert graph.planner == eager.planner and "gpu" in graph.planner
    assert graph.losses == eager.losses
    for a, b in zip(graph.logits_per_epoch, eager.logits_per_epoch):
        assert np.array_equal(a, b)
    for a, b in zip(graph.params, eager.params):
        assert np.array_equal(a, b)


def test_graph_session_io_pipeline():
    """TrainSession with host I/O (prefetch_features / fetch_logits /
    fetch_loss) around graph replays equals the eager session."""
    import torch
    from paper_2508_13716_b200 import api, hostgraph as H
    from paper_2508_13716_b200.models import _unit
    f_dim, C, P = (16, 32, 32), 7, 4
    g, ps, _, _ = workload(600, 6.0, P)
    caps = H.compute_capacities(ps, -1, [180.0] * P, 1024.0, 64.0, 2048.0, f_dim, 3)
    cfg = H.SimConfig(epochs=6, policy="jaca", staleness_bound=-1, f_dim=f_dim, L=3)
    out = {}
    for graphs in (False, True):
        with api.TrainSession(g, ps, H.unit_profiles(P), caps, cfg, model="gcn", num_classes=C,
                              gemm="3xtf32", keep_logits="none", graphs=graphs) as sess:
            eng = sess.engine
            rows = eng.D.verts.astype(np.uint64)[:, None]
            hx = torch.from_numpy(_unit(0, rows, np.arange(f_dim[0], dtype=np.uint64)[None, :]))
            hx = hx.pin_memory()
            logits = [torch.empty(eng.D.n_in, eng.C4).pin_memory() for _ in range(6)]
            loss = torch.empty(6).pin_memory()
            sess.prefetch_features(hx)
            for i in range(6):
                s = sess.step(sync=False)
                if i + 1 < 6:
                    sess.prefetch_features(hx)
                sess.fetch_logits(logits[i])
                sess.fetch_loss(s, loss[i:i + 1])
            torch.cuda.synchronize()
            sess.finish()
            out[graphs] = ([x.numpy().copy() for x in logits], loss.numpy().copy(),
                           sess.report().losses)
    (la, sa, ra), (lb, sb, rb) = out[False], out[True]
    assert ra == rb
    assert np.array_equal(sa, sb)
    for a, b in zip(la, lb):
        assert np.array_equal(a, b)


PF_CASES = [c for c in CASES if c[6] != "auto"] + [
    ("gcn", 600, 6.0, 4, (16, 32, 32), 7, 40, "jaca", 1, 6, "3xtf32"),
    ("gcn", 600, 6.0, 4, (16, 32, 32), 7, 40, "fifo", 2, 6, "3xtf32"),
    ("gcn", 500, 5.0, 4, (16, 32, 32), 6, (20, 200), "jaca", 1, 5, "3xtf32"),
    ("sage", 600, 6.0, 4, (16, 32, 32), 6, (40, 300), "jaca", 2, 6, "fp32"),
]


@pytest.mark.parametrize("case", PF_CASES, ids=lambda c: f"{c[0]}-{c[7]}-s{c[8]}-cap{c[6]}")
@pytest.mark.parametrize("graphs", [False, True], ids=["eager", "graphs"])
def test_prefetch_queue_bit_identical(case, graphs, monkeypatch):
    """R10: staging rows copied ahead on the prefetch stream (pinned-tier
    rows of every layer, all layer-0 rows) give exactly the results of the
    all-in-line staging (same rows, same values; only the stream differs)."""
    monkeypatch.setenv("CG_PREFETCH", "0")
    inline = _run(case, graphs)
    monkeypatch.setenv("CG_PREFETCH", "1")
    pf = _run(case, graphs)
    assert [r.__dict__ for r in pf.records] == [r.__dict__ for r in inline.records]
    assert sum(r.global_hits for r in pf.records) > 0   # the host tier is read
    assert pf.losses == inline.losses
    for a, b in zip(pf.logits_per_epoch, inline.logits_per_epoch):
        assert np.array_equal(a, b)
    for a, b in zip(pf.params, inline.params):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["gcn", "sage"])
def test_last_layer_transform_first_graph_equals_eager(kind, monkeypatch):
    """The transform-first last layer (forced on: the test graph is too sparse
    for the auto rule) replays bit-identically from the epoch graphs."""
    monkeypatch.setenv("CG_TFL", "1")
    case = (kind, 600, 6.0, 4, (16, 32, 32), 7, "auto", "jaca", -1, 5, "3xtf32")
    eager, graph = _run(case, False), _run(case, True)
    assert graph.losses == eager.losses
    for a, b in zip(graph.logits_per_epoch, eager.logits_per_epoch):
        assert np.array_equal(a, b)
    for a, b in zip(graph.params, eager.params):
        assert np.array_equal(a, b)
