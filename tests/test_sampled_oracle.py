"""The sampled-row oracle (oracle/sampled_port.py, used at the C3/C4 shapes)
agrees with the whole-graph partitioned oracle (model_port.Trainer) on the
rows it samples, for the plan it models (Algorithm-1 capacities, s = -1:
every halo read is the version-0 snapshot), GCN and GraphSAGE, over
weight-forced epochs."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import halo_port as ohp
from oracle import model_port as omp
from oracle import sampled_port as osp


@pytest.mark.parametrize("kind,hops", [("gcn", 1), ("sage", 2)])
def test_sampled_matches_partitioned_oracle(kind, hops):
    n, P = 600, 4
    og = ohp.er_graph(n, 7.0, 0)
    parts = ohp.random_assignment(n, P, 0)
    ops = ohp.partition_set(og, parts, hops)
    dims = [12, 16, 16, 5] if kind == "gcn" else [12, 16, 5]
    rng = np.random.default_rng(3)
    p0 = omp.init_params(kind, dims, 2)
    p1 = [x + 0.05 * rng.standard_normal(x.shape).astype(np.float32) for x in p0]
    p2 = [x + 0.05 * rng.standard_normal(x.shape).astype(np.float32) for x in p1]
    tr = omp.Trainer(og, ops.inner, ops.halo, omp.ModelSpec(kind, dims),
                     omp.features(n, dims[0], 0), omp.labels(n, dims[-1], 1), params=p0)
    ver0 = [np.zeros(h.size, np.int64) for h in ops.halo]   # every read: warm version 0
    full = [tr.step(ver0, forced_params=w).logits for w in (p0, p1, p2)]
    sg = osp.SampledGraph(og.in_off, og.in_tgt, parts, kind)
    samples = rng.choice(n, 40, replace=False)
    s, got = osp.sampled_logits(sg, dims, [p0, p1, p2], samples)
    for e in range(3):
        np.testing.assert_allclose(got[e], full[e][s], rtol=0, atol=1e-12 * max(
            1.0, np.abs(full[e]).max()))
