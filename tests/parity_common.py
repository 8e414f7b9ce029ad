"""Shared setup for GPU-vs-oracle parity tests (test-only code).

Builds one synthetic workload twice: through the product host path (native
preprocessing) for ``train()``, and through the CPU oracle for the expected
values; the integer inputs are asserted identical first.
"""

from __future__ import annotations

import numpy as np

from oracle import halo_port as ohp
from oracle import model_port as omp
from paper_2508_13716_b200 import hostgraph as H


def workload(n, deg, P, hops=1, seed=0):
    g = H.erdos_renyi(n, deg, seed)
    ps = H.build_partition_set(g, H.random_partition(n, P, seed), hops)
    og = ohp.er_graph(n, deg, seed)
    ops = ohp.partition_set(og, ohp.random_assignment(n, P, seed), hops)
    assert np.array_equal(og.in_tgt, g.in_targets)
    assert all(np.array_equal(a, b) for a, b in zip(ops.halo, ps.halo))
    return g, ps, og, ops


def oracle_run_forced(og, ops, kind, f_dim, C, caps, policy, s, params_per_epoch, seed_w=2):
    """Oracle epochs driven by the GPU's weights at the start of each epoch."""
    verts, _, _, score = ohp.influence(og, ops)
    ranked = ohp.ranked_halos(ops, verts, score)
    imp = {int(v): float(x) for v, x in zip(verts, score)}
    pr = ohp.plan_epochs(policy, (caps.c_cpu, tuple(caps.c_gpu), caps.bytes_per_entry),
                         ranked, ops.halo, imp, len(params_per_epoch), s)
    dims = list(f_dim) + [C]
    tr = omp.Trainer(og, ops.inner, ops.halo, omp.ModelSpec(kind, dims),
                     omp.features(og.n, dims[0], seed=0), omp.labels(og.n, C, seed=1),
                     params=omp.init_params(kind, dims, seed_w))
    outs = [tr.step(p.version, forced_params=w) for p, w in zip(pr.plans, params_per_epoch)]
    return pr, outs


def oracle_run(og, ops, kind, f_dim, C, caps, policy, s, epochs, seed_w=2):
    verts, _, _, score = ohp.influence(og, ops)
    ranked = ohp.ranked_halos(ops, verts, score)
    imp = {int(v): float(x) for v, x in zip(verts, score)}
    pr = ohp.plan_epochs(policy, (caps.c_cpu, tuple(caps.c_gpu), caps.bytes_per_entry),
                         ranked, ops.halo, imp, epochs, s)
    dims = list(f_dim) + [C]
    spec = omp.ModelSpec(kind, dims)
    X = omp.features(og.n, dims[0], seed=0)
    y = omp.labels(og.n, C, seed=1)
    outs, params = omp.partitioned_epochs(og, ops.inner, ops.halo,
                                          [p.version for p in pr.plans], spec, X, y,
                                          params=omp.init_params(kind, dims, seed_w))
    return pr, outs, params


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))
