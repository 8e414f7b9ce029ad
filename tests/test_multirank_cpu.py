"""World-size-2 host logic of the N>1 path, on CPU over gloo.

Each rank builds the run layout for 2 devices and checks, against the other
rank's data gathered over gloo, that every cross-device address it will
hand to the K3 staging kernel (forward halo pulls and backward gradient
pulls) names the right vertex on the owner, that the union of both ranks'
forward CSRs is the single-device CSR (same neighbour multiset per vertex),
that the redundant per-rank cache planners agree, and that the DistComm K7
all-reduce / object broadcast behave.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
from paper_2508_13716_b200 import hostgraph as H
from paper_2508_13716_b200.layout import build_layout
from paper_2508_13716_b200.planner import SequentialPlanner
from paper_2508_13716_b200.comm import DistComm

n, P = 700, 4
g = H.erdos_renyi(n, 6.0, 0)
ps = H.build_partition_set(g, H.random_partition(n, P, 0), 1)
inner = [np.asarray(x, np.int64) for x in ps.inner]
halo = [np.asarray(h, np.int64) for h in ps.halo]
caps = H.uniform_capacities(ps, 90, (16, 16))
for kind in ("gcn", "sage"):
    L2 = build_layout(g, inner, halo, caps.c_gpu, world, kind)
    L1 = build_layout(g, inner, halo, caps.c_gpu, 1, kind)
    D = L2.devices[rank]
    verts_all = [None] * world
    dist.all_gather_object(verts_all, D.verts)
    # forward: owner tables address the right vertex
    for u, od, orow in zip(L2.union, L2.owner_dev, L2.owner_row):
        assert verts_all[od][orow] == u
    # backward: remote gradient rows are pulled from the right owner row
    for v, sd, sr in zip(D.bwd_stage_vertex, D.bwd_src_dev, D.bwd_src_row):
        assert sd != rank and verts_all[sd][sr] == v
    # forward CSR: same neighbour lists as the single-device layout
    D1 = L1.devices[0]
    row1 = {{int(v): i for i, v in enumerate(D1.verts)}}
    def nbrs(DL, r):
        out = []
        for c in DL.fwd_col[DL.fwd_rowptr[r]:DL.fwd_rowptr[r + 1]]:
            out.append(int(DL.verts[c]) if c < DL.n_in else int(DL.halo_vertex[c - DL.n_in]))
        return sorted(out)
    for r, v in enumerate(D.verts):
        assert nbrs(D, r) == nbrs(D1, row1[int(v)]), (kind, v)
    assert np.array_equal(D.norm_dst, D1.norm_dst[[row1[int(v)] for v in D.verts]])
    # backward CSR: per inner row the same number of out-edges
    bdeg = np.diff(D.bwd_rowptr)
    bdeg1 = np.diff(D1.bwd_rowptr)[[row1[int(v)] for v in D.verts]]
    assert np.array_equal(bdeg, bdeg1)

# redundant planners agree across ranks
union, score = H.influence_scores(g, ps)
ranked = [h[np.lexsort((h, -score[np.searchsorted(union, h)]))] for h in ps.halo]
pl = SequentialPlanner("jaca", caps.c_cpu, caps.c_gpu, union, score, halo, ranked)
pl.warm()
counts = np.stack([pl.epoch(e, 1).counts for e in range(1, 5)])
allc = [None] * world
dist.all_gather_object(allc, counts)
assert all(np.array_equal(allc[0], c) for c in allc)

# DistComm over gloo: K7 sum + object broadcast
comm = DistComm(0)
t = torch.arange(5, dtype=torch.float32) * (rank + 1)
comm.allreduce_(t)
assert torch.equal(t, torch.arange(5, dtype=torch.float32) * 3)
assert comm.broadcast_obj("tok" if rank == 0 else None) == "tok"
comm.host_barrier()
dist.destroy_process_group()
print("rank", rank, "ok")
"""


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_world2_gloo_layout_and_plan():
    with tempfile.TemporaryDirectory() as tmp:
        script = os.path.join(tmp, "worker.py")
        with open(script, "w") as fh:
            fh.write(WORKER.format(root=ROOT))
        port = _free_port()
        procs = [subprocess.Popen([sys.executable, script],
                                  env=dict(os.environ, RANK=str(r), WORLD_SIZE="2",
                                           MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                                           CUDA_VISIBLE_DEVICES=""),
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
                 for r in range(2)]
        logs = []
        for p in procs:
            try:
                o, _ = p.communicate(timeout=300)
            except subprocess.TimeoutExpired:
                p.kill()
                o, _ = p.communicate()
            logs.append(o.decode(errors="replace"))
        assert all(p.returncode == 0 for p in procs), "\n----\n".join(logs)[-4000:]
        assert all("ok" in lg for lg in logs)
