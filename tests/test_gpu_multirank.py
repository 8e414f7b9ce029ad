"""The N>1 path (one process per partition block) on ONE GPU.

Two ranks share cuda:0 over a gloo process group: the layout spreads the
partitions over 2 "devices", peer activation/gradient buffers are exchanged
as CUDA IPC handles and pulled by the K3 staging kernel, the global tier is
the shared-memory segment registered in both processes, barriers and the K7
all-reduce go through DistComm.  (NCCL refuses two ranks on one device, so
the box's single GPU can only exercise this through gloo; the data path --
IPC-mapped peer pointers read by our kernels -- is the same as over NVLink.)

Results must equal the CPU oracle exactly for integers (per-epoch
local/global/miss counts of every partition, trace) and within 1e-4 for the
loss and logits.
"""

from __future__ import annotations

import os
import pickle
import socket
import subprocess
import sys
import tempfile

import pytest

from parity_common import oracle_run, rel_err, workload

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, pickle, sys
sys.path.insert(0, {root!r})
import torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("gloo")
from paper_2508_13716_b200 import api, hostgraph as H
n, deg, P, f_dim, C, kind, cap, policy, s, epochs = {case!r}
g = H.erdos_renyi(n, deg, 0)
ps = H.build_partition_set(g, H.random_partition(n, P, 0), 1)
caps = H.uniform_capacities(ps, cap, f_dim)
cfg = H.SimConfig(epochs=epochs, policy=policy, staleness_bound=s, f_dim=f_dim, L=len(f_dim))
rep = api.train(g, ps, H.unit_profiles(P), caps, cfg, model=kind, num_classes=C,
                keep_logits="all", record_trace=True, gemm="3xtf32")
if dist.get_rank() == 0:
    with open({out!r}, "wb") as fh:
        pickle.dump(dict(counts=[(r.epoch, r.device, r.local_hits, r.global_hits, r.misses)
                                 for r in rep.records],
                         losses=rep.losses, logits=rep.logits_per_epoch,
                         trace=rep.trace_csv, planner=rep.planner), fh)
dist.barrier()
dist.destroy_process_group()
"""


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_two_ranks(case):
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "rank0.pkl")
        script = os.path.join(tmp, "worker.py")
        with open(script, "w") as fh:
            fh.write(WORKER.format(root=ROOT, case=case, out=out))
        port = _free_port()
        procs = []
        for r in range(2):
            env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK="0",
                       MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
            procs.append(subprocess.Popen([sys.executable, script], env=env,
                                          stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
        logs = []
        for p in procs:
            try:
                o, _ = p.communicate(timeout=600)
            except subprocess.TimeoutExpired:
                p.kill()
                o, _ = p.communicate()
            logs.append(o.decode(errors="replace"))
        assert all(p.returncode == 0 for p in procs), "\n----\n".join(logs)[-4000:]
        with open(out, "rb") as fh:
            return pickle.load(fh)


CASES = [
    # n, deg, P, f_dim, C, kind, capacity, policy, s, epochs
    (600, 6.0, 4, (16, 32, 32), 7, "gcn", 80, "jaca", 1, 4),
    (500, 6.0, 2, (16, 32), 5, "sage", 120, "jaca", -1, 3),
    (500, 5.0, 4, (16, 32), 6, "gcn", 60, "lru", -1, 3),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[5]}-P{c[2]}-{c[7]}-s{c[8]}")
def test_two_ranks_match_oracle(case):
    from paper_2508_13716_b200 import hostgraph as H
    n, deg, P, f_dim, C, kind, cap, policy, s, epochs = case
    got = _run_two_ranks(case)
    g, ps, og, ops = workload(n, deg, P)
    caps = H.uniform_capacities(ps, cap, f_dim)
    pr, outs, _ = oracle_run(og, ops, kind, f_dim, C, caps, policy, s, epochs)
    exp = [(p.epoch, d, *(int(x) for x in p.counts[d])) for p in pr.plans for d in range(P)]
    assert got["counts"] == exp
    assert got["trace"] == pr.trace_csv(ops.halo)
    for e, o in enumerate(outs):
        assert abs(got["losses"][e] - o.loss) <= 1e-4 * abs(o.loss), e
        assert rel_err(got["logits"][e], o.logits) <= 1e-4, e


def test_bench_two_ranks_one_gpu():
    """bench.py's N > 1 path (torchrun, barriers, max over ranks, one JSON line
    from rank 0), two ranks sharing cuda:0 over gloo."""
    import json
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--dist-backend", "gloo",
           "--no-exchange"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["partitions_per_gpu"] == 4
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


def test_bench_self_launches_gpus_n():
    """`bench.py --gpus 2` with no launcher re-runs itself under
    torch.distributed.run (2 ranks on 127.0.0.1) and reports n_gpus 2, with
    the exchange record summed / maxed over the ranks."""
    import json
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline", "--dist-backend", "gloo"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["partitions_per_gpu"] == 4
    ex = d["exchange"]
    assert ex["lookups_per_epoch"]["misses"] > 0 and ex["k3_ms_per_epoch"]["stage"] > 0
    nv = [v for k, v in ex["wire_bytes_per_epoch"].items() if k.startswith("nvlink")][0]
    assert nv > 0          # two ranks: misses and gradient rows cross devices (IPC)
