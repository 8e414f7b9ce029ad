#!/usr/bin/env python
"""Benchmark: full-batch partitioned GCN epochs through the B200 hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): ogbn-arxiv-shaped synthetic ER
graph (169,343 vertices, 1,166,244 directed edges), 3-layer GCN with layer
inputs f_dim = (128, 256, 256) and 40 classes, P = 8 partitions (random,
seed 0) spread over the N GPUs (8/N per GPU, so total work is fixed:
strong scaling), JACA two-level cache with Algorithm-1 capacities for
180 GiB HBM / 64 GiB host, staleness bound -1 (the reference default).
One step = one training epoch (plan + forward + loss + backward + K7 +
Adam).  Metric: GTEPS = L * |E| / epoch time (BASELINE.json metric), plus
epoch ms, halo bytes/epoch and the SpMM HBM roofline fraction.

Under torchrun each rank drives one GPU; every rank prints nothing but
rank 0, which prints ONE JSON line.  ``--impl reference`` times the CPU
oracle port of the same path (the reference itself is a pure-Python
simulator with no training arithmetic) on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (C2 is the default bench line; C3 / C4 are extra
# measurement runs of the larger shapes, selected with --config)
CONFIGS = {
    "c2": dict(n=169343, e=1166244, f_dim=(128, 256, 256), classes=40, model="gcn", hops=1,
               workload="C2 ogbn-arxiv-shaped ER graph 169,343 v / 1,166,244 e, GCN 3-layer "
                        "f_dim (128,256,256) -> 40 classes, P=8 random partitions, JACA "
                        "Algorithm-1 capacities (180 GiB HBM, 64 GiB host), staleness -1"),
    "c4": dict(n=2449029, e=61859140, f_dim=(100, 256, 256), classes=47, model="gcn", hops=1,
               workload="C4 ogbn-products-shaped ER graph 2,449,029 v / 61,859,140 e, GCN "
                        "3-layer f_dim (100,256,256) -> 47 classes, P=8 partitions (random; "
                        "RAPA on identical B200 profiles only permutes slots), JACA "
                        "Algorithm-1 capacities (180 GiB HBM, 64 GiB host), staleness -1"),
    "c3": dict(n=232965, e=114615892, f_dim=(604, 256), classes=41, model="sage", hops=2,
               workload="C3 Reddit-shaped ER graph 232,965 v / 114,615,892 e, GraphSAGE-mean "
                        "2-layer f_dim (602 padded to 604, 256) -> 41 classes, 2-hop halos, "
                        "P=8 random partitions, JACA Algorithm-1 capacities, staleness -1"),
}
N_C2, E_C2 = 169343, 1166244
F_DIM, CLASSES, PARTS, MODEL, HOPS = (128, 256, 256), 40, 8, "gcn", 1
WORKLOAD = CONFIGS["c2"]["workload"]
CONFIG = "c2"


def apply_config(name: str) -> None:
    global N_C2, E_C2, F_DIM, CLASSES, MODEL, HOPS, WORKLOAD, CONFIG
    c = CONFIGS[name]
    N_C2, E_C2, F_DIM, CLASSES = c["n"], c["e"], c["f_dim"], c["classes"]
    MODEL, HOPS, WORKLOAD, CONFIG = c["model"], c["hops"], c["workload"], name


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def build_workload(parts: int):
    from paper_2508_13716_b200 import hostgraph as H
    g = H.erdos_renyi(N_C2, E_C2 / N_C2, 0)
    ps = H.build_partition_set(g, H.random_partition(N_C2, parts, 0), HOPS)
    caps = H.compute_capacities(ps, -1, [180.0] * parts, 1024.0, 64.0, 2048.0, F_DIM,
                                len(F_DIM))
    return g, ps, caps


def spmm_bytes(nnz: int, rows: int, F: int, n_halo: int) -> int:
    """Algorithmic bytes of one cg_spmm launch."""
    return nnz * (4 + 4 * F) + rows * (8 + 4 + 4 * F) + 8 + n_halo * 4


def max_over_ranks(x: float, world: int, backend: str) -> float:
    """The slowest rank's time (every multi-GPU number is max over ranks)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], device="cuda" if backend == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2508_13716_b200 import _lib, api, hostgraph as H

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one process per GPU; --dist-backend gloo exists to exercise the N > 1
    # path with several ranks sharing one GPU (NCCL refuses that)
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    t_setup = time.perf_counter()
    g, ps, caps = build_workload(args.parts)
    cfg = H.SimConfig(epochs=args.warmup + args.steps, policy="jaca",
                      staleness_bound=args.staleness, f_dim=F_DIM, L=len(F_DIM))
    # the public drop-in, stepwise: same setup as api.train()
    sess = api.TrainSession(g, ps, H.unit_profiles(args.parts), caps, cfg, model=MODEL,
                            num_classes=CLASSES, gemm=args.gemm, keep_logits="none")
    eng = sess.engine
    t_setup = time.perf_counter() - t_setup
    D = eng.D
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (includes the host-planned transient epoch and the warm fill)
    for _ in range(args.warmup):
        sess.step(sync=False)
    sess.finish()
    # ---- device-timed region: K epochs, inputs resident in HBM
    barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launches["total"]
    stats = []
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            stats.append(sess.step(sync=False))
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = _lib.launches["total"] - launches0
    sess.finish()   # completes (in place) the EpochStats of the timed epochs
    dev_ms = t0.elapsed_time(t1)
    dev_ms = max_over_ranks(dev_ms, world, args.dist_backend)
    ms_per_step = dev_ms / args.steps
    L, E = len(F_DIM), g.n_edges
    gteps = L * E * args.steps / (dev_ms / 1e3) / 1e9

    # ---- SpMM roofline (all fwd+bwd aggregation launches of the timed epochs)
    fwd_ms = np.array([s.spmm_fwd_ms for s in stats])  # (K, L)
    bwd_ms = np.array([s.spmm_bwd_ms for s in stats])  # (K, L-1)
    fb = [spmm_bytes(D.nnz_fwd, D.n_in, F, D.n_halo) for F in F_DIM]
    widths = list(F_DIM) + [eng.C4]   # backward aggregates min(F_in, F_out) wide
    bb = [spmm_bytes(D.nnz_bwd, D.n_in, min(widths[l], widths[l + 1]), 0)
          for l in range(len(F_DIM) - 1, 0, -1)]
    tot_bytes = args.steps * (sum(fb) + sum(bb))
    tot_ms = float(fwd_ms.sum() + bwd_ms.sum())
    achieved = tot_bytes / (tot_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", "spmm_traffic.json")) as fh:
            prof = json.load(fh)
        if prof.get("config", "c2") != CONFIG:
            prof = {}   # the committed ncu capture is of another workload
    except Exception:  # noqa: BLE001
        pass

    # ---- halo bytes per epoch (reference model bytes; cached vs uncached)
    bpe = caps.bytes_per_entry
    counts = stats[-1].counts
    fwd_model = int(counts[:, 2].sum()) * bpe
    fwd_uncached = int(sum(h.size for h in ps.halo)) * bpe
    bwd_model = int(sum(ps.cut_edges)) * bpe

    # ---- end-to-end through the public session API: every step uploads its
    # input rows from pinned host memory (H2D) and downloads its result, the
    # loss (D2H) -- what train() hands back per epoch.  Uploads run one step
    # ahead on a copy stream; the clock is the host wall clock around the whole
    # run including the final synchronisation.  (--e2e-logits also downloads
    # the 27 MB of logits every step.)
    from paper_2508_13716_b200.models import _unit  # deterministic host features
    rows = D.verts.astype(np.uint64)[:, None]
    host_x = torch.from_numpy(_unit(0, rows, np.arange(F_DIM[0], dtype=np.uint64)[None, :])).pin_memory()
    e2e_steps = args.steps
    host_logits = ([torch.empty(D.n_in, eng.C4).pin_memory() for _ in range(2)]
                   if args.e2e_logits else None)
    host_loss = torch.empty(e2e_steps + 2).pin_memory()

    def e2e_run(n, loss_off):
        sess.prefetch_features(host_x)
        for i in range(n):
            s = sess.step(sync=False)
            if i + 1 < n:
                sess.prefetch_features(host_x)      # next step's inputs, behind this epoch
            if args.e2e_logits:
                sess.fetch_logits(host_logits[i & 1])
            sess.fetch_loss(s, host_loss[loss_off + i:loss_off + i + 1])

    e2e_run(2, e2e_steps)        # warm-up: copy streams, staging buffer, pinned paths
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e2e_run(e2e_steps, 0)
    torch.cuda.synchronize()
    barrier()
    w_s = time.perf_counter() - w0
    sess.finish()
    w_s = max_over_ranks(w_s, world, args.dist_backend)
    e2e = {"value": L * E * e2e_steps / w_s / 1e9, "unit": "GTEPS",
           "h2d_bytes_per_step": int(host_x.numel() * 4),
           "d2h_bytes_per_step": int(D.n_in * eng.C4 * 4 + 4) if args.e2e_logits else 4,
           "steps": e2e_steps, "ms_per_step": w_s / e2e_steps * 1e3,
           "how": "api.TrainSession, 2 untimed warm-up steps, then per step: pinned-host input "
                  "rows H2D (prefetched one step ahead on a copy stream; GCN: row scaling), "
                  "epoch, loss D2H" + (" + logits D2H (overlapping the backward)"
                                       if args.e2e_logits else "") +
                  "; host wall clock incl. final sync"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if CONFIG == "c2":
            cpu = cpu_baseline(g, ps, caps, budget_s=args.cpu_budget)
        else:
            cpu = {"value": None, "unit": "GTEPS", "cores": len(os.sched_getaffinity(0)),
                   "kind": "port", "sample": "not run: one oracle-port epoch of this shape "
                   "exceeds the bench's few-minute budget (see the C2 line)"}
    sess.close()
    if rank == 0:
        line = {
            "metric": "full-batch epoch GTEPS (L*|E|/epoch time)",
            "value": gteps, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded ER graph, hash-generated features/labels, hash Glorot "
                    "weights)",
            "config": {"workload": WORKLOAD, "partitions": args.parts,
                       "partitions_per_gpu": args.parts // world, "gemm": args.gemm,
                       "staleness_bound": args.staleness,
                       "l2": "inputs larger than L2 (X_ext %.2f GB per GPU > 126 MB)"
                             % (D.n_rows * sum(F_DIM) * 4 / 1e9),
                       "planner": sorted(set(s.planner for s in stats)),
                       "setup_s": round(t_setup, 2)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "traffic": prof.get("dram_bytes_per_epoch"),
                         "traffic_basis": "per epoch (sum over the k_spmm launches of one "
                                          "epoch, ncu --set full; profiles/spmm_traffic.json), "
                                          "same basis as bytes_per_epoch",
                         "kernel": "K1/K2 fused cache-lookup + gather SpMM (k_spmm_cpa "
                                   "cp.async ring for the sparse 128/256-wide launches, "
                                   "k_spmm for the 40-wide one), all fwd+bwd launches of "
                                   "the timed epochs; per-launch CUDA-event times from the "
                                   "epoch graph's event nodes (last timed epoch)",
                         "bytes_per_epoch": sum(fb) + sum(bb),
                         "spmm_ms_per_epoch": tot_ms / args.steps,
                         "launches": [{"pass": ps_, "F": int(w), "bytes": int(b_),
                                       "ms": round(float(m), 4),
                                       "GB_s": round(b_ / (float(m) / 1e3) / 1e9, 1)}
                                      for ps_, w, b_, m in zip(
                                          ["fwd"] * len(fb) + ["bwd"] * len(bb),
                                          list(F_DIM) + [min(widths[l], widths[l + 1])
                                                         for l in range(len(F_DIM) - 1, 0, -1)],
                                          fb + bb,
                                          list(fwd_ms.mean(0)) + list(bwd_ms.mean(0)))]},
            "halo_bytes_per_epoch": {"model_fwd_cached": fwd_model,
                                     "model_fwd_uncached": fwd_uncached,
                                     "model_bwd": bwd_model},
            "loss_last": stats[-1].loss,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


class OracleSession:
    """The CPU oracle port of the same workload, stepped one epoch at a time
    (plan: pure-Python CacheSystem restatement; model: float64 numpy/scipy)."""

    def __init__(self, g, ps, caps, staleness: int = -1):
        from oracle import halo_port as ohp
        from oracle import model_port as omp
        og = ohp.GraphCSR(n=g.n_vertices, n_edges=g.n_edges, out_off=g.out_offsets,
                          out_tgt=g.out_targets, in_off=g.in_offsets, in_tgt=g.in_targets)
        opart = ohp.Partitions(n=g.n_vertices, P=ps.P, parts=None, inner=ps.inner,
                               halo=ps.halo, hops=1, overlap=ps.overlap_count,
                               cut=ps.cut_edges, all_edges=ps.all_edges)
        v, _, _, sc = ohp.influence(og, opart)
        ranked = ohp.ranked_halos(opart, v, sc)
        imp = {int(a): float(b) for a, b in zip(v, sc)}
        dims = list(F_DIM) + [CLASSES]
        self.planner = ohp.Planner("jaca", (caps.c_cpu, tuple(caps.c_gpu),
                                            caps.bytes_per_entry), ranked, ps.halo, imp)
        self.trainer = omp.Trainer(og, ps.inner, ps.halo, omp.ModelSpec(MODEL, dims),
                                   omp.features(g.n_vertices, F_DIM[0], 0),
                                   omp.labels(g.n_vertices, CLASSES, 1),
                                   params=omp.init_params(MODEL, dims, 2))
        self.s = staleness
        self.e = 0
        self.n_edges = g.n_edges

    def step(self) -> float:
        t0 = time.perf_counter()
        self.e += 1
        plan = self.planner.step(self.e, self.s)
        self.trainer.step(plan.version)
        return time.perf_counter() - t0


def cpu_baseline(g, ps, caps, budget_s: float = 20.0):
    """Oracle port timed on the host cores over a bounded sample (>= 2 epochs)."""
    sess = OracleSession(g, ps, caps)
    times = []
    t_all = time.perf_counter()
    while len(times) < 2 or (time.perf_counter() - t_all < budget_s and len(times) < 4):
        times.append(sess.step())
    per_epoch = statistics.mean(times[1:])   # epoch 1 includes the warm fill
    return {"value": len(F_DIM) * g.n_edges / per_epoch / 1e9, "unit": "GTEPS",
            "cores": len(os.sched_getaffinity(0)), "kind": "port",
            "sample": f"{len(times)} epochs of the same C2 workload through the oracle port "
                      f"(pure-Python cache plan + float64 numpy/scipy model), first epoch "
                      f"excluded; mean {per_epoch:.2f} s/epoch",
            "seconds_per_epoch": per_epoch}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    g, ps, caps = build_workload(args.parts)
    sess = OracleSession(g, ps, caps, args.staleness)
    t_start = time.perf_counter()
    times = []
    for i in range(args.warmup + args.steps):
        times.append(sess.step())
        # bound the whole run to a few minutes: keep >= 1 timed epoch
        if time.perf_counter() - t_start > args.ref_budget and len(times) > min(args.warmup, 1):
            break
    timed = times[min(args.warmup, len(times) - 1):]
    per_epoch = statistics.mean(timed)
    value = len(F_DIM) * g.n_edges / per_epoch / 1e9
    sample = (f"{len(timed)} timed epoch(s) after {len(times) - len(timed)} warm-up of the C2 "
              f"workload through the oracle port (pure-Python cache plan + float64 "
              f"numpy/scipy model); budget {args.ref_budget:.0f} s")
    line = {"impl": "reference", "metric": "full-batch epoch GTEPS (L*|E|/epoch time)",
            "value": value, "unit": "GTEPS", "n_gpus": world, "steps": len(timed),
            "warmup": len(times) - len(timed), "ms_per_step": per_epoch * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "partitions": args.parts},
            "cpu_baseline": {"value": value, "unit": "GTEPS",
                             "cores": len(os.sched_getaffinity(0)), "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--parts", type=int, default=PARTS)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-logits", action="store_true",
                    help="e2e: also download the logits every step")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help=argparse.SUPPRESS)
    ap.add_argument("--staleness", type=int, default=-1)
    ap.add_argument("--gemm", default="3xtf32", choices=["fp32", "3xtf32", "tf32"])
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=150.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    apply_config(args.config)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
