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
    "c1": dict(n=10000, e=200000, f_dim=(128, 128), classes=40, model="gcn", hops=1, parts=4,
               workload="C1 ER graph 10,000 v / 200,000 e, GCN 2-layer f_dim (128,128) -> 40 "
                        "classes, P=4 random partitions, JACA Algorithm-1 capacities, "
                        "staleness -1 (BASELINE.json configs[0], the CPU-runnable case)"),
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
    global N_C2, E_C2, F_DIM, CLASSES, MODEL, HOPS, WORKLOAD, CONFIG, PARTS
    c = CONFIGS[name]
    N_C2, E_C2, F_DIM, CLASSES = c["n"], c["e"], c["f_dim"], c["classes"]
    MODEL, HOPS, WORKLOAD, CONFIG = c["model"], c["hops"], c["workload"], name
    PARTS = c.get("parts", 8)


def mapped_repo_libs() -> list[str]:
    """Shared objects from this repo mapped into this process."""
    try:
        with open("/proc/self/maps") as fh:
            paths = {ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so")}
    except OSError:
        return []
    return sorted(os.path.relpath(p, ROOT) for p in paths if p.startswith(ROOT + os.sep))


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
    # aggregation widths in launch order (backward: min(F_in, F_out) wide;
    # GraphSAGE layer 0 transform-first when it narrows adds a backward one)
    fw, bw = eng.spmm_widths()
    fb, bb = eng.spmm_launch_bytes()
    tot_bytes = args.steps * (sum(fb) + sum(bb))
    tot_ms = float(fwd_ms.sum() + bwd_ms.sum())
    achieved = tot_bytes / (tot_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    bound = "hbm"
    if CONFIG == "c3":
        # C3's gathers are L2 hits (average in-degree 492: the 563 MB feature
        # matrix is re-read ~200x per epoch), so its roofline is the L2's
        bound, peak, peak_kind = "l2", l2_peak(), "measured (L2-resident copy, bench.l2_peak)"
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", "spmm_traffic.json")) as fh:
            prof = json.load(fh).get(CONFIG, {})   # per workload; {} = not captured
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
    # the input buffer's bare H2D rate (no epoch beside it), for the record
    dbuf = torch.empty_like(host_x, device="cuda")
    h2d_alone = 0.0
    for _ in range(3):   # best of 3 batches of 10 copies
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        for _ in range(10):
            dbuf.copy_(host_x, non_blocking=True)
        torch.cuda.synchronize()
        h2d_alone = max(h2d_alone, 10 * host_x.numel() * 4 / (time.perf_counter() - h0) / 1e9)
    del dbuf
    barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e2e_run(e2e_steps, 0)
    enq_s = time.perf_counter() - w0      # host time to enqueue the K steps
    torch.cuda.synchronize()
    barrier()
    w_s = time.perf_counter() - w0
    sess.finish()
    w_s = max_over_ranks(w_s, world, args.dist_backend)
    e2e = {"value": L * E * e2e_steps / w_s / 1e9, "unit": "GTEPS",
           "h2d_bytes_per_step": int(host_x.numel() * 4),
           "d2h_bytes_per_step": int(D.n_in * eng.C4 * 4 + 4) if args.e2e_logits else 4,
           "steps": e2e_steps, "ms_per_step": w_s / e2e_steps * 1e3,
           "host_enqueue_ms_per_step": enq_s / e2e_steps * 1e3,
           "input_h2d_alone_GB_s": h2d_alone,
           "pcie_bound_ms_per_step": host_x.numel() * 4 / h2d_alone / 1e6,
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
    del sess, eng
    exchange = exchange_pinned = None
    if CONFIG == "c2" and not args.no_exchange:
        exchange = exchange_record(args, g, ps, world)
        # the capacity-limited path (C5's shape of cache, at C2 size): small
        # HBM levels, a large pinned host tier, staleness 1 -> every other
        # epoch serves ~489K lookups as stale global hits from pinned memory
        pc = H.CacheCapacities(c_cpu=PINNED_CAP[1], c_gpu=tuple([PINNED_CAP[0]] * ps.P),
                               bytes_per_entry=caps.bytes_per_entry)
        exchange_pinned = exchange_record(
            args, g, ps, world, caps=pc, staleness=1,
            label=f"C2, c_gpu {PINNED_CAP[0]} per partition, c_cpu {PINNED_CAP[1]} (pinned "
                  "host tier), staleness 1, JACA")
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
            "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s",
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
                                          ["fwd"] * len(fb) + ["bwd"] * len(bb), fw + bw,
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
            "exchange": exchange,
            "exchange_pinned": exchange_pinned,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def sum_over_ranks(x, world: int, backend: str):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor(np.asarray(x, np.float64), device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(t)
    return t.cpu().numpy()


def l2_peak(nbytes: int = 24 << 20, reps: int = 50) -> float:
    """L2 bandwidth, GB/s, measured: the better of a device copy between two
    L2-resident buffers (2 x 24 MB << 126 MB; read + write bytes) and a
    read-only column reduction of a 48 MB L2-resident buffer (the SpMM's
    gathers are reads), best of 5 batches each."""
    import torch
    a = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda").uniform_()
    b = torch.empty_like(a)
    r = torch.empty(2 * nbytes // 4 // 1024, 1024, dtype=torch.float32, device="cuda").uniform_()
    o = torch.empty(1024, dtype=torch.float32, device="cuda")

    def best_ms(fn):
        for _ in range(3):
            fn()
        best = 1e9
        for _ in range(5):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(reps):
                fn()
            t1.record()
            torch.cuda.synchronize()
            best = min(best, t0.elapsed_time(t1) / reps)
        return best
    copy = 2 * nbytes / (best_ms(lambda: b.copy_(a)) / 1e3) / 1e9
    read = 2 * nbytes / (best_ms(lambda: torch.sum(r, dim=0, out=o)) / 1e3) / 1e9
    return max(copy, read)


def pcie_peaks(nbytes: int = 256 << 20):
    """Copy-engine H2D / D2H GB/s of one pinned buffer (best of 5)."""
    import torch
    h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    d = torch.empty_like(h, device="cuda")
    out = {}
    for name, (dst, src) in (("h2d", (d, h)), ("d2h", (h, d))):
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dst.copy_(src, non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        out[name] = nbytes / (best / 1e3) / 1e9
    return out


EXCHANGE_CAP, EXCHANGE_S = 40000, 1
PINNED_CAP = (20000, 150000)   # (c_gpu per partition, c_cpu)


def exchange_record(args, g, ps, world: int, epochs: int = 8, caps=None, staleness=None,
                    label=None):
    """The exchange path, timed: C2 with uniform capacity 40,000 per cache
    level and staleness 1 (the reference-golden case ``u40000_s1``), so every
    epoch has misses, stale global hits served from the pinned host tier,
    local-slab write-through and host-tier write-through.  Per epoch: device
    time, each K3 launch class's CUDA-event time, and the rows each class
    moved by tier (read from that epoch's plan tables), as wire bytes next to
    the reference's model bytes (simulator.py:232-236)."""
    import torch
    from paper_2508_13716_b200 import api, hostgraph as H
    if caps is None:
        caps = H.uniform_capacities(ps, EXCHANGE_CAP, F_DIM)
    staleness = EXCHANGE_S if staleness is None else staleness
    label = label or (f"C2, uniform capacity {EXCHANGE_CAP} per level (c_gpu, c_cpu), staleness "
                      f"{EXCHANGE_S}, JACA (reference golden u40000_s1)")
    cfg = H.SimConfig(epochs=args.warmup + epochs, policy="jaca", staleness_bound=staleness,
                      f_dim=F_DIM, L=len(F_DIM))
    sess = api.TrainSession(g, ps, H.unit_profiles(ps.P), caps, cfg, model=MODEL,
                            num_classes=CLASSES, gemm=args.gemm, keep_logits="none")
    eng = sess.engine
    eng.k3_timing(True)
    for _ in range(args.warmup):
        sess.step()
    classes = ("stage", "prefetch", "write_through", "write_back", "grad_pull", "snapshot")
    tiers = ("stage_host", "stage_peer", "stage_hbm", "write_through", "write_back",
             "grad_pull")
    width = eng.k3_widths()
    ep_s, k3_ms, rows, counts = [], [], [], []
    for _ in range(epochs):
        st = sess.step()                    # synchronous: events read per epoch
        ep_s.append(st.seconds)
        k3_ms.append([st.k3.get(c, 0.0) if st.k3 else 0.0 for c in classes])
        r = eng.k3_rows()
        rows.append([r[t] for t in tiers])
        counts.append(np.asarray(st.counts).sum(0))
    # the same epochs with every staging copy in line on the compute stream
    # (no prefetch queue): how much of the prefetched copies' time it hides
    eng.prefetch = False
    eng._graphs = None
    for _ in range(2):
        sess.step()
    nopf_s, nopf_stage = [], []
    for _ in range(epochs):
        st = sess.step()
        nopf_s.append(st.seconds)
        nopf_stage.append(st.k3.get("stage", 0.0) if st.k3 else 0.0)
    eng.prefetch = True
    # the same epochs without request coalescing: every co-resident requester
    # stages its own copy of a row (the wire rows coalescing saves)
    eng.coalesce = False
    eng.k6_static.coalesce = 0
    eng._graphs = None
    for _ in range(2):
        sess.step()
    noco_s, noco_rows = [], []
    for _ in range(epochs):
        st = sess.step()
        noco_s.append(st.seconds)
        r = eng.k3_rows()
        noco_rows.append([r[t] for t in tiers])
    eng.coalesce = True
    eng.k6_static.coalesce = 1
    # the same epochs with the host-tier write-through in line on the compute
    # stream (no side-stream queue): how much of its PCIe time the queue hides
    eng.wt_async = False
    eng._graphs = None            # re-capture without the fork / join
    for _ in range(2):
        sess.step()
    inl_s, inl_wt = [], []
    for _ in range(epochs):
        st = sess.step()
        inl_s.append(st.seconds)
        inl_wt.append(st.k3.get("write_through", 0.0) if st.k3 else 0.0)
    sess.close()
    noco = max_over_ranks(float(np.mean(noco_s)), world, args.dist_backend)
    noco_rows = sum_over_ranks(np.asarray(noco_rows, np.float64).mean(0), world,
                               args.dist_backend)
    nopf = max_over_ranks(float(np.mean(nopf_s)), world, args.dist_backend)
    nopf_stage = max_over_ranks(float(np.mean(nopf_stage)), world, args.dist_backend)
    inl = max_over_ranks(float(np.mean(inl_s)), world, args.dist_backend)
    inl_wt = max_over_ranks(float(np.mean(inl_wt)), world, args.dist_backend)
    ep = max_over_ranks(float(np.mean(ep_s)), world, args.dist_backend)
    k3 = np.asarray(k3_ms).mean(0)
    k3 = [max_over_ranks(float(x), world, args.dist_backend) for x in k3]
    rows_tot = sum_over_ranks(np.asarray(rows, np.float64).mean(0), world, args.dist_backend)
    wire = {t: float(rows_tot[i]) * width[t] * 4 for i, t in enumerate(tiers)}
    cnt = np.asarray(counts).mean(0)     # every rank plans every partition: no sum
    bpe = caps.bytes_per_entry
    pcie = pcie_peaks()
    k3d = dict(zip(classes, k3))
    hbm_peak, _ = peaks()

    def rate(nbytes, ms):
        return nbytes / (ms / 1e3) / 1e9 if ms > 0 else None
    stage_bytes = wire["stage_host"] + wire["stage_peer"] + wire["stage_hbm"]
    return {
        "workload": f"{label}; epochs {args.warmup + 1}..{args.warmup + epochs} "
                    "(K6-planned, period-2 plan)",
        "ms_per_epoch": ep * 1e3, "gteps": len(F_DIM) * g.n_edges / ep / 1e9,
        "lookups_per_epoch": {"local_hits": float(cnt[0]), "global_hits": float(cnt[1]),
                              "misses": float(cnt[2])},
        "model_bytes_per_epoch": {"fwd_cached": float(cnt[2]) * bpe,
                                  "fwd_uncached": float(sum(h.size for h in ps.halo)) * bpe,
                                  "bwd": float(sum(ps.cut_edges)) * bpe},
        "wire_bytes_per_epoch": {"pcie_read (global-tier hits, pinned host -> HBM)":
                                     wire["stage_host"],
                                 "pcie_write (global-tier write-through, HBM -> pinned host)":
                                     wire["write_through"],
                                 "nvlink (peer pulls: misses + backward gradient rows)":
                                     wire["stage_peer"] + wire["grad_pull"],
                                 "hbm (local-slab fills and write-back)":
                                     wire["stage_hbm"] + wire["write_back"]},
        "rows_per_epoch": {t: float(rows_tot[i]) for i, t in enumerate(tiers)},
        "k3_ms_per_epoch": k3d,
        "k3_share_of_epoch": sum(k3) / (ep * 1e3),
        "request_coalescing": {
            "ms_per_epoch_on": ep * 1e3, "ms_per_epoch_off": noco * 1e3,
            "rows_per_epoch_off": {t: float(noco_rows[i]) for i, t in enumerate(tiers)},
            "pcie_read_bytes_per_epoch_off": float(noco_rows[tiers.index("stage_host")])
                                             * width["stage_host"] * 4,
            "how": "same session, same epochs with every co-resident requester staging its "
                   "own copy (CG_COALESCE=0) vs one staged row per (vertex, source, device)"},
        "prefetch_queue": {
            "ms_per_epoch_prefetch": ep * 1e3, "ms_per_epoch_inline": nopf * 1e3,
            "stage_ms_inline": nopf_stage,
            "stage_ms_with_prefetch": {"inline (owner rows, layers >= 1)": k3d["stage"],
                                       "prefetch stream": k3d["prefetch"]},
            "hidden_frac": ((nopf - ep) * 1e3 / nopf_stage) if nopf_stage > 0 else None,
            "how": "same session, same K6-planned epochs: staging rows final before the epoch "
                   "(pinned-tier reads of every layer, all layer-0 rows) copied on a prefetch "
                   "stream right after the plan, the compute stream waiting per layer, vs every "
                   "staging copy in line; hidden = (inline - prefetch) / inline staging time"},
        "write_through_queue": {
            "ms_per_epoch_queued": ep * 1e3, "ms_per_epoch_inline": inl * 1e3,
            "write_through_ms_inline": inl_wt,
            "hidden_frac": ((inl - ep) * 1e3 / inl_wt) if inl_wt > 0 else None,
            "blocks": eng.WT_BLOCKS,
            "how": "same session, same K6-planned epochs: host-tier write-through on the "
                   "side-stream queue (forked per layer once its rows are final, all joined at "
                   "the end of the update; one graph per epoch; k3_ms_per_epoch.write_through "
                   "is its side-stream time) vs in line on the compute stream; hidden = "
                   "(inline - queued) / inline write-through time"},
        "k3_GB_s": {"stage (in line, prefetch off)": rate(stage_bytes, nopf_stage),
                    "write_through": rate(wire["write_through"], k3d["write_through"]),
                    "write_back": rate(wire["write_back"], k3d["write_back"]),
                    "grad_pull": rate(wire["grad_pull"], k3d["grad_pull"])},
        "peaks_GB_s": {"pcie_h2d_dma": pcie["h2d"], "pcie_d2h_dma": pcie["d2h"],
                       "hbm": hbm_peak, "nvlink_per_direction": 900.0},
        "note": "N=1: all 8 partitions share the GPU, so a miss reads the co-resident owner's "
                "row in place inside the SpMM gather (no K3 row, no wire byte) unless the "
                "vertex is locally cached (then it is written through into the slab, HBM); "
                "NVLink rows appear only at N>1",
    }


class OracleSession:
    """The CPU path of the same workload, one epoch per ``step()``: the
    planner port (pure-Python restatement of halopart's ``simulator.run``
    lookup loop, simulator.py:206-226) plus the PyTorch-CPU fp32 epoch
    (oracle/torch_port.py, all host cores) -- BASELINE.md §4's CPU baseline.
    Built from oracle-side graph objects only; nothing of the product."""

    def __init__(self, og, ops, caps, staleness: int = -1, threads: int | None = None):
        from oracle import halo_port as ohp
        from oracle import model_port as omp
        from oracle import torch_port as otp
        v, _, _, sc = ohp.influence(og, ops)
        ranked = ohp.ranked_halos(ops, v, sc)
        imp = {int(a): float(b) for a, b in zip(v, sc)}
        dims = list(F_DIM) + [CLASSES]
        self.planner = ohp.Planner("jaca", caps, ranked, ops.halo, imp)
        self.threads = threads or len(os.sched_getaffinity(0))
        self.trainer = otp.TorchTrainer(og, ops.inner, ops.halo, omp.ModelSpec(MODEL, dims),
                                        omp.features(og.n, F_DIM[0], 0),
                                        omp.labels(og.n, CLASSES, 1),
                                        params=omp.init_params(MODEL, dims, 2),
                                        threads=self.threads)
        self._live = otp.live_versions
        self.s = staleness
        self.e = 0
        self.plan_s, self.train_s = [], []

    def step(self):
        self.e += 1
        t0 = time.perf_counter()
        plan = self.planner.step(self.e, self.s)
        t1 = time.perf_counter()
        out = self.trainer.step(plan.version, self._live(self.planner.cache)
                                if self.e % 4 == 0 else None)
        t2 = time.perf_counter()
        self.plan_s.append(t1 - t0)
        self.train_s.append(t2 - t1)
        return t2 - t0, plan, out


def oracle_inputs(g=None, ps=None, caps=None, parts: int | None = None):
    """Oracle-side (graph, partitions, capacities): converted from the
    product's host objects when given, else built by the oracle itself (the
    reference arm must not map the product library)."""
    from oracle import halo_port as ohp
    parts = parts or PARTS
    if g is None:
        og = ohp.er_graph(N_C2, E_C2 / N_C2, 0)
        ops = ohp.partition_set(og, ohp.random_assignment(N_C2, parts, 0), HOPS)
        c = ohp.capacities_auto(ops, -1, [180.0] * parts, 1024.0, 64.0, 2048.0, F_DIM)
        return og, ops, (c[0], tuple(c[1]), c[2])
    og = ohp.GraphCSR(n=g.n_vertices, n_edges=g.n_edges, out_off=g.out_offsets,
                      out_tgt=g.out_targets, in_off=g.in_offsets, in_tgt=g.in_targets)
    ops = ohp.Partitions(n=g.n_vertices, P=ps.P, parts=None, inner=ps.inner, halo=ps.halo,
                         hops=HOPS, overlap=ps.overlap_count, cut=ps.cut_edges,
                         all_edges=ps.all_edges)
    return og, ops, (caps.c_cpu, tuple(caps.c_gpu), caps.bytes_per_entry)


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def time_cpu_path(sess: OracleSession, warmup: int, steps: int, budget_s: float):
    """Warm-up epochs, then timed epochs (at least one) within the budget."""
    t_start = time.perf_counter()
    for _ in range(warmup):
        sess.step()
    times = []
    while len(times) < steps:
        times.append(sess.step()[0])
        if time.perf_counter() - t_start > budget_s:
            break
    k = len(times)
    return statistics.mean(times), statistics.mean(sess.plan_s[-k:]), statistics.mean(sess.train_s[-k:]), k


def cpu_baseline(g, ps, caps, budget_s: float = 30.0):
    """The CPU path on the host cores over a bounded sample: 1 warm-up epoch
    (it holds the epoch-1 snapshot build), then epochs until the budget."""
    og, ops, ocaps = oracle_inputs(g, ps, caps)
    sess = OracleSession(og, ops, ocaps)
    per, plan_s, train_s, k = time_cpu_path(sess, 1, 3, budget_s)
    return {"value": len(F_DIM) * g.n_edges / per / 1e9, "unit": "GTEPS",
            "cores": sess.threads, "kind": "port",
            "sample": f"{k} timed epoch(s) after 1 warm-up of the same {CONFIG.upper()} workload: "
                      f"planner port (pure Python, 1 core) {plan_s:.2f} s + PyTorch-CPU fp32 "
                      f"epoch ({sess.threads} threads) {train_s:.2f} s per epoch",
            "seconds_per_epoch": per, "plan_s": plan_s, "train_s": train_s,
            "cpu": _cpu_model()}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    og, ops, caps = oracle_inputs(parts=args.parts)
    sess = OracleSession(og, ops, caps, args.staleness)
    per, plan_s, train_s, k = time_cpu_path(sess, args.warmup, args.steps, args.ref_budget)
    value = len(F_DIM) * og.n_edges / per / 1e9
    sample = (f"{k} timed epoch(s) after {args.warmup} warm-up of the {CONFIG.upper()} workload "
              f"(budget {args.ref_budget:.0f} s): planner port (pure Python, 1 core) "
              f"{plan_s:.2f} s + PyTorch-CPU fp32 epoch ({sess.threads} threads) {train_s:.2f} s")
    line = {"impl": "reference", "metric": "full-batch epoch GTEPS (L*|E|/epoch time)",
            "value": value, "unit": "GTEPS", "n_gpus": world, "steps": k,
            "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": WORKLOAD, "partitions": args.parts},
            "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": sess.threads,
                             "kind": "port", "sample": sample, "cpu": _cpu_model(),
                             "plan_s": plan_s, "train_s": train_s},
            "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "repo_libs_mapped": mapped_repo_libs()}
    print(json.dumps(line), flush=True)


def self_launch(args) -> int:
    """``--gpus N`` without a launcher: re-run this script under
    torch.distributed.run with N ranks on 127.0.0.1."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--parts", type=int, default=None)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-logits", action="store_true",
                    help="e2e: also download the logits every step")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help=argparse.SUPPRESS)
    ap.add_argument("--staleness", type=int, default=-1)
    ap.add_argument("--gemm", default="3xtf32", choices=["fp32", "3xtf32", "tf32"])
    ap.add_argument("--cpu-budget", type=float, default=30.0)
    ap.add_argument("--ref-budget", type=float, default=150.0)
    ap.add_argument("--no-exchange", action="store_true",
                    help="skip the exchange-path record (C2 only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    apply_config(args.config)
    if args.parts is None:
        args.parts = PARTS
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
