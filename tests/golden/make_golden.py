"""Generate golden fixtures by running the REFERENCE halopart package.

Run in the build container only (it imports halopart from /root/reference,
read-only, without installing it):

    python tests/golden/make_golden.py

Outputs (committed): tests/golden/c1.json, tests/golden/c2.json,
tests/golden/small_cases.npz, tests/golden/small_cases.json.  Nothing at test
time reads /root/reference; the tests only read these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import halopart as hp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    if isinstance(a, str):
        return hashlib.sha256(a.encode()).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def unit_profiles(P, mem=64.0):
    return [hp.DeviceProfile(id=f"u{i}", mm_s=1.0, spmm_s=1.0, h2d_s=1.0,
                             d2h_s=1.0, idt_s=1.0, mem_gb=mem) for i in range(P)]


def trace_codes(trace_csv: str) -> np.ndarray:
    code = {"hit,local": 0, "hit,global": 1, "miss,source": 2}
    rows = trace_csv.splitlines()[1:]
    return np.array([code[r.split(",", 3)[3]] for r in rows], dtype=np.int8)


def graph_digest(g):
    return {"n": int(g.n_vertices), "n_edges": int(g.n_edges),
            "out_offsets": sha(g.out_offsets.astype(np.int64)),
            "out_targets": sha(g.out_targets.astype(np.int64)),
            "in_offsets": sha(g.in_offsets.astype(np.int64)),
            "in_targets": sha(g.in_targets.astype(np.int64))}


def ps_digest(ps, table):
    ranked = []
    for h in ps.halo:
        sc = table.scores_for(h)
        ranked.append(h[np.lexsort((h, -sc))])
    return {"P": ps.P, "hops": ps.hops,
            "inner_sizes": ps.inner_sizes, "halo_sizes": ps.halo_sizes,
            "halo_sha": sha(np.concatenate(ps.halo).astype(np.int64)),
            "overlap_sha": sha(ps.overlap_count.astype(np.int64)),
            "cut_edges": [int(c) for c in ps.cut_edges],
            "all_edges": [int(c) for c in ps.all_edges],
            "union_size": int(ps.halo_union().size),
            "score_sha": sha(table.score.astype(np.float64)),
            "out_term_sha": sha(table.out_term.astype(np.float64)),
            "in_term_sha": sha(table.in_term.astype(np.float64)),
            "ranked_sha": sha(np.concatenate(ranked).astype(np.int64))}


def run_case(g, ps, caps, cfg, P):
    t0 = time.perf_counter()
    rep = hp.run(g, ps, unit_profiles(P), caps, cfg, record_trace=True)
    dt = time.perf_counter() - t0
    recs = [[r.epoch, r.device, r.fwd_bytes, r.bwd_bytes, r.local_hits,
             r.global_hits, r.misses] for r in rep.records]
    return {"caps": {"c_cpu": caps.c_cpu, "c_gpu": list(caps.c_gpu),
                     "bpe": caps.bytes_per_entry},
            "cfg": cfg.to_dict(),
            "records": recs,
            "report_json_sha": sha(rep.to_json()),
            "report_csv_sha": sha(rep.to_csv()),
            "trace_sha": sha(rep.trace_csv),
            "hit_rate_local": rep.hit_rate_local,
            "hit_rate_global": rep.hit_rate_global,
            "total_time": rep.total_time,
            "seconds": dt}, rep


def big_config(name, n, avg_deg, P, f_dim, cases):
    t0 = time.perf_counter()
    g = hp.erdos_renyi(n, avg_deg, seed=0)
    a = hp.prepartition(g, P, "random", seed=0)
    ps = hp.build_partition_set(g, a, 1)
    table = hp.influence_scores(g, ps)
    out = {"graph": graph_digest(g), "parts_sha": sha(a.parts.astype(np.int64)),
           "partitions": ps_digest(ps, table), "f_dim": list(f_dim),
           "setup_seconds": time.perf_counter() - t0, "runs": {}}
    L = len(f_dim)
    auto = hp.compute_capacities(ps, k=-1, mem_gpu=[180.0] * P,
                                 mem_gpu_res=1024.0, mem_cpu=64.0,
                                 mem_cpu_res=2048.0, f_dim=f_dim, L=L)
    out["auto_caps"] = {"c_cpu": auto.c_cpu, "c_gpu": list(auto.c_gpu)}
    for key, (policy, capspec, s, epochs) in cases.items():
        if capspec == "auto":
            caps = auto
        else:
            caps = hp.uniform_capacities(ps, int(capspec), f_dim)
        cfg = hp.SimConfig(epochs=epochs, policy=policy, staleness_bound=s,
                           f_dim=tuple(f_dim), L=L)
        res, rep = run_case(g, ps, caps, cfg, P)
        res["first_epoch_codes_sha"] = sha(trace_codes(rep.trace_csv))
        out["runs"][key] = res
        print(name, key, f"{res['seconds']:.1f}s", flush=True)
    return out


def small_cases():
    rng = np.random.default_rng(20261017)
    meta, arrays = [], {}
    idx = 0
    for trial in range(24):
        n = int(rng.integers(60, 320))
        deg = float(rng.choice([3.0, 5.0, 8.0]))
        P = int(rng.integers(2, 6))
        hops = int(rng.integers(1, 3))
        gseed = int(rng.integers(0, 1000))
        g = hp.erdos_renyi(n, deg, seed=gseed)
        a = hp.prepartition(g, P, "random", seed=gseed)
        ps = hp.build_partition_set(g, a, hops)
        table = hp.influence_scores(g, ps)
        arrays[f"g{trial}_halo"] = np.concatenate(ps.halo).astype(np.int64)
        arrays[f"g{trial}_score"] = table.score.astype(np.float64)
        arrays[f"g{trial}_overlap"] = ps.overlap_count.astype(np.int64)
        gm = {"trial": trial, "n": n, "deg": deg, "P": P, "hops": hops,
              "seed": gseed, "halo_sizes": ps.halo_sizes,
              "cut_edges": [int(c) for c in ps.cut_edges],
              "all_edges": [int(c) for c in ps.all_edges],
              "graph": graph_digest(g), "runs": []}
        hmax = max(ps.halo_sizes)
        for policy in ("jaca", "fifo", "lru"):
            for frac in (0.0, 0.2, 0.5, 1.0):
                s = int(rng.integers(-1, 3))
                c = int(round(frac * hmax))
                caps = hp.uniform_capacities(ps, c, [8, 8])
                cfg = hp.SimConfig(epochs=6, policy=policy, staleness_bound=s,
                                   f_dim=(8, 8), L=2)
                res, rep = run_case(g, ps, caps, cfg, P)
                arrays[f"r{idx}_codes"] = trace_codes(rep.trace_csv)
                res["key"] = f"r{idx}"
                res["policy"] = policy
                res["capacity"] = c
                res["staleness"] = s
                gm["runs"].append(res)
                idx += 1
        # Algorithm 1 with a top-k selection and tight budgets
        bpe = hp.feature_bytes([64, 64])
        kk = int(rng.integers(1, max(2, hmax)))
        ac = hp.compute_capacities(ps, k=kk, mem_gpu=[0.0005 * (i + 1) for i in range(P)],
                                   mem_gpu_res=0.1, mem_cpu=0.001, mem_cpu_res=0.2,
                                   f_dim=[64, 64], L=2)
        gm["algo1"] = {"k": kk, "c_cpu": ac.c_cpu, "c_gpu": list(ac.c_gpu), "bpe": bpe}
        meta.append(gm)
    return meta, arrays


def main():
    t0 = time.perf_counter()
    meta, arrays = small_cases()
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    with open(os.path.join(HERE, "small_cases.json"), "w") as fh:
        json.dump({"numpy": np.__version__, "halopart": hp.__version__,
                   "cases": meta}, fh, indent=1, sort_keys=True)
    print("small cases", f"{time.perf_counter() - t0:.1f}s", flush=True)

    c1 = big_config("c1", 10000, 20.0, 4, (128, 128), {
        "cap0": ("jaca", 0, -1, 4),
        "u3730_s1": ("jaca", 3730, 1, 4),
        "u3730_sneg": ("jaca", 3730, -1, 4),
        "u3730_s0": ("jaca", 3730, 0, 3),
        "auto": ("jaca", "auto", -1, 4),
        "fifo_u2000_s1": ("fifo", 2000, 1, 3),
        "lru_u2000_sneg": ("lru", 2000, -1, 3),
    })
    c1["numpy"] = np.__version__
    with open(os.path.join(HERE, "c1.json"), "w") as fh:
        json.dump(c1, fh, indent=1, sort_keys=True)

    n2 = 169343
    c2 = big_config("c2", n2, 1166244 / n2, 8, (128, 256, 256), {
        "auto": ("jaca", "auto", -1, 3),
        "u40000_s1": ("jaca", 40000, 1, 4),
        "cap0": ("jaca", 0, -1, 2),
    })
    c2["numpy"] = np.__version__
    with open(os.path.join(HERE, "c2.json"), "w") as fh:
        json.dump(c2, fh, indent=1, sort_keys=True)
    print("done", f"{time.perf_counter() - t0:.1f}s")


if __name__ == "__main__":
    main()
