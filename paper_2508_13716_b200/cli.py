"""Command line: ``train`` (the drop-in for ``halopart simulate``),
``cache-bench`` (halopart's policy x capacity grid, plan-only on the native
planner or with real GPU epochs) and ``profile`` (K9: B200 DeviceProfile
rows for ``halopart partition``).

    python -m paper_2508_13716_b200.cli train --graph g.txt \\
        --partition-result rapa.json --devices devices.json --out run/
    python -m paper_2508_13716_b200.cli profile --out devices.json

``train`` reads the same inputs with the same option names, defaults and
precedence as ``halopart simulate`` (defaults < --config JSON < flags,
cli.py:53-115, 230-285).  It runs the epochs on the GPU(s) and emits:
- ``sim_report.json`` / ``sim_report.csv``, byte-identical to the
  reference's for the same inputs;
- ``train_report.json``: losses, measured epoch seconds, GTEPS, planner per
  epoch;
- ``trace.csv`` with ``--trace``;
- ``manifest.json``, written last, with the inputs' sha256.

Errors exit with status 2, as in cli.py:371-377.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from . import __version__
from . import artifacts as A
from . import hostgraph as HG
from .errors import DomainError, HalopartError, ParseError

_TRAIN_DEFAULTS = {
    # halopart simulate's keys (cli.py:34-74)
    "graph": None, "devices": None, "out": ".", "seed": 0, "alpha": 0.5,
    "fdim": [256, 256, 256], "compact_ids": False, "partition_result": None,
    "policy": "jaca", "epochs": 200, "staleness": -1, "prefetch_depth": 0,
    "capacity": "auto", "layers": 3, "unit_time": 1.0, "mem_cpu": 64.0,
    "mem_gpu_res": 1024.0, "mem_cpu_res": 2048.0, "topk": -1,
    # training
    "model": "gcn", "classes": 40, "gemm": "3xtf32", "trace": False, "weight_seed": 2,
}

_PROFILE_DEFAULTS = {"out": "devices.json", "n": 16384, "reps": 50, "density": 0.004,
                     "gemm": "3xtf32", "gpus": None}


def _int_list(value) -> list[int]:
    """'256,256 256' or [256, 256] -> [256, 256]."""
    items = value.replace(",", " ").split() if isinstance(value, str) else list(value)
    out = []
    for x in items:
        try:
            out.append(int(x))
        except (TypeError, ValueError):
            raise ParseError(f"not an integer list: {value!r}") from None
    return out


def _read_config(path) -> dict:
    if path is None:
        return {}
    try:
        doc = json.loads(Path(path).read_text(encoding="utf-8"))
    except json.JSONDecodeError as exc:
        raise ParseError(f"{path}: not JSON ({exc})") from None
    if not isinstance(doc, dict):
        raise ParseError(f"{path}: the config must be a JSON object")
    return doc


def _options(args, defaults: dict) -> dict:
    """Layered options, highest first: command-line flags, then the --config
    file, then the built-in defaults (halopart's precedence, cli.py:92-115).
    Keys the command does not know are an error."""
    from collections import ChainMap
    file_cfg = _read_config(getattr(args, "config", None))
    extra = sorted(file_cfg.keys() - defaults.keys())
    if extra:
        raise ParseError(f"{args.config}: unknown keys {extra}")
    flags = {k: v for k, v in vars(args).items() if k in defaults and v is not None}
    return dict(ChainMap(flags, file_cfg, defaults))


def _needed(opts: dict, *pairs) -> None:
    for key, flag in pairs:
        if opts.get(key) is None:
            raise DomainError(f"{flag} is required (flag or config file)")


def _load_profiles(devices_opt, P: int):
    """--devices, else halopart's bundled fleet (what ``halopart simulate``
    uses without --devices, cli.py:131-139) when halopart is importable.
    Without either there is no fleet to size the caches for: error."""
    if devices_opt is not None:
        path = Path(devices_opt)
        return A.load_device_profiles(path), str(devices_opt), A.sha256_file(path)
    try:
        from importlib import resources
        ref = resources.files("halopart.data").joinpath("reference_devices.json")
        blob = ref.read_bytes()
    except (ImportError, ModuleNotFoundError, FileNotFoundError):
        raise DomainError("--devices is required here: halopart (and its bundled "
                          "reference_devices.json) is not importable") from None
    import hashlib
    import io
    return (A.load_device_profiles(io.StringIO(blob.decode("utf-8"))),
            "builtin:reference_devices.json", hashlib.sha256(blob).hexdigest())


_BENCH_DEFAULTS = {**_TRAIN_DEFAULTS, "policies": "jaca,fifo,lru", "capacities": None,
                   "train": False}


def _sim_inputs(opts: dict):
    """Graph, partition result, device profiles, capacities and SimConfig
    from the resolved options (halopart simulate's inputs, cli.py:230-285)."""
    _needed(opts, ("graph", "--graph"), ("partition_result", "--partition-result"))
    opts["fdim"] = _int_list(opts["fdim"])
    graph_path = Path(opts["graph"])
    g = A.load_edge_list(graph_path, compact_ids=bool(opts["compact_ids"]))
    result_path = Path(opts["partition_result"])
    result, ps = A.import_rapa_result(result_path)
    profiles, dev_path, dev_digest = _load_profiles(opts["devices"], ps.P)
    if len(profiles) < ps.P:
        raise DomainError(f"device file has {len(profiles)} profiles, need {ps.P}")
    profiles = profiles[:ps.P]
    if max(result.sigma) >= len(profiles):
        raise DomainError("partition result names more devices than the profile list")
    fdim, L = opts["fdim"], int(opts["layers"])
    if str(opts["capacity"]) == "auto":
        caps = HG.compute_capacities(ps, int(opts["topk"]),
                                     [profiles[result.sigma[i]].mem_gb for i in range(ps.P)],
                                     float(opts["mem_gpu_res"]), float(opts["mem_cpu"]),
                                     float(opts["mem_cpu_res"]), fdim, L)
    else:
        caps = HG.uniform_capacities(ps, int(opts["capacity"]), fdim)
    cfg = HG.SimConfig(epochs=int(opts["epochs"]), alpha=float(opts["alpha"]),
                       staleness_bound=int(opts["staleness"]),
                       prefetch_depth=int(opts["prefetch_depth"]), policy=str(opts["policy"]),
                       f_dim=tuple(fdim), L=L, seed=int(opts["seed"]),
                       unit_time=float(opts["unit_time"]))
    inputs = {"graph": {"path": str(opts["graph"]), "sha256": A.sha256_file(graph_path)},
              "partition_result": {"path": str(opts["partition_result"]),
                                   "sha256": A.sha256_file(result_path)},
              "devices": {"path": dev_path, "sha256": dev_digest}}
    return g, result, ps, profiles, caps, cfg, inputs


def _manifest(command: str, opts: dict, inputs: dict) -> dict:
    return {"tool": "paper_2508_13716_b200", "tool_version": __version__, "command": command,
            "config": {k: v for k, v in opts.items() if k != "out"}, "inputs": inputs}


def cmd_train(args) -> int:
    from . import api
    opts = _options(args, _TRAIN_DEFAULTS)
    g, result, ps, profiles, caps, cfg, inputs = _sim_inputs(opts)
    rep = api.train(g, result, profiles, caps, cfg, record_trace=bool(opts["trace"]),
                    model=str(opts["model"]), num_classes=int(opts["classes"]),
                    gemm=str(opts["gemm"]), keep_logits="none", seed=int(opts["weight_seed"]))
    train_doc = {"losses": rep.losses, "epoch_seconds": rep.epoch_seconds,
                 "gteps": [rep.gteps(i) for i in range(len(rep.epoch_seconds))],
                 "planner": rep.planner, "n_edges": rep.n_edges, "n_layers": rep.n_layers,
                 "n_devices": rep.n_devices, "model": opts["model"], "gemm": opts["gemm"]}
    artifacts = {"sim_report.json": rep.to_json().encode("utf-8"),
                 "sim_report.csv": rep.to_csv().encode("utf-8"),
                 "train_report.json": A.canon_json(train_doc)}
    if rep.trace_csv is not None:
        artifacts["trace.csv"] = rep.trace_csv.encode("utf-8")
    manifest = _manifest("train", opts, inputs)
    manifest["config"]["resolved_capacities"] = {
        "c_cpu": caps.c_cpu, "c_gpu": list(caps.c_gpu), "bytes_per_entry": caps.bytes_per_entry}
    A.emit(opts["out"], artifacts, manifest)
    return 0


def cmd_cache_bench(args) -> int:
    """halopart cache-bench (cli.py:288-301): the workload under several
    policies and capacities -> compare.csv (byte-identical to the
    reference's), plan-only on the host, or real GPU epochs with --train."""
    from . import api
    opts = _options(args, _BENCH_DEFAULTS)
    _needed(opts, ("capacities", "--capacities"))
    caps_list = _int_list(opts["capacities"])
    pol = opts["policies"]
    policies = [x for x in pol.replace(",", " ").split()] if isinstance(pol, str) else list(pol)
    if not caps_list:
        raise DomainError("need at least one capacity")
    opts["policy"] = policies[0]
    g, result, ps, profiles, _, cfg, inputs = _sim_inputs(opts)
    kw = dict(train_epochs=True, model=str(opts["model"]), num_classes=int(opts["classes"]),
              gemm=str(opts["gemm"]), keep_logits="none", seed=int(opts["weight_seed"])) \
        if opts["train"] else {}
    table = api.compare_policies(g, result, profiles, cfg, policies=policies,
                                 capacities=caps_list, **kw)
    A.emit(opts["out"], {"compare.csv": table.to_csv().encode("utf-8")},
           _manifest("cache-bench", opts, inputs))
    return 0


def cmd_profile(args) -> int:
    from . import devprofile
    opts = _options(args, _PROFILE_DEFAULTS)
    gpus = None if opts["gpus"] is None else _int_list(opts["gpus"])
    rows = devprofile.measure_all(gpus, n=int(opts["n"]), reps=int(opts["reps"]),
                                  density=float(opts["density"]), gemm=str(opts["gemm"]))
    out = Path(opts["out"])
    if out.parent and not out.parent.exists():
        out.parent.mkdir(parents=True, exist_ok=True)
    out.write_bytes((json.dumps(rows, indent=1) + "\n").encode("utf-8"))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2508_13716_b200")
    sub = ap.add_subparsers(dest="command", required=True)
    t = sub.add_parser("train", help="train on B200s; drop-in for halopart simulate")
    t.add_argument("--config")
    for flag, typ in (("graph", str), ("devices", str), ("out", str), ("seed", int),
                      ("alpha", float), ("fdim", str), ("partition-result", str),
                      ("policy", str), ("epochs", int), ("staleness", int),
                      ("prefetch-depth", int), ("capacity", str), ("layers", int),
                      ("unit-time", float), ("mem-cpu", float), ("mem-gpu-res", float),
                      ("mem-cpu-res", float), ("topk", int), ("model", str), ("classes", int),
                      ("gemm", str), ("weight-seed", int)):
        t.add_argument(f"--{flag}", type=typ, default=None)
    t.add_argument("--compact-ids", action="store_true", default=None)
    t.add_argument("--trace", action="store_true", default=None)
    t.set_defaults(func=cmd_train)
    b = sub.add_parser("cache-bench", help="halopart cache-bench: policies x capacities "
                                           "(plan-only; --train runs GPU epochs)")
    b.add_argument("--config")
    for flag, typ in (("graph", str), ("devices", str), ("out", str), ("seed", int),
                      ("alpha", float), ("fdim", str), ("partition-result", str),
                      ("epochs", int), ("staleness", int), ("prefetch-depth", int),
                      ("layers", int), ("unit-time", float), ("policies", str),
                      ("capacities", str), ("model", str), ("classes", int), ("gemm", str),
                      ("weight-seed", int)):
        b.add_argument(f"--{flag}", type=typ, default=None)
    b.add_argument("--compact-ids", action="store_true", default=None)
    b.add_argument("--train", action="store_true", default=None)
    b.set_defaults(func=cmd_cache_bench)
    p = sub.add_parser("profile", help="K9: measure DeviceProfile rows of the visible B200s")
    p.add_argument("--config")
    for flag, typ in (("out", str), ("n", int), ("reps", int), ("density", float),
                      ("gemm", str), ("gpus", str)):
        p.add_argument(f"--{flag}", type=typ, default=None)
    p.set_defaults(func=cmd_profile)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (HalopartError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
