"""Artifact I/O of the train path, format-compatible with halopart.

Readers for the reference's on-disk inputs and writers for its outputs, so a
``train`` run consumes the same files as ``halopart simulate`` and emits the
same report bytes:

  load_edge_list      graph.py:150-200        "u v" lines, '#' comments
  import_rapa_result  partitioner.py:627-676  rapa.json -> (RapaResult, PartitionSet)
  load_device_profiles devices.py:223-236     JSON array of DeviceProfile objects
  manifest / emit     cli.py:146-173          sha256 manifest, written last, rollback
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import hostgraph as HG
from .errors import DomainError, ParseError


def load_edge_list(source, compact_ids: bool = False) -> HG.Graph:
    """Parse a whitespace edge list (graph.py:150-200 semantics: duplicates
    collapse, self-loops stay, non-contiguous ids need ``compact_ids``)."""
    if isinstance(source, (str, Path)):
        with open(source, "rb") as fh:
            return load_edge_list(fh, compact_ids=compact_ids)
    us, vs = [], []
    for lineno, raw in enumerate(source, start=1):
        line = (raw.decode("utf-8") if isinstance(raw, bytes) else raw).strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) != 2:
            raise ParseError(f"line {lineno}: expected 'u v', got {line!r}")
        try:
            u, v = int(parts[0]), int(parts[1])
        except ValueError:
            raise ParseError(f"line {lineno}: non-integer vertex id in {line!r}") from None
        if u < 0 or v < 0:
            raise ParseError(f"line {lineno}: vertex ids must be unsigned, got {line!r}")
        us.append(u)
        vs.append(v)
    src = np.array(us, dtype=np.int64)
    dst = np.array(vs, dtype=np.int64)
    if src.size == 0:
        return HG.graph_from_pairs(src, dst, 0)
    ids = np.unique(np.concatenate([src, dst]))
    id_map = None
    if compact_ids:
        src = np.searchsorted(ids, src)
        dst = np.searchsorted(ids, dst)
        id_map = {int(o): i for i, o in enumerate(ids)}
        n = int(ids.size)
    else:
        n = int(ids[-1] + 1)
        if ids.size != n:
            raise DomainError(f"vertex ids are non-contiguous ({ids.size} ids, max {n - 1}); "
                              "pass compact_ids=True to remap")
    g = HG.graph_from_pairs(src, dst, n)
    g.vertex_id_map = id_map
    return g


@dataclass
class RapaResult:
    """The fields of halopart's RapaResult the train path reads."""

    sigma: tuple
    partitions: HG.PartitionSet
    feasible: bool
    iterations: int
    epsilon: float
    objective_history: list
    cost: dict


def import_rapa_result(source):
    """rapa.json -> (RapaResult, PartitionSet) (partitioner.py:627-676)."""
    if isinstance(source, bytes):
        text = source.decode("utf-8")
    elif isinstance(source, Path) or (isinstance(source, str) and Path(source).exists()):
        text = Path(source).read_text(encoding="utf-8")
    elif isinstance(source, str):
        text = source
    else:
        text = source.read()
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ParseError(f"invalid JSON: {exc}") from None
    try:
        P = len(doc["partitions"])
        inner = [np.array(p["inner"], dtype=np.int64) for p in doc["partitions"]]
        halo = [np.array(p["halo"], dtype=np.int64) for p in doc["partitions"]]
        cut = [int(p["cut_edges"]) for p in doc["partitions"]]
        all_e = [int(p["all_edges"]) for p in doc["partitions"]]
        n = int(doc["n_vertices"])
        overlap = np.zeros(n, dtype=np.int64)
        for h in halo:
            overlap[h] += 1
        ps = HG.PartitionSet(n_vertices=n, P=P, inner=inner, halo=halo, hops=int(doc["hops"]),
                             overlap_count=overlap, cut_edges=cut, all_edges=all_e)
        res = RapaResult(sigma=tuple(int(s) for s in doc["sigma"]), partitions=ps,
                         feasible=bool(doc["feasible"]), iterations=int(doc["iterations"]),
                         epsilon=float(doc["epsilon"]),
                         objective_history=[float(x) for x in doc["objective_history"]],
                         cost=dict(doc["cost"]))
    except (KeyError, TypeError, ValueError) as exc:
        raise ParseError(f"malformed refinement document: {exc}") from None
    if sorted(res.sigma) != list(range(P)):
        raise DomainError("sigma is not a permutation of the device indexes")
    return res, ps


def _profile(obj, where: str) -> HG.DeviceProfile:
    if not isinstance(obj, dict):
        raise ParseError(f"{where}: expected an object")
    try:
        p = HG.DeviceProfile(id=str(obj["id"]), mm_s=float(obj["mm_s"]),
                             spmm_s=float(obj["spmm_s"]), h2d_s=float(obj["h2d_s"]),
                             d2h_s=float(obj["d2h_s"]), idt_s=float(obj["idt_s"]),
                             mem_gb=float(obj["mem_gb"]))
    except KeyError as exc:
        raise ParseError(f"{where}: missing field {exc.args[0]!r}") from None
    except (TypeError, ValueError) as exc:
        raise ParseError(f"{where}: {exc}") from None
    if p.mem_gb <= 0:
        raise DomainError(f"{p.id}: mem_gb must be positive")
    for k in ("mm_s", "spmm_s", "h2d_s", "d2h_s", "idt_s"):
        if getattr(p, k) <= 0:
            raise DomainError(f"{p.id}: {k} must be positive")
    return p


def load_device_profiles(source) -> list:
    """JSON array of DeviceProfile objects (devices.py:223-236)."""
    if isinstance(source, (str, Path)):
        with open(source, "r", encoding="utf-8") as fh:
            return load_device_profiles(fh)
    try:
        data = json.load(source)
    except json.JSONDecodeError as exc:
        raise ParseError(f"invalid JSON: {exc}") from None
    if not isinstance(data, list):
        raise ParseError("expected a top-level JSON array of profiles")
    if not data:
        raise ParseError("profile array is empty")
    return [_profile(o, f"[{i}]") for i, o in enumerate(data)]


def sha256_file(path) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


def canon_json(doc) -> bytes:
    return (json.dumps(doc, sort_keys=True, indent=2) + "\n").encode("utf-8")


def emit(out_dir, artifacts: dict, manifest: dict) -> None:
    """Write every artifact, the manifest last; remove partial output on
    failure (cli.py:146-161)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    manifest["outputs"] = sorted(artifacts) + ["manifest.json"]
    items = list(artifacts.items()) + [("manifest.json", canon_json(manifest))]
    written = []
    try:
        for name, data in items:
            target = out / name
            target.write_bytes(data)
            written.append(target)
    except BaseException:
        for p in written:
            p.unlink(missing_ok=True)
        raise
