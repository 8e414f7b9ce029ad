"""On-disk inputs and outputs of the ``train`` command.

The files are the ones ``halopart simulate`` reads and writes, so a run can
switch tools without converting anything.  The formats are halopart's; the
code here is this package's own (vectorised parsing, schema tables, atomic
renames):

  edge list      format of graph.py:150-200     -> load_edge_list
  rapa.json      format of partitioner.py:587-676 -> import_rapa_result
  devices.json   format of devices.py:223-236   -> load_device_profiles
  outputs        contract of cli.py:146-173     -> emit (manifest last, all-or-nothing)
"""

from __future__ import annotations

import hashlib
import json
import os
import tempfile
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import hostgraph as HG
from .errors import DomainError, ParseError

# ----------------------------------------------------------------- edge list


def _edge_tokens(blob: bytes) -> tuple[np.ndarray, list[int]]:
    """Data lines of an edge list as an (m, 2) token table plus their
    1-based line numbers; '#' lines and blank lines are skipped."""
    rows, where = [], []
    for no, line in enumerate(blob.splitlines(), 1):
        s = line.strip()
        if s and not s.startswith(b"#"):
            rows.append(s.split())
            where.append(no)
    bad = next((i for i, r in enumerate(rows) if len(r) != 2), None)
    if bad is not None:
        raise ParseError(f"line {where[bad]}: want two vertex ids, got "
                         f"{b' '.join(rows[bad]).decode(errors='replace')!r}")
    return rows, where


def _to_ids(rows, where) -> np.ndarray:
    flat = [t for r in rows for t in r]
    try:
        ids = np.array([int(t) for t in flat], dtype=np.int64)
    except ValueError:
        for i, t in enumerate(flat):
            try:
                int(t)
            except ValueError:
                raise ParseError(f"line {where[i // 2]}: {t.decode(errors='replace')!r} is "
                                 "not an integer vertex id") from None
        raise
    neg = np.flatnonzero(ids < 0)
    if neg.size:
        raise ParseError(f"line {where[int(neg[0]) // 2]}: negative vertex id {ids[neg[0]]}")
    return ids.reshape(-1, 2)


def load_edge_list(source, compact_ids: bool = False) -> HG.Graph:
    """Directed edge list -> Graph (duplicate edges collapse, self-loops
    stay).  Ids must be 0..n-1 unless ``compact_ids`` renumbers them densely
    in ascending order (the map is kept on ``Graph.vertex_id_map``)."""
    if isinstance(source, (str, os.PathLike)):
        blob = Path(source).read_bytes()
    else:
        blob = source.read()
        if isinstance(blob, str):
            blob = blob.encode("utf-8")
    rows, where = _edge_tokens(blob)
    if not rows:
        return HG.graph_from_pairs(np.zeros(0, np.int64), np.zeros(0, np.int64), 0)
    pairs = _to_ids(rows, where)
    uniq, dense = np.unique(pairs, return_inverse=True)
    if compact_ids:
        g = HG.graph_from_pairs(dense.reshape(-1, 2)[:, 0], dense.reshape(-1, 2)[:, 1],
                                int(uniq.size))
        g.vertex_id_map = dict(zip(uniq.tolist(), range(uniq.size)))
        return g
    n = int(uniq[-1]) + 1
    if uniq.size != n:
        raise DomainError(f"vertex ids leave gaps ({uniq.size} distinct, largest {n - 1}); "
                          "use compact_ids=True")
    return HG.graph_from_pairs(pairs[:, 0], pairs[:, 1], n)


# ------------------------------------------------------------------ rapa.json


@dataclass
class RapaResult:
    """The RapaResult fields the train path consumes."""

    sigma: tuple
    partitions: HG.PartitionSet
    feasible: bool
    iterations: int
    epsilon: float
    objective_history: list
    cost: dict


_PART_FIELDS = (("inner", lambda v: np.asarray(v, dtype=np.int64)),
                ("halo", lambda v: np.asarray(v, dtype=np.int64)),
                ("cut_edges", int), ("all_edges", int))
_DOC_FIELDS = (("n_vertices", int), ("hops", int), ("sigma", lambda v: tuple(map(int, v))),
               ("feasible", bool), ("iterations", int), ("epsilon", float),
               ("objective_history", lambda v: [float(x) for x in v]), ("cost", dict),
               ("partitions", list))


def _fields(obj, table, where):
    if not isinstance(obj, dict):
        raise ParseError(f"{where}: expected a JSON object")
    out = {}
    for name, conv in table:
        if name not in obj:
            raise ParseError(f"{where}: field {name!r} is missing")
        try:
            out[name] = conv(obj[name])
        except (TypeError, ValueError) as exc:
            raise ParseError(f"{where}.{name}: {exc}") from None
    return out


def import_rapa_result(source):
    """A rapa.json document (path, text, bytes or file) ->
    (RapaResult, PartitionSet)."""
    if isinstance(source, os.PathLike) or (isinstance(source, str) and os.path.exists(source)):
        text = Path(source).read_text(encoding="utf-8")
    elif isinstance(source, (bytes, bytearray)):
        text = bytes(source).decode("utf-8")
    elif isinstance(source, str):
        text = source
    else:
        text = source.read()
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ParseError(f"rapa document is not JSON: {exc}") from None
    top = _fields(doc, _DOC_FIELDS, "rapa")
    parts = [_fields(p, _PART_FIELDS, f"rapa.partitions[{i}]")
             for i, p in enumerate(top["partitions"])]
    P, n = len(parts), top["n_vertices"]
    if sorted(top["sigma"]) != list(range(P)):
        raise DomainError(f"sigma {list(top['sigma'])} is not a permutation of 0..{P - 1}")
    halo = [p["halo"] for p in parts]
    overlap = (np.bincount(np.concatenate(halo), minlength=n).astype(np.int64)
               if any(h.size for h in halo) else np.zeros(n, np.int64))
    ps = HG.PartitionSet(n_vertices=n, P=P, inner=[p["inner"] for p in parts], halo=halo,
                         hops=top["hops"], overlap_count=overlap,
                         cut_edges=[p["cut_edges"] for p in parts],
                         all_edges=[p["all_edges"] for p in parts])
    res = RapaResult(sigma=top["sigma"], partitions=ps, feasible=top["feasible"],
                     iterations=top["iterations"], epsilon=top["epsilon"],
                     objective_history=top["objective_history"], cost=top["cost"])
    return res, ps


# --------------------------------------------------------------- devices.json

_TIMES = ("mm_s", "spmm_s", "h2d_s", "d2h_s", "idt_s")


def _device(obj, i: int) -> HG.DeviceProfile:
    row = _fields(obj, [("id", str)] + [(k, float) for k in _TIMES + ("mem_gb",)],
                  f"devices[{i}]")
    nonpos = [k for k in _TIMES + ("mem_gb",) if not row[k] > 0]
    if nonpos:
        raise DomainError(f"device {row['id']}: {', '.join(nonpos)} must be > 0")
    return HG.DeviceProfile(**row)


def load_device_profiles(source) -> list:
    """A JSON array of DeviceProfile objects (path or file)."""
    if isinstance(source, (str, os.PathLike)):
        text = Path(source).read_text(encoding="utf-8")
    else:
        text = source.read()
    try:
        data = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ParseError(f"device file is not JSON: {exc}") from None
    if not isinstance(data, list) or not data:
        raise ParseError("device file must hold a non-empty JSON array")
    return [_device(o, i) for i, o in enumerate(data)]


# ------------------------------------------------------------------- outputs


def sha256_file(path) -> str:
    with open(path, "rb") as fh:
        return hashlib.file_digest(fh, "sha256").hexdigest()


def canon_json(doc) -> bytes:
    """The report serialisation halopart's CLI uses (sorted keys, indent 2,
    trailing newline)."""
    return (json.dumps(doc, sort_keys=True, indent=2) + "\n").encode("utf-8")


def emit(out_dir, artifacts: dict, manifest: dict) -> None:
    """All-or-nothing output: every file is first written to a temporary
    name in ``out_dir``, then renamed into place, the manifest last.  On any
    failure the temporaries (and any already renamed file) are removed."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    manifest["outputs"] = sorted(artifacts) + ["manifest.json"]
    order = sorted(artifacts.items()) + [("manifest.json", canon_json(manifest))]
    staged, placed = [], []
    try:
        for name, data in order:
            fd, tmp = tempfile.mkstemp(prefix=f".{name}.", dir=out)
            staged.append((tmp, out / name))
            with os.fdopen(fd, "wb") as fh:
                fh.write(data)
        for tmp, final in staged:
            os.replace(tmp, final)
            placed.append(final)
    except BaseException:
        for tmp, final in staged:
            Path(tmp).unlink(missing_ok=True)
        for final in placed:
            final.unlink(missing_ok=True)
        raise
