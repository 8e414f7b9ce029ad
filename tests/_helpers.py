"""Shared test helpers (golden-file access, digests)."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a) -> str:
    if isinstance(a, str):
        return hashlib.sha256(a.encode()).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_json(name: str) -> dict:
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def load_npz(name: str):
    return np.load(os.path.join(GOLDEN, name))


def unit_profiles(P: int):
    return [dict(id=f"u{i}", mm_s=1.0, spmm_s=1.0, h2d_s=1.0, d2h_s=1.0,
                 idt_s=1.0, mem_gb=64.0) for i in range(P)]


def codes_in_lookup_order(outcomes_per_epoch, halo_sizes):
    """Flatten per-(device, position) outcome arrays into the reference's
    round-robin lookup order (simulator.py:212-225)."""
    out = []
    longest = max(halo_sizes)
    for oc in outcomes_per_epoch:
        for r in range(longest):
            for d, h in enumerate(halo_sizes):
                if r < h:
                    out.append(int(oc[d][r]))
    return np.array(out, dtype=np.int8)
