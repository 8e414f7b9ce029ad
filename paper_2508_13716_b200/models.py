"""Model definitions on the hot path: parameter shapes and deterministic init.

GCN layer  (aggregate-first):  H' = act(A_hat H W + b),
           A_hat = D_in^-1/2 (A + I) D_out^-1/2 with GLOBAL degrees.
SAGE-mean: H' = act(H W_self + mean_{N_in} H W_neigh + b).
Weights are Glorot-uniform drawn from a 32-bit counter hash (no RNG state),
so every rank and the CPU oracle start from bit-identical fp32 parameters.
"""

from __future__ import annotations

import numpy as np

_MASK = np.uint64(0xFFFFFFFF)


def _hash(seed: int, a, b) -> np.ndarray:
    x = (np.uint64(seed) * np.uint64(0x9E3779B1)
         + np.asarray(a, np.uint64) * np.uint64(0x85EBCA77)
         + np.asarray(b, np.uint64) * np.uint64(0xC2B2AE3D)) & _MASK
    for shift, mul in ((16, 0x7FEB352D), (15, 0x846CA68B)):
        x ^= x >> np.uint64(shift)
        x = (x * np.uint64(mul)) & _MASK
    return x ^ (x >> np.uint64(16))


def _unit(seed: int, a, b) -> np.ndarray:
    """fp32 uniform in [-1, 1) -- same bits as the device hash kernel."""
    top = (_hash(seed, a, b) >> np.uint64(8)).astype(np.float32)
    return top * np.float32(1.0 / 8388608.0) - np.float32(1.0)


def glorot_uniform(fan_in: int, fan_out: int, seed: int) -> np.ndarray:
    bound = np.float32(np.sqrt(6.0 / (fan_in + fan_out)))
    rows = np.arange(fan_in, dtype=np.uint64).reshape(-1, 1)
    cols = np.arange(fan_out, dtype=np.uint64).reshape(1, -1)
    return (_unit(seed, rows, cols) * bound).astype(np.float32)


def init_params(kind: str, dims, seed: int = 2) -> list[np.ndarray]:
    """Per layer l (dims[l] -> dims[l+1]): GCN [W, b]; SAGE [W_self, W_neigh, b]."""
    out = []
    for l in range(len(dims) - 1):
        fi, fo = int(dims[l]), int(dims[l + 1])
        base = seed + 16 * l
        if kind == "gcn":
            out += [glorot_uniform(fi, fo, base), np.zeros(fo, np.float32)]
        elif kind == "sage":
            out += [glorot_uniform(fi, fo, base), glorot_uniform(fi, fo, base + 1),
                    np.zeros(fo, np.float32)]
        else:
            raise ValueError(f"unknown model {kind!r}")
    return out
