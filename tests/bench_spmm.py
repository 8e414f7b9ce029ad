"""Microbenchmark (not a test): cg_spmm on a C4-shaped random CSR (products
scale: 2.45M destination rows, ~26 in-edges per row, sources over inner +
snapshot rows = 2 x n), CUDA-event timed, algorithmic GB/s per DESIGN.md §5.
Kernel choices come from the CG_SPMM_* environment knobs, so one call per
setting sweeps them:  python tests/bench_spmm.py [n_rows] [deg] [F ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13716_b200._lib import call, ptr  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2449029
    deg = float(sys.argv[2]) if len(sys.argv) > 2 else 26.25
    widths = [int(x) for x in sys.argv[3:]] or [48, 100, 256]
    n_src = 2 * n
    rng = np.random.default_rng(0)
    cnt = rng.poisson(deg, n).astype(np.int64)
    rowptr = np.concatenate(([0], np.cumsum(cnt)))
    nnz = int(rowptr[-1])
    col = rng.integers(0, n_src, nnz, dtype=np.int64).astype(np.int32)
    # ascending source order within a row, as the layout stores it
    order = np.lexsort((col, np.repeat(np.arange(n), cnt)))
    col = col[order]
    d_rp = torch.from_numpy(rowptr).cuda()
    d_col = torch.from_numpy(col).cuda()
    scale = torch.rand(n, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for F in widths:
        X = torch.rand(n_src, F, device="cuda")
        out = torch.empty(n, F, device="cuda")

        def run():
            call("cg_spmm", n, F, ptr(d_rp), ptr(d_col), 1 << 62, None, ptr(X), F, ptr(scale),
                 None, 0, None, 0, ptr(out), F, nnz, st)
        for _ in range(2):
            run()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        a.record()
        for _ in range(reps):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        byts = nnz * (4 + 4 * F) + n * (8 + 4 + 4 * F)
        knobs = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("CG_SPMM"))
        print(f"F={F:4d} nnz={nnz} {ms:8.3f} ms {byts / ms / 1e6:8.0f} GB/s  {knobs}", flush=True)
        del X, out


if __name__ == "__main__":
    main()
