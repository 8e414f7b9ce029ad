"""K9: measure a B200's DeviceProfile row (the reference's Table 1 benchmark).

PAPER.md:35 defines the row: matrix multiplication (MM), sparse-dense matrix
multiplication (SpMM, 99.6 % sparse), host-to-device, device-to-host and
intra-device transfer of a 16384 x 16384 fp32 matrix, repeated 50 times.
devices.py:23-48 stores the per-repetition seconds plus the usable memory
in GiB.  Only ratios between devices matter to RAPA (devices.py:86-105), so
what counts is that every GPU is measured by the same code:

  mm_s    cg_gemm, 16384^3, in the GEMM mode training uses (3xTF32 default)
  spmm_s  cg_spmm of a random 0.4 %-dense 16384^2 CSR times a 16384-wide
          dense matrix (in 512-column slices: the kernel's widest row)
  h2d_s / d2h_s   pinned host <-> device copy of the 1 GiB matrix
  idt_s   device-local copy of the matrix (the paper's "Intra-Device
          Transfer"); a peer copy over NVLink is measured as
          well when a second GPU is visible and reported as ``peer_s``
          (devices.py ignores unknown keys)
  mem_gb  free HBM in GiB after the benchmark buffers are released

The output is the JSON array ``halopart``'s ``load_device_profiles``
reads (devices.py:223-236), ready for ``rapa_refine``.
"""

from __future__ import annotations

import numpy as np

from ._lib import call, ptr

GEMM_MODES = {"fp32": 0, "3xtf32": 1, "tf32": 2}


def _timed(fn, reps: int) -> float:
    import torch
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def measure(device: int = 0, n: int = 16384, reps: int = 50, density: float = 0.004,
            gemm: str = "3xtf32", seed: int = 0) -> dict:
    """One profile row for cuda:<device>; seconds are per repetition."""
    import torch
    torch.cuda.set_device(device)
    dev = torch.device("cuda", device)
    st = lambda: torch.cuda.current_stream(dev).cuda_stream  # noqa: E731
    gen = torch.Generator(device=dev).manual_seed(seed)
    A = torch.rand(n, n, device=dev, generator=gen)
    B = torch.rand(n, n, device=dev, generator=gen)
    C = torch.empty(n, n, device=dev)
    mode = GEMM_MODES[gemm]

    def mm():
        call("cg_gemm", n, n, n, ptr(A), n, ptr(B), 0, None, 0, None, 0, None, 0, None, None, 0,
             ptr(C), n, mode, None, None, st())

    mm_s = _timed(mm, reps)

    # SpMM: random CSR with `density` of the n^2 entries, unit weights
    rng = np.random.default_rng(seed)
    nnz = int(round(density * n * n))
    rows = np.sort(rng.integers(0, n, nnz))
    cols = rng.integers(0, n, nnz).astype(np.int32)
    rowptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rowptr[1:])
    t_rp = torch.from_numpy(rowptr).to(dev)
    t_col = torch.from_numpy(cols).to(dev)
    W = 512

    def spmm():
        for c0 in range(0, n, W):
            call("cg_spmm", n, min(W, n - c0), ptr(t_rp), ptr(t_col), 1 << 62, None,
                 ptr(B) + 4 * c0, n, None, None, 0, None, 0, ptr(C) + 4 * c0, n, cols.size,
                 st())

    spmm_s = _timed(spmm, reps)

    host = torch.empty(n, n, pin_memory=True)
    h2d_s = _timed(lambda: A.copy_(host, non_blocking=True), reps)
    d2h_s = _timed(lambda: host.copy_(A, non_blocking=True), reps)
    idt_s = _timed(lambda: C.copy_(A, non_blocking=True), reps)
    peer_s = None
    if torch.cuda.device_count() > 1:
        other = (device + 1) % torch.cuda.device_count()
        try:
            P_ = torch.empty(n, n, device=torch.device("cuda", other))
            peer_s = _timed(lambda: P_.copy_(A, non_blocking=True), reps)
            del P_
        except RuntimeError:
            peer_s = None
    name = torch.cuda.get_device_name(dev)
    del A, B, C, host, t_rp, t_col
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info(dev)
    row = {"id": f"{name.replace(' ', '_')}-{device}", "mm_s": mm_s, "spmm_s": spmm_s,
           "h2d_s": h2d_s, "d2h_s": d2h_s, "idt_s": idt_s, "mem_gb": free / 2 ** 30,
           "bench": {"n": n, "reps": reps, "density": density, "gemm": gemm,
                     "mm_tflops": 2 * n ** 3 / mm_s / 1e12,
                     "copy_gbs": {"h2d": 4 * n * n / h2d_s / 1e9,
                                  "d2h": 4 * n * n / d2h_s / 1e9,
                                  "idt": 2 * 4 * n * n / idt_s / 1e9}}}
    if peer_s is not None:
        row["peer_s"] = peer_s
        row["bench"]["copy_gbs"]["peer"] = 4 * n * n / peer_s / 1e9
    return row


def measure_all(devices=None, **kw) -> list[dict]:
    import torch
    devs = list(range(torch.cuda.device_count())) if devices is None else list(devices)
    return [measure(d, **kw) for d in devs]
