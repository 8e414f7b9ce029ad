"""Microbenchmark (not a test): the C2 epoch's GEMM shapes through cg_gemm /
cg_wgrad in every mode, CUDA-event timed (warm L2 between reps is avoided by
the > L2 operand sizes).  Prints one line per (shape, mode)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13716_b200._lib import call, ptr  # noqa: E402

M = 169343
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
HBM = 6.65e12


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


ONLY = sys.argv[1:]  # e.g. "fwd1:1pre" "wgrad1:2" -> only these (name, mode) pairs


def want(name, tag):
    return not ONLY or f"{name}:{tag}" in ONLY


def gemm_case(name, N, K, trans_b, mask=False, row_scale=False, modes=(1, 2, 0)):
    A = torch.randn(M, K, device="cuda")
    W = torch.randn(N, K, device="cuda") if trans_b else torch.randn(K, N, device="cuda")
    Wh, Wl = torch.empty_like(W), torch.empty_like(W)
    call("cg_split_tf32", W.numel(), ptr(W), ptr(Wh), ptr(Wl), st())
    C = torch.empty(M, N, device="cuda")
    mk = torch.randn(M, N, device="cuda") if mask else None
    rs = torch.rand(M, device="cuda") if row_scale else None
    byts = 4 * (M * K + M * N + (M * N if mask else 0))
    flops = 2 * M * N * K
    for mode in modes:
        for pre in ((False, True) if mode == 1 else (False,)):
            if not want(name, f"{mode}{'pre' if pre else ''}"):
                continue
            B, lo = (Wh, Wl) if pre else (W, None)
            f = lambda: call("cg_gemm", M, N, K, ptr(A), K, ptr(B), 0, None, 0, None, trans_b,  # noqa: E731
                             None, 0, ptr(rs) if rs is not None else None,
                             ptr(mk) if mk is not None else None, N, ptr(C), N, mode,
                             ptr(lo) if lo is not None else None, None, st())
            us = timeit(f)
            print(f"{name:8s} N={N:3d} K={K:3d} tb={trans_b} mode={mode}{' pre' if pre else '    '} "
                  f"{us:8.1f} us  {byts / us / 1e6:7.0f} GB/s ({byts / us / 1e6 / (HBM / 1e9):.2f})"
                  f"  {flops * (3 if mode == 1 else 1) / us / 1e6:7.0f} GFLOP/s", flush=True)


def wgrad_case(name, K, N, modes=(1, 2, 0)):
    A = torch.randn(M, K, device="cuda")
    D = torch.randn(M, N, device="cuda")
    dW = torch.empty(K, N, device="cuda")
    ws = torch.empty(call("cg_wgrad_workspace", M, K, N), device="cuda")
    byts = 4 * (M * K + M * N)
    flops = 2 * M * N * K
    for mode in modes:
        if not want(name, str(mode)):
            continue
        f = lambda: call("cg_wgrad", M, K, N, ptr(A), K, ptr(D), N, ptr(dW), None, ptr(ws), mode, st())  # noqa: E731
        us = timeit(f)
        print(f"{name:8s} K={K:3d} N={N:3d}      mode={mode}     {us:8.1f} us  "
              f"{byts / us / 1e6:7.0f} GB/s ({byts / us / 1e6 / (HBM / 1e9):.2f})  "
              f"{flops * (3 if mode == 1 else 1) / us / 1e6:7.0f} GFLOP/s", flush=True)


if __name__ == "__main__":
    gemm_case("fwd0", 256, 128, 0, row_scale=True)
    gemm_case("fwd1", 256, 256, 0, row_scale=True)
    gemm_case("fwd2", 40, 256, 0)
    gemm_case("dgrad1", 256, 256, 1, row_scale=True)
    gemm_case("dgrad2", 256, 40, 1, mask=True)
    wgrad_case("wgrad2", 256, 40)
    wgrad_case("wgrad1", 256, 256)
    wgrad_case("wgrad0", 128, 256)
