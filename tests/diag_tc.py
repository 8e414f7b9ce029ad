"""Diagnostic (not a test): tcgen05 GEMM error patterns per layout/mode."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13716_b200._lib import call, ptr

def run(M, N, K, tb, mode, seed=0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    ref = A.astype(np.float64) @ (B.T if tb else B)
    out = torch.full((M, N), float("nan"), device="cuda")
    tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    call("cg_gemm", M, N, K, ptr(tA), K, ptr(tB), 0, None, 0, None, tb, None, 0, None, None, 0, ptr(out), N, mode, None, None,
         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    err = np.abs(got - ref) / np.abs(ref).max()
    bad = err > 1e-3
    msg = f"M{M} N{N} K{K} tb{tb} mode{mode}: maxerr {err.max():.3e} nan {np.isnan(got).mean():.3f} zero {(got==0).mean():.3f} badfrac {bad.mean():.3f}"
    if bad.any():
        r, c = np.nonzero(bad)
        msg += f" badrows[{r.min()}..{r.max()}] badcols[{c.min()}..{c.max()}] uniqcols {np.unique(c)[:12]}"
        # does got match ref with K truncated to the first 8/16/32?
        for kk in (8, 16, 32):
            if kk < K:
                part = A[:, :kk].astype(np.float64) @ ((B.T if tb else B)[:kk])
                e2 = np.abs(got - part).max() / np.abs(part).max()
                msg += f" vsK{kk} {e2:.2e}"
    print(msg, flush=True)
    return got, ref

def run_wgrad(M, K, N, mode):
    rng = np.random.default_rng(1)
    A = rng.standard_normal((M, K)).astype(np.float32)
    D = rng.standard_normal((M, N)).astype(np.float32)
    ws = torch.zeros(call("cg_wgrad_workspace", M, K, N), device="cuda")
    dW = torch.zeros(K, N, device="cuda")
    tA, tD = torch.from_numpy(A).cuda(), torch.from_numpy(D).cuda()
    call("cg_wgrad", M, K, N, ptr(tA), K, ptr(tD), N, ptr(dW), None, ptr(ws), mode, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = A.T.astype(np.float64) @ D
    got = dW.cpu().numpy()
    print(f"wgrad M{M} K{K} N{N} mode{mode}: maxerr {np.abs(got-ref).max()/np.abs(ref).max():.3e} zero {(got==0).mean():.3f} nan {np.isnan(got).mean():.3f}", flush=True)

for dbg in ("0", "1"):
    os.environ["CG_TC_DBG"] = dbg
    print("=== CG_TC_DBG", dbg)
    for mode in (2, 1):
        run(256, 128, 32, 1, mode)
        run(256, 128, 64, 1, mode)
        run(256, 128, 256, 1, mode)
        run(256, 256, 256, 1, mode)
        run(256, 128, 32, 0, mode)
        run(256, 32, 32, 0, mode)
        run(256, 128, 256, 0, mode)
        run_wgrad(64, 128, 128, mode)
        run_wgrad(4096, 128, 128, mode)
