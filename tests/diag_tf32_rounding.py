"""Diagnostic (not a test): does tcgen05 kind::tf32 truncate or round fp32
operands?  A = 1 + 2^-11 + 2^-12 (bits below the TF32 mantissa), B = 1.
Truncation gives 1.0, round-to-nearest gives 1 + 2^-10."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13716_b200._lib import call, ptr  # noqa: E402

M, N, K = 128, 16, 8
A = np.zeros((M, K), np.float32)
A[:, 0] = 1 + 2.0 ** -11 + 2.0 ** -12
A[1, 0] = -(1 + 2.0 ** -11 + 2.0 ** -12)
B = np.zeros((K, N), np.float32)
B[0, :] = 1.0
tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
out = torch.zeros(M, N, device="cuda")
call("cg_gemm", M, N, K, ptr(tA), K, ptr(tB), 0, None, 0, None, 0, None, 0, None, None, 0,
     ptr(out), N, 2, None, None, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
v, w = float(out[0, 0]), float(out[1, 0])
kind = {1.0: "truncate", 1 + 2.0 ** -10: "round-to-nearest"}.get(v, f"other {v!r}")
print(f"tf32 operand conversion: {kind} (pos {v!r}, neg {w!r})")
