"""Microbenchmark (not a test): K3 (cg_copy_rows) row-staging bandwidth from
each tier the cache plan reads -- local HBM rows and the pinned, mapped host
tier read zero-copy over PCIe -- and the write-through into the host tier.
Prints one JSON line per case."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13716_b200._lib import call, ptr  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def main():
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream().cuda_stream
    F, n_src, n = 256, 400_000, 200_000
    rng = np.random.default_rng(0)
    src_dev = torch.randn(n_src, F, device="cuda")
    host = C.c_void_p()
    nbytes = n_src * F * 4
    call("cg_host_tier_alloc", nbytes, C.addressof(host))
    hv = np.ctypeslib.as_array((C.c_float * (n_src * F)).from_address(host.value))
    hv[:] = rng.standard_normal(n_src * F).astype(np.float32)
    dst = torch.empty(n, F, device="cuda")
    rows = torch.from_numpy(rng.integers(0, n_src, n).astype(np.int32)).cuda()
    drow = torch.arange(n, dtype=torch.int32, device="cuda")
    for name, base, sid in (("hbm -> hbm (local / co-resident rows)", ptr(src_dev), 0),
                            ("pinned host -> hbm (global tier, zero-copy PCIe)", host.value, 0)):
        tab = torch.tensor([base], dtype=torch.int64, device="cuda")
        ld = torch.tensor([F], dtype=torch.int64, device="cuda")
        sids = torch.zeros(n, dtype=torch.int32, device="cuda")
        t = timed(lambda: call("cg_copy_rows", n, F, ptr(sids), ptr(rows), ptr(drow), ptr(tab),
                               ptr(ld), ptr(dst), F, st))
        print(json.dumps({"case": name, "rows": n, "row_bytes": F * 4,
                          "seconds": t, "GB_per_s": n * F * 4 / t / 1e9}), flush=True)
    # write-through: device rows -> host tier rows
    tab = torch.tensor([ptr(src_dev)], dtype=torch.int64, device="cuda")
    ld = torch.tensor([F], dtype=torch.int64, device="cuda")
    sids = torch.zeros(n, dtype=torch.int32, device="cuda")
    hdst = torch.from_numpy(rng.permutation(n_src)[:n].astype(np.int32)).cuda()
    t = timed(lambda: call("cg_copy_rows", n, F, ptr(sids), ptr(rows), ptr(hdst), ptr(tab),
                           ptr(ld), host.value, F, st))
    print(json.dumps({"case": "hbm -> pinned host (global-tier write-through)", "rows": n,
                      "row_bytes": F * 4, "seconds": t, "GB_per_s": n * F * 4 / t / 1e9}),
          flush=True)
    call("cg_host_tier_free", host.value)


if __name__ == "__main__":
    main()
