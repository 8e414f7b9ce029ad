"""Kernel-level GPU tests through the C ABI (each kernel vs a CPU reference)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(a, dtype=None):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).cuda()


def _st():
    import torch
    return torch.cuda.current_stream().cuda_stream


def _check_tf32_split(x, hi, lo):
    x, hi, lo = (np.asarray(a, np.float32) for a in (x, hi, lo))
    assert not (hi.view(np.uint32) & 0x1FFF).any()
    assert not (lo.view(np.uint32) & 0x1FFF).any()
    resid = np.abs(x.astype(np.float64) - hi.astype(np.float64) - lo.astype(np.float64))
    assert (resid <= 2.0 ** -23 * np.abs(x.astype(np.float64)) + 1e-45).all()


def _sync():
    import torch
    torch.cuda.synchronize()


@pytest.mark.parametrize("F", [4, 32, 64, 100, 128, 132, 256, 384, 500, 604])
def test_spmm_with_halo_indirection(F):
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    rng = np.random.default_rng(F)
    n_rows, n_direct, n_halo, n_extra = 300, 300, 200, 150
    X = rng.standard_normal((n_direct + n_halo + n_extra, F)).astype(np.float32)
    deg = rng.integers(0, 40, n_rows)
    rowptr = np.concatenate(([0], np.cumsum(deg))).astype(np.int64)
    col = rng.integers(0, n_direct + n_halo, rowptr[-1]).astype(np.int32)
    halo_row = rng.integers(0, X.shape[0], n_halo).astype(np.int32)
    scale = rng.random(n_rows).astype(np.float32)
    add = rng.standard_normal((n_rows, F)).astype(np.float32)
    mask = rng.standard_normal((n_rows, F)).astype(np.float32)
    mapped = np.where(col < n_direct, col, halo_row[np.maximum(col - n_direct, 0)])
    ref = np.zeros((n_rows, F), np.float64)
    for r in range(n_rows):
        ref[r] = X[mapped[rowptr[r]:rowptr[r + 1]]].astype(np.float64).sum(0)
    ref = ref * scale[:, None] + add
    ref = np.where(mask > 0, ref, 0.0)
    tX, tr, tc, th = _t(X), _t(rowptr), _t(col), _t(halo_row)
    ts, ta, tm = _t(scale), _t(add), _t(mask)
    outs = []
    # nnz = -1: the register-pipelined kernel; the true nnz (avg 20 edges/row)
    # selects the cp.async ring kernel for 128 < F <= 640.  Both in CSR order.
    for nnz in (-1, int(rowptr[-1])):
        out = torch.zeros(n_rows, F, device="cuda")
        call("cg_spmm", n_rows, F, ptr(tr), ptr(tc), n_direct, ptr(th), ptr(tX), F, ptr(ts),
             ptr(ta), F, ptr(tm), F, ptr(out), F, nnz, _st())
        _sync()
        np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-5, atol=1e-4)
        outs.append(out)
    assert torch.equal(outs[0], outs[1])


def test_copy_rows_table():
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    rng = np.random.default_rng(1)
    F = 36
    srcs = [_t(rng.standard_normal((50, F + 4 * i)).astype(np.float32)) for i in range(3)]
    tab = _t(np.array([s.data_ptr() for s in srcs], np.uint64).view(np.int64))
    ld = _t(np.array([F + 4 * i for i in range(3)], np.int64))
    n = 40
    sid = rng.integers(-1, 3, n).astype(np.int32)
    srow = rng.integers(0, 50, n).astype(np.int32)
    drow = rng.permutation(60)[:n].astype(np.int32)
    drow[::7] = -1
    dst = torch.zeros(60, F, device="cuda")
    keep = [_t(sid), _t(srow), _t(drow)]  # hold the buffers across the async launch
    call("cg_copy_rows", n, F, ptr(keep[0]), ptr(keep[1]), ptr(keep[2]), ptr(tab), ptr(ld),
         ptr(dst), F, _st())
    _sync()
    exp = np.zeros((60, F), np.float32)
    for i in range(n):
        if sid[i] >= 0 and drow[i] >= 0:
            exp[drow[i]] = srcs[sid[i]].cpu().numpy()[srow[i], :F]
    assert np.array_equal(dst.cpu().numpy(), exp)


@pytest.mark.parametrize("shape", [(1000, 40, 256, 0), (777, 256, 128, 0), (513, 64, 36, 1),
                                   (2048, 256, 256, 1)])
def test_gemm_epilogue(shape):
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    M, N, K, tb = shape
    rng = np.random.default_rng(M)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    A2 = rng.standard_normal((M, K)).astype(np.float32)
    B2 = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    rs = rng.random(M).astype(np.float32)
    Bm = B.T if tb else B
    B2m = B2.T if tb else B2
    ref = (A.astype(np.float64) @ Bm + A2.astype(np.float64) @ B2m + bias)
    ref = np.maximum(ref, 0) * rs[:, None]
    out = torch.zeros(M, N, device="cuda")
    k = [_t(A), _t(B), _t(A2), _t(B2), _t(bias), _t(rs)]
    call("cg_gemm", M, N, K, ptr(k[0]), K, ptr(k[1]), K, ptr(k[2]), K, ptr(k[3]), tb,
         ptr(k[4]), 1, ptr(k[5]), None, 0, ptr(out), N, 0, None, None, _st())
    _sync()
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-4, atol=1e-3)


def test_wgrad_colsum_deterministic():
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    rng = np.random.default_rng(3)
    M, K, N = 10000, 128, 40
    A = rng.standard_normal((M, K)).astype(np.float32)
    D = rng.standard_normal((M, N)).astype(np.float32)
    ws = torch.zeros(call("cg_wgrad_workspace", M, K, N), device="cuda")
    dW = torch.zeros(K, N, device="cuda")
    db = torch.zeros(N, device="cuda")
    tA, tD = _t(A), _t(D)
    call("cg_wgrad", M, K, N, ptr(tA), K, ptr(tD), N, ptr(dW), None, ptr(ws), 0, _st())
    call("cg_colsum", M, N, ptr(tD), N, ptr(db), ptr(ws), _st())
    _sync()
    np.testing.assert_allclose(dW.cpu().numpy(), A.T.astype(np.float64) @ D, rtol=1e-4, atol=1e-3)
    np.testing.assert_allclose(db.cpu().numpy(), D.sum(0, dtype=np.float64), rtol=1e-4, atol=1e-3)
    first = dW.clone()
    call("cg_wgrad", M, K, N, ptr(tA), K, ptr(tD), N, ptr(dW), None, ptr(ws), 0, _st())
    _sync()
    assert torch.equal(first, dW)


@pytest.mark.parametrize("Cc,ld", [(47, 47), (40, 40), (47, 48), (7, 8), (64, 64), (100, 100)])
def test_softmax_ce_and_adam(Cc, ld):
    """Both CE paths (warp per row; 4 lanes per row for C <= 64 with 16-B rows)."""
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    rng = np.random.default_rng(4)
    n = 3001
    z = rng.standard_normal((n, Cc)).astype(np.float32) * 3
    y = rng.integers(0, Cc, n).astype(np.int32)
    zp = np.zeros((n, ld), np.float32)
    zp[:, :Cc] = z
    g = torch.zeros(n, ld, device="cuda")
    loss = torch.zeros(1, device="cuda")
    ws = torch.zeros(n, device="cuda")
    tz, ty = _t(zp), _t(y)
    g2 = torch.full((n, ld), 7.0, device="cuda")   # fused row-scaled copy
    sc = _t(rng.random(n).astype(np.float32))
    call("cg_softmax_ce", n, Cc, ptr(tz), ld, ptr(ty), 1.0 / n, ptr(g), ld, ptr(loss),
         ptr(ws), ptr(g2), ld, ptr(sc), _st())
    _sync()
    # exactly grad * scale (one rounding), as the separate cg_scale_rows_to gives
    assert torch.equal(g2[:, :Cc], g[:, :Cc] * sc[:, None])
    g = g[:, :Cc]
    zz = z.astype(np.float64)
    m = zz.max(1, keepdims=True)
    lse = np.log(np.exp(zz - m).sum(1)) + m[:, 0]
    p = np.exp(zz - lse[:, None])
    ref_loss = float((lse - zz[np.arange(n), y]).sum())
    p[np.arange(n), y] -= 1
    assert abs(loss.item() - ref_loss) <= 1e-5 * abs(ref_loss)
    np.testing.assert_allclose(g.cpu().numpy(), p / n, rtol=1e-4, atol=1e-8)
    # Adam, 3 steps vs float64
    prm = rng.standard_normal(1000).astype(np.float32)
    tp, tm_, tv = _t(prm), torch.zeros(1000, device="cuda"), torch.zeros(1000, device="cuda")
    P64, M64, V64 = prm.astype(np.float64), np.zeros(1000), np.zeros(1000)
    for t in range(1, 4):
        grad = rng.standard_normal(1000).astype(np.float32)
        tg = _t(grad)
        hi, lo = torch.empty(1000, device="cuda"), torch.empty(1000, device="cuda")
        corr = None
        if t == 2:   # the graph-replay form: step scalars read from device memory
            ep, corr = torch.zeros(1, dtype=torch.int32, device="cuda"), torch.zeros(2, device="cuda")
            call("cg_set_epoch", ptr(ep), 7, ptr(corr), 0.9, 0.999, t, _st())
            _sync()
            assert int(ep.item()) == 7
            # as cg_adam: 1 - beta^t in double from the float betas, rounded to float
            b1, b2 = float(np.float32(0.9)), float(np.float32(0.999))
            assert corr.cpu().numpy().tolist() == [float(np.float32(1 - b1 ** 2)),
                                                    float(np.float32(1 - b2 ** 2))]
        call("cg_adam", 1000, ptr(tp), ptr(tg), ptr(tm_), ptr(tv), 0.01, 0.9, 0.999, 1e-8,
             99 if corr is not None else t, ptr(hi), ptr(lo),
             None if corr is None else ptr(corr), _st())
        _sync()
        # the emitted split: hi, lo are TF32 values, |param - hi - lo| <= 2^-23 |param|
        _check_tf32_split(tp.cpu().numpy(), hi.cpu().numpy(), lo.cpu().numpy())
        _sync()
        M64 = 0.9 * M64 + 0.1 * grad
        V64 = 0.999 * V64 + 0.001 * grad.astype(np.float64) ** 2
        P64 -= 0.01 * (M64 / (1 - 0.9 ** t)) / (np.sqrt(V64 / (1 - 0.999 ** t)) + 1e-8)
    _sync()
    np.testing.assert_allclose(tp.cpu().numpy(), P64, rtol=1e-5, atol=1e-6)


def test_hash_inputs_bit_exact_vs_oracle():
    import torch
    from oracle import model_port as omp
    from paper_2508_13716_b200._lib import call, ptr
    n, F, Cc = 5000, 100, 47
    v = _t(np.arange(n, dtype=np.int32))
    X = torch.zeros(n, F, device="cuda")
    y = torch.zeros(n, dtype=torch.int32, device="cuda")
    call("cg_hash_features", ptr(X), F, ptr(v), n, F, 0, None, _st())
    call("cg_hash_labels", ptr(y), ptr(v), n, Cc, 1, _st())
    _sync()
    assert np.array_equal(X.cpu().numpy(), omp.features(n, F, 0))
    assert np.array_equal(y.cpu().numpy(), omp.labels(n, Cc, 1))


TC_SHAPES = [  # M, N, K1, K2, trans_b
    (1000, 40, 256, 0, 0), (777, 256, 128, 0, 0), (513, 64, 36, 0, 1), (2048, 256, 256, 0, 1),
    (300, 128, 64, 64, 0), (4099, 48, 40, 0, 1), (128, 16, 32, 0, 0), (1536, 256, 256, 256, 0)]


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("shape", TC_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_gemm_tcgen05(shape, mode):
    """tcgen05 kind::tf32 GEMM: 3xTF32 (mode 1) ~fp32, 1xTF32 (mode 2) ~1e-3."""
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    M, N, K1, K2, tb = shape
    rng = np.random.default_rng(M + N)
    A = rng.standard_normal((M, K1)).astype(np.float32)
    B = rng.standard_normal((N, K1) if tb else (K1, N)).astype(np.float32)
    A2 = rng.standard_normal((M, K2)).astype(np.float32) if K2 else None
    B2 = (rng.standard_normal((N, K2) if tb else (K2, N)).astype(np.float32)) if K2 else None
    bias = rng.standard_normal(N).astype(np.float32)
    rs = rng.random(M).astype(np.float32)
    ref = A.astype(np.float64) @ (B.T if tb else B)
    if K2:
        ref += A2.astype(np.float64) @ (B2.T if tb else B2)
    ref = np.maximum(ref + bias, 0) * rs[:, None]
    mask = rng.standard_normal((M, N + 4)).astype(np.float32) if K2 == 0 else None
    if mask is not None:  # ReLU-backward style mask with its own leading dim
        ref = np.where(mask[:, :N] > 0, ref, 0.0)
    out = torch.full((M, N), float("nan"), device="cuda")
    k = [_t(A), _t(B), _t(A2) if K2 else None, _t(B2) if K2 else None, _t(bias), _t(rs),
         _t(mask) if mask is not None else None]
    call("cg_gemm", M, N, K1, ptr(k[0]), K1, ptr(k[1]), K2, ptr(k[2]), K2, ptr(k[3]), tb,
         ptr(k[4]), 1, ptr(k[5]), ptr(k[6]), N + 4, ptr(out), N, mode, None, None, _st())
    _sync()
    got = out.cpu().numpy()
    scale = np.abs(ref).max()
    err = np.abs(got - ref).max() / scale
    assert err < (1e-5 if mode == 1 else 2e-3), err
    if mode == 1:
        # pre-split B (the weights path, RN split) vs splitting in smem: both ~fp32
        hl = []
        for b in (k[1], k[3]):
            if b is None:
                hl += [None, None]
                continue
            h, lo = torch.empty_like(b), torch.empty_like(b)
            call("cg_split_tf32", b.numel(), ptr(b), ptr(h), ptr(lo), _st())
            hl += [h, lo]
        out2 = torch.full((M, N), float("nan"), device="cuda")
        call("cg_gemm", M, N, K1, ptr(k[0]), K1, ptr(hl[0]), K2, ptr(k[2]), K2, ptr(hl[2]), tb,
             ptr(k[4]), 1, ptr(k[5]), ptr(k[6]), N + 4, ptr(out2), N, mode, ptr(hl[1]),
             ptr(hl[3]), _st())
        _sync()
        err2 = np.abs(out2.cpu().numpy() - ref).max() / scale
        assert err2 < 1e-5, err2


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("MKN", [(10000, 128, 40), (169343 // 8, 256, 256), (5000, 256, 128), (169343, 256, 256)])
def test_wgrad_tcgen05(MKN, mode):
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    M, K, N = MKN
    rng = np.random.default_rng(K + N)
    A = rng.standard_normal((M, K)).astype(np.float32)
    D = rng.standard_normal((M, N)).astype(np.float32)
    ws = torch.zeros(call("cg_wgrad_workspace", M, K, N), device="cuda")
    dW = torch.zeros(K, N, device="cuda")
    db = torch.zeros(N, device="cuda")
    tA, tD = _t(A), _t(D)
    call("cg_wgrad", M, K, N, ptr(tA), K, ptr(tD), N, ptr(dW), ptr(db), ptr(ws), mode, _st())
    _sync()
    # bias gradient (fused column sums under 3xTF32, standalone otherwise)
    refb = D.astype(np.float64).sum(0)
    errb = np.abs(db.cpu().numpy() - refb).max() / np.abs(refb).max()
    assert errb < 1e-5, errb
    ref = A.T.astype(np.float64) @ D
    err = np.abs(dW.cpu().numpy() - ref).max() / np.abs(ref).max()
    # 3xTF32 products are ~fp32-exact; what remains is fp32 accumulation over
    # split-K chunks of up to a few thousand vertices (error ~ sqrt(chunk) ulp)
    assert err < (3e-5 if mode == 1 else 2e-3), err
    first, firstb = dW.clone(), db.clone()
    call("cg_wgrad", M, K, N, ptr(tA), K, ptr(tD), N, ptr(dW), ptr(db), ptr(ws), mode, _st())
    _sync()
    assert torch.equal(first, dW)  # deterministic split-K
    assert torch.equal(firstb, db)


def test_split_tf32_transposed():
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    rng = np.random.default_rng(7)
    shapes = [(16, 32), (5, 7), (32, 40)]
    offs, flat = [], []
    o = 0
    for r, c in shapes:
        offs.append(o)
        flat.append(rng.standard_normal(r * c).astype(np.float32))
        o += (r * c + 3) // 4 * 4
        flat.append(np.zeros((r * c + 3) // 4 * 4 - r * c, np.float32))
    x = np.concatenate(flat)
    tx = _t(x)
    hi, lo = torch.zeros_like(tx), torch.zeros_like(tx)
    keep = [_t(np.array(offs, np.int64)), _t(np.array([s[0] for s in shapes], np.int32)),
            _t(np.array([s[1] for s in shapes], np.int32))]
    call("cg_split_tf32_t", len(shapes), ptr(keep[0]), ptr(keep[1]), ptr(keep[2]), ptr(tx),
         ptr(hi), ptr(lo), max(r * c for r, c in shapes), _st())
    _sync()
    h, lw = hi.cpu().numpy(), lo.cpu().numpy()
    for (r, c), o in zip(shapes, offs):
        m = x[o:o + r * c].reshape(r, c)
        ht = h[o:o + r * c].reshape(c, r)
        lt = lw[o:o + r * c].reshape(c, r)
        _check_tf32_split(m.T, ht, lt)


def _pack_bits(x):
    """(rows, F) -> (rows, F // 32) int32: bit j of word w = x[:, 32 w + j] > 0."""
    b = (np.asarray(x) > 0).reshape(x.shape[0], -1, 32).astype(np.uint64)
    w = (b << np.arange(32, dtype=np.uint64)).sum(-1).astype(np.uint32)
    return w.view(np.int32)


@pytest.mark.parametrize("shape", [(2000, 256, 128, 0), (777, 128, 64, 1), (1500, 64, 40, 1),
                                   (900, 256, 256, 0)], ids=lambda s: "x".join(map(str, s)))
def test_relu_bits_out_and_masked_gemm_bits(shape):
    """cg_gemm_mb: a ReLU layer's bits_out equals the > 0 pattern of the
    stored output exactly, and a mask-bits GEMM equals the fp32-mask GEMM
    bit for bit (same kernel arithmetic, only the mask operand differs)."""
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    M, N, K, tb = shape
    rng = np.random.default_rng(M + N + K)
    A = _t(rng.standard_normal((M, K)).astype(np.float32))
    B = _t(rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32))
    Bh, Bl = torch.empty_like(B), torch.empty_like(B)
    call("cg_split_tf32", B.numel(), ptr(B), ptr(Bh), ptr(Bl), _st())
    bias = _t(rng.standard_normal(N).astype(np.float32))
    rs = _t(rng.random(M).astype(np.float32))
    out = torch.empty(M, N, device="cuda")
    bits = torch.full((M, N // 32), -1, dtype=torch.int32, device="cuda")
    call("cg_gemm_mb", M, N, K, ptr(A), K, ptr(Bh), 0, None, 0, None, tb, ptr(bias), 1, ptr(rs),
         None, 0, ptr(bits), N // 32, ptr(out), N, 1, ptr(Bl), None, _st())
    _sync()
    assert np.array_equal(bits.cpu().numpy(), _pack_bits(out.cpu().numpy()))
    # masked GEMM: fp32 mask = out, vs its bits
    ref = torch.empty(M, N, device="cuda")
    got = torch.empty(M, N, device="cuda")
    call("cg_gemm", M, N, K, ptr(A), K, ptr(Bh), 0, None, 0, None, tb, None, 0, None, ptr(out),
         N, ptr(ref), N, 1, ptr(Bl), None, _st())
    call("cg_gemm_mb", M, N, K, ptr(A), K, ptr(Bh), 0, None, 0, None, tb, None, 0, None,
         ptr(bits), N // 32, None, 0, ptr(got), N, 1, ptr(Bl), None, _st())
    _sync()
    assert torch.equal(ref, got)
    assert (ref == 0).any() and (ref != 0).any()


@pytest.mark.parametrize("F", [32, 128, 256])
@pytest.mark.parametrize("sparse", [False, True])
def test_spmm_mask_bits_equal_fp32_mask(F, sparse):
    """cg_spmm_mb (mask as bits) == cg_spmm (fp32 mask) bit for bit, on both
    SpMM kernels and across the 128-column slices."""
    import torch
    from paper_2508_13716_b200._lib import call, ptr
    rng = np.random.default_rng(F)
    n_rows, n_src = 3000, 5000
    deg = rng.integers(0, 16, n_rows)
    rowptr = np.concatenate(([0], np.cumsum(deg))).astype(np.int64)
    col = np.sort(rng.integers(0, n_src, rowptr[-1]).astype(np.int32))
    X = _t(rng.standard_normal((n_src, F)).astype(np.float32))
    mask = rng.standard_normal((n_rows, F)).astype(np.float32)
    tm, tb_ = _t(mask), _t(_pack_bits(mask))
    add = _t(rng.standard_normal((n_rows, F)).astype(np.float32))
    sc = _t(rng.random(n_rows).astype(np.float32))
    tr, tc = _t(rowptr), _t(col)
    nnz = int(rowptr[-1]) if sparse else -1
    for addend in (None, add):
        a = torch.empty(n_rows, F, device="cuda")
        b = torch.empty(n_rows, F, device="cuda")
        ap = None if addend is None else ptr(addend)
        call("cg_spmm", n_rows, F, ptr(tr), ptr(tc), 1 << 62, None, ptr(X), F, ptr(sc), ap, F,
             ptr(tm), F, ptr(a), F, nnz, _st())
        call("cg_spmm_mb", n_rows, F, ptr(tr), ptr(tc), 1 << 62, None, ptr(X), F, ptr(sc), ap, F,
             ptr(tb_), F // 32, ptr(b), F, nnz, _st())
        _sync()
        assert torch.equal(a, b)
