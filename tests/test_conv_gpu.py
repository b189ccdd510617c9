"""Parity of the tcgen05 implicit-GEMM convolution kernels (fwd / dgrad /
wgrad, and FC as a 1x1 conv) against a plain PyTorch fp32 CPU reference.

Tolerance: the kernels multiply in TF32 (10-bit mantissa) and accumulate in
FP32, so each product carries ~2^-11 relative rounding; we require the
relative L2 error of the whole output to be below 2e-3 and the max abs error
below 2e-2 of the output's max magnitude.
"""
import ctypes

import pytest
import torch
import torch.nn.functional as F

from paper_1901_06773_b200 import _native

pytestmark = pytest.mark.gpu

SHAPES = [
    # n, c, h, w, k, r, stride, pad
    (2, 64, 14, 14, 64, 1, 1, 0),
    (2, 64, 14, 14, 128, 3, 1, 1),
    (3, 32, 15, 13, 96, 3, 2, 1),
    (2, 128, 14, 14, 256, 1, 2, 0),
    (2, 4, 32, 32, 64, 7, 2, 3),      # stem (3 channels padded to 4)
    (4, 256, 7, 7, 512, 3, 1, 1),
    (5, 2048, 1, 1, 1000, 1, 1, 0),   # fully connected
    (1, 36, 9, 9, 20, 3, 1, 1),       # ragged channel counts / tails
    # TMA-path shapes (ResNet-152 stage geometry at small batch)
    (4, 64, 56, 56, 64, 3, 1, 1),
    (8, 256, 14, 14, 256, 3, 1, 1),
    (4, 128, 28, 28, 128, 3, 2, 1),
    (8, 256, 14, 14, 1024, 1, 1, 0),
    (8, 1024, 14, 14, 256, 1, 1, 0),
    (8, 512, 14, 14, 1024, 1, 2, 0),
    (27, 2048, 1, 1, 1000, 1, 1, 0),
    (3, 96, 10, 10, 160, 3, 1, 1),
    # stride-2 data gradients (parity-class decomposition), odd and even sizes
    (4, 64, 16, 16, 64, 3, 2, 1),
    (2, 32, 7, 9, 64, 3, 2, 1),
    (2, 64, 12, 12, 32, 1, 2, 0),
    (3, 32, 11, 11, 64, 5, 2, 2),
    # split-K heavy (small M, long K): ResNet-152 stage 3/4 at k* = 27
    (27, 1024, 7, 7, 256, 1, 1, 0),
    (27, 256, 14, 14, 256, 3, 1, 1),
]


def desc(n, c, h, w, k, r, stride, pad):
    p = (h + 2 * pad - r) // stride + 1
    q = (w + 2 * pad - r) // stride + 1
    return _native.ConvDesc(n, h, w, c, k, r, r, stride, pad, p, q), p, q


def rel_err(got, ref):
    return ((got - ref).norm() / ref.norm().clamp_min(1e-30)).item()


def check(got, ref):
    got = got.double().cpu()
    ref = ref.double()
    assert rel_err(got, ref) < 2e-3, rel_err(got, ref)
    assert (got - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-6


@pytest.fixture(params=["tma", "tma_cluster2", "tma_pair", "tma_pair_bn256_split2", "tma_pair_bn64",
                        "tma_bn64_split3", "tma_bstat", "tma_streamk", "tma_streamk_bn64",
                        "tma_kpair", "tma_kpair_bn256", "tma_kpair_bn64", "tma_padd", "tma_padd_bn256",
                        "tma_padd_cluster2", "tma_padd_pair", "cpasync"])
def impl(request):
    """TMA kernel with the analytic config, with the B tile multicast across an
    M-tile pair (cluster of 2), as a CTA pair running 2-SM MMAs (256-row
    tiles, each CTA holding half of B), with narrow tiles + forced split-K,
    and the cp.async kernel."""
    lib = _native.cuda_lib()
    lib.accudnn_set_conv_impl(0 if request.param == "cpasync" else 1)
    if request.param == "tma_cluster2":
        lib.accudnn_conv_force_cfg(0, 0, 2)
    elif request.param == "tma_pair":
        lib.accudnn_conv_force_cfg(0, 0, 4)
    elif request.param == "tma_pair_bn256_split2":
        lib.accudnn_conv_force_cfg(256, 2, 4)
    elif request.param == "tma_pair_bn64":
        lib.accudnn_conv_force_cfg(64, 1, 4)
    elif request.param == "tma_bn64_split3":
        lib.accudnn_conv_force_cfg(64, 3, 1)
    elif request.param == "tma_bstat":  # B-stationary where the B tile fits, else analytic
        lib.accudnn_conv_force_cfg(64, 0, 3)
    elif request.param == "tma_streamk":  # stream-K with the in-kernel fix-up
        lib.accudnn_conv_force_cfg(0, -1, 0)
    elif request.param == "tma_streamk_bn64":
        lib.accudnn_conv_force_cfg(64, -1, 0)
    elif request.param == "tma_kpair":  # split-K over a CTA pair, reduced through DSMEM
        lib.accudnn_conv_force_cfg(0, 0, 5)
    elif request.param == "tma_kpair_bn256":
        lib.accudnn_conv_force_cfg(256, 0, 5)
    elif request.param == "tma_kpair_bn64":
        lib.accudnn_conv_force_cfg(64, 0, 5)
    elif request.param == "tma_padd":  # 2 slices reduce-added into the zeroed output
        lib.accudnn_conv_force_cfg(0, 0, 6)
    elif request.param == "tma_padd_bn256":
        lib.accudnn_conv_force_cfg(256, 0, 6)
    elif request.param == "tma_padd_cluster2":  # the same over multicast M-tile pairs
        lib.accudnn_conv_force_cfg(0, 0, 7)
    elif request.param == "tma_padd_pair":  # the same over 2-SM MMA pairs
        lib.accudnn_conv_force_cfg(0, 0, 8)
    yield request.param
    lib.accudnn_conv_force_cfg(0, 0, 0)
    lib.accudnn_set_conv_impl(1)


@pytest.mark.parametrize("shape", SHAPES)
def test_conv_fwd_dgrad_wgrad(cuda_dev, impl, shape):
    lib = _native.cuda_lib()
    n, c, h, w, k, r, stride, pad = shape
    d, p, q = desc(*shape)
    g = torch.Generator().manual_seed(0)
    x = torch.randn(n, c, h, w, generator=g)
    wt = torch.randn(k, c, r, r, generator=g) * (1.0 / (c * r * r) ** 0.5)
    dy = torch.randn(n, k, p, q, generator=g)

    xr = x.clone().requires_grad_(True)
    wr = wt.clone().requires_grad_(True)
    y_ref = F.conv2d(xr, wr, stride=stride, padding=pad)
    y_ref.backward(dy)

    # NHWC / [K][R][S][C] on the device
    x_d = x.permute(0, 2, 3, 1).contiguous().to(cuda_dev)
    w_d = wt.permute(0, 2, 3, 1).contiguous().to(cuda_dev)
    dy_d = dy.permute(0, 2, 3, 1).contiguous().to(cuda_dev)
    y_d = torch.empty(n, p, q, k, device=cuda_dev)
    dx_d = torch.empty(n, h, w, c, device=cuda_dev)
    dw_d = torch.empty(k, r, r, c, device=cuda_dev)

    assert lib.accudnn_conv_fwd(ctypes.byref(d), x_d.data_ptr(), w_d.data_ptr(),
                                y_d.data_ptr(), 0, None) == 0
    assert lib.accudnn_conv_dgrad(ctypes.byref(d), dy_d.data_ptr(), w_d.data_ptr(),
                                  dx_d.data_ptr(), 0, None) == 0
    assert lib.accudnn_conv_wgrad(ctypes.byref(d), x_d.data_ptr(), dy_d.data_ptr(),
                                  dw_d.data_ptr(), 0, 0, None) == 0
    torch.cuda.synchronize()

    check(y_d.permute(0, 3, 1, 2), y_ref.detach())
    check(dx_d.permute(0, 3, 1, 2), xr.grad)
    check(dw_d.permute(0, 3, 1, 2), wr.grad)


def test_conv_accumulate_beta(cuda_dev):
    lib = _native.cuda_lib()
    shape = (2, 64, 8, 8, 64, 3, 1, 1)
    d, p, q = desc(*shape)
    x = torch.randn(2, 8, 8, 64, device=cuda_dev)
    w = torch.randn(64, 3, 3, 64, device=cuda_dev) * 0.05
    y0 = torch.randn(2, p, q, 64, device=cuda_dev)
    y = y0.clone()
    y1 = torch.empty_like(y0)
    assert lib.accudnn_conv_fwd(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y.data_ptr(), 1, None) == 0
    assert lib.accudnn_conv_fwd(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y1.data_ptr(), 0, None) == 0
    torch.cuda.synchronize()
    assert torch.allclose(y, y0 + y1, rtol=1e-5, atol=1e-5)


def _run_all(lib, d, x_d, w_d, dy_d, outs):
    y_d, dx_d, dw_d = outs
    assert lib.accudnn_conv_fwd(ctypes.byref(d), x_d.data_ptr(), w_d.data_ptr(),
                                y_d.data_ptr(), 0, None) == 0
    assert lib.accudnn_conv_dgrad(ctypes.byref(d), dy_d.data_ptr(), w_d.data_ptr(),
                                  dx_d.data_ptr(), 0, None) == 0
    assert lib.accudnn_conv_wgrad(ctypes.byref(d), x_d.data_ptr(), dy_d.data_ptr(),
                                  dw_d.data_ptr(), 0, 0, None) == 0
    torch.cuda.synchronize()


@pytest.mark.parametrize("shape", [(27, 1024, 14, 14, 256, 1, 1, 0), (27, 256, 14, 14, 256, 3, 1, 1),
                                   (27, 512, 14, 14, 512, 3, 2, 1), (27, 2048, 7, 7, 512, 1, 1, 0)])
def test_conv_bitwise_deterministic(cuda_dev, shape):
    """split-K partials are reduced in slice order: repeated launches (and
    launches after unrelated work reorders the SM schedule) are bit-identical."""
    lib = _native.cuda_lib()
    n, c, h, w, k, r, stride, pad = shape
    d, p, q = desc(*shape)
    g = torch.Generator(device=cuda_dev).manual_seed(1)
    x_d = torch.randn(n, h, w, c, device=cuda_dev, generator=g)
    w_d = torch.randn(k, r, r, c, device=cuda_dev, generator=g) * 0.05
    dy_d = torch.randn(n, p, q, k, device=cuda_dev, generator=g)
    a = (torch.empty(n, p, q, k, device=cuda_dev), torch.empty(n, h, w, c, device=cuda_dev),
         torch.empty(k, r, r, c, device=cuda_dev))
    b = tuple(torch.empty_like(t) for t in a)
    _run_all(lib, d, x_d, w_d, dy_d, a)
    for _ in range(3):
        torch.randn(1 << 22, device=cuda_dev).sum()  # perturb the schedule
        _run_all(lib, d, x_d, w_d, dy_d, b)
        for u, v in zip(a, b):
            assert torch.equal(u, v)


def test_conv_small_workspace_limits_splits(cuda_dev):
    """a workspace too small for any split falls back to one K-slice per
    tile and still computes the same convolution."""
    lib = _native.cuda_lib()
    shape = (27, 1024, 7, 7, 256, 1, 1, 0)
    n, c, h, w, k, r, stride, pad = shape
    d, p, q = desc(*shape)
    x_d = torch.randn(n, h, w, c, device=cuda_dev)
    w_d = torch.randn(k, r, r, c, device=cuda_dev) * 0.03
    dy_d = torch.randn(n, p, q, k, device=cuda_dev)
    a = (torch.empty(n, p, q, k, device=cuda_dev), torch.empty(n, h, w, c, device=cuda_dev),
         torch.empty(k, r, r, c, device=cuda_dev))
    b = tuple(torch.empty_like(t) for t in a)
    _run_all(lib, d, x_d, w_d, dy_d, a)
    try:
        assert lib.accudnn_conv_set_workspace(None, 0) == 0  # split-K disabled
        _run_all(lib, d, x_d, w_d, dy_d, b)
    finally:
        lib.accudnn_conv_set_workspace(None, 64 << 20)
    for u, v in zip(a, b):
        assert rel_err(u.double(), v.double()) < 1e-5


@pytest.mark.parametrize("shape", [(2, 32, 8, 8, 64, 1, 2, 0), (2, 64, 10, 10, 64, 3, 2, 1)])
def test_dgrad_strided_accumulate(cuda_dev, shape):
    """beta = 1 adds the stride-2 data gradient onto an existing one (the
    block input of a ResNet downsample receives two gradient contributions)."""
    lib = _native.cuda_lib()
    n, c, h, w, k, r, stride, pad = shape
    d, p, q = desc(*shape)
    w_d = torch.randn(k, r, r, c, device=cuda_dev) * 0.05
    dy_d = torch.randn(n, p, q, k, device=cuda_dev)
    base = torch.randn(n, h, w, c, device=cuda_dev)
    acc = base.clone()
    fresh = torch.full_like(base, float("nan"))
    assert lib.accudnn_conv_dgrad(ctypes.byref(d), dy_d.data_ptr(), w_d.data_ptr(),
                                  acc.data_ptr(), 1, None) == 0
    assert lib.accudnn_conv_dgrad(ctypes.byref(d), dy_d.data_ptr(), w_d.data_ptr(),
                                  fresh.data_ptr(), 0, None) == 0
    torch.cuda.synchronize()
    assert not torch.isnan(fresh).any()
    assert torch.allclose(acc, base + fresh, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("shape,forced", [((8, 256, 14, 14, 1024, 1, 1, 0), (0, 0, 0)),
                                          ((8, 256, 14, 14, 1024, 1, 1, 0), (128, 0, 3)),
                                          ((27, 1024, 14, 14, 256, 1, 1, 0), (256, 4, 1)),
                                          ((4, 64, 28, 28, 64, 3, 1, 1), (0, 0, 2)),
                                          ((5, 128, 14, 14, 256, 3, 1, 1), (0, 0, 4)),
                                          ((3, 96, 10, 10, 160, 3, 1, 1), (0, 0, 0))])
def test_conv_fwd_stats_and_bn_from_stats(cuda_dev, shape, forced):
    """the forward conv's epilogue (or its split-K reduce) writes per-32-row
    column sums / sums of squares of the output; a batch norm fed with them
    equals the one that reads the output itself"""
    lib = _native.cuda_lib()
    n, c, h, w, k, r, stride, pad = shape
    d, p, q = desc(*shape)
    lib.accudnn_conv_force_cfg(*forced)
    try:
        x = torch.randn(n, h, w, c, device=cuda_dev)
        wt = torch.randn(k, r, r, c, device=cuda_dev) * (1.0 / (c * r * r) ** 0.5)
        y = torch.empty(n, p, q, k, device=cuda_dev)
        M = n * p * q
        P = (M + 31) // 32
        stats = torch.full((2, P, k), float("nan"), device=cuda_dev)
        produced = ctypes.c_int(0)
        assert lib.accudnn_conv_fwd_stats(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), y.data_ptr(),
                                          stats.data_ptr(), ctypes.byref(produced), None) == 0
        torch.cuda.synchronize()
    finally:
        lib.accudnn_conv_force_cfg(0, 0, 0)
    assert produced.value == 1
    yf = y.reshape(M, k).double()
    pad_rows = P * 32 - M
    yp = torch.cat([yf, torch.zeros(pad_rows, k, device=cuda_dev, dtype=torch.float64)])
    ref1 = yp.reshape(P, 32, k).sum(1)
    ref2 = (yp * yp).reshape(P, 32, k).sum(1)
    assert rel_err(stats[0].double(), ref1) < 1e-5
    assert rel_err(stats[1].double(), ref2) < 1e-5
    g, b = torch.rand(k, device=cuda_dev) + 0.5, torch.randn(k, device=cuda_dev) * 0.1
    ws = torch.zeros(lib.accudnn_bn_workspace_bytes(k) // 4 + 1, device=cuda_dev)
    P_ = ctypes.c_void_p
    outs = []
    for use_stats in (False, True):
        yy = torch.empty_like(y)
        mean, inv = torch.empty(k, device=cuda_dev), torch.empty(k, device=cuda_dev)
        if use_stats:
            rc = lib.accudnn_bn_fwd_stats(P_(y.data_ptr()), P_(stats.data_ptr()), M, k, P_(g.data_ptr()),
                                          P_(b.data_ptr()), 1e-5, 1, P_(yy.data_ptr()), P_(mean.data_ptr()),
                                          P_(inv.data_ptr()), None, None, 0.1, P_(ws.data_ptr()), None)
        else:
            rc = lib.accudnn_bn_fwd(P_(y.data_ptr()), M, k, P_(g.data_ptr()), P_(b.data_ptr()), 1e-5, 1,
                                    P_(yy.data_ptr()), P_(mean.data_ptr()), P_(inv.data_ptr()), None,
                                    None, 0.1, P_(ws.data_ptr()), None)
        assert rc == 0
        torch.cuda.synchronize()
        outs.append((yy, mean, inv))
    assert rel_err(outs[1][1].double(), outs[0][1].double()) < 1e-5
    assert rel_err(outs[1][2].double(), outs[0][2].double()) < 1e-4
    assert rel_err(outs[1][0].double(), outs[0][0].double()) < 1e-4


@pytest.mark.parametrize("shape", [(27, 256, 14, 14, 256, 3, 1, 1), (27, 2048, 7, 7, 512, 1, 1, 0),
                                   (8, 128, 28, 28, 128, 3, 2, 1), (27, 2048, 1, 1, 1000, 1, 1, 0)])
def test_streamk_deterministic_and_accumulating(cuda_dev, shape):
    """stream-K: the tile's partial segments are summed in segment order by
    whichever CTA arrives last, so repeated launches are bit-identical; beta
    = 1 adds onto the existing output; the per-tile counters return to zero
    (a following launch is exact again)."""
    lib = _native.cuda_lib()
    n, c, h, w, k, r, stride, pad = shape
    d, p, q = desc(*shape)
    g = torch.Generator(device=cuda_dev).manual_seed(3)
    x_d = torch.randn(n, h, w, c, device=cuda_dev, generator=g)
    w_d = torch.randn(k, r, r, c, device=cuda_dev, generator=g) * 0.05
    dy_d = torch.randn(n, p, q, k, device=cuda_dev, generator=g)
    lib.accudnn_conv_force_cfg(0, -1, 0)
    try:
        a = (torch.empty(n, p, q, k, device=cuda_dev), torch.empty(n, h, w, c, device=cuda_dev),
             torch.empty(k, r, r, c, device=cuda_dev))
        _run_all(lib, d, x_d, w_d, dy_d, a)
        for _ in range(3):
            b = tuple(torch.full_like(t, float("nan")) for t in a)
            torch.randn(1 << 22, device=cuda_dev).sum()  # perturb the schedule
            _run_all(lib, d, x_d, w_d, dy_d, b)
            for u, v in zip(a, b):
                assert torch.equal(u, v)
        base = torch.randn_like(a[1])
        acc = base.clone()
        assert lib.accudnn_conv_dgrad(ctypes.byref(d), dy_d.data_ptr(), w_d.data_ptr(),
                                      acc.data_ptr(), 1, None) == 0
        torch.cuda.synchronize()
        assert torch.allclose(acc, base + a[1], rtol=1e-5, atol=1e-5)
    finally:
        lib.accudnn_conv_force_cfg(0, 0, 0)
    ref = tuple(torch.empty_like(t) for t in a)
    _run_all(lib, d, x_d, w_d, dy_d, ref)  # default config (split-K / reduce kernel)
    for u, v in zip(a, ref):
        assert rel_err(u.double(), v.double()) < 1e-5


@pytest.mark.parametrize("shape", [(27, 256, 14, 14, 256, 3, 1, 1), (42, 256, 14, 14, 256, 3, 1, 1),
                                   (42, 1024, 14, 14, 256, 1, 1, 0), (42, 256, 14, 14, 1024, 1, 1, 0),
                                   (42, 512, 7, 7, 512, 3, 1, 1), (3, 96, 10, 10, 160, 3, 1, 1)])
@pytest.mark.parametrize("bn", [64, 128, 256])
def test_kpair_equals_two_slice_workspace_reduction(cuda_dev, shape, bn):
    """The DSMEM-reduced split-K pair (cm 5) computes slice 0 + slice 1 of the
    same k-block partition as the 2-slice workspace path (splits 2), so both
    are bit-identical, for overwrite and for accumulation (beta = 1), on the
    forward and the data gradient; repeated launches are bit-identical."""
    lib = _native.cuda_lib()
    n, c, h, w, k, r, stride, pad = shape
    d, p, q = desc(*shape)
    g = torch.Generator(device=cuda_dev).manual_seed(5)
    x_d = torch.randn(n, h, w, c, device=cuda_dev, generator=g)
    w_d = torch.randn(k, r, r, c, device=cuda_dev, generator=g) * 0.05
    dy_d = torch.randn(n, p, q, k, device=cuda_dev, generator=g)
    base_y = torch.randn(n, p, q, k, device=cuda_dev, generator=g)
    base_x = torch.randn(n, h, w, c, device=cuda_dev, generator=g)

    def run(cm):
        lib.accudnn_conv_force_cfg(bn, 2, cm)
        try:
            y, dx = torch.full_like(base_y, float("nan")), torch.full_like(base_x, float("nan"))
            ya, dxa = base_y.clone(), base_x.clone()
            for out, beta in ((y, 0), (ya, 1)):
                assert lib.accudnn_conv_fwd(ctypes.byref(d), x_d.data_ptr(), w_d.data_ptr(),
                                            out.data_ptr(), beta, None) == 0
            for out, beta in ((dx, 0), (dxa, 1)):
                assert lib.accudnn_conv_dgrad(ctypes.byref(d), dy_d.data_ptr(), w_d.data_ptr(),
                                              out.data_ptr(), beta, None) == 0
            torch.cuda.synchronize()
            return y, ya, dx, dxa
        finally:
            lib.accudnn_conv_force_cfg(0, 0, 0)

    # the 2-slice workspace path needs 2 x M x N floats of workspace
    lib.accudnn_conv_set_workspace(None, ctypes.c_ulonglong(512 << 20))
    try:
        ws = run(1)
    finally:
        lib.accudnn_conv_set_workspace(None, ctypes.c_ulonglong(64 << 20))
    kp = run(5)
    again = run(5)
    for u, v, t in zip(ws, kp, again):
        assert torch.equal(u, v)
        assert torch.equal(v, t)
    # cm 6: the same two slices reduce-added into the zeroed output in L2
    # (overwrite calls; accumulating calls fall back to another config)
    pa = run(6)
    pa2 = run(6)
    for i in (0, 2):  # y, dx (beta = 0)
        assert torch.equal(ws[i], pa[i])
        assert torch.equal(pa[i], pa2[i])
    for i in (1, 3):
        assert rel_err(pa[i].double(), ws[i].double()) < 1e-5
    # cm 7 / 8: the reduce-adds over CTA pairs (multicast / 2-SM MMA) equal the
    # same pairs' 2-slice workspace reduction (cm 2 / 4, splits 2)
    for cm_ws, cm_pa in ((2, 7), (4, 8)):
        lib.accudnn_conv_set_workspace(None, ctypes.c_ulonglong(512 << 20))
        try:
            wsp = run(cm_ws)
        finally:
            lib.accudnn_conv_set_workspace(None, ctypes.c_ulonglong(64 << 20))
        pp, pp2 = run(cm_pa), run(cm_pa)
        for i in (0, 2):
            assert torch.equal(wsp[i], pp[i]), (cm_pa, i)
            assert torch.equal(pp[i], pp2[i])
        for i in (1, 3):
            assert rel_err(pp[i].double(), wsp[i].double()) < 1e-5
    ref = F.conv2d(x_d.permute(0, 3, 1, 2).double().cpu(), w_d.permute(0, 3, 1, 2).double().cpu(),
                   stride=stride, padding=pad)
    check(kp[0].permute(0, 3, 1, 2), ref)


@pytest.mark.parametrize("shape", [(8, 256, 14, 14, 256, 3, 1, 1), (8, 1024, 14, 14, 256, 1, 1, 0),
                                   (4, 128, 28, 28, 128, 3, 2, 1), (4, 64, 56, 56, 64, 3, 1, 1),
                                   (27, 2048, 1, 1, 1000, 1, 1, 0)])
def test_precise_3xtf32_on_tma_kernels(cuda_dev, shape):
    """3xTF32 with a precise scratch registered: fwd / dgrad / wgrad run as three
    TF32 tcgen05 GEMMs (hi*hi + hi*lo + lo*hi) and reach fp32 accuracy against
    an fp64 reference (relative L2 error < 5e-5, vs ~1e-3 for plain TF32), as
    the cp.async PRECISE kernel (no scratch) does."""
    lib = _native.cuda_lib()
    n, c, h, w, k, r, stride, pad = shape
    d, p, q = desc(*shape)
    g = torch.Generator().manual_seed(7)
    x = torch.randn(n, c, h, w, generator=g, dtype=torch.float64)
    wt = torch.randn(k, c, r, r, generator=g, dtype=torch.float64) / (c * r * r) ** 0.5
    dy = torch.randn(n, k, p, q, generator=g, dtype=torch.float64)
    xr = x.clone().requires_grad_(True)
    wr = wt.clone().requires_grad_(True)
    y_ref = F.conv2d(xr, wr, stride=stride, padding=pad)
    y_ref.backward(dy)
    x_d = x.float().permute(0, 2, 3, 1).contiguous().to(cuda_dev)
    w_d = wt.float().permute(0, 2, 3, 1).contiguous().to(cuda_dev)
    dy_d = dy.float().permute(0, 2, 3, 1).contiguous().to(cuda_dev)
    need = lib.accudnn_conv_precise_scratch_bytes(ctypes.byref(d))
    scratch = torch.empty(need // 4 + 64, device=cuda_dev)
    outs = {}
    lib.accudnn_set_conv_math(1)
    try:
        for tag, sc in (("tma", scratch), ("cpasync", None)):
            lib.accudnn_conv_set_precise_scratch(None, ctypes.c_void_p(sc.data_ptr() if sc is not None else 0),
                                                 ctypes.c_ulonglong(need if sc is not None else 0))
            y_d = torch.empty(n, p, q, k, device=cuda_dev)
            dx_d = torch.empty(n, h, w, c, device=cuda_dev)
            dw_d = torch.empty(k, r, r, c, device=cuda_dev)
            assert lib.accudnn_conv_fwd(ctypes.byref(d), x_d.data_ptr(), w_d.data_ptr(), y_d.data_ptr(), 0, None) == 0
            assert lib.accudnn_conv_dgrad(ctypes.byref(d), dy_d.data_ptr(), w_d.data_ptr(), dx_d.data_ptr(), 0,
                                          None) == 0
            assert lib.accudnn_conv_wgrad(ctypes.byref(d), x_d.data_ptr(), dy_d.data_ptr(), dw_d.data_ptr(), 0, 0,
                                          None) == 0
            torch.cuda.synchronize()
            outs[tag] = (y_d, dx_d, dw_d)
    finally:
        lib.accudnn_conv_set_precise_scratch(None, None, ctypes.c_ulonglong(0))
        lib.accudnn_set_conv_math(0)
    refs = (y_ref.detach(), xr.grad, wr.grad)
    for tag in ("tma", "cpasync"):
        for got, ref in zip(outs[tag], refs):
            err = rel_err(got.permute(0, 3, 1, 2).double().cpu(), ref)
            assert err < 5e-5, (tag, err)
