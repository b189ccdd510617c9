"""Parity of the HBM-bound layer kernels (csrc/kernels/pointwise.cu) against
plain PyTorch fp32 CPU references of the same ops, called through the C ABI
(include/accudnn_kernels.h).

Tolerances (stated): these kernels compute in fp32 (BN statistics finalised
in fp64), so results agree with PyTorch's fp32 CPU ops to rel-L2 1e-5 /
max-abs 1e-4 of the output scale; the routing ops (ReLU, add, max-pool, SGD)
are exact up to fp32 rounding of the same expressions.  The per-channel
reductions are deterministic: repeated launches are bit-identical.
"""
import ctypes

import pytest
import torch
import torch.nn.functional as F

from paper_1901_06773_b200 import _native

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


BN_CASES = [(27 * 14 * 14, 256, 1), (27 * 7 * 7, 2048, 0), (4 * 112 * 112, 64, 1), (6, 12, 1),
            (8 * 28 * 28, 512, 0), (300, 8192, 1)]


@pytest.mark.parametrize("M,C,relu", BN_CASES)
def test_batchnorm_fwd_bwd(cuda_dev, M, C, relu):
    lib = _native.cuda_lib()
    g = torch.Generator().manual_seed(M + C)
    x = torch.randn(M, C, generator=g) * 2.0 + 0.5
    gamma = torch.rand(C, generator=g) + 0.5
    beta = torch.randn(C, generator=g) * 0.1
    dy = torch.randn(M, C, generator=g)
    eps, mom = 1e-5, 0.1

    xr = x.clone().requires_grad_(True)
    gr = gamma.clone().requires_grad_(True)
    br = beta.clone().requires_grad_(True)
    rm, rv = torch.zeros(C), torch.ones(C)
    y_ref = F.batch_norm(xr, rm, rv, gr, br, training=True, momentum=mom, eps=eps)
    if relu:
        y_ref = F.relu(y_ref)
    y_ref.backward(dy)

    d = cuda_dev
    x_d, dy_d, g_d, b_d = x.to(d), dy.to(d), gamma.to(d), beta.to(d)
    y_d = torch.empty_like(x_d)
    mean_d, inv_d = torch.empty(C, device=d), torch.empty(C, device=d)
    rm_d, rv_d = torch.zeros(C, device=d), torch.ones(C, device=d)
    ws = torch.zeros(lib.accudnn_bn_workspace_bytes(C) // 4 + 1, device=d)
    assert lib.accudnn_bn_fwd(ptr(x_d), M, C, ptr(g_d), ptr(b_d), eps, relu, ptr(y_d), ptr(mean_d),
                              ptr(inv_d), ptr(rm_d), ptr(rv_d), mom, ptr(ws), None) == 0
    dx_d = torch.full_like(x_d, float("nan"))
    dg_d, db_d = torch.empty(C, device=d), torch.empty(C, device=d)
    assert lib.accudnn_bn_bwd(ptr(x_d), ptr(dy_d), M, C, ptr(g_d), ptr(b_d), ptr(mean_d), ptr(inv_d),
                              relu, ptr(dx_d), 0, ptr(dg_d), ptr(db_d), ptr(ws), None) == 0
    torch.cuda.synchronize()
    assert rel(y_d, y_ref.detach()) < 1e-5
    assert rel(mean_d, x.mean(0)) < 1e-5
    assert rel(rm_d, rm) < 1e-5 and rel(rv_d, rv) < 1e-5
    assert rel(dx_d, xr.grad) < 1e-4
    assert rel(dg_d, gr.grad) < 1e-4
    assert rel(db_d, br.grad) < 1e-5

    # accumulate mode + bitwise determinism of the reductions
    base = torch.randn_like(x_d)
    acc = base.clone()
    assert lib.accudnn_bn_bwd(ptr(x_d), ptr(dy_d), M, C, ptr(g_d), ptr(b_d), ptr(mean_d), ptr(inv_d),
                              relu, ptr(acc), 1, ptr(dg_d), ptr(db_d), ptr(ws), None) == 0
    y2 = torch.empty_like(y_d)
    mean2 = torch.empty_like(mean_d)
    assert lib.accudnn_bn_fwd(ptr(x_d), M, C, ptr(g_d), ptr(b_d), eps, relu, ptr(y2), ptr(mean2),
                              ptr(inv_d), None, None, mom, ptr(ws), None) == 0
    torch.cuda.synchronize()
    assert torch.allclose(acc, base + dx_d, rtol=1e-5, atol=1e-5)
    assert torch.equal(y2, y_d) and torch.equal(mean2, mean_d)


@pytest.mark.parametrize("M,C", [(42 * 56 * 56, 64), (27 * 14 * 14, 256), (8, 12)])
def test_batchnorm_large_channel_mean(cuda_dev, M, C):
    """|mean| = 1000 x std: E[x^2] - E[x]^2 in fp32 partial sums would lose
    every significant digit of the variance; the kernel's shifted sums keep
    it within 1e-4 of PyTorch's (stable) reduction."""
    lib = _native.cuda_lib()
    g = torch.Generator().manual_seed(7 + C)
    x = torch.randn(M, C, generator=g) * 0.5 + 500.0 * (1.0 + torch.rand(C, generator=g))
    gamma, beta = torch.ones(C), torch.zeros(C)
    rm, rv = torch.zeros(C, dtype=torch.float64), torch.ones(C, dtype=torch.float64)
    y_ref = F.batch_norm(x.double(), rm, rv, gamma.double(), beta.double(),
                         training=True, momentum=0.1, eps=1e-5)
    d = cuda_dev
    x_d = x.to(d)
    y_d = torch.empty_like(x_d)
    mean_d, inv_d = torch.empty(C, device=d), torch.empty(C, device=d)
    rm_d, rv_d = torch.zeros(C, device=d), torch.ones(C, device=d)
    ws = torch.zeros(lib.accudnn_bn_workspace_bytes(C) // 4 + 1, device=d)
    assert lib.accudnn_bn_fwd(ptr(x_d), M, C, ptr(gamma.to(d)), ptr(beta.to(d)), 1e-5, 0, ptr(y_d),
                              ptr(mean_d), ptr(inv_d), ptr(rm_d), ptr(rv_d), 0.1, ptr(ws), None) == 0
    torch.cuda.synchronize()
    var = x.double().var(0, unbiased=False)
    assert rel(1.0 / inv_d.double() ** 2 - 1e-5, var) < 1e-4
    assert rel(y_d, y_ref) < 1e-4
    assert rel(rv_d, rv) < 1e-4


@pytest.mark.parametrize("M,C", [(42 * 56 * 56, 256), (27 * 14 * 14, 1024), (27 * 7 * 7, 2048),
                                 (8 * 32 * 32, 16), (5, 8)])
def test_bn_add_relu(cuda_dev, M, C):
    """y = relu(bn(x) + skip) as one op, forward and backward (both input
    gradients, accumulate flags) vs torch fp32 autograd of the unfused ops."""
    lib = _native.cuda_lib()
    g = torch.Generator().manual_seed(M + 7 * C)
    x = torch.randn(M, C, generator=g) * 1.5 - 0.3
    skip = torch.randn(M, C, generator=g)
    gamma = torch.rand(C, generator=g) + 0.5
    beta = torch.randn(C, generator=g) * 0.1
    dy = torch.randn(M, C, generator=g)
    xr = x.clone().requires_grad_(True)
    gr, br = gamma.clone().requires_grad_(True), beta.clone().requires_grad_(True)
    pre = F.batch_norm(xr, None, None, gr, br, training=True, eps=1e-5) + skip
    y_ref = F.relu(pre)
    d = cuda_dev
    x_d, s_d, dy_d, g_d, b_d = x.to(d), skip.to(d), dy.to(d), gamma.to(d), beta.to(d)
    y_d = torch.empty_like(x_d)
    mean_d, inv_d = torch.empty(C, device=d), torch.empty(C, device=d)
    ws = torch.zeros(lib.accudnn_bn_workspace_bytes(C) // 4 + 1, device=d)
    assert lib.accudnn_bn_add_relu_fwd(ptr(x_d), ptr(s_d), M, C, ptr(g_d), ptr(b_d), 1e-5, ptr(y_d),
                                       ptr(mean_d), ptr(inv_d), None, None, 0.1, ptr(ws), None) == 0
    # reference backward through the device forward's ReLU mask (elements at
    # |pre-activation| ~ 1e-7 may round to the other side of 0 in torch's BN)
    g_ref = dy * (y_d.cpu() > 0)
    pre.backward(g_ref)
    dx_d = torch.full_like(x_d, float("nan"))
    base = torch.randn_like(x_d)
    ds_d = base.clone()  # the shortcut gradient accumulates (beta = 1)
    dg_d, db_d = torch.empty(C, device=d), torch.empty(C, device=d)
    assert lib.accudnn_bn_add_relu_bwd(ptr(x_d), ptr(s_d), ptr(dy_d), M, C, ptr(g_d), ptr(b_d),
                                       ptr(mean_d), ptr(inv_d), ptr(dx_d), 0, ptr(ds_d), 1,
                                       ptr(dg_d), ptr(db_d), ptr(ws), None) == 0
    torch.cuda.synchronize()
    assert rel(y_d, y_ref.detach()) < 1e-5
    assert rel(dx_d, xr.grad) < 1e-4
    assert torch.equal(ds_d.cpu(), base.cpu() + g_ref)
    assert rel(dg_d, gr.grad) < 1e-4
    assert rel(db_d, br.grad) < 1e-5


def test_batchnorm_shared_workspace_mixed_widths(cuda_dev):
    """one workspace serves layers of different channel counts in turn (as in
    the executor): every call must still finalise its own statistics."""
    lib = _native.cuda_lib()
    ws = torch.zeros(lib.accudnn_bn_workspace_bytes(512) // 4 + 1, device=cuda_dev)
    for M, C in [(4096, 16), (1024, 512), (2048, 64), (4096, 16), (512, 256)]:
        x = torch.randn(M, C, device=cuda_dev)
        g, b = torch.ones(C, device=cuda_dev), torch.zeros(C, device=cuda_dev)
        y = torch.empty_like(x)
        mean, inv = torch.empty(C, device=cuda_dev), torch.empty(C, device=cuda_dev)
        assert lib.accudnn_bn_fwd(ptr(x), M, C, ptr(g), ptr(b), 1e-5, 0, ptr(y), ptr(mean), ptr(inv),
                                  None, None, 0.1, ptr(ws), None) == 0
        dy = torch.randn_like(x)
        dx, dg, db = torch.empty_like(x), torch.empty(C, device=cuda_dev), torch.empty(C, device=cuda_dev)
        assert lib.accudnn_bn_bwd(ptr(x), ptr(dy), M, C, ptr(g), ptr(b), ptr(mean), ptr(inv), 0,
                                  ptr(dx), 0, ptr(dg), ptr(db), ptr(ws), None) == 0
        torch.cuda.synchronize()
        assert rel(mean, x.mean(0)) < 1e-5
        assert rel(db, dy.sum(0)) < 1e-5
        xh = (x - x.mean(0)) / torch.sqrt(x.var(0, unbiased=False) + 1e-5)
        assert rel(dg, (dy * xh).sum(0)) < 1e-4


def test_relu_add_copy(cuda_dev):
    lib = _native.cuda_lib()
    n = 4 * 1000
    a, b, dy = (torch.randn(n, device=cuda_dev) for _ in range(3))
    y = torch.empty_like(a)
    assert lib.accudnn_relu_fwd(ptr(a), ptr(y), n, None) == 0
    s = torch.empty_like(a)
    assert lib.accudnn_add_fwd(ptr(a), ptr(b), ptr(s), n, None) == 0
    dx = torch.empty_like(a)
    assert lib.accudnn_relu_bwd(ptr(a), ptr(dy), ptr(dx), n, 0, None) == 0
    c = b.clone()
    assert lib.accudnn_copy(ptr(a), ptr(c), n, 1, None) == 0
    torch.cuda.synchronize()
    assert torch.equal(y, torch.relu(a))
    assert torch.equal(s, a + b)
    assert torch.equal(dx, torch.where(a > 0, dy, torch.zeros_like(dy)))
    assert torch.equal(c, b + a)


@pytest.mark.parametrize("n,h,w,c,k,st,pad", [(3, 112, 112, 64, 3, 2, 1), (2, 9, 7, 8, 3, 2, 1),
                                              (2, 8, 8, 4, 2, 2, 0)])
def test_maxpool(cuda_dev, n, h, w, c, k, st, pad):
    lib = _native.cuda_lib()
    # distinct values: no ties, so the routed gradient is unambiguous
    x = torch.randperm(n * h * w * c).float().reshape(n, c, h, w) / (n * h * w * c)
    xr = x.clone().requires_grad_(True)
    y_ref = F.max_pool2d(xr, k, st, pad)
    p, q = y_ref.shape[2], y_ref.shape[3]
    dy = torch.randn(n, c, p, q)
    y_ref.backward(dy)
    x_d = x.permute(0, 2, 3, 1).contiguous().to(cuda_dev)
    dy_d = dy.permute(0, 2, 3, 1).contiguous().to(cuda_dev)
    y_d = torch.empty(n, p, q, c, device=cuda_dev)
    dx_d = torch.empty_like(x_d)
    assert lib.accudnn_maxpool_fwd(ptr(x_d), n, h, w, c, k, k, st, pad, p, q, ptr(y_d), None) == 0
    assert lib.accudnn_maxpool_bwd(ptr(x_d), ptr(dy_d), n, h, w, c, k, k, st, pad, p, q,
                                   ptr(dx_d), None) == 0
    torch.cuda.synchronize()
    assert torch.equal(y_d.permute(0, 3, 1, 2).cpu(), y_ref.detach())
    assert rel(dx_d.permute(0, 3, 1, 2), xr.grad) < 1e-6


def test_avgpool_xent_sgd(cuda_dev):
    lib = _native.cuda_lib()
    n, hw, c, classes = 5, 49, 64, 10
    x = torch.randn(n, hw, c)
    y_d = torch.empty(n, c, device=cuda_dev)
    assert lib.accudnn_avgpool_fwd(ptr(x.to(cuda_dev)), n, hw, c, ptr(y_d), None) == 0
    dy = torch.randn(n, c)
    dx_d = torch.empty(n, hw, c, device=cuda_dev)
    assert lib.accudnn_avgpool_bwd(ptr(dy.to(cuda_dev)), n, hw, c, ptr(dx_d), None) == 0
    torch.cuda.synchronize()
    assert rel(y_d, x.mean(1)) < 1e-6
    assert rel(dx_d, (dy / hw).unsqueeze(1).expand(n, hw, c)) < 1e-6

    z = torch.randn(n, classes)
    lab = torch.randint(0, classes, (n,), dtype=torch.int32)
    zr = z.clone().requires_grad_(True)
    loss_ref = F.cross_entropy(zr, lab.long())
    loss_ref.backward()
    z_d, lab_d = z.to(cuda_dev), lab.to(cuda_dev)
    loss_d = torch.zeros(1, device=cuda_dev)
    dz_d, db_d = torch.empty(n, classes, device=cuda_dev), torch.empty(classes, device=cuda_dev)
    assert lib.accudnn_xent_fwd(ptr(z_d), ptr(lab_d), n, classes, ptr(loss_d), None) == 0
    assert lib.accudnn_xent_bwd(ptr(z_d), ptr(lab_d), n, classes, ptr(dz_d), ptr(db_d), None) == 0
    torch.cuda.synchronize()
    assert abs(loss_d.item() - loss_ref.item()) < 1e-5 * abs(loss_ref.item())
    assert rel(dz_d, zr.grad) < 1e-5
    assert rel(db_d, zr.grad.sum(0)) < 1e-5

    # SGD momentum (torch.optim.SGD semantics: buf = g + wd*w first step, then mu*buf + ...)
    w = torch.randn(1000)
    gr = torch.randn(1000)
    p = torch.nn.Parameter(w.clone())
    opt = torch.optim.SGD([p], lr=0.1, momentum=0.9, weight_decay=1e-4)
    w_d, g_d, buf_d = w.to(cuda_dev), gr.to(cuda_dev), torch.zeros(1000, device=cuda_dev)
    for first in (1, 0):
        p.grad = gr.clone()
        opt.step()
        assert lib.accudnn_sgd_update(ptr(w_d), ptr(g_d), ptr(buf_d), 1000, 0.1, 0.9, 1e-4, 1.0,
                                      first, None) == 0
    torch.cuda.synchronize()
    assert rel(w_d, p.detach()) < 1e-6
