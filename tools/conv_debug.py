import ctypes, os, sys, itertools
import torch, torch.nn.functional as F
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import _native
lib = _native.cuda_lib()
dev = torch.device("cuda:0")
def run(shape):
    n, c, h, w, k, r, stride, pad = shape
    p = (h + 2 * pad - r) // stride + 1; q = (w + 2 * pad - r) // stride + 1
    d = _native.ConvDesc(n, h, w, c, k, r, r, stride, pad, p, q)
    g = torch.Generator().manual_seed(0)
    x = torch.randn(n, c, h, w, generator=g); wt = torch.randn(k, c, r, r, generator=g) * (1.0 / (c * r * r) ** 0.5)
    dy = torch.randn(n, k, p, q, generator=g)
    xr = x.clone().requires_grad_(True); wr = wt.clone().requires_grad_(True)
    y = F.conv2d(xr, wr, stride=stride, padding=pad); y.backward(dy)
    x_d = x.permute(0, 2, 3, 1).contiguous().to(dev); w_d = wt.permute(0, 2, 3, 1).contiguous().to(dev)
    dy_d = dy.permute(0, 2, 3, 1).contiguous().to(dev)
    dx_d = torch.full((n, h, w, c), 7.0, device=dev); dw_d = torch.full((k, r, r, c), 7.0, device=dev)
    lib.accudnn_conv_dgrad(ctypes.byref(d), dy_d.data_ptr(), w_d.data_ptr(), dx_d.data_ptr(), 0, None)
    lib.accudnn_conv_wgrad(ctypes.byref(d), x_d.data_ptr(), dy_d.data_ptr(), dw_d.data_ptr(), 0, 1, None)
    torch.cuda.synchronize()
    e1 = ((dx_d.permute(0,3,1,2).cpu() - xr.grad).norm() / xr.grad.norm()).item()
    e2 = ((dw_d.permute(0,3,1,2).cpu() - wr.grad).norm() / wr.grad.norm()).item()
    return e1, e2, dx_d.abs().max().item(), dw_d.abs().max().item()
shape = (2, 64, 14, 14, 64, 1, 1, 0)
shape2 = (2, 128, 14, 14, 128, 1, 1, 0)
cfgs = sys.argv[1].split(";")
for cfg in cfgs:
    os.environ["ACCUDNN_DBG_MN"] = cfg
    try:
        print(cfg, "bn64", ["%.3g" % v for v in run(shape)], "bn128", ["%.3g" % v for v in run(shape2)], flush=True)
    except Exception as ex:
        print(cfg, "EXC", str(ex)[:80]); break
