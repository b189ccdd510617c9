"""Compare the DSMEM split-K pair (cm 5) with the 2-slice workspace path on
fwd / dgrad, overwrite and accumulate."""
import ctypes
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import _native  # noqa: E402

lib = _native.cuda_lib()
dev = torch.device("cuda:0")
for shape in [(42, 1024, 14, 14, 256, 1, 1, 0), (42, 256, 14, 14, 256, 3, 1, 1), (42, 256, 14, 14, 1024, 1, 1, 0)]:
    for bn in (64, 128, 256):
        n, c, h, w, k, r, st, pad = shape
        p = (h + 2 * pad - r) // st + 1
        q = (w + 2 * pad - r) // st + 1
        d = _native.ConvDesc(n, h, w, c, k, r, r, st, pad, p, q)
        g = torch.Generator(device=dev).manual_seed(5)
        x = torch.randn(n, h, w, c, device=dev, generator=g)
        wt = torch.randn(k, r, r, c, device=dev, generator=g) * 0.05
        dy = torch.randn(n, p, q, k, device=dev, generator=g)
        by = torch.randn(n, p, q, k, device=dev, generator=g)
        bx = torch.randn(n, h, w, c, device=dev, generator=g)
        outs = {}
        for name, cm in (("ws", 1), ("kc", 5)):
            lib.accudnn_conv_force_cfg(bn, 2, cm)
            y = torch.full_like(by, float("nan")); ya = by.clone()
            dx = torch.full_like(bx, float("nan")); dxa = bx.clone()
            for o, b in ((y, 0), (ya, 1)):
                assert lib.accudnn_conv_fwd(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), o.data_ptr(), b, None) == 0
            for o, b in ((dx, 0), (dxa, 1)):
                assert lib.accudnn_conv_dgrad(ctypes.byref(d), dy.data_ptr(), wt.data_ptr(), o.data_ptr(), b, None) == 0
            torch.cuda.synchronize()
            outs[name] = (y, ya, dx, dxa)
        lib.accudnn_conv_force_cfg(0, 0, 0)
        msg = []
        for nm, u, v in zip(("y", "ya", "dx", "dxa"), outs["ws"], outs["kc"]):
            nd = (u != v).sum().item()
            msg.append(f"{nm}:{nd}" + (f"(max {((u - v).abs().max().item()):.2e}, nan {torch.isnan(v).sum().item()})" if nd else ""))
        print(shape, bn, " ".join(msg), flush=True)
