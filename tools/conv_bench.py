"""Times the tcgen05 conv kernels on representative ResNet-152 shapes (k=24)."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import _native  # noqa: E402

SHAPES = {
    "s1_conv2_3x3": (24, 64, 56, 56, 64, 3, 1, 1),
    "s1_conv3_1x1": (24, 64, 56, 56, 256, 1, 1, 0),
    "s3_conv1_1x1": (24, 1024, 14, 14, 256, 1, 1, 0),
    "s3_conv2_3x3": (24, 256, 14, 14, 256, 3, 1, 1),
    "s3_conv3_1x1": (24, 256, 14, 14, 1024, 1, 1, 0),
    "s4_conv2_3x3": (24, 512, 7, 7, 512, 3, 1, 1),
    "stem_7x7": (24, 4, 224, 224, 64, 7, 2, 3),
}


def main():
    lib = _native.cuda_lib()
    dev = torch.device("cuda:0")
    out = {}
    for name, (n, c, h, w, k, r, st, pad) in SHAPES.items():
        p = (h + 2 * pad - r) // st + 1
        q = (w + 2 * pad - r) // st + 1
        d = _native.ConvDesc(n, h, w, c, k, r, r, st, pad, p, q)
        x = torch.randn(n, h, w, c, device=dev)
        wt = torch.randn(k, r, r, c, device=dev) * 0.01
        y = torch.empty(n, p, q, k, device=dev)
        dy = torch.randn(n, p, q, k, device=dev)
        dx = torch.empty_like(x)
        dw = torch.empty_like(wt)
        flops = 2.0 * n * p * q * k * c * r * r
        res = {}
        for mode, fn in (("fwd", lambda: lib.accudnn_conv_fwd(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), y.data_ptr(), 0, None)),
                         ("dgrad", lambda: lib.accudnn_conv_dgrad(ctypes.byref(d), dy.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, None)),
                         ("wgrad", lambda: lib.accudnn_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, 0, None))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            iters = 20
            a.record()
            for _ in range(iters):
                fn()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / iters
            res[mode] = {"ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1)}
        out[name] = res
        print(name, json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
