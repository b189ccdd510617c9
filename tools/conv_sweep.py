"""Times every forced (tile width BN, split-K, CTA-pair multicast) config of
the persistent conv kernel on one shape (CUDA graph of 20 calls), next to
the tuner's choice and cuDNN TF32.
Usage: conv_sweep.py n h w c k r stride pad [fwd|dgrad|wgrad]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import _native  # noqa: E402
from conv_bench import timeit  # noqa: E402

n, h, w, c, kk, r, st, pad = (int(v) for v in sys.argv[1:9])
mode = sys.argv[9] if len(sys.argv) > 9 else "fwd"
lib = _native.cuda_lib()
tune = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "b200",
                    "conv_tune.txt")
if os.path.exists(tune):
    _native.conv_tune_import(open(tune).read())
dev = torch.device("cuda:0")
p = (h + 2 * pad - r) // st + 1
q = (w + 2 * pad - r) // st + 1
d = _native.ConvDesc(n, h, w, c, kk, r, r, st, pad, p, q)
x = torch.randn(n, h, w, c, device=dev)
wt = torch.randn(kk, r, r, c, device=dev) * 0.01
y = torch.empty(n, p, q, kk, device=dev)
dy = torch.randn(n, p, q, kk, device=dev)
dx = torch.empty_like(x)
dw = torch.empty_like(wt)
flops = 2.0 * n * p * q * kk * c * r * r
S = lambda s: ctypes.c_void_p(s.cuda_stream) if s is not None else None  # noqa: E731
fn = {"fwd": lambda s=None: lib.accudnn_conv_fwd(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), y.data_ptr(), 0, S(s)),
      "dgrad": lambda s=None: lib.accudnn_conv_dgrad(ctypes.byref(d), dy.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, S(s)),
      "wgrad": lambda s=None: lib.accudnn_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, 0, S(s))}[mode]
ms = timeit(fn, graph=True)
print(f"tuned: {ms*1e3:.1f} us {flops/ms/1e9:.0f} TF/s", flush=True)
for bn in (64, 128, 256):
    for cm in (1, 2, 4, 5, 6, 7, 8):
        for sp in ((1, 2, 3, 4, 6, 8) if cm < 5 else (2,)):
            lib.accudnn_conv_force_cfg(bn, sp, cm)
            try:
                ms = timeit(fn, graph=True)
            except Exception as e:  # noqa: BLE001
                print(bn, sp, cm, "error", e)
                continue
            print(f"bn={bn:3d} splits={sp} cm={cm}: {ms*1e3:7.1f} us {flops/ms/1e9:5.0f} TF/s", flush=True)
lib.accudnn_conv_force_cfg(0, 0, 0)
