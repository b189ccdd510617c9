"""Runs one conv shape a few times (for ncu captures of a single launch).
Usage: conv_one.py n h w c k r stride pad [fwd|dgrad|wgrad] [bn,splits,cm]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import _native  # noqa: E402

n, h, w, c, kk, r, st, pad = (int(v) for v in sys.argv[1:9])
mode = sys.argv[9] if len(sys.argv) > 9 else "fwd"
lib = _native.cuda_lib()
tune = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "b200",
                    "conv_tune.txt")
if os.path.exists(tune):
    _native.conv_tune_import(open(tune).read())
if len(sys.argv) > 10:
    lib.accudnn_conv_force_cfg(*[int(v) for v in sys.argv[10].split(",")])
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
fn = {"fwd": lambda: lib.accudnn_conv_fwd(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), y.data_ptr(), 0, None),
      "dgrad": lambda: lib.accudnn_conv_dgrad(ctypes.byref(d), dy.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, None),
      "wgrad": lambda: lib.accudnn_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, 0, None)}[mode]
for _ in range(5):
    fn()
torch.cuda.synchronize()
