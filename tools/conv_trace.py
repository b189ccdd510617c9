"""Per-CTA pipeline timeline of one TMA conv launch (debug stamps from
accudnn_conv_trace): producer issue / MMA start per k-block, epilogue per unit.
Usage: conv_trace.py mode n c h w k r stride pad [bn splits]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import _native  # noqa: E402

mode = sys.argv[1]
n, c, h, w, k, r, st, pad = (int(v) for v in sys.argv[2:10])
lib = _native.cuda_lib()
import os  # noqa: E402
_tune = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "b200",
                     "conv_tune.txt")
if os.path.exists(_tune):
    _native.conv_tune_import(open(_tune).read())
if os.environ.get("ACCUDNN_FORCE"):
    lib.accudnn_conv_force_cfg(*[int(v) for v in os.environ["ACCUDNN_FORCE"].split(",")])
p = (h + 2 * pad - r) // st + 1
q = (w + 2 * pad - r) // st + 1
d = _native.ConvDesc(n, h, w, c, k, r, r, st, pad, p, q)
dev = torch.device("cuda:0")
x = torch.randn(n, h, w, c, device=dev)
wt = torch.randn(k, r, r, c, device=dev) * 0.01
y = torch.empty(n, p, q, k, device=dev)
dy = torch.randn(n, p, q, k, device=dev)
dx = torch.empty_like(x)
dw = torch.empty_like(wt)
fn = {"fwd": lambda: lib.accudnn_conv_fwd(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), y.data_ptr(), 0, None),
      "dgrad": lambda: lib.accudnn_conv_dgrad(ctypes.byref(d), dy.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, None),
      "wgrad": lambda: lib.accudnn_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, 0, None)}[mode]
for _ in range(3):
    fn()
torch.cuda.synchronize()
buf = torch.zeros(148 * 1024, dtype=torch.int64, device=dev)
lib.accudnn_conv_trace(ctypes.c_void_p(buf.data_ptr()))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
fn()
b.record()
torch.cuda.synchronize()
lib.accudnn_conv_trace(None)
print("kernel ms %.4f  (%.1f TFLOP/s)" % (a.elapsed_time(b), 2 * n * p * q * k * c * r * r / a.elapsed_time(b) / 1e9))
t = buf.view(148, 1024).cpu().numpy()
g0 = t[:, 768][t[:, 768] > 0].min()
ent, pro, ex = t[:, 768] - g0, t[:, 769] - g0, t[:, 770] - g0
ok = t[:, 768] > 0
print("CTA entry ns: min %d max %d | prologue done ns: min %d max %d | exit ns: min %d max %d" % (
    ent[ok].min(), ent[ok].max(), pro[ok].min(), pro[ok].max(), ex[ok].min(), ex[ok].max()))
red = t[:, 771][t[:, 771] > 0]
if len(red):
    print("split-K reduce kernel block starts ns: min %d max %d" % (red.min() - g0, red.max() - g0))
for cta in (0, 1, 147):
    row = t[cta]
    prod = row[0:256]
    mma = row[256:512]
    epi = row[512:768]
    nk = int((prod > 0).sum())
    if nk == 0:
        continue
    t0 = prod[0]
    print(f"CTA {cta}: {nk} k-blocks")
    print("  producer issue (cyc from first):", (prod[:min(nk, 24)] - t0).tolist())
    print("  mma start      (cyc from first):", (mma[:min(nk, 24)] - t0).tolist())
    ne = int((epi[0::2] > 0).sum())
    print("  epilogue start/end per unit:", [(int(epi[2 * j] - t0), int(epi[2 * j + 1] - t0)) for j in range(ne)][:12])
    if nk > 1:
        dm = np.diff(mma[:nk])
        print("  mma k-block interval cycles: median %d  mean %.0f" % (np.median(dm), dm.mean()))
        lat = mma[:nk] - prod[:nk]
        print("  issue->data latency cycles: median %d  min %d max %d" % (np.median(lat), lat.min(), lat.max()))
