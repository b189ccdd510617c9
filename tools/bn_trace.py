"""Phase timeline of one BN launch (debug stamps, accudnn_bn_trace).
Usage: bn_trace.py M C relu(0/1) [bwd]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import _native  # noqa: E402

M, C, relu = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
bwd = len(sys.argv) > 4
lib = _native.cuda_lib()
dev = torch.device("cuda:0")
P = ctypes.c_void_p
x = torch.randn(M, C, device=dev)
dy = torch.randn(M, C, device=dev)
y = torch.empty_like(x)
g, b = torch.ones(C, device=dev), torch.zeros(C, device=dev)
mean, inv = torch.empty(C, device=dev), torch.empty(C, device=dev)
ws = torch.zeros(lib.accudnn_bn_workspace_bytes(C) // 4 + 1, device=dev)
def run():
    lib.accudnn_bn_fwd(P(x.data_ptr()), M, C, P(g.data_ptr()), P(b.data_ptr()), 1e-5, relu, P(y.data_ptr()),
                       P(mean.data_ptr()), P(inv.data_ptr()), None, None, 0.1, P(ws.data_ptr()), None)
    if bwd:
        lib.accudnn_bn_bwd(P(x.data_ptr()), P(dy.data_ptr()), M, C, P(g.data_ptr()), P(b.data_ptr()),
                           P(mean.data_ptr()), P(inv.data_ptr()), relu, P(y.data_ptr()), 0, None, None,
                           P(ws.data_ptr()), None)
for _ in range(3):
    run()
torch.cuda.synchronize()
buf = torch.zeros(2048 * 8, dtype=torch.int64, device=dev)
lib.accudnn_bn_trace(P(buf.data_ptr()))
run()
torch.cuda.synchronize()
lib.accudnn_bn_trace(None)
t = buf.view(-1, 8).cpu().numpy()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["entry", "phase1 loop", "partial published", "phase2 done", "phase3 done", "barrier passed"]
print(f"M={M} C={C} {'bwd' if bwd else 'fwd'} blocks={len(t)}")
for i, n in enumerate(names):
    col = t[:, i] - t0
    col = col[t[:, i] > 0]
    if len(col):
        print(f"  {n:18s} ns: min {col.min():7d} median {int(np.median(col)):7d} max {col.max():7d}")
