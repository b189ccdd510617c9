"""BN forward/backward kernels at ResNet-152 k=27 shapes: device time per
launch (CUDA graph of 20 launches, so host launch cost is excluded) and
achieved HBM-equivalent bandwidth (fwd: 2 passes over x + write y = 3S;
bwd: x, dy twice + write dx = 5S; fused residual tail relu(bn(x)+skip):
fwd 4S (x twice, skip, y), bwd 7S (x, dy twice, skip, dx, dskip)).
Usage: bn_bench.py [k]"""
import ctypes
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import _native  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 27
lib = _native.cuda_lib()
dev = torch.device("cuda:0")
P = ctypes.c_void_p
shapes = [(1, 32), (1, 512), (112 * 112, 64), (56 * 56, 64), (56 * 56, 256), (28 * 28, 128), (28 * 28, 512),
          (14 * 14, 256), (14 * 14, 1024), (7 * 7, 512), (7 * 7, 2048)]
ws = torch.zeros(lib.accudnn_bn_workspace_bytes(2048) // 4 + 1, device=dev)
s = torch.cuda.Stream()
for hw, C in shapes:
    M = k * hw if hw > 1 else 16
    x = torch.randn(M, C, device=dev)
    dy = torch.randn(M, C, device=dev)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    g, b = torch.ones(C, device=dev), torch.zeros(C, device=dev)
    mean, inv = torch.empty(C, device=dev), torch.empty(C, device=dev)
    skip = torch.randn(M, C, device=dev)
    dsk = torch.empty_like(x)
    res = []
    for mode in (0, 1, 2, 3):
        def run():
            if mode == 2:
                lib.accudnn_bn_add_relu_fwd(P(x.data_ptr()), P(skip.data_ptr()), M, C, P(g.data_ptr()),
                                            P(b.data_ptr()), 1e-5, P(y.data_ptr()), P(mean.data_ptr()),
                                            P(inv.data_ptr()), None, None, 0.1, P(ws.data_ptr()),
                                            P(s.cuda_stream))
            elif mode == 3:
                lib.accudnn_bn_add_relu_bwd(P(x.data_ptr()), P(skip.data_ptr()), P(dy.data_ptr()), M, C,
                                            P(g.data_ptr()), P(b.data_ptr()), P(mean.data_ptr()),
                                            P(inv.data_ptr()), P(dx.data_ptr()), 0, P(dsk.data_ptr()), 0,
                                            None, None, P(ws.data_ptr()), P(s.cuda_stream))
            elif mode == 0:
                lib.accudnn_bn_fwd(P(x.data_ptr()), M, C, P(g.data_ptr()), P(b.data_ptr()), 1e-5, 1,
                                   P(y.data_ptr()), P(mean.data_ptr()), P(inv.data_ptr()), None, None,
                                   0.1, P(ws.data_ptr()), P(s.cuda_stream))
            else:
                lib.accudnn_bn_bwd(P(x.data_ptr()), P(dy.data_ptr()), M, C, P(g.data_ptr()),
                                   P(b.data_ptr()), P(mean.data_ptr()), P(inv.data_ptr()), 1,
                                   P(dx.data_ptr()), 0, None, None, P(ws.data_ptr()), P(s.cuda_stream))
        with torch.cuda.stream(s):
            run()
            torch.cuda.synchronize()
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph, stream=s):
                for _ in range(20):
                    run()
            gph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            gph.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        S = M * C * 4
        res.append((us, (3, 5, 4, 7)[mode] * S / us / 1e3))
    print(f"M={M:7d} C={C:5d} S={M*C*4/1e6:6.1f}MB  fwd {res[0][0]:7.1f} us ({res[0][1]:6.0f} GB/s)  "
          f"bwd {res[1][0]:7.1f} us ({res[1][1]:6.0f} GB/s)  tail fwd {res[2][0]:7.1f} us "
          f"({res[2][1]:6.0f} GB/s)  tail bwd {res[3][0]:7.1f} us ({res[3][1]:6.0f} GB/s)", flush=True)

# floor of a trivial kernel in the same graph setting
x = torch.randn(1024, device=dev)
y = torch.empty_like(x)
with torch.cuda.stream(s):
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=s):
        for _ in range(20):
            lib.accudnn_relu_fwd(P(x.data_ptr()), P(y.data_ptr()), 1024, P(s.cuda_stream))
    gph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    gph.replay()
    e1.record(s)
torch.cuda.synchronize()
print("relu_fwd(1024 floats) in a graph: %.2f us/launch" % (e0.elapsed_time(e1) / 20 * 1e3))
