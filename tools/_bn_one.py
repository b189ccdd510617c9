import ctypes, sys
import torch
sys.path.insert(0, '.')
from paper_1901_06773_b200 import _native
lib = _native.cuda_lib(); dev = torch.device("cuda:0"); P = ctypes.c_void_p
M, C = int(sys.argv[1]), int(sys.argv[2])
ws = torch.zeros(lib.accudnn_bn_workspace_bytes(2048) // 4 + 1, device=dev)
x = torch.randn(M, C, device=dev); y = torch.empty_like(x)
g, b = torch.ones(C, device=dev), torch.zeros(C, device=dev)
mean, inv = torch.empty(C, device=dev), torch.empty(C, device=dev)
for _ in range(3):
    lib.accudnn_bn_fwd(P(x.data_ptr()), M, C, P(g.data_ptr()), P(b.data_ptr()), 1e-5, 1, P(y.data_ptr()), P(mean.data_ptr()), P(inv.data_ptr()), None, None, 0.1, P(ws.data_ptr()), None)
torch.cuda.synchronize()
