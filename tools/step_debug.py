"""Per-parameter-tensor gradient error of the B200 step vs the torch oracle,
with and without TF32 operand emulation in the oracle's convolutions."""
import os, sys
import numpy as np, torch, torch.nn.functional as F
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1901_06773_b200 import trainer
import resnet_torch
from resnet_torch import TorchResNet

def tf32(t, mode):
    i = t.contiguous().view(torch.int32)
    if mode == "trunc":
        i = i & ~0x1FFF
    else:
        i = (i + 0x1000) & ~0x1FFF
    return i.view(torch.float32)

arch, image, classes, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
_, desc = trainer.export_network(arch, image, classes)
params = trainer.init_params(desc, seed=1)
if os.environ.get("ACCUDNN_PRECISE"): trainer._lib().accudnn_set_conv_math(1)
ex = trainer.Executor(arch, image, classes, k=k)
ex.set_params(params)
g = np.random.default_rng(0)
x = g.standard_normal((k, 3, image, image)).astype(np.float32)
y = g.integers(0, classes, size=k).astype(np.int32)
out = ex.step(x, y, lr=0.0, update=False)
gd = ex.get_grads()
res = {}
orig = F.conv2d
class TF32Conv(torch.autograd.Function):
    mode = "trunc"
    @staticmethod
    def forward(ctx, x, w, stride, padding):
        ctx.save_for_backward(x, w); ctx.stride, ctx.padding = stride, padding
        m = TF32Conv.mode
        return orig(tf32(x, m), tf32(w, m), stride=stride, padding=padding)
    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors; m = TF32Conv.mode
        gx = torch.nn.grad.conv2d_input(x.shape, tf32(w, m), tf32(gy, m), stride=ctx.stride, padding=ctx.padding)
        gw = torch.nn.grad.conv2d_weight(tf32(x, m), w.shape, tf32(gy, m), stride=ctx.stride, padding=ctx.padding)
        return gx, gw, None, None
for mode in ["fp32", "trunc", "round"]:
    if mode != "fp32":
        TF32Conv.mode = mode
        resnet_torch.F.conv2d = lambda inp, w, stride=1, padding=0: TF32Conv.apply(inp, w, stride, padding)
    else:
        resnet_torch.F.conv2d = orig
    loss, gr, _, _ = TorchResNet(desc).step(params, torch.zeros(desc["n_stats"]), None, x, y, lr=0.0, update=False)
    res[mode] = (loss, gr)
    print(mode, "loss dev %.7f ref %.7f" % (out["loss"], loss), "total rel %.3e" % (np.linalg.norm(gd - gr) / np.linalg.norm(gr)))
resnet_torch.F.conv2d = orig
gr = res["fp32"][1]; gt = res["trunc"][1]; gq = res["round"][1]
print("trunc vs fp32 total %.3e ; round vs fp32 total %.3e; dev vs round %.3e" % (np.linalg.norm(gt-gr)/np.linalg.norm(gr), np.linalg.norm(gq-gr)/np.linalg.norm(gr), np.linalg.norm(gd-gq)/np.linalg.norm(gq)))
for op in desc["ops"]:
    for key, cnt in (("w_off", None), ("g_off", "channels")):
        if key not in op: continue
        off = op[key]
        n = op[cnt] if cnt else (op["cout"] * op["cin"] * op.get("r", 1) ** 2)
        a, b, c = gd[off:off + n], gr[off:off + n], gt[off:off + n]
        nb = np.linalg.norm(b) + 1e-30
        print("%-28s %-8s dev/fp32 %.2e  trunc/fp32 %.2e  dev/trunc %.2e" % (op["name"], key, np.linalg.norm(a - b) / nb, np.linalg.norm(c - b) / nb, np.linalg.norm(a - c) / nb))
