"""Per-tensor gradient error of the 3xTF32 (fp32-mode) device step against
the fp64 oracle, next to PyTorch fp32's own error: which parameter tensors
deviate.  python tools/fp32_debug.py [arch image classes k]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1901_06773_b200 import _native, trainer  # noqa: E402
from resnet_torch import TorchResNet  # noqa: E402

arch, image, classes, k = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])) \
    if len(sys.argv) > 4 else ("resnet50", 64, 8, 8)
mode = int(os.environ.get("CONV_MATH", "1"))
_native.cuda_lib().accudnn_set_conv_math(mode)
_, desc = trainer.export_network(arch, image, classes)
params = trainer.init_params(desc, seed=1)
ex = trainer.Executor(arch, image, classes, k=k)
ex.set_params(params)
g = np.random.default_rng(0)
x = g.standard_normal((k, 3, image, image)).astype(np.float32)
y = g.integers(0, classes, size=k).astype(np.int32)
out = ex.step(x, y, lr=0.0, update=False)
gd = ex.get_grads().astype(np.float64)
res = {}
for dt in (torch.float64, torch.float32):
    loss, gr, _, _ = TorchResNet(desc, dt, "exact").step(params, torch.zeros(desc["n_stats"]), None, x, y,
                                                        lr=0.0, update=False)
    res[str(dt)] = (loss, np.asarray(gr, np.float64))
l64, g64 = res["torch.float64"]
l32, g32 = res["torch.float32"]
print("loss dev %.9g fp32 %.9g fp64 %.9g" % (out["loss"], l32, l64))


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


print("total rel: dev %.3e fp32 %.3e" % (rel(gd, g64), rel(g32, g64)))
rows = []
for i, op in enumerate(desc["ops"]):
    for key, n in (("w_off", op.get("cout", 0) * op.get("cin", 0) * op.get("r", 1) ** 2),
                   ("g_off", op.get("channels", 0)), ("beta_off", op.get("channels", 0)),
                   ("b_off", op.get("cout", 0))):
        off = op.get(key, -1)
        if off is None or off < 0 or not n:
            continue
        a, b, c = gd[off:off + n], g64[off:off + n], g32[off:off + n]
        rows.append((rel(a, b), rel(c, b), i, op["kind"], key, n, float(np.linalg.norm(b))))
rows.sort(reverse=True)
for r in rows[:25]:
    print("op %3d %-12s %-8s n=%-8d |g|=%.3e dev %.3e fp32 %.3e" % (r[2], r[3], r[4], r[5], r[6], r[0], r[1]))
# first op (in forward order) whose dev error exceeds 10x fp32's
for r in sorted(rows, key=lambda r: r[2]):
    if r[0] > 10 * max(r[1], 1e-7):
        print("first large deviation (forward order): op", r[2], r[3], r[4], "%.3e vs %.3e" % (r[0], r[1]))
        break
