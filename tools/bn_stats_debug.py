"""Per-BN saved batch statistics of one executor step vs fp64 statistics of
the oracle's forward on the same weights/inputs (debug tool)."""
import os, sys
import numpy as np, torch, torch.nn.functional as F
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1901_06773_b200 import trainer
import resnet_torch

arch, image, classes, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
if os.environ.get("ACCUDNN_PRECISE"): trainer._lib().accudnn_set_conv_math(1)
_, desc = trainer.export_network(arch, image, classes)
params = trainer.init_params(desc, seed=1)
ex = trainer.Executor(arch, image, classes, k=k)
ex.set_params(params)
g = np.random.default_rng(0)
x = g.standard_normal((k, 3, image, image)).astype(np.float32)
y = g.integers(0, classes, size=k).astype(np.int32)
ex.step(x, y, lr=0.0, update=False)
st = ex.get_stats()
# oracle forward in fp64, capturing BN inputs
cap = {}
orig_bn = F.batch_norm
def bn_hook(inp, *a, **kw):
    cap[len(cap)] = inp.detach().clone()
    return orig_bn(inp, *a, **kw)
resnet_torch.F.batch_norm = bn_hook
resnet_torch.TorchResNet(desc, torch.float64).step(params, torch.zeros(desc["n_stats"]), None, x, y, lr=0.0, update=False)
i = 0
for op in desc["ops"]:
    if op["kind"] not in ("bn", "bn_relu", "bn_add_relu"): continue
    c, so = op["channels"], op["stat_off"]
    t = cap[i]; i += 1
    m = t.mean(dim=(0, 2, 3)).numpy(); v = t.var(dim=(0, 2, 3), unbiased=False).numpy()
    mean_d, inv_d = st[so:so + c], st[so + c:so + 2 * c]
    inv_ref = 1 / np.sqrt(v + 1e-5)
    em = np.abs(mean_d - m).max() / (np.sqrt(v).max() + 1e-30)
    ei = np.abs(inv_d - inv_ref).max() / np.abs(inv_ref).max()
    flag = " <==" if max(em, ei) > 1e-5 else ""
    print("%-26s M=%7d C=%4d  mean err/std %.2e  invstd rel %.2e  |mean|/std %.2f%s" % (
        op["name"], t.numel() // c, c, em, ei, np.abs(m).max() / np.sqrt(v).min(), flag))
