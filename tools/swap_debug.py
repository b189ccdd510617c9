"""Resident vs naive/dynamic executor on the same inputs: per-parameter gradient
differences (locates a swap-path ordering bug).  Usage: swap_debug.py arch image classes k"""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1901_06773_b200 import trainer

arch, image, classes, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
_, desc = trainer.export_network(arch, image, classes)
params = trainer.init_params(desc, seed=1)
g = np.random.default_rng(0)
x = g.standard_normal((k, 3, image, image)).astype(np.float32)
y = g.integers(0, classes, size=k).astype(np.int32)
res = {}
for mode in ["resident", "resident2", "naive", "naive2"]:
    ex = trainer.Executor(arch, image, classes, k=k, mode=mode.rstrip("2"))
    ex.set_params(params)
    out = ex.step(x, y, lr=0.0, update=False, profile=True)
    res[mode] = (out["loss"], ex.get_grads())
    print(mode, out["loss"], out["swapped_bytes"], flush=True)
    ex.close()
gr = res["resident"][1]
for m in ["resident2", "naive", "naive2"]:
    gd = res[m][1]
    print(m, "loss", res[m][0], "rel", np.linalg.norm(gd - gr) / np.linalg.norm(gr))
    shown = 0
    for op in desc["ops"]:
        for key, cnt in (("w_off", None), ("g_off", "channels")):
            if key not in op: continue
            off = op[key]
            n = op[cnt] if cnt else (op["cout"] * op["cin"] * op.get("r", 1) ** 2)
            a, b = gd[off:off + n], gr[off:off + n]
            e = np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30)
            if e > 1e-5 and shown < 12:
                print("   %3d %-28s %-6s %.2e" % (op["id"], op["name"], key, e)); shown += 1
