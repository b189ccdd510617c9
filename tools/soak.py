"""Soak test of the captured training step at the headline configuration:
one fixed synthetic batch, many SGD steps through the CUDA graph (weight-
gradient stream, pipelined host input); the loss must stay finite and fall
(the network memorises the batch).  Usage: soak.py [arch] [k] [steps] [lr]"""
import math
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import trainer  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet152"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 42
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
lr = float(sys.argv[4]) if len(sys.argv) > 4 else 0.02
image, classes = (224, 1000) if arch in ("resnet50", "resnet101", "resnet152") else (32, 12)
_, desc = trainer.export_network(arch, image, classes)
ex = trainer.Executor(arch, image, classes, k=k)
ex.set_params(trainer.init_params(desc, 0))
ex.set_graph(True)
g = np.random.default_rng(0)
x = g.standard_normal((k, 3, image, image)).astype(np.float32)
y = g.integers(0, classes, size=k).astype(np.int32)
losses = []
out = ex.step_pipelined(x, y, lr=lr, next_images=x)
losses.append(out["loss"])
for i in range(1, steps):
    out = ex.step_pipelined(None, y, lr=lr, next_images=x if i + 1 < steps else None)
    losses.append(out["loss"])
    if i % 20 == 0 or i == steps - 1:
        print(f"step {i:4d} loss {out['loss']:.5f} iter {out['iter_ms']:.2f} ms", flush=True)
assert all(math.isfinite(v) for v in losses), "non-finite loss"
print(f"first {losses[0]:.4f} -> last {losses[-1]:.4f} ({'fell' if losses[-1] < 0.5 * losses[0] else 'DID NOT FALL'})")
