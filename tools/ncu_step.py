"""One eager ResNet training step for ncu (launch list / full capture), after
warm-up steps, bracketed by cudaProfilerStart/Stop.
Usage: python tools/ncu_step.py [arch] [k] [warmup]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1901_06773_b200 import trainer  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet152"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 27
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 1
image, classes = (224, 1000) if arch in ("resnet50", "resnet101", "resnet152") else (32, 12)
_, desc = trainer.export_network(arch, image, classes)
_tune = os.path.join(ROOT, "profiles", "b200", "conv_tune.txt")
if os.path.exists(_tune):
    from paper_1901_06773_b200 import _native
    _native.conv_tune_import(open(_tune).read())
ex = trainer.Executor(arch, image, classes, k=k)
ex.set_params(trainer.init_params(desc, 0))
g = np.random.default_rng(0)
x = torch.from_numpy(g.standard_normal((k, 3, image, image)).astype(np.float32)).cuda()
y = torch.from_numpy(g.integers(0, classes, size=k).astype(np.int32)).cuda()
# warm-up steps (the first one autotunes the conv kernels), then exactly one
# profiled step between cudaProfilerStart/Stop (run ncu with
# --profile-from-start off)
for _ in range(max(1, warm)):
    ex.step(x, y, lr=0.01)
torch.cuda.synchronize()
torch.cuda.profiler.start()
out = ex.step(x, y, lr=0.01)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("step done", out)
