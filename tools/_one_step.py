import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1901_06773_b200 import trainer
trainer._lib().accudnn_set_conv_math(1)
_, desc = trainer.export_network("resnet20", 32, 12)
params = trainer.init_params(desc, seed=1)
ex = trainer.Executor("resnet20", 32, 12, k=4)
ex.set_params(params)
g = np.random.default_rng(0)
x = g.standard_normal((4, 3, 32, 32)).astype(np.float32)
y = g.integers(0, 12, size=4).astype(np.int32)
print(ex.step(x, y, lr=0.0, update=False))
