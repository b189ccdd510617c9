"""One tiny training step on cuda:0 checked against the CPU fp32 oracle.
Called by __graft_entry__.smoke(); the oracle is test infrastructure and is
only used here as the checker."""
import os
import sys

import numpy as np


def run():
    import torch
    assert torch.cuda.is_available(), "smoke needs a CUDA device"
    from . import trainer
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    from resnet_torch import TorchResNet

    arch, image, classes, k = "resnet20", 32, 12, 4
    _, desc = trainer.export_network(arch, image, classes)
    params = trainer.init_params(desc, seed=0)
    ex = trainer.Executor(arch, image, classes, k=k, mode="naive")  # exercises the copy streams
    ex.set_params(params)
    g = np.random.default_rng(0)
    x = g.standard_normal((k, 3, image, image)).astype(np.float32)
    y = g.integers(0, classes, size=k).astype(np.int32)
    out = ex.step(x, y, lr=0.0, update=False)
    grads = ex.get_grads()
    loss, g_ref, _, _ = TorchResNet(desc).step(params, torch.zeros(desc["n_stats"]), None, x, y,
                                               lr=0.0, update=False)
    rel_loss = abs(out["loss"] - loss) / abs(loss)
    rel_g = float(np.linalg.norm(grads - g_ref) / np.linalg.norm(g_ref))
    print(f"smoke: loss {out['loss']:.6f} (oracle {loss:.6f}, rel {rel_loss:.2e}), "
          f"grad rel-L2 {rel_g:.2e}, swapped {out['swapped_bytes']} B")
    assert rel_loss < 2e-3 and rel_g < 2e-2


if __name__ == "__main__":
    run()
