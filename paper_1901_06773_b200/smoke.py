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
    # the convolutions run on TF32 tensor cores: the device step must be as
    # close to the float64 ground truth as an fp32 step whose convolutions see
    # TF32-truncated operands (within 3x, or 2e-3) -- the tolerance of
    # tests/test_train_step_gpu.py::test_step_tf32_mode_matches_tf32_oracle
    def oracle(dtype, conv_math):
        loss, g, _, _ = TorchResNet(desc, dtype, conv_math).step(
            params, torch.zeros(desc["n_stats"]), None, x, y, lr=0.0, update=False)
        return loss, np.asarray(g, np.float64)
    l64, g64 = oracle(torch.float64, "exact")
    lt, gt = oracle(torch.float32, "tf32")
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    e_l, e_lt = abs(out["loss"] - l64) / abs(l64), abs(lt - l64) / abs(l64)
    e_g, e_gt = rel(grads, g64), rel(gt, g64)
    print(f"smoke: loss {out['loss']:.6f} (fp64 oracle {l64:.6f}); loss err {e_l:.2e} "
          f"(tf32 oracle {e_lt:.2e}); grad rel-L2 err {e_g:.2e} (tf32 oracle {e_gt:.2e}); "
          f"swapped {out['swapped_bytes']} B")
    assert e_l <= max(3 * e_lt, 2e-3) and e_g <= max(3 * e_gt, 2e-3)


if __name__ == "__main__":
    run()
