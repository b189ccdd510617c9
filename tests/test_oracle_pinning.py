"""Pins the CPU oracle (oracle/resnet_torch.py) -- the checker of the layer
math -- to canonical implementations:
  * the ResNet-50 op graph + flat-parameter mapping reproduce
    torchvision.models.resnet50 (train-mode loss and every gradient) when the
    torchvision weights are copied in;
  * the oracle's fp32 SGD update equals torch.optim.SGD(momentum, wd).
"""
import os
import sys

import numpy as np
import pytest
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_1901_06773_b200 import trainer  # noqa: E402
from resnet_torch import TorchResNet  # noqa: E402

tv = pytest.importorskip("torchvision")


def flat_from_torchvision(model, desc):
    sd = {k: v.detach().double() for k, v in model.state_dict().items()}
    p = np.zeros(desc["n_params"], dtype=np.float64)
    mapping = {}
    for op in desc["ops"]:
        name = op["name"]
        if name.startswith("stem."):
            tvname = {"stem.conv": "conv1", "stem.bn": "bn1"}.get(name)
        elif name == "fc":
            tvname = "fc"
        else:
            tvname = name.replace("downsample.conv", "downsample.0").replace("downsample.bn",
                                                                             "downsample.1")
        mapping[op["id"]] = tvname
        if op["kind"] == "conv":
            w = sd[tvname + ".weight"].permute(0, 2, 3, 1).numpy()  # [cout][r][s][cin]
            if op["in0"] == -2:
                w = np.concatenate([w, np.zeros(w.shape[:3] + (1,))], axis=3)
            p[op["w_off"]:op["w_off"] + w.size] = w.ravel()
        elif op["kind"] == "fc":
            w = sd["fc.weight"].numpy()
            p[op["w_off"]:op["w_off"] + w.size] = w.ravel()
            p[op["b_off"]:op["b_off"] + op["cout"]] = sd["fc.bias"].numpy()
        elif op["kind"] in ("bn", "bn_relu", "bn_add_relu"):
            c = op["channels"]
            p[op["g_off"]:op["g_off"] + c] = sd[tvname + ".weight"].numpy()
            p[op["beta_off"]:op["beta_off"] + c] = sd[tvname + ".bias"].numpy()
    return p, mapping


@pytest.mark.parametrize("arch", ["resnet50", "resnet152"])
def test_oracle_matches_torchvision_resnet(arch):
    """the exported op graph (fused residual tails included) + flat parameter
    layout computes torchvision's ResNet-50 / ResNet-152 exactly (fp64)"""
    torch.manual_seed(0)
    model = getattr(tv.models, arch)(num_classes=8).double().train()
    _, desc = trainer.export_network(arch, 64, 8)
    params, mapping = flat_from_torchvision(model, desc)
    g = np.random.default_rng(0)
    x = g.standard_normal((2, 3, 64, 64))
    y = g.integers(0, 8, size=2).astype(np.int32)

    out = model(torch.from_numpy(x))
    loss_tv = F.cross_entropy(out, torch.from_numpy(y).long())
    loss_tv.backward()

    loss, grads, _, _ = TorchResNet(desc, torch.float64).step(
        params, torch.zeros(desc["n_stats"]), None, x, y, lr=0.0, update=False)
    assert abs(loss - loss_tv.item()) < 1e-10
    for op in desc["ops"]:
        if op["kind"] != "conv":
            continue
        gw = model.get_submodule(mapping[op["id"]]).weight.grad.permute(0, 2, 3, 1).numpy()
        if op["in0"] == -2:
            gw = np.concatenate([gw, np.zeros(gw.shape[:3] + (1,))], axis=3)
        mine = grads[op["w_off"]:op["w_off"] + gw.size]
        rel = np.linalg.norm(mine - gw.ravel()) / np.linalg.norm(gw)
        assert rel < 1e-10, (op["name"], rel)


def test_oracle_sgd_matches_torch_optim():
    _, desc = trainer.export_network("resnet20", 32, 12)
    p0 = trainer.init_params(desc, seed=4)
    g = np.random.default_rng(1)
    oracle = TorchResNet(desc)
    w = torch.nn.Parameter(torch.from_numpy(p0.copy()))
    opt = torch.optim.SGD([w], lr=0.05, momentum=0.9, weight_decay=1e-4)
    p, buf = p0.copy(), None
    for it in range(3):
        x = g.standard_normal((2, 3, 32, 32)).astype(np.float32)
        y = g.integers(0, 12, size=2).astype(np.int32)
        _, grad, p_next, buf = oracle.step(p, torch.zeros(desc["n_stats"]), buf, x, y, lr=0.05,
                                           first=(it == 0))
        w.grad = torch.from_numpy(grad.astype(np.float32))
        opt.step()
        p = p_next
        assert np.allclose(p, w.detach().numpy(), rtol=1e-6, atol=1e-7)


def test_oracle_init_equals_product_init():
    """the CPU reference arm's parameter init (oracle) draws the same values
    as the product's"""
    import resnet_torch
    for arch, image, classes in (("resnet20", 32, 12), ("resnet152", 224, 1000)):
        _, desc = trainer.export_network(arch, image, classes)
        assert np.array_equal(resnet_torch.init_params(desc, 3), trainer.init_params(desc, 3))
