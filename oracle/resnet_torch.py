"""ORACLE / TEST INFRASTRUCTURE ONLY -- never imported by the product path.

CPU fp32 restatement of the training step the B200 executor runs, in plain
PyTorch, for the layer math the reference does not implement (the
reference's layers are FLOP/byte descriptors only, model_ir.hpp:14-32).
The network is rebuilt from the executor's own op description
(accudnn_net_export describe JSON), parameters are read from the same flat
vector layout, so both sides compute the same architecture with the same
weights:

  conv     F.conv2d       (weights stored [Cout][R][S][Cin] in the flat vector)
  bn(+relu) F.batch_norm(training=True, momentum=0.1, eps=1e-5) (+ F.relu)
  relu/add/maxpool/avgpool/fc/xent  F.relu, +, F.max_pool2d, mean, F.linear,
           F.cross_entropy (mean)
  SGD      buf = mu*buf + (g + wd*w)  (buf = g + wd*w on the first step),
           w -= lr*buf  (torch.optim.SGD semantics)
"""

import numpy as np
import torch
import torch.nn.functional as F


def tf32_truncate(t):
    """Drop the 13 low mantissa bits (what the tensor core reads from fp32)."""
    return (t.contiguous().view(torch.int32) & ~0x1FFF).view(torch.float32)


class _TF32Conv(torch.autograd.Function):
    """conv2d whose three GEMMs (fwd, dgrad, wgrad) see TF32-truncated operands,
    accumulating in fp32 -- an emulation of the tensor-core math."""

    @staticmethod
    def forward(ctx, x, w, stride, padding):
        ctx.save_for_backward(x, w)
        ctx.stride, ctx.padding = stride, padding
        return F.conv2d(tf32_truncate(x), tf32_truncate(w), stride=stride, padding=padding)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        gx = torch.nn.grad.conv2d_input(x.shape, tf32_truncate(w), tf32_truncate(gy),
                                        stride=ctx.stride, padding=ctx.padding)
        gw = torch.nn.grad.conv2d_weight(tf32_truncate(x), w.shape, tf32_truncate(gy),
                                         stride=ctx.stride, padding=ctx.padding)
        return gx, gw, None, None


class _Leaves:
    """the flat parameter vector as the forward pass slices it, backed by one
    autograd leaf per segment"""

    def __init__(self, leaves):
        self.leaves = leaves

    def __getitem__(self, sl):
        return self.leaves[(sl.start, sl.stop)]


class TorchResNet:
    """dtype: torch.float32 (default) or torch.float64 (ground truth);
    conv_math: "exact" or "tf32" (emulated tensor-core operand truncation,
    float32 only)."""

    def __init__(self, describe, dtype=torch.float32, conv_math="exact"):
        self.d = describe
        self.ops = describe["ops"]
        self.dtype = dtype
        self.conv_math = conv_math

    def _conv(self, x, w, stride, pad):
        if self.conv_math == "tf32":
            return _TF32Conv.apply(x, w, stride, pad)
        return F.conv2d(x, w, stride=stride, padding=pad)

    def _w(self, p, op):
        cout, cin, r = op["cout"], op["cin"], op["r"]
        w = p[op["w_off"]:op["w_off"] + cout * r * r * cin].view(cout, r, r, cin)
        return w.permute(0, 3, 1, 2)

    def forward(self, p, stats, images, labels):
        """images NCHW [k,3,H,W] fp32; returns the mean loss.  `stats` is the
        flat BN statistics vector (running mean/var updated in place)."""
        c4 = self.d["in_channels_padded"]
        x_img = F.pad(images, (0, 0, 0, 0, 0, c4 - images.shape[1]))
        t = {}
        for op in self.ops:
            kind = op["kind"]
            x = x_img if op["in0"] == -2 else t[op["in0"]]
            if kind == "conv":
                y = self._conv(x, self._w(p, op), op["stride"], op["pad"])
            elif kind in ("bn", "bn_relu", "bn_add_relu"):
                c = op["channels"]
                so = op["stat_off"]
                rm = stats[so + 2 * c:so + 3 * c]
                rv = stats[so + 3 * c:so + 4 * c]
                y = F.batch_norm(x, rm, rv, p[op["g_off"]:op["g_off"] + c],
                                 p[op["beta_off"]:op["beta_off"] + c], training=True,
                                 momentum=0.1, eps=1e-5)
                if kind == "bn_relu":
                    y = F.relu(y)
                elif kind == "bn_add_relu":  # relu(bn(conv) + shortcut), one op
                    y = F.relu(y + t[op["in1"]])
            elif kind == "relu":
                y = F.relu(x)
            elif kind == "add":
                y = x + t[op["in1"]]
            elif kind == "maxpool":
                y = F.max_pool2d(x, op["k"], op["stride"], op["pad"])
            elif kind == "avgpool":
                y = x.mean(dim=(2, 3))
            elif kind == "fc":
                w = p[op["w_off"]:op["w_off"] + op["cout"] * op["cin"]].view(op["cout"], op["cin"])
                b = p[op["b_off"]:op["b_off"] + op["cout"]]
                if self.conv_math == "tf32":
                    y = _TF32Conv.apply(x.reshape(x.shape[0], -1, 1, 1), w.reshape(*w.shape, 1, 1),
                                        1, 0).reshape(x.shape[0], -1) + b
                else:
                    y = F.linear(x.reshape(x.shape[0], -1), w, b)
            elif kind == "xent":
                return F.cross_entropy(x, labels.long())
            t[op["id"]] = y
        raise RuntimeError("network without a loss op")

    def _segments(self):
        segs = []
        for op in self.ops:
            if op["kind"] == "conv":
                segs.append((op["w_off"], op["cout"] * op["r"] * op["r"] * op["cin"]))
            elif op["kind"] == "fc":
                segs += [(op["w_off"], op["cout"] * op["cin"]), (op["b_off"], op["cout"])]
            elif op["kind"] in ("bn", "bn_relu", "bn_add_relu"):
                segs += [(op["g_off"], op["channels"]), (op["beta_off"], op["channels"])]
        return segs

    def step(self, params, stats, buf, images, labels, lr, momentum=0.9, wd=1e-4,
             first=True, update=True):
        """One fp32 SGD step on CPU; returns (loss, grads, new_params, new_buf).
        Every parameter segment is its own autograd leaf (slicing one flat
        leaf would make each slice's backward materialise a full-size
        gradient); the flat gradient vector is assembled afterwards."""
        leaves = {(o, o + n): torch.tensor(params[o:o + n], dtype=self.dtype, requires_grad=True)
                  for o, n in self._segments()}
        loss = self.forward(_Leaves(leaves), stats.to(self.dtype),
                            torch.as_tensor(images).to(self.dtype), torch.as_tensor(labels))
        loss.backward()
        g = np.zeros(len(params), dtype=np.float64)
        for (a, b), t in leaves.items():
            g[a:b] = t.grad.detach().numpy()
        if not update:
            return loss.item(), g, params, buf
        ft = np.float64 if self.dtype == torch.float64 else np.float32
        w = params.astype(ft)
        d = g + wd * w
        nb = d if first else momentum * buf + d
        return loss.item(), g, (w - lr * nb).astype(ft), nb.astype(ft)


def init_params(describe, seed=0):
    """Flat parameter vector with torchvision's default initialisation
    (Kaiming-normal fan_out convs, BN gamma=1 / beta=0, FC uniform
    +-1/sqrt(fan_in)) drawn from numpy's default_rng(seed) in op order -- the
    same draws as the product's trainer.init_params (tests/test_oracle_pinning
    checks they agree), restated here so the CPU reference arm of bench.py
    needs no product module."""
    rng = np.random.default_rng(seed)
    p = np.zeros(describe["n_params"], dtype=np.float32)
    for op in describe["ops"]:
        kind = op["kind"]
        if kind == "conv":
            cout, cin, r = op["cout"], op["cin"], op["r"]
            w = rng.standard_normal((cout, r, r, cin)).astype(np.float32) * (2.0 / (cout * r * r)) ** 0.5
            if op["in0"] == -2:
                w[..., describe["in_channels"]:] = 0.0
            p[op["w_off"]:op["w_off"] + w.size] = w.ravel()
        elif kind == "fc":
            cout, cin = op["cout"], op["cin"]
            bound = 1.0 / cin ** 0.5
            p[op["w_off"]:op["w_off"] + cout * cin] = rng.uniform(-bound, bound, cout * cin)
            p[op["b_off"]:op["b_off"] + cout] = rng.uniform(-bound, bound, cout)
        elif kind in ("bn", "bn_relu", "bn_add_relu"):
            p[op["g_off"]:op["g_off"] + op["channels"]] = 1.0
    return p
