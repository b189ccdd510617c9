"""The ResNet -> network.json exporter and the executor's memory model
(CPU only).

The exporter charges every executor byte outside the GMAP-resident
featuremap to the layer workspaces, so for ANY pin set the planner may
return, the executor's real device bytes never exceed the planner's
layer-wise peak (model_ir.cpp:380-449).  Checked here for random pin sets
and minibatches by replaying the GMAP running sum (build_gmap order,
model_ir.cpp:342-354) against the executor's lifetime model.
"""
import json
import random

import pytest

from paper_1901_06773_b200 import planner, trainer

ARCHS = [("resnet20", 32, 12), ("resnet50", 224, 1000), ("resnet152", 224, 1000),
         ("resnet164", 32, 12)]


def scale_size(base, k, k_base):
    raw = -(-base * k // k_base)
    return 0 if raw == 0 else -(-raw // 512) * 512


def planned_peak(net, k, pinned):
    """peak_layerwise_memory(gmap, k, pins) restated for the test."""
    layers = net["layers"]
    n, kb = len(layers), net["k_base"]
    ws = [scale_size(l["workspace_bytes_base"], k, kb) for l in layers]
    fm = [scale_size(l["featuremap_bytes_base"], k, kb) for l in layers]
    run = peak = 0
    for l in range(n):  # forward phases: alloc ws, alloc fm, offload fm, release ws
        for d in (ws[l], fm[l], 0 if pinned[l] else -fm[l], -ws[l]):
            run += d
            peak = max(peak, run)
    for l in reversed(range(n)):  # backward: prefetch fm, alloc ws, release fm, release ws
        for d in (0 if pinned[l] else fm[l], ws[l], -fm[l], -ws[l]):
            run += d
            peak = max(peak, run)
    return peak


@pytest.mark.parametrize("arch,image,classes", ARCHS)
def test_network_json_is_valid_reference_document(arch, image, classes):
    net_json, desc = trainer.export_network(arch, image, classes, k_base=8)
    rc, report = planner.validate(net_json)
    assert rc == 0 and report.startswith("ok:"), report
    net = json.loads(net_json)
    assert net["format_version"] == 1 and net["k_base"] == 8
    assert len(net["layers"]) == len(desc["ops"])
    assert all(l["flops_fwd_base"] > 0 and l["flops_bwd_base"] > 0 for l in net["layers"])


def test_parameter_counts_match_torchvision():
    expect = {"resnet50": 25_557_032, "resnet152": 60_192_808}
    for arch, n in expect.items():
        net_json, desc = trainer.export_network(arch, 224, 1000)
        layers = json.loads(net_json)["layers"]
        # the stem stores 4 input channels (3 real + 1 zero pad)
        stem_pad = 64 * 7 * 7 * 1
        assert sum(l["param_bytes"] for l in layers) // 4 - stem_pad == n


def test_conv_flops_match_survey():
    # conv training FLOPs per image (fwd + dgrad + wgrad, no
    # stem dgrad): R50 24.29 G, R152 68.83 G
    for arch, gflops in (("resnet50", 24.29), ("resnet152", 68.83)):
        _, desc = trainer.export_network(arch, 224, 1000)
        f = 0.0
        for op in desc["ops"]:
            if op["kind"] == "conv":
                h, w, _ = op["out"]
                fwd = 2.0 * h * w * op["cout"] * op["r"] * op["r"] * (3 if op["in0"] == -2 else op["cin"])
                f += fwd * (2 if op["in0"] == -2 else 3)
        assert abs(f / 1e9 - gflops) / gflops < 0.01, f / 1e9


@pytest.mark.parametrize("arch,image,classes", ARCHS)
def test_executor_never_exceeds_planned_peak(arch, image, classes):
    net_json, desc = trainer.export_network(arch, image, classes, k_base=8)
    net = json.loads(net_json)
    n = len(desc["ops"])
    rng = random.Random(0)
    for k in (1, 3, 8, 27):
        for trial in range(4):
            frac = [0.0, 1.0, 0.5, rng.random()][trial]
            pinned = [rng.random() < frac for _ in range(n)]
            live, arena = trainer.net_memory(arch, image, classes, k, [not p for p in pinned])
            peak = planned_peak(net, k, pinned)
            assert live <= peak, (k, frac, live, peak)
            # static placement of the instances costs at most 2% fragmentation
            assert arena <= peak * 1.02 + (1 << 20), (k, frac, arena, peak)


def test_describe_layout_reverse_op_order():
    """parameters are laid out in reverse op order so backward fills the
    gradient buffer front to back (all-reduce buckets are prefixes)."""
    _, desc = trainer.export_network("resnet50", 224, 1000)
    offs = [op.get("w_off", op.get("g_off")) for op in desc["ops"]
            if op.get("w_off", op.get("g_off", -1)) is not None and op.get("w_off", op.get("g_off", -1)) >= 0]
    assert offs == sorted(offs, reverse=True)


@pytest.mark.parametrize("arch,image,classes", [("resnet50", 224, 1000), ("resnet18", 224, 1000)])
def test_transient_activations_memory_bound(monkeypatch, arch, image, classes):
    """recomputed bn_relu outputs (ACCUDNN_RECOMPUTE=1): 0-byte featuremaps,
    their forward and backward instances charged to the workspaces; the
    executor still never exceeds the planned peak, the reference's k_max
    accepts the spec, and the all-pinned (resident) peak shrinks."""
    net0, _ = trainer.export_network(arch, image, classes, k_base=8)
    monkeypatch.setenv("ACCUDNN_RECOMPUTE", "1")
    net_json, desc = trainer.export_network(arch, image, classes, k_base=8)
    assert any(o.get("transient") for o in desc["ops"])
    net = json.loads(net_json)
    for o, l in zip(desc["ops"], net["layers"]):
        assert (l["featuremap_bytes_base"] == 0) == bool(o.get("transient"))
    n = len(desc["ops"])
    rng = random.Random(1)
    for k in (1, 8, 27):
        for frac in (0.0, 1.0, 0.5):
            pinned = [rng.random() < frac for _ in range(n)]
            live, arena = trainer.net_memory(arch, image, classes, k, [not p for p in pinned])
            peak = planned_peak(net, k, pinned)
            assert live <= peak, (k, frac, live, peak)
    hw = trainer.hardware_json(8 << 30, trainer.default_m_others(desc, image, 8 << 30), 50e9)
    assert planner.kmax(net_json, hw) >= planner.kmax(net0, hw)
    resident = planned_peak(net, 32, [True] * n)
    resident0 = planned_peak(json.loads(net0), 32, [True] * n)
    assert resident < 0.9 * resident0, (resident, resident0)
