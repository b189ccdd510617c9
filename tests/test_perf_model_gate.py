"""Perf-model gate on the B200 measurements.

The reference checks that its fitted model reproduces in-sample rates within
15% (/root/reference/proj/tests/test_perf_model.cpp:217-230) on synthetic
profiles drawn from one saturating curve per layer type -- where a per-type
fit is exact by construction.  Real B200 layers of one type differ by shape
(a 1x1 and a 3x3 convolution of equal FLOPs do not take equal time), so the
per-sample bound does not transfer; what the planner consumes is the sum
over phases (Eq. 2/3, the iteration time that enters the stall constraint and
Eq. 8).  The gate here is that sum:
  * in-sample: for every profiled minibatch of every committed B200 profile,
    the model's iteration compute time is within 15% of the measured one;
  * Table 1: the measured iteration time of every (k, mode) cell of the
    committed ResNet-152 sweep (tools/table1.py, executor on a B200) is
    within 15% of the sweep's prediction, and the prediction is reproduced
    bit-for-bit by the planner from the committed documents now.
"""
import csv
import io
import json
import os

import pytest

from paper_1901_06773_b200 import planner, trainer

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles", "b200")
ARCHS = [("resnet20", 32, 12), ("resnet50", 224, 1000), ("resnet152", 224, 1000),
         ("resnet1001", 32, 12)]


@pytest.mark.parametrize("arch,image,classes", ARCHS, ids=[a[0] for a in ARCHS])
def test_in_sample_iteration_compute_within_15_percent(arch, image, classes):
    net, hw, model, _ = trainer.config_documents(arch, image, classes, 8 << 30)
    rows = list(csv.DictReader(open(os.path.join(PROF, f"{arch}_compute_profile.csv"))))
    ks = sorted({int(r["minibatch"]) for r in rows})
    assert len(ks) >= 4
    for k in ks:
        pred = sum(planner.phase_times(net, model, k)) * 1e-9
        meas = sum(float(r["time_s"]) for r in rows if int(r["minibatch"]) == k)
        assert abs(pred - meas) / meas < 0.15, (arch, k, pred, meas)


def _table1():
    # round 2 on: the executor measured with the same documents as the
    # prediction (hardware.json's cap drives its swap-in queue); the round-1
    # sweep ran the executor without them (fixed one-phase prefetch lookahead)
    p = os.path.join(ROOT, "profiles", "r02", "table1_r152.json")
    if not os.path.exists(p):
        pytest.skip("no committed round-2 Table-1 sweep")
    return p, json.load(open(p))


def test_table1_measured_cells_within_15_percent():
    path, t = _table1()
    cap = int(t["cap_gib"] * (1 << 30))
    net, hw, model, _ = trainer.config_documents(t["arch"], 224, 1000, cap)
    ks = sorted({r["k"] for r in t["rows"]})
    pred = {(int(r["k"]), r["mode"]): r for r in
            csv.DictReader(io.StringIO(planner.sweep(net, hw, model, ks, "naive,dynamic,resident")))}
    for r in t["rows"]:
        p = pred[(r["k"], r["mode"])]
        assert float(p["iter_time_s"]) == pytest.approx(r["predicted_iter_s"], abs=1e-9), r
        err = (r["measured_iter_s"] - r["predicted_iter_s"]) / r["predicted_iter_s"]
        assert abs(err) < 0.15, (os.path.relpath(path, ROOT), r["k"], r["mode"], err)
