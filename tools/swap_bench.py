"""Swap-executor stress on ResNet-152 (the tuned 8 GiB plan swaps nothing on a
B200): the same step at a given k with (a) every featuremap resident, (b) the
planner's pin set for k (k_override, may swap), (c) naive mode (every
featuremap offloaded after its forward and prefetched for its backward).
Reports device ms/step, swapped bytes and the exposed swap time (compute
gaps in front of phases that waited on a copy stream).
Usage: swap_bench.py [k] [json_out]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1901_06773_b200 import _native, planner, trainer  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
out_path = sys.argv[2] if len(sys.argv) > 2 else None
arch, image, classes = "resnet152", 224, 1000
tune = os.path.join(ROOT, "profiles", "b200", "conv_tune.txt")
if os.path.exists(tune):
    _native.conv_tune_import(open(tune).read())
net, desc = trainer.export_network(arch, image, classes, k_base=8)
link = json.load(open(os.path.join(ROOT, "profiles", "b200", "host_link.json")))
hw = trainer.hardware_json(8 << 30, trainer.default_m_others(desc, image), link["d2h"] * 1e9)
comp = open(os.path.join(ROOT, "profiles", "b200", f"{arch}_compute_profile.csv")).read()
tran = open(os.path.join(ROOT, "profiles", "b200", f"{arch}_transfer_profile.csv")).read()
model = planner.fit(net, [comp, tran], hw, eta=0.95)
g = np.random.default_rng(0)
x = torch.from_numpy(g.standard_normal((k, 3, image, image)).astype(np.float32)).cuda()
y = torch.from_numpy(g.integers(0, classes, size=k).astype(np.int32)).cuda()
res = {"arch": arch, "k": k, "host_link_gbs": link}
modes = [("resident", None)]
try:
    modes.append(("dynamic", planner.plan(net, hw, model, k_override=k)))
except planner.PlannerError as e:
    res["dynamic_plan_error"] = str(e)
modes.append(("naive", None))
for mode, plan in modes:
    ex = trainer.Executor(arch, image, classes, k=k, mode=mode, plan_json=plan)
    ex.set_params(trainer.init_params(desc, 0))
    for _ in range(2):
        ex.step(x, y, lr=0.01)
    ms = []
    for _ in range(3):
        ms.append(ex.step(x, y, lr=0.01)["iter_ms"])
    prof = ex.step(x, y, lr=0.01, update=False, profile=True)
    res[mode] = {"ms_per_step": round(float(np.median(ms)), 3),
                 "img_per_s": round(k / (float(np.median(ms)) * 1e-3), 1),
                 "swapped_bytes": int(prof["swapped_bytes"]),
                 "exposed_swap_ms_profiled": round(prof["exposed_swap_ms"], 3),
                 "profiled_iter_ms": round(prof["iter_ms"], 3),
                 "pinned": None if plan is None else len(json.loads(plan)["pinned_objects"])}
    swap_ms = prof["swapped_bytes"] / (link["d2h"] * 1e9) * 1e3 if prof["swapped_bytes"] else 0.0
    res[mode]["swap_time_at_link_bw_ms"] = round(swap_ms, 3)
    ex.close()
    print(mode, json.dumps(res[mode]), flush=True)
print(json.dumps(res))
if out_path:
    json.dump(res, open(out_path, "w"), indent=1)
