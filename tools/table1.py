"""Measured Table-1-style sweep: for each k and mode
{naive, dynamic, resident} the B200 executor's measured iteration time and
peak device bytes next to the planner/simulator prediction of the same cell
(sweep_grid, the reference's `swapsched sweep`).  The perf model is fitted
from the committed B200 profiles, so the comparison validates the model
(the reference tolerates 15% in-sample, test_perf_model.cpp:217-230).
Usage: table1.py [arch] [k,k,...] [cap_gib] [json_out]"""
import csv
import io
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1901_06773_b200 import _native, planner, trainer  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet152"
ks = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "8,16,32,42").split(",")]
cap = float(sys.argv[3]) if len(sys.argv) > 3 else 8.0
out_path = sys.argv[4] if len(sys.argv) > 4 else None
image, classes = (224, 1000) if arch in ("resnet50", "resnet101", "resnet152") else (32, 12)
tune = os.path.join(ROOT, "profiles", "b200", "conv_tune.txt")
if os.path.exists(tune):
    _native.conv_tune_import(open(tune).read())
net, desc = trainer.export_network(arch, image, classes, k_base=8)
link = json.load(open(os.path.join(ROOT, "profiles", "b200", "host_link.json")))
hw = trainer.hardware_json(int(cap * (1 << 30)), trainer.default_m_others(desc, image, int(cap * (1 << 30))),
                           link["d2h"] * 1e9)
prof = os.path.join(ROOT, "profiles", "b200")
model = planner.fit(net, [open(os.path.join(prof, f"{arch}_compute_profile.csv")).read(),
                          open(os.path.join(prof, f"{arch}_transfer_profile.csv")).read()], hw, eta=0.95)
pred = {(int(r["k"]), r["mode"]): r for r in
        csv.DictReader(io.StringIO(planner.sweep(net, hw, model, ks, "naive,dynamic,resident")))}
rows = []
g = np.random.default_rng(0)
for k in ks:
    x = torch.from_numpy(g.standard_normal((k, 3, image, image)).astype(np.float32)).cuda()
    y = torch.from_numpy(g.integers(0, classes, size=k).astype(np.int32)).cuda()
    for mode in os.environ.get("TABLE1_MODES", "resident,dynamic,naive").split(","):
        p = pred[(k, mode)]
        plan = None
        if mode == "dynamic":
            try:
                plan = planner.plan(net, hw, model, k_override=k)
            except planner.PlannerError:
                rows.append({"k": k, "mode": mode, "note": "no plan"})
                continue
        try:
            # the same documents as the prediction: the executor's cap and
            # swap-in queue follow hardware.json (without them a naive plan
            # falls back to a fixed one-phase prefetch lookahead)
            ex = trainer.Executor(arch, image, classes, k=k, mode=mode, plan_json=plan,
                                  network_json=net, hardware_json=hw)
        except Exception as e:  # does not fit the device
            rows.append({"k": k, "mode": mode, "note": str(e)[:80]})
            continue
        ex.set_params(trainer.init_params(desc, 0))
        ex.set_graph(True)
        for _ in range(3):
            ex.step(x, y, lr=0.01)
        ms = float(np.median([ex.step(x, y, lr=0.01)["iter_ms"] for _ in range(5)]))
        arena, fixed = ex.memory()
        ex.close()
        rec = {"k": k, "mode": mode, "measured_iter_s": round(ms * 1e-3, 6),
               "predicted_iter_s": float(p["iter_time_s"]), "predicted_feasible": p["feasible"],
               "measured_peak_bytes": int(arena + fixed),
               "predicted_peak_bytes": int(p["peak_mem_bytes"]),
               "measured_img_per_s": round(k / (ms * 1e-3), 1)}
        rec["iter_rel_err"] = round(rec["measured_iter_s"] / rec["predicted_iter_s"] - 1.0, 4)
        rows.append(rec)
        print(json.dumps(rec), flush=True)
res = {"arch": arch, "cap_gib": cap, "rows": rows}
if out_path:
    json.dump(res, open(out_path, "w"), indent=1)
