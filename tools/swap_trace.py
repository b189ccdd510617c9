"""Swap-executor timeline on a BASELINE config: captured-step time of the
plan's swapping vs all-resident, and the real trace / summary documents of a
profiled step next to the simulator's for the same documents and plan.

  python tools/swap_trace.py resnet20 32 12 8 [cap_gib] [pins: plan|every3|naive] [outdir]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_06773_b200 import planner, trainer  # noqa: E402

arch, image, classes, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cap = int(float(sys.argv[5]) * (1 << 30)) if len(sys.argv) > 5 else 8 << 30
pins = sys.argv[6] if len(sys.argv) > 6 else "plan"
out = sys.argv[7] if len(sys.argv) > 7 else "gpurun_out/swap_trace"
os.makedirs(out, exist_ok=True)
net, hw, model, desc = trainer.config_documents(arch, image, classes, cap)
plan = planner.plan(net, hw, model, k_override=k)
n = len(desc["ops"])
if pins != "plan":
    p = json.loads(plan)
    p["pinned_objects"] = [f"fm{l}" for l in range(1, n + 1, 3)] if pins == "every3" else []
    plan = json.dumps(p)
g = np.random.default_rng(0)
x = g.standard_normal((k, 3, image, image)).astype(np.float32)
y = g.integers(0, classes, size=k).astype(np.int32)
params = trainer.init_params(desc, 0)
res = {}
for name, mode in (("resident", "resident"), ("dynamic", "dynamic")):
    ex = trainer.Executor(arch, image, classes, k=k, mode=mode, plan_json=plan, network_json=net,
                          hardware_json=hw)
    ex.set_params(params)
    ex.set_graph(True)
    for _ in range(3):
        ex.step(x, y, lr=0.01)
    ts = [ex.step(x, y, lr=0.01)["iter_ms"] for _ in range(30)]
    prof = ex.step(x, y, lr=0.01, update=False, profile=True)
    arena, fixed = ex.memory()
    res[name] = {"graph_ms_median": float(np.median(ts)), "graph_ms_min": float(np.min(ts)),
                 "profiled_iter_ms": prof["iter_ms"], "exposed_swap_ms": prof["exposed_swap_ms"],
                 "swapped_bytes": prof["swapped_bytes"], "arena": arena, "fixed": fixed}
    if mode == "dynamic":
        for doc in ("trace", "summary", "stall_bars", "mem_curves", "order"):
            with open(os.path.join(out, f"real_{doc}.{'json' if doc == 'summary' else 'csv'}"), "w") as f:
                f.write(ex.document(doc))
    ex.close()
rc, summ, trace = planner.simulate(net, hw, model, plan, "dynamic", k)
with open(os.path.join(out, "sim_trace.csv"), "w") as f:
    f.write(trace)
with open(os.path.join(out, "sim_summary.json"), "w") as f:
    f.write(summ)
s = json.loads(summ)
res["simulated"] = {"iter_ms": s.get("iter_time_s", 0) * 1e3, "stall_ms": s.get("total_stall_s", 0) * 1e3}
res["exposed_frac_graph"] = res["dynamic"]["graph_ms_median"] / res["resident"]["graph_ms_median"] - 1
print(json.dumps(res, indent=1))
with open(os.path.join(out, "summary.json"), "w") as f:
    json.dump(res, f, indent=1)
