"""Swap-executor stress (BASELINE config 5 and forced swap plans): for each
case the captured step with the case's swap plan next to the same step all
resident, and the simulator's prediction of both for the same documents.

  exposed_swap_ms      = graph step (swap plan) - graph step (resident)
  sim_exposed_ms       = simulated iter (swap plan) - simulated iter (resident)
  sim_total_stall_ms   = simulate_iteration's total_stall of the swap plan

Cases: ResNet-1001 @32 and ResNet-152 @224 with every featuremap offloaded
(naive) and with every third pinned (forced dynamic), ResNet-20 @32 with the
planner's own plan (config 1).

  python tools/swap_stress.py [json_out]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_06773_b200 import _native, planner, trainer  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/swap_stress.json"
tune = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "b200",
                    "conv_tune.txt")
if os.path.exists(tune):
    _native.conv_tune_import(open(tune).read())

CASES = [  # arch, image, classes, cap GiB, k, pins
    ("resnet20", 32, 12, 8, 8, "plan"),
    ("resnet20", 32, 12, 8, 8, "naive"),   # config 1's naive-mode run
    ("resnet1001", 32, 12, 8, 41, "naive"),
    ("resnet1001", 32, 12, 8, 41, "every3"),
    ("resnet152", 224, 1000, 8, 8, "naive"),
    ("resnet152", 224, 1000, 8, 16, "every3"),
]


def timed(ex, x, y, steps):
    ex.set_graph(True)
    for _ in range(3):
        ex.step(x, y, lr=0.01)
    return float(np.median([ex.step(x, y, lr=0.01)["iter_ms"] for _ in range(steps)]))


rows = []
for arch, image, classes, cap_gib, k, pins in CASES:
    net, hw, model, desc = trainer.config_documents(arch, image, classes, cap_gib << 30)
    n = len(desc["ops"])
    base = json.loads(planner.plan(net, hw, model, k_override=k)) if pins == "plan" else None
    if base is None:
        # a plan document at k for the forced pin set (t_ready etc. are not
        # read by the executor; the simulator's dynamic mode uses the pins)
        try:
            base = json.loads(planner.plan(net, hw, model, k_override=k))
        except planner.PlannerError:
            base = json.loads(planner.plan(net, hw, model))
            base["k_star"] = k
        base["pinned_objects"] = ([] if pins == "naive" else
                                  [f"fm{l}" for l in range(1, n + 1, 3)])
    plan = json.dumps(base)
    g = np.random.default_rng(0)
    x = g.standard_normal((k, 3, image, image)).astype(np.float32)
    y = g.integers(0, classes, size=k).astype(np.int32)
    params = trainer.init_params(desc, 0)
    steps = 10 if arch == "resnet152" else 30
    r = {"arch": arch, "image": image, "k": k, "cap_gib": cap_gib, "pins": pins,
         "pinned": len(base["pinned_objects"]), "featuremaps": n}
    res = trainer.Executor(arch, image, classes, k=k, network_json=net, hardware_json=hw)
    res.set_params(params)
    r["resident_ms"] = timed(res, x, y, steps)
    res.close()
    dyn = trainer.Executor(arch, image, classes, k=k, mode="dynamic", plan_json=plan,
                           network_json=net, hardware_json=hw)
    dyn.set_params(params)
    r["swap_ms"] = timed(dyn, x, y, steps)
    st = dyn.step(x, y, lr=0.01, update=False, profile=True)
    r["swapped_bytes_each_way"] = st["swapped_bytes"]
    arena, fixed = dyn.memory()
    r["swap_device_bytes"] = arena + fixed
    dyn.close()
    r["exposed_swap_ms"] = r["swap_ms"] - r["resident_ms"]
    r["exposed_frac"] = r["exposed_swap_ms"] / r["resident_ms"]
    _, s_dyn, _ = planner.simulate(net, hw, model, plan, "dynamic", k)
    _, s_res, _ = planner.simulate(net, hw, model, None, "resident", k)
    sd, sr = json.loads(s_dyn), json.loads(s_res)
    r["sim_swap_ms"] = sd["iter_time_s"] * 1e3
    r["sim_resident_ms"] = sr["iter_time_s"] * 1e3
    r["sim_exposed_ms"] = r["sim_swap_ms"] - r["sim_resident_ms"]
    r["sim_total_stall_ms"] = sd["total_stall_s"] * 1e3
    r["link_bound_ms"] = r["swapped_bytes_each_way"] / (json.loads(hw)["pcie_nominal_bytes_per_s"]
                                                       if "pcie_nominal_bytes_per_s" in json.loads(hw)
                                                       else 56e9) * 1e3
    print(json.dumps(r), flush=True)
    rows.append(r)
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump({"rows": rows}, f, indent=1)
