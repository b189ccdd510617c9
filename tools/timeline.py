"""Kernel timeline of the captured training step (CUPTI via torch.profiler):
busy time vs gaps on the device, per-kernel in-situ durations.
Usage: timeline.py [arch] [k] [steps] [json_out]"""
import collections
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1901_06773_b200 import trainer  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet152"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 27
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
out_path = sys.argv[4] if len(sys.argv) > 4 else None
image, classes = (224, 1000) if arch in ("resnet50", "resnet101", "resnet152") else (32, 12)
_, desc = trainer.export_network(arch, image, classes)
# PDL lets a kernel start (and CUPTI's clock for it run) while it waits for its
# predecessor: per-kernel durations are only meaningful with ACCUDNN_PDL=0
if "ACCUDNN_PDL" in os.environ:
    trainer._lib().accudnn_set_pdl(int(os.environ["ACCUDNN_PDL"]))
_tune = os.path.join(ROOT, "profiles", "b200", "conv_tune.txt")
if os.path.exists(_tune):
    from paper_1901_06773_b200 import _native
    _native.conv_tune_import(open(_tune).read())
ex = trainer.Executor(arch, image, classes, k=k)
ex.set_params(trainer.init_params(desc, 0))
ex.set_graph(True)
g = np.random.default_rng(0)
x = torch.from_numpy(g.standard_normal((k, 3, image, image)).astype(np.float32)).cuda()
y = torch.from_numpy(g.integers(0, classes, size=k).astype(np.int32)).cuda()
for _ in range(4):
    ex.step(x, y, lr=0.01)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        ex.step(x, y, lr=0.01)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs
               if "memcpy" not in e.name.lower() and "memset" not in e.name.lower()])
if not kern:
    print("no kernel events captured")
    sys.exit(1)
span = kern[-1][1] - kern[0][0]
busy, last_end, gaps, big = 0.0, kern[0][0], [], []
prev = ""
for s, e, nm in kern:
    if s > last_end:
        gaps.append(s - last_end)
        big.append((s - last_end, prev[:50], nm[:50]))
    busy += max(0.0, e - max(s, last_end))
    last_end = max(last_end, e)
    prev = nm
agg = collections.defaultdict(lambda: [0, 0.0])
for s, e, n in kern:
    key = n.replace("(anonymous namespace)::", "").replace("accudnn::", "").replace("void ", "")
    key = key.split("(")[0][:60]
    agg[key][0] += 1
    agg[key][1] += e - s
gaps = np.array(gaps) if gaps else np.zeros(1)
res = {"arch": arch, "k": k, "steps": steps, "kernels_per_step": len(kern) / steps,
       "span_ms_per_step": span / steps / 1e3, "busy_ms_per_step": busy / steps / 1e3,
       "gap_ms_per_step": gaps.sum() / steps / 1e3, "gap_us_median": float(np.median(gaps)),
       "gap_us_p90": float(np.percentile(gaps, 90)),
       "top": sorted(([n, c // steps, round(t / steps / 1e3, 3), round(t / c, 2)]
                      for n, (c, t) in agg.items()), key=lambda r: -r[2])[:25]}
print(json.dumps({k_: v for k_, v in res.items() if k_ != "top"}, indent=1))
print("largest gaps (us, before -> after):")
for gp in sorted(big, reverse=True)[:8]:
    print("  %.1f  %s -> %s" % gp)
print("kernel | launches/step | ms/step | us/launch")
for r in res["top"]:
    print(" | ".join(str(v) for v in r))

# per-stream view (chrome trace carries the stream of every kernel): the
# critical path runs on the compute stream (the one launching batch norms);
# its idle time is where it waited on the weight-gradient stream or on SMs
import tempfile  # noqa: E402
with tempfile.NamedTemporaryFile(suffix=".json") as tf:
    prof.export_chrome_trace(tf.name)
    trace = json.load(open(tf.name))
per_stream = collections.defaultdict(list)
for ev in trace.get("traceEvents", []):
    if ev.get("cat") == "kernel":
        per_stream[ev.get("args", {}).get("stream", ev.get("tid"))].append(
            (float(ev["ts"]), float(ev["ts"]) + float(ev.get("dur", 0)), ev.get("name", "")))
streams = {}
for sid, ks in per_stream.items():
    ks.sort()
    busy_s, end_s, idle = 0.0, ks[0][0], []
    for a0, a1, nm in ks:
        if a0 > end_s:
            idle.append((a0 - end_s, nm[:50]))
        busy_s += max(0.0, a1 - max(a0, end_s))
        end_s = max(end_s, a1)
    streams[str(sid)] = {"kernels_per_step": len(ks) / steps,
                         "busy_ms_per_step": busy_s / steps / 1e3,
                         "idle_ms_per_step": sum(i for i, _ in idle) / steps / 1e3,
                         "has_bn": any("bn_fused" in nm for _, _, nm in ks),
                         "largest_idle": [[round(i, 1), nm] for i, nm in sorted(idle, reverse=True)[:6]]}
res["streams"] = streams
print(json.dumps(streams, indent=1))
if out_path:
    json.dump(res, open(out_path, "w"), indent=1)
