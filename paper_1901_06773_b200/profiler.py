"""B200 profiler: measured phase times and host-link transfers in the
reference's profile CSV formats (profiles.cpp:57-154), the input of the
perf-model fit (the paper's profiling stage).

  compute rows  minibatch,phase,layer_type,flops,time_s
                one row per phase (1..2N) per sampled minibatch; time = CUDA
                events around the phase's kernels on the compute stream of an
                instrumented (eager, serial) step, scaled so that the phases sum
                to the measured CUDA-graph step at that minibatch (the step the
                executor actually runs: no launch gaps, weight gradients
                overlapped) -- the phases keep their measured shares
  transfer rows minibatch,seq_no,bytes,time_s
                one row per featuremap offload (GMAP sequence number of the
                offload op) per sampled minibatch; time = CUDA events around
                a FIFO burst of pinned-memory D2H copies of that many bytes,
                per copy (the executor's swap-out stream)

The sampling grid is 1/8, 1/4, 1/2, 2/3, 1 x k_ref (synthetic.cpp:102); k_ref
is the largest minibatch that trains resident on one B200 with headroom
(not the budget's k_max: its host-side featuremap store would not fit).
"""

import json

import numpy as np

from . import trainer


def grid(k_ref):
    ks = []
    for f in (1 / 8, 1 / 4, 1 / 2, 2 / 3, 1.0):
        k = max(1, int(round(f * k_ref)))
        if k not in ks:
            ks.append(k)
    return ks


def _scale_flops(flops_base, k, k_base):
    # C4: (flops*k + k_base/2) / k_base in integers (profiles.cpp:174-182)
    return (flops_base * k + k_base // 2) // k_base


def phase_table(network_json):
    """[(phase, type_key, flops_base)] for phases 1..2N (model_ir.cpp:238-264)."""
    net = json.loads(network_json)
    layers = net["layers"]
    n = len(layers)
    out = []
    for j in range(1, 2 * n + 1):
        l = layers[j - 1] if j <= n else layers[2 * n - j]
        key = l.get("type_tag") if l["layer_type"] == "other" else l["layer_type"]
        fl = l["flops_fwd_base"] if j <= n else l["flops_bwd_base"]
        out.append((j, key, int(fl)))
    return out, int(net["k_base"])


def profile_compute(arch, image, classes, network_json, ks, steps=2, seed=0, graph_steps=4,
                    scale_to_graph=True):
    phases, k_base = phase_table(network_json)
    _, desc = trainer.export_network(arch, image, classes)
    params = trainer.init_params(desc, seed=seed)
    rows = ["minibatch,phase,layer_type,flops,time_s"]
    for k in ks:
        ex = trainer.Executor(arch, image, classes, k=k)
        ex.set_params(params)
        g = np.random.default_rng(seed)
        x = g.standard_normal((k, 3, image, image)).astype(np.float32)
        y = g.integers(0, classes, size=k).astype(np.int32)
        times = None
        for _ in range(steps):
            ex.step(x, y, lr=0.0, update=False, profile=True)
            tr = ex.trace().strip().splitlines()[1:]
            t = {int(r.split(",")[0]): float(r.split(",")[2]) - float(r.split(",")[1]) for r in tr}
            times = t if times is None else {j: min(times[j], t[j]) for j in t}
        scale = 1.0
        if scale_to_graph:
            # the captured step (lr = 0: parameters unchanged), min over steps
            ex.set_graph(True)
            graph_ms = min(ex.step(x, y, lr=0.0)["iter_ms"] for _ in range(graph_steps + 1))
            total = sum(times.values())
            if total > 0 and graph_ms > 0:
                scale = graph_ms / total
        for j, key, fl in phases:
            rows.append(f"{k},{j},{key},{_scale_flops(fl, k, k_base)},{times[j] * scale * 1e-3:.12g}")
        ex.close()
    return "\n".join(rows) + "\n"


def profile_transfer(network_json, ks, repeats=2, burst=8):
    """Pinned-memory D2H copy time of every featuremap at every k, as the
    executor's swap-out stream sees it: the steady-state time per copy of a
    FIFO burst of `burst` back-to-back copies of that size (per-copy DMA
    set-up and inter-copy gaps included, which dominate for the sub-MB
    featuremaps of the CIFAR nets), best of `repeats` bursts."""
    import torch
    net = json.loads(network_json)
    k_base = int(net["k_base"])
    layers = net["layers"]
    rows = ["minibatch,seq_no,bytes,time_s"]
    max_bytes = max(-(-int(l["featuremap_bytes_base"]) * max(ks) // k_base) for l in layers)
    dev = torch.empty(max_bytes // 4 + 1024, dtype=torch.float32, device="cuda")
    host = torch.empty(max_bytes // 4 + 1024, dtype=torch.float32, pin_memory=True)
    s = torch.cuda.Stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in ks:
        for l in layers:
            raw = -(-int(l["featuremap_bytes_base"]) * k // k_base)
            nbytes = (raw + 511) // 512 * 512 if raw else 0  # scale_size (C3)
            if nbytes == 0:
                continue
            n = nbytes // 4
            best = None
            with torch.cuda.stream(s):
                for _ in range(repeats):
                    a.record(s)
                    for _ in range(burst):
                        host[:n].copy_(dev[:n], non_blocking=True)
                    b.record(s)
                    b.synchronize()
                    ms = a.elapsed_time(b) / burst
                    best = ms if best is None else min(best, ms)
            seq = 4 * (int(l["index"]) - 1) + 2  # GMAP offload op of layer l
            rows.append(f"{k},{seq},{nbytes},{best * 1e-3:.12g}")
    return "\n".join(rows) + "\n"


def host_link_bandwidth(nbytes=1 << 28, repeats=5):
    """(D2H, H2D, concurrent-both) GB/s with pinned memory."""
    import torch
    dev = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    dev2 = torch.empty_like(dev)
    host = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    host2 = torch.empty_like(host, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("d2h", "h2d", "both"):
        best = None
        for _ in range(repeats):
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            if name in ("d2h", "both"):
                s1.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s1):
                    host.copy_(dev, non_blocking=True)
            if name in ("h2d", "both"):
                s2.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s2):
                    dev2.copy_(host2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            b.record()
            b.synchronize()
            ms = a.elapsed_time(b)
            best = ms if best is None else min(best, ms)
        moved = nbytes * (2 if name == "both" else 1)
        res[name] = moved / (best * 1e-3) / 1e9
    return res
