"""ResNet-152 images/s at the tuner-chosen minibatch under a device memory
cap on 1..8 B200s (BASELINE.json `metric`, configs[2]/[3]).

A "step" is one full training iteration of the hot path at k* images per
GPU: forward, backward, swap traffic of the plan, bucketed NCCL gradient
all-reduce (N > 1), SGD-momentum update.  Before timing, the path's host
side runs exactly as a user would: export network.json, fit model.json from
the B200 profile CSVs (profiles/b200/, measured by tools/profile_b200.py),
plan (Algorithm 2 + greedy pinning -> k*, pin set), adapted learning rate
(Eq. 9), executor on the plan.

  value  images/s with inputs already in HBM (device time, CUDA events on
         the executor's compute stream, max over ranks)
  e2e    images/s through the C ABI step with pinned HOST inputs: the H2D
         copy of the batch and the loss read-back are inside the timed step

`--impl reference` times the CPU implementation of the same step (oracle
port: plain PyTorch fp32 on all host cores, oracle/resnet_torch.py) on a
bounded sample, plus the reference planner (oracle/_ref) on the same
documents.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GIB = 1 << 30


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arch", default="resnet152")
    ap.add_argument("--image", type=int, default=224)
    ap.add_argument("--classes", type=int, default=1000)
    ap.add_argument("--cap-gib", type=float, default=8.0)
    ap.add_argument("--k", type=int, default=0, help="override k* (0 = tuner)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=2, help="images in the CPU baseline step")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        """NVML (a few µs per sample): the same fields as the nvidia-smi query."""
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while not self._stop.is_set():
            sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
            self._stop.wait(0.01)
        N.nvmlShutdown()

    def _run(self):
        try:
            return self._run_nvml()
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def plan_for(args, network_json, hardware_json):
    """fit model.json from the committed B200 profiles and run the tuner."""
    from paper_1901_06773_b200 import planner, profiler
    pdir = os.path.join(ROOT, "profiles", "b200")
    cpath = os.path.join(pdir, f"{args.arch}_compute_profile.csv")
    tpath = os.path.join(pdir, f"{args.arch}_transfer_profile.csv")
    if os.path.exists(cpath) and os.path.exists(tpath):
        comp, tran = open(cpath).read(), open(tpath).read()
        source = os.path.relpath(cpath, ROOT)
    else:  # profile live (first run on a new config)
        ks = profiler.grid(32)
        comp = profiler.profile_compute(args.arch, args.image, args.classes, network_json, ks)
        tran = profiler.profile_transfer(network_json, ks)
        source = "live"
    model_json = planner.fit(network_json, [comp, tran], hardware_json, eta=0.95)
    t0 = time.perf_counter()
    if args.k > 0:
        plan_json = planner.plan(network_json, hardware_json, model_json, k_override=args.k)
    else:
        plan_json = planner.plan(network_json, hardware_json, model_json)
    plan_s = time.perf_counter() - t0
    return model_json, plan_json, plan_s, source


def conv_flops_per_image(desc):
    f = 0.0
    for op in desc["ops"]:
        if op["kind"] in ("conv", "fc"):
            h, w, c = op["out"]
            fwd = 2.0 * h * w * op["cout"] * op["cin"] * op["r"] * op["r"]
            f += fwd * (2.0 if op["in0"] == -2 else 3.0)
    return f


def count_kernel_launches(step_fn):
    """kernels of one (captured) training step, counted from the CUPTI
    activity records of our library (names in namespace accudnn)."""
    import warnings

    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step_fn()
            torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    return sum(1 for n in names if "accudnn" in n), len(names)


def roofline_from_trace(desc, trace_csv, k, peak_tflops, n_ops):
    """conv / fc phases of a profiled step -> achieved TFLOP/s of the implicit
    GEMM kernels (phase j <= N: forward of op j-1; phase j > N: backward of op
    2N+1-j, plus op 0 in phase 2N)."""
    rows = [r.split(",") for r in trace_csv.strip().splitlines()[1:]]
    t = {int(r[0]): float(r[2]) - float(r[1]) for r in rows}
    ops = desc["ops"]
    conv_ms, total_ms, conv_flops = 0.0, 0.0, 0.0
    for j, ms in t.items():
        total_ms += ms
        ids = [j - 1] if j <= n_ops else ([2 * n_ops + 1 - j] if 2 * n_ops + 1 - j < n_ops else [])
        if j == 2 * n_ops:
            ids.append(0)
        for o in ids:
            op = ops[o]
            if op["kind"] in ("conv", "fc"):
                h, w, c = op["out"]
                fwd = 2.0 * h * w * op["cout"] * op["cin"] * op["r"] * op["r"] * k
                conv_flops += fwd if j <= n_ops else fwd * (1.0 if op["in0"] == -2 else 2.0)
                conv_ms += ms / len(ids)
    achieved = conv_flops / (conv_ms * 1e-3) / 1e12 if conv_ms > 0 else 0.0
    return {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak_tflops,
            "unit": "TFLOP/s", "frac": round(achieved / peak_tflops, 4), "traffic": None,
            "kernel": "conv_sm100_kernel (persistent, TMA + tcgen05 kind::tf32, TMEM accumulators)",
            "conv_share_of_step": round(conv_ms / total_ms, 4) if total_ms else None,
            "flops_per_launch_note": "sum of conv/fc fwd+dgrad+wgrad FLOPs per step / sum of "
                                     "their phase times (CUDA events on the compute stream)",
            "conv_flops_per_step": conv_flops}


def conv_kernel_us(step_fn):
    """device durations (CUPTI) of the convolution kernels of one step: the
    persistent TMA/tcgen05 kernel, the cp.async kernel and the split-K reduce
    that completes a split GEMM."""
    import warnings

    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            out = step_fn()
            torch.cuda.synchronize()
    keys = ("conv_sm100_kernel", "conv_igemm_kernel", "conv_splitk_reduce")
    cuda = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs = [e for e in cuda if any(q in e.name for q in keys)]
    bn = [e for e in cuda if "bn_fused_kernel" in e.name]
    conv_kernel_us.bn_us = sum(e.time_range.end - e.time_range.start for e in bn)
    conv_kernel_us.bn_launches = len(bn)
    return out, sum(e.time_range.end - e.time_range.start for e in evs), len(evs)


def bn_min_bytes_per_step(desc, k):
    """algorithmic (single-touch) HBM bytes of the step's batch-norm passes:
    forward reads x (+ the shortcut) and writes y; backward reads x, dy (+ the
    shortcut for the ReLU mask) and writes dx (+ d(shortcut))."""
    total = 0
    for op in desc["ops"]:
        if op["kind"] not in ("bn", "bn_relu", "bn_add_relu"):
            continue
        h, w, c = op["out"]
        S = 4 * k * h * w * c
        tail = op["kind"] == "bn_add_relu"
        total += (3 if tail else 2) * S + (5 if tail else 3) * S
    return total


# ---------------------------------------------------------------------------
def cpu_step_rate(arch, image, classes, k, threads, seed=0):
    """oracle port: plain PyTorch fp32 training step on the host cores."""
    import numpy as np
    import torch
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from resnet_torch import TorchResNet
    from paper_1901_06773_b200 import trainer
    torch.set_num_threads(threads)
    _, desc = trainer.export_network(arch, image, classes)
    params = trainer.init_params(desc, seed)
    g = np.random.default_rng(seed)
    x = g.standard_normal((k, 3, image, image)).astype(np.float32)
    y = g.integers(0, classes, size=k).astype(np.int32)
    o = TorchResNet(desc)
    stats = torch.zeros(desc["n_stats"])
    o.step(params, stats, None, x, y, lr=0.1)  # warm-up
    t0 = time.perf_counter()
    o.step(params, stats, None, x, y, lr=0.1)
    dt = time.perf_counter() - t0
    return k / dt, dt


def reference_planner_seconds(network_json, hardware_json, model_json):
    path = os.path.join(ROOT, "oracle", "_ref", "libswapsched_ref.so")
    if not os.path.exists(path):
        return None
    import ctypes
    from paper_1901_06773_b200 import _native, planner
    lib = ctypes.CDLL(path)
    _native.declare_planner_symbols(lib, "oracle_")
    t0 = time.perf_counter()
    try:
        planner.plan(network_json, hardware_json, model_json, lib=lib, prefix="oracle_", step=16)
    except planner.PlannerError:
        pass
    return time.perf_counter() - t0


# ---------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from paper_1901_06773_b200 import trainer
    k = args.k or 24
    rates = []
    for _ in range(max(1, args.warmup)):
        cpu_step_rate(args.arch, args.image, args.classes, args.cpu_sample, threads)
    for _ in range(max(1, args.steps)):
        r, _ = cpu_step_rate(args.arch, args.image, args.classes, args.cpu_sample, threads)
        rates.append(r)
    value = sum(rates) / len(rates)
    line = {
        "impl": "reference", "metric": "images/s (ResNet-152 training step, tuned minibatch, "
        "device cap)", "value": round(value, 3), "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * args.cpu_sample / value, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) images, uniform labels, torchvision-style init",
        "config": {"workload": f"{args.arch}@{args.image} training step, k*={k} per GPU "
                   f"(bounded sample of {args.cpu_sample} images per timed step)",
                   "cap_gib": args.cap_gib},
        "cpu_baseline": {"value": round(value, 3), "unit": "images/s", "cores": threads,
                         "kind": "port", "sample": f"{args.cpu_sample} images/step, torch fp32 "
                         "CPU restatement (oracle/resnet_torch.py)"},
        "e2e": {"value": round(value, 3), "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1901_06773_b200 import planner, trainer

    world, rank, local = dist_env()
    if "ACCUDNN_PDL" in os.environ:  # A/B switch for programmatic dependent launch
        trainer._lib().accudnn_set_pdl(int(os.environ["ACCUDNN_PDL"]))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    # ---- host side of the path: spec, profiles -> model, tuner -> plan, LR ----
    network_json, desc = trainer.export_network(args.arch, args.image, args.classes, k_base=8)
    link = {}
    lp = os.path.join(ROOT, "profiles", "b200", "host_link.json")
    if os.path.exists(lp):
        link = json.load(open(lp))
    pcie = float(link.get("d2h", 50.0)) * 1e9
    m_others = trainer.default_m_others(desc, args.image, int(args.cap_gib * GIB))
    hardware_json = trainer.hardware_json(int(args.cap_gib * GIB), m_others, pcie)
    model_json, plan_json, plan_s, prof_src = plan_for(args, network_json, hardware_json)
    plan = json.loads(plan_json)
    k = plan["k_star"]
    q = world * k / 8.0
    lr, _, _ = planner.tune_lr(0.1, 1.0, max(1.0, q))

    # conv (tile width, split-K) table tuned on B200 and committed with the
    # profiles; shapes it lacks are tuned in the first (eager) step
    from paper_1901_06773_b200 import _native
    tune_path = os.path.join(ROOT, "profiles", "b200", "conv_tune.txt")
    if os.path.exists(tune_path) and not os.environ.get("ACCUDNN_RETUNE"):
        _native.conv_tune_import(open(tune_path).read())
    ex = trainer.Executor(args.arch, args.image, args.classes, mode="dynamic", plan_json=plan_json,
                          network_json=network_json, hardware_json=hardware_json, device=local)
    ex.set_params(trainer.init_params(desc, seed=0))
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(trainer.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        ex.set_comm(uid.cpu().numpy().tobytes(), rank, world)
    ex.set_graph(not args.no_graph)

    g = np.random.default_rng(100 + rank)
    x_host = torch.from_numpy(g.standard_normal((k, 3, args.image, args.image)).astype(np.float32)).pin_memory()
    y_host = torch.from_numpy(g.integers(0, args.classes, size=k).astype(np.int32)).pin_memory()
    x_dev, y_dev = x_host.to(dev), y_host.to(dev)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up (first step captures the CUDA graph on the second call)
    for _ in range(max(3, args.warmup)):
        ex.step(x_dev, y_dev, lr=lr)
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", "conv_tune.txt"), "w") as f:
            f.write(_native.conv_tune_export())

    # ---- timed: device-resident inputs ----
    barrier()
    dev_ms = 0.0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            st = ex.step(x_dev, y_dev, lr=lr)
            dev_ms += st["iter_ms"]
    barrier()
    ms_per_step = max_over_ranks(dev_ms / args.steps)
    value = world * k / (ms_per_step * 1e-3)

    # ---- timed: end to end with pinned host inputs ----
    # pipelined input (the user-facing data path): every step copies the next
    # batch H2D from pinned host memory on a side stream while it computes,
    # and reads the loss back; one batch copy + one loss read per timed step
    ex.step_pipelined(x_host, y_host, lr=lr, next_images=x_host)  # prime the pipeline
    barrier()
    t0 = time.perf_counter()
    e2e_dev_ms = 0.0
    for _ in range(args.steps):
        st = ex.step_pipelined(None, y_host, lr=lr, next_images=x_host)
        e2e_dev_ms += st["iter_ms"]
    barrier()
    e2e_wall = max_over_ranks((time.perf_counter() - t0) / args.steps)
    e2e_value = world * k / e2e_wall
    ex.step(x_dev, y_dev, lr=lr)  # drop the outstanding prefetch before the profiled steps

    ours_launches, all_device_ops = count_kernel_launches(lambda: ex.step(x_dev, y_dev, lr=lr))

    # ---- one profiled step (not timed): exposed swap + conv roofline ----
    # (the profiled step runs every kernel on the compute stream, in order:
    # the conv kernels' CUPTI durations are undilated by the weight-gradient
    # stream)
    prof, conv_us, conv_launches = conv_kernel_us(
        lambda: ex.step(x_dev, y_dev, lr=lr, update=False, profile=True))
    trace = ex.trace()
    peaks = {}
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        peaks = json.load(open(pp))
    bf16 = float(peaks.get("bf16_tflops_sustained", 1405.3))
    # the convolutions run TF32: the denominator is the measured sustained
    # cuBLAS TF32 GEMM rate on this pool's B200s (profiles/b200/tf32_peak.json,
    # tools/measure_tf32_peak.py); fallback 1/2 of the measured bf16 figure
    tf32_path = os.path.join(ROOT, "profiles", "b200", "tf32_peak.json")
    if os.path.exists(tf32_path):
        tf32_peak = float(json.load(open(tf32_path))["tf32_tflops_sustained"])
        peak_note = ("measured sustained cuBLAS TF32 GEMM 8192^3 on B200 (profiles/b200/"
                     "tf32_peak.json); 1/2 of MEASURED_PEAKS bf16 sustained would be %.1f" % (bf16 / 2))
    else:
        tf32_peak = round(bf16 / 2.0, 1)
        peak_note = ("TF32 dense peak taken as 1/2 of the measured cuBLAS bf16 sustained "
                     "figure in MEASURED_PEAKS.json (nominal 1.1 vs 2.25 PF)")
    roof = roofline_from_trace(desc, trace, k, tf32_peak, len(desc["ops"]))
    roof["peak_note"] = peak_note
    # achieved = algorithmic FLOPs of the step's conv GEMMs / the summed device
    # duration of the kernels computing them (per the roofline definition: work
    # per launch / that kernel's launch duration); the phase-event figure, which
    # also counts launch gaps inside the eager profiled step, is kept beside it
    if conv_us > 0:
        ach = roof["conv_flops_per_step"] / (conv_us * 1e-6) / 1e12
        roof["achieved_phase_events"] = roof["achieved"]
        roof["frac_phase_events"] = roof["frac"]
        roof["achieved"] = round(ach, 2)
        roof["frac"] = round(ach / tf32_peak, 4)
        roof["conv_kernel_ms_per_step"] = round(conv_us / 1e3, 3)
    # the second-largest kernel family, HBM-bound: batch norm (single-touch
    # algorithmic bytes / CUPTI device time of its kernels, same profiled step)
    hbm_peak = float(peaks.get("hbm_gbs", 0.0)) or 6650.0  # fallback: B200_PROFILING.md
    bn_us = getattr(conv_kernel_us, "bn_us", 0.0)
    roofline_bn = None
    if bn_us > 0:
        ach_bn = bn_min_bytes_per_step(desc, k) / (bn_us * 1e-6) / 1e9
        roofline_bn = {"bound": "hbm", "kernel": "bn_fused_kernel (cooperative / cluster single-kernel BN)",
                       "achieved": round(ach_bn, 1), "peak": hbm_peak, "unit": "GB/s",
                       "frac": round(ach_bn / hbm_peak, 4) if hbm_peak else None,
                       "launches_per_step": conv_kernel_us.bn_launches,
                       "kernel_ms_per_step": round(bn_us / 1e3, 3),
                       "note": "algorithmic bytes = one read of every input and one write of every "
                               "output per pass (the two-pass kernels re-read x, partly from L2); "
                               "peak = MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"}
        roof["conv_kernel_launches_per_step"] = conv_launches
        roof["flops_per_launch_note"] = (
            "achieved = conv/fc fwd+dgrad+wgrad FLOPs per step / summed CUPTI device duration of "
            "their kernels (TMA/tcgen05 conv, cp.async conv, split-K reduce) in the profiled "
            "serial step; achieved_phase_events = same FLOPs / CUDA-event phase times")
    # DRAM traffic of the conv kernels per launch, from the committed ncu
    # launch list of the same step (profiles/r01, dram__bytes_read+write)
    ls_path = os.path.join(ROOT, "profiles", "r01", f"launch_summary_k{k}.json")
    if os.path.exists(ls_path):
        summ = json.load(open(ls_path))
        cv = [v for n, v in summ.items() if "conv_sm100_kernel" in n or "conv_igemm_kernel" in n]
        n_launch = sum(v["launches"] for v in cv)
        if n_launch:
            roof["traffic"] = round(sum(v["dram_bytes"] for v in cv) / n_launch)
            roof["traffic_unit"] = "DRAM bytes per conv launch (ncu, cold cache, serialised)"
            roof["algorithmic_flops_per_launch"] = round(k * conv_flops_per_image(desc) / n_launch)
    arena, fixed = ex.memory()
    f_conv = conv_flops_per_image(desc)
    swapped = prof["swapped_bytes"]
    t_conv = k * f_conv / (tf32_peak * 1e12)
    t_swap = swapped / pcie if swapped else 0.0
    img_roof = k / max(t_conv, t_swap)

    if rank != 0:
        return
    threads = os.cpu_count() or 1
    try:
        cpu_rate, cpu_dt = cpu_step_rate(args.arch, args.image, args.classes, args.cpu_sample,
                                         threads)
    except Exception as e:  # never fail the GPU line on the CPU baseline
        cpu_rate, cpu_dt = None, str(e)
    ref_plan_s = None
    try:
        ref_plan_s = reference_planner_seconds(network_json, hardware_json, model_json)
    except Exception:
        pass
    clk = clocks.summary()
    n_fm = len(desc["ops"])
    line = {
        "metric": "images/s (ResNet-152 training step, tuned minibatch, device cap)",
        "value": round(value, 2), "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (TF32 tensor-core convolutions)",
        "data": "synthetic N(0,1) 224x224 images, uniform labels, torchvision-style random init",
        "config": {"workload": f"{args.arch}@{args.image}, {args.cap_gib:g} GiB device cap per GPU, "
                   f"tuner k*={k} per GPU, global batch {world * k}",
                   "model": args.arch, "global_batch": world * k, "k_star": k,
                   "parallelism": f"dp{world}", "cap_bytes": int(args.cap_gib * GIB),
                   "pinned_featuremaps": f"{len(plan['pinned_objects'])}/{n_fm}",
                   "lr_alpha_star": lr, "cuda_graph": not args.no_graph,
                   "l2": "inputs > L2: each step streams ~k*273 MiB of activations",
                   "profiles": prof_src},
        "e2e": {"value": round(e2e_value, 2), "unit": "images/s",
                "h2d_bytes_per_step": int(x_host.numel() * 4 + y_host.numel() * 4),
                "d2h_bytes_per_step": 4},
        "gpu_launches": ours_launches,
        "gpu_launches_note": f"kernels of one captured step counted from CUPTI records "
                             f"({all_device_ops} device activities incl. copies)",
        "roofline": roof,
        "roofline_bn": roofline_bn,
        "roofline_official": {"img_per_s_roof": round(img_roof * world, 2),
                              "frac": round(value / (img_roof * world), 4),
                              "definition": "k / max(k*F_conv/P_tf32, B_swap/BW_host) per GPU"},
        "memory": {"peak_device_bytes": int(arena + fixed), "arena_bytes": int(arena),
                   "fixed_bytes": int(fixed), "cap_bytes": int(args.cap_gib * GIB)},
        "swap": {"swapped_bytes_per_step": int(swapped),
                 "exposed_swap_ms": round(prof["exposed_swap_ms"], 3),
                 "exposed_swap_frac": round(prof["exposed_swap_ms"] / max(prof["iter_ms"], 1e-9), 4)},
        "planner": {"plan_seconds_b200_host": round(plan_s, 4),
                    "reference_planner_seconds_step16": None if ref_plan_s is None else round(ref_plan_s, 3)},
        "clocks": clk,
        "cpu_baseline": {"value": None if cpu_rate is None else round(cpu_rate, 3),
                         "unit": "images/s", "cores": threads, "kind": "port",
                         "sample": f"{args.cpu_sample} images, one torch fp32 CPU step "
                                   f"({cpu_dt if isinstance(cpu_dt, str) else round(cpu_dt, 2)} s)"},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
