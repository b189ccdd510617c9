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

`--gpus N` without torchrun re-launches itself under torch.distributed.run
(one process per GPU, 127.0.0.1 rendezvous); under torchrun every rank runs
its replica and rank 0 prints the line.

`--impl reference` times the reference's CPU path on the same documents
(tests/golden/headline_docs, no product library loaded): the reference
planner (oracle/_ref, Algorithm 2 at step 1), its simulator's modelled
images/s for that plan, and the CPU training step (plain PyTorch fp32
restatement, oracle/resnet_torch.py, all host cores) on a bounded sample of
the k* batch -- its images/s is the line's value.
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
    ap.add_argument("--cpu-sample", type=int, default=4,
                    help="images of the k* batch per CPU (reference / baseline) step")
    ap.add_argument("--conv-math", default="tf32", choices=["tf32", "3xtf32"],
                    help="3xtf32: fp32-accurate convolutions (split operands, 3 MMAs)")
    ap.add_argument("--dry-run", action="store_true",
                    help="host side only (documents, plan, rendezvous, max over ranks); no GPU")
    ap.add_argument("--nccl-allowance-mib", type=int, default=768,
                    help="device MiB charged to m_others for NCCL's buffers when N > 1")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch_distributed(args):
    """`--gpus N` (N > 1) outside torchrun: run this script under
    torch.distributed.run with N local ranks on a free 127.0.0.1 port and
    return its exit code (rank 0 prints the JSON line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    # NCCL's init log (ranks, channels, NVLS) on stderr, stdout stays one line
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return subprocess.run(cmd, env=env).returncode


def headline_docs(arch, image, cap_gib):
    """committed copies of the documents bench.py plans on (written by
    tests/golden/make_golden.py from the exporter; tests pin them equal)"""
    stem = os.path.join(ROOT, "tests", "golden", "headline_docs", f"{arch}_{image}_{int(cap_gib)}GiB")
    if not os.path.exists(stem + ".network.json"):
        return None
    return {k: open(f"{stem}.{k}.json").read() for k in ("network", "hardware", "model", "describe")}


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
def plan_for(args, m_others_extra=0):
    """documents -> k*: network.json from the exporter, model.json fitted
    from the committed B200 profiles (trainer.config_documents, the same
    documents the headline goldens pin), then the tuner."""
    from paper_1901_06773_b200 import planner, profiler, trainer
    cap = int(args.cap_gib * GIB)
    pdir = os.path.join(ROOT, "profiles", "b200")
    if os.path.exists(os.path.join(pdir, f"{args.arch}_compute_profile.csv")):
        network_json, hardware_json, model_json, desc = trainer.config_documents(
            args.arch, args.image, args.classes, cap)
        source = f"profiles/b200/{args.arch}_compute_profile.csv"
    else:  # profile live (first run on a new config)
        network_json, desc = trainer.export_network(args.arch, args.image, args.classes, k_base=8)
        link = json.load(open(os.path.join(pdir, "host_link.json")))
        hardware_json = trainer.hardware_json(cap, trainer.default_m_others(desc, args.image, cap),
                                              float(link.get("d2h", 50.0)) * 1e9)
        ks = profiler.grid(32)
        comp = profiler.profile_compute(args.arch, args.image, args.classes, network_json, ks)
        tran = profiler.profile_transfer(network_json, ks)
        model_json = planner.fit(network_json, [comp, tran], hardware_json, eta=0.95)
        source = "live"
    if m_others_extra:
        # data parallel: NCCL's device buffers are part of the fixed overhead
        hw = json.loads(hardware_json)
        hw["m_others_bytes"] += int(m_others_extra)
        hardware_json = json.dumps(hw, indent=2) + "\n"
    t0 = time.perf_counter()
    plan_json = planner.plan(network_json, hardware_json, model_json, k_override=max(0, args.k))
    plan_s = time.perf_counter() - t0
    return network_json, hardware_json, model_json, desc, plan_json, plan_s, source


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
def _oracle_torch():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import resnet_torch
    return resnet_torch


def cpu_step_seconds(desc, image, classes, sample, threads, steps=1, warmup=1, seed=0):
    """CPU training step (oracle port: plain PyTorch fp32 on the host cores,
    oracle/resnet_torch.py) on `sample` images; returns per-step seconds."""
    import numpy as np
    import torch
    rt = _oracle_torch()
    torch.set_num_threads(threads)
    params = rt.init_params(desc, seed)
    g = np.random.default_rng(seed)
    x = g.standard_normal((sample, 3, image, image)).astype(np.float32)
    y = g.integers(0, classes, size=sample).astype(np.int32)
    o = rt.TorchResNet(desc)
    stats = torch.zeros(desc["n_stats"])
    buf = None
    for _ in range(warmup):
        _, _, params, buf = o.step(params, stats, buf, x, y, lr=0.1, first=buf is None)
    out = []
    for _ in range(steps):
        t0 = time.perf_counter()
        _, _, params, buf = o.step(params, stats, buf, x, y, lr=0.1, first=buf is None)
        out.append(time.perf_counter() - t0)
    return out


def reference_cpu_path(network_json, hardware_json, model_json, k_ours=None, plan_ours=None):
    """The reference's own CPU implementation of the host path (oracle/_ref,
    compiled from /root/reference/proj/src): Algorithm 2 at step 1 on the
    same documents (planner.cpp:346-424), timed, and simulate_iteration of
    its plan (simulator.cpp:79-370) -> the reference's modelled images/s.
    With plan_ours, plan_parity says whether the documents are identical."""
    path = os.path.join(ROOT, "oracle", "_ref", "libswapsched_ref.so")
    if not os.path.exists(path):
        return {"unavailable": "oracle/_ref/libswapsched_ref.so not built"}
    import ctypes
    from paper_1901_06773_b200 import _native, planner
    lib = ctypes.CDLL(path)
    _native.declare_planner_symbols(lib, "oracle_")
    R = dict(lib=lib, prefix="oracle_")
    t0 = time.perf_counter()
    plan_ref = planner.plan(network_json, hardware_json, model_json, step=1, **R)
    plan_s = time.perf_counter() - t0
    k = json.loads(plan_ref)["k_star"]
    t0 = time.perf_counter()
    _, summ, _ = planner.simulate(network_json, hardware_json, model_json, plan_ref, "dynamic", k, **R)
    sim_s = time.perf_counter() - t0
    summ = json.loads(summ)
    out = {"kind": "reference", "k_star": k, "planner_seconds_step1": round(plan_s, 3),
           "simulate_seconds": round(sim_s, 4),
           "modelled_iter_ms": None if summ.get("oom") else round(summ["iter_time_s"] * 1e3, 3),
           "modelled_images_per_s": None if summ.get("oom") else round(k / summ["iter_time_s"], 2),
           "modelled_stall_ms": None if summ.get("oom") else round(summ["total_stall_s"] * 1e3, 4)}
    # the reference's parallel grid sweep (sweep.cpp, OpenMP over cells on all
    # host cores; the bench/sweep_bench.cpp:46-64 method) on the same documents
    ks = sorted({8, 16, 32, k})
    t0 = time.perf_counter()
    sw_ref = planner.sweep(network_json, hardware_json, model_json, ks, "naive,dynamic,resident",
                           parallel=True, **R)
    out["sweep_seconds_parallel"] = round(time.perf_counter() - t0, 4)
    out["sweep_cells"] = 3 * len(ks)
    out["sweep_threads"] = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    if plan_ours is not None:
        out["plan_parity"] = plan_ref == plan_ours
        # the same grid through the B200 host library: identical CSV
        t0 = time.perf_counter()
        sw = planner.sweep(network_json, hardware_json, model_json, ks, "naive,dynamic,resident")
        out["sweep_seconds_b200_host"] = round(time.perf_counter() - t0, 4)
        out["sweep_parity"] = sw == sw_ref
    return out


def loaded_repo_libraries():
    """shared objects under the repo mapped into this process"""
    try:
        maps = open("/proc/self/maps").read().splitlines()
    except OSError:
        return None
    libs = {ln.split()[-1] for ln in maps if ln.endswith(".so") and ROOT in ln}
    return sorted(os.path.relpath(p, ROOT) for p in libs)


# ---------------------------------------------------------------------------
def run_reference(args):
    """CPU reference arm: no product library on this path (documents from
    tests/golden/headline_docs, the reference planner/simulator from
    oracle/_ref, the CPU step from oracle/resnet_torch.py)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    docs = headline_docs(args.arch, args.image, args.cap_gib)
    if docs is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no committed documents for {args.arch}@{args.image} "
                          f"{args.cap_gib:g} GiB (tests/golden/make_golden.py HEADLINE)"}), flush=True)
        return
    threads = os.cpu_count() or 1
    ref = reference_cpu_path(docs["network"], docs["hardware"], docs["model"])
    k = args.k or ref.get("k_star") or 0
    desc = json.loads(docs["describe"])
    # bounded sample: as many of the k* images per step as keep the whole
    # --steps/--warmup run within ~150 s on this host (at most --cpu-sample)
    steps, warm = max(1, args.steps), max(1, args.warmup)
    probe = cpu_step_seconds(desc, args.image, args.classes, 1, threads, steps=1, warmup=1)[0]
    sample = int(max(1, min(args.cpu_sample, k or args.cpu_sample, 150.0 / ((steps + warm) * probe))))
    secs = cpu_step_seconds(desc, args.image, args.classes, sample, threads, steps=steps,
                            warmup=max(0, warm - 1))
    ms = 1e3 * sum(secs) / len(secs)
    value = sample / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": "images/s (ResNet-152 training step, tuned minibatch, "
        "device cap)", "value": round(value, 3), "unit": "images/s", "n_gpus": 0,
        "launched_with_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": round(ms, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) images, uniform labels, torchvision-style init",
        "config": {"workload": f"{args.arch}@{args.image}, {args.cap_gib:g} GiB device cap per GPU, "
                   f"tuner k*={k} per GPU, global batch {k}",
                   "model": args.arch, "k_star": k, "cap_bytes": int(args.cap_gib * GIB),
                   "same_config": True,
                   "sample": f"{sample} of the k*={k} images per timed step (a bounded sample; "
                             "images/s = sample / step time)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "images/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{sample} images per step, {steps} steps: the training "
                                   "step restated in plain PyTorch fp32 (oracle/resnet_torch.py; the "
                                   "reference has no layer math)"},
        "reference_planner": ref,
        "e2e": {"value": round(value, 3), "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "native_libraries_loaded": loaded_repo_libraries(),
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1901_06773_b200 import planner, trainer

    world, rank, local = dist_env()
    if args.dry_run:
        return run_dry(args, world, rank)
    if "ACCUDNN_PDL" in os.environ:  # A/B switch for programmatic dependent launch
        trainer._lib().accudnn_set_pdl(int(os.environ["ACCUDNN_PDL"]))
    if args.conv_math == "3xtf32":
        trainer._lib().accudnn_set_conv_math(1)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    # ---- host side of the path: spec, profiles -> model, tuner -> plan, LR ----
    # (every rank plans on identical documents: identical k* and pins; N > 1
    # charges NCCL's device buffers to the fixed overhead before planning)
    extra = (args.nccl_allowance_mib << 20) if world > 1 else 0
    if args.conv_math == "3xtf32":
        # the 3xTF32 convolutions' low-part scratch is a fixed device allocation
        _, d0 = trainer.export_network(args.arch, args.image, args.classes)
        extra += trainer.precise_scratch_allowance(d0, args.image, args.cap_gib * (1 << 30))
    network_json, hardware_json, model_json, desc, plan_json, plan_s, prof_src = plan_for(args, extra)
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
    torch.cuda.synchronize()
    free_before_exec, _ = torch.cuda.mem_get_info(dev)
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
    # launch list of the same step (latest round first, dram__bytes_read+write)
    ls_path = next((p for p in (os.path.join(ROOT, "profiles", r, f"launch_summary_k{k}.json")
                                for r in ("r02", "r01")) if os.path.exists(p)), "")
    if ls_path:
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
    # host-link bandwidth the plan was made with (hardware.json)
    pcie = float(json.loads(hardware_json).get("pcie_nominal_bytes_per_s", 0.0)) or 56e9
    t_swap = swapped / pcie if swapped else 0.0
    img_roof = k / max(t_conv, t_swap)

    # data parallel: all-reduce device time and the compute stream's wait at
    # its join, measured in the profiled step; the exposed part is the
    # reference's per-iteration delta_sync_s (model_ir.hpp:108,
    # perf_model.cpp:141-143), written back into hardware.json
    dp = None
    if world > 1:
        ar = max_over_ranks(prof.get("exposed_allreduce_ms", 0.0))
        hw = json.loads(hardware_json)
        hw["delta_sync_s"] = ar * 1e-3
        hw_delta = json.dumps(hw, indent=2) + "\n"
        pred = json.loads(plan_json).get("predicted_iter_time_s")
        dp = {"allreduce_ms": round(max_over_ranks(prof.get("allreduce_ms", 0.0)), 3),
              "exposed_allreduce_ms": round(ar, 3), "delta_sync_s": ar * 1e-3,
              "grad_bytes": 4 * desc["n_params"], "bucket_bytes": 25 << 20,
              "nccl_device_bytes": int(max_over_ranks(float(ex.comm_bytes()))),
              "nccl_allowance_bytes": extra,
              "predicted_iter_ms_with_delta": None if pred is None else round((pred + ar * 1e-3) * 1e3, 3)}
        if rank == 0:
            os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
            with open(os.path.join(ROOT, "gpurun_out", f"hardware_dp{world}.json"), "w") as f:
                f.write(hw_delta)
    free_after, total_mem = torch.cuda.mem_get_info(dev)
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # ---- CPU legs (after the timed region): the reference's planner +
    # simulator on the same documents (plan parity), and the CPU step ----
    try:
        km = planner.kmax(network_json, hardware_json)
        if km > 5000:
            # the reference scans k_max..1 serially (planner.cpp:376-408) at ~48 s per
            # evaluation for ResNet-1001: days.  Parity for this config is pinned by
            # tests/golden/resnet1001_plan.json (reference evaluations at k*, k*+1).
            ref = {"kind": "reference", "skipped": f"reference step-1 scan over k_max = {km} "
                   "candidates is not bounded here; evaluations at k*, k*+1 pinned by "
                   "tests/golden/resnet1001_plan.json"}
        else:
            ref = reference_cpu_path(network_json, hardware_json, model_json, plan_ours=plan_json)
    except Exception as e:  # never fail the GPU line on a baseline
        ref = {"error": str(e)}
    try:
        secs = cpu_step_seconds(desc, args.image, args.classes, min(k, args.cpu_sample), threads)
        cpu_rate, cpu_dt = min(k, args.cpu_sample) / secs[0], secs[0]
    except Exception as e:
        cpu_rate, cpu_dt = None, str(e)
    clk = clocks.summary()
    n_fm = len(desc["ops"])
    arch_name = {"resnet152": "ResNet-152", "resnet50": "ResNet-50", "resnet20": "ResNet-20",
                 "resnet1001": "ResNet-1001"}.get(args.arch, args.arch)
    line = {
        "metric": f"images/s ({arch_name} training step, tuned minibatch, device cap)",
        "value": round(value, 2), "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (TF32 tensor-core convolutions)" if args.conv_math == "tf32"
                 else "f32 (3xTF32 convolutions: fp32-accurate)",
        "data": f"synthetic N(0,1) {args.image}x{args.image} images, uniform labels, "
                "torchvision-style random init",
        "config": {"workload": f"{args.arch}@{args.image}, {args.cap_gib:g} GiB device cap per GPU, "
                   f"tuner k*={k} per GPU, global batch {world * k}",
                   "model": args.arch, "global_batch": world * k, "k_star": k,
                   "parallelism": f"dp{world}", "cap_bytes": int(args.cap_gib * GIB),
                   "pinned_featuremaps": f"{len(plan['pinned_objects'])}/{n_fm}",
                   "lr_alpha_star": lr, "cuda_graph": not args.no_graph,
                   "conv_math": args.conv_math,
                   "l2": "inputs > L2: each step streams the batch's activations "
                         f"(~{sum(4 * o['out'][0] * o['out'][1] * o['out'][2] for o in desc['ops']) * k >> 20} MiB)",
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
        "memory": {"peak_device_bytes": int(arena + fixed + ex.comm_bytes()), "arena_bytes": int(arena),
                   "fixed_bytes": int(fixed), "nccl_bytes": int(ex.comm_bytes()),
                   "cap_bytes": int(args.cap_gib * GIB),
                   "measured_executor_device_bytes": int(free_before_exec - free_after),
                   "measured_process_device_bytes": int(total_mem - free_after),
                   "note": "measured_* = cudaMemGetInfo deltas: executor = free before its "
                           "construction minus free after the timed steps (arena, fixed "
                           "buffers, NCCL, CUDA-graph and library internals); process "
                           "additionally holds the CUDA context and torch's input tensors"},
        "swap": {"swapped_bytes_per_step": int(swapped),
                 "exposed_swap_ms": round(prof["exposed_swap_ms"], 3),
                 "exposed_swap_frac": round(prof["exposed_swap_ms"] / max(prof["iter_ms"], 1e-9), 4)},
        "dp": dp,
        "planner": {"plan_seconds_b200_host": round(plan_s, 4), "reference": ref,
                    "plan_parity": ref.get("plan_parity")},
        "clocks": clk,
        "cpu_baseline": {"value": None if cpu_rate is None else round(cpu_rate, 3),
                         "unit": "images/s", "cores": threads, "kind": "port",
                         "sample": f"{min(k, args.cpu_sample)} of the k* images, one torch fp32 CPU "
                                   f"step ({cpu_dt if isinstance(cpu_dt, str) else round(cpu_dt, 2)} s; "
                                   "oracle/resnet_torch.py -- the reference has no layer math); "
                                   "the reference's own CPU path (planner + simulator) is "
                                   "planner.reference"},
    }
    print(json.dumps(line), flush=True)


def run_dry(args, world, rank):
    """Host side of every rank without a GPU (CPU tests of the launcher):
    documents and plan per rank, gloo rendezvous, k* / plan digest gathered
    and checked equal across ranks, max over ranks, one line from rank 0."""
    import hashlib

    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    extra = (args.nccl_allowance_mib << 20) if world > 1 else 0
    t0 = time.perf_counter()
    network_json, hardware_json, model_json, desc, plan_json, plan_s, src = plan_for(args, extra)
    k = json.loads(plan_json)["k_star"]
    digest = int(hashlib.sha256(plan_json.encode()).hexdigest()[:12], 16)
    mine = torch.tensor([float(k), float(digest), time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        allv = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allv, mine)
        dist.barrier()
    else:
        allv = [mine]
    same = all(float(v[0]) == k and float(v[1]) == digest for v in allv)
    if rank == 0:
        print(json.dumps({"metric": "images/s (dry run: host side only)", "value": None,
                          "unit": "images/s", "n_gpus": world, "dry_run": True, "k_star": k,
                          "global_batch": world * k, "plans_identical_across_ranks": same,
                          "host_seconds_max_over_ranks": round(max(float(v[2]) for v in allv), 4),
                          "m_others_extra_bytes": extra}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    world, _, _ = dist_env()
    if args.gpus > 1 and world == 1 and "TORCHELASTIC_RUN_ID" not in os.environ:
        sys.exit(relaunch_distributed(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
