"""Command-line front end, compatible with the reference `swapsched` CLI
(/root/reference/proj/tools/swapsched.cpp:539-674): the same subcommands,
flags, output documents and exit codes (0 ok, 1 validation / infeasible,
2 I/O, 3 internal), over the B200 planner library (include/accudnn_plan.h).
Documents carry the same `manifest_digest` (FNV-1a over the subcommand, the
input files' bytes and `key=value;` parameters, swapsched.cpp:76-91).

B200 additions:
  export   ResNet -> network.json (+ hardware.json for a cap) through the
           executor's exporter (csrc/runtime/net.cpp)
  execute  run the planned training iteration on the GPU and write the
           measured per-phase trace (trace.csv) next to the simulator's, with
           summary.json (iteration time, exposed swap, peak bytes)

    python -m paper_1901_06773_b200.cli plan --network n.json --hardware h.json \\
        --model model.json --out plan.json
"""
import argparse
import json
import os
import sys

from . import planner


class CliError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _read(path):
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError as e:
        raise CliError(2, f"cannot open {path}: {e.strerror}")


def _text(path):
    return _read(path).decode()


def _write(path, content):
    d = os.path.dirname(path)
    try:
        if d:
            os.makedirs(d, exist_ok=True)
        with open(path, "w") as f:
            f.write(content)
    except OSError as e:
        raise CliError(2, f"cannot write {path}: {e.strerror}")


def manifest_digest(subcommand, inputs, params):
    """FNV-1a 64 over subcommand, input file bytes, then "key=value;" params
    (swapsched.cpp:76-91)."""
    h = 1469598103934665603
    def mix(data):
        nonlocal h
        for c in data:
            h ^= c
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    mix(subcommand.encode())
    for p in inputs:
        mix(_read(p))
    for k, v in params:
        mix(f"{k}={v};".encode())
    return "%016x" % h


def _with_digest(doc, digest):
    """Serialised by the library's JSON writer, as the reference CLI does
    (swapsched.cpp:114-118): sorted keys, indent 2, trailing newline."""
    return planner.with_digest(doc, digest)


def _cpp_double(x):
    """std::to_string(double) formatting (%f)."""
    return "%f" % x


def _forbid_overwrite(inputs, outputs):
    for o in outputs:
        for i in inputs:
            if os.path.exists(o) and os.path.realpath(o) == os.path.realpath(i):
                raise CliError(1, f"output would overwrite input {i}")


def _map_planner_error(e):
    code = e.code if e.code in (1, 2, 3) else 3
    return CliError(code, str(e))


def cmd_validate(a):
    inputs = [a.network] + ([a.hardware] if a.hardware else [])
    for p in inputs:
        _read(p)
    rc, report = planner.validate(_text(a.network))
    for line in (report or "").splitlines():
        print(line if rc == 0 else f"diagnostic: {line}")
    return 1 if rc == 1 else 0


def cmd_fit(a):
    inputs = [a.network] + list(a.profiles) + ([a.hardware] if a.hardware else [])
    _forbid_overwrite(inputs, [a.out])
    digest = manifest_digest("fit", inputs, [("eta", _cpp_double(a.eta))])
    model = planner.fit(_text(a.network), [_text(p) for p in a.profiles],
                        _text(a.hardware) if a.hardware else None, eta=a.eta)
    _write(a.out, _with_digest(model, digest))
    m = json.loads(model)
    print("bandwidth_avail: %.3e bytes/s" % m.get("bandwidth_avail_bytes_per_s", 0.0))
    return 0


def cmd_plan(a):
    inputs = [a.network, a.hardware, a.model]
    _forbid_overwrite(inputs, [a.out])
    params = [("step", str(a.step)), ("k", str(a.k)), ("epochs", str(a.epochs)),
              ("dataset_size", str(a.dataset_size))]
    if a.budget_bytes:
        params.append(("budget", str(a.budget_bytes)))
    digest = manifest_digest("plan", inputs, params)
    try:
        doc = planner.plan(_text(a.network), _text(a.hardware), _text(a.model), step=a.step,
                           k_override=a.k, epochs=a.epochs, dataset_size=a.dataset_size,
                           budget_override=a.budget_bytes)
    except planner.PlannerError as e:
        if e.code == 1:
            status = "infeasible"
            try:
                status = json.loads(e.document).get("status", status)
            except (TypeError, ValueError):
                pass
            print(f"{status}: {e.message}")
            return 1
        raise _map_planner_error(e)
    _write(a.out, _with_digest(doc, digest))
    p = json.loads(doc)
    print(f"k_star: {p['k_star']}")
    print(f"pinned: {len(p.get('pinned_objects', []))} featuremaps")
    print("predicted_iter_time_s: %.6f" % p.get("predicted_iter_time_s", 0.0))
    return 0


def _write_sim_outputs(out_dir, r, digest):
    """write_sim_outputs (swapsched.cpp:162-170)."""
    _write(os.path.join(out_dir, "trace.csv"), r["trace"])
    _write(os.path.join(out_dir, "summary.json"), _with_digest(r["summary"], digest))
    _write(os.path.join(out_dir, "mem_curves.csv"), r["mem_curves"])
    _write(os.path.join(out_dir, "stall_bars.csv"), r["stall_bars"])


def cmd_simulate(a):
    inputs = [a.network, a.hardware, a.model] + ([a.plan] if a.plan else [])
    params = [("mode", a.mode), ("k", str(a.k)), ("tolerance", _cpp_double(a.tolerance))]
    if a.budget_bytes:
        params.append(("budget", str(a.budget_bytes)))
    outs = [os.path.join(a.out_dir, f) for f in
            ("trace.csv", "summary.json", "mem_curves.csv", "stall_bars.csv")]
    _forbid_overwrite(inputs, outs)
    digest = manifest_digest("simulate", inputs, params)
    try:
        rc, r = planner.simulate_report(_text(a.network), _text(a.hardware), _text(a.model),
                                        _text(a.plan) if a.plan else None, a.mode, a.k,
                                        budget_override=a.budget_bytes, tolerance=a.tolerance)
    except planner.PlannerError as e:
        raise _map_planner_error(e)
    _write_sim_outputs(a.out_dir, r, digest)
    s = json.loads(r["summary"])
    if s.get("oom"):
        print(f"oom: {s.get('oom_detail', '')}")
        return 1
    print("iter_time_s: %.6f" % s.get("iter_time_s", 0.0))
    print("total_stall_s: %.6f" % s.get("total_stall_s", 0.0))
    print("peak_mem_bytes: %d" % s.get("peak_mem_bytes", 0))
    if r["verify"]:
        _write(os.path.join(a.out_dir, "verify.json"), _with_digest(r["verify"], digest))
        print("verify: %s" % ("pass" if json.loads(r["verify"])["pass"] else "fail"))
    return 1 if rc == 1 else 0


def cmd_sweep(a):
    inputs = [a.network, a.hardware, a.model]
    _forbid_overwrite(inputs, [a.out])
    csv = planner.sweep(_text(a.network), _text(a.hardware), _text(a.model), list(a.k),
                        a.modes, parallel=a.parallel)
    _write(a.out, csv)
    print(f"{max(0, csv.count(chr(10)) - 1)} cells -> {a.out}")
    return 0


def cmd_tune_lr(a):
    alpha, residual, iters = planner.tune_lr(a.alpha_base, a.convexity, a.q, mu=a.mu,
                                             iters_base=a.iters_base)
    print("alpha_star: %.10g" % alpha)
    print("contraction_residual: %.6e" % residual)
    print("adjusted_iterations: %d" % iters)
    return 0


def cmd_gen(a):
    fx = planner.generate_fixture(a.seed, a.min_layers, a.max_layers)
    _write(os.path.join(a.out_dir, "network.json"), fx["network"])
    _write(os.path.join(a.out_dir, "hardware.json"), fx["hardware"])
    _write(os.path.join(a.out_dir, "compute_profile.csv"), fx["compute_csv"])
    _write(os.path.join(a.out_dir, "transfer_profile.csv"), fx["transfer_csv"])
    n = json.loads(fx["network"])
    print(f"wrote fixture ({n['num_layers']} layers, k_base {n['k_base']}) to {a.out_dir}")
    return 0


def cmd_pipeline(a):
    """validate -> fit -> plan -> simulate -> verify under one manifest digest
    (run_pipeline, swapsched.cpp:458-533)."""
    inputs = [a.network, a.hardware] + list(a.profiles)
    names = ("model.json", "plan.json", "trace.csv", "summary.json", "mem_curves.csv",
             "stall_bars.csv", "verify.json")
    _forbid_overwrite(inputs, [os.path.join(a.out_dir, f) for f in names])
    digest = manifest_digest("pipeline", inputs, [("eta", _cpp_double(a.eta)),
                                                 ("tolerance", _cpp_double(a.tolerance))])
    net, hw = _text(a.network), _text(a.hardware)
    rc, report = planner.validate(net)
    if rc == 1:
        for line in (report or "").splitlines():
            print(f"diagnostic: {line}")
        return 1
    print("validate: ok")
    model = planner.fit(net, [_text(p) for p in a.profiles], hw, eta=a.eta)
    _write(os.path.join(a.out_dir, "model.json"), _with_digest(model, digest))
    m = json.loads(model)
    print("fit: %d curves, bandwidth %.3e B/s" % (len(m.get("curves", [])),
                                                   m.get("bandwidth_avail_bytes_per_s", 0.0)))
    try:
        plan = planner.plan(net, hw, model)
    except planner.PlannerError as e:
        if e.code == 1:
            print(f"plan: {e.message}")
            return 1
        raise _map_planner_error(e)
    _write(os.path.join(a.out_dir, "plan.json"), _with_digest(plan, digest))
    p = json.loads(plan)
    print(f"plan: k_star {p['k_star']}, {len(p.get('pinned_objects', []))} pinned")
    rc, r = planner.simulate_report(net, hw, model, plan, "dynamic", 0, tolerance=a.tolerance)
    _write_sim_outputs(a.out_dir, r, digest)
    s = json.loads(r["summary"])
    if s.get("oom"):
        print(f"simulate: oom ({s.get('oom_detail', '')})")
        return 1
    print("simulate: iter %.6f s, stall %.6f s" % (s.get("iter_time_s", 0.0),
                                                   s.get("total_stall_s", 0.0)))
    _write(os.path.join(a.out_dir, "verify.json"), _with_digest(r["verify"], digest))
    ok = json.loads(r["verify"])["pass"]
    print("verify: %s" % ("pass" if ok else "fail"))
    return 0 if ok else 1


def cmd_export(a):
    from . import trainer
    net, desc = trainer.export_network(a.arch, a.image, a.classes, k_base=a.k_base)
    _write(a.out, net)
    if a.hardware_out:
        hw = trainer.hardware_json(int(a.cap_gib * (1 << 30)),
                                   trainer.default_m_others(desc, a.image, int(a.cap_gib * (1 << 30))),
                                   a.pcie_gbs * 1e9)
        _write(a.hardware_out, hw)
    print(f"exported {a.arch}@{a.image}: {len(desc['ops'])} layers -> {a.out}")
    return 0


def cmd_execute(a):
    import numpy as np
    from . import trainer
    plan_json = _text(a.plan)
    k = json.loads(plan_json)["k_star"]
    _, desc = trainer.export_network(a.arch, a.image, a.classes)
    ex = trainer.Executor(a.arch, a.image, a.classes, mode=a.mode, plan_json=plan_json,
                          network_json=_text(a.network), hardware_json=_text(a.hardware))
    ex.set_params(trainer.init_params(desc, seed=a.seed))
    g = np.random.default_rng(a.seed)
    x = g.standard_normal((k, 3, a.image, a.image)).astype(np.float32)
    y = g.integers(0, a.classes, size=k).astype(np.int32)
    for _ in range(a.warmup):
        ex.step(x, y, lr=0.0, update=False)
    st = ex.step(x, y, lr=0.0, update=False, profile=True)
    arena, fixed = ex.memory()
    _write(os.path.join(a.out_dir, "trace.csv"), ex.trace())
    summary = {"format_version": 1, "k": k, "mode": a.mode, "iter_time_s": st["iter_ms"] * 1e-3,
               "exposed_swap_s": st["exposed_swap_ms"] * 1e-3,
               "swapped_bytes": st["swapped_bytes"], "peak_device_bytes": arena + fixed,
               "loss": st["loss"]}
    _write(os.path.join(a.out_dir, "summary.json"), json.dumps(summary, indent=2) + "\n")
    print("iter_time_s: %.6f" % summary["iter_time_s"])
    print("exposed_swap_s: %.6f" % summary["exposed_swap_s"])
    print(f"peak_device_bytes: {summary['peak_device_bytes']}")
    return 0


def build_parser():
    ap = argparse.ArgumentParser(prog="swapsched-b200", description=(
        "planner and discrete-event simulator for memory-swap schedules in DNN training "
        "(B200 build)"))
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("validate")
    p.add_argument("--network", required=True)
    p.add_argument("--hardware")
    p = sub.add_parser("fit")
    p.add_argument("--network", required=True)
    p.add_argument("--profiles", nargs="+", required=True)
    p.add_argument("--hardware")
    p.add_argument("--eta", type=float, default=0.95)
    p.add_argument("--out", default="out.json")
    p = sub.add_parser("plan")
    for f in ("--network", "--hardware", "--model"):
        p.add_argument(f, required=True)
    p.add_argument("--budget-bytes", type=int, default=0)
    p.add_argument("--step", type=int, default=1)
    p.add_argument("--k", type=int, default=0)
    p.add_argument("--epochs", type=int, default=1)
    p.add_argument("--dataset-size", type=int, default=0)
    p.add_argument("--out", default="out.json")
    p = sub.add_parser("simulate")
    for f in ("--network", "--hardware", "--model"):
        p.add_argument(f, required=True)
    p.add_argument("--plan")
    p.add_argument("--mode", default="naive")
    p.add_argument("--k", type=int, default=0)
    p.add_argument("--budget-bytes", type=int, default=0)
    p.add_argument("--tolerance", type=float, default=0.02)
    p.add_argument("--out-dir", default="out")
    p = sub.add_parser("sweep")
    for f in ("--network", "--hardware", "--model"):
        p.add_argument(f, required=True)
    p.add_argument("--k", type=int, nargs="+", required=True)
    p.add_argument("--modes", default="naive,dynamic,resident")
    p.add_argument("--parallel", action="store_true")
    p.add_argument("--epochs", type=int, default=1)
    p.add_argument("--dataset-size", type=int, default=0)
    p.add_argument("--out", default="out.json")
    p = sub.add_parser("tune-lr")
    p.add_argument("--alpha-base", type=float, required=True)
    p.add_argument("--convexity", type=float, required=True)
    p.add_argument("--mu", type=float, default=1.0)
    p.add_argument("--q", type=float, required=True)
    p.add_argument("--iters-base", type=int, default=1000)
    p = sub.add_parser("gen")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--min-layers", type=int, default=0)
    p.add_argument("--max-layers", type=int, default=0)
    p.add_argument("--out-dir", default="out")
    p = sub.add_parser("pipeline")
    p.add_argument("--network", required=True)
    p.add_argument("--hardware", required=True)
    p.add_argument("--profiles", nargs="+", required=True)
    p.add_argument("--eta", type=float, default=0.95)
    p.add_argument("--tolerance", type=float, default=0.02)
    p.add_argument("--out-dir", default="out")
    p = sub.add_parser("export")
    p.add_argument("--arch", default="resnet152")
    p.add_argument("--image", type=int, default=224)
    p.add_argument("--classes", type=int, default=1000)
    p.add_argument("--k-base", type=int, default=8)
    p.add_argument("--out", default="network.json")
    p.add_argument("--hardware-out")
    p.add_argument("--cap-gib", type=float, default=8.0)
    p.add_argument("--pcie-gbs", type=float, default=56.0)
    p = sub.add_parser("execute")
    for f in ("--network", "--hardware", "--plan"):
        p.add_argument(f, required=True)
    p.add_argument("--arch", default="resnet152")
    p.add_argument("--image", type=int, default=224)
    p.add_argument("--classes", type=int, default=1000)
    p.add_argument("--mode", default="dynamic")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--out-dir", default="out")
    return ap


COMMANDS = {"validate": cmd_validate, "fit": cmd_fit, "plan": cmd_plan,
            "simulate": cmd_simulate, "sweep": cmd_sweep, "tune-lr": cmd_tune_lr,
            "gen": cmd_gen, "pipeline": cmd_pipeline, "export": cmd_export,
            "execute": cmd_execute}


def main(argv=None):
    a = build_parser().parse_args(argv)
    try:
        return COMMANDS[a.cmd](a)
    except CliError as e:
        print(f"[error] {e}", file=sys.stderr)
        return e.code
    except planner.PlannerError as e:
        err = _map_planner_error(e)
        print(f"[error] {err}", file=sys.stderr)
        return err.code
    except Exception as e:  # internal invariant breach
        print(f"[error] internal error: {e}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
