"""Generates tests/golden/*.json from the compiled REFERENCE planner
(oracle/_ref/libswapsched_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Test infrastructure: run here, commit the outputs; the
tests then pin the B200 planner against them without the reference tree.

  planner_fixtures.json  for seeds of the reference's fixture generator
                         (synthetic.cpp:170-195): the four input documents'
                         digests, model.json, plan.json, evaluate_minibatch at
                         k*, k*+1, k_max, simulate(dynamic) summary + trace
                         FNV-1a, sweep CSV
  resnet_plans.json      exported ResNet network.json + B200 profiles ->
                         per-k evaluations and small-budget full plans
  headline_plans.json    BASELINE configs 2-4 on bench.py's documents: the
                         reference's full step-1 search (plan.json) and its
                         evaluations at k* and k*+1
  resnet1001_plan.json   (--with-r1001, ~2 min) config 5: reference evaluations
                         at k* and k*+1 of ResNet-1001 under 8 GiB
"""
import ctypes
import hashlib
import json
import os
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1901_06773_b200 import _native, planner  # noqa: E402

SEEDS = [1, 5, 7, 42, 99, 3, 11, 23, 64, 77, 101, 202, 303, 404, 505, 606]


def fnv1a(data):
    h = 1469598103934665603
    for c in data:
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def t_ready_digest(ns):
    return fnv1a(struct.pack("<%dq" % len(ns), *ns))


def ref_lib():
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libswapsched_ref.so"))
    _native.declare_planner_symbols(lib, "oracle_")
    return dict(lib=lib, prefix="oracle_")


def fixture_record(seed, R):
    fx = planner.generate_fixture(seed, **R)
    model = planner.fit(fx["network"], [fx["compute_csv"], fx["transfer_csv"]], fx["hardware"], **R)
    rec = {"seed": seed,
           "docs_sha256": {k: hashlib.sha256(v.encode()).hexdigest() for k, v in fx.items()},
           "model_json": model, "k_max": planner.kmax(fx["network"], fx["hardware"], **R)}
    try:
        plan = planner.plan(fx["network"], fx["hardware"], model, **R)
        rec["plan_json"] = plan
        k = json.loads(plan)["k_star"]
        evals = {}
        for kk in sorted({1, k, k + 1, rec["k_max"]}):
            evals[str(kk)] = planner.evaluate_k(fx["network"], fx["hardware"], model, kk, **R)
        rec["evals"] = evals
        rec["t_ready_fnv1a"] = t_ready_digest(evals[str(k)]["t_ready_ns"])
        sims = {}
        for mode in ("naive", "dynamic", "resident"):
            rc, summ, trace = planner.simulate(fx["network"], fx["hardware"], model, plan, mode, k, **R)
            sims[mode] = {"rc": rc, "summary": summ, "trace_fnv1a": fnv1a(trace.encode())}
        rec["sim"] = sims
        rec["sweep_csv"] = planner.sweep(fx["network"], fx["hardware"], model,
                                         sorted({1, max(1, k // 2), k, k + 1}), **R)
    except planner.PlannerError as e:
        rec["plan_error"] = {"code": e.code, "document": e.document}
    return rec


def resnet_records(R):
    from paper_1901_06773_b200 import trainer
    out = []
    cases = [("resnet20", 32, 12, 64 << 20, "resnet20"), ("resnet50", 224, 1000, 12 << 30, "resnet50"),
             ("resnet152", 224, 1000, 8 << 30, "resnet152")]
    link = json.load(open(os.path.join(ROOT, "profiles", "b200", "host_link.json")))
    for arch, image, classes, budget, prof in cases:
        net, desc = trainer.export_network(arch, image, classes, k_base=8)
        hw = trainer.hardware_json(budget, trainer.default_m_others(desc, image), link["d2h"] * 1e9)
        pdir = os.path.join(ROOT, "profiles", "b200")
        csvs = []
        for kind in ("compute", "transfer"):
            p = os.path.join(pdir, f"{prof}_{kind}_profile.csv")
            if os.path.exists(p):
                csvs.append(open(p).read())
        if len(csvs) < 2:  # no measured profile: flat B200-like synthetic curves
            continue
        model = planner.fit(net, csvs, hw, **R)
        km = planner.kmax(net, hw, **R)
        rec = {"arch": arch, "image": image, "classes": classes, "budget": budget,
               "network_sha256": hashlib.sha256(net.encode()).hexdigest(), "model_json": model,
               "hardware_json": hw, "k_max": km, "evals": {}}
        for kk in (1, 8, 16, 24, 27, 32, 48, 64):
            if kk <= km:
                rec["evals"][str(kk)] = planner.evaluate_k(net, hw, model, kk, **R)
        if arch == "resnet20":
            rec["plan_json"] = planner.plan(net, hw, model, **R)
        out.append(rec)
    return out


def resnet1001_record(R):
    """BASELINE config 5 (ResNet-1001 @32, 8 GiB): the reference's
    evaluate_minibatch at k* = 41 and k* + 1 (~48 s each on one core; the
    reference's full k_max = 32,136 scan does not finish)."""
    from paper_1901_06773_b200 import trainer
    net, desc = trainer.export_network("resnet1001", 32, 12, k_base=8)
    link = json.load(open(os.path.join(ROOT, "profiles", "b200", "host_link.json")))
    hw = trainer.hardware_json(8 << 30, trainer.default_m_others(desc, 32), link["d2h"] * 1e9)
    pdir = os.path.join(ROOT, "profiles", "b200")
    csvs = [open(os.path.join(pdir, f"resnet1001_{k}_profile.csv")).read()
            for k in ("compute", "transfer")]
    model = planner.fit(net, csvs, hw, eta=0.95, **R)
    rec = {"arch": "resnet1001", "image": 32, "classes": 12, "budget": 8 << 30,
           "network_sha256": hashlib.sha256(net.encode()).hexdigest(), "model_json": model,
           "hardware_json": hw, "k_max": planner.kmax(net, hw, **R), "evals": {}}
    for k in (41, 42):
        rec["evals"][str(k)] = planner.evaluate_k(net, hw, model, k, **R)
    return rec


HEADLINE = [("resnet152", 224, 1000, 8 << 30),    # BASELINE config 3 (the bench line)
            ("resnet50", 224, 1000, 12 << 30),    # config 2
            ("resnet152", 224, 1000, 12 << 30)]   # config 4 (per GPU)


def headline_records(R):
    """Full Algorithm-2 searches of the reference (step = 1, planner.cpp:346-424)
    on exactly the documents bench.py builds (trainer.config_documents), plus
    its evaluations at k* and k*+1 (maximality)."""
    import time
    from paper_1901_06773_b200 import trainer
    out = []
    for arch, image, classes, cap in HEADLINE:
        net, hw, model_ours, desc = trainer.config_documents(arch, image, classes, cap)
        # the documents themselves, so the reference arm of bench.py can plan,
        # simulate and run the CPU step without loading any product library
        ddir = os.path.join(HERE, "headline_docs")
        os.makedirs(ddir, exist_ok=True)
        stem = os.path.join(ddir, f"{arch}_{image}_{cap >> 30}GiB")
        for ext, text in (("network", net), ("hardware", hw), ("model", model_ours),
                          ("describe", json.dumps(desc, indent=0))):
            with open(f"{stem}.{ext}.json", "w") as f:
                f.write(text)
        pdir = os.path.join(ROOT, "profiles", "b200")
        csvs = [open(os.path.join(pdir, f"{arch}_{k}_profile.csv")).read()
                for k in ("compute", "transfer")]
        model = planner.fit(net, csvs, hw, eta=0.95, **R)
        t0 = time.perf_counter()
        plan = planner.plan(net, hw, model, step=1, **R)
        secs = time.perf_counter() - t0
        k = json.loads(plan)["k_star"]
        rec = {"arch": arch, "image": image, "classes": classes, "cap_bytes": cap,
               "network_sha256": hashlib.sha256(net.encode()).hexdigest(),
               "hardware_json": hw, "model_json": model, "plan_json": plan,
               "k_max": planner.kmax(net, hw, **R),
               "reference_plan_seconds_step1": round(secs, 2),
               "evals": {str(kk): planner.evaluate_k(net, hw, model, kk, **R) for kk in (k, k + 1)}}
        print(arch, cap >> 30, "GiB: k* =", k, "reference step-1 search %.1f s" % secs, flush=True)
        out.append(rec)
    return out


def main():
    R = ref_lib()
    if "--headline-only" in sys.argv:
        with open(os.path.join(HERE, "headline_plans.json"), "w") as f:
            json.dump(headline_records(R), f, indent=1)
        return
    with open(os.path.join(HERE, "headline_plans.json"), "w") as f:
        json.dump(headline_records(R), f, indent=1)
    if "--with-r1001" in sys.argv:
        with open(os.path.join(HERE, "resnet1001_plan.json"), "w") as f:
            json.dump(resnet1001_record(R), f, indent=1)
    fixtures = [fixture_record(s, R) for s in SEEDS]
    with open(os.path.join(HERE, "planner_fixtures.json"), "w") as f:
        json.dump(fixtures, f, indent=1)
    with open(os.path.join(HERE, "resnet_plans.json"), "w") as f:
        json.dump(resnet_records(R), f, indent=1)
    print("wrote", len(fixtures), "fixtures")


if __name__ == "__main__":
    main()
