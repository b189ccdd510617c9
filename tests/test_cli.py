"""The swapsched-compatible CLI (paper_1901_06773_b200/cli.py): subcommands,
exit codes (0 ok, 1 validation/infeasible, 2 I/O) and documents identical to
the reference library's on the same inputs (the reference's own CLI needs
CLI11, absent here, so the comparison goes through the oracle library's C ABI
with the same manifest-digest rule, swapsched.cpp:76-91)."""
import json
import os

import pytest

from paper_1901_06773_b200 import cli, planner


def run(*argv):
    return cli.main(list(argv))


@pytest.fixture
def fixture_dir(tmp_path):
    assert run("gen", "--seed", "7", "--out-dir", str(tmp_path / "fx")) == 0
    return tmp_path


def paths(d):
    fx = d / "fx"
    return (str(fx / "network.json"), str(fx / "hardware.json"),
            str(fx / "compute_profile.csv"), str(fx / "transfer_profile.csv"))


def test_cli_end_to_end_matches_reference(fixture_dir, oracle):
    net, hw, comp, tran = paths(fixture_dir)
    model = str(fixture_dir / "model.json")
    plan = str(fixture_dir / "plan.json")
    assert run("validate", "--network", net, "--hardware", hw) == 0
    assert run("fit", "--network", net, "--profiles", comp, tran, "--hardware", hw,
               "--out", model) == 0
    assert run("plan", "--network", net, "--hardware", hw, "--model", model, "--out", plan) == 0
    assert run("simulate", "--network", net, "--hardware", hw, "--model", model, "--plan", plan,
               "--mode", "dynamic", "--out-dir", str(fixture_dir / "sim")) == 0
    assert run("sweep", "--network", net, "--hardware", hw, "--model", model, "--k", "4", "8",
               "--out", str(fixture_dir / "sweep.csv")) == 0
    # same documents from the reference library (digest excluded: it is added by the CLI)
    R = dict(lib=oracle, prefix="oracle_")
    texts = [open(p).read() for p in (net, hw, comp, tran)]
    ref_model = json.loads(planner.fit(texts[0], texts[2:], texts[1], eta=0.95, **R))
    mine_model = json.load(open(model))
    assert mine_model.pop("manifest_digest")
    assert mine_model == ref_model
    ref_plan = json.loads(planner.plan(texts[0], texts[1], json.dumps(ref_model), **R))
    mine_plan = json.load(open(plan))
    digest = mine_plan.pop("manifest_digest")
    assert mine_plan == ref_plan
    # the digest is FNV-1a over subcommand, input bytes and parameters
    assert digest == cli.manifest_digest("plan", [net, hw, model],
                                         [("step", "1"), ("k", "0"), ("epochs", "1"),
                                          ("dataset_size", "0")])


def test_cli_exit_codes(fixture_dir):
    net, hw, comp, tran = paths(fixture_dir)
    model = str(fixture_dir / "model.json")
    assert run("fit", "--network", net, "--profiles", comp, tran, "--out", model) == 0
    assert run("plan", "--network", str(fixture_dir / "missing.json"), "--hardware", hw,
               "--model", model) == 2
    assert run("plan", "--network", net, "--hardware", hw, "--model", model,
               "--budget-bytes", "1000", "--out", str(fixture_dir / "p.json")) == 1
    assert run("plan", "--network", net, "--hardware", hw, "--model", model, "--out", net) == 1
    assert run("tune-lr", "--alpha-base", "0.1", "--convexity", "1", "--q", "2") == 0


def test_cli_export_resnet(tmp_path):
    out = str(tmp_path / "net.json")
    hw = str(tmp_path / "hw.json")
    assert run("export", "--arch", "resnet50", "--out", out, "--hardware-out", hw,
               "--cap-gib", "12") == 0
    n = json.load(open(out))
    assert n["num_layers"] == len(n["layers"]) and n["k_base"] == 8
    assert json.load(open(hw))["memory_budget_bytes"] == 12 << 30
    assert run("validate", "--network", out) == 0


@pytest.mark.gpu
def test_cli_execute_on_gpu(tmp_path, cuda_dev):
    """export -> fit (committed B200 profiles) -> plan -> execute: the real
    iteration's per-phase trace and summary next to the simulator's"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prof = os.path.join(root, "profiles", "b200")
    net, hw = str(tmp_path / "net.json"), str(tmp_path / "hw.json")
    model, plan = str(tmp_path / "model.json"), str(tmp_path / "plan.json")
    assert run("export", "--arch", "resnet20", "--image", "32", "--classes", "12", "--out", net,
               "--hardware-out", hw, "--cap-gib", "0.25") == 0
    assert run("fit", "--network", net, "--profiles", os.path.join(prof, "resnet20_compute_profile.csv"),
               os.path.join(prof, "resnet20_transfer_profile.csv"), "--hardware", hw,
               "--out", model) == 0
    assert run("plan", "--network", net, "--hardware", hw, "--model", model, "--k", "16",
               "--out", plan) == 0
    out = tmp_path / "exec"
    assert run("execute", "--network", net, "--hardware", hw, "--plan", plan, "--arch", "resnet20",
               "--image", "32", "--classes", "12", "--out-dir", str(out)) == 0
    s = json.load(open(out / "summary.json"))
    assert s["k"] == 16 and s["iter_time_s"] > 0 and s["peak_device_bytes"] <= 0.25 * (1 << 30)
    rows = open(out / "trace.csv").read().strip().splitlines()
    assert len(rows) == 1 + 2 * json.load(open(net))["num_layers"]


def test_plan_cache_keyed_by_manifest_digest(fixture_dir):
    net, hw, comp, tran = (open(p).read() for p in paths(fixture_dir))
    model = planner.fit(net, [comp, tran], hw)
    cache = str(fixture_dir / "cache")
    p1, hit1 = planner.plan_cached(net, hw, model, cache)
    p2, hit2 = planner.plan_cached(net, hw, model, cache)
    assert (hit1, hit2) == (False, True) and p1 == p2 == planner.plan(net, hw, model)
    p3, hit3 = planner.plan_cached(net, hw, model, cache, k_override=4)
    assert not hit3 and json.loads(p3)["k_star"] == 4
    # the key is the manifest digest of a `plan` run on files with these bytes
    for name, text in (("n.json", net), ("h.json", hw), ("m.json", model)):
        (fixture_dir / name).write_text(text)
    d = cli.manifest_digest("plan", [str(fixture_dir / n) for n in ("n.json", "h.json", "m.json")],
                            [("step", "1"), ("k", "0"), ("epochs", "1"), ("dataset_size", "0")])
    assert os.path.exists(os.path.join(cache, f"plan-{d}.json"))
