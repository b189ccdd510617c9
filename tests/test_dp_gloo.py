"""Data-parallel host logic with world_size 2 on gloo (CPU):
  * every rank plans independently and gets the identical plan (the planner
    is deterministic, so k* / the pin set need no broadcast);
  * the gradient buckets the executor all-reduces (prefixes of the flat
    buffer in reverse op order) reproduce a whole-buffer all-reduce;
  * the learning rate uses q = W * k* / k_base (Eq. 9).
"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_06773_b200 import planner, trainer


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def buckets(desc, bucket_floats):
    """prefix buckets in backward order, as executor.cu builds them"""
    n = len(desc["ops"])
    ends = []
    done = 0
    for op in reversed(desc["ops"]):
        end = -1
        if op.get("w_off", -1) >= 0:
            end = max(end, op["w_off"] + op["cout"] * op["r"] * op["r"] * op["cin"])
        if op.get("b_off", -1) >= 0:
            end = max(end, op["b_off"] + op["cout"])
        if op.get("beta_off", -1) >= 0:
            end = max(end, op["beta_off"] + op["channels"])
        done = max(done, end)
        ends.append(min(done, desc["n_params"]))
    out, start = [], 0
    for i, e in enumerate(ends):
        if e - start >= bucket_floats or (i == len(ends) - 1 and e > start):
            out.append((start, e))
            start = e
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fx = planner.generate_fixture(42)
    model = planner.fit(fx["network"], [fx["compute_csv"], fx["transfer_csv"]], fx["hardware"])
    plan = planner.plan(fx["network"], fx["hardware"], model)
    plans = [None] * world
    dist.all_gather_object(plans, plan)

    _, desc = trainer.export_network("resnet20", 32, 12)
    g = torch.from_numpy(np.random.default_rng(rank).standard_normal(desc["n_params"]).astype(np.float32))
    full = g.clone()
    dist.all_reduce(full)
    bucketed = g.clone()
    bl = buckets(desc, 16384)
    for a, b in bl:
        view = bucketed[a:b]
        dist.all_reduce(view)
    covered = sum(b - a for a, b in bl)
    k_star = json.loads(plan)["k_star"]
    lr = planner.tune_lr(0.1, 1.0, world * k_star / 8.0)[0]
    q.put((rank, plans[0] == plans[1], float((full - bucketed).abs().max()), covered,
           desc["n_params"], lr))
    dist.destroy_process_group()


def test_two_rank_plan_and_buckets():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, same_plan, diff, covered, n_params, lr in res:
        assert same_plan
        assert diff == 0.0
        assert covered == n_params or n_params - covered < 4
        assert 0.1 < lr < 1.0
    assert res[0][5] == res[1][5]


@pytest.mark.parametrize("gpus", [2, 3])
def test_bench_launcher_spawns_ranks(gpus):
    """`python bench.py --gpus N` outside torchrun re-launches itself under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous); every rank
    plans on identical documents with NCCL's allowance charged to m_others,
    and rank 0 alone prints one JSON line with n_gpus = N (--dry-run: host
    side only, gloo)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run",
                          "--gpus", str(gpus)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == gpus and rec["plans_identical_across_ranks"]
    assert rec["m_others_extra_bytes"] == 768 << 20
    assert rec["global_batch"] == gpus * rec["k_star"]
