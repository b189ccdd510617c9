"""Runs the B200 profiler for the BASELINE configs and writes the reference
format profile CSVs + host-link bandwidths under profiles/b200/ (committed;
bench.py fits the performance model from them)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1901_06773_b200 import profiler, trainer  # noqa: E402

CONFIGS = {
    "resnet152": (224, 1000, 32),
    "resnet50": (224, 1000, 48),
    # grid 8, 16, 32, 43, 64: config 1 runs at k = 8 (k_override), inside it
    "resnet20": (32, 12, 64),
    "resnet1001": (32, 12, 32),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--archs", default="resnet152,resnet50")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "b200"))
    ap.add_argument("--k-base", type=int, default=8)
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    bw = profiler.host_link_bandwidth()
    with open(os.path.join(args.out, "host_link.json"), "w") as f:
        json.dump({k: round(v, 2) for k, v in bw.items()}, f, indent=1)
    print("host link GB/s", bw, flush=True)
    for arch in args.archs.split(","):
        image, classes, k_ref = CONFIGS[arch]
        net_json, _ = trainer.export_network(arch, image, classes, k_base=args.k_base)
        ks = profiler.grid(k_ref)
        t0 = time.time()
        comp = profiler.profile_compute(arch, image, classes, net_json, ks)
        tran = profiler.profile_transfer(net_json, ks)
        with open(os.path.join(args.out, f"{arch}_compute_profile.csv"), "w") as f:
            f.write(comp)
        with open(os.path.join(args.out, f"{arch}_transfer_profile.csv"), "w") as f:
            f.write(tran)
        print(arch, "grid", ks, "rows", comp.count("\n") - 1, tran.count("\n") - 1,
              "%.1fs" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    main()
