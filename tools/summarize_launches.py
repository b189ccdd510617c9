"""Per-kernel share of one profiled step from an ncu launch list
(--metrics gpu__time_duration.sum --csv).  Usage: summarize_launches.py launches.csv"""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        name = name.split("(CUtensorMap")[0].split("(const")[0].split("(float")[0].split("(int")[0]
        name = name.split("(unnamed")[0].split("(Args")[0]
        v = float(r[vi].replace(",", ""))
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print(f"| kernel | launches | ms (ncu, serialised) | share |\n|---|---|---|---|")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"| `{k[:70]}` | {c} | {v / 1e6:.3f} | {100 * v / tot:.1f}% |")
    print(f"| **total** | {sum(c for c, _ in agg.values())} | {tot / 1e6:.3f} | 100% |")


if __name__ == "__main__":
    main(sys.argv[1])
