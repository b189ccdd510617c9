"""Per-kernel share of one profiled step from an ncu launch list
(--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum,...] --csv).
Usage: summarize_launches.py launches.csv [json_out]"""
import collections
import csv
import json
import sys


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "").replace("accudnn::", "")
    for cut in ("(CUtensorMap", "(const", "(float", "(int", "(unnamed", "(Args", "(BnArgs", "(Prob"):
        name = name.split(cut)[0]
    return name.strip()


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, mi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        rec = launches.setdefault(r[ii], {"name": short(r[ki])})
        rec[r[mi]] = float(r[vi].replace(",", ""))
    return list(launches.values())


def main(path, out=None):
    ls = load(path)
    agg = collections.defaultdict(lambda: collections.Counter())
    for l in ls:
        a = agg[l["name"]]
        a["n"] += 1
        a["ns"] += l.get("gpu__time_duration.sum", 0)
        a["dram"] += l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
    tot = sum(a["ns"] for a in agg.values())
    has_dram = any(a["dram"] for a in agg.values())
    print("| kernel | launches | ms (ncu, serialised) | share |" + (" DRAM MB/launch |" if has_dram else ""))
    print("|---|---|---|---|" + ("---|" if has_dram else ""))
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ns"])[:30]:
        line = f"| `{k[:60]}` | {a['n']} | {a['ns'] / 1e6:.3f} | {100 * a['ns'] / tot:.1f}% |"
        if has_dram:
            line += f" {a['dram'] / a['n'] / 1e6:.2f} |"
        print(line)
    print(f"| **total** | {sum(a['n'] for a in agg.values())} | {tot / 1e6:.3f} | 100% |")
    if out:
        json.dump({k: {"launches": a["n"], "ms": a["ns"] / 1e6, "dram_bytes": a["dram"]}
                   for k, a in agg.items()}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
