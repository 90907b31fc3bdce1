"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv --log-file x.csv`):
launches, total us and share per kernel (template arguments kept, parameters dropped).
usage: python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import OrderedDict


def short(name):
    name = name.replace("void ", "").replace("unnamed>::", "").replace("(anonymous namespace)::", "")
    depth, out = 0, []
    for ch in name:  # cut the parameter list: the first '(' outside template brackets
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            break
        out.append(ch)
    return "".join(out).strip()


def main(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    kn, mn, mv, mu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), \
        h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[mn] != "gpu__time_duration.sum":
            continue
        us = float(r[mv].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                               "nsecond": 1e-3, "msecond": 1e3}[r[mu]]
        k = short(r[kn])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    tot = sum(t for _, t in agg.values())
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f} % |")
    print(f"\ntotal {tot / 1e3:.2f} ms over the captured step, "
          f"{sum(n for n, _ in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
