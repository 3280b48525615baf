"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel name.

  python tools/summarize_launches.py gpurun_out/launches.csv > profiles/r01_launches.md
The per-launch times are cold-cache and serialised (ncu), so compare SHARES, not absolutes.
"""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    name = name.replace("mls::", "").replace("(anonymous namespace)::", "")
    return name.strip()


def main(path):
    rows = list(csv.reader(open(path)))
    # find header
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    kn, mn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        v = float(r[mv].replace(",", ""))
        unit = r[mu]
        us = v / 1e3 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1e3)
        k = short(r[kn])
        agg[k][0] += 1
        agg[k][1] += us
        total += us
    print(f"# ncu launch list summary ({path})\n")
    print(f"total {sum(a[0] for a in agg.values())} launches, {total/1e3:.2f} ms (cold-cache, serialised)\n")
    print("| kernel | launches | total ms | share | mean us |")
    print("|---|---|---|---|---|")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {us/1e3:.2f} | {100*us/total:.1f}% | {us/n:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
