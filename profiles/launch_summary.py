"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.

usage: python profiles/launch_summary.py launches.csv [steps]
Prints per-kernel total / count / mean (ncu: cold cache, serialised launches,
so compare shares, not absolutes).
"""
import collections
import csv
import sys


def main(path, steps=1):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        name = r[ik].split("(")[0]
        for pre in ("void ", "slide::"):
            name = name.replace(pre, "")
        agg[name[:70]][0] += 1
        agg[name[:70]][1] += float(r[iv].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot / 1e3:.1f} us total")
    print(f"{'us total':>10} {'share':>6} {'n':>5} {'us mean':>9}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{v[1] / 1e3:10.1f} {100 * v[1] / tot:5.1f}% {v[0]:5d} {v[1] / 1e3 / v[0]:9.2f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
