"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum --csv): count, total and mean
time per kernel, in first-launch order.

    python tools/launch_table.py gpurun_out/launches.csv [--md]
"""

from __future__ import annotations

import collections
import csv
import sys


def table(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ns = v * {"ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1.0}.get(unit, 1.0)
        a = agg.setdefault(r[ki], [0, 0.0])
        a[0] += 1
        a[1] += ns
    return agg


def main():
    agg = table(sys.argv[1])
    tot = sum(t for _, t in agg.values())
    md = "--md" in sys.argv
    if md:
        print("| launches | total us | mean us | share | kernel |\n|---:|---:|---:|---:|---|")
    for k, (c, t) in agg.items():
        name = k if len(k) < 90 else k[:87] + "..."
        if md:
            print(f"| {c} | {t / 1e3:.1f} | {t / c / 1e3:.1f} | {100 * t / tot:.1f}% | `{name}` |")
        else:
            print(f"{c:5d} {t / 1e3:10.1f} us  mean {t / c / 1e3:8.1f}  {100 * t / tot:5.1f}%  {name}")


if __name__ == "__main__":
    main()
