#!/usr/bin/env python
"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python scripts/launch_summary.py launches.csv "<header line>" > summary.txt
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    header = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    cols = rows[h]
    ki, mi, vi, ui = (cols.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0, "s": 1e3,
                 "second": 1e3}[r[ui]]
        name = r[ki].split("(")[0][:60]
        n, t = tot.get(name, (0, 0.0))
        tot[name] = (n + 1, t + float(r[vi].replace(",", "")) * scale)
    total = sum(t for _, t in tot.values())
    print(header)
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>12s} {'share':>8s}")
    for name, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:60s} {n:8d} {t:12.3f} {t / total:8.5f}")


if __name__ == "__main__":
    main()
