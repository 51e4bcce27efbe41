#!/usr/bin/env python
"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv --log-file X`) as a
markdown table: per kernel name, launches, total us, share of all kernel time.

  python tools/launches_md.py gpurun_out/launches.csv "title" > profiles/rNN_launches.md
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        rows.append((r["Kernel Name"], v * scale))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for name, us in rows:
        tot[name] += us
        cnt[name] += 1
    allus = sum(tot.values())
    print(f"# ncu launch list — {title}\n")
    print("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares, "
          "not absolute times).\n")
    print(f"{len(rows)} launches, {allus:.1f} us of kernel time.\n")
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for name, us in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{name[:90]}` | {cnt[name]} | {us:.1f} | {100 * us / allus:.1f}% |")


if __name__ == "__main__":
    main()
