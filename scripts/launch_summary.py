"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X.csv ...`) into one barrier's launches and per-kernel shares.

A barrier is cut out as the launches from one `select_args_kernel` (the first
kernel of a graph-mode barrier) to the next one. Usage:
  python scripts/launch_summary.py launches.csv [barrier_index] > summary.md
"""
from __future__ import annotations

import csv
import sys
from collections import OrderedDict


def main() -> None:
    path = sys.argv[1]
    which = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(lines)
    head = next(rd)
    col = {h: i for i, h in enumerate(head)}
    for r in rd:
        if r[col["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[col["Metric Value"]].replace(",", ""))
        unit = r[col["Metric Unit"]]
        us = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        name = r[col["Kernel Name"]].split("(")[0].replace("tgb::<unnamed>::", "").replace("(anonymous namespace)::", "")
        rows.append((int(r[col["ID"]]), name, r[col["Grid Size"]], us))
    starts = [i for i, r in enumerate(rows) if r[1].startswith("select_args_kernel")]
    if len(starts) < which + 2:
        raise SystemExit(f"only {len(starts)} barrier starts in the list")
    bar = rows[starts[which]:starts[which + 1]]
    total = sum(r[3] for r in bar)
    print(f"barrier {which}: {total:.1f} us serialised over {len(bar)} kernel launches\n")
    print("| # | kernel | grid | us | share |\n|---|---|---|---|---|")
    for n, r in enumerate(bar):
        print(f"| {n} | {r[1][:60]} | {r[2]} | {r[3]:.1f} | {100 * r[3] / total:.1f}% |")
    agg: "OrderedDict[str, list]" = OrderedDict()
    for r in bar:
        a = agg.setdefault(r[1][:60], [0.0, 0])
        a[0] += r[3]
        a[1] += 1
    print("\nAggregated:\n\n| kernel | launches | us | share |\n|---|---|---|---|")
    for k, (us, n) in sorted(agg.items(), key=lambda t: -t[1][0]):
        print(f"| {k} | {n} | {us:.1f} | {100 * us / total:.1f}% |")


if __name__ == "__main__":
    main()
