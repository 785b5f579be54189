"""Summarise an `ncu --set full` report: per launch duration, DRAM bytes and
achieved HBM GB/s, L2 bytes, and the tensor-pipe utilisation columns.

Usage: python scripts/ncu_summary.py REPORT.ncu-rep [HBM_PEAK_GBPS]
(needs the ncu CLI; reads `ncu -i REPORT --page raw --csv`).
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys


def main() -> None:
    rep = sys.argv[1]
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6549.1
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}

    def get(r, name, scale=1.0):
        i = col.get(name)
        if i is None or r[i] in ("", "n/a"):
            return None
        v = float(r[i].replace(",", ""))
        u = units[i]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
                "msecond": 1e3}.get(u, 1.0)
        return v * mult * scale

    tensor_cols = [h for h in head if h == "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
    print(f"| # | kernel | grid | us | DRAM read MB | DRAM write MB | HBM GB/s | % of {peak:.0f} GB/s "
          f"| L2 hit % | L2 thru % | SM thru % | tensor pipe % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for n, r in enumerate(data):
        name = r[col["Kernel Name"]].split("(")[0].replace("tgb::<unnamed>::", "").replace("tgb::", "").replace("unnamed>::", "")
        grid = r[col["Grid Size"]] if "Grid Size" in col else ""
        us = get(r, "gpu__time_duration.sum")
        rd = get(r, "dram__bytes_read.sum") or 0.0
        wr = get(r, "dram__bytes_write.sum") or 0.0
        hit = get(r, "lts__t_sector_hit_rate.pct")
        l2t = get(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed")
        smt = get(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed")
        tens = [get(r, h) for h in tensor_cols]
        tens = max([t for t in tens if t is not None], default=None)
        gbs = (rd + wr) / (us * 1e-6) / 1e9 if us else 0.0
        print(f"| {n} | {name} | {grid} | {us:.1f} | {rd / 1e6:.2f} | {wr / 1e6:.2f} | {gbs:.0f} | "
              f"{100 * gbs / peak:.1f} | "
              f"{'' if hit is None else f'{hit:.1f}'} | {'' if l2t is None else f'{l2t:.1f}'} | "
              f"{'' if smt is None else f'{smt:.1f}'} | {'' if tens is None else f'{tens:.1f}'} |")
    if tensor_cols:
        print(f"\ntensor-pipe column(s): {', '.join(tensor_cols)}")


if __name__ == "__main__":
    main()
