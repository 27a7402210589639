"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.

Usage: python tools/launch_summary.py launches.csv [--last N]
--last N keeps only the last N launches (one bench step is the tail of the run).
"""
import csv
import re
import sys
from collections import OrderedDict


def load(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
        rows.append((int(r["ID"]), re.sub(r"\(.*", "", r["Kernel Name"]), v * scale))
    return rows


def main():
    path = sys.argv[1]
    last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else None
    rows = load(path)
    if last:
        rows = rows[-last:]
    agg = OrderedDict()
    for _, k, us in rows:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':60s} {'n':>6s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:6d} {us:10.1f} {us / n:9.1f} {us / tot:6.1%}")
    print(f"{'total':60s} {sum(a[0] for a in agg.values()):6d} {tot:10.1f}")


if __name__ == "__main__":
    main()
