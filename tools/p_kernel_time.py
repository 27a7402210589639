"""Mean ncu launch duration of the P-frame kernels of a config-3 bench step, per plane size.
Usage: ncu --metrics gpu__time_duration.sum,launch__grid_size -k regex:frame_kernel --csv \
          --log-file gpurun_out/pk.csv python bench.py --steps 1 --warmup 1 --no-cpu
       python tools/p_kernel_time.py gpurun_out/pk.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.DictReader(ln for ln in open(sys.argv[1]) if ln.startswith('"'))]
by = defaultdict(dict)
for r in rows:
    by[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
acc = defaultdict(list)
for (i, name), m in by.items():
    kind = "P" if "(bool)1" in name or "<1," in name or "<true" in name else "I"
    acc[(kind, int(m.get("launch__grid_size", 0)))].append(m["gpu__time_duration.sum"] / 1e3)
for k, v in sorted(acc.items()):
    print(f"{k[0]} grid {k[1]:6d}: {len(v):4d} launches, mean {sum(v) / len(v):7.2f} us, min {min(v):7.2f}")
