"""Per-kernel averages of an ncu --metrics capture of bench.py's own launches.

    ncu --metrics <METRICS> -k regex:"cg_tile|cg_cluster|frame_kernel|restrict" \\
        --clock-control none --csv --log-file cap.csv python bench.py --steps 1 --warmup 3 --no-cpu
    python tools/ncu_kernel_summary.py cap.csv --out profiles/r02_kernel_metrics.json

Writes, per kernel (template arguments kept, so the P-frame and I-frame
variants of frame_kernel are separate rows): the launch count and the mean
per launch of every captured metric.  bench.py reads the file for the
`traffic` of each roofline row (DRAM, L2 and shared-memory bytes measured
on its own launches); the durations here are serialised ncu replays, so
bench.py takes the dominant kernel's time from its own live timing.
"""

from __future__ import annotations

import argparse
import collections
import csv
import json
import re
import time

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
]

SCALE = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name.replace("void ", "").replace("hivc::", ""))
    return name.strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out")
    ap.add_argument("--command", default="")
    args = ap.parse_args()
    lines = [ln for ln in open(args.csv) if ln.startswith('"')]
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    launches = collections.defaultdict(set)
    for r in csv.DictReader(lines):
        k = short(r["Kernel Name"])
        unit = r.get("Metric Unit", "") or ""
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(unit, 1.0)
        per[k][r["Metric Name"]].append(v)
        launches[k].add(r["ID"])
    out = {"source": args.csv, "command": args.command, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "units": "per launch: duration ns, bytes, counts; wavefront = one shared-memory pipe cycle (<= 128 B)",
           "kernels": {}}
    for k, m in per.items():
        row = {"launches": len(launches[k])}
        for name, vals in m.items():
            row[name] = sum(vals) / len(vals)
        dram = row.get("dram__bytes_read.sum", 0) + row.get("dram__bytes_write.sum", 0)
        row["dram_bytes"] = dram
        row["smem_bytes_upper"] = 128.0 * row.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0)
        out["kernels"][k] = row
    text = json.dumps(out, indent=1)
    if args.out:
        open(args.out, "w").write(text + "\n")
    for k, row in sorted(out["kernels"].items(), key=lambda kv: -kv[1]["launches"] * kv[1].get("gpu__time_duration.sum", 0)):
        print(f"{k[:60]:60s} n={row['launches']:5d} t={row.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us "
              f"dram={row['dram_bytes'] / 1e6:8.2f} MB l2={row.get('lts__t_bytes.sum', 0) / 1e6:8.2f} MB "
              f"smem<={row['smem_bytes_upper'] / 1e6:8.2f} MB")


if __name__ == "__main__":
    main()
