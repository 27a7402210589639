"""Measure the on-chip peaks once per pod (BASELINE.md §2 asks for L2, TF32 and
FP64): shared-memory and L2 bandwidth, FP64 issue rates and barrier latencies
from tools/onchip_peaks.cu, plus cuBLAS TF32 and FP64 GEMM throughput through
torch.  Writes one JSON object (stdout, and --out).

    python tools/onchip_peaks.py --out profiles/r02_onchip_peaks.json
"""

from __future__ import annotations

import argparse
import json
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent


def gemm_tflops(dtype, n, tf32=False, reps=10):
    import torch

    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    del c
    torch.backends.cuda.matmul.allow_tf32 = False
    return 2 * n ** 3 / best / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    exe = Path("/tmp/onchip_peaks")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", str(exe),
                    str(REPO / "tools" / "onchip_peaks.cu")], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, check=True)
    res = json.loads(r.stdout.strip().splitlines()[-1])
    res["tf32_cublas_TFLOPs"] = gemm_tflops(__import__("torch").float32, 8192, tf32=True)
    res["fp64_cublas_TFLOPs"] = gemm_tflops(__import__("torch").float64, 4096)
    res["how"] = ("tools/onchip_peaks.cu: LDS.128 on every SM (128 KiB smem, 1024 threads), ld.global.cg over a "
                  "32 MiB L2-resident buffer x20, 2 GiB streamed read, DADD/DMUL with 8 independent chains, "
                  "cooperative grid barrier (acq_rel atomic + acquire poll, 144 CTAs x 512 threads) and 16-CTA "
                  "cluster barrier, best of 5 (CUDA events); cuBLAS via torch: fp32 8192^3 with TF32 allowed, "
                  "fp64 4096^3, best of 10")
    res["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    try:
        q = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm", "--format=csv,noheader"],
                           capture_output=True, text=True).stdout.strip()
        res["gpu"] = q
    except OSError:
        pass
    line = json.dumps(res)
    print(line)
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    sys.exit(main())
