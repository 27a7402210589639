"""Time codec.encode on one config-3 GOP (12 frames, 1080p Y or 540p Cb/Cr) and
compare its bytes with the reference encoder's GOP payload (tests/golden/streams).

    python tools/encode_probe.py [--plane Y] [--gops 1] [--repeat 2]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plane", default="Y")
    ap.add_argument("--gops", type=int, default=1)
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    import torch

    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.bitstream import read_stream
    from paper_2008_10273_b200.frame import Frame
    from paper_2008_10273_b200.synth import synth_420

    t0 = time.perf_counter()
    y, cb, cr = synth_420(12 * a.gops, 1080, 1920, blobs=40, rects=12, v=6.0, seed=3)
    planes = {"Y": y, "Cb": cb, "Cr": cr}[a.plane]
    print(f"synth {time.perf_counter() - t0:.1f}s", flush=True)
    ref = read_stream((REPO / "tests/golden/streams" / f"cfg3_{a.plane}.hivc").read_bytes())[1]
    frames = [Frame((p,), colorspace="gray") for p in planes]
    cfg = codec.EncoderConfig(gop_size=12)
    for r in range(a.repeat):
        tim = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        stream = codec.encode(frames, cfg, timings=tim)
        dt = time.perf_counter() - t0
        got = read_stream(stream)[1]
        same = [g == ref[i] for i, g in enumerate(got)]
        print(json.dumps({"repeat": r, "seconds": round(dt, 3), "fps": round(len(frames) / dt, 2),
                          "gop_bytes_equal": same, "bytes": len(stream),
                          "stages": {k: round(v, 3) for k, v in sorted(tim.items(), key=lambda kv: -kv[1])}}),
              flush=True)


if __name__ == "__main__":
    main()
