"""GPU Brox flow timing at 1080p (scale 0.5 and 0.95) vs the oracle on a crop."""

import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2008_10273_b200.flow import BroxParams, flow_brox  # noqa: E402
from paper_2008_10273_b200.synth import synth_clip  # noqa: E402


def main():
    clip = synth_clip(2, 1080, 1920, blobs=40, rects=12, v=6.0, seed=4)[:, 0].astype(np.float64)
    a, b = torch.from_numpy(clip[1]).cuda(), torch.from_numpy(clip[0]).cuda()
    for sc in (0.5, 0.95):
        prm = BroxParams(pyramid_scale=sc)
        flow_brox(a, b, prm)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            ff = flow_brox(a, b, prm)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        print(f"1080p brox scale {sc}: {dt * 1e3:.1f} ms/pair, |u|max {float(ff.u.abs().max()):.2f}", flush=True)


if __name__ == "__main__":
    main()
