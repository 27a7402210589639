"""One warm 1080p decode-mode solve + one config-1 solve, for ncu captures."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2008_10273_b200 import homogeneous  # noqa: E402
from paper_2008_10273_b200.synth import random_mask, synth_clip  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    plane = synth_clip(1, 1080, 1920, blobs=40, rects=12, v=6.0, seed=1)[0, 0].astype(np.float64)
    for dens, tol, mi, strict in [(0.04, 1e-4, 160, False), (0.02, 1e-6, 10000, True)]:
        m = random_mask(plane.shape, dens, 1001)
        f = torch.from_numpy(np.where(m, plane, 0.0)).cuda()
        mt = torch.from_numpy(m).cuda()
        for _ in range(reps):
            st = {}
            homogeneous.solve_homogeneous(f, mt, tol=tol, max_iter=mi, strict=strict, stats=st)
        torch.cuda.synchronize()
        print(dens, st["level_iterations"])


if __name__ == "__main__":
    main()
