"""Ad-hoc GPU timings used while developing (not the benchmark contract)."""

import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2008_10273_b200 import codec, homogeneous  # noqa: E402
from paper_2008_10273_b200.synth import random_mask, synth_clip  # noqa: E402

REPO = Path(__file__).resolve().parent.parent


def main():
    data = (REPO / "tests/golden/streams/cfg0.hivc").read_bytes()
    out = torch.empty(codec.frames_shape(data), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        codec.decode_frames(data, out=out)
    tm = {}
    t0 = time.perf_counter()
    for _ in range(10):
        codec.decode_frames(data, out=out, timings=tm)
    dt = (time.perf_counter() - t0) / 10
    print(f"cfg0 decode: {dt * 1e3:.2f} ms/stream = {10 / dt:.0f} fps; stages {({k: round(v / 10 * 1e3, 3) for k, v in tm.items()})}")
    plane = synth_clip(1, 1080, 1920, blobs=40, rects=12, v=6.0, seed=1)[0, 0].astype(np.float64)
    for dens, tol, mi, strict in [(0.04, 1e-4, 160, False), (0.02, 1e-6, 10000, True)]:
        m = random_mask(plane.shape, dens, 1001)
        f = torch.from_numpy(np.where(m, plane, 0.0)).cuda()
        mt = torch.from_numpy(m).cuda()
        st = {}
        homogeneous.solve_homogeneous(f, mt, tol=tol, max_iter=mi, strict=strict, stats=st)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            homogeneous.solve_homogeneous(f, mt, tol=tol, max_iter=mi, strict=strict)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"1080p solve dens={dens} tol={tol}: {dt * 1e3:.2f} ms, iters {st['level_iterations']}")


if __name__ == "__main__":
    main()
