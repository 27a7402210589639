"""Time one cascadic solve per plane size with the HIVC_CG_TRACE phase breakdown
of its finest level (run under HIVC_DEBUG=cg_trace; packed mode is the
packed band layout for single solves)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10273_b200 import homogeneous  # noqa: E402
from paper_2008_10273_b200.synth import random_mask, synth_clip  # noqa: E402

SIZES = [(540, 960), (1080, 1920)] if len(sys.argv) < 2 else [tuple(map(int, sys.argv[1].split("x")))]
for h, w in SIZES:
    plane = synth_clip(1, h, w, blobs=40, rects=12, v=6.0, seed=1)[0, 0].astype(np.float64)
    m = random_mask(plane.shape, 0.09, 1001)
    f = torch.from_numpy(np.where(m, plane, 0.0)).cuda()
    mt = torch.from_numpy(m).cuda()
    for _ in range(3):
        st = {}
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        homogeneous.solve_homogeneous(f, mt, tol=1e-4, max_iter=160, strict=False, stats=st)
        ev1.record()
        torch.cuda.synchronize()
    print((h, w), st["level_iterations"], f"{ev0.elapsed_time(ev1):.3f} ms", flush=True)
