"""Determinism stress: repeated solves of the same problems must be bit-identical."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10273_b200.homogeneous import solve_homogeneous  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
bad = 0
for (h, w) in [(300, 500), (1080, 1920), (540, 960), (301, 517)]:
    rng = np.random.default_rng(5)
    m = rng.uniform(size=(h, w)) < 0.03
    f = np.where(m, rng.uniform(0, 255, m.shape), 0.0)
    ft, mt = torch.from_numpy(f).cuda(), torch.from_numpy(m).cuda()
    ref = solve_homogeneous(f, m, tol=1e-4, max_iter=160, strict=False)
    for i in range(reps):
        o = solve_homogeneous(ft, mt, tol=1e-4, max_iter=160, strict=False).cpu().numpy()
        d = np.abs(o - ref).max()
        if d != 0:
            bad += 1
            idx = np.unravel_index(np.argmax(np.abs(o - ref)), o.shape)
            print((h, w), "rep", i, "max diff", d, "at", idx, flush=True)
print("mismatches", bad)
