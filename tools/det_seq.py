"""Reproduce the GPU test sequence, then check determinism of a 300x500 solve."""
import sys
from pathlib import Path

import numpy as np
import pytest  # noqa: F401
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from paper_2008_10273_b200.homogeneous import solve_homogeneous  # noqa: E402


def det(tag):
    rng = np.random.default_rng(5)
    m = rng.uniform(size=(300, 500)) < 0.03
    f = np.where(m, rng.uniform(0, 255, m.shape), 0.0)
    outs = []
    for i in range(6):
        st = {}
        if i % 2:
            o = solve_homogeneous(f, m, tol=1e-4, max_iter=160, strict=False, stats=st)
        else:
            o = solve_homogeneous(torch.from_numpy(f).cuda(), torch.from_numpy(m).cuda(), tol=1e-4, max_iter=160,
                                  strict=False, stats=st).cpu().numpy()
        outs.append((o, st["level_iterations"]))
    diffs = [float(np.abs(o - outs[0][0]).max()) for o, _ in outs]
    print(tag, diffs, [it[-1] for _, it in outs], flush=True)


det("fresh")
import test_gpu_blocks as tb  # noqa: E402
import test_gpu_parity as tp  # noqa: E402
import conftest  # noqa: E402

g = np.load(Path(__file__).resolve().parent.parent / "tests" / "golden" / "golden.npz", allow_pickle=True)
for name in dir(tb):
    if name.startswith("test_"):
        fn = getattr(tb, name)
        try:
            fn(g) if fn.__code__.co_argcount else fn()
        except TypeError:
            pass
det("after blocks")
for i in range(8):
    try:
        tp.test_solve_homogeneous_matches_reference(g, i)
    except TypeError:
        tp.test_solve_homogeneous_matches_reference(i)
det("after matches_reference")
tp.test_solve_homogeneous_1080p_vs_oracle()
det("after 1080p")
tp.test_solve_homogeneous_errors()
det("after errors")
