"""Golden vectors for prediction.optimize_mask_values (the encoder's tonal
optimisation), produced by importing the REFERENCE here:

    OMP_NUM_THREADS=1 python tests/golden/make_tonal.py   ->  tests/golden/golden_tonal.npz

Cases: a luma-like plane with the reference's own error-driven subdivision
mask (prediction.py's encoder path), a 2-plane (chroma) case sharing a
random mask, a full mask (returned verbatim) and a 1-point mask.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")

from paper_2008_10273_b200.synth import synth_clip  # noqa: E402


def main():
    from hivc import prediction as rp
    from hivc import subdivision as rs

    g = {}
    clip = synth_clip(1, 72, 96, blobs=5, rects=2, v=2.0, seed=21, channels=3)[0]
    y = np.clip(np.rint(clip[0]), 0, 255)
    tree = rs.subdivide_by_error(y, int(0.08 * y.size))
    m0 = rs.mask_from_tree(tree)
    cases = [
        ([y], m0),
        ([clip[1], clip[2]], np.random.default_rng(22).uniform(size=(72, 96)) < 0.05),
        ([y[:16, :24]], np.ones((16, 24), bool)),
        ([y[:20, :30]], np.pad(np.ones((1, 1), bool), ((7, 12), (11, 18)))),
    ]
    for i, (planes, mask) in enumerate(cases):
        out = rp.optimize_mask_values(planes, mask)
        g[f"tonal{i}_planes"] = np.stack([np.asarray(p, dtype=np.float64) for p in planes])
        g[f"tonal{i}_mask"] = mask
        g[f"tonal{i}_out"] = np.stack(out)
    np.savez_compressed(HERE / "golden_tonal.npz", **g)
    print("wrote", HERE / "golden_tonal.npz", [g[f"tonal{i}_out"].shape for i in range(len(cases))])


if __name__ == "__main__":
    main()
