"""Golden vectors at the BENCHMARK configurations, produced by the REFERENCE.

Run here (the container that has /root/reference), never on the GPU box:

    python tests/golden/make_bench_pins.py cfg1          # ~20 s
    python tests/golden/make_bench_pins.py brox05        # ~1-2 min
    python tests/golden/make_bench_pins.py brox095       # ~10 min

Writes tests/golden/pin_<name>.npz.  The inputs are stored exactly (mask
indices + float32 values for config 1, uint8 frames for Brox), so the GPU
test rebuilds them bit for bit without re-running the synthetic generator
(whose numpy `exp` may round differently on another host CPU).  Full-size
float64 outputs do not fit in the repo, so each output is stored as its exact
row sums, column sums and a strided sub-grid of values.

* cfg1: BASELINE config 1 — 1080p x 3 channels (synth seed 1, 40 blobs,
  12 rectangles), shared uniform-random 2 % mask (seed 1001),
  `solve_homogeneous(tol=1e-6, max_iter=10000, strict=True)` per channel
  (homogeneous.py:157-212) with the per-level iteration counts.
* brox05 / brox095: `flow_brox` (flow.py:187-278) on a 1440x810 pair
  (> 2^20 px, so the GPU's two-sweep level kernel runs on the two finest
  levels) at pyramid_scale 0.5 and 0.95, other BroxParams at their defaults.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

ROW_STEP, COL_STEP = 8, 4  # strided sub-grid of stored output values


def summarise(prefix: str, a: np.ndarray, g: dict) -> None:
    g[f"{prefix}_rows"] = a.sum(axis=1)
    g[f"{prefix}_cols"] = a.sum(axis=0)
    g[f"{prefix}_grid"] = a[::ROW_STEP, ::COL_STEP].copy()


def cfg1() -> None:
    import hivc.homogeneous as rh

    from paper_2008_10273_b200.synth import random_mask, synth_clip

    clip = synth_clip(1, 1080, 1920, blobs=40, rects=12, v=6.0, seed=1, channels=3)[0]  # float32
    m = random_mask((1080, 1920), 0.02, 1001)
    idx = np.flatnonzero(m).astype(np.int32)
    g = {"shape": np.array([1080, 1920]), "mask_idx": idx}
    for c in range(3):
        vals = clip[c].ravel()[idx].astype(np.float32)
        f = np.zeros(1080 * 1920)
        f[idx] = vals.astype(np.float64)
        f = f.reshape(1080, 1920)
        st = {}
        t0 = time.perf_counter()
        u = rh.solve_homogeneous(f, m, tol=1e-6, max_iter=10000, strict=True, stats=st)
        print(f"channel {c}: {time.perf_counter() - t0:.1f} s, iterations {st['level_iterations']}", flush=True)
        g[f"vals{c}"] = vals
        g[f"iters{c}"] = np.array(st["level_iterations"], dtype=np.int64)
        summarise(f"u{c}", u, g)
    np.savez_compressed(HERE / "pin_cfg1.npz", **g)


def brox(scale: float, name: str) -> None:
    import hivc.flow as rf

    from paper_2008_10273_b200.synth import synth_clip

    clip = synth_clip(2, 810, 1440, blobs=24, rects=8, v=4.0, seed=7)
    frames = np.rint(clip[:, 0]).astype(np.uint8)
    t0 = time.perf_counter()
    fl = rf.flow_brox(frames[1].astype(np.float64), frames[0].astype(np.float64),
                      rf.BroxParams(pyramid_scale=scale))
    print(f"brox {scale}: {time.perf_counter() - t0:.1f} s", flush=True)
    g = {"frames": frames, "scale": np.array(scale)}
    summarise("u", fl.u, g)
    summarise("v", fl.v, g)
    np.savez_compressed(HERE / f"pin_{name}.npz", **g)


if __name__ == "__main__":
    what = sys.argv[1:] or ["cfg1", "brox05", "brox095"]
    for w in what:
        if w == "cfg1":
            cfg1()
        elif w == "brox05":
            brox(0.5, "brox05")
        elif w == "brox095":
            brox(0.95, "brox095")
        else:
            raise SystemExit(f"unknown pin {w}")
