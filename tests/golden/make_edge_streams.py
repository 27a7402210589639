"""Edge-size streams made and decoded by the REFERENCE codec (run in this
container only):

    OMP_NUM_THREADS=1 python tests/golden/make_edge_streams.py  ->  tests/golden/golden_edge.npz

Frame sizes from 1x1 up to odd sizes that cross the 8x8 tile grid and the
solver's level / kernel thresholds, gray and RGB, one and several GOPs, the
lossless full-mask configuration and Horn-Schunck flows.  Stored: the stream
bytes and the reference decoder's frames, so the GPU decoder (and encoder)
can be checked on sizes the benchmark clips never hit.
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

from paper_2008_10273_b200.synth import synth_clip, to_codec_planes  # noqa: E402

CASES = [
    # (name, n, h, w, channels, encoder kwargs)
    # one-pixel-wide frames: I-frames only (the reference's flow needs 2x2 planes)
    ("g1x1", 2, 1, 1, 1, dict(gop_size=1)),
    ("g1x7", 3, 1, 7, 1, dict(gop_size=1, intra_mask_fraction=0.3)),
    ("g7x1", 3, 7, 1, 1, dict(gop_size=1, intra_mask_fraction=0.3)),
    ("g2x2", 2, 2, 2, 1, dict(gop_size=2, flow_points=3)),
    ("g5x3", 3, 5, 3, 1, dict(gop_size=3, intra_mask_fraction=0.5, flow_points=15)),
    ("g9x17", 4, 9, 17, 1, dict(gop_size=2, intra_mask_fraction=0.2)),
    ("g33x65", 4, 33, 65, 1, dict(gop_size=4, intra_mask_fraction=0.05)),
    ("g130x250", 3, 130, 250, 1, dict(gop_size=3, intra_mask_fraction=0.03)),
    ("g257x129", 3, 257, 129, 1, dict(gop_size=3, intra_mask_fraction=0.02, flow_method="horn-schunck")),
    ("c3x4", 2, 3, 4, 3, dict(gop_size=2, flow_points=5)),
    ("c17x23", 3, 17, 23, 3, dict(gop_size=3, intra_mask_fraction=0.15)),
    ("c45x61", 4, 45, 61, 3, dict(gop_size=2, intra_mask_fraction=0.08, residual_points=9)),
    ("lossless21x19", 2, 21, 19, 3, dict(gop_size=1, intra_mask_fraction=1.0, intra_levels=256)),
]


def main():
    from hivc import codec
    from hivc.frame import Frame

    g = {}
    for i, (name, n, h, w, ch, kw) in enumerate(CASES):
        clip = to_codec_planes(synth_clip(n, h, w, blobs=3, rects=1, v=1.0, seed=50 + i, channels=ch))
        cs = "rgb" if ch == 3 else "gray"
        frames = [Frame(tuple(f[c] for c in range(ch)), colorspace=cs) for f in clip]
        stream = codec.encode(frames, codec.EncoderConfig(**kw))
        dec = codec.decode(stream)
        g[f"{name}_src"] = clip.astype(np.uint8)
        g[f"{name}_cfg"] = np.array(repr(kw))
        g[f"{name}_stream"] = np.frombuffer(stream, dtype=np.uint8)
        g[f"{name}_frames"] = np.stack([np.stack(f.planes) for f in dec]).astype(np.int16)
        print(name, len(stream), "bytes", flush=True)
    g["names"] = np.array([c[0] for c in CASES])
    np.savez_compressed(HERE / "golden_edge.npz", **g)


if __name__ == "__main__":
    main()
