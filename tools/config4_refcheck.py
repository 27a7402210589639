"""Config 4, GOP 0: the UNMODIFIED reference encoder (baseline/_ref,
hivc.codec.encode, codec.py:426-471) on the same 12 frames with the same
injected flows must produce the GOP payload our encoder wrote.

    python tools/config4_refcheck.py --gop0 /tmp/cfg4_gop0.npz --streams DIR [--planes Y Cb Cr]

One process per plane (the reference is single-threaded numpy: luma takes a
few minutes).  Prints one JSON line per plane: byte-identical or not, sizes,
reference seconds.
"""

from __future__ import annotations

import argparse
import json
import struct
import sys
import time
from multiprocessing import get_context
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent


def _one(args):
    plane, gop0, streams = args
    sys.path.insert(0, str(REPO / "baseline" / "_ref"))
    from hivc import codec as rc
    from hivc.flow import FlowField
    from hivc.frame import Frame

    g = np.load(gop0)
    frames = [Frame((p.astype(np.int32),), colorspace="gray") for p in g[plane]]
    if plane == "Y":
        flows = [FlowField(u, v) for u, v in zip(g["lu"], g["lv"])]
    else:
        flows = [FlowField(u, v) for u, v in zip(g["cu"], g["cv"])]
    t0 = time.perf_counter()
    ref = rc.encode(frames, rc.EncoderConfig(gop_size=12), _flows=[flows])
    dt = time.perf_counter() - t0
    ours = (Path(streams) / f"cfg4_{plane}.hivc").read_bytes()
    (ln,) = struct.unpack_from("<I", ours, 22)
    ours_gop0 = ours[26 : 26 + ln]
    (rln,) = struct.unpack_from("<I", ref, 22)
    ref_gop0 = ref[26 : 26 + rln]
    return {"plane": plane, "gop0_identical": ours_gop0 == ref_gop0, "ours_bytes": len(ours_gop0),
            "reference_bytes": len(ref_gop0), "reference_seconds": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gop0", required=True)
    ap.add_argument("--streams", required=True)
    ap.add_argument("--planes", nargs="+", default=["Y", "Cb", "Cr"])
    a = ap.parse_args()
    with get_context("spawn").Pool(len(a.planes)) as pool:
        for r in pool.imap_unordered(_one, [(p, a.gop0, a.streams) for p in a.planes]):
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
