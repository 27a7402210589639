"""How many config-3 frames decode bit-identical to the reference (per plane)."""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10273_b200 import codec  # noqa: E402

g = Path(__file__).resolve().parent.parent / "tests" / "golden"
for plane in ("Y", "Cb", "Cr"):
    ref = np.load(g / f"cfg3_{plane}_sums.npz")
    out = codec.decode_frames((g / "streams" / f"cfg3_{plane}.hivc").read_bytes()).numpy()
    exact = [hashlib.sha256(out[i, 0].tobytes()).hexdigest() == ref["sha256"][i] for i in range(out.shape[0])]
    drift = [int(np.abs(out[i, 0].sum(axis=1).astype(np.int64) - ref["row_sums"][i]).sum()) for i in range(out.shape[0])]
    print(plane, "exact frames", sum(exact), "/", len(exact), "max row-sum drift", max(drift), "total", sum(drift))
