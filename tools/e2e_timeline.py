"""Per-item timeline of one host-output decode (HIVC_DEBUG=timeline=path): where
the D2H tail of the e2e step comes from.  python tools/e2e_timeline.py out.csv"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10273_b200 import _native as N  # noqa: E402
from paper_2008_10273_b200 import codec  # noqa: E402

REPO = Path(__file__).resolve().parent.parent
streams = [(REPO / "tests/golden/streams" / f"cfg3_{p}.hivc").read_bytes() for p in ("Y", "Cb", "Cr")]
ctx = N.Context(0)
shapes = [codec.frames_shape(s, 0, None) for s in streams]
host = [torch.empty(s, dtype=torch.uint8, pin_memory=True) for s in shapes]
for _ in range(5):
    codec.decode_streams(streams, host, ctx=ctx)
torch.cuda.synchronize()
