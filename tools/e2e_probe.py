"""Wall time vs device span of decode_streams, device vs pinned-host outputs.

    python tools/e2e_probe.py [reps]
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10273_b200 import _native as N  # noqa: E402
from paper_2008_10273_b200 import codec  # noqa: E402

REPO = Path(__file__).resolve().parent.parent
streams = [(REPO / "tests/golden/streams" / f"cfg3_{p}.hivc").read_bytes() for p in ("Y", "Cb", "Cr")]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
ctx = N.Context(0)
N.check(N.lib.hivc_ctx_set_stage_timing(ctx.handle, 0))
shapes = [codec.frames_shape(s, 0, None) for s in streams]
dev = [torch.empty(s, dtype=torch.uint8, device="cuda") for s in shapes]
host = [torch.empty(s, dtype=torch.uint8, pin_memory=True) for s in shapes]
for name, outs in (("device", dev), ("host", host), ("device", dev), ("host", host)):
    walls, spans = [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        span = codec.decode_streams(streams, outs, ctx=ctx)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
        spans.append(span)
    print(f"{name:6s} wall ms: " + " ".join(f"{1e3 * w:.1f}" for w in walls))
    print(f"{name:6s} span ms: " + " ".join(f"{1e3 * s:.1f}" for s in spans))
