"""Per-phase device timing of the batched I-frame solves of one config-3 decode
(HIVC_DEBUG=batch_trace prints one line per phase from the CgProbe marks)."""
import os
import sys
from pathlib import Path

os.environ.setdefault("HIVC_DEBUG", "batch_trace")
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10273_b200 import _native as N  # noqa: E402
from paper_2008_10273_b200 import codec  # noqa: E402

REPO = Path(__file__).resolve().parent.parent
streams = [(REPO / "tests/golden/streams" / f"cfg3_{p}.hivc").read_bytes() for p in ("Y", "Cb", "Cr")]
ctx = N.Context(0)
outs = [torch.empty(codec.frames_shape(s), dtype=torch.uint8, device="cuda") for s in streams]
N.check(N.lib.hivc_ctx_set_stage_timing(ctx.handle, 0))
for _ in range(4):
    codec.decode_streams(streams, outs, ctx=ctx)
torch.cuda.synchronize()
N.check(N.lib.hivc_ctx_set_stage_timing(ctx.handle, 1))
sys.stderr.flush()
print("---- traced call", flush=True)
t = {}
codec.decode_streams(streams, outs, ctx=ctx, timings=t)
torch.cuda.synchronize()
print({k: round(v * 1e3, 3) for k, v in t.items()})
