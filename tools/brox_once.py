"""One 1080p Brox pair (config-4 content) for profiling: python tools/brox_once.py [scale] [reps]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2008_10273_b200.flow import BroxParams, flow_brox  # noqa: E402
from paper_2008_10273_b200.synth import synth_clip  # noqa: E402

sc = float(sys.argv[1]) if len(sys.argv) > 1 else 0.95
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
clip = synth_clip(2, 1080, 1920, blobs=40, rects=12, v=6.0, seed=4)[:, 0].astype(np.float64)
a, b = torch.from_numpy(clip[1]).cuda(), torch.from_numpy(clip[0]).cuda()
for _ in range(reps):
    f = flow_brox(a, b, BroxParams(pyramid_scale=sc))
torch.cuda.synchronize()
print("ok", float(f.u.abs().max()))
