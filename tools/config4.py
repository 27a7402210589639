"""Config 4: 1080p 4:2:0 encode + decode, measured on a GOP sample.

Workload per GOP (12 frames): Brox flows on luma only at pyramid_scale 0.95
(alpha = gamma = 40 defaults), chroma flows = luma flow 2x2-averaged and
halved, three gray streams (Y 1080x1920, Cb/Cr 540x960) encoded with the
injected flows (`codec.encode(..., _flows=...)`, EncoderConfig(gop_size=12)),
then decoded.  Content: synth_420(seed=4), frames generated for the sampled
GOPs only (the 480-frame clip's first GOPs: the per-frame noise draws are
sequential, so these are exactly its frames).

GOPs are independent (one process per GPU, GOP ranges per rank:
`shard.encode_sharded`), so the 480-frame / 40-GOP job on P GPUs takes
ceil(40 / P) GOP times; the script reports the measured per-GOP times and
that extrapolation, labelled as such.

    python tools/config4.py [--gops 2] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gops", type=int, default=2)
    ap.add_argument("--json", default=None)
    ap.add_argument("--workers", type=int, default=1, help="GOPs encoded concurrently (threads, one context each)")
    a = ap.parse_args()
    import torch

    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.flow import BroxParams, FlowField, flow_brox
    from paper_2008_10273_b200.frame import Frame
    from paper_2008_10273_b200.synth import downsample2, synth_420

    G = 12
    t0 = time.perf_counter()
    planes = synth_420(G * a.gops, 1080, 1920, blobs=40, rects=12, v=6.0, seed=4)
    print(f"synth {time.perf_counter() - t0:.1f}s", flush=True)
    cfg = codec.EncoderConfig(gop_size=G)
    bp = BroxParams(pyramid_scale=0.95)
    def one_gop(g):
        s, e = g * G, (g + 1) * G
        t0 = time.perf_counter()
        y = planes[0][s:e].astype(np.float64)
        lflows = [flow_brox(y[i], y[i - 1], bp) for i in range(1, G)]
        t_flow = time.perf_counter() - t0
        cflows = [FlowField(downsample2(f.u) * 0.5, downsample2(f.v) * 0.5) for f in lflows]
        streams = []
        t1 = time.perf_counter()
        for pi, fl in enumerate([lflows, cflows, cflows]):
            frames = [Frame((p,), colorspace="gray") for p in planes[pi][s:e]]
            streams.append(codec.encode(frames, cfg, _flows=[fl]))
        t_enc = time.perf_counter() - t1
        t2 = time.perf_counter()
        out = [torch.empty(codec.frames_shape(st), dtype=torch.uint8, device="cuda") for st in streams]
        codec.decode_streams(streams, out)
        torch.cuda.synchronize()
        t_dec = time.perf_counter() - t2
        psnr = []
        for pi, o in enumerate(out):
            d = o.cpu().numpy()[:, 0].astype(np.float64) - planes[pi][s:e]
            psnr.append(round(10 * np.log10(255.0**2 / max(np.mean(d * d), 1e-12)), 2))
        rec = {"gop": g, "brox_s": round(t_flow, 3), "brox_ms_per_pair": round(1e3 * t_flow / (G - 1), 1),
               "encode_s": round(t_enc, 3), "decode_s": round(t_dec, 4),
               "bytes": [len(st) for st in streams], "psnr_db": psnr}
        print(json.dumps(rec), flush=True)
        return rec

    one_gop(0)  # warm-up (graphs, workspaces, first-touch)
    torch.cuda.synchronize()
    t_all = time.perf_counter()
    if a.workers > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(a.workers) as ex:
            per_gop = list(ex.map(one_gop, range(a.gops)))
    else:
        per_gop = [one_gop(g) for g in range(a.gops)]
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_all
    gop_s = wall / a.gops  # throughput: wall time per GOP (GOPs overlap when workers > 1)
    dec_s = float(np.mean([r["decode_s"] for r in per_gop]))
    summary = {
        "config": "config4 sample: 1080p 4:2:0, GOP 12, Brox 0.95 on luma, injected chroma flows",
        "gops_measured": a.gops,
        "workers": a.workers,
        "wall_s": round(wall, 3),
        "encode_gop_s": round(gop_s, 3),
        "encode_fps_per_gpu": round(G / gop_s, 2),
        "decode_gop_s": round(dec_s, 4),
        "extrapolated_480_frames": {f"{p}gpu_encode_s": round(-(-40 // p) * gop_s, 1) for p in (1, 2, 4, 8)},
        "extrapolated_encode_fps": {f"{p}gpu": round(480 / (-(-40 // p) * gop_s), 2) for p in (1, 2, 4, 8)},
        "note": "extrapolated from the measured per-GOP time (GOP-sharded, no cross-GOP work)",
    }
    print(json.dumps(summary), flush=True)
    if a.json:
        Path(a.json).write_text(json.dumps({"gops": per_gop, "summary": summary}, indent=1))


if __name__ == "__main__":
    main()
