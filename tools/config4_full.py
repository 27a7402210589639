"""BASELINE config 4, run in full on one GPU: the 480-frame 1080p 4:2:0 clip
(synth seed 4, 40 blobs, 12 rectangles, v = 6; 40 GOPs of 12) encoded end to
end and decoded.

Per GOP: Brox flows on luma at pyramid_scale 0.95 (alpha = gamma = 40, the
reference defaults; flow.py:187-278) for the 11 frame pairs, chroma flows =
luma flow 2x2-averaged and halved, three gray streams (Y 1080x1920, Cb/Cr
540x960) encoded with the injected flows (`codec.encode_gops(..., _flows)`,
EncoderConfig(gop_size=12), codec.py:426-471).  Frames are generated one at
a time (`synth.synth_420_frames`, the same draws as `synth_420`).  GOP 0's
planes and flows go to --gop0 for the reference-encoder check
(tools/config4_refcheck.py).  Then the 40-GOP streams are decoded
(`codec.decode_streams`, device output) and checked against the encoder's own
reconstructions (per-frame SHA-256).

    python tools/config4_full.py --out DIR [--gops 40] [--gop0 /tmp/cfg4_gop0.npz] [--json out.json]

Writes DIR/cfg4_{Y,Cb,Cr}.hivc and prints one JSON line: encode frames/s
(wall, Brox and encode split), decode frames/s (median of 5, CUDA events),
stream sizes.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
G = 12
PLANES = ("Y", "Cb", "Cr")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--gops", type=int, default=40)
    ap.add_argument("--gop0", default=None)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    import torch

    from paper_2008_10273_b200 import codec, encoder
    from paper_2008_10273_b200 import _native as N
    from paper_2008_10273_b200.bitstream import StreamHeader, write_stream
    from paper_2008_10273_b200.flow import BroxParams, FlowField, flow_brox
    from paper_2008_10273_b200.frame import Frame
    from paper_2008_10273_b200.synth import downsample2, synth_420_frames

    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    cfg = codec.EncoderConfig(gop_size=G)
    bp = BroxParams(pyramid_scale=0.95)
    nframes = G * a.gops
    # input clip first (host numpy, not codec work): uint8 planes
    t0 = time.perf_counter()
    clip = [tuple(p.astype(np.uint8) for p in f)
            for f in synth_420_frames(nframes, 1080, 1920, blobs=40, rects=12, v=6.0, seed=4)]
    t_synth = time.perf_counter() - t0
    print(f"synthesis {t_synth:.1f} s", file=sys.stderr, flush=True)
    payloads = {p: [None] * a.gops for p in PLANES}
    recon_sha = {p: [None] * a.gops for p in PLANES}
    t_flow = t_enc = 0.0

    def flows_of(g):  # Brox on luma (GPU) + the derived chroma flows
        fr = clip[g * G:(g + 1) * G]
        yd = [torch.from_numpy(f[0].astype(np.float64)).cuda() for f in fr]
        lf = [flow_brox(yd[i], yd[i - 1], bp) for i in range(1, G)]
        lf = [FlowField(f.u.cpu().numpy(), f.v.cpu().numpy()) for f in lf]
        cf = [FlowField(downsample2(f.u) * 0.5, downsample2(f.v) * 0.5) for f in lf]
        return lf, cf

    def encode_gop(g, lf, cf):
        fr = clip[g * G:(g + 1) * G]
        for k, p in enumerate(PLANES):
            frames = [Frame((f[k].astype(np.int32),), colorspace="gray") for f in fr]
            pay, rec = encoder.encode_gops(frames, cfg, 0, 1, [lf if k == 0 else cf], workers=1)
            payloads[p][g] = pay[0]
            recon_sha[p][g] = [hashlib.sha256(np.asarray(r[0], dtype=np.uint8).tobytes()).hexdigest() for r in rec[0]]

    # pipelined: the flows of GOP g+1 are estimated on the GPU while GOP g is
    # encoded (host C++ + GPU fits / tonal solves); GOPs are independent
    import queue
    import threading

    q = queue.Queue(maxsize=2)
    t_all = time.perf_counter()

    def producer():
        nonlocal t_flow
        for g in range(a.gops):
            t0 = time.perf_counter()
            lf, cf = flows_of(g)
            t_flow += time.perf_counter() - t0
            if g == 0 and a.gop0:
                fr = clip[:G]
                np.savez(a.gop0, Y=np.stack([f[0] for f in fr]), Cb=np.stack([f[1] for f in fr]),
                         Cr=np.stack([f[2] for f in fr]), lu=np.stack([f.u for f in lf]), lv=np.stack([f.v for f in lf]),
                         cu=np.stack([f.u for f in cf]), cv=np.stack([f.v for f in cf]))
            q.put((g, lf, cf))
        q.put(None)

    th = threading.Thread(target=producer)
    th.start()
    while True:
        item = q.get()
        if item is None:
            break
        g, lf, cf = item
        t0 = time.perf_counter()
        encode_gop(g, lf, cf)
        t_enc += time.perf_counter() - t0
        print(f"GOP {g}: {time.perf_counter() - t_all:.1f} s", file=sys.stderr, flush=True)
    th.join()
    t_total = time.perf_counter() - t_all
    payloads = {p: payloads[p] for p in PLANES}
    recon_sha = {p: [h for gop in recon_sha[p] for h in gop] for p in PLANES}
    streams = []
    for p in PLANES:
        h, w = (1080, 1920) if p == "Y" else (540, 960)
        hdr = StreamHeader(width=w, height=h, frame_count=nframes, fps_num=cfg.fps_num, fps_den=cfg.fps_den,
                           gop_size=G, channels=1, intra_levels=cfg.intra_levels, flow_levels=cfg.flow_levels,
                           residual_levels=cfg.residual_levels)
        s = write_stream(hdr, payloads[p])
        (out / f"cfg4_{p}.hivc").write_bytes(s)
        streams.append(s)
    # ---- decode (1 GPU): device output, median of 5 after 2 warm-ups; frames vs the encoder's reconstructions
    ctx = N.Context(0)
    outs = [torch.empty(codec.frames_shape(s), dtype=torch.uint8, device="cuda") for s in streams]
    times = []
    for i in range(7):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        codec.decode_streams(streams, outs, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            times.append(e0.elapsed_time(e1) / 1e3)
    exact = {}
    for p, o in zip(PLANES, outs):
        a_ = o.cpu().numpy()
        exact[p] = sum(hashlib.sha256(a_[i, 0].tobytes()).hexdigest() == recon_sha[p][i] for i in range(a_.shape[0]))
    dec = statistics.median(times)
    line = {
        "config": 4, "what": f"{nframes}-frame 1080p 4:2:0 clip, {a.gops} GOPs of 12, Brox 0.95 on luma, one GPU",
        "encode_seconds": t_total, "encode_fps": nframes / t_total,
        "encode_busy_s": {"brox_flows_thread": t_flow, "encode_3_streams_thread": t_enc},
        "encode_note": "wall time of the pipelined encode (flows of GOP g+1 on the GPU while GOP g is encoded); "
                       "the input clip is synthesised beforehand and not counted",
        "input_synthesis_s": t_synth,
        "decode_seconds": dec, "decode_fps": nframes / dec,
        "decode_frames_equal_encoder_recon": exact, "frames": nframes,
        "stream_bytes": {p: len(s) for p, s in zip(PLANES, streams)},
        "stream_sha256": {p: hashlib.sha256(s).hexdigest() for p, s in zip(PLANES, streams)},
    }
    print(json.dumps(line), flush=True)
    if a.json:
        Path(a.json).write_text(json.dumps(line, indent=1) + "\n")


if __name__ == "__main__":
    main()
