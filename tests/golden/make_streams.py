"""Produce the benchmark bitstreams with the REFERENCE encoder and record
the reference decoder's output for them.

Run here (the container that has /root/reference), never on the GPU box:

    OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python tests/golden/make_streams.py [cfg0] [rgb] [cfg3]

Outputs (committed, small):
  tests/golden/streams/cfg0.hivc            config 0: 320x180 gray, 10 frames, GOP 10, intra 4 %
  tests/golden/streams/rgb.hivc             colour: 96x128 RGB, 7 frames, GOP 4 (RCT path)
  tests/golden/rgb_frames.npz               reference-decoded colour frames (uint8, n x 3 x h x w)
  tests/golden/streams/cfg3_{Y,Cb,Cr}.hivc  config 3: 60-frame 1080p 4:2:0 as three gray streams, GOP 12
  tests/golden/cfg0_frames.npz              reference-decoded config-0 frames (uint8)
  tests/golden/cfg3_{plane}_sums.npz        per-frame sha256 + row/column sums of the reference decode
  tests/golden/streams/manifest.json        sha256 of every stream, reference decode timings

Config 3 is encoded GOP by GOP in a process pool (the reference encoder
has no cross-GOP state: `codec.py:459-462` loops GOPs independently and
`codec.py:496` resets `prev` per GOP) and the single-GOP payloads are
spliced with the reference's own `write_stream`.  Flows are the
reference's own Brox flows (`flow.py:187`, default `BroxParams`, which is
what `codec._estimate_flow` uses, `codec.py:369-372`), computed per plane.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool
from pathlib import Path

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

from paper_2008_10273_b200.synth import synth_420, synth_clip, to_codec_planes  # noqa: E402

STREAMS = HERE / "streams"
WORK = Path("/tmp/hivc_streams_work")


def _ref():
    import hivc.bitstream as bs
    import hivc.codec as codec
    import hivc.flow as flow
    from hivc.frame import Frame

    return codec, flow, bs, Frame


def _sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


# ----------------------------------------------------------------------------- config 0


def make_cfg0():
    codec, _, _, Frame = _ref()
    clip = to_codec_planes(synth_clip(10, 180, 320, blobs=8, rects=3, v=3.0, seed=0)[:, 0])
    frames = [Frame((p,), colorspace="gray") for p in clip]
    cfg = codec.EncoderConfig(gop_size=10, intra_mask_fraction=0.04)
    t0 = time.perf_counter()
    stream = codec.encode(frames, cfg)
    t_enc = time.perf_counter() - t0
    t0 = time.perf_counter()
    timings = {}
    dec = codec.decode(stream, timings)
    t_dec = time.perf_counter() - t0
    STREAMS.mkdir(parents=True, exist_ok=True)
    (STREAMS / "cfg0.hivc").write_bytes(stream)
    out = np.stack([f.planes[0] for f in dec]).astype(np.uint8)
    np.savez_compressed(HERE / "cfg0_frames.npz", frames=out, source=clip.astype(np.uint8))
    return {
        "cfg0.hivc": {
            "sha256": _sha(stream),
            "bytes": len(stream),
            "encode_s": t_enc,
            "decode_s": t_dec,
            "timings": timings,
        }
    }


# ----------------------------------------------------------------------------- colour (RCT) stream


def make_rgb():
    """A small 3-channel RGB clip (RCT domain inside the codec, frame.py:70-93):
    7 frames of 96x128 in GOPs of 4 (I P P P | I P P), intra 6 %, encoded and
    decoded by the reference; exercises the colour path (shared chroma tree,
    the U/V intra levels 2L-1, the [-255, 255] chroma clip, RCT inverse)."""
    codec, _, _, Frame = _ref()
    clip = to_codec_planes(synth_clip(7, 96, 128, blobs=6, rects=3, v=2.0, seed=7, channels=3))
    frames = [Frame(tuple(f[c] for c in range(3)), colorspace="rgb") for f in clip]
    cfg = codec.EncoderConfig(gop_size=4, intra_mask_fraction=0.06)
    t0 = time.perf_counter()
    stream = codec.encode(frames, cfg)
    t_enc = time.perf_counter() - t0
    timings = {}
    t0 = time.perf_counter()
    dec = codec.decode(stream, timings)
    t_dec = time.perf_counter() - t0
    (STREAMS / "rgb.hivc").write_bytes(stream)
    out = np.stack([np.stack(f.planes) for f in dec]).astype(np.uint8)
    np.savez_compressed(HERE / "rgb_frames.npz", frames=out, colorspace=np.array([f.colorspace for f in dec]))
    return {"rgb.hivc": {"sha256": _sha(stream), "bytes": len(stream), "encode_s": t_enc, "decode_s": t_dec,
                         "timings": timings}}


# ----------------------------------------------------------------------------- config 3

GOP = 12
NF = 60
PLANES = ("Y", "Cb", "Cr")


def _planes3():
    cache = WORK / "cfg3_planes.npz"
    if cache.exists():
        z = np.load(cache)
        return {k: z[k] for k in PLANES}
    y, cb, cr = synth_420(NF, 1080, 1920, blobs=40, rects=12, v=6.0, seed=3)
    WORK.mkdir(parents=True, exist_ok=True)
    np.savez(cache, Y=y, Cb=cb, Cr=cr)
    return {"Y": y, "Cb": cb, "Cr": cr}


def _flow_job(args):
    plane, i = args
    path = WORK / f"flow_{plane}_{i:03d}.npz"
    if path.exists():
        return path
    _, flow, _, _ = _ref()
    p = _planes3()[plane]
    t0 = time.perf_counter()
    f = flow.flow_brox(p[i].astype(np.float64), p[i - 1].astype(np.float64), flow.BroxParams())
    np.savez(path, u=f.u, v=f.v, seconds=time.perf_counter() - t0)
    return path


def _encode_job(args):
    plane, g = args
    path = WORK / f"gop_{plane}_{g}.hivc"
    if path.exists():
        return path
    codec, flow, _, Frame = _ref()
    p = _planes3()[plane]
    s, e = g * GOP, min((g + 1) * GOP, NF)
    frames = [Frame((p[i],), colorspace="gray") for i in range(s, e)]
    flows = []
    for i in range(s + 1, e):
        z = np.load(WORK / f"flow_{plane}_{i:03d}.npz")
        flows.append(flow.FlowField(z["u"], z["v"]))
    cfg = codec.EncoderConfig(gop_size=GOP)
    t0 = time.perf_counter()
    stream = codec.encode(frames, cfg, _flows=[flows])
    dt = time.perf_counter() - t0
    path.write_bytes(stream)
    (WORK / f"gop_{plane}_{g}.json").write_text(json.dumps({"encode_s": dt}))
    return path


def _decode_job(args):
    plane, g = args
    codec, _, _, _ = _ref()
    stream = (WORK / f"gop_{plane}_{g}.hivc").read_bytes()
    timings = {}
    t0 = time.perf_counter()
    dec = codec.decode(stream, timings)
    dt = time.perf_counter() - t0
    rows = []
    for f in dec:
        a = f.planes[0].astype(np.uint8)
        rows.append((_sha(a.tobytes()), a.sum(axis=1).astype(np.int32), a.sum(axis=0).astype(np.int32)))
    return plane, g, rows, dt, timings


def make_cfg3(nproc: int = 8):
    planes = _planes3()
    del planes
    flow_jobs = [(pl, i) for pl in PLANES for i in range(NF) if i % GOP != 0]
    t0 = time.perf_counter()
    with Pool(nproc) as pool:
        for k, _ in enumerate(pool.imap_unordered(_flow_job, flow_jobs)):
            if k % 10 == 0:
                print(f"[cfg3] flows {k + 1}/{len(flow_jobs)}  {time.perf_counter() - t0:.0f}s", flush=True)
        gop_jobs = [(pl, g) for pl in PLANES for g in range(NF // GOP)]
        list(pool.imap_unordered(_encode_job, gop_jobs))
        print(f"[cfg3] encoded {time.perf_counter() - t0:.0f}s", flush=True)
        decoded = list(pool.imap_unordered(_decode_job, gop_jobs))
    print(f"[cfg3] decoded {time.perf_counter() - t0:.0f}s", flush=True)

    _, _, bs, _ = _ref()
    manifest = {}
    for pl in PLANES:
        payloads = []
        header0 = None
        for g in range(NF // GOP):
            h, pays = bs.read_stream((WORK / f"gop_{pl}_{g}.hivc").read_bytes())
            header0 = header0 or h
            payloads.extend(pays)
        header = bs.StreamHeader(
            width=header0.width,
            height=header0.height,
            frame_count=NF,
            fps_num=header0.fps_num,
            fps_den=header0.fps_den,
            gop_size=GOP,
            channels=1,
            intra_levels=header0.intra_levels,
            flow_levels=header0.flow_levels,
            residual_levels=header0.residual_levels,
        )
        stream = bs.write_stream(header, payloads)
        (STREAMS / f"cfg3_{pl}.hivc").write_bytes(stream)
        rows = sorted([d for d in decoded if d[0] == pl], key=lambda d: d[1])
        shas, rsum, csum = [], [], []
        dec_s = 0.0
        tim = {}
        for _, _, fr, dt, t in rows:
            dec_s += dt
            for k, v in t.items():
                tim[k] = tim.get(k, 0.0) + v
            for s, r, c in fr:
                shas.append(s)
                rsum.append(r)
                csum.append(c)
        np.savez_compressed(
            HERE / f"cfg3_{pl}_sums.npz", sha256=np.array(shas), row_sums=np.stack(rsum), col_sums=np.stack(csum)
        )
        enc_s = sum(json.loads((WORK / f"gop_{pl}_{g}.json").read_text())["encode_s"] for g in range(NF // GOP))
        manifest[f"cfg3_{pl}.hivc"] = {
            "sha256": _sha(stream),
            "bytes": len(stream),
            "reference_decode_s_1proc_sum": dec_s,
            "reference_encode_s_sum_excl_flow": enc_s,
            "timings": tim,
        }
    return manifest


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg0", "cfg3"]
    STREAMS.mkdir(parents=True, exist_ok=True)
    mpath = STREAMS / "manifest.json"
    manifest = json.loads(mpath.read_text()) if mpath.exists() else {}
    if "cfg0" in which:
        manifest.update(make_cfg0())
        mpath.write_text(json.dumps(manifest, indent=1, sort_keys=True))
    if "rgb" in which:
        manifest.update(make_rgb())
        mpath.write_text(json.dumps(manifest, indent=1, sort_keys=True))
    if "cfg3" in which:
        manifest.update(make_cfg3())
        mpath.write_text(json.dumps(manifest, indent=1, sort_keys=True))
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "timings"} for k, v in manifest.items()}, indent=1))
