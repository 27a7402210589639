"""Golden vectors for the encoder primitives,
produced by importing the REFERENCE here:

    OMP_NUM_THREADS=1 python tests/golden/make_encoder.py   ->  tests/golden/golden_encoder.npz

Cases:
  sub*      subdivision.subdivide_by_error trees (bits + preorder leaves) on
            integer planes, float (flow-like) planes with min_error=0, joint
            two-plane errors, 8x8 tiles and a constant plane;
  means*    subdivision.leaf_means of float planes over those trees;
  flow*     flow.compress_flow payloads of smooth synthetic flow fields;
  res*      codec._encode_residual payloads of integer residual planes
            (1 and 3 planes, ragged sizes, lambda 0 / 1, 4 and 9 points);
  intra*    prediction.encode_intra payloads (gray and 3-plane).
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

from paper_2008_10273_b200.synth import synth_clip  # noqa: E402


def _smooth(rng, h, w, k=6, amp=3.0):
    """Sum of random Gaussian bumps: a flow-like smooth float field."""
    yy, xx = np.mgrid[0:h, 0:w]
    out = np.zeros((h, w))
    for _ in range(k):
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        s = rng.uniform(0.1, 0.4) * max(h, w)
        out += rng.normal(0, amp) * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * s * s))
    return out


def _residual(rng, h, w, scale=6.0, frac=0.3):
    r = np.rint(rng.laplace(0, scale, (h, w))).astype(np.int64)
    keep = rng.uniform(size=(h // 8 + 1, w // 8 + 1)) < frac  # most tiles zero, like a real P-frame
    return r * np.kron(keep, np.ones((8, 8), dtype=np.int64))[:h, :w]


def main():
    from hivc import codec as rc
    from hivc import flow as rf
    from hivc import prediction as rp
    from hivc import subdivision as rs

    g = {}
    rng = np.random.default_rng(31)
    clip = synth_clip(1, 60, 84, blobs=5, rects=2, v=2.0, seed=32, channels=3)[0]
    ints = np.clip(np.rint(clip[0]), 0, 255).astype(np.float64)
    flt = _smooth(rng, 61, 83)  # float64 (the encoder subdivides float64 planes)
    u2, v2 = _smooth(rng, 45, 70), _smooth(rng, 45, 70)
    sub_cases = [
        ("int", [ints], 400, None),
        ("flt", [flt], 100, 0.0),
        ("flt_full", [flt], 700, None),
        ("joint", [u2, v2], 250, None),
        ("tile", [np.asarray(rng.integers(-9, 9, (8, 8)), dtype=np.float64)], 4, None),
        ("tile_ragged", [np.asarray(rng.integers(-9, 9, (5, 8)), dtype=np.float64)], 9, None),
        ("const", [np.full((33, 17), 2.5)], 50, 0.0),
        ("ties", [np.tile(np.array([[0.0, 1.0], [1.0, 0.0]]), (16, 16))], 64, None),
    ]
    for i, (name, planes, target, min_error) in enumerate(sub_cases):
        err = rs.joint_ssd_error(planes) if len(planes) > 1 else None
        tree = rs.subdivide_by_error(planes[0], target, error_fn=err, min_error=min_error)
        g[f"sub{i}_name"] = np.array(name)
        g[f"sub{i}_planes"] = np.stack(planes)
        g[f"sub{i}_target"] = np.array(target)
        g[f"sub{i}_min_error"] = np.array(np.nan if min_error is None else min_error)
        g[f"sub{i}_bits"] = np.array(tree.bits, dtype=np.uint8)
        g[f"sub{i}_leaves"] = np.array(tree.leaves(), dtype=np.int32)
        g[f"sub{i}_means"] = rs.leaf_means(tree, planes[0])

    for i, (h, w, budget, levels) in enumerate([(61, 83, 100, 256), (45, 70, 37, 64), (20, 30, 5, 256)]):
        f = rf.FlowField(_smooth(rng, h, w, amp=2.0), _smooth(rng, h, w, amp=2.0))
        g[f"flow{i}_u"], g[f"flow{i}_v"] = f.u, f.v
        g[f"flow{i}_cfg"] = np.array([budget, levels])
        g[f"flow{i}_payload"] = np.frombuffer(rf.compress_flow(f, budget, levels), dtype=np.uint8)
    # zero flow: a single-leaf tree per component (min_error early stop)
    z = rf.FlowField(np.zeros((24, 40)), np.zeros((24, 40)))
    g["flow3_u"], g["flow3_v"], g["flow3_cfg"] = z.u, z.v, np.array([100, 256])
    g["flow3_payload"] = np.frombuffer(rf.compress_flow(z, 100, 256), dtype=np.uint8)

    res_cases = [
        (1, 72, 96, 4, 63, 1.0),
        (1, 61, 83, 4, 63, 0.0),
        (3, 45, 70, 4, 63, 1.0),
        (1, 40, 56, 9, 31, 0.5),
        (3, 27, 35, 7, 63, 0.0),
    ]
    for i, (nch, h, w, pts, levels, lam) in enumerate(res_cases):
        planes = [_residual(rng, h, w, scale=6.0 if c == 0 else 9.0) for c in range(nch)]
        g[f"res{i}_planes"] = np.stack(planes)
        g[f"res{i}_cfg"] = np.array([pts, levels, lam])
        g[f"res{i}_payload"] = np.frombuffer(rc._encode_residual(planes, pts, levels, lam), dtype=np.uint8)
        # the tile plan of the Y group (codec._plan_group): coded tiles, 8x8 masks, tree bits
        tiles = __import__("hivc.pseudodiff", fromlist=["block_grid"]).block_grid(h, w)
        coded, trees, masks = rc._plan_group(planes[:1], tiles, pts)
        g[f"res{i}_plan_coded"] = np.array(coded, dtype=np.int64)
        g[f"res{i}_plan_masks"] = np.array(masks, dtype=bool).reshape(-1, 64)
        g[f"res{i}_plan_bits"] = np.array([b for t in trees for b in t.bits], dtype=np.uint8)
        if nch == 3:
            coded, trees, masks = rc._plan_group(planes[1:], tiles, pts)
            g[f"res{i}_plan2_coded"] = np.array(coded, dtype=np.int64)
            g[f"res{i}_plan2_masks"] = np.array(masks, dtype=bool).reshape(-1, 64)
            g[f"res{i}_plan2_bits"] = np.array([b for t in trees for b in t.bits], dtype=np.uint8)
    # an all-zero residual: the 1-byte empty marker
    g["res5_planes"] = np.zeros((1, 16, 24), dtype=np.int64)
    g["res5_cfg"] = np.array([4, 63, 1.0])
    g["res5_payload"] = np.frombuffer(rc._encode_residual([g["res5_planes"][0]], 4, 63, 1.0), dtype=np.uint8)

    clip3 = synth_clip(1, 48, 64, blobs=4, rects=2, v=2.0, seed=33, channels=3)[0]
    gray = np.clip(np.rint(clip3[0]), 0, 255).astype(np.int64)
    yuv = [gray, np.rint(clip3[1] - clip3[0]).astype(np.int64), np.rint(clip3[2] - clip3[0]).astype(np.int64)]
    for i, (planes, budget, levels) in enumerate([([gray], 180, 256), (yuv, 250, 256), ([gray], 48 * 64, 64)]):
        g[f"intra{i}_planes"] = np.stack(planes)
        g[f"intra{i}_cfg"] = np.array([budget, levels])
        g[f"intra{i}_payload"] = np.frombuffer(rp.encode_intra(planes, budget, levels), dtype=np.uint8)

    # Horn-Schunck baseline flow (flow.py:281-316) on a small synthetic pair
    pair = synth_clip(2, 40, 56, blobs=4, rects=2, v=2.0, seed=34)[:, 0].astype(np.float64)
    hs = rf.flow_horn_schunck(pair[1], pair[0])
    g["hs_pair"], g["hs_u"], g["hs_v"] = pair, hs.u, hs.v
    hs2 = rf.flow_horn_schunck(pair[1], pair[0], alpha=5.0, iterations=7)
    g["hs2_u"], g["hs2_v"] = hs2.u, hs2.v

    # whole-encoder cases: Horn-Schunck flows, and encode_target_ratio's bisection (codec.py:604-642)
    from hivc.frame import Frame

    clip5 = np.clip(np.rint(synth_clip(5, 40, 52, blobs=3, rects=2, v=2.0, seed=35)[:, 0]), 0, 255).astype(np.int32)
    frames = [Frame((p,), colorspace="gray") for p in clip5]
    g["enc_hs_frames"] = clip5
    g["enc_hs_stream"] = np.frombuffer(
        rc.encode(frames, rc.EncoderConfig(gop_size=3, intra_mask_fraction=0.1, flow_method="horn-schunck")),
        dtype=np.uint8)
    stream, ratio, cfg = rc.encode_target_ratio(frames, rc.EncoderConfig(gop_size=5, intra_mask_fraction=0.05), 10.0)
    g["enc_tr_stream"] = np.frombuffer(stream, dtype=np.uint8)
    g["enc_tr_ratio"] = np.array(ratio)
    g["enc_tr_cfg"] = np.array([cfg.intra_mask_fraction, cfg.residual_points, cfg.flow_points, cfg.intra_levels,
                                cfg.residual_levels, cfg.residual_lambda])

    np.savez_compressed(HERE / "golden_encoder.npz", **g)
    print(f"wrote {len(g)} arrays")


if __name__ == "__main__":
    main()
