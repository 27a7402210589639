"""Function-level microbenchmarks of BASELINE.json configs 1, 2 and the Brox part of 4.

    python tools/microbench.py [--reps R] [--cpu]

One JSON line per measurement.  GPU times: wall clock around calls that
synchronise their own CUDA stream (the C ABI returns after the device work),
median of R repetitions after one warm-up.  --cpu also times the oracle port
(the reference algorithm in numpy) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def config1(reps, cpu):
    import torch

    from paper_2008_10273_b200.homogeneous import solve_homogeneous
    from paper_2008_10273_b200.synth import random_mask, synth_clip

    clip = synth_clip(1, 1080, 1920, blobs=40, rects=12, v=6.0, seed=1, channels=3)[0].astype(np.float64)
    m = random_mask((1080, 1920), 0.02, 1001)
    mt = torch.from_numpy(m).cuda()
    fs = [torch.from_numpy(np.where(m, clip[c], 0.0)).cuda() for c in range(3)]
    stats = []

    def run():
        stats.clear()
        for f in fs:
            st = {}
            solve_homogeneous(f, mt, tol=1e-6, max_iter=10000, strict=True, stats=st)
            stats.append(st["level_iterations"])

    dt = timed(run, reps)
    alg = sum(n * (49 * it + 49) for s in stats for n, it in s)
    line = {"config": 1, "what": "homogeneous inpainting 1080p x3 channels, 2% random mask, tol 1e-6, strict",
            "seconds": dt, "seconds_per_channel": dt / 3, "level_iterations": stats[0],
            "total_iterations": [sum(it for _, it in s) for s in stats],
            "algorithmic_GBps": alg / dt / 1e9, "dtype": "f64"}
    if cpu:
        from oracle import inpaint

        t0 = time.perf_counter()
        inpaint.solve(np.where(m, clip[0], 0.0), m, tol=1e-6, max_iter=10000, strict=True)
        line["cpu_oracle_seconds_per_channel"] = time.perf_counter() - t0
    print(json.dumps(line), flush=True)


def config2(reps, cpu):
    import torch
    from scipy.ndimage import uniform_filter

    from paper_2008_10273_b200.pseudodiff import FLAT_BLOCK_MASK, reconstruct_plane_masks, reconstruct_plane_shared_mask

    rng = np.random.default_rng(2)
    res = uniform_filter(rng.laplace(0.0, 8.0, (1080, 1920)), size=3, mode="reflect").astype(np.float32)
    nblk = 135 * 240
    rt = torch.from_numpy(res).cuda()
    dt = timed(lambda: reconstruct_plane_shared_mask(rt), reps)
    # the floor for moving the same bytes in one launch: a device copy of the plane (8.3 MB in + 8.3 MB out)
    dst = torch.empty_like(rt)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    cps = []
    for _ in range(reps + 2):
        ev[0].record()
        dst.copy_(rt)
        ev[1].record()
        torch.cuda.synchronize()
        cps.append(ev[0].elapsed_time(ev[1]) * 1e-3)
    cp = statistics.median(cps[2:])
    print(json.dumps({"config": "2a", "what": "shared 4-point mask, fit+rebuild as one 64x64 operator, 3xTF32 tcgen05 "
                      "(TMA-fed persistent kernel)", "blocks": nblk, "seconds": dt, "blocks_per_s": nblk / dt,
                      "GBps": nblk * 512 / dt / 1e9, "flops_per_block": 3 * 2 * 64 * 64,
                      "same_bytes_device_copy_seconds": cp,
                      "note": "seconds: through the API (host call + launch + sync); the kernel alone is in the ncu "
                              "capture; a plain device copy of the same 16.6 MB is the one-launch floor at this size"}),
          flush=True)
    mrng = np.random.default_rng(1002)
    masks = mrng.uniform(size=(nblk, 8, 8)) < 0.05
    empty = ~masks.reshape(nblk, 64).any(1)
    for i in np.flatnonzero(empty):
        masks[i, mrng.integers(0, 8), mrng.integers(0, 8)] = True
    from paper_2008_10273_b200.pseudodiff import _mask_words

    words = torch.from_numpy(_mask_words(masks).view(np.int64)).cuda()
    dt = timed(lambda: reconstruct_plane_masks(rt, words), reps)  # masks resident on the device
    ks = masks.reshape(nblk, 64).sum(1)
    print(json.dumps({"config": "2b", "what": "per-block Bernoulli(0.05) masks, float64 smem bordered solves",
                      "blocks": nblk, "seconds": dt, "blocks_per_s": nblk / dt,
                      "GBps": float(np.sum(520 + 4 * (ks + 1))) / dt / 1e9,
                      "k_hist": np.bincount(ks).tolist()}), flush=True)


def config4_brox(reps, cpu):
    import torch

    from paper_2008_10273_b200.flow import BroxParams, flow_brox
    from paper_2008_10273_b200.synth import synth_clip

    clip = synth_clip(2, 1080, 1920, blobs=40, rects=12, v=6.0, seed=4)[:, 0].astype(np.float64)
    a, b = torch.from_numpy(clip[1]).cuda(), torch.from_numpy(clip[0]).cuda()
    for sc in (0.95, 0.5):
        dt = timed(lambda: flow_brox(a, b, BroxParams(pyramid_scale=sc)), reps)
        print(json.dumps({"config": 4, "what": f"Brox flow 1080p pair, pyramid_scale {sc}", "seconds_per_pair": dt,
                          "pairs_per_s": 1 / dt, "dtype": "f64",
                          "cpu_reference_seconds_per_pair_survey": 948.2 if sc == 0.95 else 126.4}), flush=True)


def tonal(reps, cpu):
    """prediction.optimize_mask_values on a 1080p luma
    I-frame with the reference encoder's own mask (config-3 Y stream, GOP 0)."""
    import ctypes as C

    from paper_2008_10273_b200 import _native as N
    from paper_2008_10273_b200.prediction import optimize_mask_values
    from paper_2008_10273_b200.synth import synth_420

    data = (REPO / "tests/golden/streams/cfg3_Y.hivc").read_bytes()
    h, w = 1080, 1920
    # mask points of GOP 0's I-frame: the first frame record's tree (native parser)
    pos = 22 + 4 + 2 + 5
    nbits = int.from_bytes(data[pos:pos + 4], "little")
    cap = h * w
    rects = (C.c_int32 * (4 * cap))()
    nl, used = C.c_size_t(), C.c_uint64()
    blob = data[pos + 4: pos + 4 + (nbits + 7) // 8]
    N.check(N.lib.hivc_parse_tree(blob, len(blob), nbits, 0, w, h, rects, cap, C.byref(nl), C.byref(used)))
    r = np.frombuffer(rects, dtype=np.int32)[: 4 * nl.value].reshape(-1, 4)
    mask = np.zeros((h, w), bool)
    mask[r[:, 1] + r[:, 3] // 2, r[:, 0] + r[:, 2] // 2] = True
    y = synth_420(1, h, w, blobs=40, rects=12, v=6.0, seed=3)[0][0].astype(np.float64)
    st = {}
    sec = timed(lambda: optimize_mask_values([y], mask, stats=st), reps)
    print(json.dumps({"config": "f1", "what": "tonal optimisation (LSQR x12 over GPU inpainting solves), 1080p luma "
                      "I-frame, reference encoder mask", "mask_points": int(mask.sum()), "seconds": sec,
                      "solver_iterations": st.get("solver_iterations"),
                      "cpu_reference_seconds_survey": 112.0}), flush=True)


def encoder_parts(reps, cpu):
    """SURVEY §8(f) ranks 2-3 on 1080p content (config-3 luma, frames 0-1):
    the residual encoder on the frame-difference residual, the 9 % intra
    subdivision and the tANS encode of its 186,624 values.  Reference CPU
    times (1 core, measured in the build container with the reference package):
    _encode_residual 6.08 s, subdivide_by_error 7.38 s, encode_symbols 0.177 s."""
    import torch

    from paper_2008_10273_b200.encoder import _encode_residual_rec
    from paper_2008_10273_b200.entropy import encode_symbols
    from paper_2008_10273_b200.subdivision import subdivide_by_error
    from paper_2008_10273_b200.synth import synth_420

    y, _, _ = synth_420(2, 1080, 1920, blobs=40, rects=12, v=6.0, seed=3)
    res = y[1].astype(np.int64) - y[0].astype(np.int64)
    dt = timed(lambda: (_encode_residual_rec([res], 4, 63, 1.0), torch.cuda.synchronize()), reps)
    print(json.dumps({"config": "f2", "what": "residual encoder, 1080p frame-difference residual (tile plans C++, "
                      "GPU fits + keep rebuilds, tANS)", "seconds": dt, "cpu_reference_seconds": 6.08}), flush=True)
    p = y[0].astype(np.float64)
    target = int(round(0.09 * p.size))
    dt = timed(lambda: subdivide_by_error(p, target), reps)
    print(json.dumps({"config": "f3", "what": "intra subdivision 1080p, 9 % (186,624 leaves), numpy-order float64",
                      "seconds": dt, "cpu_reference_seconds": 7.38}), flush=True)
    sym = np.random.default_rng(0).integers(0, 256, 186624)
    dt = timed(lambda: encode_symbols(sym), reps)
    print(json.dumps({"config": "f3", "what": "tANS encode of 186,624 symbols (256-letter alphabet)",
                      "seconds": dt, "cpu_reference_seconds": 0.177}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--only", default="1,2,4,f1,f2")
    a = ap.parse_args()
    only = a.only.split(",")
    if "1" in only:
        config1(a.reps, a.cpu)
    if "2" in only:
        config2(a.reps, a.cpu)
    if "4" in only:
        config4_brox(max(1, a.reps // 2), a.cpu)
    if "f1" in only:
        tonal(max(1, a.reps // 2), a.cpu)
    if "f2" in only:
        encoder_parts(max(1, a.reps // 2), a.cpu)


if __name__ == "__main__":
    main()
