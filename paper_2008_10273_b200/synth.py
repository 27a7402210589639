"""Seeded synthetic video content for the benchmark configurations.

BASELINE.json names no public dataset (the paper's Sintel clip is not in
this container), so every configuration runs on content drawn here, with
the shapes, sizes and value distributions SURVEY.md §8(d) fixes:

* frame t = sum of translated isotropic Gaussian blobs
  (sigma U[8,30] px, amplitude U[40,120] per channel)
  + axis-aligned constant rectangles (value U[0,255] per channel)
  + i.i.d. N(0, 2) noise drawn per frame and channel, clipped to [0, 255];
* every blob and rectangle moves at its own velocity U[-v, v]^2 px/frame.

Draw order from ``numpy.random.default_rng(seed)`` is fixed (centres,
sigmas, amplitudes, blob velocities, rectangle origins, sizes, values,
rectangle velocities, then per-frame noise) so a (seed, shape) pair
always yields the same clip.  This is harness code, not part of the
decode path.
"""

from __future__ import annotations

import numpy as np


def synth_frames(
    n_frames: int,
    height: int,
    width: int,
    blobs: int = 8,
    rects: int = 3,
    v: float = 3.0,
    seed: int = 0,
    channels: int = 1,
):
    """Frames of ``synth_clip`` one at a time (same draws, same values): a
    generator of float32 (channels, height, width) arrays, so long clips
    (config 4: 480 frames at 1080p) never sit in memory whole."""
    rng = np.random.default_rng(seed)
    bc = np.stack([rng.uniform(0, width, blobs), rng.uniform(0, height, blobs)], axis=1)
    bs = rng.uniform(8.0, 30.0, blobs)
    ba = rng.uniform(40.0, 120.0, (blobs, channels))
    bv = rng.uniform(-v, v, (blobs, 2))
    ro = np.stack([rng.uniform(0, width, rects), rng.uniform(0, height, rects)], axis=1)
    rs = np.stack(
        [rng.uniform(0.05 * width, 0.3 * width, rects), rng.uniform(0.05 * height, 0.3 * height, rects)],
        axis=1,
    )
    rval = rng.uniform(0.0, 255.0, (rects, channels))
    rv = rng.uniform(-v, v, (rects, 2))

    xs = np.arange(width, dtype=np.float64) + 0.5
    ys = np.arange(height, dtype=np.float64) + 0.5
    for t in range(n_frames):
        acc = np.zeros((channels, height, width))
        for i in range(blobs):
            cx, cy = bc[i] + bv[i] * t
            gx = np.exp(-((xs - cx) ** 2) / (2.0 * bs[i] ** 2))
            gy = np.exp(-((ys - cy) ** 2) / (2.0 * bs[i] ** 2))
            g = gy[:, None] * gx[None, :]
            for c in range(channels):
                acc[c] += ba[i, c] * g
        for i in range(rects):
            x0, y0 = ro[i] + rv[i] * t
            inx = (xs >= x0) & (xs < x0 + rs[i, 0])
            iny = (ys >= y0) & (ys < y0 + rs[i, 1])
            ind = iny[:, None] & inx[None, :]
            for c in range(channels):
                acc[c][ind] += rval[i, c]
        for c in range(channels):
            acc[c] += rng.normal(0.0, 2.0, (height, width))
        yield np.clip(acc, 0.0, 255.0).astype(np.float32)


def synth_clip(
    n_frames: int,
    height: int,
    width: int,
    blobs: int = 8,
    rects: int = 3,
    v: float = 3.0,
    seed: int = 0,
    channels: int = 1,
) -> np.ndarray:
    """Float32 clip of shape (n_frames, channels, height, width) in [0, 255]."""
    out = np.empty((n_frames, channels, height, width), dtype=np.float32)
    for t, f in enumerate(synth_frames(n_frames, height, width, blobs, rects, v, seed, channels)):
        out[t] = f
    return out


def to_codec_planes(clip: np.ndarray) -> np.ndarray:
    """Round half-even then clip to the codec's integer input domain."""
    return np.clip(np.rint(clip), 0, 255).astype(np.int32)


def downsample2(plane: np.ndarray) -> np.ndarray:
    """2x2 mean (ceil halving on odd sizes) for 4:2:0 chroma."""
    h, w = plane.shape[-2:]
    ph, pw = h + (h & 1), w + (w & 1)
    p = np.pad(plane.astype(np.float64), [(0, 0)] * (plane.ndim - 2) + [(0, ph - h), (0, pw - w)], mode="edge")
    return 0.25 * (p[..., 0::2, 0::2] + p[..., 1::2, 0::2] + p[..., 0::2, 1::2] + p[..., 1::2, 1::2])


def synth_420_frames(n_frames: int, height: int, width: int, blobs: int, rects: int, v: float, seed: int):
    """``synth_420`` one frame at a time: yields (Y, Cb, Cr) int32 planes."""
    for f in synth_frames(n_frames, height, width, blobs, rects, v, seed, channels=3):
        yield (to_codec_planes(f[0]), to_codec_planes(downsample2(f[1])), to_codec_planes(downsample2(f[2])))


def synth_420(n_frames: int, height: int, width: int, blobs: int, rects: int, v: float, seed: int):
    """4:2:0 clip as three integer plane stacks: Y (H, W), Cb and Cr (H/2, W/2).

    The chroma planes come from the same geometry with per-channel values,
    generated at full resolution and 2x2-mean downsampled, then rounded.
    """
    clip = synth_clip(n_frames, height, width, blobs, rects, v, seed, channels=3)
    y = to_codec_planes(clip[:, 0])
    cb = to_codec_planes(downsample2(clip[:, 1]))
    cr = to_codec_planes(downsample2(clip[:, 2]))
    return y, cb, cr


def random_mask(shape, density: float, seed: int) -> np.ndarray:
    """Uniform-random known-pixel mask (config 0 function check, config 1)."""
    return np.random.default_rng(seed).uniform(size=shape) < density
