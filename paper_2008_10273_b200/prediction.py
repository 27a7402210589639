"""Per-frame prediction signals on the B200 (reference: prediction.py).

``decode_intra`` (prediction.py:185-208): native tree/tANS parse, then the
GPU cascadic-CG solve per channel with the decoder's fixed budget
(tol 1e-4, 160 iterations, non-strict).  ``predict_inter``
(prediction.py:220-223): GPU bilinear backward warp.
"""

from __future__ import annotations

import struct

import numpy as np

from paper_2008_10273_b200.entropy import decode_symbols
from paper_2008_10273_b200.errors import QuantizeError, TruncatedStream
from paper_2008_10273_b200.flow import _tree_leaves, warp_planes
from paper_2008_10273_b200.homogeneous import solve_homogeneous

INTRA_SOLVE_ITERS = 160  # prediction.py:35
INTRA_SOLVE_TOL = 1e-4  # prediction.py:36


def chroma_levels(levels: int) -> int:
    return 2 * levels - 1  # prediction.py:111-114


def _read_tree(data: bytes, pos: int, width: int, height: int):
    if pos + 4 > len(data):  # prediction.py:149-159
        raise TruncatedStream("intra payload truncated")
    (nbits,) = struct.unpack_from("<I", data, pos)
    pos += 4
    nbytes = (nbits + 7) // 8
    if pos + nbytes > len(data):
        raise TruncatedStream("intra payload truncated")
    leaves = _tree_leaves(data, pos, nbits, width, height)
    mask = np.zeros((height, width), dtype=bool)
    if len(leaves):
        mask[leaves[:, 1] + leaves[:, 3] // 2, leaves[:, 0] + leaves[:, 2] // 2] = True
    return mask, pos + nbytes


def _decode_plane_values(data: bytes, pos: int, levels: int):
    if pos + 4 > len(data):  # prediction.py:133-139
        raise TruncatedStream("intra payload truncated")
    lo, hi = struct.unpack_from("<hh", data, pos)
    idx, pos = decode_symbols(data, pos + 4)
    lo, hi = float(lo), float(hi)
    if not lo < hi:
        raise QuantizeError("need lo < hi")
    return lo + idx.astype(np.float64) * ((hi - lo) / (levels - 1)), pos


def decode_intra(data: bytes, pos: int, shape, channels: int, levels: int):
    """Decode an intra payload into float prediction planes; returns (planes, next position)."""
    h, w = shape
    mask_y, pos = _read_tree(data, pos, w, h)
    vals_y, pos = _decode_plane_values(data, pos, levels)
    jobs = [(mask_y, vals_y)]
    if channels == 3:
        mask_c, pos = _read_tree(data, pos, w, h)
        for _ in range(2):
            vals, pos = _decode_plane_values(data, pos, chroma_levels(levels))
            jobs.append((mask_c, vals))
    planes = []
    for mask, vals in jobs:
        f = np.zeros(mask.shape)
        f.ravel()[np.flatnonzero(mask.ravel())] = vals
        planes.append(solve_homogeneous(f, mask, tol=INTRA_SOLVE_TOL, max_iter=INTRA_SOLVE_ITERS, strict=False))
    return planes, pos


def predict_inter(prev_planes, flow):
    """Motion-compensated prediction: previous reconstruction sampled at (x+u, y+v)."""
    return warp_planes([np.asarray(p, dtype=np.float64) for p in prev_planes], flow.u, flow.v)
