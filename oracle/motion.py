"""Oracle: backward bilinear warp and flow-payload decoding (TEST INFRASTRUCTURE ONLY).

Restates reference ``flow.py:94-132`` (warp) and ``343-372`` (flow
decompression).  The Brox estimator oracle lives in ``oracle/brox.py``.
"""

from __future__ import annotations

import struct

import numpy as np

from oracle.parse import Bits, Truncated, decode_symbols, paint, tree_leaves, uniform_dequant


def warp(planes, u: np.ndarray, v: np.ndarray):
    """Sample every plane at (x + u, y + v), clamped bilinear (``flow.py:94-127``).

    Coordinates are clamped before flooring; the four taps are summed in
    the order w00*p00 + w01*p01 + w10*p10 + w11*p11.
    """
    h, w = planes[0].shape
    gy, gx = np.mgrid[0:h, 0:w]
    sx = np.clip(gx + u, 0, w - 1)
    sy = np.clip(gy + v, 0, h - 1)
    ix0 = np.floor(sx).astype(np.int64)
    iy0 = np.floor(sy).astype(np.int64)
    ix1 = np.minimum(ix0 + 1, w - 1)
    iy1 = np.minimum(iy0 + 1, h - 1)
    ax = sx - ix0
    ay = sy - iy0
    k00 = (1 - ay) * (1 - ax)
    k01 = (1 - ay) * ax
    k10 = ay * (1 - ax)
    k11 = ay * ax
    res = []
    for p in planes:
        q = np.ascontiguousarray(p, dtype=np.float64)
        res.append(k00 * q[iy0, ix0] + k01 * q[iy0, ix1] + k10 * q[iy1, ix0] + k11 * q[iy1, ix1])
    return res


def decode_flow_component(data: bytes, pos: int, shape, levels: int):
    """One flow component: f32 lo/hi, u32 nbits, tree, tANS leaf indices (``flow.py:343-356``)."""
    if pos + 12 > len(data):
        raise Truncated("flow payload truncated")
    lo, hi, nbits = struct.unpack_from("<ffI", data, pos)
    pos += 12
    nb = (nbits + 7) // 8
    if pos + nb > len(data):
        raise Truncated("flow payload truncated")
    leaves = tree_leaves(Bits(data[pos : pos + nb], nbits), shape[1], shape[0])
    pos += nb
    idx, pos = decode_symbols(data, pos)
    vals = uniform_dequant(idx, float(lo), float(hi), levels)
    return paint(leaves, vals, shape[1], shape[0]), pos


def decode_flow(data: bytes, pos: int, shape, levels: int):
    """(u, v, next pos) — reference ``flow.py:368-372``."""
    u, pos = decode_flow_component(data, pos, shape, levels)
    v, pos = decode_flow_component(data, pos, shape, levels)
    if not (np.isfinite(u).all() and np.isfinite(v).all()):
        raise ValueError("non-finite flow values")
    return u, v, pos
