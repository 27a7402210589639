"""Error-driven rectangular subdivision through the native encoder (reference: subdivision.py).

``subdivide_by_error`` (subdivision.py:76-130) runs the greedy worst-leaf
split in C++ (csrc/encode.cpp) with region errors summed in numpy's exact
float64 association order, so trees (and the bits serialised from them) are
identical to the reference's.  ``error_fn`` accepts the reference's two
error rules: ``None`` (region_ssd, subdivision.py:133-135) and
``joint_ssd_error(planes)`` (subdivision.py:138-144).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from paper_2008_10273_b200 import _native as N
from paper_2008_10273_b200.errors import SubdivisionError


@dataclass(frozen=True)
class SubdivisionTree:
    """Preorder split bits over a root rectangle (subdivision.py:38-73), with the
    preorder leaf rectangles (x, y, w, h) the encoder already knows."""

    x: int
    y: int
    w: int
    h: int
    bits: tuple
    rects: np.ndarray  # (n_leaves, 4) int32, preorder

    def leaves(self):
        return [tuple(int(v) for v in r) for r in self.rects]

    @property
    def leaf_count(self):
        return int(self.rects.shape[0])

    @property
    def packed(self) -> bytes:
        """Tree bits as serialize_tree writes them (MSB first, zero-padded)."""
        return np.packbits(np.asarray(self.bits, dtype=np.uint8)).tobytes()


class _JointError:
    def __init__(self, planes):
        self.planes = [np.ascontiguousarray(p, dtype=np.float64) for p in planes]


def joint_ssd_error(planes):
    """Error rule summing region SSD over several planes (chroma rule)."""
    return _JointError(planes)


def split_children(x: int, y: int, w: int, h: int):
    """Children of a rectangle: halve the longer side, ties halve width (subdivision.py:25-35)."""
    if w < 1 or h < 1:
        raise SubdivisionError(f"degenerate rectangle {w}x{h}")
    if w == 1 and h == 1:
        raise SubdivisionError("cannot split a single pixel")
    if h > w:
        h1 = (h + 1) // 2
        return (x, y, w, h1), (x, y + h1, w, h - h1)
    w1 = (w + 1) // 2
    return (x, y, w1, h), (x + w1, y, w - w1, h)


def subdivide_by_error(plane, target_points: int, error_fn=None, min_error=None) -> SubdivisionTree:
    """Greedy split of the worst-error leaf until ``target_points`` leaves exist."""
    p = np.ascontiguousarray(plane, dtype=np.float64)
    if p.ndim != 2:
        raise SubdivisionError("expected a 2-D plane")
    h, w = p.shape
    target_points = int(target_points)
    if target_points < 1:
        raise SubdivisionError("target_points must be >= 1")
    if target_points > w * h:
        raise SubdivisionError("target_points exceeds pixel count")
    if error_fn is None:
        planes = [p]
    elif isinstance(error_fn, _JointError):
        planes = error_fn.planes
        if any(q.shape != p.shape for q in planes):
            raise SubdivisionError("joint error planes must match the plane's shape")
    else:
        raise SubdivisionError("error_fn must be None or joint_ssd_error(planes)")
    arr = (C.c_void_p * len(planes))(*[q.ctypes.data for q in planes])
    bits = np.zeros((2 * target_points - 1 + 7) // 8 + 1, dtype=np.uint8)
    rects = np.empty((target_points, 4), dtype=np.int32)
    nbits, nleaves = C.c_uint64(), C.c_size_t()
    N.check(N.lib.hivc_subdivide(arr, len(planes), w, h, target_points, int(min_error is not None),
                                 float(min_error or 0.0), bits.ctypes.data, C.byref(nbits), rects.ctypes.data,
                                 C.byref(nleaves)))
    b = tuple(int(v) for v in np.unpackbits(bits)[: nbits.value])
    return SubdivisionTree(0, 0, w, h, b, rects[: nleaves.value].copy())


def region_ssd(plane, x: int, y: int, w: int, h: int) -> float:
    region = np.asarray(plane)[y : y + h, x : x + w]
    return float(np.sum((region - region.mean()) ** 2))


def mask_from_tree(tree: SubdivisionTree) -> np.ndarray:
    """Boolean mask with one point at the floor midpoint of each leaf (subdivision.py:147-152)."""
    mask = np.zeros((tree.h, tree.w), dtype=bool)
    r = tree.rects
    mask[r[:, 1] + r[:, 3] // 2, r[:, 0] + r[:, 2] // 2] = True
    return mask


def leaf_means(tree: SubdivisionTree, plane) -> np.ndarray:
    """Mean of ``plane`` over each leaf, preorder, in numpy's summation order (subdivision.py:155-159)."""
    p = np.ascontiguousarray(plane, dtype=np.float64)
    rects = np.ascontiguousarray(tree.rects, dtype=np.int32)
    out = np.empty(rects.shape[0])
    N.check(N.lib.hivc_region_means(p.ctypes.data, p.shape[1], p.shape[0], rects.ctypes.data, rects.shape[0],
                                    out.ctypes.data))
    return out


def serialize_tree(tree: SubdivisionTree, writer):
    """Append the preorder bits to a ``bits.BitWriter``-like writer (subdivision.py:178-181)."""
    for b in tree.bits:
        writer.write_bit(b)
