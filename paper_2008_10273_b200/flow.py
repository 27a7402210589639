"""Backward flow: warping and flow-payload decoding on the B200 (reference: flow.py).

``warp_planes`` / ``bilinear_warp`` keep the reference signatures
(flow.py:94-132) and run ``hivc_warp`` (csrc/recon.cu) in float64 with the
reference's clamp-then-floor coordinates and tap order.  Inside
``codec.decode`` the warp is fused with the residual and rounding and the
dense flow field is never materialised (csrc/recon.cu: frame_kernel).
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from paper_2008_10273_b200 import _native as N
from paper_2008_10273_b200._tensors import back, is_cuda_tensor, ptr, to_device, torch
from paper_2008_10273_b200.errors import FlowError


@dataclass(frozen=True)
class FlowField:
    u: object  # horizontal displacement, pixels
    v: object  # vertical displacement, pixels

    def __post_init__(self):  # flow.py:45-49
        if tuple(self.u.shape) != tuple(self.v.shape):
            raise FlowError("flow component shape mismatch")
        if is_cuda_tensor(self.u):
            t = torch()
            ok = bool(t.isfinite(self.u).all()) and bool(t.isfinite(self.v).all())
        else:
            ok = bool(np.isfinite(self.u).all() and np.isfinite(self.v).all())
        if not ok:
            raise FlowError("non-finite flow values")

    @property
    def shape(self):
        return tuple(self.u.shape)


@dataclass(frozen=True)
class BroxParams:  # flow.py:56-66
    alpha: float = 40.0
    gamma: float = 40.0
    pyramid_scale: float = 0.5
    min_size: int = 16
    warps: int = 3
    fixed_point_iters: int = 5
    solver_iters: int = 30
    eps: float = 1e-3
    presmooth_sigma: float = 0.8


def warp_planes(planes, u, v):
    """Sample each plane at (x + u, y + v), bilinear with border clamping (flow.py:94-127)."""
    t = torch()
    ut = to_device(u, t.float64)
    dev = ut.device
    vt = to_device(v, t.float64, dev)
    h, w = ut.shape
    src = [to_device(p, t.float64, dev) for p in planes]
    for s in src:
        if tuple(s.shape) != (h, w):
            raise ValueError("plane/flow shape mismatch")
    dst = [t.empty_like(s) for s in src]
    ctx = N.context(dev.index)
    t.cuda.current_stream(dev).synchronize()
    sp = (C.c_void_p * len(src))(*[ptr(s) for s in src])
    dp = (C.c_void_p * len(dst))(*[ptr(d) for d in dst])
    N.check(N.lib.hivc_warp(ctx.handle, sp, len(src), ptr(ut), ptr(vt), h, w, dp))
    return [back(d, p) for d, p in zip(dst, planes)]


def bilinear_warp(plane, u, v):
    """Sample plane at (x + u, y + v) with bilinear interpolation, clamped (flow.py:130-132)."""
    return warp_planes([plane], u, v)[0]


def _gaussian_taps(sigma: float, truncate: float = 4.0) -> np.ndarray:
    """scipy.ndimage's normalised 1-D Gaussian taps (gaussian_filter1d, order 0);
    computed with numpy exactly as scipy does so the device filter is bit-identical."""
    radius = int(truncate * float(sigma) + 0.5)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
    return np.ascontiguousarray(phi / phi.sum(), dtype=np.float64)


def flow_brox(frame_t, frame_prev, params: BroxParams | None = None) -> FlowField:
    """Backward flow from frame_t to frame_prev, coarse-to-fine with warping (flow.py:187-278).

    The whole estimator runs on the GPU in float64 (csrc/brox.cu).  numpy
    inputs give a numpy FlowField; CUDA tensors keep u, v on the device.
    """
    if params is None:
        params = BroxParams()
    t = torch()
    f1 = to_device(frame_t, t.float64)
    f0 = to_device(frame_prev, t.float64, f1.device)
    if tuple(f1.shape) != tuple(f0.shape) or f1.dim() != 2:
        raise FlowError("frame shape mismatch")
    if not (bool(t.isfinite(f1).all()) and bool(t.isfinite(f0).all())):
        raise FlowError("non-finite input planes")
    h, w = f1.shape
    u = t.empty_like(f1)
    v = t.empty_like(f1)
    prm = N.BroxParamsC(params.alpha, params.gamma, params.pyramid_scale, params.min_size, params.warps,
                        params.fixed_point_iters, params.solver_iters, params.eps, params.presmooth_sigma)
    tp = _gaussian_taps(params.presmooth_sigma) if params.presmooth_sigma > 0 else np.ones(1)
    ta = _gaussian_taps(0.5 / params.pyramid_scale)
    ctx = N.context(f1.device.index)
    t.cuda.current_stream(f1.device).synchronize()
    N.check(N.lib.hivc_brox(ctx.handle, ptr(f1), ptr(f0), h, w, C.byref(prm), tp.ctypes.data_as(N.c_dbl_p), tp.size,
                            ta.ctypes.data_as(N.c_dbl_p), ta.size, ptr(u), ptr(v)))
    return FlowField(back(u, frame_t), back(v, frame_t))


def flow_horn_schunck(frame_t, frame_prev, alpha: float = 15.0, iterations: int = 400) -> FlowField:
    """Quadratic-penalty flow, Jacobi sweeps on the Euler-Lagrange equations (flow.py:281-316),
    on the GPU in float64 (csrc/brox.cu: hs_deriv_kernel, hs_iter_kernel)."""
    t = torch()
    f1 = to_device(frame_t, t.float64)
    f0 = to_device(frame_prev, t.float64, f1.device)
    if tuple(f1.shape) != tuple(f0.shape) or f1.dim() != 2:
        raise FlowError("frame shape mismatch")
    if not (bool(t.isfinite(f1).all()) and bool(t.isfinite(f0).all())):
        raise FlowError("non-finite input planes")
    h, w = f1.shape
    u = t.empty_like(f1)
    v = t.empty_like(f1)
    ctx = N.context(f1.device.index)
    t.cuda.current_stream(f1.device).synchronize()
    N.check(N.lib.hivc_horn_schunck(ctx.handle, ptr(f1), ptr(f0), h, w, float(alpha), int(iterations), ptr(u),
                                    ptr(v)))
    return FlowField(back(u, frame_t), back(v, frame_t))


def _tree_leaves(data: bytes, pos: int, nbits: int, width: int, height: int, bit_offset: int = 0, with_used=False):
    """Preorder leaf rectangles (x, y, w, h) via the native parser (subdivision.py:183-222)."""
    nbytes = (nbits + 7) // 8
    buf = C.create_string_buffer(bytes(data[pos : pos + nbytes]), max(nbytes, 1))
    n = C.c_size_t()
    used = C.c_uint64()
    N.check(N.lib.hivc_parse_tree(buf, nbytes, nbits, bit_offset, width, height, None, 0, C.byref(n), C.byref(used)))
    rects = (C.c_int32 * max(4 * n.value, 1))()
    N.check(N.lib.hivc_parse_tree(buf, nbytes, nbits, bit_offset, width, height, rects, n.value, C.byref(n),
                                  C.byref(used)))
    out = np.frombuffer(rects, dtype=np.int32)[: 4 * n.value].reshape(-1, 4).copy()
    return (out, int(used.value)) if with_used else out


def _decompress_plane(data: bytes, pos: int, shape, levels: int):
    """One flow component painted on a host float64 plane (flow.py:343-356,
    quantize.py:78-82, subdivision.py:162-170) by one native call."""
    h, w = shape
    out = np.empty((h, w), dtype=np.float64)
    nxt = C.c_size_t()
    N.check(N.lib.hivc_flow_component(None, bytes(data), len(data), pos, h, w, levels,
                                      out.ctypes.data_as(C.c_void_p), C.byref(nxt)))
    return out, int(nxt.value)


def _decompress_plane_device(data: bytes, pos: int, shape, levels: int, device):
    """_decompress_plane with the leaves painted on the GPU by one launch (the
    encoder's closed loop keeps the dense flow on the device for the warp)."""
    h, w = shape
    t = torch()
    out = t.empty((h, w), dtype=t.float64, device=device)
    nxt = C.c_size_t()
    N.check(N.lib.hivc_flow_component(N.context(out.device.index).handle, bytes(data), len(data), pos, h, w, levels,
                                      ptr(out), C.byref(nxt)))
    return out, int(nxt.value)


def decompress_flow(data: bytes, pos: int, shape, quant_levels: int):
    """Decode a compressed flow payload; returns (FlowField, next position) (flow.py:368-372)."""
    u, pos = _decompress_plane(data, pos, shape, quant_levels)
    v, pos = _decompress_plane(data, pos, shape, quant_levels)
    return FlowField(u, v), pos


def _compress_plane(plane, budget: int, levels: int) -> bytes:
    """Tree bits + quantised leaf means of one flow component (flow.py:324-340)."""
    from paper_2008_10273_b200.entropy import encode_symbols
    from paper_2008_10273_b200.quantize import uniform_quantize
    from paper_2008_10273_b200.subdivision import leaf_means, subdivide_by_error

    p = np.ascontiguousarray(plane.cpu().numpy() if is_cuda_tensor(plane) else plane, dtype=np.float64)
    tree = subdivide_by_error(p, budget, min_error=0.0)  # early stop on exactly representable regions
    means = leaf_means(tree, p)
    lo, hi = float(means.min()), float(means.max())
    if hi <= lo:
        hi = lo + 1e-6
    idx = uniform_quantize(means, lo, hi, levels)
    return struct.pack("<ffI", lo, hi, len(tree.bits)) + tree.packed + encode_symbols(idx, table_log=8)


def compress_flow(flow: FlowField, points_budget: int, quant_levels: int) -> bytes:
    """Encode u and v independently: tree bits + quantized leaf averages (flow.py:359-365)."""
    if points_budget < 1:
        raise FlowError("points budget must be >= 1")
    # the two components are independent: subdivide them on two host threads
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(2) as ex:
        pu = ex.submit(_compress_plane, flow.u, points_budget, quant_levels)
        pv = ex.submit(_compress_plane, flow.v, points_budget, quant_levels)
        return pu.result() + pv.result()
