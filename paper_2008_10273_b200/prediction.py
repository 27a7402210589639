"""Per-frame prediction signals on the B200 (reference: prediction.py).

``decode_intra`` (prediction.py:185-208): native tree/tANS parse, then the
GPU cascadic-CG solve per channel with the decoder's fixed budget
(tol 1e-4, 160 iterations, non-strict).  ``predict_inter``
(prediction.py:220-223): GPU bilinear backward warp.  Encoder side:
``optimize_mask_values`` (prediction.py:63-96): LSQR over
GPU inpainting solves and their adjoint.
"""

from __future__ import annotations

import struct

import numpy as np

from paper_2008_10273_b200.entropy import decode_symbols
from paper_2008_10273_b200.errors import QuantizeError, TruncatedStream
from paper_2008_10273_b200.flow import _tree_leaves, warp_planes
from paper_2008_10273_b200._tensors import ptr, torch
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
    """Motion-compensated prediction: previous reconstruction sampled at (x+u, y+v)
    (numpy planes -> numpy, CUDA tensors -> CUDA tensors)."""
    from paper_2008_10273_b200._tensors import is_cuda_tensor

    return warp_planes([p if is_cuda_tensor(p) else np.asarray(p, dtype=np.float64) for p in prev_planes],
                       flow.u, flow.v)


# ----------------------------------------------------------------------------- tonal optimisation (encoder)

TONAL_ITERS = 12  # prediction.py:40
# the reference factorises the inpainting system exactly (splu); the GPU
# operator solves it with CG to this relative residual instead
TONAL_SOLVE_TOL = 1e-12
TONAL_SOLVE_MAX_ITER = 200000


class _InpaintOperator:
    """The LSQR operator of ``optimize_mask_values`` (prediction.py:72-81):
    ``matvec(v) = A^-1 [v scattered on the mask points]`` and
    ``rmatvec(w) = (A^-T w)[mask points]`` with A = diag(d) + diag(1-d) L
    (prediction.py:43-61).  The forward solve is the cascadic CG of
    ``solve_homogeneous``; the adjoint solves the interior system
    L_II z_I = w_I and takes z_M = w_M - (L z)_M (``hivc_poisson_interior``,
    ``hivc_mask_adjoint``).  Vectors are float64 CUDA tensors."""

    def __init__(self, mask, tol=TONAL_SOLVE_TOL, max_iter=TONAL_SOLVE_MAX_ITER):
        import ctypes as C

        from paper_2008_10273_b200 import _native as N
        from paper_2008_10273_b200._tensors import to_device

        self._C, self._N = C, N
        self.t = torch()
        self.m = to_device(mask, self.t.bool).to(self.t.uint8)
        self.h, self.w = int(self.m.shape[0]), int(self.m.shape[1])
        self.n = self.h * self.w
        self.pts = self.t.nonzero(self.m.reshape(-1)).reshape(-1).to(self.t.int32)
        self.npts = int(self.pts.numel())
        self.tol, self.max_iter = float(tol), int(max_iter)
        self.ctx = N.context(self.m.device.index)
        self.solver_iters = []

    def _sync(self):
        self.t.cuda.current_stream(self.m.device).synchronize()

    def matvec(self, v):
        C, N, t = self._C, self._N, self.t
        f = t.zeros(self.n, dtype=t.float64, device=self.m.device)
        f[self.pts.long()] = v
        u = t.empty_like(f)
        sizes, iters, nlev = (C.c_int32 * 32)(), (C.c_int32 * 32)(), C.c_int32()
        self._sync()
        N.check(N.lib.hivc_homog_solve(self.ctx.handle, ptr(f), ptr(self.m), self.h, self.w, self.tol, self.max_iter,
                                       0, ptr(u), sizes, iters, C.byref(nlev)))
        self.solver_iters.append(int(iters[nlev.value - 1]))
        return u

    def rmatvec(self, wv):
        C, N, t = self._C, self._N, self.t
        wv = wv.contiguous()
        z = t.empty_like(wv)
        out = t.empty(self.npts, dtype=t.float64, device=self.m.device)
        it = C.c_int32()
        self._sync()
        N.check(N.lib.hivc_poisson_interior(self.ctx.handle, ptr(wv), ptr(self.m), self.h, self.w, self.tol,
                                            self.max_iter, ptr(z), C.byref(it)))
        N.check(N.lib.hivc_mask_adjoint(self.ctx.handle, ptr(wv), ptr(z), ptr(self.pts), self.npts, self.h, self.w,
                                        ptr(out)))
        self.solver_iters.append(int(it.value))
        return out


def _sym_ortho(a: float, b: float):
    """Stable Givens rotation (c, s, r) with r = sqrt(a^2 + b^2) (Paige & Saunders)."""
    import math

    if b == 0:
        return math.copysign(1.0, a) if a != 0 else 0.0, 0.0, abs(a)
    if a == 0:
        return 0.0, math.copysign(1.0, b), abs(b)
    if abs(b) > abs(a):
        tau = a / b
        s = math.copysign(1.0, b) / math.sqrt(1 + tau * tau)
        return s * tau, s, b / s
    tau = b / a
    c = math.copysign(1.0, a) / math.sqrt(1 + tau * tau)
    return c, c * tau, a / c


def _lsqr(op, b, iter_lim: int, x0, atol: float = 1e-6, btol: float = 1e-6, conlim: float = 1e8):
    """LSQR (Paige & Saunders 1982) for min ||A x - b||, damp = 0, started at x0 —
    the algorithm and stopping tests of the reference's ``scipy.sparse.linalg.lsqr``
    call (prediction.py:91, scipy 1.18.1; default atol/btol/conlim).  Scalars on
    the host, vectors on the device."""
    import math

    t = torch()
    eps = float(np.finfo(np.float64).eps)
    ctol = 1.0 / conlim if conlim > 0 else 0.0
    bnorm = float(t.linalg.vector_norm(b))
    x = x0.clone()
    u = b - op.matvec(x)
    beta = float(t.linalg.vector_norm(u))
    if beta > 0:
        u = u * (1.0 / beta)
        v = op.rmatvec(u)
        alfa = float(t.linalg.vector_norm(v))
    else:
        v = x.clone()
        alfa = 0.0
    if alfa > 0:
        v = v * (1.0 / alfa)
    w = v.clone()
    rhobar, phibar = alfa, beta
    anorm = acond = ddnorm = res2 = xnorm = xxnorm = z = 0.0
    cs2, sn2 = -1.0, 0.0
    if alfa * beta == 0:
        return x
    itn = 0
    while itn < iter_lim:
        itn += 1
        u = op.matvec(v) - alfa * u
        beta = float(t.linalg.vector_norm(u))
        if beta > 0:
            u = u * (1.0 / beta)
            anorm = math.sqrt(anorm**2 + alfa**2 + beta**2)
            v = op.rmatvec(u) - beta * v
            alfa = float(t.linalg.vector_norm(v))
            if alfa > 0:
                v = v * (1.0 / alfa)
        cs, sn, rho = _sym_ortho(rhobar, beta)
        theta = sn * alfa
        rhobar = -cs * alfa
        phi = cs * phibar
        phibar = sn * phibar
        tau = sn * phi
        t1, t2 = phi / rho, -theta / rho
        ddnorm += float(t.linalg.vector_norm(w * (1.0 / rho))) ** 2
        x = x + t1 * w
        w = v + t2 * w
        delta = sn2 * rho
        gambar = -cs2 * rho
        rhs = phi - delta * z
        zbar = rhs / gambar
        xnorm = math.sqrt(xxnorm + zbar**2)
        gamma = math.sqrt(gambar**2 + theta**2)
        cs2, sn2 = gambar / gamma, theta / gamma
        z = rhs / gamma
        xxnorm += z**2
        acond = anorm * math.sqrt(ddnorm)
        rnorm = math.sqrt(phibar**2 + res2)
        arnorm = alfa * abs(tau)
        test1 = rnorm / bnorm
        test2 = arnorm / (anorm * rnorm + eps)
        test3 = 1 / (acond + eps)
        t1n = test1 / (1 + anorm * xnorm / bnorm)
        rtol = btol + atol * anorm * xnorm / bnorm
        if (itn >= iter_lim or 1 + test3 <= 1 or 1 + test2 <= 1 or 1 + t1n <= 1 or test3 <= ctol or test2 <= atol
                or test1 <= rtol):
            break
    return x


def optimize_mask_values(planes, mask, stats: dict | None = None):
    """Least-squares refinement of the transmitted mask values
    (prediction.optimize_mask_values, prediction.py:63-96): LSQR, 12
    iterations from the point samples, over the inpainting operator (GPU
    solves), then the box projection onto each plane's [min, max].  Returns
    a list of float64 numpy arrays (one per plane, raster order of the mask
    points), like the reference."""
    from paper_2008_10273_b200._tensors import to_device

    t = torch()
    mask = np.asarray(mask, dtype=bool) if not hasattr(mask, "is_cuda") else mask
    m_np = mask if isinstance(mask, np.ndarray) else mask.cpu().numpy()
    pts = np.flatnonzero(m_np.ravel())
    samples = [np.asarray(p, dtype=np.float64).ravel()[pts] for p in planes]
    if m_np.all():
        return samples
    op = _InpaintOperator(m_np)
    out = []
    for plane, x0 in zip(planes, samples):
        target = to_device(np.asarray(plane, dtype=np.float64).ravel(), t.float64)
        v = _lsqr(op, target, TONAL_ITERS, to_device(x0, t.float64))
        lo, hi = float(target.min()), float(target.max())
        out.append(t.clamp(v, lo, hi).cpu().numpy())
    if stats is not None:
        stats["solver_iterations"] = list(op.solver_iters)
    return out


# ----------------------------------------------------------------------------- intra payload (encoder)


def chroma_budget(luma_budget: int, plane_size: int) -> int:
    """Chroma shares one mask with half the luma points; a full luma mask stays full (prediction.py:99-108)."""
    if luma_budget >= plane_size:
        return plane_size
    return (luma_budget + 1) // 2


def _encode_plane_values(values, levels: int) -> bytes:
    from paper_2008_10273_b200.entropy import encode_symbols
    from paper_2008_10273_b200.quantize import uniform_quantize

    values = np.asarray(values, dtype=np.float64)  # prediction.py:122-130
    lo = int(np.floor(values.min()))
    hi = int(np.ceil(values.max()))
    if hi <= lo:
        hi = lo + 1
    idx = uniform_quantize(values, float(lo), float(hi), levels)
    return struct.pack("<hh", lo, hi) + encode_symbols(idx)


def _tree_record(tree) -> bytes:
    return struct.pack("<I", len(tree.bits)) + tree.packed  # prediction.py:142-146


def encode_intra(planes, luma_budget: int, levels: int, stats: dict | None = None) -> bytes:
    """Subdivision masks (native), tonal optimisation (GPU LSQR), quantised
    values (native tANS): the intra payload of prediction.encode_intra
    (prediction.py:162-182), byte for byte."""
    from paper_2008_10273_b200.encoder import _stage
    from paper_2008_10273_b200.subdivision import joint_ssd_error, mask_from_tree, subdivide_by_error

    if luma_budget < 1:
        raise ValueError("luma mask budget must be >= 1")
    y = np.ascontiguousarray(planes[0], dtype=np.float64)
    with _stage("intra_subdivide"):
        tree_y = subdivide_by_error(y, min(luma_budget, y.size))
    with _stage("intra_tonal"):
        (vals_y,) = optimize_mask_values([y], mask_from_tree(tree_y), stats)
    out = bytearray(_tree_record(tree_y))
    out += _encode_plane_values(vals_y, levels)
    if len(planes) == 3:
        u = np.ascontiguousarray(planes[1], dtype=np.float64)
        v = np.ascontiguousarray(planes[2], dtype=np.float64)
        with _stage("intra_subdivide"):
            tree_c = subdivide_by_error(u, chroma_budget(min(luma_budget, y.size), u.size),
                                        error_fn=joint_ssd_error([u, v]))
        with _stage("intra_tonal"):
            vals_u, vals_v = optimize_mask_values([u, v], mask_from_tree(tree_c))
        out += _tree_record(tree_c)
        out += _encode_plane_values(vals_u, chroma_levels(levels))
        out += _encode_plane_values(vals_v, chroma_levels(levels))
    return bytes(out)
