"""Oracle: 8x8 block pseudodifferential inpainting (TEST INFRASTRUCTURE ONLY).

Restates reference ``pseudodiff.py``: the float AAN DCT-II / DCT-III
butterflies (``47-117``), their diagonal scale factors derived against
the exact orthonormal DCT matrix (``120-138``), the harmonic Green's
eigenvalues (``160-171``), batched reconstruction (``275-279``), the
64x64 Green's matrix (``190-201``) and the bordered coefficient fit
(``218-263``).
"""

from __future__ import annotations

import math

import numpy as np

# AAN factorisation constants (same real numbers as pseudodiff.py:40-44, 85-88)
F_C4 = 0.70710678118654752440  # cos(pi/4)
F_C6R2 = 0.54119610014619698439  # sqrt(2) cos(3pi/8)
F_C2R2 = 1.30656296487637652785  # sqrt(2) cos(pi/8)
F_C6 = 0.38268343236508977173  # cos(3pi/8)
I_R2 = 1.41421356237309504880  # sqrt(2)
I_2C2 = 1.84775906502257351226  # 2 cos(pi/8)
I_K3 = 1.08239220029239396879
I_K4 = 2.61312592975275305571


def fwd_butterfly(v: np.ndarray) -> np.ndarray:
    """Unscaled forward AAN pass along the last axis."""
    a = [v[..., i] for i in range(8)]
    s07, d07 = a[0] + a[7], a[0] - a[7]
    s16, d16 = a[1] + a[6], a[1] - a[6]
    s25, d25 = a[2] + a[5], a[2] - a[5]
    s34, d34 = a[3] + a[4], a[3] - a[4]
    e0, e3 = s07 + s34, s07 - s34
    e1, e2 = s16 + s25, s16 - s25
    out = [None] * 8
    out[0] = e0 + e1
    out[4] = e0 - e1
    rot = (e2 + e3) * F_C4
    out[2] = e3 + rot
    out[6] = e3 - rot
    o0 = d34 + d25
    o1 = d25 + d16
    o2 = d16 + d07
    q = (o0 - o2) * F_C6
    ra = F_C6R2 * o0 + q
    rb = F_C2R2 * o2 + q
    rc = o1 * F_C4
    lo_, hi_ = d07 + rc, d07 - rc
    out[5] = hi_ + ra
    out[3] = hi_ - ra
    out[1] = lo_ + rb
    out[7] = lo_ - rb
    return np.stack(out, axis=-1)


def inv_butterfly(v: np.ndarray) -> np.ndarray:
    """Unscaled inverse AAN pass along the last axis."""
    a = [v[..., i] for i in range(8)]
    p0, p1 = a[0] + a[4], a[0] - a[4]
    q13 = a[2] + a[6]
    q12 = (a[2] - a[6]) * I_R2 - q13
    e0, e3 = p0 + q13, p0 - q13
    e1, e2 = p1 + q12, p1 - q12
    m13 = a[5] + a[3]
    m10 = a[5] - a[3]
    m11 = a[1] + a[7]
    m12 = a[1] - a[7]
    o7 = m11 + m13
    o11 = (m11 - m13) * I_R2
    z = (m10 + m12) * I_2C2
    o10 = I_K3 * m12 - z
    o12 = -I_K4 * m10 + z
    o6 = o12 - o7
    o5 = o11 - o6
    o4 = o10 + o5
    return np.stack([e0 + o7, e1 + o6, e2 + o5, e3 - o4, e3 + o4, e2 - o5, e1 - o6, e0 - o7], axis=-1)


def dct_matrix() -> np.ndarray:
    k = np.arange(8)[:, None]
    n = np.arange(8)[None, :]
    c = np.cos(np.pi * (2 * n + 1) * k / 16.0)
    c[0, :] *= math.sqrt(1.0 / 8.0)
    c[1:, :] *= math.sqrt(2.0 / 8.0)
    return c


C8 = dct_matrix()
FWD_SCALE = np.diag(C8 @ np.linalg.inv(fwd_butterfly(np.eye(8)).T))
INV_SCALE = np.diag(np.linalg.inv(inv_butterfly(np.eye(8)).T) @ C8.T)
FWD_SCALE2 = np.outer(FWD_SCALE, FWD_SCALE)
INV_SCALE2 = np.outer(INV_SCALE, INV_SCALE)


def dct2(b: np.ndarray) -> np.ndarray:
    t = fwd_butterfly(b)
    t = fwd_butterfly(np.swapaxes(t, -1, -2))
    return np.swapaxes(t, -1, -2) * FWD_SCALE2


def idct2(c: np.ndarray) -> np.ndarray:
    t = inv_butterfly(c * INV_SCALE2)
    t = inv_butterfly(np.swapaxes(t, -1, -2))
    return np.swapaxes(t, -1, -2)


def greens_eig() -> np.ndarray:
    d = 2.0 - 2.0 * np.cos(np.pi * np.arange(8) / 8.0)
    mu = d[:, None] + d[None, :]
    lam = np.zeros((8, 8))
    lam[mu > 0] = 1.0 / mu[mu > 0]
    return lam


def reconstruct(mc: np.ndarray, a: np.ndarray, eig: np.ndarray | None = None) -> np.ndarray:
    """IDCT(eig * DCT(mc)) + a per block, (n, 8, 8)."""
    if eig is None:
        eig = greens_eig()
    return idct2(eig * dct2(mc)) + np.asarray(a)[:, None, None]


def greens_matrix() -> np.ndarray:
    """64x64 G = C2^T diag(eig) C2 with C2 = kron(C8, C8)."""
    c2 = np.kron(C8, C8)
    return (c2.T * greens_eig().reshape(-1)) @ c2


def fit(f_blocks: np.ndarray, masks: np.ndarray):
    """Bordered fit [[G_KK, 1], [1^T, 0]] [c; a] = [f_K; 0] for blocks sharing K."""
    n = f_blocks.shape[0]
    fm = masks.reshape(n, 64)
    k = int(fm[0].sum())
    g = greens_matrix()
    pos = np.argwhere(fm)[:, 1].reshape(n, k)
    A = np.empty((n, k + 1, k + 1))
    A[:, :k, :k] = g[pos[:, :, None], pos[:, None, :]]
    A[:, :k, k] = 1.0
    A[:, k, :k] = 1.0
    A[:, k, k] = 0.0
    rhs = np.zeros((n, k + 1))
    rhs[:, :k] = np.take_along_axis(f_blocks.reshape(n, 64), pos, axis=1)
    sol = np.linalg.solve(A, rhs[:, :, None])[:, :, 0]
    return sol[:, :k], sol[:, k]


def tile_grid(h: int, w: int):
    """Raster-order (y0, x0, bh, bw) tiles (``pseudodiff.py:290-296``)."""
    return [(y, x, min(8, h - y), min(8, w - x)) for y in range(0, h, 8) for x in range(0, w, 8)]
