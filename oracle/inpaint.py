"""Oracle: homogeneous-diffusion inpainting by cascadic CG (TEST INFRASTRUCTURE ONLY).

Restates reference ``homogeneous.py:27-212`` in numpy float64 with the
same association of every sum, so the only divergence from the reference
is BLAS dot-product summation order.
"""

from __future__ import annotations

import numpy as np

COARSEST = 16  # homogeneous.py:15
LEVEL_TOL = 1e-4  # homogeneous.py:16


class InpaintErr(ValueError):
    kind = "InpaintingError"


class NotConverged(RuntimeError):
    kind = "ConvergenceError"


def lap5(u: np.ndarray) -> np.ndarray:
    """Reflecting 5-point Laplacian (``homogeneous.py:27-43``).

    Accumulation order per pixel: -4u, +north, +south, +west, +east, where a
    missing neighbour is the pixel itself.
    """
    north = np.concatenate([u[:1], u[:-1]], axis=0)
    south = np.concatenate([u[1:], u[-1:]], axis=0)
    west = np.concatenate([u[:, :1], u[:, :-1]], axis=1)
    east = np.concatenate([u[:, 1:], u[:, -1:]], axis=1)
    return (((u * -4.0 + north) + south) + west) + east


def _pair_sum(a: np.ndarray) -> np.ndarray:
    """2x2 block sums with ceiling halving: rows first, then columns
    (the order of ``np.add.reduceat`` over axis 0 then axis 1)."""
    h, w = a.shape
    if h & 1:
        a = np.concatenate([a, np.zeros((1, w))], axis=0)
    rows = a[0::2] + a[1::2] if a.shape[0] > 1 else a
    if h & 1:
        rows[-1] = a[-2]
    if w & 1:
        rows = np.concatenate([rows, np.zeros((rows.shape[0], 1))], axis=1)
    out = rows[:, 0::2] + rows[:, 1::2]
    if w & 1:
        out[:, -1] = rows[:, -2]
    return out


def pyramid(f: np.ndarray, mask: np.ndarray):
    """Finest-first list of (values, mask) (``homogeneous.py:96-130``)."""
    lv = [(np.asarray(f, dtype=np.float64), np.asarray(mask, dtype=bool))]
    while max(lv[-1][0].shape) > COARSEST:
        fv, mv = lv[-1]
        cnt = _pair_sum(mv.astype(np.float64))
        ssum = _pair_sum(np.where(mv, fv, 0.0))
        ones = _pair_sum(np.ones_like(fv))
        mean_all = _pair_sum(fv) / ones
        cm = cnt > 0
        lv.append((np.where(cm, ssum / np.maximum(cnt, 1.0), mean_all), cm))
    return lv


def prolong(c: np.ndarray, shape) -> np.ndarray:
    """Pixel-centre bilinear up-sampling (``homogeneous.py:133-154``)."""
    h, w = shape
    ch, cw = c.shape
    if (ch, cw) == (h, w):
        return c.copy()
    ys = np.clip((np.arange(h) + 0.5) * (ch / h) - 0.5, 0, ch - 1)
    xs = np.clip((np.arange(w) + 0.5) * (cw / w) - 0.5, 0, cw - 1)
    y0 = np.floor(ys).astype(int)
    x0 = np.floor(xs).astype(int)
    y1 = np.minimum(y0 + 1, ch - 1)
    x1 = np.minimum(x0 + 1, cw - 1)
    fy = (ys - y0)[:, None]
    fx = (xs - x0)[None, :]
    top = (1 - fx) * c[y0][:, x0] + fx * c[y0][:, x1]
    bot = (1 - fx) * c[y1][:, x0] + fx * c[y1][:, x1]
    return (1 - fy) * top + fy * bot


def masked_cg(f, mask, x0, tol, max_iter, denom=None):
    """CG on the non-mask unknowns (``homogeneous.py:55-93``); returns (u, iterations)."""
    keep = (~mask).astype(np.float64)
    ud = np.where(mask, f, 0.0)
    b = lap5(ud) * keep
    x = x0 * keep
    r = b - (-lap5(x) * keep)
    bn = float(np.linalg.norm(b)) if denom is None else denom
    if bn == 0.0:
        return ud + x, 0
    p = r.copy()
    rs = float(np.vdot(r, r))
    k = 0
    for k in range(1, max_iter + 1):
        ap = -lap5(p) * keep
        pap = float(np.vdot(p, ap))
        if pap <= 0.0 or rs < 1e-300:
            break
        alpha = rs / pap
        x += alpha * p
        r -= alpha * ap
        rs1 = float(np.vdot(r, r))
        if np.sqrt(rs1) <= tol * bn:
            break
        p = r + (rs1 / rs) * p
        rs = rs1
    return ud + x, k


def solve(f, mask, tol=1e-6, max_iter=10000, strict=True, stats=None):
    """Cascadic coarse-to-fine solve (``homogeneous.py:157-212``)."""
    f = np.asarray(f, dtype=np.float64)
    mask = np.asarray(mask, dtype=bool)
    if f.shape != mask.shape:
        raise InpaintErr("plane/mask shape mismatch")
    if not mask.any():
        raise InpaintErr("empty inpainting mask")
    if strict and tol <= 0:
        raise InpaintErr("tol must be positive")
    lv = pyramid(f, mask)
    u = None
    its = []
    for i in range(len(lv) - 1, -1, -1):
        fv, mv = lv[i]
        x0 = np.full_like(fv, float(fv[mv].mean())) if u is None else prolong(u, fv.shape)
        if mv.all():
            u = fv.copy()
            its.append((fv.size, 0))
            continue
        ltol = tol if i == 0 else max(LEVEL_TOL, tol)
        den = float(np.linalg.norm(fv[mv])) if i == 0 else None
        if den == 0.0:
            den = None
        u, k = masked_cg(fv, mv, x0, ltol, max_iter, denom=den)
        its.append((fv.size, k))
    if stats is not None:
        stats["level_iterations"] = its
    if strict:
        res = np.where(mask, u - f, lap5(u))
        den = float(np.linalg.norm(f[mask]))
        rel = float(np.linalg.norm(res)) / den if den > 0 else float(np.linalg.norm(res))
        if den > 0 and rel > tol:
            raise NotConverged(f"relative residual {rel:.3e} > tol {tol:.3e}")
    return u


def solve_dense(f, mask):
    """Direct dense solve, small planes only (``homogeneous.py:215-229``)."""
    f = np.asarray(f, dtype=np.float64)
    m = np.asarray(mask, dtype=bool).ravel().astype(np.float64)
    h, w = f.shape
    n = h * w
    lap = np.zeros((n, n))
    for yy in range(h):
        for xx in range(w):
            i = yy * w + xx
            for dy, dx in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                ny, nx = yy + dy, xx + dx
                if 0 <= ny < h and 0 <= nx < w:
                    lap[i, ny * w + nx] += 1.0
                    lap[i, i] -= 1.0
    A = np.diag(m) + (np.eye(n) - np.diag(m)) @ lap
    return np.linalg.solve(A, m * f.ravel()).reshape(h, w)
