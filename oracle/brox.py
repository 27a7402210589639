"""Oracle: Brox-style variational backward flow (TEST INFRASTRUCTURE ONLY).

Restates reference ``flow.py:56-86,135-184,187-278`` in numpy float64 with
the reference's association of every expression.  The reference calls two
third-party filters, ``scipy.ndimage.gaussian_filter`` (mode 'reflect',
truncate 4.0) and ``median_filter`` (size 3, mode 'nearest'), scipy 1.18.1
in this image.  ``gaussian`` below restates scipy's published algorithm —
separable 1-D correlations along axis 0 then axis 1 with normalised
``exp(-x^2 / (2 sigma^2))`` taps and the symmetric accumulation order of
scipy's ``NI_Correlate1D`` (centre tap first, then the outermost pair
inwards) — and is pinned bit-for-bit against scipy in tests/test_oracle.py.
The 3x3 median is an order statistic (exact); the oracle uses scipy's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Params:  # flow.py:56-66
    alpha: float = 40.0
    gamma: float = 40.0
    pyramid_scale: float = 0.5
    min_size: int = 16
    warps: int = 3
    fixed_point_iters: int = 5
    solver_iters: int = 30
    eps: float = 1e-3
    presmooth_sigma: float = 0.8


def gauss_taps(sigma: float, truncate: float = 4.0):
    """Normalised taps and radius of scipy's 1-D Gaussian."""
    r = int(truncate * float(sigma) + 0.5)
    x = np.arange(-r, r + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
    return phi / phi.sum(), r


def _corr_axis(a, taps, r, axis):
    a = np.moveaxis(a, axis, -1)
    n = a.shape[-1]
    idx = np.arange(-r, n + r)
    src = np.where(idx < 0, -idx - 1, np.where(idx >= n, 2 * n - idx - 1, idx))  # 'reflect'
    ext = a[..., src]
    acc = ext[..., r : r + n] * taps[r]
    for j in range(-r, 0):
        acc = acc + (ext[..., r + j : r + j + n] + ext[..., r - j : r - j + n]) * taps[r + j]
    return np.moveaxis(acc, -1, axis)


def gaussian(a, sigma):
    taps, r = gauss_taps(sigma)
    return _corr_axis(_corr_axis(np.asarray(a, dtype=np.float64), taps, r, 0), taps, r, 1)


def median3(a):
    from scipy.ndimage import median_filter

    return median_filter(a, size=3, mode="nearest")


def resize(img, shape):
    """Pixel-centre bilinear resample (flow.py:69-86)."""
    h, w = shape
    ih, iw = img.shape
    if (ih, iw) == (h, w):
        return img.copy()
    ys = np.clip((np.arange(h) + 0.5) * (ih / h) - 0.5, 0, ih - 1)
    xs = np.clip((np.arange(w) + 0.5) * (iw / w) - 0.5, 0, iw - 1)
    y0 = np.floor(ys).astype(int)
    x0 = np.floor(xs).astype(int)
    y1 = np.minimum(y0 + 1, ih - 1)
    x1 = np.minimum(x0 + 1, iw - 1)
    fy = (ys - y0)[:, None]
    fx = (xs - x0)[None, :]
    top = (1 - fx) * img[y0][:, x0] + fx * img[y0][:, x1]
    bot = (1 - fx) * img[y1][:, x0] + fx * img[y1][:, x1]
    return (1 - fy) * top + fy * bot


def ddx(a):  # flow.py:135-140
    g = np.empty_like(a)
    g[:, 1:-1] = 0.5 * (a[:, 2:] - a[:, :-2])
    g[:, 0] = a[:, 1] - a[:, 0]
    g[:, -1] = a[:, -1] - a[:, -2]
    return g


def ddy(a):  # flow.py:143-148
    g = np.empty_like(a)
    g[1:-1, :] = 0.5 * (a[2:, :] - a[:-2, :])
    g[0, :] = a[1, :] - a[0, :]
    g[-1, :] = a[-1, :] - a[-2, :]
    return g


def level_shapes(h, w, scale, min_size):  # flow.py:151-159
    out = [(h, w)]
    while min(out[-1]) > min_size:
        nh = max(int(round(out[-1][0] * scale)), min_size)
        nw = max(int(round(out[-1][1] * scale)), min_size)
        if (nh, nw) == out[-1]:
            break
        out.append((nh, nw))
    return out


def _edge(a):
    return np.pad(a, 1, mode="edge")


def nbr_sum(f, wn, ws, ww, we):  # flow.py:162-170
    p = _edge(f)
    return wn * p[:-2, 1:-1] + ws * p[2:, 1:-1] + ww * p[1:-1, :-2] + we * p[1:-1, 2:]


def half_weights(psi):  # flow.py:173-184
    p = _edge(psi)
    wn = 0.5 * (psi + p[:-2, 1:-1])
    ws = 0.5 * (psi + p[2:, 1:-1])
    ww = 0.5 * (psi + p[1:-1, :-2])
    we = 0.5 * (psi + p[1:-1, 2:])
    wn[0, :] = 0.0
    ws[-1, :] = 0.0
    ww[:, 0] = 0.0
    we[:, -1] = 0.0
    return wn, ws, ww, we


def warp1(plane, u, v):
    from oracle.motion import warp

    return warp([plane], u, v)[0]


def brox(frame_t, frame_prev, prm: Params | None = None):
    """Backward flow frame_t -> frame_prev (flow.py:187-278); returns (u, v)."""
    prm = prm or Params()
    f1 = np.asarray(frame_t, dtype=np.float64)
    f0 = np.asarray(frame_prev, dtype=np.float64)
    if prm.presmooth_sigma > 0:
        f1 = gaussian(f1, prm.presmooth_sigma)
        f0 = gaussian(f0, prm.presmooth_sigma)
    shapes = level_shapes(*f1.shape, prm.pyramid_scale, prm.min_size)
    refs, tgts = [f1], [f0]
    aa = 0.5 / prm.pyramid_scale
    for shp in shapes[1:]:
        refs.append(resize(gaussian(refs[-1], aa), shp))
        tgts.append(resize(gaussian(tgts[-1], aa), shp))
    eps2 = prm.eps * prm.eps
    a = prm.alpha
    u = v = None
    for lvl in range(len(shapes) - 1, -1, -1):
        h, w = shapes[lvl]
        ref, tgt = refs[lvl], tgts[lvl]
        if u is None:
            u, v = np.zeros((h, w)), np.zeros((h, w))
        else:
            u = resize(u, (h, w)) * (w / shapes[lvl + 1][1])
            v = resize(v, (h, w)) * (h / shapes[lvl + 1][0])
        for _ in range(prm.warps):
            wp = warp1(tgt, u, v)
            ix = 0.5 * (ddx(wp) + ddx(ref))
            iy = 0.5 * (ddy(wp) + ddy(ref))
            iz = wp - ref
            ixx, ixy, iyy = ddx(ix), ddy(ix), ddy(iy)
            ixz = ddx(wp) - ddx(ref)
            iyz = ddy(wp) - ddy(ref)
            du, dv = np.zeros_like(u), np.zeros_like(v)
            for _ in range(prm.fixed_point_iters):
                rb = iz + ix * du + iy * dv
                psi_d = 1.0 / np.sqrt(rb * rb + eps2)
                rgx = ixz + ixx * du + ixy * dv
                rgy = iyz + ixy * du + iyy * dv
                psi_g = prm.gamma / np.sqrt(rgx * rgx + rgy * rgy + eps2)
                ut, vt = u + du, v + dv
                g2 = ddx(ut) ** 2 + ddy(ut) ** 2 + ddx(vt) ** 2 + ddy(vt) ** 2
                psi_s = np.maximum(1.0 / np.sqrt(g2 + eps2), 0.05)
                wn, ws, ww, we = half_weights(psi_s)
                wsum = wn + ws + ww + we
                a11 = psi_d * ix * ix + psi_g * (ixx * ixx + ixy * ixy) + a * wsum
                a12 = psi_d * ix * iy + psi_g * (ixx * ixy + ixy * iyy)
                a22 = psi_d * iy * iy + psi_g * (ixy * ixy + iyy * iyy) + a * wsum
                b1f = -psi_d * ix * iz - psi_g * (ixx * ixz + ixy * iyz)
                b2f = -psi_d * iy * iz - psi_g * (ixy * ixz + iyy * iyz)
                su = nbr_sum(u, wn, ws, ww, we) - wsum * u
                sv = nbr_sum(v, wn, ws, ww, we) - wsum * v
                for _ in range(prm.solver_iters):
                    b1 = b1f + a * (su + nbr_sum(du, wn, ws, ww, we))
                    b2 = b2f + a * (sv + nbr_sum(dv, wn, ws, ww, we))
                    det = a11 * a22 - a12 * a12
                    det = np.where(np.abs(det) < 1e-12, 1e-12, det)
                    dun = (a22 * b1 - a12 * b2) / det
                    dvn = (a11 * b2 - a12 * b1) / det
                    du = 0.5 * du + 0.5 * dun
                    dv = 0.5 * dv + 0.5 * dvn
                np.clip(du, -1.0, 1.0, out=du)
                np.clip(dv, -1.0, 1.0, out=dv)
            u = median3(u + du)
            v = median3(v + dv)
    bound = float(max(f1.shape))
    return np.clip(u, -bound, bound), np.clip(v, -bound, bound)
