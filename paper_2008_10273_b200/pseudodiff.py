"""Block pseudodifferential residual inpainting on the B200 (reference: pseudodiff.py).

``reconstruct_blocks`` (pseudodiff.py:275-279) runs the AAN DCT ->
Green's eigenvalues -> AAN IDCT chain per 8x8 block on the GPU in float64,
operation for operation (csrc/device.cuh: block_reconstruct_8lanes);
``solve_block_coefficients_batch`` (pseudodiff.py:243-263) solves every
block's bordered (K+1)^2 system in shared memory (csrc/recon.cu:
block_fit_kernel) and, unlike the reference, accepts any mix of K.
"""

from __future__ import annotations

import numpy as np

from paper_2008_10273_b200 import _native as N
from paper_2008_10273_b200._tensors import back, is_cuda_tensor, ptr, to_device, torch
from paper_2008_10273_b200.errors import PseudodiffError

BLOCK = 8


def greens_eigenvalues_harmonic() -> np.ndarray:
    """Eigenvalues of G = pinv(-L) on an 8x8 block in the DCT-II basis (pseudodiff.py:160-171)."""
    p = 2.0 - 2.0 * np.cos(np.pi * np.arange(8) / 8.0)
    mu = p[:, None] + p[None, :]
    lam = np.zeros((8, 8))
    lam[mu > 0] = 1.0 / mu[mu > 0]
    return lam


def block_grid(height: int, width: int):
    """Raster-order list of (y0, x0, bh, bw) tiles of size <= 8 (pseudodiff.py:290-296)."""
    return [
        (y0, x0, min(BLOCK, height - y0), min(BLOCK, width - x0))
        for y0 in range(0, height, BLOCK)
        for x0 in range(0, width, BLOCK)
    ]


def reconstruct_blocks(mc, a, eig=None):
    """Batched decode of scattered coefficient blocks (n, 8, 8) + constants (n,)."""
    t = torch()
    mct = to_device(mc, t.float64)
    n = int(mct.shape[0])
    if tuple(mct.shape[1:]) != (8, 8):
        raise PseudodiffError("expected (n, 8, 8) coefficient blocks")
    at = to_device(a, t.float64, mct.device).reshape(-1)
    if at.numel() != n:
        raise PseudodiffError("one constant per block expected")
    eigt = None if eig is None else to_device(eig, t.float64, mct.device).reshape(64)
    out = t.empty_like(mct)
    ctx = N.context(mct.device.index)
    t.cuda.current_stream(mct.device).synchronize()
    N.check(N.lib.hivc_block_reconstruct(ctx.handle, ptr(mct), ptr(at), ptr(eigt) if eigt is not None else None, n,
                                         ptr(out)))
    return back(out, mc)


def _mask_words(masks) -> np.ndarray:
    m = np.asarray(masks.cpu().numpy() if is_cuda_tensor(masks) else masks, dtype=bool).reshape(-1, 64)
    weights = (np.uint64(1) << np.arange(64, dtype=np.uint64))
    return (m.astype(np.uint64) * weights).sum(axis=1, dtype=np.uint64)


def solve_block_coefficients_batch(f_blocks, masks):
    """Coefficient fit [[G_KK,1],[1^T,0]][c;a] = [f_K;0] for every block.

    f_blocks: (n, 8, 8), masks: (n, 8, 8) bool sharing one popcount K (as in
    the reference).  Returns (c: (n, K), a: (n,)).
    """
    t = torch()
    ft = to_device(f_blocks, t.float64)
    n = int(ft.shape[0])
    words = _mask_words(masks)
    ks = np.array([bin(int(x)).count("1") for x in words]) if n else np.zeros(0, dtype=int)
    if n and (ks != ks[0]).any():
        raise PseudodiffError("blocks in one batch must share K (use solve_blocks_any_k)")
    c_full, a = solve_blocks_any_k(ft, words)
    k = int(ks[0]) if n else 0
    mflat = t.from_numpy(np.asarray(masks.cpu().numpy() if is_cuda_tensor(masks) else masks, dtype=bool).reshape(n, 64))
    mflat = mflat.to(ft.device)
    c = c_full.reshape(n, 64)[mflat].reshape(n, k)
    return back(c, f_blocks), back(a, f_blocks)


def solve_blocks_any_k(f_blocks, mask_words):
    """Fit for blocks with arbitrary masks; returns the scattered M c (n, 8, 8) and a (n,)."""
    t = torch()
    ft = to_device(f_blocks, t.float64)
    n = int(ft.shape[0])
    mw = to_device(np.asarray(mask_words, dtype=np.uint64).view(np.int64), t.int64, ft.device)
    c = t.empty((n, 8, 8), dtype=t.float64, device=ft.device)
    a = t.empty((n,), dtype=t.float64, device=ft.device)
    ctx = N.context(ft.device.index)
    t.cuda.current_stream(ft.device).synchronize()
    N.check(N.lib.hivc_block_fit(ctx.handle, ptr(ft), ptr(mw), n, ptr(c), ptr(a)))
    return c, a


# The reference's flat-block 4-point layout: mask_from_tree(subdivide_by_error(zeros((8, 8)), 4)),
# points (y, x) = (2,1), (2,3), (4,6), (6,2) (subdivision.py:76-130, 173-178); bit y*8+x.
FLAT_BLOCK_MASK = (1 << 17) | (1 << 19) | (1 << 38) | (1 << 50)


def reconstruct_plane_shared_mask(plane, mask=FLAT_BLOCK_MASK):
    """Fit + rebuild every 8x8 tile of a float32 plane with ONE shared mask layout.

    Equivalent to ``inpaint_plane_blockwise`` (pseudodiff.py:299-324) with the
    same mask in every tile: the fit and the rebuild collapse into a fixed
    64x64 operator, applied to all tiles as a 3xTF32 tcgen05 tensor-core
    contraction (csrc/blockgemm.cu).  ``mask``: 8x8 bool array or int bitmask.
    Returns the reconstructed plane (float32; numpy in -> numpy out).
    """
    t = torch()
    if not isinstance(mask, int):
        mask = int(_mask_words(np.asarray(mask, dtype=bool).reshape(1, 64))[0])
    pt = to_device(plane, t.float32)
    h, w = pt.shape
    pts = [(b // 8, b % 8) for b in range(64) if (mask >> b) & 1]
    if not pts:
        raise PseudodiffError("block mask needs at least one point")
    if (h % 8 and max(y for y, _ in pts) >= h % 8) or (w % 8 and max(x for _, x in pts) >= w % 8):
        raise PseudodiffError("mask point outside true pixels of edge block")  # pseudodiff.py:317-318
    out = t.empty_like(pt)
    ctx = N.context(pt.device.index)
    t.cuda.current_stream(pt.device).synchronize()
    N.check(N.lib.hivc_block_operator(ctx.handle, ptr(pt), h, w, mask, ptr(out)))
    return back(out, plane)


def reconstruct_plane_masks(plane, masks):
    """Per-tile mask layouts (raster tile order, (ntiles, 8, 8) bool or uint64 words,
    or a CUDA int64 tensor of the words already on the device): each tile solves
    its own bordered system (float64) and is rebuilt."""
    t = torch()
    pt = to_device(plane, t.float32)
    h, w = pt.shape
    if is_cuda_tensor(masks) and masks.dtype == t.int64:
        mw = masks.contiguous()
    else:
        words = masks if (isinstance(masks, np.ndarray) and masks.dtype == np.uint64) else _mask_words(masks)
        mw = to_device(np.asarray(words, dtype=np.uint64).view(np.int64), t.int64, pt.device)
    if mw.numel() != ((h + 7) // 8) * ((w + 7) // 8):
        raise PseudodiffError("one mask per 8x8 tile expected")
    out = t.empty_like(pt)
    ctx = N.context(pt.device.index)
    t.cuda.current_stream(pt.device).synchronize()
    N.check(N.lib.hivc_block_perblock(ctx.handle, ptr(pt), h, w, ptr(mw), ptr(out)))
    return back(out, plane)


# Reference-compatible aliases for the decode-side helpers
__all__ = [
    "FLAT_BLOCK_MASK",
    "reconstruct_plane_shared_mask",
    "reconstruct_plane_masks",
    "BLOCK",
    "block_grid",
    "greens_eigenvalues_harmonic",
    "reconstruct_blocks",
    "solve_block_coefficients_batch",
    "solve_blocks_any_k",
]
