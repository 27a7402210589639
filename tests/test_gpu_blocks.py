"""Config-2 block fit + rebuild on the GPU vs the oracle (reference algorithm)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _oracle_plane(plane, masks):
    """inpaint_plane_blockwise (pseudodiff.py:299-324) with the oracle's fit + reconstruct."""
    from oracle import blocks

    h, w = plane.shape
    out = np.zeros((h, w))
    tiles = blocks.tile_grid(h, w)
    fb = np.zeros((len(tiles), 8, 8))
    for i, (y0, x0, bh, bw) in enumerate(tiles):
        fb[i, :bh, :bw] = plane[y0 : y0 + bh, x0 : x0 + bw]
    ks = masks.reshape(len(tiles), 64).sum(1)
    rec = np.zeros((len(tiles), 8, 8))
    for k in np.unique(ks):
        sel = np.flatnonzero(ks == k)
        c, a = blocks.fit(fb[sel], masks[sel])
        mc = np.zeros((len(sel), 64))
        for j, i in enumerate(sel):
            mc[j, masks[i].ravel()] = c[j]
        rec[sel] = blocks.reconstruct(mc.reshape(-1, 8, 8), a)
    for i, (y0, x0, bh, bw) in enumerate(tiles):
        out[y0 : y0 + bh, x0 : x0 + bw] = rec[i, :bh, :bw]
    return out


def _residual(h, w, seed):
    from scipy.ndimage import uniform_filter

    rng = np.random.default_rng(seed)
    return uniform_filter(rng.laplace(0.0, 8.0, (h, w)), size=3, mode="reflect").astype(np.float32)


def test_shared_mask_tensor_core_matches_oracle():
    from paper_2008_10273_b200.pseudodiff import FLAT_BLOCK_MASK, reconstruct_plane_shared_mask

    plane = _residual(120, 200, 2)
    m = np.array([[(FLAT_BLOCK_MASK >> (y * 8 + x)) & 1 for x in range(8)] for y in range(8)], bool)
    ntiles = 15 * 25
    ref = _oracle_plane(plane.astype(np.float64), np.broadcast_to(m, (ntiles, 8, 8)).copy())
    got = reconstruct_plane_shared_mask(plane)
    err = np.abs(got.astype(np.float64) - ref).max()
    # 3xTF32: ~fp32 accuracy; the north-star float bar is 1e-3
    assert err < 1e-3, err


def test_per_block_masks_match_oracle():
    from paper_2008_10273_b200.pseudodiff import reconstruct_plane_masks

    plane = _residual(100, 136, 3)  # edge tiles of 4 rows
    rng = np.random.default_rng(1002)
    tiles = 13 * 17
    masks = rng.uniform(size=(tiles, 8, 8)) < 0.05
    for i in range(tiles):  # points only on true pixels of edge tiles; empty tiles get one point
        ty = i // 17
        if ty == 12:
            masks[i, 4:] = False
        if not masks[i].any():
            masks[i, rng.integers(0, 4), rng.integers(0, 8)] = True
    ref = _oracle_plane(plane.astype(np.float64), masks)
    got = reconstruct_plane_masks(plane, masks)
    assert np.abs(got.astype(np.float64) - ref).max() < 1e-4  # float64 solve, float32 output


def test_shared_mask_rejects_points_outside_edge_tiles():
    from paper_2008_10273_b200.errors import PseudodiffError
    from paper_2008_10273_b200.pseudodiff import FLAT_BLOCK_MASK, reconstruct_plane_shared_mask

    with pytest.raises(PseudodiffError):
        reconstruct_plane_shared_mask(np.zeros((20, 16), np.float32), FLAT_BLOCK_MASK)


def test_per_block_masks_dense_blocks_use_wide_systems():
    """Blocks with more than 16 points take the wide-system kernel variant."""
    from paper_2008_10273_b200.pseudodiff import reconstruct_plane_masks

    plane = _residual(32, 48, 4)
    rng = np.random.default_rng(7)
    tiles = 4 * 6
    masks = rng.uniform(size=(tiles, 8, 8)) < 0.05
    masks[3] = rng.uniform(size=(8, 8)) < 0.5  # ~32 points
    masks[10] = rng.uniform(size=(8, 8)) < 0.35  # ~22 points
    for i in range(tiles):
        if not masks[i].any():
            masks[i, rng.integers(0, 8), rng.integers(0, 8)] = True
    ref = _oracle_plane(plane.astype(np.float64), masks)
    got = reconstruct_plane_masks(plane, masks)
    assert np.abs(got.astype(np.float64) - ref).max() < 1e-3
