"""The CPU oracle against the reference's own outputs (golden vectors made by
importing the reference, tests/golden/make_golden.py / make_streams.py).
CPU only."""

import numpy as np
import pytest

from oracle import blocks, decoder, inpaint, motion, parse


def test_oracle_decodes_rgb_like_the_reference():
    """Colour stream (RCT, shared chroma tree, [-255, 255] chroma clip) decoded by the
    reference decoder (tests/golden/make_streams.py rgb)."""
    from conftest import GOLDEN

    stream = (GOLDEN / "streams" / "rgb.hivc").read_bytes()
    ref = np.load(GOLDEN / "rgb_frames.npz")["frames"]
    got = np.stack([np.stack(f) for f in decoder.decode_stream(stream)])
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)


def test_oracle_decodes_config0_like_the_reference(cfg0_stream, cfg0_frames):
    frames = decoder.decode_stream(cfg0_stream)
    got = np.stack([f[0] for f in frames]).astype(np.uint8)
    assert np.array_equal(got, cfg0_frames)


@pytest.mark.parametrize("i", range(8))
def test_oracle_homogeneous_matches_reference(golden, i):
    f, m, u = golden[f"homog{i}_f"], golden[f"homog{i}_m"], golden[f"homog{i}_u"]
    tol, mi, strict = golden[f"homog{i}_cfg"]
    st = {}
    got = inpaint.solve(f, m, tol=tol, max_iter=int(mi), strict=bool(strict), stats=st)
    assert np.array_equal(np.array(st["level_iterations"]), golden[f"homog{i}_iters"])
    # identical algorithm; only BLAS dot-product order may differ
    assert np.abs(got - u).max() <= 1e-9 * max(1.0, np.abs(u).max())
    if f"homog{i}_dense" in golden and strict:
        assert np.sqrt(np.mean((got - golden[f"homog{i}_dense"]) ** 2)) < 1e-3


def test_oracle_blocks_match_reference(golden):
    assert np.array_equal(blocks.reconstruct(golden["blocks_mc"], golden["blocks_a"]), golden["blocks_rec"])
    assert np.array_equal(blocks.greens_eig(), golden["blocks_eig"])
    assert np.array_equal(blocks.FWD_SCALE2, golden["fscale2"])
    assert np.array_equal(blocks.INV_SCALE2, golden["iscale2"])
    assert np.array_equal(blocks.greens_matrix(), golden["g8"])


def test_oracle_block_fit_matches_reference(golden):
    f, masks = golden["fit_f"], golden["fit_masks"]
    n = f.shape[0]
    ks = masks.reshape(n, 64).sum(1)
    for k in np.unique(ks):
        sel = np.flatnonzero(ks == k)
        c, a = blocks.fit(f[sel], masks[sel])
        np.testing.assert_allclose(a, golden["fit_a"][sel], rtol=0, atol=1e-9)
        cf = golden["fit_c"][sel].reshape(len(sel), 64)[masks[sel].reshape(len(sel), 64)].reshape(len(sel), k)
        np.testing.assert_allclose(c, cf, rtol=0, atol=1e-9)


def test_oracle_warp_matches_reference(golden):
    out = motion.warp(list(golden["warp_planes"]), golden["warp_u"], golden["warp_v"])
    assert np.array_equal(np.stack(out), golden["warp_out"])


def test_oracle_entropy_matches_reference(payloads):
    for key in payloads:
        if key.endswith("_payload") and key.startswith("sym"):
            name = key[: -len("_payload")]
            out, pos = parse.decode_symbols(payloads[key].tobytes(), 0)
            assert pos == payloads[key].size
            assert np.array_equal(out, payloads[name + "_in"])
        if key.endswith("_payload") and key.startswith("sv"):
            name = key[: -len("_payload")]
            out, pos = parse.decode_signed_values(payloads[key].tobytes(), 0)
            assert pos == payloads[key].size
            assert np.array_equal(out, payloads[name + "_in"])


def test_oracle_trees_match_reference(payloads):
    i = 0
    while f"tree{i}_bits" in payloads:
        h, w = payloads[f"tree{i}_shape"]
        rd = parse.Bits(payloads[f"tree{i}_bits"].tobytes(), int(payloads[f"tree{i}_nbits"][0]))
        leaves = parse.tree_leaves(rd, int(w), int(h))
        assert np.array_equal(np.array(leaves).reshape(-1, 4), payloads[f"tree{i}_leaves"])
        rd = parse.Bits(payloads[f"tree{i}_bits"].tobytes(), int(payloads[f"tree{i}_nbits"][0]))
        assert np.array_equal(parse.tree_mask(rd, int(w), int(h)), payloads[f"tree{i}_mask"])
        i += 1


def test_oracle_dense_known_answers():
    # homogeneous.py / test_homogeneous.py known answers: full mask copies,
    # a single point gives a constant, maximum principle
    f = np.arange(12.0).reshape(3, 4)
    assert np.array_equal(inpaint.solve(f, np.ones((3, 4), bool)), f)
    m = np.zeros((5, 6), bool)
    m[2, 3] = True
    g = np.zeros((5, 6))
    g[2, 3] = 7.0
    np.testing.assert_allclose(inpaint.solve(g, m), 7.0, atol=1e-6)
    rng = np.random.default_rng(3)
    m = rng.uniform(size=(10, 11)) < 0.2
    m[0, 0] = True
    f = np.where(m, rng.uniform(10, 20, (10, 11)), 0.0)
    u = inpaint.solve(f, m)
    assert u.min() >= f[m].min() - 1e-6 and u.max() <= f[m].max() + 1e-6
    np.testing.assert_allclose(u, inpaint.solve_dense(f, m), atol=1e-4)


def test_oracle_gaussian_restatement_is_scipy_bit_exact():
    from scipy.ndimage import gaussian_filter

    from oracle import brox

    rng = np.random.default_rng(2)
    for shape in ((16, 17), (48, 64), (90, 33)):
        a = rng.uniform(0, 255, shape)
        for s in (0.8, 1.0, 0.5 / 0.95, 2.5):
            assert np.array_equal(brox.gaussian(a, s), gaussian_filter(a, s))


@pytest.mark.parametrize("tag,scale", [("05", 0.5), ("095", 0.95)])
def test_oracle_brox_matches_reference(golden, tag, scale):
    from oracle import brox

    pair = golden["brox_pair"]
    u, v = brox.brox(pair[1], pair[0], brox.Params(pyramid_scale=scale))
    assert np.array_equal(u, golden[f"brox{tag}_u"]) and np.array_equal(v, golden[f"brox{tag}_v"])


def test_oracle_decodes_edge_size_streams():
    """The oracle against the reference decoder on edge frame sizes (tests/golden/make_edge_streams.py)."""
    from pathlib import Path

    from oracle import decoder

    g = np.load(Path(__file__).resolve().parent / "golden" / "golden_edge.npz")
    for name in (str(n) for n in g["names"]):
        ref = g[f"{name}_frames"].astype(np.int32)
        got = np.stack([np.stack(f) for f in decoder.decode_stream(g[f"{name}_stream"].tobytes())])
        assert np.array_equal(got, ref), name


def test_oracle_config1_channel0_matches_reference():
    """Config 1 at its full size (1080p, 2 % mask, tol 1e-6, strict), channel 0:
    the oracle against the reference's iterations and solution (make_bench_pins.py)."""
    from conftest import GOLDEN

    g = np.load(GOLDEN / "pin_cfg1.npz")
    h, w = (int(x) for x in g["shape"])
    f = np.zeros(h * w)
    f[g["mask_idx"]] = g["vals0"].astype(np.float64)
    m = np.zeros(h * w, bool)
    m[g["mask_idx"]] = True
    st = {}
    u = inpaint.solve(f.reshape(h, w), m.reshape(h, w), tol=1e-6, max_iter=10000, strict=True, stats=st)
    assert np.array_equal(np.array(st["level_iterations"]), g["iters0"])
    assert np.abs(u[::8, ::4] - g["u0_grid"]).max() <= 1e-9
    assert np.abs(u.sum(axis=1) - g["u0_rows"]).max() <= 1e-9 * w
