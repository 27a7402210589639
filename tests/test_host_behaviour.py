"""Host-side behaviour (no GPU), restating the checks of the reference's own
suite (reference pkg/tests/test_entropy.py, test_subdivision.py,
test_quantize.py, test_frame.py, test_bitstream.py) against this package."""

import math

import numpy as np
import pytest


# ----------------------------------------------------------------------------- entropy


def test_categories_are_a_bijection():
    from paper_2008_10273_b200.entropy import MAX_MAGNITUDE, from_category, to_category
    from paper_2008_10273_b200.errors import EntropyError

    assert to_category(0) == (0, 0) and to_category(5) == (3, 5) and to_category(-1) == (1, 0)
    for v in list(range(-1024, 1025)) + [MAX_MAGNITUDE, -MAX_MAGNITUDE]:
        assert from_category(*to_category(v)) == v
    with pytest.raises(EntropyError):
        to_category(MAX_MAGNITUDE + 1)


def test_normalize_counts_invariants():
    from paper_2008_10273_b200.entropy import normalize_counts
    from paper_2008_10273_b200.errors import EntropyError

    assert normalize_counts(np.ones(256, dtype=np.int64), 8).tolist() == [1] * 256
    c = normalize_counts([900, 90, 10], 8)
    assert c.sum() == 256 and (c >= 1).all()
    rng = np.random.default_rng(0)
    for tl in (5, 8, 12):
        h = rng.integers(0, 50, 20)
        h[3] = 1
        c = normalize_counts(h, tl)
        assert c.sum() == 1 << tl and ((c > 0) == (h > 0)).all()
    with pytest.raises(EntropyError):
        normalize_counts(np.zeros(4, dtype=np.int64), 8)


def test_entropy_payload_sizes():
    from paper_2008_10273_b200 import entropy

    assert len(entropy.encode_symbols([7] * 4000)) < 40  # one symbol: no information
    b = entropy.encode_symbols([])
    assert entropy.decode_symbols(b)[0].size == 0
    rng = np.random.default_rng(1)
    p = np.array([0.5, 0.25, 0.125, 0.0625, 0.0625])
    s = rng.choice(5, size=200_000, p=p)
    bits = 8 * len(entropy.encode_symbols(s))
    h = -(p * np.log2(p)).sum() * s.size
    assert bits <= 1.02 * h + 2048  # within 2 % of the entropy


def test_entropy_decoder_rejects_corruption_and_truncation():
    from paper_2008_10273_b200 import entropy
    from paper_2008_10273_b200.errors import EntropyError, TruncatedStream

    b = entropy.encode_symbols(np.random.default_rng(2).integers(0, 9, 3000))
    for cut in (0, 3, len(b) // 2, len(b) - 1):
        with pytest.raises((TruncatedStream, EntropyError)):
            entropy.decode_symbols(b[:cut])
    rng = np.random.default_rng(3)
    for _ in range(50):
        m = bytearray(b)
        m[int(rng.integers(0, len(m)))] ^= int(rng.integers(1, 256))
        try:
            entropy.decode_symbols(bytes(m))
        except (TruncatedStream, EntropyError):
            pass


# ----------------------------------------------------------------------------- subdivision


def test_split_rules():
    from paper_2008_10273_b200.subdivision import split_children

    assert split_children(0, 0, 8, 8) == ((0, 0, 4, 8), (4, 0, 4, 8))  # tie: width
    assert split_children(0, 0, 4, 8) == ((0, 0, 4, 4), (0, 4, 4, 4))  # taller: height
    assert split_children(2, 3, 7, 5) == ((2, 3, 4, 5), (6, 3, 3, 5))  # ceiling halves
    assert split_children(0, 0, 1, 3) == ((0, 0, 1, 2), (0, 2, 1, 1))


def test_subdivision_on_constant_and_step_planes():
    from paper_2008_10273_b200 import subdivision as S

    t = S.subdivide_by_error(np.full((16, 16), 3.0), 10, min_error=0.0)
    assert t.leaf_count == 1 and t.bits == (0,)
    a = S.subdivide_by_error(np.full((16, 16), 3.0), 10)
    assert a.leaf_count == 10 and a.leaves() == S.subdivide_by_error(np.full((16, 16), 3.0), 10).leaves()
    step = np.zeros((16, 32))
    step[:, 16:] = 100.0
    t = S.subdivide_by_error(step, 2)
    assert t.leaves() == [(0, 0, 16, 16), (16, 0, 16, 16)]


def test_subdivision_masks_and_means():
    from paper_2008_10273_b200 import subdivision as S

    rng = np.random.default_rng(4)
    p = rng.normal(size=(21, 34)) * 10
    t = S.subdivide_by_error(p, 50)
    m = S.mask_from_tree(t)
    assert m.sum() == t.leaf_count == 50
    for x, y, w, h in t.leaves():
        assert m[y + h // 2, x + w // 2]
    means = S.leaf_means(t, p)
    for (x, y, w, h), v in zip(t.leaves(), means):
        assert v == p[y : y + h, x : x + w].mean()


def test_subdivision_error_falls_with_budget():
    from paper_2008_10273_b200 import subdivision as S

    p = np.cumsum(np.random.default_rng(5).normal(size=(40, 40)), axis=1)
    errs = []
    for n in (4, 16, 64, 256):
        t = S.subdivide_by_error(p, n)
        approx = np.empty_like(p)
        for (x, y, w, h), v in zip(t.leaves(), S.leaf_means(t, p)):
            approx[y : y + h, x : x + w] = v
        errs.append(float(((p - approx) ** 2).sum()))
    assert errs == sorted(errs, reverse=True)


def test_serialised_trees_parse_back():
    from paper_2008_10273_b200 import subdivision as S
    from paper_2008_10273_b200.flow import _tree_leaves

    rng = np.random.default_rng(6)
    for _ in range(20):
        h, w = (int(v) for v in rng.integers(1, 40, 2))
        n = int(rng.integers(1, h * w + 1))
        t = S.subdivide_by_error(rng.normal(size=(h, w)), n)
        got = _tree_leaves(t.packed, 0, len(t.bits), w, h)
        assert got.tolist() == [list(r) for r in t.leaves()]


# ----------------------------------------------------------------------------- quantisers


def test_quantiser_semantics():
    from paper_2008_10273_b200 import quantize as Q
    from paper_2008_10273_b200.errors import QuantizeError

    assert Q.map_coefficients(np.zeros(3), 2.0).tolist() == [0.0] * 3
    assert Q.map_coefficients([10.0, -10.0], 1.0).tolist() == [127.0, -127.0]
    assert Q.map_coefficients([2.0], 2.0)[0] == 127.0
    x = np.linspace(-1.9, 1.9, 7)
    assert np.allclose(Q.unmap_coefficients(Q.map_coefficients(x, 2.0), 2.0), x)
    with pytest.raises(QuantizeError):
        Q.coefficient_scale(np.zeros(0))
    step = Q.deadzone_step(63)
    assert Q.deadzone_quantize([0.0, 0.99 * step, step, -step, -1.5 * step], 63).tolist() == [0, 0, 1, -1, -1]
    assert Q.deadzone_dequantize([0], 63)[0] == 0.0
    with pytest.raises(QuantizeError):
        Q.deadzone_step(4)
    assert Q.uniform_quantize([0.0, 255.0], 0.0, 255.0, 256).tolist() == [0, 255]
    assert Q.uniform_quantize(np.arange(256.0), 0.0, 255.0, 256).tolist() == list(range(256))
    v = np.random.default_rng(7).uniform(-3, 9, 1000)
    r = Q.uniform_dequantize(Q.uniform_quantize(v, -3.0, 9.0, 17), -3.0, 9.0, 17)
    assert np.abs(r - v).max() <= 0.5 * 12.0 / 16 + 1e-12


# ----------------------------------------------------------------------------- frames and container


def test_rct_and_psnr():
    from paper_2008_10273_b200.errors import FrameError
    from paper_2008_10273_b200.frame import Frame, clip_plane, psnr, rct_forward, rct_inverse

    one = lambda *v: tuple(np.full((1, 1), x, dtype=np.int32) for x in v)  # noqa: E731
    yuv = rct_forward(Frame(one(255, 0, 0)))
    assert [int(p[0, 0]) for p in yuv.planes] == [63, 0, 255]
    rng = np.random.default_rng(8)
    f = Frame(tuple(rng.integers(0, 256, (9, 13)).astype(np.int32) for _ in range(3)))
    yuv = rct_forward(f)
    assert rct_inverse(yuv) == f
    assert 0 <= yuv.planes[0].min() and yuv.planes[0].max() <= 255
    assert max(np.abs(yuv.planes[1]).max(), np.abs(yuv.planes[2]).max()) <= 255
    with pytest.raises(FrameError):
        rct_forward(Frame(one(1), colorspace="gray"))
    with pytest.raises(FrameError):
        rct_inverse(Frame(one(0, 300, 0), colorspace="yuv"))
    assert psnr(f, f) == math.inf
    z = Frame(tuple(np.zeros((4, 4), np.int32) for _ in range(3)))
    w = Frame(tuple(np.full((4, 4), 255, np.int32) for _ in range(3)))
    assert psnr(z, w) == 0.0 and psnr(z, w) == psnr(w, z)
    assert clip_plane(np.array([-3.4, 260.6]), 0, "rgb").tolist() == [0, 255]
    assert clip_plane(np.array([-300.0, 2.5]), 1, "yuv").tolist() == [-255, 2]


def test_stream_header_validation_and_gop_framing():
    from paper_2008_10273_b200.bitstream import StreamHeader, read_stream, write_stream
    from paper_2008_10273_b200.errors import BadMagic, BitstreamError, LengthMismatch, Truncated, UnsupportedVersion

    h = StreamHeader(64, 48, 3, 25, 1, 2, 1, 256, 256, 63)
    for bad in (dict(width=0), dict(channels=2), dict(gop_size=0), dict(intra_levels=1), dict(residual_levels=4)):
        with pytest.raises(BitstreamError):
            StreamHeader(**{**h.__dict__, **bad})
    s = write_stream(h, [b"\x02\x00abc", b"\x01\x00de"])
    hh, gops = read_stream(s)
    assert hh == h and gops == [b"\x02\x00abc", b"\x01\x00de"]
    with pytest.raises(BadMagic):
        read_stream(b"XXXX" + s[4:])
    with pytest.raises(UnsupportedVersion):
        read_stream(s[:4] + b"\x09" + s[5:])
    with pytest.raises(Truncated):
        read_stream(s[:-1])
    with pytest.raises(LengthMismatch):
        read_stream(write_stream(h, [b"\x02\x00abc"]))


def test_corrupt_gop_frame_count_sizes_outputs_by_records(cfg0_stream):
    """A GOP whose u16 frame count is corrupt (60000 instead of 10) must not size
    the output buffers: frames_shape counts the records that fit."""
    import struct

    from paper_2008_10273_b200 import codec

    d = bytearray(cfg0_stream)
    struct.pack_into("<H", d, 26, 60000)  # GOP 0's frame count (22-byte header + u32 length)
    assert codec.frames_shape(bytes(d))[0] == 10
    assert codec.frames_shape(cfg0_stream)[0] == 10
