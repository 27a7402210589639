"""Codec-level behaviour on the B200, restating the checks of the reference's
own test suite (reference pkg/tests/test_codec.py, test_prediction.py,
test_flow.py) against this package: round trips, losslessness, rate-distortion
ordering, rate control, determinism, corrupt-stream handling.  Needs a B200."""

import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _rgb_clip(n, h, w, seed):
    from paper_2008_10273_b200.frame import Frame
    from paper_2008_10273_b200.synth import synth_clip, to_codec_planes

    clip = to_codec_planes(synth_clip(n, h, w, blobs=4, rects=2, v=2.0, seed=seed, channels=3))
    return [Frame(tuple(f[c] for c in range(3)), colorspace="rgb") for f in clip]


def _gray(clip):
    from paper_2008_10273_b200.frame import Frame

    return [Frame((f.planes[0],), colorspace="gray") for f in clip]


def _mean_psnr(a, b):
    from paper_2008_10273_b200.frame import psnr

    return float(np.mean([psnr(x, y) for x, y in zip(a, b)]))


def test_lossless_configuration_round_trips_exactly():
    """Full mask, 256 levels, GOP 1: every frame (RGB through the RCT) comes back exactly."""
    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.frame import Frame

    cfg = codec.EncoderConfig(gop_size=1, intra_mask_fraction=1.0, intra_levels=256, self_check=True)
    clip = _rgb_clip(3, 40, 48, seed=1)
    assert codec.decode(codec.encode(clip, cfg)) == clip
    rng = np.random.default_rng(2)
    noise = Frame(tuple(rng.integers(0, 256, (24, 24)).astype(np.int32) for _ in range(3)))
    assert codec.decode(codec.encode([noise], cfg))[0] == noise


def test_gray_and_lossy_round_trip_quality():
    from paper_2008_10273_b200 import codec

    gray = _gray(_rgb_clip(4, 48, 48, seed=3))
    out = codec.decode(codec.encode(gray, codec.EncoderConfig(gop_size=4, intra_mask_fraction=0.2, self_check=True)))
    assert len(out) == 4 and all(f.colorspace == "gray" for f in out)
    assert _mean_psnr(gray, out) >= 28.0
    clip = _rgb_clip(5, 48, 64, seed=4)
    cfg = codec.EncoderConfig(gop_size=5, intra_mask_fraction=0.15, residual_points=8, self_check=True)
    assert _mean_psnr(clip, codec.decode(codec.encode(clip, cfg))) >= 30.0


def test_static_video_inter_frame_is_nearly_free():
    """A flat clip: the P-frame is a zero flow and an empty residual."""
    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.bitstream import read_stream
    from paper_2008_10273_b200.frame import Frame

    flat = Frame(tuple(np.full((160, 240), v, dtype=np.int32) for v in (90, 120, 60)), colorspace="rgb")
    stream = codec.encode([flat, flat], codec.EncoderConfig(gop_size=2, intra_mask_fraction=0.1, self_check=True))
    payload = read_stream(stream)[1][0]
    pos, sizes = 2, []
    for _ in range(2):
        pred_len = struct.unpack_from("<BI", payload, pos)[1]
        pos += 5 + pred_len
        (res_len,) = struct.unpack_from("<I", payload, pos)
        pos += 4 + res_len
        sizes.append(9 + pred_len + res_len)
    assert sizes[1] < 0.10 * sizes[0]


def test_multi_gop_stream_and_determinism():
    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.bitstream import read_stream

    clip = _rgb_clip(7, 40, 48, seed=8)
    cfg = codec.EncoderConfig(gop_size=3, intra_mask_fraction=0.2, self_check=True)
    stream = codec.encode(clip, cfg)
    assert len(read_stream(stream)[1]) == 3
    assert codec.encode(clip, cfg, workers=1) == stream  # threads do not change the bytes
    a, b = codec.decode(stream), codec.decode(stream)
    assert len(a) == 7 and a == b


def test_rate_distortion_ordering():
    """Larger budgets: quality does not drop and the ratio does not rise (medians)."""
    from paper_2008_10273_b200 import codec

    budgets = [
        codec.EncoderConfig(gop_size=4, intra_mask_fraction=0.02, residual_points=2, flow_points=20,
                            residual_levels=31),
        codec.EncoderConfig(gop_size=4, intra_mask_fraction=0.08, residual_points=6, flow_points=80,
                            residual_levels=63),
        codec.EncoderConfig(gop_size=4, intra_mask_fraction=0.32, residual_points=18, flow_points=320,
                            residual_levels=127),
    ]
    ratio, quality = [[], [], []], [[], [], []]
    for seed in (10, 11):
        clip = _rgb_clip(4, 48, 64, seed=seed)
        for i, cfg in enumerate(budgets):
            s = codec.encode(clip, cfg)
            ratio[i].append(4 * 48 * 64 * 3 / len(s))
            quality[i].append(_mean_psnr(clip, codec.decode(s)))
    q, r = [np.median(x) for x in quality], [np.median(x) for x in ratio]
    assert q[0] <= q[1] <= q[2]
    assert r[0] >= r[1] >= r[2]


def test_target_ratio_hits_the_target():
    from paper_2008_10273_b200 import codec

    clip = _rgb_clip(6, 48, 96, seed=12)
    stream, ratio, used = codec.encode_target_ratio(clip, codec.EncoderConfig(gop_size=6), 15.0)
    raw = 6 * 48 * 96 * 3
    assert abs(raw / len(stream) - 15.0) / 15.0 <= 0.10
    assert ratio == pytest.approx(raw / len(stream))
    assert isinstance(used, codec.EncoderConfig)
    with pytest.raises(ValueError):
        codec.encode_target_ratio(clip[:1], codec.EncoderConfig(), 1.0)


def test_corrupt_streams_raise_bitstream_errors():
    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.errors import BitstreamError

    stream = codec.encode(_rgb_clip(2, 32, 32, seed=13), codec.EncoderConfig(gop_size=2))
    for cut in (10, len(stream) - 3):
        with pytest.raises(BitstreamError):
            codec.decode(stream[:cut])
    rng = np.random.default_rng(15)
    for _ in range(40):
        m = bytearray(stream)
        m[int(rng.integers(30, len(m)))] ^= int(rng.integers(1, 256))
        try:
            codec.decode(bytes(m))
        except (BitstreamError, ValueError):
            pass


def test_intra_prediction_properties():
    """Constant frame: one point reproduces it; the payload decodes the same way twice."""
    from paper_2008_10273_b200.prediction import decode_intra, encode_intra

    const = [np.full((20, 30), 77, dtype=np.int64)]
    payload = encode_intra(const, 1, 256)
    pred, pos = decode_intra(payload, 0, (20, 30), 1, 256)
    assert pos == len(payload) and np.array_equal(np.rint(pred[0]), np.full((20, 30), 77.0))
    clip = _rgb_clip(1, 40, 56, seed=20)[0]
    planes = [p.astype(np.int64) for p in clip.planes]
    payload = encode_intra(planes, 200, 256)
    a, _ = decode_intra(payload, 0, (40, 56), 3, 256)
    b, _ = decode_intra(payload, 0, (40, 56), 3, 256)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert all(np.abs(np.asarray(p)).max() < 600 for p in a)


def test_flow_compression_properties():
    """Zero flow: tiny exact payload.  Piecewise-constant flow on tree cells: exact."""
    from paper_2008_10273_b200.flow import FlowField, compress_flow, decompress_flow

    z = FlowField(np.zeros((30, 40)), np.zeros((30, 40)))
    b = compress_flow(z, 50, 256)
    dec, pos = decompress_flow(b, 0, (30, 40), 256)
    assert pos == len(b) and len(b) < 64
    assert not np.asarray(dec.u).any() and not np.asarray(dec.v).any()
    u = np.zeros((32, 32))
    u[:, 16:] = 2.0  # one split of the root separates the two halves exactly
    v = np.zeros((32, 32))
    v[16:, :] = -1.0
    dec, _ = decompress_flow(compress_flow(FlowField(u, v), 8, 256), 0, (32, 32), 256)
    assert np.abs(np.asarray(dec.u) - u).max() < 1e-6 and np.abs(np.asarray(dec.v) - v).max() < 1e-6


def test_inter_prediction_zero_flow_is_identity():
    from paper_2008_10273_b200.flow import FlowField
    from paper_2008_10273_b200.prediction import predict_inter

    planes = [np.random.default_rng(5).integers(0, 256, (24, 36)).astype(np.int64) for _ in range(3)]
    out = predict_inter(planes, FlowField(np.zeros((24, 36)), np.zeros((24, 36))))
    assert all(np.array_equal(o, p.astype(np.float64)) for o, p in zip(out, planes))


def test_420_three_stream_round_trip():
    """yuv420.encode_420: luma flows estimated once, chroma flows derived; decode_420
    decodes the three streams in one native call, equal to per-stream decodes."""
    from paper_2008_10273_b200 import codec, yuv420
    from paper_2008_10273_b200.flow import flow_brox
    from paper_2008_10273_b200.synth import synth_420

    y, cb, cr = synth_420(5, 40, 56, blobs=4, rects=2, v=2.0, seed=30)
    cfg = codec.EncoderConfig(gop_size=3, intra_mask_fraction=0.1)
    streams = yuv420.encode_420(y, cb, cr, cfg)
    yf = y.astype(np.float64)
    flows = [[flow_brox(yf[1], yf[0]), flow_brox(yf[2], yf[1])], [flow_brox(yf[4], yf[3])]]
    frames = [codec.Frame((p,), colorspace="gray") for p in y]
    assert streams[0] == codec.encode(frames, cfg, _flows=flows)
    dy, dcb, dcr = yuv420.decode_420(streams)
    for dec, s in zip((dy, dcb, dcr), streams):
        ref = np.stack([f.planes[0] for f in codec.decode(s)])
        assert np.array_equal(dec.astype(np.int32), ref)
    gy, _, _ = yuv420.decode_420(yuv420.unpack(yuv420.pack(streams)), device="cuda")
    assert np.array_equal(gy.cpu().numpy(), dy)
    assert _psnr_arr(dy, y) > 25 and _psnr_arr(dcb, cb) > 25


def _psnr_arr(a, b):
    d = a.astype(np.float64) - b
    return 10 * np.log10(255.0**2 / max(np.mean(d * d), 1e-12))


def test_corrupt_gop_frame_count_raises_reference_error(cfg0_stream):
    """The reference decodes the 10 records, then raises Truncated("frame record
    cut short in group 0") (codec.py:497-499); so must the GPU decode, without
    first sizing 60000 frames of output."""
    import struct

    from paper_2008_10273_b200 import codec, errors

    d = bytearray(cfg0_stream)
    struct.pack_into("<H", d, 26, 60000)
    with pytest.raises(errors.Truncated, match="frame record cut short in group 0"):
        codec.decode(bytes(d))
