"""PNM / YUV4MPEG2 files and the 4:2:0 three-stream container (host only)."""

import numpy as np
import pytest


def _rgb(seed, h=9, w=13):
    from paper_2008_10273_b200.frame import Frame

    rng = np.random.default_rng(seed)
    return Frame(tuple(rng.integers(0, 256, (h, w)).astype(np.int32) for _ in range(3)), colorspace="rgb")


def test_pnm_round_trips(tmp_path):
    from paper_2008_10273_b200.frame import Frame
    from paper_2008_10273_b200.video_io import VideoIOError, read_frames, read_pnm, write_pnm

    f = _rgb(0)
    write_pnm(tmp_path / "a.ppm", f)
    assert read_pnm(tmp_path / "a.ppm") == f
    g = Frame((f.planes[0],), colorspace="gray")
    write_pnm(tmp_path / "b.pgm", g)
    assert read_pnm(tmp_path / "b.pgm") == g
    (tmp_path / "c.pgm").write_bytes(b"P5\n# comment\n2 1\n255\n\x07\x09")
    assert read_pnm(tmp_path / "c.pgm").planes[0].tolist() == [[7, 9]]
    for bad in (b"P2 1 1 255\n0", b"P5 2 2 255\n\x00", b"P5 1 1 65535\n\x00\x00"):
        (tmp_path / "d.pgm").write_bytes(bad)
        with pytest.raises(VideoIOError):
            read_pnm(tmp_path / "d.pgm")
    d = tmp_path / "seq"
    d.mkdir()
    for i in range(3):
        write_pnm(d / f"f{i:02d}.ppm", _rgb(i))
    frames, fps = read_frames(d)
    assert fps == (25, 1) and frames == [_rgb(i) for i in range(3)]
    assert read_frames(str(d / "f0*.ppm"))[0] == frames


def test_y4m_round_trips(tmp_path):
    from paper_2008_10273_b200.frame import Frame
    from paper_2008_10273_b200.video_io import VideoIOError, read_y4m, read_y4m_420, write_y4m, write_y4m_420

    clip = [_rgb(i) for i in range(4)]
    write_y4m(tmp_path / "a.y4m", clip, fps=(30000, 1001))
    frames, fps = read_y4m(tmp_path / "a.y4m")
    assert frames == clip and fps == (30000, 1001)
    gray = [Frame((f.planes[1],), colorspace="gray") for f in clip]
    write_y4m(tmp_path / "g.y4m", gray)
    assert read_y4m(tmp_path / "g.y4m")[0] == gray
    rng = np.random.default_rng(5)
    y = rng.integers(0, 256, (3, 9, 13), dtype=np.uint8)
    cb = rng.integers(0, 256, (3, 5, 7), dtype=np.uint8)
    cr = rng.integers(0, 256, (3, 5, 7), dtype=np.uint8)
    write_y4m_420(tmp_path / "c.y4m", y, cb, cr)
    y2, cb2, cr2, fps = read_y4m_420(tmp_path / "c.y4m")
    assert np.array_equal(y2, y) and np.array_equal(cb2, cb) and np.array_equal(cr2, cr)
    with pytest.raises(VideoIOError):
        read_y4m(tmp_path / "c.y4m")
    with pytest.raises(VideoIOError):
        write_y4m_420(tmp_path / "x.y4m", y, cb[:, :4], cr)
    (tmp_path / "t.y4m").write_bytes((tmp_path / "a.y4m").read_bytes()[:-5])
    with pytest.raises(VideoIOError):
        read_y4m(tmp_path / "t.y4m")
    (tmp_path / "u.y4m").write_bytes(b"YUV4MPEG2 W2 H2 C422\nFRAME\n" + bytes(8))
    with pytest.raises(VideoIOError):
        read_y4m(tmp_path / "u.y4m")


def test_420_container_and_chroma_flow():
    from paper_2008_10273_b200 import yuv420
    from paper_2008_10273_b200.errors import BitstreamError, Truncated
    from paper_2008_10273_b200.flow import FlowField
    from paper_2008_10273_b200.synth import downsample2

    s = (b"HIVCaaa", b"HIVCbb", b"")
    assert yuv420.unpack(yuv420.pack(s)) == s
    with pytest.raises(Truncated):
        yuv420.unpack(yuv420.pack(s)[:-3] + b"")
    with pytest.raises(BitstreamError):
        yuv420.unpack(b"XXXX")
    a = np.random.default_rng(1).normal(size=(7, 10))
    assert np.array_equal(yuv420.half_plane(a), downsample2(a))  # the config-4 recipe
    f = yuv420.chroma_flow(FlowField(a, -a))
    assert f.u.shape == (4, 5) and np.array_equal(f.u, downsample2(a) * 0.5)
