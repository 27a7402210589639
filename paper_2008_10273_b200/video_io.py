"""Image and sequence files (reference: video_io.py).

Binary PNM stills (P5 gray / P6 colour, maxval 255) and YUV4MPEG2 sequences:
`C444 XCS=RGB` (untransformed R, G, B planes — the codec applies its own RCT)
and `Cmono` as in the reference (video_io.py:92-160), plus 8-bit 4:2:0
(`C420jpeg` / `C420paldv` / `C420mpeg2` / `C420`) for the three-stream 4:2:0
path of `yuv420.py`.  Plain host byte work: numpy views over the file bytes.
"""

from __future__ import annotations

import glob
import os
import re

import numpy as np

from paper_2008_10273_b200.frame import Frame

_Y4M = b"YUV4MPEG2"
_C420 = (b"420jpeg", b"420paldv", b"420mpeg2", b"420")


class VideoIOError(IOError):
    pass


# ----------------------------------------------------------------------------- PNM


def _pnm_header(data: bytes):
    """(width, height, maxval, offset of the pixel bytes); '#' comments allowed."""
    vals, pos = [], 2
    while len(vals) < 3:
        if pos >= len(data):
            raise VideoIOError("truncated header")
        c = data[pos : pos + 1]
        if c == b"#":
            end = data.find(b"\n", pos)
            if end < 0:
                raise VideoIOError("truncated header")
            pos = end + 1
        elif c.isspace():
            pos += 1
        else:
            m = re.match(rb"\d+", data[pos:])
            if m is None:
                raise VideoIOError("malformed header")
            vals.append(int(m.group()))
            pos += m.end()
    return vals[0], vals[1], vals[2], pos + 1  # one whitespace byte after maxval


def read_pnm(path) -> Frame:
    data = open(path, "rb").read()
    if data[:2] not in (b"P5", b"P6"):
        raise VideoIOError(f"unsupported image format {data[:2]!r}")
    w, h, maxval, pos = _pnm_header(data)
    if maxval != 255:
        raise VideoIOError(f"only maxval 255 supported, got {maxval}")
    ch = 3 if data[:2] == b"P6" else 1
    if len(data) - pos < w * h * ch:
        raise VideoIOError("pixel data truncated")
    px = np.frombuffer(data, dtype=np.uint8, count=w * h * ch, offset=pos).astype(np.int32)
    if ch == 3:
        px = px.reshape(h, w, 3)
        return Frame((px[..., 0], px[..., 1], px[..., 2]), colorspace="rgb")
    return Frame((px.reshape(h, w),), colorspace="gray")


def write_pnm(path, frame: Frame):
    if frame.channels == 3:
        body = np.stack(frame.planes, axis=-1).astype(np.uint8).tobytes()
        head = b"P6 %d %d 255\n" % (frame.width, frame.height)
    else:
        body = frame.planes[0].astype(np.uint8).tobytes()
        head = b"P5 %d %d 255\n" % (frame.width, frame.height)
    with open(path, "wb") as fh:
        fh.write(head + body)


# ----------------------------------------------------------------------------- YUV4MPEG2


def _y4m_params(data: bytes):
    nl = data.find(b"\n")
    if nl < 0 or not data.startswith(_Y4M):
        raise VideoIOError("not a YUV4MPEG2 stream")
    w = h = None
    fps, mode = (25, 1), b"444"
    for tok in data[len(_Y4M) : nl].split():
        key, val = tok[:1], tok[1:]
        if key == b"W":
            w = int(val)
        elif key == b"H":
            h = int(val)
        elif key == b"F":
            a, b = val.split(b":")
            fps = (int(a), int(b))
        elif key == b"C":
            mode = val
    if not w or not h:
        raise VideoIOError("missing frame dimensions")
    if not (mode == b"mono" or mode.startswith(b"444") or mode in _C420):
        raise VideoIOError(f"unsupported chroma mode C{mode.decode()}")
    return w, h, fps, mode, nl + 1


def _y4m_frames(data: bytes, pos: int, plane_sizes):
    """Split the FRAME records into lists of planes with the given (h, w) sizes."""
    out, need = [], sum(a * b for a, b in plane_sizes)
    while pos < len(data):
        nl = data.find(b"\n", pos)
        if nl < 0 or not data[pos:nl].startswith(b"FRAME"):
            raise VideoIOError(f"bad frame marker at byte {pos}")
        pos = nl + 1
        if pos + need > len(data):
            raise VideoIOError("frame data truncated")
        planes = []
        for ph, pw in plane_sizes:
            planes.append(np.frombuffer(data, dtype=np.uint8, count=ph * pw, offset=pos).reshape(ph, pw))
            pos += ph * pw
        out.append(planes)
    if not out:
        raise VideoIOError("stream holds no frames")
    return out


def read_y4m(path):
    """4:4:4 (RGB) or mono sequence -> (frames, (fps_num, fps_den)) (video_io.py:110-160)."""
    data = open(path, "rb").read()
    w, h, fps, mode, pos = _y4m_params(data)
    if mode in _C420:
        raise VideoIOError("4:2:0 sequence: use read_y4m_420")
    ch = 1 if mode == b"mono" else 3
    recs = _y4m_frames(data, pos, [(h, w)] * ch)
    cs = "rgb" if ch == 3 else "gray"
    return [Frame(tuple(p.astype(np.int32) for p in r), colorspace=cs) for r in recs], fps


def write_y4m(path, frames, fps=(25, 1)):
    """RGB frames as C444 XCS=RGB, gray frames as Cmono (video_io.py:92-107)."""
    if not frames:
        raise VideoIOError("no frames to write")
    f0 = frames[0]
    tag = b"C444 XCS=RGB" if f0.channels == 3 else b"Cmono"
    with open(path, "wb") as fh:
        fh.write(_Y4M + b" W%d H%d F%d:%d Ip A1:1 %s\n" % (f0.width, f0.height, fps[0], fps[1], tag))
        for f in frames:
            if (f.width, f.height, f.channels) != (f0.width, f0.height, f0.channels):
                raise VideoIOError("frame geometry mismatch")
            fh.write(b"FRAME\n")
            for p in f.planes:
                fh.write(np.ascontiguousarray(p, dtype=np.uint8).tobytes())


def read_y4m_420(path):
    """8-bit 4:2:0 sequence -> (Y (n, H, W), Cb, Cr (n, ceil(H/2), ceil(W/2)) uint8, fps)."""
    data = open(path, "rb").read()
    w, h, fps, mode, pos = _y4m_params(data)
    if mode not in _C420:
        raise VideoIOError(f"not a 4:2:0 sequence (C{mode.decode()})")
    cw, chh = (w + 1) // 2, (h + 1) // 2
    recs = _y4m_frames(data, pos, [(h, w), (chh, cw), (chh, cw)])
    return tuple(np.stack([r[i] for r in recs]) for i in range(3)) + (fps,)


def write_y4m_420(path, y, cb, cr, fps=(25, 1)):
    y, cb, cr = (np.asarray(a) for a in (y, cb, cr))
    n, h, w = y.shape
    if cb.shape != (n, (h + 1) // 2, (w + 1) // 2) or cr.shape != cb.shape:
        raise VideoIOError("chroma planes must be (n, ceil(H/2), ceil(W/2))")
    with open(path, "wb") as fh:
        fh.write(_Y4M + b" W%d H%d F%d:%d Ip A1:1 C420jpeg\n" % (w, h, fps[0], fps[1]))
        for i in range(n):
            fh.write(b"FRAME\n")
            for p in (y[i], cb[i], cr[i]):
                fh.write(np.ascontiguousarray(np.clip(p, 0, 255), dtype=np.uint8).tobytes())


def read_frames(path):
    """A .y4m file, one PNM image, a glob over PNM images or a directory of them
    (sorted by name) -> (frames, fps) (video_io.py:163-184)."""
    path = str(path)
    if path.endswith(".y4m"):
        return read_y4m(path)
    if os.path.isdir(path) or any(c in path for c in "*?["):
        if os.path.isdir(path):
            names = sorted(os.path.join(path, n) for n in os.listdir(path) if n.endswith((".pgm", ".ppm", ".pnm")))
        else:
            names = sorted(glob.glob(path))
        if not names:
            raise VideoIOError(f"no frames match {path!r}")
        return [read_pnm(n) for n in names], (25, 1)
    return [read_pnm(path)], (25, 1)
