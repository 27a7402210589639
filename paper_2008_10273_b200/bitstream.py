"""Container framing through the native parser (reference: bitstream.py)."""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from paper_2008_10273_b200 import _native as N
from paper_2008_10273_b200.errors import (  # noqa: F401  (re-exports)
    BadMagic,
    BitstreamError,
    LengthMismatch,
    Truncated,
    UnsupportedVersion,
)

MAGIC = b"HIVC"
VERSION = 1
HEADER_SIZE = 22


@dataclass(frozen=True)
class StreamHeader:
    width: int
    height: int
    frame_count: int
    fps_num: int
    fps_den: int
    gop_size: int
    channels: int
    intra_levels: int
    flow_levels: int
    residual_levels: int


def _view(data):
    a = np.frombuffer(data, dtype=np.uint8) if len(data) else np.zeros(1, dtype=np.uint8)
    return a, a.ctypes.data_as(C.c_void_p)


def stream_info(data: bytes) -> N.StreamInfo:
    """Validated header + GOP count (bitstream.py:102-154)."""
    data = bytes(data)
    a, p = _view(data)
    info = N.StreamInfo()
    N.check(N.lib.hivc_parse_header(p, len(data), C.byref(info)))
    del a
    return info


def unpack_header(data: bytes) -> StreamHeader:
    i = stream_info(data)
    return StreamHeader(i.width, i.height, i.frame_count, i.fps_num, i.fps_den, i.gop_size, i.channels,
                        i.intra_levels, i.flow_levels, i.residual_levels)


def read_stream(data: bytes):
    """Split a stream into (header, list of group payloads) (bitstream.py:132-154)."""
    data = bytes(data)
    header = unpack_header(data)
    pos = HEADER_SIZE
    payloads = []
    while pos < len(data):
        (n,) = struct.unpack_from("<I", data, pos)
        payloads.append(data[pos + 4 : pos + 4 + n])
        pos += 4 + n
    return header, payloads


def gop_frame_counts(data: bytes):
    data = bytes(data)
    a, p = _view(data)
    info = stream_info(data)
    counts = (C.c_int32 * max(info.gop_count, 1))()
    n = C.c_int32()
    N.check(N.lib.hivc_gop_frame_counts(p, len(data), counts, info.gop_count, C.byref(n)))
    del a
    return [int(counts[i]) for i in range(n.value)]
