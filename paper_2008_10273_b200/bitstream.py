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

    def __post_init__(self):  # bitstream.py:70-82
        if not (1 <= self.width <= 65535 and 1 <= self.height <= 65535):
            raise BitstreamError("bad frame dimensions")
        if self.channels not in (1, 3):
            raise BitstreamError("channels must be 1 or 3")
        if self.gop_size < 1 or self.gop_size > 255:
            raise BitstreamError("gop_size out of range")
        if not (2 <= self.intra_levels <= 256 and 2 <= self.flow_levels <= 256):
            raise BitstreamError("quantizer levels out of range")
        if self.residual_levels < 3 or self.residual_levels % 2 == 0:
            raise BitstreamError("residual_levels must be odd and >= 3")

    def pack(self) -> bytes:
        """22-byte little-endian header; quantiser level counts stored minus one (bitstream.py:84-99)."""
        return MAGIC + struct.pack("<BHHIHHBBBBB", VERSION, self.width, self.height, self.frame_count, self.fps_num,
                                   self.fps_den, self.gop_size, self.channels, self.intra_levels - 1,
                                   self.flow_levels - 1, self.residual_levels)


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


def write_stream(header: StreamHeader, gop_payloads) -> bytes:
    """Header, then each GOP payload behind a u32 length (bitstream.py:124-129)."""
    out = bytearray(header.pack())
    for payload in gop_payloads:
        out += struct.pack("<I", len(payload))
        out += payload
    return bytes(out)


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
