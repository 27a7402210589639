"""Oracle: integer/byte parsing of the HIVC container (TEST INFRASTRUCTURE ONLY).

Restates, in plain Python, the reference's bit reader, LEB128 varints,
tANS ("FSE") decoder, category/extra-bit signed values, subdivision-tree
parsing and container framing.  Everything here is integer work and must
be bit-exact; the CUDA library's C++ host parser is compared against it.
"""

from __future__ import annotations

import struct

import numpy as np


class OracleError(Exception):
    """Base class; ``kind`` names the reference exception it stands for."""

    kind = "BitstreamError"


class Truncated(OracleError):
    kind = "Truncated"  # bitstream.Truncated / bits.TruncatedStream


class EntropyErr(OracleError):
    kind = "EntropyError"


class SubdivisionErr(OracleError):
    kind = "SubdivisionError"


class CodecErr(OracleError):
    kind = "CodecError"


class BadMagic(OracleError):
    kind = "BadMagic"


class UnsupportedVersion(OracleError):
    kind = "UnsupportedVersion"


class LengthMismatch(OracleError):
    kind = "LengthMismatch"


class QuantizeErr(OracleError):
    kind = "QuantizeError"


# ----------------------------------------------------------------------------- bits


class Bits:
    """MSB-first reader with a hard bit limit (reference ``bits.py:41-78``)."""

    def __init__(self, buf: bytes, nbits: int | None = None):
        self.buf = bytes(buf)
        self.limit = len(self.buf) * 8 if nbits is None else int(nbits)
        if self.limit > len(self.buf) * 8:
            raise Truncated("bit length exceeds buffer")
        self.pos = 0

    def take(self, n: int) -> int:
        if n == 0:
            return 0
        if self.pos + n > self.limit:
            raise Truncated("bit stream exhausted")
        v = 0
        for _ in range(n):
            byte = self.buf[self.pos >> 3]
            v = (v << 1) | ((byte >> (7 - (self.pos & 7))) & 1)
            self.pos += 1
        return v


def uvarint(data: bytes, pos: int):
    """LEB128 (reference ``bits.py:95-108``)."""
    val = 0
    sh = 0
    while True:
        if pos >= len(data):
            raise Truncated("varint runs past end of buffer")
        b = data[pos]
        pos += 1
        val |= (b & 0x7F) << sh
        if not (b & 0x80):
            return val, pos
        sh += 7
        if sh > 63:
            raise OracleError("varint too long")


# ----------------------------------------------------------------------------- tANS

MAX_STREAM_SYMBOLS = 1 << 28  # reference entropy.py:28


def fse_tables(counts, table_log: int):
    """(symbol, x, nbits) per slot — reference ``entropy.py:108-130``.

    Slots are visited with stride (S/2 + S/8 + 3) mod S and filled with
    the symbols in order, each repeated by its normalised count.  Within a
    symbol, slots in increasing slot index get x = count, count+1, ...;
    nbits = table_log + 1 - bit_length(x).
    """
    size = 1 << table_log
    counts = [int(c) for c in counts]
    if sum(counts) != size:
        raise EntropyErr("normalized counts must sum to table size")
    stride = (size >> 1) + (size >> 3) + 3
    sym_of = [0] * size
    k = 0
    for s, c in enumerate(counts):
        for _ in range(c):
            sym_of[(k * stride) & (size - 1)] = s
            k += 1
    nxt = list(counts)
    xs = [0] * size
    nbs = [0] * size
    for slot in range(size):
        s = sym_of[slot]
        xs[slot] = nxt[s]
        nxt[s] += 1
        nbs[slot] = table_log + 1 - xs[slot].bit_length()
    return sym_of, xs, nbs


def decode_symbols(data: bytes, pos: int = 0):
    """Self-contained tANS payload -> (int64 symbols, next pos).

    Reference ``entropy.py:227-240`` (header) and ``276-291`` / ``175-211``.
    """
    if pos >= len(data):
        raise Truncated("entropy payload truncated")
    table_log = data[pos]
    pos += 1
    if not 5 <= table_log <= 12:
        raise EntropyErr("bad table_log")
    nsym, pos = uvarint(data, pos)
    if nsym == 0 or nsym > (1 << table_log):
        raise EntropyErr("bad alphabet size")
    counts = []
    for _ in range(nsym):
        c, pos = uvarint(data, pos)
        counts.append(c)
    if pos + 10 > len(data):
        raise Truncated("entropy payload truncated")
    count, state, bit_len = struct.unpack_from("<IHI", data, pos)
    pos += 10
    if count > MAX_STREAM_SYMBOLS:
        raise EntropyErr("implausible symbol count")
    nbytes = (bit_len + 7) // 8
    if pos + nbytes > len(data):
        raise Truncated("entropy payload truncated")
    sym_of, xs, nbs = fse_tables(counts, table_log)
    rd = Bits(data[pos : pos + nbytes], bit_len)
    out = np.empty(count, dtype=np.int64)
    if count:
        size = 1 << table_log
        if not size <= state < 2 * size:
            raise EntropyErr("corrupt stream: initial state out of range")
        for i in range(count):
            slot = state - size
            out[i] = sym_of[slot]
            nb = nbs[slot]
            state = (xs[slot] << nb) | rd.take(nb) if nb else xs[slot]
        if state != size:
            raise EntropyErr("corrupt stream: final state mismatch")
    return out, pos + nbytes


def decode_signed_values(data: bytes, pos: int = 0):
    """Category symbols + raw MSB-first extra bits (reference ``entropy.py:311-338``).

    A category-k value with extra bits e is e when e >= 2^(k-1), else
    e - 2^k + 1 (JPEG sign convention, ``entropy.py:52-60``).
    """
    cats, pos = decode_symbols(data, pos)
    if pos + 4 > len(data):
        raise Truncated("entropy payload truncated")
    (bit_len,) = struct.unpack_from("<I", data, pos)
    pos += 4
    nbytes = (bit_len + 7) // 8
    if pos + nbytes > len(data):
        raise Truncated("entropy payload truncated")
    if cats.size and int(cats.max()) > 16:
        raise EntropyErr("bad category in stream")
    if int(cats.sum()) != bit_len:
        raise EntropyErr("extra-bits length mismatch")
    rd = Bits(data[pos : pos + nbytes], bit_len)
    vals = np.zeros(cats.size, dtype=np.int64)
    for i, k in enumerate(cats.tolist()):
        if k:
            e = rd.take(k)
            vals[i] = e if e >= (1 << (k - 1)) else e - (1 << k) + 1
    return vals, pos + nbytes


# ----------------------------------------------------------------------------- subdivision trees


def tree_leaves(rd: Bits, w: int, h: int):
    """Preorder leaf rectangles (x, y, w, h) of one serialised tree.

    Reference ``subdivision.py:198-222`` (parse_mask) and ``183-195`` /
    ``53-69`` (deserialize_tree + leaves): bit 1 halves the longer side
    (ties halve the width, first half rounded up), bit 0 is a leaf.
    """
    out = []
    todo = [(0, 0, w, h)]
    while todo:
        x, y, rw, rh = todo.pop()
        if rd.take(1):
            if rw == 1 and rh == 1:
                raise SubdivisionErr("split of a single pixel")
            if rh > rw:
                top = (rh + 1) // 2
                todo.append((x, y + top, rw, rh - top))
                todo.append((x, y, rw, top))
            else:
                left = (rw + 1) // 2
                todo.append((x + left, y, rw - left, rh))
                todo.append((x, y, left, rh))
        else:
            out.append((x, y, rw, rh))
    return out


def tree_mask(rd: Bits, w: int, h: int) -> np.ndarray:
    """Leaf-midpoint mask: point at (y + h//2, x + w//2) per leaf."""
    m = np.zeros((h, w), dtype=bool)
    for x, y, rw, rh in tree_leaves(rd, w, h):
        m[y + rh // 2, x + rw // 2] = True
    return m


def paint(leaves, values, w: int, h: int) -> np.ndarray:
    """Piecewise-constant plane from preorder leaf values (``subdivision.py:162-170``)."""
    if len(values) != len(leaves):
        raise SubdivisionErr("leaf value count mismatch")
    out = np.empty((h, w), dtype=np.float64)
    for (x, y, rw, rh), v in zip(leaves, values):
        out[y : y + rh, x : x + rw] = v
    return out


# ----------------------------------------------------------------------------- quantisers


def uniform_dequant(idx, lo: float, hi: float, levels: int) -> np.ndarray:
    """lo + idx * ((hi - lo) / (levels - 1)) — reference ``quantize.py:78-82``."""
    if not lo < hi:
        raise QuantizeErr("need lo < hi")
    step = (hi - lo) / (levels - 1)
    return lo + np.asarray(idx, dtype=np.float64) * step


def deadzone_unmap(idx, levels: int, scale: float) -> np.ndarray:
    """(idx * 127/((L-1)//2)) / 127 * scale — ``quantize.py:43-47,59-62,39-40``."""
    step = 127.0 / ((levels - 1) // 2)
    return np.asarray(idx, dtype=np.float64) * step / 127.0 * scale


# ----------------------------------------------------------------------------- container

HEADER_FMT = "<4sBHHIHHBBBBB"
HEADER_SIZE = struct.calcsize(HEADER_FMT)


def read_container(data: bytes):
    """(header dict, list of GOP payloads) — reference ``bitstream.py:102-154``."""
    if len(data) < HEADER_SIZE:
        raise Truncated("stream shorter than header")
    f = struct.unpack_from(HEADER_FMT, data, 0)
    if f[0] != b"HIVC":
        raise BadMagic("not a compressed video stream")
    if f[1] != 1:
        raise UnsupportedVersion("unsupported stream version")
    hdr = dict(
        width=f[2], height=f[3], frame_count=f[4], fps_num=f[5], fps_den=f[6], gop_size=f[7],
        channels=f[8], intra_levels=f[9] + 1, flow_levels=f[10] + 1, residual_levels=f[11],
    )
    if not (1 <= hdr["width"] and 1 <= hdr["height"]):
        raise OracleError("bad frame dimensions")
    if hdr["channels"] not in (1, 3):
        raise OracleError("channels must be 1 or 3")
    if hdr["gop_size"] < 1:
        raise OracleError("gop_size out of range")
    if hdr["intra_levels"] < 2 or hdr["flow_levels"] < 2:
        raise OracleError("quantizer levels out of range")
    if hdr["residual_levels"] < 3 or hdr["residual_levels"] % 2 == 0:
        raise OracleError("residual_levels must be odd and >= 3")
    if hdr["fps_num"] < 1 or hdr["fps_den"] < 1:
        raise OracleError("bad frame rate")
    pos = HEADER_SIZE
    gops = []
    while pos < len(data):
        if pos + 4 > len(data):
            raise Truncated("group length prefix cut short")
        (n,) = struct.unpack_from("<I", data, pos)
        pos += 4
        if pos + n > len(data):
            raise Truncated("group payload cut short")
        gops.append(data[pos : pos + n])
        pos += n
    want = -(-hdr["frame_count"] // hdr["gop_size"]) if hdr["frame_count"] else 0
    if len(gops) != want:
        raise LengthMismatch("group count does not match header")
    return hdr, gops
