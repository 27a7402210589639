"""tANS / category payloads through the native coder (reference: entropy.py).

``decode_symbols`` (entropy.py:276-291), ``decode_signed_values``
(entropy.py:311-338), ``encode_symbols`` (entropy.py:255-273) and
``encode_signed_values`` (entropy.py:294-308) keep their signatures and run
the bit-exact C++ coder of libhivc_b200 (csrc/parse.cpp, csrc/encode.cpp) —
host code, no GPU needed.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2008_10273_b200 import _native as N
from paper_2008_10273_b200.errors import EntropyError  # noqa: F401  (re-export)


def _call(fn, data, pos):
    data = bytes(data)
    buf = C.create_string_buffer(data, max(len(data), 1))
    count = C.c_size_t()
    nxt = C.c_size_t()
    N.check(fn(buf, len(data), pos, None, 0, C.byref(count), C.byref(nxt)))
    out = np.empty(count.value, dtype=np.int64)
    N.check(fn(buf, len(data), pos, out.ctypes.data_as(N.c_i64_p), count.value, C.byref(count), C.byref(nxt)))
    return out, int(nxt.value)


def decode_symbols(data: bytes, pos: int = 0):
    """Inverse of encode_symbols; returns (symbols, next position)."""
    return _call(N.lib.hivc_parse_symbols, data, pos)


def decode_signed_values(data: bytes, pos: int = 0):
    """Inverse of encode_signed_values; returns (values, next position)."""
    return _call(N.lib.hivc_parse_signed_values, data, pos)


def _encode(fn, values, table_log):
    v = np.ascontiguousarray(np.asarray(values, dtype=np.int64).reshape(-1))
    tl = -1 if table_log is None else int(table_log)
    cap = 64 + 4 * v.size
    for _ in range(2):
        buf = C.create_string_buffer(cap)
        size = C.c_size_t()
        N.check(fn(v.ctypes.data if v.size else None, v.size, tl, buf, cap, C.byref(size)))
        if size.value <= cap:
            return buf.raw[: size.value]
        cap = size.value
    raise RuntimeError("encoder payload size changed between calls")


def encode_symbols(symbols, table_log: int | None = None) -> bytes:
    """Self-contained FSE payload of a nonnegative integer symbol stream."""
    return _encode(N.lib.hivc_encode_symbols, symbols, table_log)


def encode_signed_values(values, table_log: int | None = None) -> bytes:
    """Category + extra-bits + FSE payload for signed integer streams."""
    return _encode(N.lib.hivc_encode_signed_values, values, table_log)


MAX_MAGNITUDE = (1 << 15) - 1  # entropy.py:26


def to_category(v: int):
    """(category, extra-bits value) of a signed integer, bijective (entropy.py:40-49)."""
    if abs(v) > MAX_MAGNITUDE:
        raise EntropyError(f"magnitude overflow: {v}")
    if v == 0:
        return 0, 0
    k = int(abs(v)).bit_length()
    return (k, v) if v > 0 else (k, v + (1 << k) - 1)


def from_category(category: int, extra: int) -> int:
    """Inverse of to_category (entropy.py:52-60)."""
    if category == 0:
        return 0
    if category > 16:
        raise EntropyError(f"bad category {category}")
    return extra if extra >= 1 << (category - 1) else extra - (1 << category) + 1


def normalize_counts(hist, table_log: int) -> np.ndarray:
    """Histogram -> tANS table counts summing to 2**table_log (entropy.py:68-106), native."""
    h = np.ascontiguousarray(np.asarray(hist, dtype=np.int64).reshape(-1))
    out = np.empty(h.size, dtype=np.int64)
    N.check(N.lib.hivc_normalize_counts(h.ctypes.data if h.size else None, h.size, int(table_log), out.ctypes.data))
    return out
