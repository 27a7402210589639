"""tANS / category payload decoding through the native parser (reference: entropy.py).

``decode_symbols`` (entropy.py:276-291) and ``decode_signed_values``
(entropy.py:311-338) keep their signatures and run the bit-exact C++
parser of libhivc_b200 (csrc/parse.cpp) — host code, no GPU needed.
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
