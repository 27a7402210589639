"""Exception classes with the reference's names and bases.

Reference: bitstream.py:37-54, bits.py:6, codec.py:69, entropy.py:31,
subdivision.py:21, homogeneous.py:19-24, flow.py:36, frame.py:15,
quantize.py:16, pseudodiff.py:27.  The C ABI returns a status code per
class (include/hivc_b200.h); ``raise_for`` maps it back.
"""

from __future__ import annotations


class BitstreamError(Exception):
    """Base class for malformed or unreadable streams."""


class BadMagic(BitstreamError):
    pass


class UnsupportedVersion(BitstreamError):
    pass


class Truncated(BitstreamError):
    pass


class LengthMismatch(BitstreamError):
    pass


class CodecError(BitstreamError):
    """Decoding failed on structurally valid but inconsistent payloads."""


class TruncatedStream(ValueError):
    """A reader ran past the end of its buffer."""


class EntropyError(ValueError):
    pass


class SubdivisionError(ValueError):
    pass


class InpaintingError(ValueError):
    pass


class ConvergenceError(RuntimeError):
    """Solver failed to reach the requested tolerance within max_iter."""


class FlowError(ValueError):
    pass


class FrameError(ValueError):
    pass


class QuantizeError(ValueError):
    pass


class PseudodiffError(ValueError):
    pass


class NativeError(RuntimeError):
    """CUDA / library failure (no device, launch error, out of memory)."""


STATUS = {
    1: Truncated,
    2: BadMagic,
    3: UnsupportedVersion,
    4: LengthMismatch,
    5: CodecError,
    6: EntropyError,
    7: SubdivisionError,
    8: InpaintingError,
    9: ConvergenceError,
    10: FlowError,
    11: FrameError,
    12: QuantizeError,
    13: BitstreamError,
    14: PseudodiffError,
    15: TruncatedStream,
    20: ValueError,
    21: NativeError,
    22: MemoryError,
}


def raise_for(status: int, message: str):
    cls = STATUS.get(status, NativeError)
    raise cls(message)
