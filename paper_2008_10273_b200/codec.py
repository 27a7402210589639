"""Decoder orchestration on the B200 (reference: codec.py).

``decode(data, timings)`` keeps the reference signature (codec.py:484) and
returns the same ``Frame`` list; underneath, ONE native call
(``hivc_decode``, csrc/decode.cu) parses every GOP on host threads and runs
the whole reconstruction on the GPU.  ``decode_frames`` is the zero-copy
variant (uint8 frames into a caller buffer, host or device) that the
benchmark and the multi-GPU sharding use.
"""

from __future__ import annotations

import ctypes as C
import struct
import time

import numpy as np

from paper_2008_10273_b200 import _native as N
from paper_2008_10273_b200._tensors import torch
from paper_2008_10273_b200.bitstream import gop_frame_counts, stream_info
from paper_2008_10273_b200.errors import CodecError, Truncated  # noqa: F401  (re-exports)
from paper_2008_10273_b200.frame import Frame

STAGES = ("intra_solve", "flow_parse", "warp", "residual_parse", "residual_transform", "finalize", "total")
MAX_RESIDUAL_POINTS = 48  # codec.py:65


def frames_shape(data: bytes, gop_begin: int = 0, gop_end: int | None = None):
    """(n_frames, channels, height, width) of the uint8 output for a GOP range."""
    info = stream_info(data)
    counts = gop_frame_counts(data)
    gop_end = info.gop_count if gop_end is None else gop_end
    return (sum(counts[gop_begin:gop_end]), info.channels, info.height, info.width)


def decode_frames(data: bytes, out=None, gop_begin: int = 0, gop_end: int | None = None, timings: dict | None = None,
                  device: int | None = None, ctx=None):
    """Decode GOPs [gop_begin, gop_end) into uint8 frames (n, C, H, W).

    ``out``: a CUDA uint8 tensor (frames stay in HBM), a pinned/CPU uint8
    tensor or numpy array, or None (a pinned host tensor is allocated).
    Returns ``out``.
    """
    data = bytes(data)
    shape = frames_shape(data, gop_begin, gop_end)
    t = torch()
    if out is None:
        out = t.empty(shape, dtype=t.uint8, pin_memory=True)
    if isinstance(out, np.ndarray):
        on_dev = False
        optr = out.ctypes.data
        if out.shape != shape or out.dtype != np.uint8 or not out.flags.c_contiguous:
            raise ValueError(f"out must be contiguous uint8 {shape}")
    else:
        on_dev = bool(out.is_cuda)
        optr = out.data_ptr()
        if tuple(out.shape) != shape or out.dtype != t.uint8 or not out.is_contiguous():
            raise ValueError(f"out must be contiguous uint8 {shape}")
        if on_dev:
            device = out.device.index
    if ctx is None:
        ctx = N.context(device)
    buf = np.frombuffer(data, dtype=np.uint8)
    stage = (C.c_double * 8)()
    gend = -1 if gop_end is None else gop_end
    if on_dev:
        t.cuda.current_stream(out.device).synchronize()
    N.check(N.lib.hivc_decode(ctx.handle, buf.ctypes.data_as(C.c_void_p), len(data), gop_begin, gend, optr,
                              int(on_dev), stage))
    if timings is not None:
        for k, v in zip(STAGES + ("device_span",), stage):
            timings[k] = timings.get(k, 0.0) + float(v)
    return out


def decode_streams(streams, outs, gop_ranges=None, ctx=None, timings: dict | None = None,
                   peer: bool = False) -> float:
    """Decode several streams (e.g. the Y/Cb/Cr gray streams of a 4:2:0 video)
    in ONE native call sharing the decode lanes.  ``outs[k]``: uint8 buffer of
    ``frames_shape(streams[k], *gop_ranges[k])`` (all on the device or all on
    the host).  ``peer=True``: ``outs`` are device addresses (ints) of a peer
    GPU's frame buffer (``shard.PeerFrames``); every frame is copied there over
    NVLink as it completes (``ctx`` required).  Returns the device-side span in
    seconds (CUDA events)."""
    t = torch()
    n = len(streams)
    datas = [np.frombuffer(bytes(s), dtype=np.uint8) for s in streams]
    on_dev = peer or bool(getattr(outs[0], "is_cuda", False))
    if peer and ctx is None:
        raise ValueError("peer output needs the decoding GPU's context")
    if ctx is None:
        ctx = N.context(outs[0].device.index if on_dev else None)
    dptr = (C.c_void_p * n)(*[d.ctypes.data for d in datas])
    lens = (C.c_size_t * n)(*[len(d) for d in datas])
    gb = (C.c_int32 * n)(*[(r[0] if gop_ranges else 0) for r in (gop_ranges or [None] * n)])
    ge = (C.c_int32 * n)(*[(r[1] if gop_ranges and r[1] is not None else -1) for r in (gop_ranges or [None] * n)])
    optr = (C.c_void_p * n)(*[(int(o) if peer else o.data_ptr() if hasattr(o, "data_ptr") else o.ctypes.data)
                              for o in outs])
    stage = (C.c_double * 8)()
    if on_dev and not peer:
        t.cuda.current_stream(outs[0].device).synchronize()
    N.check(N.lib.hivc_decode_multi(ctx.handle, n, dptr, lens, gb, ge, optr, 2 if peer else int(on_dev), stage))
    if timings is not None:
        for k, v in zip(STAGES + ("device_span",), stage):
            timings[k] = timings.get(k, 0.0) + float(v)
    return float(stage[7])


def decode(data: bytes, timings: dict | None = None):
    """Decode a stream into output frames (RGB or gray) (codec.py:484-563)."""
    t0 = time.perf_counter()
    local = {} if timings is not None else None
    frames_u8 = decode_frames(bytes(data), timings=local)
    t1 = time.perf_counter()
    arr = frames_u8.numpy() if hasattr(frames_u8, "numpy") else frames_u8
    cs = "gray" if arr.shape[1] == 1 else "rgb"
    frames = [Frame(tuple(arr[i, c] for c in range(arr.shape[1])), colorspace=cs) for i in range(arr.shape[0])]
    if timings is not None:
        local["finalize"] += time.perf_counter() - t1  # Frame construction (codec.py:552-555)
        local["total"] = time.perf_counter() - t0
        for k, v in local.items():
            timings[k] = timings.get(k, 0.0) + v
    return frames


def _decode_residual(data, pos, shape, channels, levels, timings=None):
    """Residual planes (float64) of one residual payload (codec.py:248-340).

    Parsing goes through the native entropy/tree parser; the block
    transform runs on the GPU (``pseudodiff.reconstruct_blocks``).
    """
    from paper_2008_10273_b200.entropy import decode_signed_values
    from paper_2008_10273_b200.flow import _tree_leaves
    from paper_2008_10273_b200.pseudodiff import block_grid, reconstruct_blocks

    h, w = shape
    tiles = block_grid(h, w)
    nskip = (len(tiles) + 7) // 8
    if pos + 1 > len(data):
        raise Truncated("residual payload truncated")
    marker = data[pos]
    pos += 1
    if marker == 0:
        return [np.zeros((h, w)) for _ in range(channels)], pos
    if marker != 1:
        raise CodecError("bad residual payload marker")
    if pos + 8 > len(data):
        raise Truncated("residual payload truncated")
    c_fp, a_fp = struct.unpack_from("<II", data, pos)
    pos += 8
    if c_fp == 0 or a_fp == 0:
        raise CodecError("zero coefficient scale")
    c_scale, a_scale = c_fp / 65536.0, a_fp / 65536.0
    step = 127.0 / ((levels - 1) // 2)
    planes = []
    nbx, nby = -(-w // 8), -(-h // 8)
    for nplanes in [1] + ([2] if channels == 3 else []):
        if pos + nskip > len(data):
            raise Truncated("residual payload truncated")
        bits = np.unpackbits(np.frombuffer(data, dtype=np.uint8, count=nskip, offset=pos))[: len(tiles)]
        pos += nskip
        coded = np.flatnonzero(bits)
        if pos + 4 > len(data):
            raise Truncated("residual payload truncated")
        (tb,) = struct.unpack_from("<I", data, pos)
        pos += 4
        tnb = (tb + 7) // 8
        if pos + tnb > len(data):
            raise Truncated("residual payload truncated")
        masks = np.zeros((len(coded), 64), dtype=bool)
        # concatenated per-tile trees: parse tile by tile, tracking the bit offset
        bitpos = 0
        for bi, ti in enumerate(coded):
            _, _, bh, bw = tiles[ti]
            leaves, used = _tree_leaves(data, pos, tb, bw, bh, bit_offset=bitpos, with_used=True)
            bitpos += used
            for x, y, lw, lh in leaves.tolist():
                masks[bi, (y + lh // 2) * 8 + (x + lw // 2)] = True
        pos += tnb
        c_sym, pos = decode_signed_values(data, pos)
        a_sym, pos = decode_signed_values(data, pos)
        rows, cols = np.nonzero(masks)
        if c_sym.size != rows.size * nplanes or a_sym.size != len(coded) * nplanes:
            raise CodecError("residual payload inconsistent with block masks")
        c_vals = c_sym.astype(np.float64) * step / 127.0 * c_scale
        a_vals = a_sym.astype(np.float64) * step / 127.0 * a_scale
        mc = np.zeros((nplanes, len(coded), 64))
        for ci in range(nplanes):
            mc[ci, rows, cols] = c_vals[ci * rows.size : (ci + 1) * rows.size]
        rec = (
            reconstruct_blocks(mc.reshape(-1, 8, 8), a_vals).reshape(nplanes, len(coded), 8, 8) if len(coded) else None
        )
        for ci in range(nplanes):
            pad = np.zeros((nby * 8, nbx * 8))
            if rec is not None:
                view = pad.reshape(nby, 8, nbx, 8).transpose(0, 2, 1, 3)
                view[coded // nbx, coded % nbx] = rec[ci]
            planes.append(pad[:h, :w])
    return planes, pos


# the encoder lives in encoder.py; codec.encode & co. keep the reference's import path (codec.py:74-105, 426-471, 604-642)
from paper_2008_10273_b200.encoder import EncoderConfig, encode, encode_target_ratio  # noqa: E402,F401
