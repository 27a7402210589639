"""4:2:0 video as three gray HIVC streams.

The reference codec is 4:4:4 (RCT) or gray; 4:2:0 material is carried as
three independent gray streams — Y at full resolution, Cb and Cr at half
resolution — exactly how the benchmark streams are built.  The encoder
estimates flow on luma only and gives the chroma streams the luma flow
2x2-averaged and halved (config 4's recipe); the decoder runs all three
streams in one native call (`codec.decode_streams`), sharing the GPU's decode
lanes.  `pack` / `unpack` hold the three streams in one byte string
(`HV42`, then three u32-length-prefixed HIVC streams).
"""

from __future__ import annotations

import struct

import numpy as np

from paper_2008_10273_b200.errors import BitstreamError, FrameError, Truncated

MAGIC = b"HV42"


def half_plane(a) -> np.ndarray:
    """2x2 mean with edge replication on odd sizes: (H, W) -> (ceil(H/2), ceil(W/2))."""
    a = np.asarray(a, dtype=np.float64)
    h, w = a.shape
    p = np.pad(a, ((0, h & 1), (0, w & 1)), mode="edge")
    return 0.25 * (p[0::2, 0::2] + p[1::2, 0::2] + p[0::2, 1::2] + p[1::2, 1::2])


def chroma_flow(flow):
    """Luma flow -> chroma-plane flow: 2x2-averaged and halved (displacements in chroma pixels)."""
    from paper_2008_10273_b200.flow import FlowField

    return FlowField(half_plane(np.asarray(flow.u)) * 0.5, half_plane(np.asarray(flow.v)) * 0.5)


def _gray_frames(planes):
    from paper_2008_10273_b200.frame import Frame

    return [Frame((np.asarray(p, dtype=np.int32),), colorspace="gray") for p in planes]


def encode_420(y, cb, cr, cfg=None, luma_flows=None, brox_params=None, workers: int = 2):
    """Encode (n, H, W) Y and (n, ceil(H/2), ceil(W/2)) Cb / Cr integer planes.

    ``luma_flows``: per-GOP lists of luma FlowFields (as ``codec.encode``'s
    ``_flows``) or None to estimate them (Brox with ``brox_params`` on luma,
    or Horn-Schunck when ``cfg.flow_method`` says so).  Returns the three
    streams (bytes)."""
    from paper_2008_10273_b200.encoder import EncoderConfig, _split_gops, encode
    from paper_2008_10273_b200.flow import flow_brox, flow_horn_schunck

    cfg = cfg or EncoderConfig()
    y, cb, cr = (np.asarray(a) for a in (y, cb, cr))
    if y.ndim != 3 or len(y) == 0:
        raise FrameError("expected a non-empty (n, H, W) luma stack")
    n, h, w = y.shape
    if cb.shape != (n, (h + 1) // 2, (w + 1) // 2) or cr.shape != cb.shape:
        raise FrameError("chroma planes must be (n, ceil(H/2), ceil(W/2))")
    if luma_flows is None:
        yf = y.astype(np.float64)
        est = (lambda a, b: flow_horn_schunck(a, b)) if cfg.flow_method == "horn-schunck" else (
            lambda a, b: flow_brox(a, b, brox_params))
        luma_flows = [[est(yf[i], yf[i - 1]) for i in range(s + 1, e)] for s, e in _split_gops(n, cfg.gop_size)]
    cflows = [[chroma_flow(f) for f in g] for g in luma_flows]
    return (encode(_gray_frames(y), cfg, _flows=luma_flows, workers=workers),
            encode(_gray_frames(cb), cfg, _flows=cflows, workers=workers),
            encode(_gray_frames(cr), cfg, _flows=cflows, workers=workers))


def decode_420(streams, device: str | None = None):
    """Decode the three streams in one native call -> (Y, Cb, Cr) uint8 stacks
    (torch CUDA tensors when ``device`` is given, else numpy)."""
    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200._tensors import torch

    t = torch()
    if len(streams) != 3:
        raise BitstreamError("a 4:2:0 video is three streams (Y, Cb, Cr)")
    shapes = [codec.frames_shape(s) for s in streams]
    if any(sh[1] != 1 for sh in shapes) or len({sh[0] for sh in shapes}) != 1:
        raise BitstreamError("4:2:0 streams must be gray and hold the same number of frames")
    if device is not None:
        outs = [t.empty(sh, dtype=t.uint8, device=device) for sh in shapes]
    else:
        outs = [t.empty(sh, dtype=t.uint8).pin_memory() for sh in shapes]
    codec.decode_streams(list(streams), outs)
    res = [o[:, 0] for o in outs]
    return tuple(res) if device is not None else tuple(r.numpy() for r in res)


def pack(streams) -> bytes:
    """One byte string holding the Y, Cb, Cr streams."""
    if len(streams) != 3:
        raise BitstreamError("a 4:2:0 video is three streams (Y, Cb, Cr)")
    return MAGIC + b"".join(struct.pack("<I", len(s)) + bytes(s) for s in streams)


def unpack(data: bytes):
    data = bytes(data)
    if data[:4] != MAGIC:
        raise BitstreamError("not a 4:2:0 HIVC container")
    out, pos = [], 4
    for _ in range(3):
        if pos + 4 > len(data):
            raise Truncated("4:2:0 container cut short")
        (n,) = struct.unpack_from("<I", data, pos)
        if pos + 4 + n > len(data):
            raise Truncated("4:2:0 container cut short")
        out.append(data[pos + 4 : pos + 4 + n])
        pos += 4 + n
    if pos != len(data):
        raise BitstreamError("trailing bytes after the three streams")
    return tuple(out)
