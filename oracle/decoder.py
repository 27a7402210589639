"""Oracle: whole-stream decode (TEST INFRASTRUCTURE ONLY).

Restates reference ``codec.py:248-340`` (residual payload),
``prediction.py:133-208`` (intra payload) and ``codec.py:484-563`` (GOP /
frame loop, rint + clip finalisation, ``frame.py:118-124``).  Gray
streams return uint8 planes; colour streams return the RCT-inverted RGB
planes as int32 (``codec.py:474-481``, ``frame.py:84-93``).
"""

from __future__ import annotations

import struct

import numpy as np

from oracle import blocks, inpaint, motion
from oracle.parse import (
    Bits,
    CodecErr,
    Truncated,
    decode_signed_values,
    decode_symbols,
    deadzone_unmap,
    read_container,
    tree_mask,
    uniform_dequant,
)

INTRA_ITERS = 160  # prediction.py:35
INTRA_TOL = 1e-4  # prediction.py:36


def _intra_mask(data: bytes, pos: int, w: int, h: int):
    if pos + 4 > len(data):
        raise Truncated("intra payload truncated")
    (nbits,) = struct.unpack_from("<I", data, pos)
    pos += 4
    nb = (nbits + 7) // 8
    if pos + nb > len(data):
        raise Truncated("intra payload truncated")
    return tree_mask(Bits(data[pos : pos + nb], nbits), w, h), pos + nb


def _intra_values(data: bytes, pos: int, levels: int):
    if pos + 4 > len(data):
        raise Truncated("intra payload truncated")
    lo, hi = struct.unpack_from("<hh", data, pos)
    idx, pos = decode_symbols(data, pos + 4)
    return uniform_dequant(idx, float(lo), float(hi), levels), pos


def intra_planes_input(data: bytes, pos: int, shape, channels: int, levels: int):
    """Parse an intra payload into [(mask, f)] solver inputs (``prediction.py:185-208``)."""
    h, w = shape
    my, pos = _intra_mask(data, pos, w, h)
    vy, pos = _intra_values(data, pos, levels)
    jobs = [(my, vy)]
    if channels == 3:
        mc, pos = _intra_mask(data, pos, w, h)
        for _ in range(2):
            vc, pos = _intra_values(data, pos, 2 * levels - 1)
            jobs.append((mc, vc))
    out = []
    for m, vals in jobs:
        f = np.zeros(m.shape)
        f.ravel()[np.flatnonzero(m.ravel())] = vals
        out.append((m, f))
    return out, pos


def decode_intra(data: bytes, pos: int, shape, channels: int, levels: int):
    jobs, pos = intra_planes_input(data, pos, shape, channels, levels)
    planes = [inpaint.solve(f, m, tol=INTRA_TOL, max_iter=INTRA_ITERS, strict=False) for m, f in jobs]
    return planes, pos


def residual_blocks(data: bytes, pos: int, shape, channels: int, levels: int):
    """Parse a residual payload into per-group (coded tiles, masks, mc, a).

    Returns (groups, pos) with groups = [] for the all-zero marker.
    """
    h, w = shape
    tiles = blocks.tile_grid(h, w)
    nskip = (len(tiles) + 7) // 8
    if pos + 1 > len(data):
        raise Truncated("residual payload truncated")
    marker = data[pos]
    pos += 1
    if marker == 0:
        return None, pos
    if marker != 1:
        raise CodecErr("bad residual payload marker")
    if pos + 8 > len(data):
        raise Truncated("residual payload truncated")
    c_fp, a_fp = struct.unpack_from("<II", data, pos)
    pos += 8
    if c_fp == 0 or a_fp == 0:
        raise CodecErr("zero coefficient scale")
    cs, as_ = c_fp / 65536.0, a_fp / 65536.0
    groups = []
    for npl in [1] + ([2] if channels == 3 else []):
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
        rd = Bits(data[pos : pos + tnb], tb)
        pos += tnb
        masks = np.zeros((len(coded), 8, 8), dtype=bool)
        for bi, ti in enumerate(coded):
            _, _, bh, bw = tiles[ti]
            masks[bi, :bh, :bw] = tree_mask(rd, bw, bh)
        csym, pos = decode_signed_values(data, pos)
        asym, pos = decode_signed_values(data, pos)
        rr, cc = np.nonzero(masks.reshape(len(coded), 64))
        if csym.size != rr.size * npl or asym.size != len(coded) * npl:
            raise CodecErr("residual payload inconsistent with block masks")
        cv = deadzone_unmap(csym, levels, cs)
        av = deadzone_unmap(asym, levels, as_)
        mc = np.zeros((npl, len(coded), 64))
        for ci in range(npl):
            mc[ci, rr, cc] = cv[ci * rr.size : (ci + 1) * rr.size]
        groups.append((npl, coded, masks, mc.reshape(npl * len(coded), 8, 8), av))
    return groups, pos


def decode_residual(data: bytes, pos: int, shape, channels: int, levels: int):
    """Residual planes (float64) — reference ``codec.py:248-340``."""
    h, w = shape
    groups, pos = residual_blocks(data, pos, shape, channels, levels)
    if groups is None:
        return [np.zeros((h, w)) for _ in range(channels)], pos
    nbx, nby = -(-w // 8), -(-h // 8)
    planes = []
    for npl, coded, _masks, mc, av in groups:
        rec = blocks.reconstruct(mc, av).reshape(npl, len(coded), 8, 8) if len(coded) else None
        for ci in range(npl):
            pad = np.zeros((nby * 8, nbx * 8))
            if rec is not None:
                view = pad.reshape(nby, 8, nbx, 8).transpose(0, 2, 1, 3)
                view[coded // nbx, coded % nbx] = rec[ci]
            planes.append(pad[:h, :w])
    return planes, pos


def _clip_range(ci: int, channels: int):
    return (-255, 255) if (channels == 3 and ci > 0) else (0, 255)


def decode_stream(data: bytes, record=None):
    """Decode every frame; returns list of per-frame plane lists (int32).

    ``record`` (optional dict) collects per-frame float predictions and
    residuals for teacher-forced stage checks.
    """
    hdr, gops = read_container(data)
    ch = hdr["channels"]
    shape = (hdr["height"], hdr["width"])
    frames = []
    for gi, pay in enumerate(gops):
        if len(pay) < 2:
            raise Truncated("group payload too small")
        (nfr,) = struct.unpack_from("<H", pay, 0)
        pos = 2
        prev = None
        for _ in range(nfr):
            if pos + 5 > len(pay):
                raise Truncated("frame record cut short")
            ftype, plen = struct.unpack_from("<BI", pay, pos)
            pos += 5
            if ftype not in (0, 1):
                raise CodecErr("unknown frame type")
            if pos + plen > len(pay):
                raise Truncated("prediction payload cut short")
            pdata = pay[pos : pos + plen]
            pos += plen
            if ftype == 0:
                pred, used = decode_intra(pdata, 0, shape, ch, hdr["intra_levels"])
            else:
                if prev is None:
                    raise CodecErr("group starts with an inter frame")
                u, v, used = motion.decode_flow(pdata, 0, shape, hdr["flow_levels"])
                pred = motion.warp([p.astype(np.float64) for p in prev], u, v)
            if used != plen:
                raise CodecErr("prediction payload length mismatch")
            if pos + 4 > len(pay):
                raise Truncated("frame record cut short")
            (rlen,) = struct.unpack_from("<I", pay, pos)
            pos += 4
            if pos + rlen > len(pay):
                raise Truncated("residual payload cut short")
            res, used = decode_residual(pay[pos : pos + rlen], 0, shape, ch, hdr["residual_levels"])
            if used != rlen:
                raise CodecErr("residual payload length mismatch")
            pos += rlen
            recon = []
            for ci, (p, r) in enumerate(zip(pred, res)):
                lo, hi = _clip_range(ci, ch)
                recon.append(np.clip(np.rint(np.rint(p).astype(np.int64) + r), lo, hi).astype(np.int32))
            if record is not None:
                record.setdefault("pred", []).append(pred)
                record.setdefault("res", []).append(res)
            prev = recon
            frames.append(_finalize(recon, ch))
        if pos != len(pay):
            raise CodecErr("trailing bytes in group")
    if len(frames) != hdr["frame_count"]:
        raise CodecErr("frame count mismatch")
    return frames


def _finalize(recon, channels):
    if channels == 1:
        return recon
    y, u, v = (p.astype(np.int64) for p in recon)
    g = y - ((u + v) >> 2)
    return [np.clip(p, 0, 255).astype(np.int32) for p in (v + g, g, u + g)]
