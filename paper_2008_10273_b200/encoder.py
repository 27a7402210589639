"""Encoder orchestration on the B200 (reference: codec.py:74-475, 576-642).

``encode(frames, cfg, _flows)`` produces the reference encoder's stream byte
for byte (tests/test_gpu_encoder.py pins it against streams made by the
reference).  Heavy steps run natively:

* Brox flow between source frames: GPU (``flow.flow_brox``, csrc/brox.cu);
* intra mask subdivision, tANS coding, residual tile planning: C++
  (csrc/encode.cpp), numpy's float64 summation order replayed exactly;
* tonal optimisation of the intra mask values: GPU LSQR over CG solves
  (``prediction.optimize_mask_values``);
* closed loop: the decoder's own GPU kernels rebuild every frame
  (``prediction.decode_intra``, ``flow.decompress_flow`` +
  ``prediction.predict_inter``, ``codec._decode_residual``);
* residual block fits and the keep-decision rebuilds: GPU
  (``pseudodiff.solve_blocks_any_k``, ``pseudodiff.reconstruct_blocks``).

GOPs are independent (``prev`` resets per GOP): ``encode`` runs them on a
small thread pool so the host-side steps of one GOP overlap the GPU work of
another.
"""

from __future__ import annotations

import ctypes as C
import struct
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, replace

import numpy as np

from paper_2008_10273_b200 import _native as N
from paper_2008_10273_b200.bitstream import StreamHeader, write_stream
from paper_2008_10273_b200.errors import CodecError, FrameError
from paper_2008_10273_b200.frame import Frame, clip_plane, rct_forward, rct_inverse

MAX_RESIDUAL_POINTS = 48  # codec.py:65
_SCALE_FP = 65536.0  # codec.py:66


@dataclass(frozen=True)
class EncoderConfig:  # codec.py:74-105
    gop_size: int = 16
    intra_mask_fraction: float = 0.09
    residual_points: int = 4
    flow_points: int = 100
    intra_levels: int = 256
    flow_levels: int = 256
    residual_levels: int = 63
    residual_lambda: float = 1.0
    fps_num: int = 25
    fps_den: int = 1
    flow_method: str = "brox"
    self_check: bool = False

    def __post_init__(self):
        if not 0.0 < self.intra_mask_fraction <= 1.0:
            raise ValueError("intra_mask_fraction must lie in (0, 1]")
        if not 1 <= self.residual_points <= MAX_RESIDUAL_POINTS:
            raise ValueError(f"residual_points must lie in [1, {MAX_RESIDUAL_POINTS}]")
        if self.flow_points < 1:
            raise ValueError("flow_points must be >= 1")
        if self.flow_method not in ("brox", "horn-schunck"):
            raise ValueError(f"unknown flow method {self.flow_method!r}")
        if self.gop_size < 1 or self.gop_size > 255:
            raise ValueError("gop_size must lie in [1, 255]")
        if self.residual_lambda < 0.0:
            raise ValueError("residual_lambda must be >= 0")


# per-stage wall time of the last encode(timings=...) call (probe / bench instrumentation)
_stage_times: dict | None = None


class _stage:
    def __init__(self, key: str):
        self.key = key

    def __enter__(self):
        self.t = time.perf_counter()

    def __exit__(self, *exc):
        if _stage_times is not None:
            _stage_times[self.key] = _stage_times.get(self.key, 0.0) + time.perf_counter() - self.t


# ----------------------------------------------------------------------------- residual coding


def _plan_group(gplanes, points: int):
    """codec._plan_group (codec.py:118-137) in C++: coded tiles, their 8x8 mask words and tree bits."""
    h, w = gplanes[0].shape
    arrs = [np.ascontiguousarray(p, dtype=np.int64) for p in gplanes]
    nt = ((h + 7) // 8) * ((w + 7) // 8)
    coded = np.empty(nt, dtype=np.uint8)
    masks = np.empty(nt, dtype=np.uint64)
    tbits = np.empty((nt, 16), dtype=np.uint8)
    tnb = np.empty(nt, dtype=np.uint8)
    pp = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    N.check(N.lib.hivc_plan_residual_tiles(pp, len(arrs), h, w, points, 0, coded.ctypes.data, masks.ctypes.data,
                                           tbits.ctypes.data, tnb.ctypes.data))
    idx = np.flatnonzero(coded)
    return idx, masks[idx], tbits[idx], tnb[idx]


def _tile_blocks(arrs, idx) -> np.ndarray:
    """Tiles `idx` of int64 planes embedded top-left into zero-padded 8x8 blocks,
    (nplanes, n, 64) float64 (codec._tile_residuals, codec.py:108-115), in C++."""
    h, w = arrs[0].shape
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty((len(arrs), idx.size, 64))
    pp = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    N.check(N.lib.hivc_gather_tiles(pp, len(arrs), h, w, idx.ctypes.data if idx.size else None, idx.size,
                                    out.ctypes.data))
    return out


def _encode_residual(planes, points: int, levels: int, lam: float = 0.0) -> bytes:
    """Serialise integer residual planes, Y alone and U,V jointly (codec.py:156-245)."""
    return _encode_residual_rec(planes, points, levels, lam)[0]


def _encode_residual_rec(planes, points: int, levels: int, lam: float = 0.0):
    """``_encode_residual`` plus the residual planes the decoder will rebuild from
    the payload.  Per channel group: tile plans and tile gather in C++; the
    bordered-system fits, the dead-zone quantisation, the rebuilds and the
    keep decision on the GPU (``hivc_block_fit``, ``hivc_residual_keep``); the
    frame's coefficient scales (99.9th percentiles over every group and plane)
    on the host.  The kept blocks' rebuilds are exactly the decoder's residual
    (same dequantisation expression, same per-block transform), so the closed
    loop needs no second parse (codec._decode_residual stays the self-check)."""
    from paper_2008_10273_b200._tensors import ptr, torch
    from paper_2008_10273_b200.entropy import encode_signed_values
    from paper_2008_10273_b200.pseudodiff import solve_blocks_any_k
    from paper_2008_10273_b200.quantize import coefficient_scale, deadzone_step

    t = torch()
    dev = t.device("cuda", t.cuda.current_device())
    h, w = planes[0].shape
    nby, nbx = (h + 7) // 8, (w + 7) // 8
    ntiles = nby * nbx
    groups = [[planes[0]]] + ([[planes[1], planes[2]]] if len(planes) == 3 else [])
    deadzone_step(levels)  # validates the level count (QuantizeError)
    plans, all_c, all_a = [], [], []
    for gplanes in groups:
        arrs = [np.ascontiguousarray(p, dtype=np.int64) for p in gplanes]
        with _stage("res_plan"):
            idx, words, tbits, tnb = _plan_group(arrs, points)
        n = idx.size
        bitmask = ((words[:, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).astype(bool)  # (n, 64)
        fits = []
        with _stage("res_fit"):
            fb = t.from_numpy(_tile_blocks(arrs, idx)).to(dev) if n else None  # (npl, n, 64)
            wd = t.from_numpy(words.view(np.int64)).to(dev) if n else None
            for ci in range(len(arrs)):
                if n:
                    c_sc, a = solve_blocks_any_k(fb[ci].view(n, 8, 8), words)  # GPU bordered-system fits
                    c_sc = c_sc.view(n, 64)
                    fits.append((c_sc, a))
                    all_c.append(c_sc.cpu().numpy()[bitmask])  # block by block, raster mask order
                    all_a.append(a.cpu().numpy())
        plans.append((idx, words, bitmask, tbits, tnb, fits, fb, wd, len(arrs)))

    c_flat = np.concatenate(all_c) if all_c else np.zeros(0)
    a_flat = np.concatenate(all_a) if all_a else np.zeros(0)
    c_scale = coefficient_scale(c_flat) if c_flat.size else 1.0
    a_scale = coefficient_scale(a_flat) if a_flat.size else 1.0
    c_fp = min(int(round(c_scale * _SCALE_FP)), 0xFFFFFFFF) or 1
    a_fp = min(int(round(a_scale * _SCALE_FP)), 0xFFFFFFFF) or 1
    c_scale, a_scale = c_fp / _SCALE_FP, a_fp / _SCALE_FP
    bits_per_sym = max(1, int(np.ceil(np.log2(levels))))
    ctx = N.context(dev.index)

    kept_total = 0
    out = bytearray(struct.pack("<II", c_fp, a_fp))
    rec_planes = []
    for idx, words, bitmask, tbits, tnb, fits, fb, wd, npl in plans:
        n = idx.size
        keep = np.zeros(0, dtype=np.int64)
        q = qa = rec = None
        if n:
            q = t.empty((npl, n, 64), dtype=t.int32, device=dev)
            qa = t.empty((npl, n), dtype=t.int32, device=dev)
            rec = t.empty((npl, n, 64), dtype=t.float64, device=dev)
            kp = t.empty(n, dtype=t.uint8, device=dev)
            arr = lambda xs: (C.c_void_p * npl)(*[ptr(x) for x in xs])  # noqa: E731
            with _stage("res_keep_rebuild"):
                t.cuda.current_stream(dev).synchronize()
                N.check(N.lib.hivc_residual_keep(ctx.handle, npl, arr([f[0] for f in fits]), arr([f[1] for f in fits]),
                                                 arr([fb[ci] for ci in range(npl)]), ptr(wd), n, levels, bits_per_sym,
                                                 c_scale, a_scale, float(lam), arr([q[ci] for ci in range(npl)]),
                                                 arr([qa[ci] for ci in range(npl)]),
                                                 arr([rec[ci] for ci in range(npl)]), ptr(kp)))
                keep = np.flatnonzero(kp.cpu().numpy())
        kept_total += keep.size
        # decoded residual planes: kept blocks' rebuilds placed on the tile grid (GPU scatter)
        for ci in range(npl):
            full = t.zeros((ntiles, 64), dtype=t.float64, device=dev)
            if keep.size:
                kd = t.from_numpy(keep).to(dev)
                full[t.from_numpy(idx[keep]).to(dev)] = rec[ci].index_select(0, kd)
            rec_planes.append(full.view(nby, nbx, 8, 8).permute(0, 2, 1, 3).reshape(nby * 8, nbx * 8)[:h, :w]
                              .cpu().numpy())
        coded_bits = np.zeros(ntiles, dtype=np.uint8)
        coded_bits[idx[keep]] = 1
        out += np.packbits(coded_bits).tobytes()
        tb = np.unpackbits(tbits[keep], axis=1)[np.arange(128)[None, :] < tnb[keep, None].astype(np.int64)]
        out += struct.pack("<I", int(tb.size))
        out += np.packbits(tb).tobytes()
        # plane-major: every kept block's coefficients of plane 0, then plane 1 (codec.py:232-241)
        c_sym, a_sym = [], []
        if keep.size:
            kd = t.from_numpy(keep).to(dev)
            qk = q.index_select(1, kd).cpu().numpy()  # (npl, nk, 64)
            qak = qa.index_select(1, kd).cpu().numpy()
            mk = bitmask[keep]
            for ci in range(npl):
                c_sym.append(qk[ci][mk].astype(np.int64))
                a_sym.append(qak[ci].astype(np.int64))
        with _stage("res_entropy"):
            out += encode_signed_values(np.concatenate(c_sym) if c_sym else np.zeros(0, np.int64))
            out += encode_signed_values(np.concatenate(a_sym) if a_sym else np.zeros(0, np.int64))
    if kept_total == 0:
        return b"\x00", [np.zeros((h, w)) for _ in planes]  # nothing survived quantisation anywhere
    return b"\x01" + bytes(out), rec_planes


# ----------------------------------------------------------------------------- frame and group coding


def _reconstruct(pred_int, res_planes, colorspace):
    return [clip_plane(p + r, ci, colorspace) for ci, (p, r) in enumerate(zip(pred_int, res_planes))]


def _code_frame(planes, pred_planes, cfg: EncoderConfig, colorspace: str):
    """Residual-code one frame against its prediction, closed loop (codec.py:355-366)."""
    from paper_2008_10273_b200.codec import _decode_residual

    pred_int = [np.rint(np.asarray(p)).astype(np.int64) for p in pred_planes]
    residual = [np.asarray(o, dtype=np.int64) - p for o, p in zip(planes, pred_int)]
    with _stage("residual_encode"):
        payload, res_dec = _encode_residual_rec(residual, cfg.residual_points, cfg.residual_levels,
                                                cfg.residual_lambda)
    if cfg.self_check:  # the reference's decode of its own payload (codec.py:362-365)
        with _stage("residual_decode"):
            res_chk, consumed = _decode_residual(payload, 0, planes[0].shape, len(planes), cfg.residual_levels)
        if consumed != len(payload) or any(not np.array_equal(a, b) for a, b in zip(res_chk, res_dec)):
            raise CodecError("residual payload does not decode to the encoder's reconstruction")
    return payload, _reconstruct(pred_int, res_dec, colorspace)


def _estimate_flow(y_t, y_prev, method: str):
    from paper_2008_10273_b200.flow import BroxParams, flow_brox, flow_horn_schunck

    if method == "horn-schunck":
        return flow_horn_schunck(y_t, y_prev)
    return flow_brox(y_t, y_prev, BroxParams())


def _encode_gop(frames_planes, cfg: EncoderConfig, colorspace: str, flows_raw):
    """One group: I-frame, then P-frames against the previous reconstruction (codec.py:375-400)."""
    from paper_2008_10273_b200._tensors import torch
    from paper_2008_10273_b200.flow import FlowField, _decompress_plane_device, compress_flow
    from paper_2008_10273_b200.prediction import decode_intra, encode_intra, predict_inter

    h, w = frames_planes[0][0].shape
    luma_budget = max(1, int(round(cfg.intra_mask_fraction * h * w)))
    out = bytearray(struct.pack("<H", len(frames_planes)))
    recons = []
    for i, planes in enumerate(frames_planes):
        if i == 0:
            with _stage("intra_encode"):
                pred_payload = encode_intra(planes, luma_budget, cfg.intra_levels)
            with _stage("intra_decode"):
                pred, consumed = decode_intra(pred_payload, 0, (h, w), len(planes), cfg.intra_levels)
            ftype = 0
        else:
            with _stage("flow_compress"):
                pred_payload = compress_flow(flows_raw[i - 1], cfg.flow_points, cfg.flow_levels)
            with _stage("inter_predict"):
                # decompress_flow + predict_inter with the dense flow painted and warped on the device
                dev = torch().device("cuda", torch().cuda.current_device())
                u, pos = _decompress_plane_device(pred_payload, 0, (h, w), cfg.flow_levels, dev)
                v, consumed = _decompress_plane_device(pred_payload, pos, (h, w), cfg.flow_levels, dev)
                prev = [torch().from_numpy(np.ascontiguousarray(p)).to(dev).double() for p in recons[-1]]
                pred = [q.cpu().numpy() for q in predict_inter(prev, FlowField(u, v))]
            ftype = 1
        if consumed != len(pred_payload):
            raise CodecError("prediction payload not consumed exactly")
        res_payload, recon = _code_frame(planes, pred, cfg, colorspace)
        recons.append(recon)
        out += struct.pack("<BI", ftype, len(pred_payload))
        out += pred_payload
        out += struct.pack("<I", len(res_payload))
        out += res_payload
    return bytes(out), recons


def _split_gops(n: int, gop_size: int):
    return [(s, min(s + gop_size, n)) for s in range(0, n, gop_size)]


def _to_yuv_planes(frame: Frame):
    if frame.colorspace == "rgb":
        frame = rct_forward(frame)
    return [p.astype(np.int64) for p in frame.planes]


def _compute_gop_flows(y_planes, cfg: EncoderConfig):
    """Flow fields between consecutive source frames, one list per group (codec.py:413-423)."""
    return [[_estimate_flow(y_planes[i], y_planes[i - 1], cfg.flow_method) for i in range(s + 1, e)]
            for s, e in _split_gops(len(y_planes), cfg.gop_size)]


def _finalize_frame(recon_planes, channels: int) -> Frame:
    if channels == 1:
        return Frame((recon_planes[0],), colorspace="gray")
    rgb = rct_inverse(Frame(tuple(recon_planes), colorspace="yuv"))
    return Frame(tuple(np.clip(p, 0, 255).astype(np.int32) for p in rgb.planes), colorspace="rgb")


def encode(frames, cfg: EncoderConfig | None = None, _flows=None, workers: int = 2, timings: dict | None = None) -> bytes:
    """Compress a frame sequence into a self-contained byte stream (codec.py:426-471).

    ``timings`` (optional dict) receives per-stage wall seconds (GOPs run
    sequentially when it is given, so the stages add up)."""
    global _stage_times
    from paper_2008_10273_b200.codec import decode

    if timings is not None:
        _stage_times, workers = timings, 1
    try:
        return _encode(frames, cfg, _flows, workers, decode)
    finally:
        _stage_times = None


def _check_frames(frames, cfg):
    cfg = cfg or EncoderConfig()
    if not frames:
        raise FrameError("nothing to encode")
    first = frames[0]
    if any(f.width != first.width or f.height != first.height or f.channels != first.channels for f in frames):
        raise FrameError("all frames must share geometry and channel count")
    if first.colorspace not in ("rgb", "gray"):
        raise FrameError(f"unsupported input colorspace {first.colorspace!r}")
    return cfg, first


def stream_header(frames, cfg: EncoderConfig | None = None) -> StreamHeader:
    """The container header ``encode`` writes for these frames (codec.py:442-453)."""
    cfg, first = _check_frames(frames, cfg)
    return StreamHeader(first.width, first.height, len(frames), cfg.fps_num, cfg.fps_den, cfg.gop_size,
                        first.channels, cfg.intra_levels, cfg.flow_levels, cfg.residual_levels)


def encode_gops(frames, cfg: EncoderConfig | None = None, gop_begin: int = 0, gop_end: int | None = None,
                _flows=None, workers: int = 2):
    """GOP payloads [gop_begin, gop_end) of ``encode(frames, cfg)`` and their
    reconstructions: GOPs are independent (codec.py:459-462), so ranks (or
    threads) encode disjoint ranges.  ``_flows``: all GOPs' flow lists, or
    None to estimate each GOP's flows inside its job (codec.py:413-423)."""
    cfg, first = _check_frames(frames, cfg)
    colorspace = "yuv" if first.channels == 3 else "gray"
    spans = _split_gops(len(frames), cfg.gop_size)
    gop_end = len(spans) if gop_end is None else gop_end

    def one(gi):
        s, e = spans[gi]
        yuv = [_to_yuv_planes(f) for f in frames[s:e]]
        if _flows is None:
            with _stage("flow_estimate"):
                y = [p[0].astype(np.float64) for p in yuv]
                flows = [_estimate_flow(y[i], y[i - 1], cfg.flow_method) for i in range(1, len(y))]
        else:
            flows = _flows[gi]
        return _encode_gop(yuv, cfg, colorspace, flows)

    gis = range(gop_begin, gop_end)
    if workers > 1 and len(gis) > 1:
        with ThreadPoolExecutor(max_workers=min(workers, len(gis))) as ex:
            results = list(ex.map(one, gis))
    else:
        results = [one(gi) for gi in gis]
    return [r[0] for r in results], [r[1] for r in results]


def _encode(frames, cfg, _flows, workers, decode):
    cfg, first = _check_frames(frames, cfg)
    header = stream_header(frames, cfg)
    payloads, recons = encode_gops(frames, cfg, 0, None, _flows, workers)
    stream = write_stream(header, payloads)
    if cfg.self_check:
        recons = [rc for r in recons for rc in r]
        for i, frame in enumerate(decode(stream)):
            if frame != _finalize_frame(recons[i], first.channels):
                raise CodecError(f"self-check failed at frame {i}")
    return stream


# ----------------------------------------------------------------------------- rate control


def _scaled_config(cfg: EncoderConfig, m: float, pixels: int) -> EncoderConfig:
    """Budgets scaled by the multiplier m (codec.py:576-601)."""
    frac = min(1.0, max(cfg.intra_mask_fraction * m**0.15, 1.0 / pixels))
    pts = min(MAX_RESIDUAL_POINTS, max(1, int(round(cfg.residual_points * m))))
    fpts = max(1, int(round(cfg.flow_points * m**1.5)))
    lam = cfg.residual_lambda / m**6
    lv, ilv = cfg.residual_levels, cfg.intra_levels
    if m < 1.0:
        lv = max(3, int(round(cfg.residual_levels * m)) | 1)
        ilv = max(16, int(round(cfg.intra_levels * m**0.5)))
    return replace(cfg, intra_mask_fraction=frac, residual_points=pts, flow_points=fpts, intra_levels=ilv,
                   residual_levels=lv, residual_lambda=lam)


def encode_target_ratio(frames, cfg: EncoderConfig, target_ratio: float, tol=0.03, max_iter=14):
    """Bisect a budget multiplier until raw/stream bytes hits the target (codec.py:604-642).
    Returns (stream, achieved ratio, config used)."""
    if target_ratio <= 1.0:
        raise ValueError("target ratio must exceed 1")
    first = frames[0]
    raw = len(frames) * first.width * first.height * first.channels
    pixels = first.width * first.height
    flows = _compute_gop_flows([_to_yuv_planes(f)[0].astype(np.float64) for f in frames], cfg)

    def run(m):
        stream = encode(frames, _scaled_config(cfg, m, pixels), _flows=flows)
        return stream, raw / len(stream)

    lo = hi = None
    m = 1.0
    stream, ratio = run(m)
    best = (stream, ratio, m)
    for _ in range(max_iter):
        if abs(ratio - target_ratio) / target_ratio <= tol:
            break
        if ratio > target_ratio:
            lo = m
            m = m * 2 if hi is None else (lo * hi) ** 0.5
        else:
            hi = m
            m = m / 2 if lo is None else (lo * hi) ** 0.5
        stream, ratio = run(m)
        if abs(ratio - target_ratio) < abs(best[1] - target_ratio):
            best = (stream, ratio, m)
    else:
        stream, ratio, m = best
    return stream, ratio, _scaled_config(cfg, m, pixels)
