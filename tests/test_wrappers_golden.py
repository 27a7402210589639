"""Function-level decoder wrappers against the reference's own outputs.

golden_wrappers.npz (tests/golden/make_wrappers.py) holds, for the frame
records of the reference-encoded cfg0 (gray) and rgb (colour) streams, what
the reference's `prediction.decode_intra` (prediction.py:185-208),
`flow.decompress_flow` (flow.py:368-372) and `codec._decode_residual`
(codec.py:248-340) return on the record's payloads, called as
`codec.decode` calls them (codec.py:491-543).

CPU tests pin the oracle on all three and check the package's host-side
`decompress_flow` (native tree parse + leaf painting); the GPU tests check the
package's decode_intra (CUDA cascadic CG) and _decode_residual (CUDA block
rebuild).
"""

from __future__ import annotations

import struct

import numpy as np
import pytest

from conftest import GOLDEN

STREAMS = ("cfg0", "rgb")


@pytest.fixture(scope="module")
def wg():
    return dict(np.load(GOLDEN / "golden_wrappers.npz"))


def _records(name):
    from oracle.parse import read_container

    data = (GOLDEN / "streams" / f"{name}.hivc").read_bytes()
    hdr, payloads = read_container(data)
    out = {}
    for gi, payload in enumerate(payloads):
        (nframes,) = struct.unpack_from("<H", payload, 0)
        pos = 2
        for fi in range(nframes):
            ftype, pred_len = struct.unpack_from("<BI", payload, pos)
            pos += 5
            pred = payload[pos : pos + pred_len]
            pos += pred_len
            (res_len,) = struct.unpack_from("<I", payload, pos)
            pos += 4
            out[f"{name}_g{gi}_f{fi}"] = (ftype, pred, payload[pos : pos + res_len])
            pos += res_len
    return hdr, out


def _cases(wg, kind):
    return sorted(k[: -len(kind) - 1] for k in wg if k.endswith("_" + kind))


def _hdr(h):
    """(shape, channels, intra, flow, residual levels) from the oracle's header tuple or dict."""
    if isinstance(h, dict):
        return (h["height"], h["width"]), h["channels"], h["intra_levels"], h["flow_levels"], h["residual_levels"]
    return (h.height, h.width), h.channels, h.intra_levels, h.flow_levels, h.residual_levels


def test_golden_covers_every_wrapper(wg):
    assert len(_cases(wg, "intra")) == 3 and len(_cases(wg, "flow")) == 6 and len(_cases(wg, "res")) == 9


# ------------------------------------------------------------------ CPU: oracle pinned, host-side flow decode


@pytest.mark.parametrize("name", STREAMS)
def test_oracle_wrappers_match_reference(wg, name):
    from oracle import decoder, motion

    hdr, recs = _records(name)
    shape, ch, il, fl, rl = _hdr(hdr)
    for key in _cases(wg, "flow"):
        if key.startswith(name + "_"):
            _, pred, _ = recs[key]
            u, v, used = motion.decode_flow(pred, 0, shape, fl)
            assert used == int(wg[key + "_flow_used"])
            assert np.array_equal(np.stack([u, v]), wg[key + "_flow"])
    for key in _cases(wg, "res"):
        if key.startswith(name + "_"):
            _, _, res = recs[key]
            planes, used = decoder.decode_residual(res, 0, shape, ch, rl)
            assert used == int(wg[key + "_res_used"])
            assert np.abs(np.stack(planes) - wg[key + "_res"]).max() <= 1e-9
    for key in _cases(wg, "intra"):
        if key.startswith(name + "_"):
            _, pred, _ = recs[key]
            planes, used = decoder.decode_intra(pred, 0, shape, ch, il)
            assert used == int(wg[key + "_intra_used"])
            assert np.abs(np.stack(planes) - wg[key + "_intra"]).max() <= 1e-9


@pytest.mark.parametrize("name", STREAMS)
def test_decompress_flow_matches_reference(wg, name):
    """Host-side API (native tree parse + native leaf painting): bit-exact."""
    from paper_2008_10273_b200.flow import decompress_flow

    hdr, recs = _records(name)
    shape, _, _, fl, _ = _hdr(hdr)
    keys = [k for k in _cases(wg, "flow") if k.startswith(name + "_")]
    assert keys
    for key in keys:
        _, pred, _ = recs[key]
        flow, used = decompress_flow(pred, 0, shape, fl)
        assert used == int(wg[key + "_flow_used"]) == len(pred)
        assert flow.u.dtype == np.float64 and flow.u.shape == shape
        assert np.array_equal(np.stack([flow.u, flow.v]), wg[key + "_flow"])


# ------------------------------------------------------------------ GPU: the CUDA-backed wrappers


@pytest.mark.gpu
@pytest.mark.parametrize("name", STREAMS)
def test_decode_intra_matches_reference(wg, name):
    from paper_2008_10273_b200.prediction import decode_intra

    hdr, recs = _records(name)
    shape, ch, il, _, _ = _hdr(hdr)
    keys = [k for k in _cases(wg, "intra") if k.startswith(name + "_")]
    assert keys
    for key in keys:
        _, pred, _ = recs[key]
        planes, used = decode_intra(pred, 0, shape, ch, il)
        assert used == int(wg[key + "_intra_used"]) == len(pred)
        got = np.stack([np.asarray(p) for p in planes])
        assert got.shape == wg[key + "_intra"].shape
        # float64 replay of the reference's cascadic CG: same iterations, <= 1e-9 grey
        assert np.abs(got - wg[key + "_intra"]).max() <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("name", STREAMS)
def test_decode_residual_matches_reference(wg, name):
    from paper_2008_10273_b200.codec import _decode_residual

    hdr, recs = _records(name)
    shape, ch, _, _, rl = _hdr(hdr)
    keys = [k for k in _cases(wg, "res") if k.startswith(name + "_")]
    assert keys
    for key in keys:
        _, _, res = recs[key]
        planes, used = _decode_residual(res, 0, shape, ch, rl)
        assert used == int(wg[key + "_res_used"]) == len(res)
        got = np.stack([np.asarray(p) for p in planes])
        # the float64 AAN rebuild replays the reference's operation order: bit-identical
        assert np.array_equal(got, wg[key + "_res"])


@pytest.mark.gpu
def test_decompress_flow_device_paint_matches_reference(wg):
    """The encoder's closed-loop flow decode (leaves painted by one CUDA launch)."""
    import torch

    from paper_2008_10273_b200.flow import _decompress_plane_device

    hdr, recs = _records("cfg0")
    shape, _, _, fl, _ = _hdr(hdr)
    for key in [k for k in _cases(wg, "flow") if k.startswith("cfg0_")]:
        _, pred, _ = recs[key]
        u, pos = _decompress_plane_device(pred, 0, shape, fl, torch.device("cuda:0"))
        v, pos = _decompress_plane_device(pred, pos, shape, fl, torch.device("cuda:0"))
        assert pos == len(pred) and u.is_cuda
        assert np.array_equal(np.stack([u.cpu().numpy(), v.cpu().numpy()]), wg[key + "_flow"])


def test_decompress_flow_error_classes():
    """Corrupt flow payloads raise the reference's classes in its order
    (flow.py:343-356, quantize.py:78-82, subdivision.py:162-170)."""
    from paper_2008_10273_b200 import errors
    from paper_2008_10273_b200.flow import decompress_flow

    hdr, recs = _records("cfg0")
    shape, _, _, fl, _ = _hdr(hdr)
    _, pred, _ = recs["cfg0_g0_f1"]
    with pytest.raises(errors.TruncatedStream):
        decompress_flow(pred[:11], 0, shape, fl)  # no room for lo/hi/nbits
    lo, hi, nbits = struct.unpack_from("<ffI", pred, 0)
    with pytest.raises(errors.TruncatedStream):
        decompress_flow(pred[: 12 + (nbits + 7) // 8 - 1], 0, shape, fl)  # tree cut short
    swapped = struct.pack("<ff", hi, lo) + pred[8:]
    with pytest.raises(errors.QuantizeError):
        decompress_flow(swapped, 0, shape, fl)  # lo >= hi
    # the tree followed by a 3-value symbol block: more leaves than values
    from paper_2008_10273_b200.entropy import encode_symbols

    short = pred[: 12 + (nbits + 7) // 8] + encode_symbols(np.array([1, 2, 3]), table_log=8)
    with pytest.raises(errors.SubdivisionError, match="leaf value count mismatch"):
        decompress_flow(short, 0, shape, fl)
