"""The C ABI library on the CPU: it loads, exports every symbol the header
declares, and its bit-exact host parser matches the oracle / reference
payloads, including the reference's error classes on corrupt input."""

import struct

import numpy as np
import pytest

from oracle import parse as P
from paper_2008_10273_b200 import _native as N
from paper_2008_10273_b200 import bitstream, entropy, errors
from paper_2008_10273_b200.flow import _tree_leaves


def test_library_exports_every_header_symbol():
    names = N.exported_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(N.lib, name), name
    assert b"sm_100a" in N.lib.hivc_version()


def test_symbols_match_reference_payloads(payloads):
    for key, val in payloads.items():
        if key.endswith("_payload") and key.startswith("sym"):
            out, pos = entropy.decode_symbols(val.tobytes(), 0)
            assert pos == val.size
            assert np.array_equal(out, payloads[key[:-8] + "_in"]), key


def test_signed_values_match_reference_payloads(payloads):
    for key, val in payloads.items():
        if key.endswith("_payload") and key.startswith("sv"):
            out, pos = entropy.decode_signed_values(val.tobytes(), 0)
            assert pos == val.size
            assert np.array_equal(out, payloads[key[:-8] + "_in"]), key


def test_trees_match_reference(payloads):
    i = 0
    while f"tree{i}_bits" in payloads:
        h, w = (int(x) for x in payloads[f"tree{i}_shape"])
        leaves = _tree_leaves(payloads[f"tree{i}_bits"].tobytes(), 0, int(payloads[f"tree{i}_nbits"][0]), w, h)
        assert np.array_equal(leaves, payloads[f"tree{i}_leaves"])
        i += 1


def test_header_and_gops(cfg0_stream):
    h = bitstream.unpack_header(cfg0_stream)
    ref = P.read_container(cfg0_stream)[0]
    for k, v in ref.items():
        assert getattr(h, k) == v
    assert bitstream.gop_frame_counts(cfg0_stream) == [10]


def _walk_records(stream):
    """Yield (kind, payload bytes) of every prediction and residual payload."""
    _, gops = P.read_container(stream)
    for pay in gops:
        (nf,) = struct.unpack_from("<H", pay, 0)
        pos = 2
        for _ in range(nf):
            ftype, plen = struct.unpack_from("<BI", pay, pos)
            pos += 5
            yield ("intra" if ftype == 0 else "flow"), pay[pos : pos + plen]
            pos += plen
            (rlen,) = struct.unpack_from("<I", pay, pos)
            pos += 4
            yield "res", pay[pos : pos + rlen]
            pos += rlen


def test_every_entropy_payload_of_config0_matches_oracle(cfg0_stream):
    n = 0
    for kind, data in _walk_records(cfg0_stream):
        if kind == "intra":
            (nbits,) = struct.unpack_from("<I", data, 0)
            nb = (nbits + 7) // 8
            leaves = _tree_leaves(data, 4, nbits, 320, 180)
            ref = P.tree_leaves(P.Bits(data[4 : 4 + nb], nbits), 320, 180)
            assert np.array_equal(leaves, np.array(ref))
            pos = 4 + nb + 4
            a, p1 = entropy.decode_symbols(data, pos)
            b, p2 = P.decode_symbols(data, pos)
            assert p1 == p2 and np.array_equal(a, b)
            n += 1
        elif kind == "res" and data[0] == 1:
            # skip marker, scales, bitmap, trees -> c and a streams
            ntiles = 40 * 23
            pos = 1 + 8 + (ntiles + 7) // 8
            (tb,) = struct.unpack_from("<I", data, pos)
            pos += 4 + (tb + 7) // 8
            for _ in range(2):
                a, p1 = entropy.decode_signed_values(data, pos)
                b, p2 = P.decode_signed_values(data, pos)
                assert p1 == p2 and np.array_equal(a, b)
                pos = p1
            assert pos == len(data)
            n += 1
    assert n >= 5


@pytest.mark.parametrize("cut", [0, 1, 5, 21, 22, 30, 100, 1000])
def test_truncated_streams_raise_reference_classes(cfg0_stream, cut):
    data = cfg0_stream[:cut]
    with pytest.raises(errors.BitstreamError):
        bitstream.stream_info(data)


def test_header_errors(cfg0_stream):
    with pytest.raises(errors.BadMagic):
        bitstream.stream_info(b"XIVC" + cfg0_stream[4:])
    with pytest.raises(errors.UnsupportedVersion):
        bitstream.stream_info(cfg0_stream[:4] + b"\x02" + cfg0_stream[5:])
    with pytest.raises(errors.LengthMismatch):
        # header promises 11 frames with gop 10 -> 2 groups, stream holds 1
        bitstream.stream_info(cfg0_stream[:9] + struct.pack("<I", 11) + cfg0_stream[13:])


def test_entropy_errors(payloads):
    good = payloads["sym4_payload"].tobytes()
    with pytest.raises(errors.EntropyError):
        entropy.decode_symbols(b"\x04" + good[1:], 0)  # table_log out of range
    with pytest.raises(errors.TruncatedStream):
        entropy.decode_symbols(good[:-3], 0)
    with pytest.raises(errors.TruncatedStream):
        entropy.decode_symbols(b"", 0)
    # corrupting the coded bits must be caught by the final-state check (or a read past the end)
    bad = bytearray(good)
    bad[-1] ^= 0xFF
    bad[-5] ^= 0x5A
    with pytest.raises((errors.EntropyError, errors.TruncatedStream)):
        entropy.decode_symbols(bytes(bad), 0)


def test_byte_flip_fuzz_matches_oracle_error_class(payloads):
    """Same accept/reject decision and exception class as the oracle."""
    rng = np.random.default_rng(7)
    src = payloads["sv3_payload"].tobytes()
    kinds = {"Truncated": errors.TruncatedStream, "EntropyError": errors.EntropyError}
    for _ in range(200):
        b = bytearray(src)
        i = int(rng.integers(len(b)))
        b[i] ^= int(rng.integers(1, 256))
        b = bytes(b)
        try:
            ref, rpos = P.decode_signed_values(b, 0)
            ref_err = None
        except P.OracleError as e:
            ref_err = e.kind
        except ValueError:
            ref_err = "ValueError"
        if ref_err is None:
            out, pos = entropy.decode_signed_values(b, 0)
            assert pos == rpos and np.array_equal(out, ref)
        else:
            with pytest.raises(kinds.get(ref_err, ValueError)):
                entropy.decode_signed_values(b, 0)


def _parse_stream_stats(data):
    """hivc_parse_stream's per-frame stats rows (type, intra points, ...)."""
    import ctypes as C

    cap = 8 * 4096
    stats = (C.c_int64 * cap)()
    nf = C.c_int64()
    secs = C.c_double()
    buf = C.create_string_buffer(data, len(data))
    N.check(N.lib.hivc_parse_stream(buf, len(data), stats, cap, C.byref(nf), C.byref(secs)))
    return np.array(stats[: 8 * nf.value], dtype=np.int64).reshape(-1, 8)


def _first_intra_tree(stream):
    """(offset of the tree's u32 bit count in the stream, nbits) of GOP 0's I-frame."""
    hdr = bitstream.read_stream(stream)
    gop0 = 22 + 4  # header, then the first GOP's u32 length
    off = gop0 + 2 + 5  # frame count, record type + prediction length
    (nbits,) = struct.unpack_from("<I", stream, off)
    return hdr, off, nbits


def test_medium_gray_tree_two_thread_walk_matches_oracle():
    """540p gray I-frames take the two-thread walk (tree subtrees shared with
    the value-decode helper): mask point counts equal the oracle's leaves."""
    from pathlib import Path

    data = (Path(__file__).parent / "golden" / "streams" / "cfg3_Cb.hivc").read_bytes()
    rows = _parse_stream_stats(data)
    _, off, nbits = _first_intra_tree(data)
    nb = (nbits + 7) // 8
    ref = P.tree_leaves(P.Bits(data[off + 4 : off + 4 + nb], nbits), 960, 540)
    assert rows[0, 0] == 0 and rows[0, 1] == len(ref)


@pytest.mark.parametrize("seed", [5, 9, 10, 11])
def test_medium_gray_tree_corruption_matches_oracle_error_class(seed):
    """Corrupt 540p trees (seeds whose flips the oracle rejects) raise the
    oracle's class through the two-thread walk (its failure path reruns the
    sequential walk for the first error in stream order)."""
    from pathlib import Path

    data = bytearray((Path(__file__).parent / "golden" / "streams" / "cfg3_Cb.hivc").read_bytes())
    _, off, nbits = _first_intra_tree(bytes(data))
    nb = (nbits + 7) // 8
    rng = np.random.default_rng(seed)
    for _ in range(3):  # flip bytes inside the tree
        i = off + 4 + int(rng.integers(nb))
        data[i] ^= int(rng.integers(1, 256))
    try:
        P.tree_leaves(P.Bits(bytes(data[off + 4 : off + 4 + nb]), nbits), 960, 540)
        ref_err = None
    except P.OracleError as e:
        ref_err = e.kind
    assert ref_err is not None
    kinds = {"Truncated": errors.TruncatedStream, "SubdivisionError": errors.SubdivisionError}
    with pytest.raises(kinds[ref_err]):
        _parse_stream_stats(bytes(data))


def test_medium_gray_tree_truncated_raises_truncated():
    from pathlib import Path

    data = bytearray((Path(__file__).parent / "golden" / "streams" / "cfg3_Cb.hivc").read_bytes())
    _, off, nbits = _first_intra_tree(bytes(data))
    nb = (nbits + 7) // 8
    tail = bytes(data[off + 4 + nb // 2 : off + 4 + nb])
    data[off + 4 + nb // 2 : off + 4 + nb] = bytes(len(tail))  # the tree's second half all splits? no: zeros = leaves
    for k in range(off + 4 + nb // 2, off + 4 + nb):
        data[k] = 0xFF  # all splits: the tree runs out of bits
    with pytest.raises((errors.TruncatedStream, errors.SubdivisionError)):
        _parse_stream_stats(bytes(data))
