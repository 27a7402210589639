"""Host-side encoder primitives (native C++, no GPU) against the reference's
own outputs (tests/golden/make_encoder.py, make_golden.py): tANS payloads,
subdivision trees, leaf means, flow payloads, residual tile plans."""

import numpy as np
import pytest


def test_encode_symbols_matches_reference_payloads(payloads):
    from paper_2008_10273_b200 import entropy

    names = sorted({k[:-3] for k in payloads if k.endswith("_in") and k.startswith(("sym", "sv"))})
    assert len(names) >= 13
    for k in names:
        tl = int(k[5:]) if k.startswith("symtl") else None
        fn = entropy.encode_signed_values if k.startswith("sv") else entropy.encode_symbols
        assert fn(payloads[k + "_in"], tl) == payloads[k + "_payload"].tobytes(), k


def test_encode_decode_round_trip_and_errors():
    from paper_2008_10273_b200 import entropy
    from paper_2008_10273_b200.errors import EntropyError

    rng = np.random.default_rng(3)
    for n, hi in [(0, 1), (1, 1), (5, 300), (4096, 3), (70000, 40), (3000, 4000)]:
        s = rng.integers(0, hi, n)
        got, pos = entropy.decode_symbols(entropy.encode_symbols(s))
        assert np.array_equal(got, s)
        v = rng.integers(-hi, hi + 1, n)
        b = entropy.encode_signed_values(v)
        got, pos = entropy.decode_signed_values(b)
        assert np.array_equal(got, v) and pos == len(b)
    with pytest.raises(EntropyError):
        entropy.encode_symbols([1, -1])
    with pytest.raises(EntropyError):
        entropy.encode_symbols([0, 1], table_log=4)
    with pytest.raises(EntropyError):
        entropy.encode_signed_values([1 << 15])


def _sub_case(g, i):
    from paper_2008_10273_b200 import subdivision as S

    planes = list(g[f"sub{i}_planes"])
    me = float(g[f"sub{i}_min_error"])
    err = S.joint_ssd_error(planes) if len(planes) > 1 else None
    return S.subdivide_by_error(planes[0], int(g[f"sub{i}_target"]), error_fn=err,
                                min_error=None if np.isnan(me) else me), planes


@pytest.mark.parametrize("i", range(8))
def test_subdivide_by_error_matches_reference(enc_golden, i):
    from paper_2008_10273_b200 import subdivision as S

    tree, planes = _sub_case(enc_golden, i)
    assert np.array_equal(np.array(tree.bits, dtype=np.uint8), enc_golden[f"sub{i}_bits"])
    assert np.array_equal(tree.rects, enc_golden[f"sub{i}_leaves"])
    # float64 means in numpy's association order: bit-identical
    assert np.array_equal(S.leaf_means(tree, planes[0]), enc_golden[f"sub{i}_means"])


def test_subdivision_properties_and_errors():
    from paper_2008_10273_b200 import subdivision as S
    from paper_2008_10273_b200.errors import SubdivisionError

    rng = np.random.default_rng(9)
    p = rng.normal(size=(37, 53))
    t = S.subdivide_by_error(p, 300)
    assert t.leaf_count == 300 and len(t.bits) == 599
    assert S.mask_from_tree(t).sum() == 300
    area = np.zeros(p.shape, dtype=int)  # leaves tile the plane exactly once
    for x, y, w, h in t.leaves():
        area[y : y + h, x : x + w] += 1
    assert (area == 1).all()
    full = S.subdivide_by_error(p, p.size)
    assert full.leaf_count == p.size
    for bad in (0, p.size + 1):
        with pytest.raises(SubdivisionError):
            S.subdivide_by_error(p, bad)


@pytest.mark.parametrize("i", range(4))
def test_compress_flow_matches_reference(enc_golden, i):
    from paper_2008_10273_b200.flow import FlowField, compress_flow

    b, levels = (int(v) for v in enc_golden[f"flow{i}_cfg"])
    f = FlowField(enc_golden[f"flow{i}_u"], enc_golden[f"flow{i}_v"])
    assert compress_flow(f, b, levels) == enc_golden[f"flow{i}_payload"].tobytes()


@pytest.mark.parametrize("i", range(5))
def test_residual_tile_plan_matches_reference(enc_golden, i):
    from paper_2008_10273_b200.encoder import _plan_group

    planes = enc_golden[f"res{i}_planes"]
    pts = int(enc_golden[f"res{i}_cfg"][0])
    for key, group in [("plan", planes[:1])] + ([("plan2", planes[1:])] if len(planes) == 3 else []):
        idx, words, tbits, tnb = _plan_group(list(group), pts)
        assert np.array_equal(idx, enc_golden[f"res{i}_{key}_coded"])
        m = ((words[:, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).astype(bool)
        assert np.array_equal(m, enc_golden[f"res{i}_{key}_masks"])
        bits = np.concatenate([np.unpackbits(tbits[j])[: tnb[j]] for j in range(len(idx))]) if len(idx) else []
        assert np.array_equal(np.asarray(bits, dtype=np.uint8), enc_golden[f"res{i}_{key}_bits"])


def test_stream_header_pack_round_trip(cfg0_stream):
    from paper_2008_10273_b200.bitstream import HEADER_SIZE, read_stream, unpack_header, write_stream

    h, payloads = read_stream(cfg0_stream)
    assert h.pack() == cfg0_stream[:HEADER_SIZE]
    assert write_stream(h, payloads) == cfg0_stream
    assert unpack_header(cfg0_stream) == h
