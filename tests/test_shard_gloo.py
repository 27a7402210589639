"""N>1 host logic on the CPU: GOP-range sharding + the rank-0 frame gather,
world_size 2 over gloo.  Each rank decodes its GOP range with the oracle (the
CUDA decode needs a B200); rank 0 must reassemble exactly the full decode."""

import os
import struct
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parent.parent


def _one_gop_stream(data: bytes, gops, g):
    pay = gops[g]
    (nf,) = struct.unpack_from("<H", pay, 0)
    head = bytearray(data[:22])
    struct.pack_into("<I", head, 9, nf)
    return bytes(head) + struct.pack("<I", len(pay)) + pay


def _worker(rank, world, port, data, out_path):
    sys.path.insert(0, str(REPO))
    import torch
    import torch.distributed as dist

    from oracle import decoder, parse
    from paper_2008_10273_b200.shard import gather_frames, gop_ranges

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, gops = parse.read_container(data)
    b, e = gop_ranges(len(gops), world)[rank]
    frames = []
    for g in range(b, e):
        frames += [f[0].astype(np.uint8) for f in decoder.decode_stream(_one_gop_stream(data, gops, g))]
    local = torch.from_numpy(np.stack(frames).reshape(-1)) if frames else torch.zeros(0, dtype=torch.uint8)
    full = gather_frames(local, world, rank)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.destroy_process_group()


def test_gop_ranges_partition():
    from paper_2008_10273_b200.shard import gop_ranges

    for n in (1, 5, 40):
        for p in (1, 2, 4, 8):
            r = gop_ranges(n, p)
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [e - b for b, e in r]
            assert max(sizes) - min(sizes) <= 1


def test_tile_stream_is_a_valid_container(cfg0_stream):
    from oracle import parse
    from paper_2008_10273_b200.shard import tile_stream

    t = tile_stream(cfg0_stream, 3)
    hdr, gops = parse.read_container(t)
    assert hdr["frame_count"] == 30 and len(gops) == 3


def test_two_rank_gop_shard_and_gather(tmp_path, cfg0_stream):
    from oracle import decoder
    from paper_2008_10273_b200.shard import tile_stream

    data = tile_stream(cfg0_stream, 3)  # 3 GOPs -> ranks get 1 and 2 GOPs
    out = tmp_path / "full.npy"
    port = 29500 + (os.getpid() % 1000)
    mp.start_processes(_worker, args=(2, port, data, str(out)), nprocs=2, join=True, start_method="spawn")
    full = np.load(out)
    ref = np.stack([f[0].astype(np.uint8) for f in decoder.decode_stream(data)]).reshape(-1)
    assert np.array_equal(full, ref)


if __name__ == "__main__":  # pragma: no cover
    pytest.main([__file__, "-q"])


def _enc_worker(rank, world, port, data, out_path):
    sys.path.insert(0, str(REPO))
    import torch.distributed as dist

    from oracle import parse
    from paper_2008_10273_b200 import encoder
    from paper_2008_10273_b200.frame import Frame
    from paper_2008_10273_b200.shard import encode_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hdr, gops = parse.read_container(data)
    frames = [Frame((np.zeros((hdr["height"], hdr["width"]), np.int32),), colorspace="gray")
              for _ in range(hdr["frame_count"])]
    cfg = encoder.EncoderConfig(gop_size=hdr["gop_size"], intra_mask_fraction=0.04)
    seen = []

    def stub(frames_, cfg_, b, e, flows_):  # the per-GOP encoder needs a GPU: replay the stream's payloads
        seen.append((b, e))
        return [gops[g] for g in range(b, e)], None

    out = encode_sharded(frames, cfg, world, rank, encode_gops=stub)
    assert len(seen) == 1
    if rank == 0:
        Path(out_path).write_bytes(out)
    else:
        assert out is None
    dist.destroy_process_group()


def test_two_rank_sharded_encode_container(tmp_path, cfg0_stream):
    """Rank-0 assembly of GOP payloads encoded on two ranks equals the single-process stream."""
    from paper_2008_10273_b200.shard import tile_stream

    data = tile_stream(cfg0_stream, 3)
    out = tmp_path / "stream.hivc"
    port = 30500 + (os.getpid() % 1000)
    mp.start_processes(_enc_worker, args=(2, port, data, str(out)), nprocs=2, join=True, start_method="spawn")
    assert out.read_bytes() == data
