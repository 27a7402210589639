"""The fused multi-GPU gather's mechanics on one GPU: two processes (one per
"rank", both on cuda:0 — they never wait on each other's kernels, only on a
host barrier), rank 0 exports its frame buffer through CUDA IPC, rank 1 maps it
and decodes its GOP range with per-frame device-to-device copies into its slice
(out_on_device = 2); rank 0 decodes the other range the same way.  The buffer
must equal a single-process decode of the whole stream."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
REPO = Path(__file__).resolve().parent.parent


def _worker(rank, world, port, data, out_path):
    sys.path.insert(0, str(REPO))
    import torch
    import torch.distributed as dist

    from paper_2008_10273_b200 import _native as N
    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.shard import PeerFrames, gop_ranges

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    info = codec.stream_info(data)
    n, c, h, w = codec.frames_shape(data)
    frame_bytes = c * h * w
    pf = PeerFrames(n * frame_bytes, world, rank, 0)
    g0, g1 = gop_ranges(info.gop_count, world)[rank]
    first = codec.frames_shape(data, 0, g0)[0] if g0 > 0 else 0
    ctx = N.Context(0)
    codec.decode_streams([data], [pf.base + first * frame_bytes], gop_ranges=[(g0, g1)], ctx=ctx, peer=True)
    dist.barrier()
    if rank == 0:
        np.save(out_path, pf.to_host())
    dist.barrier()
    pf.close()
    dist.destroy_process_group()


def test_peer_frames_two_processes(tmp_path, cfg0_stream):
    import torch.multiprocessing as mp

    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.shard import tile_stream

    data = tile_stream(cfg0_stream, 3)  # 3 GOPs: rank 0 gets 1, rank 1 gets 2
    out = tmp_path / "buf.npy"
    port = 31500 + (os.getpid() % 1000)
    mp.start_processes(_worker, args=(2, port, data, str(out)), nprocs=2, join=True, start_method="spawn")
    ref = codec.decode_frames(data).numpy().reshape(-1)
    assert np.array_equal(np.load(out), ref)


def test_staged_device_output_equals_direct():
    """out_on_device = 2 into a local buffer: same frames as the direct device write."""
    from paper_2008_10273_b200 import _native as N
    from paper_2008_10273_b200 import codec

    data = (REPO / "tests" / "golden" / "streams" / "rgb.hivc").read_bytes()
    shape = codec.frames_shape(data)
    direct = torch.empty(shape, dtype=torch.uint8, device="cuda")
    codec.decode_streams([data], [direct])
    staged = torch.zeros(shape, dtype=torch.uint8, device="cuda")
    codec.decode_streams([data], [staged.data_ptr()], ctx=N.context(0), peer=True)
    assert torch.equal(direct, staged)
