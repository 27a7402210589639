"""GOP sharding across GPUs (one process per GPU) and the decoded-frame gather.

GOP records are length-prefixed and self-contained and ``prev`` resets per GOP
(reference bitstream.py:124-154, codec.py:491-496), so contiguous GOP ranges
decode independently on each rank with no data-path collective.  The only
exchange is gathering the decoded frames on rank 0 (NCCL over NVLink on the
GPU box; gloo in the CPU tests).
"""

from __future__ import annotations

import struct


def gop_ranges(n_gops: int, world: int):
    """Contiguous GOP ranges [r*G/P, (r+1)*G/P) per rank."""
    return [((r * n_gops) // world, ((r + 1) * n_gops) // world) for r in range(world)]


def tile_stream(data: bytes, times: int) -> bytes:
    """The stream's GOP sequence repeated `times` times; a valid container
    whose header frame count is scaled to match (bitstream.py:57-99)."""
    if times == 1:
        return bytes(data)
    hdr = bytearray(data[:22])
    (fc,) = struct.unpack_from("<I", hdr, 9)
    struct.pack_into("<I", hdr, 9, fc * times)
    return bytes(hdr) + bytes(data[22:]) * times


def gather_frames(local, world: int, rank: int, dst: int = 0):
    """Gather every rank's flat uint8 frame buffer on `dst`, in rank order.

    ``local``: 1-D uint8 torch tensor (any length; lengths may differ per
    rank).  Returns the concatenation on `dst`, None elsewhere.
    """
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    n = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes)
    buf = local
    if local.numel() < cap:
        buf = torch.zeros(cap, dtype=local.dtype, device=local.device)
        buf[: local.numel()].copy_(local)
    parts = [torch.empty(cap, dtype=local.dtype, device=local.device) for _ in range(world)] if rank == dst else None
    dist.gather(buf, parts, dst=dst)
    if rank != dst:
        return None
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])
