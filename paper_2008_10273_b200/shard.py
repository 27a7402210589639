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


def gather_payloads(payloads, world: int, rank: int, dst: int = 0):
    """Gather every rank's list of byte strings on `dst`, in rank order
    (one flat uint8 gather of [u32 count, (u32 len, bytes)...] records)."""
    import numpy as np
    import torch

    rec = bytearray(struct.pack("<I", len(payloads)))
    for p in payloads:
        rec += struct.pack("<I", len(p)) + p
    local = torch.from_numpy(np.frombuffer(bytes(rec), dtype=np.uint8).copy())
    if world > 1:
        import torch.distributed as dist

        if dist.get_backend() == "nccl":  # NCCL moves device buffers only
            local = local.cuda()
    full = gather_frames(local, world, rank, dst) if world > 1 else local
    if full is None:
        return None
    data = full.cpu().numpy().tobytes()
    out, pos = [], 0
    while pos < len(data):  # one record per rank
        (n,) = struct.unpack_from("<I", data, pos)
        pos += 4
        for _ in range(n):
            (ln,) = struct.unpack_from("<I", data, pos)
            out.append(data[pos + 4 : pos + 4 + ln])
            pos += 4 + ln
    return out


def encode_sharded(frames, cfg=None, world: int = 1, rank: int = 0, _flows=None, encode_gops=None):
    """codec.encode across ranks: rank r encodes GOPs [r*G/P, (r+1)*G/P)
    (flows estimated on its own GPU), the GOP payloads (kB each) are gathered
    to rank 0, which writes the container.  Returns
    the stream on rank 0 (identical to a single-process encode), None elsewhere.
    ``encode_gops`` defaults to ``encoder.encode_gops`` (override for tests)."""
    from paper_2008_10273_b200 import encoder

    enc = encode_gops or encoder.encode_gops
    cfg = cfg or encoder.EncoderConfig()
    header = encoder.stream_header(frames, cfg)
    n_gops = -(-len(frames) // cfg.gop_size)
    b, e = gop_ranges(n_gops, world)[rank]
    payloads = enc(frames, cfg, b, e, _flows)[0] if e > b else []
    allp = gather_payloads(payloads, world, rank)
    if allp is None:
        return None
    from paper_2008_10273_b200.bitstream import write_stream

    return write_stream(header, allp)


class PeerFrames:
    """The job's decoded-frame buffer on rank ``owner``'s GPU, mapped into every
    rank's address space through CUDA IPC (``hivc_peer_alloc`` / ``hivc_peer_open``).

    Ranks decode with ``codec.decode_streams(..., peer=True)`` into their slice:
    each finished frame is copied device-to-device over NVLink by the decoder's
    copy streams while later frames decode, so the gather to rank 0 is fused
    into the decode instead of following it (an NCCL gather of 186 MB per rank
    and step would serialise after the last frame).  The handle travels over
    ``torch.distributed`` (any backend); one process per GPU.
    """

    def __init__(self, nbytes: int, world: int, rank: int, device: int, owner: int = 0):
        import ctypes as C

        import torch.distributed as dist

        from paper_2008_10273_b200 import _native as N

        self.nbytes, self.rank, self.owner, self.device = int(nbytes), rank, owner, device
        self._N = N
        self.ptr = C.c_void_p()
        handle = (C.c_uint8 * 64)()
        ok = True
        if rank == owner:
            ok = N.lib.hivc_peer_alloc(device, self.nbytes, C.byref(self.ptr), handle) == 0
        box = [bytes(handle) if rank == owner and ok else None]
        if world > 1:
            dist.broadcast_object_list(box, src=owner)  # every rank takes part, even on failure
        if box[0] is None:
            raise RuntimeError("peer frame buffer allocation failed on the owner rank")
        if rank != owner:
            h = (C.c_uint8 * 64).from_buffer_copy(box[0])
            N.check(N.lib.hivc_peer_open(device, h, C.byref(self.ptr)))

    @property
    def base(self) -> int:
        return int(self.ptr.value)

    def to_host(self, offset: int = 0, nbytes: int | None = None):
        """Copy (part of) the buffer into a numpy uint8 array (synchronous)."""
        import numpy as np

        n = self.nbytes - offset if nbytes is None else nbytes
        out = np.empty(n, dtype=np.uint8)
        self._N.check(self._N.lib.hivc_memcpy(out.ctypes.data, self.base + offset, n))
        return out

    def close(self):
        if self.ptr.value:
            if self.rank == self.owner:
                self._N.check(self._N.lib.hivc_peer_free(self.ptr))
            else:
                self._N.check(self._N.lib.hivc_peer_close(self.ptr))
            self.ptr.value = None
