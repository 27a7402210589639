"""The N > 1 paths with the CUDA decode, on the one GPU the pool gives a call.

* bench.py under torchrun with WORLD_SIZE 2, both ranks on cuda:0 over gloo
  (HIVC_BENCH_DEVICE / HIVC_DIST_BACKEND): the GOP shard of each rank is
  decoded by the CUDA path and copied frame by frame into rank 0's CUDA-IPC
  mapped buffer; the bench's own check (`gather_verified`) compares rank 0's
  buffer with every rank's decode.  Timings of such a run mean nothing.
* GOP-range shards decoded with the CUDA path on two processes and gathered
  to rank 0 over gloo reassemble exactly the reference decoder's frames
  (tests/golden/cfg3_*_sums.npz).
The ranks never wait on each other inside a kernel (they only meet at host
barriers), so sharing one GPU cannot deadlock.
"""

import hashlib
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REPO = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def test_bench_two_ranks_gather_verified():
    env = dict(os.environ, HIVC_BENCH_DEVICE="0", HIVC_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(REPO / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1", "--no-cpu"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=str(REPO))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["frames_per_rank"] == 60
    assert d.get("gather_verified") is True, d


def _decode_worker(rank, world, port, out_path):
    sys.path.insert(0, str(REPO))
    import torch
    import torch.distributed as dist

    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.shard import gather_frames, gop_ranges

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    streams = [(REPO / "tests" / "golden" / "streams" / f"cfg3_{p}.hivc").read_bytes() for p in ("Y", "Cb", "Cr")]
    b, e = gop_ranges(codec.stream_info(streams[0]).gop_count, world)[rank]
    outs = [torch.empty(codec.frames_shape(s, b, e), dtype=torch.uint8, device="cuda") for s in streams]
    codec.decode_streams(streams, outs, gop_ranges=[(b, e)] * 3)
    torch.cuda.synchronize()
    local = torch.cat([o.view(-1).cpu() for o in outs])  # gloo gathers host tensors
    full = gather_frames(local, world, rank)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.destroy_process_group()


def test_two_rank_cuda_decode_gather_matches_reference(tmp_path):
    import torch.multiprocessing as mp

    out = tmp_path / "full.npy"
    mp.start_processes(_decode_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True, start_method="spawn")
    full = np.load(out)
    # rank r's block: its GOP range of Y, then Cb, then Cr; ranks in order
    sums = {p: np.load(REPO / "tests" / "golden" / f"cfg3_{p}_sums.npz")["sha256"] for p in ("Y", "Cb", "Cr")}
    shapes = {"Y": (1080, 1920), "Cb": (540, 960), "Cr": (540, 960)}
    pos = 0
    for b, e in [(0, 2), (2, 5)]:
        for p in ("Y", "Cb", "Cr"):
            h, w = shapes[p]
            for i in range(12 * b, 12 * e):
                fr = full[pos : pos + h * w]
                pos += h * w
                assert hashlib.sha256(fr.tobytes()).hexdigest() == sums[p][i], (p, i)
    assert pos == full.size
