"""Decode the config-3 streams once (device output) — for ncu captures."""

import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

from paper_2008_10273_b200 import codec  # noqa: E402


def main():
    planes = sys.argv[1:] or ["Y"]
    for p in planes:
        data = (REPO / "tests/golden/streams" / f"cfg3_{p}.hivc").read_bytes()
        out = torch.empty(codec.frames_shape(data), dtype=torch.uint8, device="cuda")
        codec.decode_frames(data, out=out)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
