"""Config-2a shared-layout block operator, a few launches — for ncu captures."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2008_10273_b200.pseudodiff import reconstruct_plane_shared_mask  # noqa: E402


def main():
    rng = np.random.default_rng(2)
    res = torch.from_numpy(rng.laplace(0.0, 8.0, (1080, 1920)).astype(np.float32)).cuda()
    for _ in range(3):
        reconstruct_plane_shared_mask(res)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
