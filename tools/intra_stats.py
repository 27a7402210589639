"""Per-level CG iteration counts + GPU solve times of the config-3 I-frames."""

import struct
import sys
import time
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

from oracle import decoder, parse  # noqa: E402
from paper_2008_10273_b200 import homogeneous  # noqa: E402


def main():
    for plane in ("Y", "Cb"):
        data = (REPO / "tests/golden/streams" / f"cfg3_{plane}.hivc").read_bytes()
        hdr, gops = parse.read_container(data)
        shape = (hdr["height"], hdr["width"])
        for g, pay in enumerate(gops[:2]):
            ftype, plen = struct.unpack_from("<BI", pay, 2)
            jobs, _ = decoder.intra_planes_input(pay[7 : 7 + plen], 0, shape, 1, hdr["intra_levels"])
            m, f = jobs[0]
            ft, mt = torch.from_numpy(f).cuda(), torch.from_numpy(m).cuda()
            st = {}
            homogeneous.solve_homogeneous(ft, mt, tol=1e-4, max_iter=160, strict=False, stats=st)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                homogeneous.solve_homogeneous(ft, mt, tol=1e-4, max_iter=160, strict=False)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 5
            print(f"{plane} gop{g}: mask {m.mean():.4f}, {dt * 1e3:.2f} ms, iters {st['level_iterations']}", flush=True)


if __name__ == "__main__":
    main()
