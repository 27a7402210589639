"""Golden vectors for the decoder's function-level wrappers, from the REFERENCE.

Run here (the container that has /root/reference), never on the GPU box:

    python tests/golden/make_wrappers.py

For every frame record of the committed reference-encoded streams cfg0.hivc
(gray 320x180) and rgb.hivc (colour), the reference's own
`prediction.decode_intra` (prediction.py:185-208), `flow.decompress_flow`
(flow.py:368-372) and `codec._decode_residual` (codec.py:248-340) are run on
the record's payloads exactly as `codec.decode` calls them (codec.py:491-543),
and their outputs and consumed lengths are stored in golden_wrappers.npz.
"""

from __future__ import annotations

import struct
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import hivc.bitstream as rbs  # noqa: E402
import hivc.codec as rcodec  # noqa: E402
import hivc.flow as rflow  # noqa: E402
import hivc.prediction as rpred  # noqa: E402


def records(data: bytes):
    """(gop, frame, ftype, pred_data, res_data) per frame record (codec.py:491-540)."""
    header, payloads = rbs.read_stream(data)
    for gi, payload in enumerate(payloads):
        (nframes,) = struct.unpack_from("<H", payload, 0)
        pos = 2
        for fi in range(nframes):
            ftype, pred_len = struct.unpack_from("<BI", payload, pos)
            pos += 5
            pred = payload[pos : pos + pred_len]
            pos += pred_len
            (res_len,) = struct.unpack_from("<I", payload, pos)
            pos += 4
            res = payload[pos : pos + res_len]
            pos += res_len
            yield header, gi, fi, ftype, pred, res


def main():
    g = {}
    for name in ("cfg0", "rgb"):
        data = (HERE / "streams" / f"{name}.hivc").read_bytes()
        n_intra = n_flow = 0
        for header, gi, fi, ftype, pred, res in records(data):
            shape = (header.height, header.width)
            key = f"{name}_g{gi}_f{fi}"
            if ftype == 0:
                planes, used = rpred.decode_intra(pred, 0, shape, header.channels, header.intra_levels)
                g[f"{key}_intra"] = np.stack(planes)
                g[f"{key}_intra_used"] = np.int64(used)
                n_intra += 1
            elif n_flow < 3:  # three flow records per stream are plenty (the GPU decode pins all of them)
                flow, used = rflow.decompress_flow(pred, 0, shape, header.flow_levels)
                g[f"{key}_flow"] = np.stack([flow.u, flow.v])
                g[f"{key}_flow_used"] = np.int64(used)
                n_flow += 1
            else:
                continue
            res_planes, used = rcodec._decode_residual(res, 0, shape, header.channels, header.residual_levels)
            g[f"{key}_res"] = np.stack(res_planes)
            g[f"{key}_res_used"] = np.int64(used)
        print(name, "intra records", n_intra, "flow records", n_flow)
    np.savez_compressed(HERE / "golden_wrappers.npz", **g)
    print("wrote", HERE / "golden_wrappers.npz", (HERE / "golden_wrappers.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
