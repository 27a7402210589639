"""Edge frame sizes (1x1 up to odd sizes crossing the tile grid and the
solver's level / kernel thresholds; gray, RGB, lossless, Horn-Schunck):
the GPU decoder reproduces the reference decoder's frames and the encoder
reproduces the reference encoder's bytes (tests/golden/make_edge_streams.py)."""

import ast
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

G = np.load(Path(__file__).resolve().parent / "golden" / "golden_edge.npz")
NAMES = [str(n) for n in G["names"]]


@pytest.mark.parametrize("name", NAMES)
def test_edge_decode_matches_reference(name):
    from paper_2008_10273_b200 import codec

    stream = G[f"{name}_stream"].tobytes()
    ref = G[f"{name}_frames"].astype(np.int32)
    got = np.stack([np.stack(f.planes) for f in codec.decode(stream)])
    assert got.shape == ref.shape and np.array_equal(got, ref)
    dev = codec.decode_frames(stream, out=torch.empty(ref.shape, dtype=torch.uint8, device="cuda"))
    if ref.shape[1] == 1:
        assert np.array_equal(dev.cpu().numpy().astype(np.int32), ref)


@pytest.mark.parametrize("name", NAMES)
def test_edge_encode_matches_reference(name):
    from paper_2008_10273_b200 import codec
    from paper_2008_10273_b200.frame import Frame

    src = G[f"{name}_src"].astype(np.int32)
    kw = ast.literal_eval(str(G[f"{name}_cfg"]))  # encoder settings written by make_edge_streams.py
    cs = "rgb" if src.shape[1] == 3 else "gray"
    frames = [Frame(tuple(f), colorspace=cs) for f in src]
    assert codec.encode(frames, codec.EncoderConfig(**kw)) == G[f"{name}_stream"].tobytes()
