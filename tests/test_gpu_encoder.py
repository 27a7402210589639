"""Encoder-side kernels beyond the decode path: the
tonal optimisation of the transmitted mask values, against golden vectors
from the reference (tests/golden/make_tonal.py).  Needs a B200."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLD = Path(__file__).resolve().parent / "golden" / "golden_tonal.npz"


@pytest.mark.parametrize("i", range(4))
def test_optimize_mask_values_matches_reference(i):
    from paper_2008_10273_b200.prediction import optimize_mask_values

    g = np.load(GOLD)
    planes, mask, ref = g[f"tonal{i}_planes"], g[f"tonal{i}_mask"], g[f"tonal{i}_out"]
    got = np.stack(optimize_mask_values(list(planes), mask))
    assert got.shape == ref.shape
    # the reference factorises the system (splu); here CG solves to 1e-12: agreement to ~1e-9
    scale = max(1.0, float(np.abs(ref).max()))
    assert np.abs(got - ref).max() <= 1e-6 * scale, np.abs(got - ref).max()


def test_tonal_adjoint_is_the_transpose():
    """<A v, w> == <v, A^T w> for the GPU operator pair (random v, w)."""
    from paper_2008_10273_b200.prediction import _InpaintOperator

    rng = np.random.default_rng(3)
    mask = rng.uniform(size=(40, 50)) < 0.1
    op = _InpaintOperator(mask)
    v = torch.from_numpy(rng.normal(size=int(mask.sum()))).cuda()
    w = torch.from_numpy(rng.normal(size=mask.size)).cuda()
    lhs = float(torch.dot(op.matvec(v), w))
    rhs = float(torch.dot(v, op.rmatvec(w)))
    assert abs(lhs - rhs) <= 1e-9 * max(1.0, abs(lhs))
