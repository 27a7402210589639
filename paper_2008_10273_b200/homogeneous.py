"""Homogeneous diffusion inpainting on the B200 (reference: homogeneous.py).

``solve_homogeneous`` keeps the reference signature (homogeneous.py:157-164)
and replays its cascadic coarse-to-fine CG on the GPU in float64 through
``hivc_homog_solve`` (csrc/inpaint.cu): same pyramid, prolongation, initial
guesses, per-level tolerances, denominators and stopping rules, so the
per-level iteration counts in ``stats["level_iterations"]`` match the
reference's.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2008_10273_b200 import _native as N
from paper_2008_10273_b200._tensors import back, is_cuda_tensor, ptr, to_device, torch
from paper_2008_10273_b200.errors import ConvergenceError, InpaintingError  # noqa: F401  (re-export)

COARSEST_SIZE = 16  # homogeneous.py:15
LEVEL_TOL = 1e-4  # homogeneous.py:16


def solve_homogeneous(f, mask, tol: float = 1e-6, max_iter: int = 10000, strict: bool = True, stats: dict | None = None):
    """Cascadic CG solve of homogeneous diffusion inpainting (homogeneous.py:157-212).

    ``f``/``mask`` may be numpy arrays (result returned as float64 numpy) or
    CUDA tensors (result stays on the device).
    """
    if tuple(f.shape) != tuple(mask.shape) or len(f.shape) != 2:
        raise InpaintingError("plane/mask shape mismatch")
    if not is_cuda_tensor(mask) and not np.asarray(mask).any():
        raise InpaintingError("empty inpainting mask")
    if strict and tol <= 0:
        raise InpaintingError("tol must be positive")
    t = torch()
    ft = to_device(f, t.float64)
    mt = to_device(mask, t.bool).to(t.uint8)
    h, w = ft.shape
    u = t.empty_like(ft)
    ctx = N.context(ft.device.index)
    sizes = (C.c_int32 * 32)()
    iters = (C.c_int32 * 32)()
    nlev = C.c_int32()
    # the C side works on the context's stream: order it after torch's copies
    t.cuda.current_stream(ft.device).synchronize()
    status = N.lib.hivc_homog_solve(
        ctx.handle, ptr(ft), ptr(mt), h, w, float(tol), int(max_iter), int(bool(strict)), ptr(u), sizes, iters,
        C.byref(nlev),
    )
    if stats is not None and status in (0, 9):
        stats["level_iterations"] = [(int(sizes[i]), int(iters[i])) for i in range(nlev.value)]
    N.check(status)
    return back(u, f)
