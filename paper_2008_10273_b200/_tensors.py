"""Host <-> device hand-off: PyTorch is only used for device memory here."""

from __future__ import annotations

import numpy as np


def torch():
    import torch as _t

    return _t


def is_cuda_tensor(x) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor) and x.is_cuda


def to_device(x, dtype, device=None):
    """numpy / CPU tensor / CUDA tensor -> contiguous CUDA tensor of `dtype`."""
    t = torch()
    if isinstance(x, t.Tensor):
        dev = x.device if x.is_cuda else (device if device is not None else t.device("cuda", t.cuda.current_device()))
        return x.to(device=dev, dtype=dtype).contiguous()
    a = np.ascontiguousarray(x)
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    return t.from_numpy(a).to(device=dev, dtype=dtype).contiguous()


def ptr(t) -> int:
    return int(t.data_ptr())


def back(t, like):
    """Return `t` in the caller's convention: numpy in -> numpy out."""
    if is_cuda_tensor(like):
        return t
    return t.cpu().numpy()
