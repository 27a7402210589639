"""ctypes binding of libhivc_b200.so (include/hivc_b200.h).

There is no fallback: if the library is missing the import fails loudly,
and every compute call needs a CUDA device (the C side checks for sm_100).
The host-only parse entry points work without a GPU.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from paper_2008_10273_b200.errors import raise_for

LIB_PATH = Path(__file__).resolve().parent / "libhivc_b200.so"
if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2008_10273_b200.build` "
        "(there is no CPU fallback for the HIVC CUDA path)"
    )
lib = C.CDLL(str(LIB_PATH))

c_int_p = C.POINTER(C.c_int32)
c_size_p = C.POINTER(C.c_size_t)
c_u64_p = C.POINTER(C.c_uint64)
c_i64_p = C.POINTER(C.c_int64)
c_dbl_p = C.POINTER(C.c_double)


class StreamInfo(C.Structure):
    _fields_ = [
        (name, C.c_int32)
        for name in (
            "width", "height", "frame_count", "fps_num", "fps_den", "gop_size", "channels",
            "intra_levels", "flow_levels", "residual_levels", "gop_count",
        )
    ]


def _proto(name, restype, *argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = list(argtypes)
    return fn


_proto("hivc_last_error", C.c_char_p)
_proto("hivc_version", C.c_char_p)
_proto("hivc_ctx_create", C.c_int, C.c_int, C.POINTER(C.c_void_p))
_proto("hivc_ctx_destroy", C.c_int, C.c_void_p)
_proto("hivc_ctx_stream", C.c_void_p, C.c_void_p)
_proto("hivc_ctx_synchronize", C.c_int, C.c_void_p)
_proto("hivc_ctx_launch_count", C.c_int64, C.c_void_p)
_proto("hivc_parse_header", C.c_int, C.c_void_p, C.c_size_t, C.POINTER(StreamInfo))
_proto("hivc_gop_frame_counts", C.c_int, C.c_void_p, C.c_size_t, c_int_p, C.c_int32, c_int_p)
_proto("hivc_parse_stream", C.c_int, C.c_void_p, C.c_size_t, c_i64_p, C.c_int64, c_i64_p, c_dbl_p)
_proto("hivc_parse_symbols", C.c_int, C.c_void_p, C.c_size_t, C.c_size_t, c_i64_p, C.c_size_t, c_size_p, c_size_p)
_proto("hivc_parse_signed_values", C.c_int, C.c_void_p, C.c_size_t, C.c_size_t, c_i64_p, C.c_size_t, c_size_p, c_size_p)
_proto("hivc_parse_tree", C.c_int, C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, c_int_p,
       C.c_size_t, c_size_p, c_u64_p)
_proto("hivc_homog_solve", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_int32,
       C.c_int32, C.c_void_p, c_int_p, c_int_p, c_int_p)
_proto("hivc_poisson_interior", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_double,
       C.c_int32, C.c_void_p, c_int_p)
_proto("hivc_mask_adjoint", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
       C.c_void_p)
_proto("hivc_flow_component", C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_int32, C.c_int32,
       C.c_int32, C.c_void_p, c_size_p)
_proto("hivc_warp", C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
       C.c_int32, C.POINTER(C.c_void_p))
_proto("hivc_block_reconstruct", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p)
_proto("hivc_block_fit", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p)
_proto("hivc_decode", C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
       c_dbl_p)
_proto("hivc_decode_multi", C.c_int, C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), c_size_p, c_int_p, c_int_p,
       C.POINTER(C.c_void_p), C.c_int32, c_dbl_p)
_proto("hivc_peer_alloc", C.c_int, C.c_int32, C.c_size_t, C.POINTER(C.c_void_p), C.c_void_p)
_proto("hivc_peer_open", C.c_int, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p))
_proto("hivc_peer_close", C.c_int, C.c_void_p)
_proto("hivc_peer_free", C.c_int, C.c_void_p)
_proto("hivc_memcpy", C.c_int, C.c_void_p, C.c_void_p, C.c_size_t)
_proto("hivc_ctx_bytes", C.c_int, C.c_void_p, c_i64_p, c_i64_p)
_proto("hivc_encode_symbols", C.c_int, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p, C.c_size_t, c_size_p)
_proto("hivc_normalize_counts", C.c_int, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)
_proto("hivc_encode_signed_values", C.c_int, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p, C.c_size_t, c_size_p)
_proto("hivc_subdivide", C.c_int, C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
       C.c_double, C.c_void_p, c_u64_p, C.c_void_p, c_size_p)
_proto("hivc_region_means", C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p)
_proto("hivc_gather_tiles", C.c_int, C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t,
       C.c_void_p)
_proto("hivc_residual_keep", C.c_int, C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
       C.POINTER(C.c_void_p), C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
       C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p)
_proto("hivc_plan_residual_tiles", C.c_int, C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
       C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
_proto("hivc_horn_schunck", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_double,
       C.c_int32, C.c_void_p, C.c_void_p)
_proto("hivc_block_operator", C.c_int, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p)
_proto("hivc_block_perblock", C.c_int, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p)


class BroxParamsC(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("gamma", C.c_double), ("pyramid_scale", C.c_double),
        ("min_size", C.c_int32), ("warps", C.c_int32), ("fixed_point_iters", C.c_int32), ("solver_iters", C.c_int32),
        ("eps", C.c_double), ("presmooth_sigma", C.c_double),
    ]


_proto("hivc_brox", C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(BroxParamsC),
       c_dbl_p, C.c_int32, c_dbl_p, C.c_int32, C.c_void_p, C.c_void_p)
_proto("hivc_ctx_set_stage_timing", C.c_int, C.c_void_p, C.c_int32)
_proto("hivc_ctx_decode_stats", C.c_int, C.c_void_p, c_dbl_p, C.c_int32)


def check(status: int):
    if status != 0:
        raise_for(status, lib.hivc_last_error().decode(errors="replace"))


_tls = threading.local()


class Context:
    """One device + CUDA stream + scratch (hivc_ctx)."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        check(lib.hivc_ctx_create(device, C.byref(h)))
        self.handle = h

    @property
    def stream(self) -> int:
        return lib.hivc_ctx_stream(self.handle) or 0

    def synchronize(self):
        check(lib.hivc_ctx_synchronize(self.handle))

    @property
    def launches(self) -> int:
        return int(lib.hivc_ctx_launch_count(self.handle))

    def close(self):
        if self.handle:
            lib.hivc_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def context(device: int | None = None) -> Context:
    """Per-thread context (the reference may call solves from a thread pool)."""
    if device is None:
        import torch

        device = torch.cuda.current_device()
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def exported_symbols():
    """Function names declared in include/hivc_b200.h."""
    import re

    hdr = (Path(__file__).resolve().parent.parent / "include" / "hivc_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(hivc_\w+)\s*\(", hdr, flags=re.M)))
