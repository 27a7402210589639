"""B200-native HIVC per-frame reconstruction path (arXiv 2008.10273).

Module layout mirrors the reference package ``hivc`` for the hot path:
``codec.decode``, ``homogeneous.solve_homogeneous``, ``flow.warp_planes`` /
``bilinear_warp`` / ``decompress_flow``, ``prediction.decode_intra`` /
``predict_inter``, ``pseudodiff.reconstruct_blocks`` /
``solve_block_coefficients_batch``, ``entropy.decode_symbols`` /
``decode_signed_values``, ``bitstream.read_stream``.  All of them call
``libhivc_b200.so`` (C ABI: include/hivc_b200.h) — sm_100a CUDA kernels
plus a bit-exact C++ parser.  Submodules are imported lazily so that
``synth`` and ``build`` work without the native library.
"""

import os as _os

# A decode keeps ~3 CUDA streams per (stream, GOP) item in flight; with the
# default 8 hardware work queues, a copy or kernel waiting on one item's event
# blocks unrelated items that share its queue (measured on config 3: chroma
# frame copies completing 6 ms after their kernels).  32 queues remove those
# false dependencies.  Effective only if set before the process creates its
# CUDA context (importing this package before using CUDA is enough); an
# explicit user setting wins.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

__all__ = [
    "bitstream",
    "codec",
    "entropy",
    "errors",
    "flow",
    "frame",
    "homogeneous",
    "prediction",
    "pseudodiff",
]
