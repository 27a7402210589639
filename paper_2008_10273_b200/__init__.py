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
