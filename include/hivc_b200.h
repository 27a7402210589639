/*
 * hivc_b200.h — C ABI of the B200-native HIVC per-frame reconstruction path.
 *
 * The reference (arXiv 2008.10273, package `hivc`, /root/reference/pkg/src/hivc)
 * is pure Python/numpy and has no FFI of its own; these entry points are the
 * functions its Python signatures bind to (see INTEGRATION.md for the ctypes
 * stubs).  Each declaration names the reference interface it replaces.
 *
 * Conventions
 *  - Every function returns an int status (HIVC_OK == 0).  On failure a
 *    thread-local message is available from hivc_last_error(); the status
 *    code names the reference exception class to raise.
 *  - "device" pointers are CUDA device addresses (e.g. torch.cuda tensors'
 *    data_ptr()); "host" pointers are ordinary CPU memory.
 *  - Floating-point planes are row-major float64 (the reference computes in
 *    float64); masks are uint8 0/1; decoded frames are uint8.
 *  - No torch types cross this boundary.
 */
#ifndef HIVC_B200_H
#define HIVC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
enum hivc_status {
    HIVC_OK = 0,
    HIVC_E_TRUNCATED = 1,          /* bitstream.Truncated           (bitstream.py:49) */
    HIVC_E_BAD_MAGIC = 2,          /* bitstream.BadMagic            (bitstream.py:41) */
    HIVC_E_UNSUPPORTED_VERSION = 3,/* bitstream.UnsupportedVersion  (bitstream.py:45) */
    HIVC_E_LENGTH_MISMATCH = 4,    /* bitstream.LengthMismatch      (bitstream.py:53) */
    HIVC_E_CODEC = 5,              /* codec.CodecError              (codec.py:69) */
    HIVC_E_ENTROPY = 6,            /* entropy.EntropyError          (entropy.py:31) */
    HIVC_E_SUBDIVISION = 7,        /* subdivision.SubdivisionError  (subdivision.py:21) */
    HIVC_E_INPAINTING = 8,         /* homogeneous.InpaintingError   (homogeneous.py:19) */
    HIVC_E_CONVERGENCE = 9,        /* homogeneous.ConvergenceError  (homogeneous.py:23) */
    HIVC_E_FLOW = 10,              /* flow.FlowError                (flow.py:36) */
    HIVC_E_FRAME = 11,             /* frame.FrameError              (frame.py:15) */
    HIVC_E_QUANTIZE = 12,          /* quantize.QuantizeError        (quantize.py:16) */
    HIVC_E_BITSTREAM = 13,         /* bitstream.BitstreamError (generic header validation, bitstream.py:37,80-91) */
    HIVC_E_PSEUDODIFF = 14,        /* pseudodiff.PseudodiffError    (pseudodiff.py:27) */
    HIVC_E_TRUNCATED_STREAM = 15,  /* bits.TruncatedStream          (bits.py:6) */
    HIVC_E_ARGUMENT = 20,          /* bad call arguments (ValueError) */
    HIVC_E_CUDA = 21,              /* CUDA runtime failure (no device, launch error, ...) */
    HIVC_E_NOMEM = 22
};

/* Thread-local message of the last failing call on this thread. */
const char* hivc_last_error(void);
/* Library build string (arch, flags). */
const char* hivc_version(void);

/* ------------------------------------------------------------------ context
 * One context = one device + one CUDA stream + device scratch.  Contexts are
 * independent; use one per host thread (runtime.map_tasks, runtime.py:37-43).
 */
typedef struct hivc_ctx hivc_ctx;
int hivc_ctx_create(int device, hivc_ctx** out);
int hivc_ctx_destroy(hivc_ctx* ctx);
/* cudaStream_t the context launches on (as an opaque pointer). */
void* hivc_ctx_stream(hivc_ctx* ctx);
/* Wait for all work queued on the context's stream. */
int hivc_ctx_synchronize(hivc_ctx* ctx);
/* Number of device kernels this context has launched so far. */
int64_t hivc_ctx_launch_count(hivc_ctx* ctx);

/* ------------------------------------------------------------------ container
 * Replaces bitstream.unpack_header / read_stream (bitstream.py:102-154).
 */
typedef struct hivc_stream_info {
    int32_t width, height;
    int32_t frame_count;
    int32_t fps_num, fps_den;
    int32_t gop_size;
    int32_t channels;          /* 1 gray, 3 colour (RCT) */
    int32_t intra_levels, flow_levels, residual_levels;
    int32_t gop_count;
} hivc_stream_info;
int hivc_parse_header(const uint8_t* data, size_t len, hivc_stream_info* info);
/* Frames per GOP record (the u16 at the head of each GOP payload, codec.py:494). */
int hivc_gop_frame_counts(const uint8_t* data, size_t len, int32_t* counts, int32_t cap, int32_t* ngops);

/* Host-only parse of every frame record of a stream (the parse half of
 * codec.decode, codec.py:491-561, no GPU needed): 8 int64 per frame — type,
 * intra mask points, flow leaves (u, v), residual marker, coded blocks and
 * mask points of group 0, coded blocks of group 1.  *seconds: parse time. */
int hivc_parse_stream(const uint8_t* data, size_t len, int64_t* stats, int64_t cap, int64_t* nframes,
                      double* seconds);

/* ------------------------------------------------------------------ entropy (host, bit-exact)
 * Replaces entropy.decode_symbols (entropy.py:276-291).  Writes at most `cap`
 * symbols; *count receives the stream's symbol count (call with cap=0 to size).
 */
int hivc_parse_symbols(const uint8_t* data, size_t len, size_t pos,
                       int64_t* out, size_t cap, size_t* count, size_t* next_pos);
/* Replaces entropy.decode_signed_values (entropy.py:311-338). */
int hivc_parse_signed_values(const uint8_t* data, size_t len, size_t pos,
                             int64_t* out, size_t cap, size_t* count, size_t* next_pos);
/* Replaces subdivision.deserialize_tree + SubdivisionTree.leaves (subdivision.py:183-195, 53-69)
 * and parse_mask (198-222): preorder leaf rectangles (x, y, w, h) of a tree
 * over a (width x height) root, read from `nbits` bits of `data` starting at
 * bit `bit_offset` (trees of coded residual tiles are concatenated, codec.py:298-303).
 * Writes at most `cap` leaves (4 int32 each); *nleaves gets the true count,
 * *bits_used the bits consumed. */
int hivc_parse_tree(const uint8_t* data, size_t nbytes, uint64_t nbits, uint64_t bit_offset,
                    int32_t width, int32_t height,
                    int32_t* rects, size_t cap, size_t* nleaves, uint64_t* bits_used);

/* ------------------------------------------------------------------ homogeneous diffusion inpainting
 * Replaces homogeneous.solve_homogeneous (homogeneous.py:157-212): cascadic
 * coarse-to-fine CG, replayed step for step on the GPU (float64).
 * f, mask, u: device pointers (h*w).  level_iters/level_sizes: host arrays of
 * capacity >= 32 receiving (coarse->fine) per-level pixel counts and CG
 * iterations, *nlevels their length (stats["level_iterations"]).
 * Returns HIVC_E_CONVERGENCE in strict mode when the final relative residual
 * exceeds tol (u is still written).
 */
int hivc_homog_solve(hivc_ctx* ctx, const double* f, const uint8_t* mask, int32_t h, int32_t w,
                     double tol, int32_t max_iter, int32_t strict,
                     double* u, int32_t* level_sizes, int32_t* level_iters, int32_t* nlevels);

/* ------------------------------------------------------------------ tonal optimisation operator
 * The two solves of prediction.optimize_mask_values (prediction.py:43-96),
 * whose LSQR operator is v -> A^-1 [v on the mask points] and its adjoint
 * w -> (A^-T w)[mask points], A = diag(d) + diag(1 - d) L (prediction.py:43-61,
 * factorised there with splu).  The forward solve is hivc_homog_solve; the
 * adjoint needs the interior system L_II z_I = w_I (zeros on the mask) and
 * then z_M = w_M - (L z)_M:
 *   hivc_poisson_interior: CG from 0 until ||r|| <= tol ||w_I||; z gets the
 *     full plane (zeros on the mask); *iters the CG iterations.
 *   hivc_mask_adjoint: out[k] = w[pts[k]] - sum of z over pts[k]'s existing
 *     4-neighbours.
 * All pointers are device pointers.
 */
int hivc_poisson_interior(hivc_ctx* ctx, const double* w_full, const uint8_t* mask, int32_t h, int32_t w,
                          double tol, int32_t max_iter, double* z, int32_t* iters);
int hivc_mask_adjoint(hivc_ctx* ctx, const double* w_full, const double* z, const int32_t* pts, int32_t npts,
                      int32_t h, int32_t w, double* out);

/* ------------------------------------------------------------------ flow component decode
 * Replaces flow._decompress_plane (flow.py:343-356) with its
 * uniform_dequantize (quantize.py:78-82) and paint_leaf_values
 * (subdivision.py:162-170): reads f32 lo/hi, u32 nbits, the subdivision tree
 * and the tANS leaf indices at `pos`, and paints each leaf's value on the
 * (h x w) float64 plane `out`.  ctx == NULL: `out` is host memory (painted by
 * the calling thread); else `out` is a device pointer on ctx's device (one
 * kernel launch on ctx's stream, synchronised).  *next_pos: the position
 * after the component.  Errors in the reference's order and classes:
 * HIVC_E_TRUNCATED_STREAM, tree/entropy errors, HIVC_E_QUANTIZE (lo >= hi),
 * HIVC_E_SUBDIVISION (leaf value count mismatch).
 */
int hivc_flow_component(hivc_ctx* ctx, const uint8_t* data, size_t len, size_t pos, int32_t h, int32_t w,
                        int32_t levels, double* out, size_t* next_pos);

/* ------------------------------------------------------------------ warp
 * Replaces flow.warp_planes (flow.py:94-127): every plane sampled at
 * (x+u, y+v), clamped bilinear, float64.  src/dst: host arrays of `nplanes`
 * device pointers; u, v: device pointers.
 */
int hivc_warp(hivc_ctx* ctx, const double* const* src, int32_t nplanes, const double* u, const double* v,
              int32_t h, int32_t w, double* const* dst);

/* ------------------------------------------------------------------ block pseudodifferential residual
 * Replaces pseudodiff.reconstruct_blocks (pseudodiff.py:275-279):
 * out[i] = IDCT_AAN(eig * DCT_AAN(mc[i])) + a[i].  mc/out: device (n*64),
 * a: device (n), eig: device (64) or NULL for greens_eigenvalues_harmonic().
 */
int hivc_block_reconstruct(hivc_ctx* ctx, const double* mc, const double* a, const double* eig,
                           int32_t n, double* out);
/* Replaces pseudodiff.solve_block_coefficients_batch (pseudodiff.py:243-263)
 * for ANY mix of mask layouts: per block the bordered (K+1)^2 system
 * [[G_KK,1],[1^T,0]][c;a] = [f_K;0] is solved in shared memory.
 * f_blocks: device (n*64); masks: device (n) uint64, bit (y*8+x);
 * c_out: device (n*64) — c of block i at its K mask positions, zero elsewhere
 * (the scattered "M c" layout reconstruct_blocks consumes); a_out: device (n). */
int hivc_block_fit(hivc_ctx* ctx, const double* f_blocks, const uint64_t* masks, int32_t n,
                   double* c_out, double* a_out);

/* Replaces the per-block quantise / rebuild / keep loop of codec._encode_residual
 * (codec.py:181-221) for one channel group of npl (1 or 2) planes: all device
 * pointers, per plane c (n x 64 fitted M c), a (n), fb (n x 64 residual tiles);
 * words (n) 8x8 mask words; outputs q (n x 64 int32 indices, 0 off the mask),
 * qa (n), rec (n x 64 rebuilt blocks = the decoder's residual), keep (n). */
int hivc_residual_keep(hivc_ctx* ctx, int32_t npl, const double* const* c, const double* const* a,
                       const double* const* fb, const uint64_t* words, int32_t n, int32_t levels,
                       int32_t bits_per_sym, double c_scale, double a_scale, double lam, int32_t* const* q,
                       int32_t* const* qa, double* const* rec, uint8_t* keep);
/* Fit + rebuild of every 8x8 tile of a float32 residual plane (config 2;
 * solve_block_coefficients_batch + reconstruct_blocks, pseudodiff.py:243-279,
 * edge tiles embedded top-left as in inpaint_plane_blockwise, 299-324).
 * hivc_block_operator: ONE mask layout shared by all tiles (bit y*8+x of
 * `mask`): the fit+rebuild is the fixed 64x64 operator R (float64 on the host),
 * applied to all tiles as a 3xTF32 tcgen05 tensor-core contraction.
 * hivc_block_perblock: per-tile masks (device uint64 array, raster tile order),
 * float64 bordered solves in shared memory.  plane/out: device float32 (h*w). */
int hivc_block_operator(hivc_ctx* ctx, const float* plane, int32_t h, int32_t w, uint64_t mask, float* out);
int hivc_block_perblock(hivc_ctx* ctx, const float* plane, int32_t h, int32_t w, const uint64_t* masks, float* out);

/* ------------------------------------------------------------------ Brox optic flow (encoder side)
 * Replaces flow.flow_brox (flow.py:187-278): backward flow frame_t -> frame_prev,
 * float64, same pyramid / warps / lagged nonlinearity / damped Jacobi / median
 * as the reference.  frame_t, frame_prev, u, v: device float64 planes (h*w).
 * taps_presmooth / taps_antialias: HOST arrays with scipy's normalised 1-D
 * Gaussian taps for sigma = presmooth_sigma and 0.5 / pyramid_scale
 * (scipy.ndimage._gaussian_kernel1d, truncate 4.0; length 2r+1).
 */
typedef struct hivc_brox_params {
    double alpha, gamma, pyramid_scale;
    int32_t min_size, warps, fixed_point_iters, solver_iters;
    double eps, presmooth_sigma;
} hivc_brox_params;
int hivc_brox(hivc_ctx* ctx, const double* frame_t, const double* frame_prev, int32_t h, int32_t w,
              const hivc_brox_params* params, const double* taps_presmooth, int32_t ntaps_presmooth,
              const double* taps_antialias, int32_t ntaps_antialias, double* u, double* v);

/* Replaces flow.flow_horn_schunck (flow.py:281-316): the quadratic-penalty
 * baseline flow, `iterations` Jacobi sweeps in float64 replayed operation for
 * operation (device pointers, planes h x w >= 2 x 2). */
int hivc_horn_schunck(hivc_ctx* ctx, const double* frame_t, const double* frame_prev, int32_t h, int32_t w,
                      double alpha, int32_t iterations, double* u, double* v);

/* ------------------------------------------------------------------ stream decode
 * Replaces codec.decode (codec.py:484-563) for the GOP range [gop_begin, gop_end):
 * frames are written as uint8 planes, layout [frame][channel][h][w] (gray: the
 * Y plane; colour: R, G, B after rct_inverse, frame.py:84-93).  out_on_device:
 * 0 = `out` is host memory (pinned recommended; each frame is copied out as it
 * completes), 1 = device memory written directly, 2 = device memory reached
 * through per-frame device-to-device copies on a copy stream (a peer GPU's
 * buffer, e.g. CUDA-IPC-mapped: the multi-GPU gather fused into the decode).
 * stage_seconds (nullable, 8 doubles) receives the reference timing
 * keys: intra_solve, flow_parse, warp, residual_parse, residual_transform,
 * finalize, total (codec.py:509-562), then the device-side span of the call
 * measured with CUDA events (first lane start -> last lane's final copy).
 * gop_end < 0 means "to the last GOP".
 */
int hivc_decode(hivc_ctx* ctx, const uint8_t* data, size_t len, int32_t gop_begin, int32_t gop_end,
                uint8_t* out, int32_t out_on_device, double* stage_seconds);
/* Several streams in one call (e.g. the Y, Cb, Cr gray streams of a 4:2:0
 * video): all (stream, GOP) pairs share the decode lanes.  Per-stream arrays;
 * gop_begin/gop_end may be NULL (whole streams). */
int hivc_decode_multi(hivc_ctx* ctx, int32_t nstreams, const uint8_t* const* data, const size_t* len,
                      const int32_t* gop_begin, const int32_t* gop_end, uint8_t* const* out,
                      int32_t out_on_device, double* stage_seconds);
/* Peer frame buffers for the fused multi-GPU gather: rank 0 allocates the whole
 * job's frame buffer and exports a 64-byte CUDA IPC handle; every other rank
 * maps it for its own device and decodes with out_on_device = 2 into its slice
 * (each finished frame is copied over NVLink while the next ones decode). */
int hivc_peer_alloc(int32_t device, size_t bytes, void** ptr, uint8_t* ipc_handle);
int hivc_peer_open(int32_t device, const uint8_t* ipc_handle, void** ptr);
int hivc_peer_close(void* ptr);
int hivc_peer_free(void* ptr);
/* Synchronous copy between any two (host / device / peer) addresses. */
int hivc_memcpy(void* dst, const void* src, size_t bytes);
/* Host<->device bytes moved by this context's decodes so far. */
int hivc_ctx_bytes(hivc_ctx* ctx, int64_t* h2d, int64_t* d2h);
/* Accumulated statistics of timed decodes (stage timing on), 10 doubles:
 * CG solves, sum N_l*it_l, sum N_l, cooperative level-kernel launches, their
 * device seconds, their sum N_l*it_l, their sum N_l, P frames, P-kernel device
 * seconds, I frames.  reset != 0 clears them. */
int hivc_ctx_decode_stats(hivc_ctx* ctx, double* out, int32_t reset);
/* Per-frame CUDA-event stage breakdown on (default) or off (pure throughput runs). */
int hivc_ctx_set_stage_timing(hivc_ctx* ctx, int32_t enable);

/* ------------------------------------------------------------------ encoder primitives (host, bit-exact)
 * Output buffers: `cap` bytes at `out`; *size receives the payload size.  A
 * payload larger than `cap` is not written (call again with *size bytes). */
/* Replaces entropy.encode_symbols (entropy.py:255-273); table_log < 0 = automatic
 * (entropy.py:243-252), else 5..12. */
int hivc_encode_symbols(const int64_t* symbols, size_t n, int32_t table_log, uint8_t* out, size_t cap,
                        size_t* size);
/* Replaces entropy.normalize_counts (entropy.py:68-106): histogram of n symbols -> table
 * counts summing to 2^table_log (every present symbol keeps >= 1), written to out[n]. */
int hivc_normalize_counts(const int64_t* hist, size_t n, int32_t table_log, int64_t* out);
/* Replaces entropy.encode_signed_values (entropy.py:294-308). */
int hivc_encode_signed_values(const int64_t* values, size_t n, int32_t table_log, uint8_t* out, size_t cap,
                              size_t* size);
/* Replaces subdivision.subdivide_by_error + serialize_tree + SubdivisionTree.leaves
 * (subdivision.py:76-130, 178-181, 53-69) over C-contiguous float64 planes of
 * width x height: error = region_ssd (nplanes == 1) or joint_ssd_error (nplanes > 1,
 * subdivision.py:133-144) in numpy's float64 summation order; min_error applies when
 * use_min_error != 0.  Tree bits MSB-first into `bits` (ceil(2*target-1 / 8) bytes
 * suffice), *nbits; preorder leaves (x, y, w, h) into `rects` (4*target int32), *nleaves. */
int hivc_subdivide(const double* const* planes, int32_t nplanes, int32_t width, int32_t height, int64_t target,
                   int32_t use_min_error, double min_error, uint8_t* bits, uint64_t* nbits, int32_t* rects,
                   size_t* nleaves);
/* Replaces subdivision.leaf_means (subdivision.py:155-159): numpy-order mean of
 * a float64 plane over each (x, y, w, h) rectangle. */
int hivc_region_means(const double* plane, int32_t width, int32_t height, const int32_t* rects, size_t n,
                      double* out);
/* codec._tile_residuals (codec.py:108-115): tiles `tiles[0..n)` of nplanes int64
 * planes (h x w) embedded top-left into zero-padded 8x8 float64 blocks, out[p][i][64]. */
int hivc_gather_tiles(const int64_t* const* planes, int32_t nplanes, int32_t h, int32_t w, const int64_t* tiles,
                      size_t n, double* out);
/* Replaces codec._plan_group (codec.py:118-137) for one channel group of 1 or 2
 * int64 residual planes (h x w): per raster 8x8 tile t, coded[t] (0: zero in every
 * plane), mask word masks[t] (bit y*8+x), tree bits at tree_bits[16*t] (MSB first)
 * and tree_nbits[t].  threads <= 0: all hardware threads. */
int hivc_plan_residual_tiles(const int64_t* const* planes, int32_t nplanes, int32_t h, int32_t w, int32_t points,
                             int32_t threads, uint8_t* coded, uint64_t* masks, uint8_t* tree_bits,
                             uint8_t* tree_nbits);

#ifdef __cplusplus
}
#endif
#endif /* HIVC_B200_H */
