// Host interface of the reconstruction kernels (recon.cu): the fused
// per-frame finalize (prediction + block residual + rint + clip [+ RCT]),
// the standalone warp / block-reconstruct kernels of the function-level
// API, and the intra mask scatter.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hivc {

struct ResGroupDev {
    int nplanes = 0, nblocks = 0, npoints = 0;
    const uint64_t* tile_words = nullptr;  // bit t%64 of word t/64: tile t coded
    const int32_t* word_prefix = nullptr;  // coded tiles before each word
    const uint64_t* block_mask = nullptr;  // per coded block: bit y*8+x
    const int32_t* block_off = nullptr;    // per coded block: first point index
    const int32_t* c_sym = nullptr;        // plane-major, nplanes * npoints
    const int32_t* a_sym = nullptr;        // plane-major, nplanes * nblocks
};

struct ResDev {
    int ngroups = 0;                            // 0: all-zero residual
    double dz_step = 0, c_scale = 0, a_scale = 0;  // dead-zone step 127/((L-1)/2), c_fp/65536, a_fp/65536
    // optional: qtab[s + 127] = s * dz_step / 127.0 for |s| <= 127 (then one
    // multiply by the scale dequantises a symbol, same rounding as the reference)
    const double* qtab = nullptr;
    ResGroupDev g[2];
};

struct FlowDev {
    const int32_t* nodes[2] = {nullptr, nullptr};  // u, v trees (parse.h: parse_flow_tree)
    const double* vals[2] = {nullptr, nullptr};
    const uint16_t* tiles[2] = {nullptr, nullptr};  // per-tile covering leaf, 0xFFFF = mixed
    int nleaves[2] = {0, 0};                        // leaves (values) per tree; nodes = 2 * leaves - 1
};

struct FrameArgs {
    int h = 0, w = 0, channels = 1;
    const double* u[3] = {nullptr, nullptr, nullptr};  // intra: inpainted planes
    const void* prev[3] = {nullptr, nullptr, nullptr}; // inter: previous reconstruction
    FlowDev flow;
    ResDev res;
    void* recon[3] = {nullptr, nullptr, nullptr};      // out: reconstruction (uint8 gray / int16 colour)
    uint8_t* rgb[3] = {nullptr, nullptr, nullptr};     // out: RGB planes (colour only)
};

// kInter: warp prediction from prev + flow trees; else prediction = u.
void launch_frame(const FrameArgs& a, bool inter, cudaStream_t s);

// f.ravel()[pts] = vals; mask.ravel()[pts] = 1 (prediction.py:203-208) after zero fill.
void launch_scatter(const int32_t* pts, const double* vals, int npts, double* f, uint8_t* m, cudaStream_t s);

// subdivision.paint_leaf_values (subdivision.py:162-170): out[y:y+h, x:x+w] = vals[i]
// for every preorder leaf rect i (x, y, w, h int32 quadruples), plane width `pw`.
void launch_paint_leaves(const int32_t* rects, const double* vals, int nleaves, int pw, double* out, cudaStream_t s);

// flow.warp_planes on float64 planes (flow.py:94-127).
void launch_warp(const double* const* src, int nplanes, const double* u, const double* v, int h, int w,
                 double* const* dst, cudaStream_t s);

// pseudodiff.reconstruct_blocks (pseudodiff.py:275-279).
void launch_block_reconstruct(const double* mc, const double* a, const double* eig, int n, double* out,
                              cudaStream_t s);

// pseudodiff.solve_block_coefficients_batch (pseudodiff.py:243-263), any mask mix.
void launch_block_fit(const double* f, const uint64_t* masks, int n, double* c_out, double* a_out, int* status,
                      cudaStream_t s);

// codec._encode_residual's quantise + keep decision for one channel group (codec.py:181-221).
struct KeepArgs {
    const double* c[2];   // fitted M c per plane (n x 64, zero off the mask)
    const double* a[2];   // fitted constants per plane (n)
    const double* fb[2];  // residual tiles per plane (n x 64)
    const uint64_t* words;
    int n, npl, lmax, bits_per_sym;
    double c_scale, a_scale, step, lam;
    int32_t* q[2];   // out: quantised coefficient indices (n x 64, 0 off the mask)
    int32_t* qa[2];  // out: quantised constants (n)
    double* rec[2];  // out: rebuilt blocks (n x 64)
    uint8_t* keep;   // out
};
void launch_residual_keep(const KeepArgs& A, cudaStream_t s);

const double* device_default_eig();  // greens_eigenvalues_harmonic() in device memory

}  // namespace hivc
