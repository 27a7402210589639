// Per-frame reconstruction kernels.
//
// frame_kernel: one CTA per strip of 8 tiles (64x8 pixels).  Warps 0..7 first
// rebuild the coded 8x8 residual blocks of their tile (dequantise the compact
// symbols, scatter onto the mask, AAN DCT -> Green's eigenvalues -> AAN IDCT,
// + a; codec.py:316-335, pseudodiff.py:275-279) into shared memory; then every
// thread forms the prediction for its pixels — the inpainted plane (I) or the
// clamped bilinear backward warp of the previous reconstruction along the flow
// trees (P; flow.py:94-127) — and writes clip(rint(rint(pred) + res))
// (codec.py:545-550, frame.py:118-124), with the RCT inverse for colour
// (frame.py:84-93).  The residual planes and the dense flow field never touch
// HBM.  Float64, FMA contraction off, numpy's association order.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "device.cuh"
#include "inpaint.h"
#include "recon.h"
#include "func_attr.h"

namespace hivc {

// Leaf node of the flow tree containing pixel (x, y); the tree may sit in
// shared or global memory (parse.h: parse_flow_tree layout).
__device__ __forceinline__ int flow_leaf(const int32_t* __restrict__ nodes, int x, int y, int start = 0) {
    int i = start;
    int a = __ldg(nodes + 2 * i);
    while (a & 3) {
        int coord = a >> 2;
        bool right = ((a & 3) == 1 ? x : y) >= coord;
        i = right ? __ldg(nodes + 2 * i + 1) : i + 1;
        a = __ldg(nodes + 2 * i);
    }
    return i;
}

// Exact int <-> double without the quarter-rate conversion pipe (B200: DADD
// runs at 64/clk/SM, I2F/F2I/FRND.F64 at ~16): place the integer in the
// mantissa of 2^52 (or 1.5 * 2^52) and subtract.
__device__ __forceinline__ double u32_to_d(unsigned n) {  // exact, any n
    return __hiloint2double(0x43300000, (int)n) - 4503599627370496.0;
}
__device__ __forceinline__ double s32_to_d(int n) {  // exact, any n: biased by 2^31
    return __hiloint2double(0x43380000, n ^ (int)0x80000000) - 6755401588539392.0;
}
// rint (round half to even) for |v| < 2^51: adding 1.5 * 2^52 rounds to an
// integer.  Used only where the result is then clipped to [-255, 255]: a
// larger |v| (a corrupt residual) saturates the clip either way.
__device__ __forceinline__ double rint_clip(double v) { return (v + 6755399441055744.0) - 6755399441055744.0; }
// (int)v for an integral v with |v| < 2^31: its value sits in the low mantissa word of v + 1.5 * 2^52
__device__ __forceinline__ int d_to_int_exact(double v) { return __double2loint(v + 6755399441055744.0); }

__device__ __forceinline__ double to_d(uint8_t v) { return u32_to_d((unsigned)v); }
__device__ __forceinline__ double to_d(int16_t v) { return s32_to_d((int)v); }

template <typename RT>
__device__ __forceinline__ double ld_plane(const void* p, int k) {
    const RT v = __ldg(reinterpret_cast<const RT*>(p) + k);
    if (sizeof(RT) == 1) return u32_to_d((unsigned)v);
    return s32_to_d((int)v);
}

// sym * dz_step / 127 * scale (codec.py:316-321), the first two factors from the table
__device__ __forceinline__ double dequant(const ResDev& R, int sym, double scale) {
    if (R.qtab && sym >= -127 && sym <= 127) return __ldg(R.qtab + sym + 127) * scale;
    return (double)sym * R.dz_step / 127.0 * scale;
}

// Row stride of the residual tiles in shared memory: 9 doubles, so the AAN
// row passes (lane j reads row j) spread over all banks.
constexpr int kResLd = 9;

// Residual block of coded block b, plane ci of group G, built by lanes 0..7.
__device__ __forceinline__ void residual_block(const ResDev& R, const ResGroupDev& G, int b, int ci, double* t,
                                               int lane, unsigned mask8) {
    const uint64_t mask = __ldg(G.block_mask + b);
    const int off = __ldg(G.block_off + b);
    // scatter dequantised coefficients onto the mask (codec.py:316-321)
    const uint64_t below = mask & ((1ull << (lane * 8)) - 1ull);
    int rank = __popcll(below);
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        double v = 0.0;
        if ((mask >> (lane * 8 + x)) & 1ull) {
            const int sym = __ldg(G.c_sym + ci * G.npoints + off + rank);
            ++rank;
            v = dequant(R, sym, R.c_scale);
        }
        t[lane * kResLd + x] = v;
    }
    double a = dequant(R, __ldg(G.a_sym + ci * G.nblocks + b), R.a_scale);
    __syncwarp(mask8);
    block_reconstruct_8lanes<kResLd>(t, lane, kGreensEig, a, mask8);
}

// min(max(v, lo), hi) for finite v (np.clip; the flow values are checked finite)
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    v = v < lo ? lo : v;
    return v > hi ? hi : v;
}

// Layout: a warp covers kWarpTiles horizontally adjacent 8x8 tiles; each
// tile gets kLanesTile lanes — lane (column gl, row half rh) owns column gl
// of the tile for kRowsL rows (rh * kRowsL ...), so every load/store row is
// consecutive pixels and each lane has kRowsL independent prediction chains
// in flight (the warp is latency-bound: tile map -> flow value -> 4 gathers).
// The coded residual blocks of the warp's tiles are rebuilt side by side by
// the first 8 lanes of each tile's group.
#ifndef HIVC_FRAME_ROWS
#define HIVC_FRAME_ROWS 4
#endif
constexpr int kRowsL = HIVC_FRAME_ROWS;          // rows per lane (8 or 4)
constexpr int kLanesTile = 8 * (8 / kRowsL);     // lanes per tile
constexpr int kWarpTiles = 32 / kLanesTile;
constexpr int kFrameWarps = 2;
#ifndef HIVC_FRAME_MIN_BLOCKS
#define HIVC_FRAME_MIN_BLOCKS 16
#endif
// 2-warp CTAs, <= 64 registers.  Measured (ncu, config-3 P frames, 1080p /
// 540p): 8 rows per lane at <= 80 registers 24.4 / 16.5 us; 4 rows 21.2 /
// 12.5 us; 2 rows (one tile per warp) 24.0-25.7 / 12.0 us (profiles/r02_summary.md)
constexpr int kFrameMinBlocks = HIVC_FRAME_MIN_BLOCKS;

template <bool kInter, int C, typename RT>
__global__ void __launch_bounds__(32 * kFrameWarps, kFrameMinBlocks) frame_kernel(FrameArgs A) {
    __shared__ double s_res[kFrameWarps][C][kWarpTiles][8 * kResLd];
    const int h = A.h, w = A.w;
    const int nbx = (w + 7) >> 3;
    const int ty = blockIdx.y;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / kLanesTile, sub = lane % kLanesTile;
    const int gl = sub & 7, r0 = (sub >> 3) * kRowsL;  // column within the tile, first own row
    const int tx = (blockIdx.x * kFrameWarps + wid) * kWarpTiles + grp;
    const bool tile_ok = tx < nbx;
    const int x = tx * 8 + gl;
    const bool col_ok = tile_ok && x < w;
    const int y_base = ty * 8 + r0;
    const int rows = min(kRowsL, h - y_base);  // (<= 0: no rows of this lane in a bottom edge tile)
    // gray: one residual group (see the residual section)
    const bool res_on = C == 1 && A.res.ngroups > 0 && tile_ok;
    const int t_res = ty * nbx + (tile_ok ? tx : 0);
    double pred[kRowsL][C];
    // ---- prediction
    if (kInter) {
        // the host rasterised each flow tree to tiles: most tiles lie inside one
        // leaf (one (u, v) for the tile); tiles on a leaf boundary walk the tree
        const int tt = ty * nbx + (tile_ok ? tx : 0);
        const int lu = __ldg(A.flow.tiles[0] + tt), lv = __ldg(A.flow.tiles[1] + tt);
        const double* __restrict__ vals0 = A.flow.vals[0];
        const double* __restrict__ vals1 = A.flow.vals[1];
        const double wm1 = (double)(w - 1), hm1 = (double)(h - 1);
        const double xd = u32_to_d((unsigned)x), yd0 = u32_to_d((unsigned)y_base);
        // tile map: < 0x8000 leaf (value) index; else walk per pixel from node (t - 0x8000), 0xFFFF: root
        const bool mu = lu >= 0x8000, mv = lv >= 0x8000;
        const int su = lu == 0xFFFF ? 0 : lu - 0x8000, sv = lv == 0xFFFF ? 0 : lv - 0x8000;
        const double u_tile = mu ? 0.0 : __ldg(vals0 + lu);
        const double v_tile = mv ? 0.0 : __ldg(vals1 + lv);
#pragma unroll
        for (int r = 0; r < kRowsL; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) pred[r][c] = 0.0;
        if (col_ok && !mu && !mv) {
            // uniform flow over the tile: one source column pair for all 8 rows;
            // the 8 rows' 32 taps are issued before any is used
            const double sx = clampd(xd + u_tile, 0.0, wm1);
            const int x0 = __double2int_rd(sx);  // floor; sx >= 0
            const int x1 = min(x0 + 1, w - 1);
            const double fx = sx - u32_to_d((unsigned)x0);
            int ra[kRowsL], rb[kRowsL];
            double fy[kRowsL];
#pragma unroll
            for (int r = 0; r < kRowsL; ++r) {
                const double sy = clampd((yd0 + (double)r) + v_tile, 0.0, hm1);
                const int y0 = __double2int_rd(sy);
                ra[r] = y0 * w;
                rb[r] = min(y0 + 1, h - 1) * w;
                fy[r] = sy - u32_to_d((unsigned)y0);
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const RT* __restrict__ p = reinterpret_cast<const RT*>(A.prev[c]);
                RT t00[kRowsL], t01[kRowsL], t10[kRowsL], t11[kRowsL];
                if (sizeof(RT) == 1) {
                    // gray: one address per tap row, the right taps at +1.  Where the
                    // reference clamps x1 = x0 (x0 = w-1) the coordinate was clamped to
                    // exactly w-1, so fx = 0 and w01 = w11 = 0 multiply whatever byte
                    // follows (the next row's first, or the first byte of the frame
                    // after the previous one in the GOP buffer): the sum is unchanged.
                    // (rows past the plane's bottom edge load clamped, in-plane taps and are
                    // never stored: no per-row branch)
#pragma unroll
                    for (int r = 0; r < kRowsL; ++r) {
                        const RT* qa = p + (ra[r] + x0);
                        const RT* qb = p + (rb[r] + x0);
                        t00[r] = __ldg(qa);
                        t01[r] = __ldg(qa + 1);
                        t10[r] = __ldg(qb);
                        t11[r] = __ldg(qb + 1);
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < kRowsL; ++r) {
                        if (r < rows) {
                            t00[r] = __ldg(p + ra[r] + x0);
                            t01[r] = __ldg(p + ra[r] + x1);
                            t10[r] = __ldg(p + rb[r] + x0);
                            t11[r] = __ldg(p + rb[r] + x1);
                        }
                    }
                }
#pragma unroll
                for (int r = 0; r < kRowsL; ++r) {
                    if (sizeof(RT) != 1 && r >= rows) break;
                    const double w00 = (1 - fy[r]) * (1 - fx), w01 = (1 - fy[r]) * fx, w10 = fy[r] * (1 - fx),
                                 w11 = fy[r] * fx;
                    pred[r][c] = ((w00 * to_d(t00[r]) + w01 * to_d(t01[r])) + w10 * to_d(t10[r])) + w11 * to_d(t11[r]);
                }
            }
        } else if (col_ok) {
            // a tile on a leaf boundary: descend both trees for the 8 rows in
            // lockstep (one 8-byte node load per row and tree per level), then
            // the 8 rows' flow values and taps
            int iu[kRowsL], iv[kRowsL];  // node -> (at the end) value index per row
#pragma unroll
            for (int r = 0; r < kRowsL; ++r) {
                iu[r] = mu ? su : -1;
                iv[r] = mv ? sv : -1;
            }
            const int2* __restrict__ n0 = reinterpret_cast<const int2*>(A.flow.nodes[0]);
            const int2* __restrict__ n1 = reinterpret_cast<const int2*>(A.flow.nodes[1]);
            bool more = true;
            while (more) {
                more = false;
                int2 e0[kRowsL], e1[kRowsL];
#pragma unroll
                for (int r = 0; r < kRowsL; ++r) {
                    e0[r] = iu[r] >= 0 ? __ldg(n0 + iu[r]) : make_int2(0, 0);
                    e1[r] = iv[r] >= 0 ? __ldg(n1 + iv[r]) : make_int2(0, 0);
                }
#pragma unroll
                for (int r = 0; r < kRowsL; ++r) {
                    const int y = y_base + r;
                    if (iu[r] >= 0 && (e0[r].x & 3)) {  // split: x-split code 1, y-split code 2
                        const bool right = ((e0[r].x & 3) == 1 ? x : y) >= (e0[r].x >> 2);
                        iu[r] = right ? e0[r].y : iu[r] + 1;
                        more = true;
                    }
                    if (iv[r] >= 0 && (e1[r].x & 3)) {
                        const bool right = ((e1[r].x & 3) == 1 ? x : y) >= (e1[r].x >> 2);
                        iv[r] = right ? e1[r].y : iv[r] + 1;
                        more = true;
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < kRowsL; ++r) {  // leaf node -> its value index
                iu[r] = iu[r] >= 0 ? __ldg(n0 + iu[r]).y : -1;
                iv[r] = iv[r] >= 0 ? __ldg(n1 + iv[r]).y : -1;
            }
#pragma unroll
            for (int r = 0; r < kRowsL; ++r) {
                if (r >= rows) break;
                // flow.py:94-127 — coordinates clamped before flooring, taps summed w00..w11
                const double u = iu[r] >= 0 ? __ldg(vals0 + iu[r]) : u_tile;
                const double v = iv[r] >= 0 ? __ldg(vals1 + iv[r]) : v_tile;
                const double sx = clampd(xd + u, 0.0, wm1);
                const double sy = clampd((yd0 + (double)r) + v, 0.0, hm1);
                const int x0 = __double2int_rd(sx), y0 = __double2int_rd(sy);  // floor; sx, sy >= 0
                const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
                const double fx = sx - u32_to_d((unsigned)x0), fy = sy - u32_to_d((unsigned)y0);
                const double w00 = (1 - fy) * (1 - fx), w01 = (1 - fy) * fx, w10 = fy * (1 - fx), w11 = fy * fx;
                const int i00 = y0 * w + x0, i01 = y0 * w + x1, i10 = y1 * w + x0, i11 = y1 * w + x1;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const void* p = A.prev[c];
                    pred[r][c] = ((w00 * ld_plane<RT>(p, i00) + w01 * ld_plane<RT>(p, i01)) + w10 * ld_plane<RT>(p, i10)) +
                                 w11 * ld_plane<RT>(p, i11);
                }
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < kRowsL; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c)
                pred[r][c] = (col_ok && r < rows) ? __ldg(A.u[c] + (size_t)(y_base + r) * w + x) : 0.0;
    }
    // pred_int = rint(pred) (codec.py:545), in place: |pred| <= 255 for a P frame
    // (a convex combination of frame values) and bounded by the inpainted plane
    // for an I frame, so the 1.5 * 2^52 rounding is exact
#pragma unroll
    for (int r = 0; r < kRowsL; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) pred[r][c] = rint_clip(pred[r][c]);
    // ---- residual block(s): lanes 8g..8g+7 rebuild tile g's coded blocks
    bool coded[2] = {false, false};
    if (C == 1) {
        // gray: one group with a static index, so `coded` stays in registers (a
        // runtime group index put it in local memory, read back in the epilogue);
        // loading the tile word ahead of the prediction measured no better
        if (res_on) {
            const unsigned mask8 = 0xFFu << (kLanesTile * grp);
            const ResGroupDev& G = A.res.g[0];
            const uint64_t word0 = __ldg(G.tile_words + (t_res >> 6));
            coded[0] = (word0 >> (t_res & 63)) & 1ull;
            if (coded[0] && sub < 8) {
                const int b = __ldg(G.word_prefix + (t_res >> 6)) + __popcll(word0 & ((1ull << (t_res & 63)) - 1ull));
                residual_block(A.res, G, b, 0, &s_res[wid][0][grp][0], gl, mask8);
            }
        }
    } else if (A.res.ngroups > 0 && tile_ok) {
        const int t = ty * nbx + tx;
        const unsigned mask8 = 0xFFu << (kLanesTile * grp);
        int chan = 0;
        for (int gi = 0; gi < A.res.ngroups; ++gi) {
            const ResGroupDev& G = A.res.g[gi];
            const uint64_t word = __ldg(G.tile_words + (t >> 6));
            coded[gi] = (word >> (t & 63)) & 1ull;
            if (coded[gi] && sub < 8) {
                const int b = __ldg(G.word_prefix + (t >> 6)) + __popcll(word & ((1ull << (t & 63)) - 1ull));
                for (int ci = 0; ci < G.nplanes; ++ci)
                    residual_block(A.res, G, b, ci, &s_res[wid][chan + ci][grp][0], gl, mask8);
            }
            chan += G.nplanes;
        }
    }
    __syncwarp();
    if (!col_ok) return;
#pragma unroll
    for (int r = 0; r < kRowsL; ++r) {
        if (r >= rows) continue;  // (predicated, no loop exit)
        const size_t k = (size_t)(y_base + r) * w + x;
        int rec[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int gi = c == 0 ? 0 : 1;
            const double res = coded[gi] ? s_res[wid][c][grp][(r0 + r) * kResLd + gl] : 0.0;
            double v = rint_clip(pred[r][c] + res);
            const double lo = (C == 3 && c > 0) ? -255.0 : 0.0;
            v = clampd(v, lo, 255.0);
            rec[c] = d_to_int_exact(v);
            reinterpret_cast<RT*>(A.recon[c])[k] = (RT)rec[c];
        }
        if (C == 3) {
            // rct_inverse (frame.py:84-93) + clip to [0, 255] (codec.py:479-480)
            const int g = rec[0] - ((rec[1] + rec[2]) >> 2);
            const int rr = rec[2] + g, bb = rec[1] + g;
            A.rgb[0][k] = (uint8_t)min(max(rr, 0), 255);
            A.rgb[1][k] = (uint8_t)min(max(g, 0), 255);
            A.rgb[2][k] = (uint8_t)min(max(bb, 0), 255);
        }
    }
}

void launch_frame(const FrameArgs& a, bool inter, cudaStream_t s) {
    const int tiles_per_cta = kFrameWarps * kWarpTiles;
    dim3 grid((((a.w + 7) / 8) + tiles_per_cta - 1) / tiles_per_cta, (a.h + 7) / 8);
    const int nt = 32 * kFrameWarps;
    if (a.channels == 1) {
        if (inter)
            frame_kernel<true, 1, uint8_t><<<grid, nt, 0, s>>>(a);
        else
            frame_kernel<false, 1, uint8_t><<<grid, nt, 0, s>>>(a);
    } else {
        if (inter)
            frame_kernel<true, 3, int16_t><<<grid, nt, 0, s>>>(a);
        else
            frame_kernel<false, 3, int16_t><<<grid, nt, 0, s>>>(a);
    }
    CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------- intra scatter

__global__ void scatter_kernel(const int32_t* __restrict__ pts, const double* __restrict__ vals, int npts,
                               double* __restrict__ f, uint8_t* __restrict__ m) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npts) return;
    int p = pts[i];
    f[p] = vals[i];
    if (m) m[p] = 1;
}

void launch_scatter(const int32_t* pts, const double* vals, int npts, double* f, uint8_t* m, cudaStream_t s) {
    if (npts <= 0) return;
    scatter_kernel<<<(npts + 255) / 256, 256, 0, s>>>(pts, vals, npts, f, m);
    CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------- standalone warp (function-level API)

struct WarpArgs {
    const double* src[8];
    double* dst[8];
    int nplanes;
};

__global__ void warp_kernel(WarpArgs P, const double* __restrict__ u, const double* __restrict__ v, int h, int w) {
    int n = h * w;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        int y = k / w, x = k % w;
        double sx = fmin(fmax((double)x + u[k], 0.0), (double)(w - 1));
        double sy = fmin(fmax((double)y + v[k], 0.0), (double)(h - 1));
        int x0 = (int)floor(sx), y0 = (int)floor(sy);
        int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
        double fx = sx - (double)x0, fy = sy - (double)y0;
        double w00 = (1 - fy) * (1 - fx), w01 = (1 - fy) * fx, w10 = fy * (1 - fx), w11 = fy * fx;
        size_t i00 = (size_t)y0 * w + x0, i01 = (size_t)y0 * w + x1, i10 = (size_t)y1 * w + x0,
               i11 = (size_t)y1 * w + x1;
        for (int c = 0; c < P.nplanes; ++c) {
            const double* p = P.src[c];
            P.dst[c][k] = ((w00 * __ldg(p + i00) + w01 * __ldg(p + i01)) + w10 * __ldg(p + i10)) + w11 * __ldg(p + i11);
        }
    }
}

void launch_warp(const double* const* src, int nplanes, const double* u, const double* v, int h, int w,
                 double* const* dst, cudaStream_t s) {
    for (int c0 = 0; c0 < nplanes; c0 += 8) {
        WarpArgs P;
        P.nplanes = nplanes - c0 < 8 ? nplanes - c0 : 8;
        for (int c = 0; c < P.nplanes; ++c) {
            P.src[c] = src[c0 + c];
            P.dst[c] = dst[c0 + c];
        }
        int n = h * w;
        int nb = (n + 255) / 256;
        if (nb > 148 * 16) nb = 148 * 16;
        warp_kernel<<<nb, 256, 0, s>>>(P, u, v, h, w);
        CUDA_CHECK(cudaGetLastError());
    }
}

// ---------------------------------------------------------------- leaf painting

// One CTA column per leaf (blockIdx.x), blockIdx.y strides the leaf's rows; a
// row is written by consecutive threads (coalesced 8-byte stores).  Leaves
// tile the plane, so every pixel is written exactly once.
__global__ void paint_leaves_kernel(const int4* __restrict__ rects, const double* __restrict__ vals, int pw,
                                    double* __restrict__ out) {
    const int4 r = rects[blockIdx.x];
    const double v = vals[blockIdx.x];
    for (int y = blockIdx.y; y < r.w; y += gridDim.y) {
        double* row = out + (size_t)(r.y + y) * pw + r.x;
        for (int x = threadIdx.x; x < r.z; x += blockDim.x) row[x] = v;
    }
}

void launch_paint_leaves(const int32_t* rects, const double* vals, int nleaves, int pw, double* out, cudaStream_t s) {
    if (nleaves <= 0) return;
    // rect fields are (x, y, w, h): int4 .x=x .y=y .z=w .w=h
    paint_leaves_kernel<<<dim3(nleaves, 8), 128, 0, s>>>(reinterpret_cast<const int4*>(rects), vals, pw, out);
    CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------- standalone block reconstruct

__global__ void block_reconstruct_kernel(const double* __restrict__ mc, const double* __restrict__ a,
                                         const double* __restrict__ eig, int n, double* __restrict__ out) {
    __shared__ double t[8][64];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * 8 + wid;
    if (b >= n || lane >= 8) return;
    for (int x = 0; x < 8; ++x) t[wid][lane * 8 + x] = mc[(size_t)b * 64 + lane * 8 + x];
    __syncwarp(0xffu);
    block_reconstruct_8lanes(&t[wid][0], lane, eig, a[b], 0xffu);
    for (int x = 0; x < 8; ++x) out[(size_t)b * 64 + lane * 8 + x] = t[wid][lane * 8 + x];
}

__global__ void block_reconstruct_default_eig(const double* __restrict__ mc, const double* __restrict__ a, int n,
                                              double* __restrict__ out) {
    __shared__ double t[8][64];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * 8 + wid;
    if (b >= n || lane >= 8) return;
    for (int x = 0; x < 8; ++x) t[wid][lane * 8 + x] = mc[(size_t)b * 64 + lane * 8 + x];
    __syncwarp(0xffu);
    block_reconstruct_8lanes(&t[wid][0], lane, kGreensEig, a[b], 0xffu);
    for (int x = 0; x < 8; ++x) out[(size_t)b * 64 + lane * 8 + x] = t[wid][lane * 8 + x];
}

void launch_block_reconstruct(const double* mc, const double* a, const double* eig, int n, double* out,
                              cudaStream_t s) {
    if (n <= 0) return;
    if (eig)
        block_reconstruct_kernel<<<(n + 7) / 8, 256, 0, s>>>(mc, a, eig, n, out);
    else
        block_reconstruct_default_eig<<<(n + 7) / 8, 256, 0, s>>>(mc, a, n, out);
    CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------- residual encoder: quantise + keep decision
// codec._encode_residual's per-block loop (codec.py:181-221) for one channel
// group of npl planes, 8 lanes (rows) per block: map + dead-zone quantise the
// fitted coefficients and constant (quantize.py:32-58), dequantise + unmap,
// rebuild the block (the decoder's AAN path), and keep it when it has a
// nonzero index and gain = sum_planes(sum(r*r) - sum((r-rec)^2)) exceeds
// lam * (8 + npl (K+1) bits_per_sym).  Sums in numpy's order for 64 terms
// (8 column accumulators over rows, then the pairwise tree).

__device__ __forceinline__ int32_t deadzone_q(double c, double scale, double step, int lmax) {
    double m = c / scale * 127.0;  // map_coefficients
    m = fmin(fmax(m, -127.0), 127.0);
    const double sg = m > 0.0 ? 1.0 : (m < 0.0 ? -1.0 : 0.0);
    double idx = sg * floor(fabs(m) / step);  // deadzone_quantize
    idx = fmin(fmax(idx, (double)-lmax), (double)lmax);
    return (int32_t)idx;
}

__global__ void residual_keep_kernel(const __grid_constant__ KeepArgs A) {
    __shared__ double t[8][64];
    __shared__ double u[8][64];
    __shared__ double g[8][8];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * 8 + wid;
    if (b >= A.n || lane >= 8) return;
    const unsigned m8 = 0xffu;
    const uint64_t word = A.words[b];
    const int j = lane;
    bool nz = false;
    double gain = 0.0;
    for (int ci = 0; ci < A.npl; ++ci) {
        // quantise this row's coefficients, dequantise + unmap into the rebuild buffer
        for (int x = 0; x < 8; ++x) {
            const int k = j * 8 + x;
            double mc = 0.0;
            int32_t qv = 0;
            if ((word >> k) & 1ull) {
                qv = deadzone_q(A.c[ci][(size_t)b * 64 + k], A.c_scale, A.step, A.lmax);
                mc = (double)qv * A.step / 127.0 * A.c_scale;  // unmap(deadzone_dequantize)
            }
            nz |= qv != 0;
            A.q[ci][(size_t)b * 64 + k] = qv;
            t[wid][k] = mc;
        }
        const int32_t qa = deadzone_q(A.a[ci][b], A.a_scale, A.step, A.lmax);
        nz |= qa != 0;
        if (j == 0) A.qa[ci][b] = qa;
        const double a_hat = (double)qa * A.step / 127.0 * A.a_scale;
        __syncwarp(m8);
        block_reconstruct_8lanes(&t[wid][0], j, kGreensEig, a_hat, m8);
        // r*r and (r-rec)^2 of this row, then column sums down the rows in order
        for (int x = 0; x < 8; ++x) {
            const int k = j * 8 + x;
            const double r = A.fb[ci][(size_t)b * 64 + k], rc = t[wid][k];
            A.rec[ci][(size_t)b * 64 + k] = rc;
            const double d = r - rc;
            u[wid][k] = r * r;
            t[wid][k] = d * d;
        }
        __syncwarp(m8);
        double s1 = u[wid][j], s2 = t[wid][j];  // accumulator j: elements j, j+8, ..., j+56
        for (int row = 1; row < 8; ++row) {
            s1 += u[wid][row * 8 + j];
            s2 += t[wid][row * 8 + j];
        }
        g[wid][j] = s1;
        __syncwarp(m8);
        const double S1 = ((g[wid][0] + g[wid][1]) + (g[wid][2] + g[wid][3])) +
                          ((g[wid][4] + g[wid][5]) + (g[wid][6] + g[wid][7]));
        __syncwarp(m8);
        g[wid][j] = s2;
        __syncwarp(m8);
        const double S2 = ((g[wid][0] + g[wid][1]) + (g[wid][2] + g[wid][3])) +
                          ((g[wid][4] + g[wid][5]) + (g[wid][6] + g[wid][7]));
        __syncwarp(m8);
        gain = gain + (S1 - S2);
    }
    nz = __any_sync(m8, nz);
    if (j == 0) {
        const int k = __popcll(word);
        const double cost = (double)(8 + A.npl * (k + 1) * A.bits_per_sym);
        A.keep[b] = nz && gain > A.lam * cost;
    }
}

void launch_residual_keep(const KeepArgs& A, cudaStream_t s) {
    if (A.n <= 0) return;
    residual_keep_kernel<<<(A.n + 7) / 8, 256, 0, s>>>(A);
    CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------- block coefficient fit (any mask layout)
// One warp per block: the bordered (K+1)x(K+1) system [[G_KK,1],[1^T,0]] is
// assembled in shared memory from the 64x64 Green's matrix and solved by
// Gaussian elimination with partial pivoting (LAPACK gesv's pivot rule),
// lanes owning columns.  Output is the scattered M c layout + a.
constexpr int kFitWarps = 4;
constexpr int kFitMaxK = 64;
constexpr int kFitLd = kFitMaxK + 2;

__global__ void __launch_bounds__(kFitWarps * 32) block_fit_kernel(const double* __restrict__ f,
                                                                   const uint64_t* __restrict__ masks, int n,
                                                                   double* __restrict__ c_out,
                                                                   double* __restrict__ a_out, int* status) {
    extern __shared__ double smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * kFitWarps + wid;
    if (b >= n) return;
    double* M = smem + (size_t)wid * (kFitMaxK + 1) * kFitLd;
    int* pos = reinterpret_cast<int*>(smem + (size_t)kFitWarps * (kFitMaxK + 1) * kFitLd) + wid * 64;
    const uint64_t mask = masks[b];
    const int K = __popcll(mask);
    if (K == 0) {
        if (lane == 0) atomicExch(status, 1);
        for (int j = lane; j < 64; j += 32) c_out[(size_t)b * 64 + j] = 0.0;
        if (lane == 0) a_out[b] = 0.0;
        return;
    }
    // mask positions in raster order
    for (int j = lane; j < 64; j += 32) {
        if ((mask >> j) & 1ull) pos[__popcll(mask & ((1ull << j) - 1ull))] = j;
    }
    __syncwarp();
    const int N = K + 1;
    // augmented matrix [A | rhs], row-major, ld = kFitLd
    for (int e = lane; e < N * N; e += 32) {
        int i = e / N, j = e % N;
        double v;
        if (i < K && j < K)
            v = kGreens64[pos[i] * 64 + pos[j]];
        else if (i == K && j == K)
            v = 0.0;
        else
            v = 1.0;
        M[i * kFitLd + j] = v;
    }
    for (int i = lane; i < N; i += 32) M[i * kFitLd + N] = i < K ? f[(size_t)b * 64 + pos[i]] : 0.0;
    __syncwarp();
    bool singular = false;
    for (int col = 0; col < N; ++col) {
        // pivot: first row with max |a| (idamax)
        int piv = col;
        double best = -1.0;
        for (int i = col; i < N; ++i) {
            double v = fabs(M[i * kFitLd + col]);
            if (v > best) {
                best = v;
                piv = i;
            }
        }
        if (best == 0.0) {
            singular = true;
            break;
        }
        if (piv != col)
            for (int j = lane; j <= N; j += 32) {
                double t = M[col * kFitLd + j];
                M[col * kFitLd + j] = M[piv * kFitLd + j];
                M[piv * kFitLd + j] = t;
            }
        __syncwarp();
        const double d = M[col * kFitLd + col];
        for (int i = col + 1; i < N; ++i) {
            const double l = M[i * kFitLd + col] / d;
            for (int j = col + 1 + lane; j <= N; j += 32) M[i * kFitLd + j] = M[i * kFitLd + j] - l * M[col * kFitLd + j];
            __syncwarp();
        }
    }
    if (singular) {
        if (lane == 0) atomicExch(status, 2);
        return;
    }
    // back substitution (serial, tiny)
    if (lane == 0) {
        for (int i = N - 1; i >= 0; --i) {
            double s = M[i * kFitLd + N];
            for (int j = i + 1; j < N; ++j) s = s - M[i * kFitLd + j] * M[j * kFitLd + N];
            M[i * kFitLd + N] = s / M[i * kFitLd + i];
        }
    }
    __syncwarp();
    for (int j = lane; j < 64; j += 32) c_out[(size_t)b * 64 + j] = 0.0;
    __syncwarp();
    for (int i = lane; i < K; i += 32) c_out[(size_t)b * 64 + pos[i]] = M[i * kFitLd + N];
    if (lane == 0) a_out[b] = M[K * kFitLd + N];
}

void launch_block_fit(const double* f, const uint64_t* masks, int n, double* c_out, double* a_out, int* status,
                      cudaStream_t s) {
    if (n <= 0) return;
    size_t smem = (size_t)kFitWarps * (kFitMaxK + 1) * kFitLd * sizeof(double) + kFitWarps * 64 * sizeof(int);
    ensure_func_attr((const void*)block_fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    block_fit_kernel<<<(n + kFitWarps - 1) / kFitWarps, kFitWarps * 32, smem, s>>>(f, masks, n, c_out, a_out, status);
    CUDA_CHECK(cudaGetLastError());
}

}  // namespace hivc
