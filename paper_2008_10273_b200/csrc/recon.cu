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

#include "device.cuh"
#include "inpaint.h"
#include "recon.h"

namespace hivc {

// Leaf node of the flow tree containing pixel (x, y).
__device__ __forceinline__ int flow_leaf(const int32_t* __restrict__ nodes, int x, int y) {
    int i = 0;
    int a = __ldg(nodes);
    while (a & 3) {
        int coord = a >> 2;
        bool right = ((a & 3) == 1 ? x : y) >= coord;
        i = right ? __ldg(nodes + 2 * i + 1) : i + 1;
        a = __ldg(nodes + 2 * i);
    }
    return i;
}

__device__ __forceinline__ double flow_lookup(const int32_t* __restrict__ nodes, const double* __restrict__ vals, int x,
                                              int y) {
    return __ldg(vals + __ldg(nodes + 2 * flow_leaf(nodes, x, y) + 1));
}

template <typename RT>
__device__ __forceinline__ double ld_plane(const void* p, size_t k) {
    return (double)__ldg(reinterpret_cast<const RT*>(p) + k);
}

// Residual block of coded block b, plane ci of group G, built by lanes 0..7.
__device__ __forceinline__ void residual_block(const ResDev& R, const ResGroupDev& G, int b, int ci, double* t,
                                               int lane) {
    const uint64_t mask = __ldg(G.block_mask + b);
    const int off = __ldg(G.block_off + b);
    // scatter dequantised coefficients onto the mask (codec.py:316-321)
    for (int x = 0; x < 8; ++x) {
        int bit = lane * 8 + x;
        double v = 0.0;
        if ((mask >> bit) & 1ull) {
            int rank = __popcll(mask & ((1ull << bit) - 1ull));
            int sym = __ldg(G.c_sym + (size_t)ci * G.npoints + off + rank);
            v = (double)sym * R.dz_step / 127.0 * R.c_scale;
        }
        t[lane * 8 + x] = v;
    }
    double a = (double)__ldg(G.a_sym + (size_t)ci * G.nblocks + b) * R.dz_step / 127.0 * R.a_scale;
    __syncwarp(0xffu);
    block_reconstruct_8lanes(t, lane, kGreensEig, a, 0xffu);
}

template <bool kInter, int C, typename RT>
__global__ void __launch_bounds__(256) frame_kernel(FrameArgs A) {
    __shared__ double s_res[C][8][64];
    const int h = A.h, w = A.w;
    const int nbx = (w + 7) >> 3;
    const int ty = blockIdx.y;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tx = blockIdx.x * 8 + wid;

    // One warp per 8x8 tile: lane l owns column l % 8 of rows l / 8 and l / 8 + 4.
    // The prediction loads are issued first; the tile's residual block is
    // rebuilt (lanes 0..7) while they are in flight; no CTA-wide barrier.
    const int lx = lane & 7, ly = lane >> 3;
    const int x = tx * 8 + lx;
    const bool tile_ok = tx < nbx;
    double pred[2][C];
    bool live[2];
    // ---- prediction
    if (kInter) {
        // the host rasterised each flow tree to tiles: most tiles lie inside one
        // leaf (one (u, v) for the tile); tiles on a leaf boundary walk the tree
        const size_t tt = (size_t)ty * nbx + (tile_ok ? tx : 0);
        const int lu = __ldg(A.flow.tiles[0] + tt), lv = __ldg(A.flow.tiles[1] + tt);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int y = ty * 8 + ly + 4 * rr;
            live[rr] = tile_ok && x < w && y < h;
            if (!live[rr]) continue;
            // flow.py:94-127 — coordinates clamped before flooring, taps summed w00..w11
            double u = lu != 0xFFFF ? __ldg(A.flow.vals[0] + lu) : flow_lookup(A.flow.nodes[0], A.flow.vals[0], x, y);
            double v = lv != 0xFFFF ? __ldg(A.flow.vals[1] + lv) : flow_lookup(A.flow.nodes[1], A.flow.vals[1], x, y);
            double sx = fmin(fmax((double)x + u, 0.0), (double)(w - 1));
            double sy = fmin(fmax((double)y + v, 0.0), (double)(h - 1));
            int x0 = (int)floor(sx), y0 = (int)floor(sy);
            int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
            double fx = sx - (double)x0, fy = sy - (double)y0;
            double w00 = (1 - fy) * (1 - fx), w01 = (1 - fy) * fx, w10 = fy * (1 - fx), w11 = fy * fx;
            size_t i00 = (size_t)y0 * w + x0, i01 = (size_t)y0 * w + x1, i10 = (size_t)y1 * w + x0,
                   i11 = (size_t)y1 * w + x1;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const void* p = A.prev[c];
                pred[rr][c] = ((w00 * ld_plane<RT>(p, i00) + w01 * ld_plane<RT>(p, i01)) + w10 * ld_plane<RT>(p, i10)) +
                              w11 * ld_plane<RT>(p, i11);
            }
        }
    } else {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int y = ty * 8 + ly + 4 * rr;
            live[rr] = tile_ok && x < w && y < h;
#pragma unroll
            for (int c = 0; c < C; ++c) pred[rr][c] = live[rr] ? __ldg(A.u[c] + (size_t)y * w + x) : 0.0;
        }
    }
    // ---- residual block(s) of this tile
    bool coded[2] = {false, false};
    if (A.res.ngroups > 0 && tile_ok) {
        const size_t t = (size_t)ty * nbx + tx;
        int chan = 0;
        for (int gi = 0; gi < A.res.ngroups; ++gi) {
            const ResGroupDev& G = A.res.g[gi];
            uint64_t word = __ldg(G.tile_words + (t >> 6));
            coded[gi] = (word >> (t & 63)) & 1ull;
            if (coded[gi]) {
                int b = __ldg(G.word_prefix + (t >> 6)) + __popcll(word & ((1ull << (t & 63)) - 1ull));
                if (lane < 8)
                    for (int ci = 0; ci < G.nplanes; ++ci) residual_block(A.res, G, b, ci, &s_res[chan + ci][wid][0], lane);
            }
            chan += G.nplanes;
        }
        __syncwarp();
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        if (!live[rr]) continue;
        const int row = ly + 4 * rr;
        const int y = ty * 8 + row;
        const size_t k = (size_t)y * w + x;
        int rec[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int gi = c == 0 ? 0 : 1;
            double res = coded[gi] ? s_res[c][wid][row * 8 + lx] : 0.0;
            double v = rint(rint(pred[rr][c]) + res);
            const double lo = (C == 3 && c > 0) ? -255.0 : 0.0;
            v = fmin(fmax(v, lo), 255.0);
            rec[c] = (int)v;
            reinterpret_cast<RT*>(A.recon[c])[k] = (RT)rec[c];
        }
        if (C == 3) {
            // rct_inverse (frame.py:84-93) + clip to [0, 255] (codec.py:479-480)
            int g = rec[0] - ((rec[1] + rec[2]) >> 2);
            int r = rec[2] + g, b = rec[1] + g;
            A.rgb[0][k] = (uint8_t)min(max(r, 0), 255);
            A.rgb[1][k] = (uint8_t)min(max(g, 0), 255);
            A.rgb[2][k] = (uint8_t)min(max(b, 0), 255);
        }
    }
}

void launch_frame(const FrameArgs& a, bool inter, cudaStream_t s) {
    dim3 grid((((a.w + 7) / 8) + 7) / 8, (a.h + 7) / 8);
    if (a.channels == 1) {
        if (inter)
            frame_kernel<true, 1, uint8_t><<<grid, 256, 0, s>>>(a);
        else
            frame_kernel<false, 1, uint8_t><<<grid, 256, 0, s>>>(a);
    } else {
        if (inter)
            frame_kernel<true, 3, int16_t><<<grid, 256, 0, s>>>(a);
        else
            frame_kernel<false, 3, int16_t><<<grid, 256, 0, s>>>(a);
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
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(block_fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    block_fit_kernel<<<(n + kFitWarps - 1) / kFitWarps, kFitWarps * 32, smem, s>>>(f, masks, n, c_out, a_out, status);
    CUDA_CHECK(cudaGetLastError());
}

}  // namespace hivc
