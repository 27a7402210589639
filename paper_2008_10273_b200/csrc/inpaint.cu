// Homogeneous-diffusion inpainting on the GPU: the reference's cascadic
// conjugate-gradient scheme (homogeneous.py:55-212) replayed step for step.
//
//  * pyramid: 2x2 ceiling-halving restriction, any-child mask, mean of the
//    set children (homogeneous.py:96-130) — one kernel per level;
//  * per level one persistent kernel runs the whole CG: setup (prolongation
//    of the coarser solution, x0 * interior, b = L(u_D) * interior,
//    r = b - A x), then the iteration loop with both global dot products per
//    iteration reduced in a fixed order, so every CTA takes the same
//    alpha/beta/stop decisions and the result is bit-reproducible;
//  * large levels run on one CTA per SM with a software grid barrier
//    (cooperative launch); small levels run in a single CTA with
//    __syncthreads only.
// Float64 throughout, FMA contraction off, sums associated as in numpy.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "device.cuh"
#include "inpaint.h"

namespace hivc {

constexpr int kCoarsest = 16;      // homogeneous.py:15
constexpr double kLevelTol = 1e-4;  // homogeneous.py:16
constexpr int kThreads = 1024;
constexpr int kSingleCtaMaxPx = 16384;

// ---------------------------------------------------------------- pyramid

struct RestrictBatch {  // blockIdx.y = solve
    const double* f[16];
    const uint8_t* m[16];
    double* fc[16];
    uint8_t* mc[16];
};

// One coarse pixel i of a 2x restriction (homogeneous.py:110-130): mask = any
// fine mask pixel, f = mean of the masked fine values (else of all of them);
// np.add.reduceat over rows, then over columns (homogeneous.py:121-122).
__device__ __forceinline__ void restrict_px(const double* __restrict__ f, const uint8_t* __restrict__ m,
                                            double* __restrict__ fc, uint8_t* __restrict__ mc, int h, int w, int wc,
                                            int i) {
    int cy = i / wc, cx = i % wc;
    int r0 = 2 * cy, c0 = 2 * cx;
    bool hr = r0 + 1 < h, hcol = c0 + 1 < w;
    auto at = [&](int r, int c, int kind) -> double {
        size_t k = (size_t)r * w + c;
        bool mk = m[k] != 0;
        switch (kind) {
            case 0: return mk ? 1.0 : 0.0;
            case 1: return mk ? f[k] : 0.0;
            case 2: return 1.0;
            default: return f[k];
        }
    };
    double tot[4];
#pragma unroll
    for (int kind = 0; kind < 4; ++kind) {
        double s0 = hr ? at(r0, c0, kind) + at(r0 + 1, c0, kind) : at(r0, c0, kind);
        double t = s0;
        if (hcol) {
            double s1 = hr ? at(r0, c0 + 1, kind) + at(r0 + 1, c0 + 1, kind) : at(r0, c0 + 1, kind);
            t = s0 + s1;
        }
        tot[kind] = t;
    }
    double avg = tot[3] / tot[2];
    bool cm = tot[0] > 0.0;
    fc[i] = cm ? tot[1] / fmax(tot[0], 1.0) : avg;
    mc[i] = cm ? 1 : 0;
}

__global__ void restrict_kernel(const __grid_constant__ RestrictBatch B, int h, int w, int hc, int wc) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hc * wc) return;
    restrict_px(B.f[blockIdx.y], B.m[blockIdx.y], B.fc[blockIdx.y], B.mc[blockIdx.y], h, w, wc, i);
}

// The small levels of the pyramid in one launch: one 8-CTA cluster per solve
// (blockIdx.y) restricts level after level, a cluster barrier between them
// (release / acquire at cluster scope: the level just written is visible to
// every CTA of the cluster).  Replaces one ~5 us latency-bound launch per level.
constexpr int kRestrictChainMax = 8;
constexpr int kRestrictCluster = 8;
constexpr int kRestrictChainMaxPx = 8192;  // coarse pixels of the largest chained level
struct RestrictChain {
    int nlev;  // restrictions: level l -> l + 1 for l < nlev
    int h[kRestrictChainMax + 1], w[kRestrictChainMax + 1];
    const double* f[kMaxBatch][kRestrictChainMax + 1];
    const uint8_t* m[kMaxBatch][kRestrictChainMax + 1];
};
__global__ void __cluster_dims__(kRestrictCluster, 1, 1) __launch_bounds__(512)
    restrict_chain_kernel(const __grid_constant__ RestrictChain C) {
    const int j = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x, nth = kRestrictCluster * blockDim.x;
    for (int l = 0; l < C.nlev; ++l) {
        const int nc = C.h[l + 1] * C.w[l + 1];
        for (int i = t; i < nc; i += nth)
            restrict_px(C.f[j][l], C.m[j][l], const_cast<double*>(C.f[j][l + 1]), const_cast<uint8_t*>(C.m[j][l + 1]),
                        C.h[l], C.w[l], C.w[l + 1], i);
        if (l + 1 < C.nlev) cooperative_groups::this_cluster().sync();
    }
}

// ---------------------------------------------------------------- CG level kernel

struct CgParams {
    int h, w, n;
    const double* f;
    const uint8_t* m;
    const double* uc;  // coarser solution (nullptr at the coarsest level)
    int hc, wc;
    double* x;
    double* r;
    double* pa;
    double* pb;
    double* ap;
    double* u;  // level solution out
    double tol;
    int max_iter;
    int finest;
    double* partials;  // [gridDim.x * 4]
    unsigned int* bar;
    int* iters;         // out: iterations of this level
    double* margin;     // out: min |sqrt(rs)-tol*bn|/(tol*bn) over stop tests (parity diagnostics)
    // band kernel: CTA b owns rows [b*band_rows, min(h, (b+1)*band_rows))
    int band_rows;
    double* ex_r;  // [nbands][2][w]: first/last owned row of r
    int x_rows = 0;  // tile: leading rows whose x lives in shared memory (the rest streams)
    // tile kernel: tiles of band_rows x tile_cols, ntc tiles per row of tiles
    int tile_cols = 0, ntc = 1;
    unsigned long long* trace = nullptr;  // diagnostics: per-iteration phase timestamps of CTA 0
    unsigned long long* stamp = nullptr;  // probe: globaltimer at kernel entry / exit (CTA 0)
};

__device__ __forceinline__ double prolong_at(const CgParams& P, int y, int xx) {
    // homogeneous.py:133-154, evaluated at one fine pixel
    double ys = ((double)y + 0.5) * ((double)P.hc / (double)P.h) - 0.5;
    double xs = ((double)xx + 0.5) * ((double)P.wc / (double)P.w) - 0.5;
    ys = fmin(fmax(ys, 0.0), (double)(P.hc - 1));
    xs = fmin(fmax(xs, 0.0), (double)(P.wc - 1));
    int y0 = (int)floor(ys), x0 = (int)floor(xs);
    int y1 = min(y0 + 1, P.hc - 1), x1 = min(x0 + 1, P.wc - 1);
    double wy = ys - (double)y0, wx = xs - (double)x0;
    const double* c = P.uc;
    double c00 = __ldg(c + (size_t)y0 * P.wc + x0), c01 = __ldg(c + (size_t)y0 * P.wc + x1);
    double c10 = __ldg(c + (size_t)y1 * P.wc + x0), c11 = __ldg(c + (size_t)y1 * P.wc + x1);
    return (1 - wy) * ((1 - wx) * c00 + wx * c01) + wy * ((1 - wx) * c10 + wx * c11);
}

// 5-point reflecting Laplacian of a field given by an accessor (homogeneous.py:27-43).
template <class G>
__device__ __forceinline__ double lap_at(int y, int xx, int h, int w, double c, G get) {
    double north = y > 0 ? get(y - 1, xx) : c;
    double south = y < h - 1 ? get(y + 1, xx) : c;
    double west = xx > 0 ? get(y, xx - 1) : c;
    double east = xx < w - 1 ? get(y, xx + 1) : c;
    return (((c * -4.0 + north) + south) + west) + east;
}

// Consecutive grid reductions alternate between two banks of partials (by
// barrier epoch): a CTA released from barrier e may already publish its
// partial for barrier e + 1 while a slower CTA still sums the partials of
// barrier e; it cannot reach barrier e + 2 (same bank) before every CTA has
// arrived at e + 1.
constexpr int kPartialBank = 2048;  // doubles per bank (<= 512 CTAs x 4 values)

template <bool kGrid, int NV>
__device__ __forceinline__ void reduce(double (&v)[NV], double* sh, const CgParams& P, unsigned int& epoch) {
    block_sum<NV>(v, sh);
    if (!kGrid) return;
    const double* part = P.partials + ((epoch + 1) & 1) * kPartialBank;  // see grid_reduce
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) const_cast<double*>(part)[blockIdx.x * 4 + k] = v[k];
    grid_barrier(P.bar, gridDim.x, epoch);
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
            for (int g = lane; g < (int)gridDim.x; g += 32) s += __ldcg(part + g * 4 + k);
            s = warp_sum(s);
            if (lane == 0) sh[k * 32] = s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = sh[k * 32];
    __syncthreads();
}

// Fixed-order sum of the n CTA partials of each of the NV values (lane l
// adds partials l, l + 32, ... in order, then warp_sum); warp k sums value k,
// and each lane issues all its loads before the first add, so the partials
// arrive in ONE L2 round trip (a runtime-bound loop took two or more).
constexpr int kSumPer = 5;  // unrolled loads per lane: n <= 160 (one CTA per SM)
template <int NV>
__device__ __forceinline__ void sum_partials(const double* part, int n, double* bc) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (wid >= NV) return;
    double s = 0.0;
    if (n <= 32 * kSumPer) {
        double vals[kSumPer];
#pragma unroll
        for (int j = 0; j < kSumPer; ++j) {
            const int g = lane + 32 * j;
            vals[j] = g < n ? __ldcg(part + g * 4 + wid) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kSumPer; ++j)
            if (lane + 32 * j < n) s += vals[j];
    } else {
        for (int g = lane; g < n; g += 32) s += __ldcg(part + g * 4 + wid);
    }
    s = warp_sum(s);
    if (lane == 0) bc[wid] = s;
}

// This CTA's partial of each value into part[0..NV): warp sums, one CTA
// barrier, then lane k of warp 0 adds the warp partials of value k in warp
// order (block_sum1's order, without every thread re-reading them).
template <int NV>
__device__ __forceinline__ void cta_partial(double (&v)[NV], double* sh, int& par, double* part) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* buf = sh + par * NV * 32;
    par ^= 1;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) buf[k * 32 + wid] = v[k];
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int i = 0; i < nw; ++i) s += buf[threadIdx.x * 32 + i];
        part[threadIdx.x] = s;
    }
    if (threadIdx.x < 32) __syncwarp();  // lanes 1..NV-1's stores before lane 0's arrival (release)
}

// Grid-wide fixed-order sum with 3 CTA barriers: cta_partial, the grid
// arrival/wait, and the broadcast of the sums over the CTA partials.
// sh: 2*4*32 (block_sum1 buffers) + 2*4 (broadcast buffers) doubles.
struct RedState {
    unsigned int epoch = 0;
    int par = 0, bpar = 0;
};
// idx / n: this CTA's slot and the number of CTAs taking part (one solve of a batch).
// Consecutive reductions alternate between two banks of partials (kPartialBank).
template <int NV>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], double* sh, const CgParams& P, RedState& st, int idx,
                                            int n) {
    double* part = P.partials + ((st.epoch + 1) & 1) * kPartialBank;
    cta_partial<NV>(v, sh, st.par, part + idx * 4);
    grid_arrive_wait(P.bar, n, st.epoch);
    double* bc = sh + 2 * 4 * 32 + st.bpar * 4;
    st.bpar ^= 1;
    sum_partials<NV>(part, n, bc);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = bc[k];
}
// grid_reduce in two halves: publish this CTA's partial and arrive; ...; wait and sum.
template <int NV>
__device__ __forceinline__ void grid_reduce_arrive(double (&v)[NV], double* sh, const CgParams& P, RedState& st,
                                                   int idx) {
    double* part = P.partials + ((st.epoch + 1) & 1) * kPartialBank;
    cta_partial<NV>(v, sh, st.par, part + idx * 4);
    grid_arrive(P.bar, st.epoch);
}
template <int NV>
__device__ __forceinline__ void grid_reduce_finish(double (&v)[NV], double* sh, const CgParams& P, RedState& st,
                                                   int n) {
    grid_wait(P.bar, n, st.epoch);
    const double* part = P.partials + (st.epoch & 1) * kPartialBank;
    double* bc = sh + 2 * 4 * 32 + st.bpar * 4;
    st.bpar ^= 1;
    sum_partials<NV>(part, n, bc);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = bc[k];
}
template <int NV>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], double* sh, const CgParams& P, RedState& st) {
    grid_reduce<NV>(v, sh, P, st, (int)blockIdx.x, (int)gridDim.x);
}

template <bool kGrid>
__global__ void __launch_bounds__(kThreads, 1) cg_level_kernel(CgParams P) {
    __shared__ double sh[4 * 32];
    __shared__ double s_mean;
    __shared__ double s_vals[kCoarsest * kCoarsest];
    unsigned int epoch = 0;
    if (P.stamp && blockIdx.x == 0 && threadIdx.x == 0) P.stamp[0] = globaltimer_ns();
    const int h = P.h, w = P.w, n = P.n;
    const int stride = gridDim.x * blockDim.x;
    const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
    const double* __restrict__ f = P.f;
    const uint8_t* __restrict__ m = P.m;

    // coarsest level: x0 = mean(f[mask]) with numpy's pairwise sum (homogeneous.py:188)
    if (P.uc == nullptr) {
        if (threadIdx.x == 0) {
            int c = 0;
            for (int i = 0; i < n; ++i)
                if (m[i]) s_vals[c++] = f[i];
            s_mean = np_pairwise_sum(s_vals, c) / (double)c;
        }
        __syncthreads();
    }
    const double mean0 = P.uc == nullptr ? s_mean : 0.0;
    auto x0_at = [&](int y, int xx) -> double { return P.uc ? prolong_at(P, y, xx) : mean0; };

    // ---- setup: x = x0*interior, b = L(u_D)*interior, r = b - A x (homogeneous.py:64-77)
    double acc[4] = {0.0, 0.0, 0.0, 0.0};  // r.r, b.b, |f_mask|^2, #interior
    for (int i = t0; i < n; i += stride) {
        int y = i / w, xx = i % w;
        bool mi = m[i] != 0;
        double interior = mi ? 0.0 : 1.0;
        auto ud = [&](int yy, int xq) -> double {
            size_t k = (size_t)yy * w + xq;
            return m[k] ? __ldg(f + k) : 0.0;
        };
        auto xv = [&](int yy, int xq) -> double {
            size_t k = (size_t)yy * w + xq;
            return x0_at(yy, xq) * (m[k] ? 0.0 : 1.0);
        };
        double udi = mi ? __ldg(f + i) : 0.0;
        double xi = x0_at(y, xx) * interior;
        double b = lap_at(y, xx, h, w, udi, ud) * interior;
        double ax = -lap_at(y, xx, h, w, xi, xv) * interior;
        double ri = b - ax;
        P.x[i] = xi;
        P.r[i] = ri;
        P.pa[i] = ri;
        acc[0] += ri * ri;
        acc[1] += b * b;
        acc[2] += mi ? udi * udi : 0.0;
        acc[3] += interior;
    }
    reduce<kGrid, 4>(acc, sh, P, epoch);
    double rs = acc[0];
    double bn;
    bool all_mask = acc[3] == 0.0;
    if (P.finest && acc[2] != 0.0)
        bn = sqrt(acc[2]);  // ||f restricted to mask|| (homogeneous.py:198)
    else
        bn = sqrt(acc[1]);  // ||b||
    int it = 0;
    double margin = 1e300;
    double* pold = P.pa;
    double* pnew = P.pb;
    if (!all_mask && bn != 0.0) {
        double beta = 0.0;  // first iteration: p = r
        for (int k = 1; k <= P.max_iter; ++k) {
            it = k;
            // phase 1: p = r + beta p (fused), ap = -L(p)*interior, p.ap
            double d[1] = {0.0};
            for (int i = t0; i < n; i += stride) {
                int y = i / w, xx = i % w;
                auto pv = [&](int yy, int xq) -> double {
                    size_t q = (size_t)yy * w + xq;
                    return __ldcg(P.r + q) + beta * __ldcg(pold + q);
                };
                double pi = pv(y, xx);
                double interior = m[i] ? 0.0 : 1.0;
                double api = -lap_at(y, xx, h, w, pi, pv) * interior;
                pnew[i] = pi;
                P.ap[i] = api;
                d[0] += pi * api;
            }
            reduce<kGrid, 1>(d, sh, P, epoch);
            double pap = d[0];
            if (pap <= 0.0 || rs < 1e-300) break;
            double alpha = rs / pap;
            // phase 2: x += alpha p, r -= alpha ap, r.r
            double e[1] = {0.0};
            for (int i = t0; i < n; i += stride) {
                double pi = pnew[i];
                double xi = P.x[i] + alpha * pi;
                double ri = __ldcg(P.r + i) - alpha * P.ap[i];
                P.x[i] = xi;
                P.r[i] = ri;
                e[0] += ri * ri;
            }
            reduce<kGrid, 1>(e, sh, P, epoch);
            double rs1 = e[0];
            double lhs = sqrt(rs1), rhs = P.tol * bn;
            if (rhs > 0.0) margin = fmin(margin, fabs(lhs - rhs) / rhs);
            if (lhs <= rhs) break;
            beta = rs1 / rs;
            rs = rs1;
            double* t = pold;
            pold = pnew;
            pnew = t;
        }
    }
    // level solution: u = u_D + x (or a copy of f when the mask is full)
    for (int i = t0; i < n; i += stride) {
        bool mi = m[i] != 0;
        double udi = mi ? __ldg(f + i) : 0.0;
        P.u[i] = all_mask ? __ldg(f + i) : udi + P.x[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *P.iters = it;
        if (P.margin) *P.margin = margin;
        if (P.stamp) P.stamp[1] = globaltimer_ns();
    }
}

#include "cg_setup.cuh"
#include "cg_tile.cuh"
#include "cg_cluster.cuh"
#include "cg_cluster_col.cuh"

// ---------------------------------------------------------------- strict residual check

__global__ void residual_partials(const double* __restrict__ u, const double* __restrict__ f,
                                  const uint8_t* __restrict__ m, int h, int w, double* partials) {
    __shared__ double sh[2 * 32];
    double acc[2] = {0.0, 0.0};
    int n = h * w;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int y = i / w, xx = i % w;
        double res;
        if (m[i]) {
            res = u[i] - f[i];
            acc[1] += f[i] * f[i];
        } else {
            res = lap_at(y, xx, h, w, u[i], [&](int yy, int xq) { return u[(size_t)yy * w + xq]; });
        }
        acc[0] += res * res;
    }
    block_sum<2>(acc, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x * 2] = acc[0];
        partials[blockIdx.x * 2 + 1] = acc[1];
    }
}

// ---------------------------------------------------------------- host side

void pyramid_shapes(int h, int w, std::vector<std::pair<int, int>>& shapes) {
    shapes.clear();
    shapes.push_back({h, w});
    while (std::max(shapes.back().first, shapes.back().second) > kCoarsest) {
        auto s = shapes.back();
        shapes.push_back({(s.first + 1) / 2, (s.second + 1) / 2});
    }
}

void InpaintWorkspace::reserve(int h, int w, int dev) {
    size_t n = (size_t)h * w;
    if (n <= cap_px && (size_t)w <= cap_w && dev == device) return;
    release();
    device = dev;
    cudaDeviceProp prop;
    CUDA_CHECK(cudaGetDeviceProperties(&prop, dev));
    num_sms = prop.multiProcessorCount;
    int occ = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cg_level_kernel<true>, kThreads, 0));
    grid_ctas = occ >= 1 ? num_sms : 0;
    // finest-level vectors + every coarser level's f, m, u
    std::vector<std::pair<int, int>> shapes;
    pyramid_shapes(h, w, shapes);
    size_t coarse = 0;
    for (size_t l = 1; l < shapes.size(); ++l) coarse += (size_t)shapes[l].first * shapes[l].second;
    size_t nd = 5 * n + 2 * coarse + n /* u of level 0 scratch */;
    CUDA_CHECK(cudaMalloc(&dbl, nd * sizeof(double)));
    CUDA_CHECK(cudaMalloc(&bytes, coarse + 64));
    // CG partials (grid_ctas x 4) and the strict-residual partials (<= 1024 blocks x 2)
    // [0, 4096): band-setup partials at 4096 (kSetupCtas x 4)
    CUDA_CHECK(cudaMalloc(&partials, (size_t)(4096 + kSetupCtas * 4 + 64) * sizeof(double)));
    CUDA_CHECK(cudaMalloc(&bar, 64 * sizeof(unsigned int)));
    CUDA_CHECK(cudaMemset(bar, 0, 64 * sizeof(unsigned int)));
    CUDA_CHECK(cudaMalloc(&iters, 64 * sizeof(int)));
    CUDA_CHECK(cudaMalloc(&margins, 64 * sizeof(double)));
    // tile-kernel edge exchange: r + 2 parities of p, every tile's perimeter
    ex_cap = (size_t)3 * std::max(num_sms, 1) * (2 * (size_t)kTileCols + 2 * (size_t)kTileRows);
    CUDA_CHECK(cudaMalloc(&ex, ex_cap * sizeof(double)));
    cap_px = n;
    cap_w = w;
    cap_coarse = coarse;
    for (TileKernelFn fn : {tile_kernel_for(30, 480), tile_kernel_for(23, 480), tile_kernel_for(15, 480),
                            tile_kernel_for(0, 0)})
        CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem));
    // 16-CTA clusters (non-portable size) for the coarse/mid levels, when this device can host one
    cluster_ok = cudaFuncSetAttribute(cg_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                     cudaSuccess &&
                 cudaFuncSetAttribute(cg_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ==
                     cudaSuccess;
    if (cluster_ok) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kClusterSize);
        cfg.blockDim = dim3(kClThreads);
        cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kClusterSize;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        cluster_ok = cudaOccupancyMaxActiveClusters(&nclusters, cg_cluster_kernel, &cfg) == cudaSuccess && nclusters > 0;
    }
    if (cluster_ok)
        cluster_ok = cudaFuncSetAttribute(cg_cluster_col_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                         cudaSuccess &&
                     cudaFuncSetAttribute(cg_cluster_col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          200 * 1024) == cudaSuccess;
    cudaGetLastError();  // clear a rejected attribute
}

void InpaintWorkspace::release() {
    if (dbl) cudaFree(dbl);
    if (bytes) cudaFree(bytes);
    if (partials) cudaFree(partials);
    if (bar) cudaFree(bar);
    if (iters) cudaFree(iters);
    if (margins) cudaFree(margins);
    if (ex) cudaFree(ex);
    ex = nullptr;
    dbl = nullptr;
    bytes = nullptr;
    partials = nullptr;
    bar = nullptr;
    iters = nullptr;
    margins = nullptr;
    cap_px = 0;
}

int solve_homogeneous_async(InpaintWorkspace& ws, cudaStream_t s, const double* f, const uint8_t* m, int h, int w,
                            double tol, int max_iter, double* u_out, int64_t* launches, CgProbe* probe) {
    SolveJob job{&ws, f, m, u_out};
    return solve_batch_async(&job, 1, h, w, tol, max_iter, s, launches, probe);
}

namespace {

// 2-D tile layout of a grid level for cg_tile_kernel: at most `budget` tiles
// of <= kTileRows rows x <= 512 columns, p + as many x rows as fit in smem.
struct TilePlan {
    bool ok = false;
    int trows = 0, tcols = 0, ntc = 0, nt = 0, xr = 0;
    size_t smem = 0, ex = 0;  // dynamic smem bytes, exchange doubles (the tiles' r edges)
};
TilePlan plan_tiles(int h, int w, int budget) {
    TilePlan T;
    const int tc = (w + kTileThreads - 1) / kTileThreads;
    const int tcols = (w + tc - 1) / tc;
    const int tr_max = budget / tc;
    if (tr_max < 1) return T;
    const int trows = (h + tr_max - 1) / tr_max;
    if (trows > kTileRows || trows < 1) return T;
    const int ntr = (h + trows - 1) / trows;
    const size_t p_bytes = (size_t)(trows + 2) * (tcols + 2) * sizeof(double);
    if (p_bytes > (size_t)kTileSmem) return T;
    const int xr = (int)std::min<size_t>((size_t)trows, ((size_t)kTileSmem - p_bytes) / ((size_t)tcols * sizeof(double)));
    T.ok = true;
    T.trows = trows;
    T.tcols = tcols;
    T.ntc = tc;
    T.nt = ntr * tc;
    T.xr = xr;
    T.smem = p_bytes + (size_t)xr * tcols * sizeof(double);
    T.ex = (size_t)T.nt * (2 * (size_t)tcols + 2 * (size_t)trows);
    return T;
}

// Per-job views of its workspace: finest CG vectors + every level's f, m, u.
struct JobLevels {
    double* x;
    double* r;
    double* pa;
    double* pb;
    double* ap;
    std::vector<const double*> f;
    std::vector<const uint8_t*> m;
    std::vector<double*> u;
};

CgParams level_params(const JobLevels& J, InpaintWorkspace& ws, const std::vector<std::pair<int, int>>& shapes, int l,
                      double tol, int max_iter) {
    const int L = (int)shapes.size();
    CgParams P{};
    P.h = shapes[l].first;
    P.w = shapes[l].second;
    P.n = P.h * P.w;
    P.f = J.f[l];
    P.m = J.m[l];
    P.uc = l == L - 1 ? nullptr : J.u[l + 1];
    P.hc = l == L - 1 ? 0 : shapes[l + 1].first;
    P.wc = l == L - 1 ? 0 : shapes[l + 1].second;
    P.x = J.x;
    P.r = J.r;
    P.pa = J.pa;
    P.pb = J.pb;
    P.ap = J.ap;
    P.u = J.u[l];
    P.tol = l == 0 ? tol : std::max(kLevelTol, tol);
    P.max_iter = max_iter;
    P.finest = l == 0;
    P.partials = ws.partials;
    P.bar = ws.bar;
    P.iters = ws.iters + (L - 1 - l);
    P.margin = ws.margins + (L - 1 - l);
    return P;
}

}  // namespace

int solve_batch_async(const SolveJob* jobs, int K, int h, int w, double tol, int max_iter, cudaStream_t s,
                      int64_t* launches, CgProbe* probe, cudaStream_t s_pre) {
    if (K < 1 || K > kMaxBatch) fail(HIVC_E_ARGUMENT, "solve batch size out of range");
    InpaintWorkspace& ws0 = *jobs[0].ws;
    // pyramid + cluster/single-CTA levels never wait on other CTAs' progress
    // across launches, so they may run on a side stream next to another
    // batch's grid-barrier levels; the grid levels stay on s
    const cudaStream_t sp = s_pre ? s_pre : s;
    std::vector<bool> recorded(K, false);
    std::vector<std::pair<int, int>> shapes;
    pyramid_shapes(h, w, shapes);
    const int L = (int)shapes.size();
    const size_t n0 = (size_t)h * w;
    std::vector<JobLevels> J(K);
    for (int j = 0; j < K; ++j) {
        InpaintWorkspace& ws = *jobs[j].ws;
        JobLevels& V = J[j];
        V.x = ws.dbl;
        V.r = V.x + n0;
        V.pa = V.r + n0;
        V.pb = V.pa + n0;
        V.ap = V.pb + n0;
        double* cur = V.ap + n0;  // coarse f / u storage
        uint8_t* cm = ws.bytes;
        V.f.assign(L, nullptr);
        V.m.assign(L, nullptr);
        V.u.assign(L, nullptr);
        V.f[0] = jobs[j].f;
        V.m[0] = jobs[j].m;
        V.u[0] = jobs[j].u;
        for (int l = 1; l < L; ++l) {
            const size_t nl = (size_t)shapes[l].first * shapes[l].second;
            V.f[l] = cur;
            cur += nl;
            V.u[l] = cur;
            cur += nl;
            V.m[l] = cm;
            cm += nl;
        }
    }
    const bool bt = probe && debug_opt("batch_trace");
    auto mb = [&](const std::string& label, cudaStream_t st) {
        if (bt) probe->mark_begin(st, label + " K=" + std::to_string(K) + " " + std::to_string(h) + "x" + std::to_string(w));
    };
    auto me = [&](cudaStream_t st) {
        if (bt) probe->mark_end(st);
    };
    // ---- pyramid (homogeneous.py:96-130): one launch per level for the whole batch
    mb("restrict", sp);
    int l_chain = L;  // levels >= l_chain - 1 restricted by the chained cluster launch
    while (l_chain - 1 >= 1 && L - (l_chain - 1) <= kRestrictChainMax &&
           (size_t)shapes[l_chain - 1].first * shapes[l_chain - 1].second <= (size_t)kRestrictChainMaxPx)
        --l_chain;
    if (L - l_chain < 2) l_chain = L;  // a single small level: the plain launch
    for (int l = 1; l < l_chain; ++l) {
        RestrictBatch RB{};
        for (int j = 0; j < K; ++j) {
            RB.f[j] = J[j].f[l - 1];
            RB.m[j] = J[j].m[l - 1];
            RB.fc[j] = const_cast<double*>(J[j].f[l]);
            RB.mc[j] = const_cast<uint8_t*>(J[j].m[l]);
        }
        const size_t nl = (size_t)shapes[l].first * shapes[l].second;
        restrict_kernel<<<dim3((unsigned)((nl + 255) / 256), K), 256, 0, sp>>>(
            RB, shapes[l - 1].first, shapes[l - 1].second, shapes[l].first, shapes[l].second);
        ++*launches;
    }
    if (l_chain < L) {
        RestrictChain RC{};
        RC.nlev = L - l_chain;
        for (int q = 0; q <= RC.nlev; ++q) {
            RC.h[q] = shapes[l_chain - 1 + q].first;
            RC.w[q] = shapes[l_chain - 1 + q].second;
            for (int j = 0; j < K; ++j) {
                RC.f[j][q] = J[j].f[l_chain - 1 + q];
                RC.m[j][q] = J[j].m[l_chain - 1 + q];
            }
        }
        restrict_chain_kernel<<<dim3(kRestrictCluster, K), 512, 0, sp>>>(RC);
        ++*launches;
    }
    me(sp);
    CUDA_CHECK(cudaGetLastError());
    const int first_solve = probe ? (int)probe->solves.size() : 0;
    // ---- coarse and mid levels: one cluster per solve (levels whose 16 row
    // bands fit on chip), else one single-CTA launch per solve for the tiny ones
    int l_start = L - 1;
    if (ws0.cluster_ok) {
        ClusterBatch CB{};
        size_t smem = 0;
        int nlev = 0;
        int l = L - 1;
        while (l >= 0 && nlev < kClMaxLevels) {
            const int hh = shapes[l].first, ww = shapes[l].second;
            const int br = (hh + kClusterSize - 1) / kClusterSize;
            const size_t need =
                ((size_t)(br + 2) * (ww + 2) + (size_t)br * ww + 6 * (size_t)ww) * sizeof(double) + (size_t)br * ww;
            if ((size_t)br * ww > (size_t)kClPx * kClThreads || ww > kClMaxW || need > 200 * 1024) break;
            for (int j = 0; j < K; ++j) {
                ClusterLevels& S = CB.S[j];
                S.h[nlev] = hh;
                S.w[nlev] = ww;
                S.f[nlev] = J[j].f[l];
                S.m[nlev] = J[j].m[l];
                S.u[nlev] = J[j].u[l];
                S.iters[nlev] = jobs[j].ws->iters + (L - 1 - l);
            }
            ++nlev;
            smem = std::max(smem, need);
            --l;
        }
        if (nlev > 0) {
            for (int j = 0; j < K; ++j) {
                ClusterLevels& S = CB.S[j];
                S.nlev = nlev;
                S.uc0 = nullptr;
                S.last_is_finest = l < 0;
                S.tol = tol;
                S.max_iter = max_iter;
                S.trace = nullptr;
            }
            if (debug_opt("cg_trace_cluster") && K == 1) {
                if (!ws0.trace) CUDA_CHECK(cudaMalloc(&ws0.trace, kTraceLen * sizeof(unsigned long long)));
                CUDA_CHECK(cudaMemsetAsync(ws0.trace, 0, kTraceLen * sizeof(unsigned long long), sp));
                CB.S[0].trace = ws0.trace;
            }
            // column-walk variant when every band is <= kColRows x kClThreads
            bool col = true;
            for (int i = 0; i < nlev && col; ++i)
                col = CB.S[0].w[i] <= kClThreads && (CB.S[0].h[i] + kClusterSize - 1) / kClusterSize <= kColRows;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(kClusterSize * K);
            cfg.blockDim = dim3(kClThreads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = sp;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = kClusterSize;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            mb("cluster nlev=" + std::to_string(nlev), sp);
            if (col)
                CUDA_CHECK(cudaLaunchKernelEx(&cfg, cg_cluster_col_kernel, CB));
            else
                CUDA_CHECK(cudaLaunchKernelEx(&cfg, cg_cluster_kernel, CB));
            me(sp);
            ++*launches;
            l_start = l;
        }
    }
    if (sp != s) {  // the grid levels (and the caller's next work on s) follow the side-stream levels
        if (!ws0.pre_done) CUDA_CHECK(cudaEventCreateWithFlags(&ws0.pre_done, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventRecord(ws0.pre_done, sp));
        CUDA_CHECK(cudaStreamWaitEvent(s, ws0.pre_done, 0));
    }
    // ---- remaining (large) levels
    for (int l = l_start; l >= 0; --l) {
        std::vector<CgParams> P(K);
        for (int j = 0; j < K; ++j) P[j] = level_params(J[j], *jobs[j].ws, shapes, l, tol, max_iter);
        const int hh = P[0].h, ww = P[0].w;
        const bool grid = !(P[0].n <= kSingleCtaMaxPx || ws0.grid_ctas == 0);
        // on-chip 2-D tile kernel (every level above the cluster levels of the
        // benchmark pyramids); packed solves share the SMs, at most 4 side by
        // side (a lone solve gets the whole GPU); other shapes: the streaming
        // grid kernel, or one CTA for the small ones
        const int kc = (ww + kTileCols - 1) / kTileCols;
        const int waves = (K + 3) / 4;
        const int side = (K + waves - 1) / waves;  // even waves: 5 solves -> 3 + 2, not 4 + 1
        const bool pack_t = ws0.pack_bands && kc <= 2 && side > 1;
        const TilePlan TP = plan_tiles(hh, ww, pack_t ? ws0.num_sms / side : ws0.num_sms);
        const bool tile = grid && P[0].uc != nullptr && TP.ok && TP.ex <= ws0.ex_cap;
        CgProbe::Launch rec{};
        if (probe && grid) {
            rec.stamp_base = probe->next_stamp;
            probe->next_stamp += K;
            for (int j = 0; j < K; ++j) P[j].stamp = probe->stamp_slot(rec.stamp_base + j);
        }
        auto rec_begin = [&]() {
            if (!(probe && grid)) return;
            CUDA_CHECK(cudaEventCreate(&rec.start));
            CUDA_CHECK(cudaEventCreate(&rec.stop));
            CUDA_CHECK(cudaEventRecord(rec.start, s));
        };
        if (!grid) {
            rec_begin();
            for (int j = 0; j < K; ++j) {
                cg_level_kernel<false><<<1, kThreads, 0, s>>>(P[j]);
                ++*launches;
            }
        } else if (tile) {
            SetupBatch SB{};
            TileBatch TB{};
            const size_t E = 2 * (size_t)TP.tcols + 2 * (size_t)TP.trows;
            for (int j = 0; j < K; ++j) {
                InpaintWorkspace& ws = *jobs[j].ws;
                P[j].band_rows = TP.trows;
                P[j].tile_cols = TP.tcols;
                P[j].ntc = TP.ntc;
                P[j].x_rows = TP.xr;
                P[j].ex_r = ws.ex;
                SB.P[j] = P[j];
                SB.partials[j] = ws.partials + 4096;
                TB.P[j] = P[j];
                TB.setup[j] = ws.partials + 4096;
            }
            if (debug_opt("cg_trace") && l == 0 && K == 1) {
                if (!ws0.trace) CUDA_CHECK(cudaMalloc(&ws0.trace, kTraceLen * sizeof(unsigned long long)));
                CUDA_CHECK(cudaMemsetAsync(ws0.trace, 0, kTraceLen * sizeof(unsigned long long), s));
                SB.P[0].trace = TB.P[0].trace = ws0.trace;
            }
            unsigned int* ticket = ws0.bar + 32;
            const bool ticketed = pack_t && K > 1;
            SB.ticket = ticketed ? ticket : nullptr;
            mb("setup l=" + std::to_string(l), s);
            cg_setup_x_kernel<<<dim3((unsigned)(ww + 255) / 256, (unsigned)(hh + kSetupXRows - 1) / kSetupXRows, K), 256, 0, s>>>(SB);
            cg_setup_kernel<<<dim3(kSetupCtas, K), 512, 0, s>>>(SB);
            me(s);
            *launches += 2;
            mb(std::string(ticketed ? "tile-ticket" : "tile-coop") + " l=" + std::to_string(l) + " nt=" +
                   std::to_string(TP.nt) + " " + std::to_string(TP.trows) + "x" + std::to_string(TP.tcols),
               s);
            rec_begin();
            TB.nt = TP.nt;
            if (ticketed) {
                TB.ticket = ticket;
                tile_kernel_for(TP.trows, TP.tcols)<<<TP.nt * K, kTileThreads,
                                                            TP.smem, s>>>(TB);
                ++*launches;
            } else {
                for (int j = 0; j < K; ++j) {
                    TileBatch one{};
                    one.P[0] = TB.P[j];
                    one.setup[0] = TB.setup[j];
                    one.nt = TP.nt;
                    one.ticket = nullptr;
                    void* args[] = {&one};
                    CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)tile_kernel_for(TP.trows, TP.tcols),
                                                           dim3(TP.nt),
                                                           dim3(kTileThreads), args,
                                                           TP.smem, s));
                    ++*launches;
                    if (l == 0 && jobs[j].done) {
                        CUDA_CHECK(cudaEventRecord(jobs[j].done, s));
                        recorded[j] = true;
                    }
                }
            }
        } else {
            rec_begin();
            for (int j = 0; j < K; ++j) {
                CUDA_CHECK(cudaMemsetAsync(jobs[j].ws->bar, 0, sizeof(unsigned int), s));  // barrier epoch counter
                void* args[] = {&P[j]};
                CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)cg_level_kernel<true>, dim3(ws0.grid_ctas),
                                                       dim3(kThreads), args, 0, s));
                ++*launches;
            }
        }
        CUDA_CHECK(cudaGetLastError());
        if (tile) me(s);
        if (probe && grid) {
            CUDA_CHECK(cudaEventRecord(rec.stop, s));
            rec.pixels = P[0].n;
            rec.first_solve = first_solve;
            rec.nsolves = K;
            rec.level = L - 1 - l;
            probe->launches.push_back(rec);
        }
    }
    for (int j = 0; j < K; ++j)
        if (jobs[j].done && !recorded[j]) CUDA_CHECK(cudaEventRecord(jobs[j].done, s));
    if (probe) {
        // per-level iteration counts of each solve, read back after the stream syncs
        for (int j = 0; j < K; ++j) {
            CgProbe::Solve sv;
            sv.nlevels = L;
            for (int l = 0; l < L; ++l) sv.pixels[l] = (int64_t)shapes[L - 1 - l].first * shapes[L - 1 - l].second;
            sv.host_iters = probe->alloc_iters();
            if (sv.host_iters)
                CUDA_CHECK(cudaMemcpyAsync(sv.host_iters, jobs[j].ws->iters, L * sizeof(int), cudaMemcpyDeviceToHost, s));
            probe->solves.push_back(sv);
        }
    }
    return L;
}

// out[k] = w[pts[k]] - sum of z over the existing 4-neighbours of pts[k]
// (z is zero on the mask): the mask rows of A^T z = w solved for z_M once
// z_I is known (A = diag(d) + diag(1 - d) L, L the reflecting graph Laplacian).
__global__ void mask_adjoint_kernel(const double* __restrict__ w_full, const double* __restrict__ z,
                                    const int32_t* __restrict__ pts, int npts, int h, int w, double* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= npts) return;
    const int p = pts[k], y = p / w, x = p - y * w;
    double s = 0.0;  // neighbours in the order of the sparse row (north, south, west, east)
    if (y > 0) s += z[p - w];
    if (y < h - 1) s += z[p + w];
    if (x > 0) s += z[p - 1];
    if (x < w - 1) s += z[p + 1];
    out[k] = w_full[p] - s;
}

int solve_poisson_interior(InpaintWorkspace& ws, cudaStream_t s, const double* rhs, const uint8_t* m, int h, int w,
                           double tol, int max_iter, double* z_out, int64_t* launches) {
    // single level, x0 = 0; the level kernel writes u = (mask ? f : 0) + x with f = 0
    const size_t n = (size_t)h * w;
    double* x = ws.dbl;
    double* r = x + n;
    double* zero_f = r + 3 * n;  // (the ap slot: unused by the tile kernel) zeroed as f
    CUDA_CHECK(cudaMemsetAsync(zero_f, 0, n * sizeof(double), s));
    CgParams P{};
    P.h = h;
    P.w = w;
    P.n = (int)n;
    P.f = zero_f;
    P.m = m;
    P.uc = nullptr;
    P.x = x;
    P.r = r;
    P.pa = r + n;
    P.pb = r + 2 * n;
    P.ap = zero_f;
    P.u = z_out;
    P.tol = tol;
    P.max_iter = max_iter;
    P.finest = 0;  // denominator ||b||
    P.partials = ws.partials;
    P.bar = ws.bar;
    P.iters = ws.iters;
    P.margin = ws.margins;
    const TilePlan TP = plan_tiles(h, w, ws.num_sms);
    if (!TP.ok || TP.ex > ws.ex_cap) fail(HIVC_E_ARGUMENT, "plane shape not supported by the interior solver");
    const size_t E = 2 * (size_t)TP.tcols + 2 * (size_t)TP.trows;
    P.band_rows = TP.trows;
    P.tile_cols = TP.tcols;
    P.ntc = TP.ntc;
    P.x_rows = TP.xr;
    P.ex_r = ws.ex;
    double* setup = ws.partials + 4096;
    cg_setup_rhs_kernel<<<kSetupCtas, 512, 0, s>>>(P, rhs, setup);
    TileBatch one{};
    one.P[0] = P;
    one.setup[0] = setup;
    one.nt = TP.nt;
    one.ticket = nullptr;
    void* args[] = {&one};
    CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)tile_kernel_for(TP.trows, TP.tcols), dim3(TP.nt),
                                           dim3(kTileThreads), args,
                                           TP.smem, s));
    *launches += 3;
    CUDA_CHECK(cudaGetLastError());
    int it = 0;
    CUDA_CHECK(cudaMemcpyAsync(&it, ws.iters, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    return it;
}

void launch_mask_adjoint(const double* w_full, const double* z, const int32_t* pts, int npts, int h, int w, double* out,
                         cudaStream_t s) {
    if (npts <= 0) return;
    mask_adjoint_kernel<<<(npts + 255) / 256, 256, 0, s>>>(w_full, z, pts, npts, h, w, out);
    CUDA_CHECK(cudaGetLastError());
}

int* CgProbe::alloc_iters() {
    if (!host) {
        if (cudaHostAlloc(&host, kCap * 32 * sizeof(int), cudaHostAllocDefault) != cudaSuccess) host = nullptr;
    }
    if (!host || used >= kCap) return nullptr;
    return host + 32 * used++;
}

unsigned long long* CgProbe::stamp_slot(int i) {
    if (!stamps_dev) {
        if (cudaMalloc(&stamps_dev, kStampCap * 2 * sizeof(unsigned long long)) != cudaSuccess) stamps_dev = nullptr;
        if (stamps_dev) cudaMemset(stamps_dev, 0, kStampCap * 2 * sizeof(unsigned long long));
    }
    if (!stamps_dev || i >= kStampCap) return nullptr;
    return stamps_dev + 2 * i;
}

void CgProbe::mark_begin(cudaStream_t s, const std::string& label) {
    Mark m{label, nullptr, nullptr};
    CUDA_CHECK(cudaEventCreate(&m.a));
    CUDA_CHECK(cudaEventCreate(&m.b));
    CUDA_CHECK(cudaEventRecord(m.a, s));
    marks.push_back(m);
}

void CgProbe::mark_end(cudaStream_t s) { CUDA_CHECK(cudaEventRecord(marks.back().b, s)); }

void CgProbe::reset() {
    for (auto& m : marks) {
        cudaEventDestroy(m.a);
        cudaEventDestroy(m.b);
    }
    marks.clear();
    for (auto& l : launches) {
        if (l.start) cudaEventDestroy(l.start);
        if (l.stop) cudaEventDestroy(l.stop);
    }
    launches.clear();
    solves.clear();
    used = 0;
    next_stamp = 0;
}

CgProbe::~CgProbe() {
    reset();
    if (host) cudaFreeHost(host);
    if (stamps_dev) cudaFree(stamps_dev);
}

void CgProbe::harvest(CgTotals& t) {
    if (!marks.empty()) {
        float t0 = 0;
        for (auto& m : marks) {
            float a = 0, d = 0;
            cudaEventElapsedTime(&a, marks[0].a, m.a);
            cudaEventElapsedTime(&d, m.a, m.b);
            std::fprintf(stderr, "[batch] %-28s start %9.1f us  dur %8.1f us\n", m.label.c_str(), a * 1e3, d * 1e3);
            t0 = a;
        }
        (void)t0;
    }
    // after the stream synchronised: accumulate iteration-weighted pixel counts
    // and the grid-mode launches' device time
    std::vector<int> it_of_solve_level;
    if (!marks.empty())
        for (const Solve& sv : solves) {  // level iterations per solve, coarsest first
            std::string line = "[batch] solve " + std::to_string(sv.pixels[0]) + " px levels:";
            for (int l = 0; l < sv.nlevels; ++l) line += " " + std::to_string(sv.host_iters ? sv.host_iters[l] : -1);
            std::fprintf(stderr, "%s\n", line.c_str());
        }
    for (const Solve& sv : solves) {
        t.solves += 1;
        for (int l = 0; l < sv.nlevels; ++l) {
            int it = sv.host_iters ? sv.host_iters[l] : 0;
            t.pixel_iters += sv.pixels[l] * it;
            t.pixel_levels += sv.pixels[l];
        }
    }
    // in-kernel globaltimer stamps give the kernel's own duration; the stream
    // events around a cooperative launch also contain time spent queued
    // behind other lanes' kernels, so they are only the fallback
    std::vector<unsigned long long> st;
    if (stamps_dev && !launches.empty()) {
        st.resize(2 * std::min<size_t>(next_stamp, kStampCap));
        cudaMemcpy(st.data(), stamps_dev, st.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        cudaMemset(stamps_dev, 0, st.size() * sizeof(unsigned long long));
    }
    for (size_t i = 0; i < launches.size(); ++i) {
        const Launch& l = launches[i];
        // span of the launch: first solve's entry to last solve's exit
        unsigned long long t0 = ~0ull, t1 = 0;
        bool ok = true;
        for (int j = 0; j < l.nsolves; ++j) {
            const size_t k = 2 * (size_t)(l.stamp_base + j);
            if (k + 1 >= st.size() || !st[k] || st[k + 1] <= st[k]) {
                ok = false;
                break;
            }
            t0 = std::min(t0, st[k]);
            t1 = std::max(t1, st[k + 1]);
        }
        float ms = 0;
        if (ok && l.nsolves > 0)
            ms = (float)((t1 - t0) * 1e-6);
        else
            cudaEventElapsedTime(&ms, l.start, l.stop);
        t.grid_launches += 1;
        t.grid_seconds += ms * 1e-3;
        for (int j = 0; j < l.nsolves; ++j) {
            const Solve& sv = solves[l.first_solve + j];
            const int it = sv.host_iters ? sv.host_iters[l.level] : 0;
            t.grid_pixel_iters += l.pixels * it;
            t.grid_pixels += l.pixels;
        }
    }
    reset();
}

double strict_relative_residual(InpaintWorkspace& ws, cudaStream_t s, const double* u, const double* f,
                                const uint8_t* m, int h, int w, int64_t* launches) {
    int nb = std::min(1024, (h * w + 255) / 256);
    residual_partials<<<nb, 256, 0, s>>>(u, f, m, h, w, ws.partials);
    ++*launches;
    CUDA_CHECK(cudaGetLastError());
    std::vector<double> host((size_t)nb * 2);
    CUDA_CHECK(cudaMemcpyAsync(host.data(), ws.partials, host.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    double rr = 0.0, ff = 0.0;
    for (int b = 0; b < nb; ++b) {
        rr += host[2 * b];
        ff += host[2 * b + 1];
    }
    double den = std::sqrt(ff);
    double num = std::sqrt(rr);
    // homogeneous.py:206-211
    return den > 0 ? num / den : -1.0;
}

}  // namespace hivc
