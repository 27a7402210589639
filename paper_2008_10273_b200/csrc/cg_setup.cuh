// Level setup for the tile CG kernel (included by inpaint.cu): x = x0 *
// interior, r = b - A x in global memory and the per-CTA partials of r.r,
// b.b, |f_mask|^2 and #interior (homogeneous.py:64-77), which the level kernel
// sums in a fixed order.  Batched: blockIdx.y = solve.
#pragma once

// Optional phase timestamps of CTA 0 / thread 0 (HIVC_CG_TRACE=1, diagnostics only).
#define HIVC_TRACE(slot)                                                                      \
    do {                                                                                      \
        if (P.trace && band == 0 && tid == 0 && k < 256) P.trace[k * 8 + (slot)] = globaltimer_ns(); \
    } while (0)

constexpr int kSetupCtas = 296;
constexpr int kTileSmem = 224 * 1024;  // tile kernel dynamic smem cap (+ 2.1 KB static <= the 227 KB opt-in limit)

struct SetupBatch {
    CgParams P[kMaxBatch];
    double* partials[kMaxBatch];
    unsigned int* ticket;  // reset with the solves' barrier counters (nullable)
};

// setup pass 1: x = x0 * interior, x0 prolonged from the coarser level (homogeneous.py:71)
__global__ void __launch_bounds__(512) cg_setup_x_kernel(const __grid_constant__ SetupBatch B) {
    const CgParams& P = B.P[blockIdx.y];
    const int w = P.w, n = P.n;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // the band launch that follows starts a fresh barrier epoch
        P.bar[0] = 0;
        if (blockIdx.y == 0 && B.ticket) *B.ticket = 0;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        P.x[i] = prolong_at(P, i / w, i % w) * (P.m[i] ? 0.0 : 1.0);
}

// Poisson mode (LSQR adjoint, prediction.optimize_mask_values): x = 0,
// r = b = -rhs on the interior (zero on the mask) and the level partials
// (r.r, b.b, 0, #interior), so the level kernel solves (-L_II) x = -rhs_I,
// i.e. L_II x = rhs_I with zero values held on the mask.
__global__ void __launch_bounds__(512) cg_setup_rhs_kernel(CgParams P, const double* __restrict__ rhs,
                                                           double* partials) {
    __shared__ double sh[4 * 32];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (blockIdx.x == 0 && threadIdx.x == 0) P.bar[0] = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        const bool mi = P.m[i] != 0;
        const double b = mi ? 0.0 : -__ldg(rhs + i);
        P.x[i] = 0.0;
        P.r[i] = b;
        acc[0] += b * b;
        acc[1] += b * b;
        acc[3] += mi ? 0.0 : 1.0;
    }
    block_sum<4>(acc, sh);
    if (threadIdx.x == 0)
        for (int k = 0; k < 4; ++k) partials[blockIdx.x * 4 + k] = acc[k];
}

// setup pass 2: b = L(u_D) * interior, r = b - A x and the level partials
__global__ void __launch_bounds__(512) cg_setup_kernel(const __grid_constant__ SetupBatch B) {
    __shared__ double sh[4 * 32];
    const CgParams& P = B.P[blockIdx.y];
    double* partials = B.partials[blockIdx.y];
    const int h = P.h, w = P.w, n = P.n;
    const double* __restrict__ f = P.f;
    const uint8_t* __restrict__ m = P.m;
    const double* __restrict__ xg = P.x;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int y = i / w, xx = i % w;
        bool mi = m[i] != 0;
        double interior = mi ? 0.0 : 1.0;
        auto ud = [&](int yy, int xq) -> double {
            size_t k = (size_t)yy * w + xq;
            return m[k] ? __ldg(f + k) : 0.0;
        };
        auto xv = [&](int yy, int xq) -> double { return xg[(size_t)yy * w + xq]; };
        double udi = mi ? __ldg(f + i) : 0.0;
        double xi = xg[i];
        double b = lap_at(y, xx, h, w, udi, ud) * interior;
        double ax = -lap_at(y, xx, h, w, xi, xv) * interior;
        double ri = b - ax;
        P.r[i] = ri;
        acc[0] += ri * ri;
        acc[1] += b * b;
        acc[2] += mi ? udi * udi : 0.0;
        acc[3] += interior;
    }
    block_sum<4>(acc, sh);
    if (threadIdx.x == 0)
        for (int k = 0; k < 4; ++k) partials[blockIdx.x * 4 + k] = acc[k];
}

