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

// setup pass 1: x = x0 * interior, x0 prolonged from the coarser level
// (homogeneous.py:71, 133-154).  2-D: blockIdx.x = 256-column strip,
// blockIdx.y = band of kSetupXRows rows, blockIdx.z = solve; a thread owns one
// column, so the column's interpolation position and weights are computed
// once and the row's once per row (the same expressions as prolong_at).
constexpr int kSetupXRows = 8;
__global__ void __launch_bounds__(256) cg_setup_x_kernel(const __grid_constant__ SetupBatch B) {
    const CgParams& P = B.P[blockIdx.z];
    const int w = P.w, h = P.h;
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {  // the level launch that follows starts a fresh barrier epoch
        P.bar[0] = 0;
        if (blockIdx.z == 0 && B.ticket) *B.ticket = 0;
    }
    const int xx = blockIdx.x * blockDim.x + threadIdx.x;
    if (xx >= w) return;
    double xs = ((double)xx + 0.5) * ((double)P.wc / (double)P.w) - 0.5;
    xs = fmin(fmax(xs, 0.0), (double)(P.wc - 1));
    const int x0 = (int)floor(xs);
    const int x1 = min(x0 + 1, P.wc - 1);
    const double wx = xs - (double)x0;
    const double* c = P.uc;
    const int y_end = min(h, (int)(blockIdx.y + 1) * kSetupXRows);
    for (int y = blockIdx.y * kSetupXRows; y < y_end; ++y) {
        double ys = ((double)y + 0.5) * ((double)P.hc / (double)P.h) - 0.5;
        ys = fmin(fmax(ys, 0.0), (double)(P.hc - 1));
        const int y0 = (int)floor(ys);
        const int y1 = min(y0 + 1, P.hc - 1);
        const double wy = ys - (double)y0;
        const double c00 = __ldg(c + (size_t)y0 * P.wc + x0), c01 = __ldg(c + (size_t)y0 * P.wc + x1);
        const double c10 = __ldg(c + (size_t)y1 * P.wc + x0), c11 = __ldg(c + (size_t)y1 * P.wc + x1);
        const double x0v = (1 - wy) * ((1 - wx) * c00 + wx * c01) + wy * ((1 - wx) * c10 + wx * c11);
        const size_t i = (size_t)y * w + xx;
        P.x[i] = x0v * (P.m[i] ? 0.0 : 1.0);
    }
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
    // grid-stride over the flat index as before (same pixels per thread, same
    // accumulation order); (y, x) advanced without a division, and every load
    // of the 5-point stencils issued before the first use
    const int stride = gridDim.x * blockDim.x;
    const int sy = stride / w, sx = stride - sy * w;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int y = i / w, xx = i - y * w;
    for (; i < n; i += stride) {
        const bool hn = y > 0, hs = y < h - 1, hw = xx > 0, he = xx < w - 1;
        const uint8_t mc = m[i];
        const uint8_t mn = hn ? m[i - w] : 0, ms = hs ? m[i + w] : 0, mw = hw ? m[i - 1] : 0, me = he ? m[i + 1] : 0;
        const double fc = __ldg(f + i);
        const double fn = hn ? __ldg(f + i - w) : 0.0, fs = hs ? __ldg(f + i + w) : 0.0;
        const double fw = hw ? __ldg(f + i - 1) : 0.0, fe = he ? __ldg(f + i + 1) : 0.0;
        const double xi = xg[i];
        const double xn = hn ? xg[i - w] : xi, xs = hs ? xg[i + w] : xi;
        const double xw = hw ? xg[i - 1] : xi, xe = he ? xg[i + 1] : xi;
        const bool mi = mc != 0;
        const double interior = mi ? 0.0 : 1.0;
        const double udi = mi ? fc : 0.0;
        // lap_at's reflecting 5-point Laplacian (homogeneous.py:27-43), same association
        const double un = hn ? (mn ? fn : 0.0) : udi, us = hs ? (ms ? fs : 0.0) : udi;
        const double uw = hw ? (mw ? fw : 0.0) : udi, ue = he ? (me ? fe : 0.0) : udi;
        const double b = ((((udi * -4.0 + un) + us) + uw) + ue) * interior;
        const double ax = -((((xi * -4.0 + xn) + xs) + xw) + xe) * interior;
        const double ri = b - ax;
        P.r[i] = ri;
        acc[0] += ri * ri;
        acc[1] += b * b;
        acc[2] += mi ? udi * udi : 0.0;
        acc[3] += interior;
        xx += sx;
        y += sy;
        if (xx >= w) xx -= w, ++y;
    }
    block_sum<4>(acc, sh);
    if (threadIdx.x == 0)
        for (int k = 0; k < 4; ++k) partials[blockIdx.x * 4 + k] = acc[k];
}

