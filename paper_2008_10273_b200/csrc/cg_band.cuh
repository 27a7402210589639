// On-chip CG level kernel (included by inpaint.cu).
//
// One CTA per horizontal band of <= 8 rows (one CTA per SM, cooperative
// launch).  For the whole level the band's residual r lives in REGISTERS and
// its search direction p (plus one halo row above/below and one pad column
// left/right holding the reflected edge value) in SHARED memory; x streams
// through global memory.  Only the first/last owned rows of r and p cross
// CTAs: each CTA publishes them to small exchange buffers and, after the grid
// barrier, its neighbours rebuild their halo p = r + beta p from them.
// A p is recomputed from shared memory in phase 2 instead of being stored.
// Per iteration a CTA moves x (16 B/px) + 4 exchange rows; everything else is
// on-chip.  The per-pixel float64 expressions are those of cg_level_kernel.
//
// Pixel mapping: thread t owns columns t + 512k (k < 4) of each owned row, so
// the per-thread register array r[row * 4 + k] is statically indexed.
#pragma once

// Optional phase timestamps of CTA 0 / thread 0 (HIVC_CG_TRACE=1, diagnostics only).
#define HIVC_TRACE(slot)                                                                      \
    do {                                                                                      \
        if (P.trace && band == 0 && tid == 0 && k < 256) P.trace[k * 8 + (slot)] = globaltimer_ns(); \
    } while (0)

constexpr int kBandThreads = 512;
constexpr int kBandCols = 4;  // column slots per thread: w <= 2048
constexpr int kBandRows = 8;  // rows per band
constexpr int kPackRows = 16; // rows per band in throughput mode (w <= 1024)
constexpr int kBandPx = kBandCols * kBandRows;
constexpr int kSetupCtas = 296;
constexpr int kBand2Smem = 224 * 1024;  // band2 dynamic smem cap (+ 2.1 KB static <= the 227 KB opt-in limit)

// A batch of same-shape level solves (kernel parameter, __grid_constant__).
// ticket != nullptr: CTAs take (solve, band) = divmod(ticket, nb) in the order
// they start, so the CTAs of a solve are resident together as long as nb
// CTAs fit the GPU (the first solves finish and free SMs for the rest); the
// batch never runs concurrently with another spinning launch (one solver stream).
struct BandBatch {
    CgParams P[kMaxBatch];
    const double* setup[kMaxBatch];
    int nb;
    unsigned int* ticket;
};
struct SetupBatch {
    CgParams P[kMaxBatch];
    double* partials[kMaxBatch];
    unsigned int* ticket;  // reset with the solves' barrier counters (nullable)
};

// Setup for the band kernel: x = x0*interior, r = b - A x (global), and the
// per-CTA partials of r.r, b.b, |f_mask|^2, #interior (homogeneous.py:64-77).
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

__global__ void __launch_bounds__(kBandThreads, 1) cg_band_kernel(CgParams P, const double* __restrict__ setup) {
    extern __shared__ double sp[];  // (kBandRows + 2) x (w + 2)
    __shared__ double sh[2 * 4 * 32 + 8];
    RedState red;
    const int h = P.h, w = P.w, W2 = w + 2;
    const int band = blockIdx.x, nb = gridDim.x;
    const int y0 = band * P.band_rows;
    const int rows = min(P.band_rows, h - y0);
    const int tid = threadIdx.x;
    const bool top = y0 == 0, bottom = y0 + rows == h;
    uint8_t* smask = reinterpret_cast<uint8_t*>(sp + (size_t)(kBandRows + 2) * W2);
    const double* __restrict__ f = P.f;
    const uint8_t* __restrict__ m = P.m;
    if (P.stamp && band == 0 && tid == 0) P.stamp[0] = globaltimer_ns();

    // ---- level scalars from the setup partials (fixed order in every CTA)
    if (tid < 32) {
        for (int k = 0; k < 4; ++k) {
            double s = 0.0;
            for (int g = tid; g < kSetupCtas; g += 32) s += setup[g * 4 + k];
            s = warp_sum(s);
            if (tid == 0) sh[k * 32] = s;
        }
    }
    __syncthreads();
    double rs = sh[0];
    const bool all_mask = sh[96] == 0.0;
    const double bn = (P.finest && sh[64] != 0.0) ? sqrt(sh[64]) : sqrt(sh[32]);
    __syncthreads();

    // ---- r into registers, p = 0 (first iteration has beta = 0: p = r + 0 * 0 = r)
    double r[kBandPx];
#pragma unroll
    for (int j = 0; j < kBandPx; ++j) {
        const int row = j / kBandCols, col = tid + kBandThreads * (j % kBandCols);
        r[j] = 0.0;
        if (row < rows && col < w) {
            size_t gi = (size_t)(y0 + row) * w + col;
            r[j] = __ldcg(P.r + gi);
            sp[(row + 1) * W2 + col + 1] = 0.0;
            smask[row * w + col] = m[gi];
        }
    }
    const size_t pstride = (size_t)nb * 2 * w;
    int it = 0;
    double margin = 1e300;
    if (!all_mask && bn != 0.0) {
        double beta = 0.0;
        for (int k = 1; k <= P.max_iter; ++k) {
            it = k;
            const size_t prev_par = (size_t)((k - 1) & 1) * pstride, cur_par = (size_t)(k & 1) * pstride;
            // ---- phase 1: p = r + beta p on the band, its halo rows and pads; then p.Ap
            HIVC_TRACE(0);
            for (int c = tid; c < w; c += kBandThreads) {
                if (!top) {
                    double rv, pv;
                    if (k == 1) {
                        rv = pv = __ldcg(P.r + (size_t)(y0 - 1) * w + c);
                    } else {
                        size_t e = ((size_t)(band - 1) * 2 + 1) * w + c;
                        rv = __ldcg(P.ex_r + e);
                        pv = __ldcg(P.ex_p + prev_par + e);
                    }
                    sp[c + 1] = rv + beta * pv;
                }
                if (!bottom) {
                    double rv, pv;
                    if (k == 1) {
                        rv = pv = __ldcg(P.r + (size_t)(y0 + rows) * w + c);
                    } else {
                        size_t e = ((size_t)(band + 1) * 2 + 0) * w + c;
                        rv = __ldcg(P.ex_r + e);
                        pv = __ldcg(P.ex_p + prev_par + e);
                    }
                    sp[(rows + 1) * W2 + c + 1] = rv + beta * pv;
                }
            }
#pragma unroll
            for (int j = 0; j < kBandPx; ++j) {
                const int row = j / kBandCols, col = tid + kBandThreads * (j % kBandCols);
                if (row < rows && col < w) {
                    double* q = sp + (row + 1) * W2 + col + 1;
                    const double pn = r[j] + beta * (k == 1 ? 0.0 : *q);
                    *q = pn;
                    if (col == 0) q[-1] = pn;                 // reflecting pad (west of column 0)
                    if (col == w - 1) q[1] = pn;              // reflecting pad (east of the last column)
                    if (top && row == 0) q[-W2] = pn;         // north of row 0 is row 0
                    if (bottom && row == rows - 1) q[W2] = pn;  // south of the last row is itself
                }
            }
            __syncthreads();
            HIVC_TRACE(1);
            double d[1] = {0.0};
#pragma unroll
            for (int j = 0; j < kBandPx; ++j) {
                const int row = j / kBandCols, col = tid + kBandThreads * (j % kBandCols);
                if (row < rows && col < w) {
                    const double* q = sp + (row + 1) * W2 + col + 1;
                    const double c0 = q[0];
                    const double lap = (((c0 * -4.0 + q[-W2]) + q[W2]) + q[-1]) + q[1];
                    const double api = -lap * (smask[row * w + col] ? 0.0 : 1.0);
                    d[0] += c0 * api;
                }
            }
            for (int c = tid; c < w; c += kBandThreads) {
                P.ex_p[cur_par + ((size_t)band * 2 + 0) * w + c] = sp[W2 + c + 1];
                P.ex_p[cur_par + ((size_t)band * 2 + 1) * w + c] = sp[rows * W2 + c + 1];
            }
            HIVC_TRACE(2);
            grid_reduce<1>(d, sh, P, red);
            HIVC_TRACE(3);
            const double pap = d[0];
            if (pap <= 0.0 || rs < 1e-300) break;
            const double alpha = rs / pap;
            // ---- phase 2: x += alpha p, r -= alpha Ap (recomputed), r.r; publish r's edge rows
            double e1[1] = {0.0};
#pragma unroll
            for (int j = 0; j < kBandPx; ++j) {
                const int row = j / kBandCols, col = tid + kBandThreads * (j % kBandCols);
                if (row < rows && col < w) {
                    const double* q = sp + (row + 1) * W2 + col + 1;
                    const double c0 = q[0];
                    const double lap = (((c0 * -4.0 + q[-W2]) + q[W2]) + q[-1]) + q[1];
                    const double api = -lap * (smask[row * w + col] ? 0.0 : 1.0);
                    size_t gi = (size_t)(y0 + row) * w + col;
                    P.x[gi] = P.x[gi] + alpha * c0;
                    r[j] = r[j] - alpha * api;
                    e1[0] += r[j] * r[j];
                    if (row == 0) P.ex_r[((size_t)band * 2 + 0) * w + col] = r[j];
                    if (row == rows - 1) P.ex_r[((size_t)band * 2 + 1) * w + col] = r[j];
                }
            }
            HIVC_TRACE(4);
            grid_reduce<1>(e1, sh, P, red);
            HIVC_TRACE(5);
            const double rs1 = e1[0];
            const double lhs = sqrt(rs1), rhs = P.tol * bn;
            if (rhs > 0.0) margin = fmin(margin, fabs(lhs - rhs) / rhs);
            if (lhs <= rhs) break;
            beta = rs1 / rs;
            rs = rs1;
        }
    }
    // level solution u = u_D + x (or f when the mask is full)
    for (int row = 0; row < rows; ++row)
        for (int col = tid; col < w; col += kBandThreads) {
            size_t gi = (size_t)(y0 + row) * w + col;
            bool mi = m[gi] != 0;
            P.u[gi] = all_mask ? __ldg(f + gi) : (mi ? __ldg(f + gi) : 0.0) + P.x[gi];
        }
    if (band == 0 && tid == 0) {
        *P.iters = it;
        if (P.margin) *P.margin = margin;
        if (P.stamp) P.stamp[1] = globaltimer_ns();
    }
}
