// On-chip CG level kernel, column-streaming variant (included by inpaint.cu).
//
// Same data placement and exchange protocol as cg_band_kernel (one CTA per
// band of <= ROWS rows, r in registers, padded p in shared memory, x streamed,
// edge rows of r/p exchanged through global memory, two grid reductions per
// iteration), but every thread owns whole COLUMNS of its band
// (c = tid + 512 k, k < KC) and walks them top to bottom: the 5-point stencil
// reuses the column's previous/current/next p values from registers, so it
// reads 3 shared-memory values per pixel instead of 5, the mask is a bit set
// in one register, and with STORE_AP the phase-1 A p values stay in registers
// for phase 2 (small bands) instead of being recomputed.
#pragma once

constexpr int kXG = 8;  // streamed-x values per batch of loads

template <int ROWS, int KC, bool STORE_AP>
__global__ void __launch_bounds__(kBandThreads, 1) cg_band2_kernel(const __grid_constant__ BandBatch B) {
    static_assert(ROWS * KC <= 32, "mask bits");
    extern __shared__ double sp[];  // (ROWS + 2) x (w + 2)
    __shared__ double sh[2 * 4 * 32 + 8];
    __shared__ int s_ticket;
    int t = blockIdx.x;
    if (B.ticket) {
        if (threadIdx.x == 0) s_ticket = (int)atomicAdd(B.ticket, 1u);
        __syncthreads();
        t = s_ticket;
    }
    const int nb = B.nb, band = t % nb;
    const CgParams& P = B.P[t / nb];
    const double* __restrict__ setup = B.setup[t / nb];
    RedState red;
    const int h = P.h, w = P.w, W2 = w + 2;
    const int y0 = band * P.band_rows;
    const int rows = min(P.band_rows, h - y0);
    const int tid = threadIdx.x;
    const bool top = y0 == 0, bottom = y0 + rows == h;
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

    // resident x rows behind the padded p
    double* sx = sp + (size_t)(ROWS + 2) * W2;
    const int xr = min(P.x_rows, rows);
    for (int i = tid; i < xr * w; i += kBandThreads) sx[i] = __ldcg(P.x + (size_t)y0 * w + i);
    // ---- r into registers (index row * KC + k), mask bits, p = 0
    double r[ROWS * KC];
    double ap[STORE_AP ? ROWS * KC : 1];
    uint32_t mbits = 0;
#pragma unroll
    for (int k = 0; k < KC; ++k) {
        const int c = tid + kBandThreads * k;
#pragma unroll
        for (int row = 0; row < ROWS; ++row) {
            r[row * KC + k] = 0.0;
            if (row < rows && c < w) {
                const size_t gi = (size_t)(y0 + row) * w + c;
                r[row * KC + k] = __ldcg(P.r + gi);
                sp[(row + 1) * W2 + c + 1] = 0.0;
                if (m[gi]) mbits |= 1u << (row * KC + k);
            }
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
            HIVC_TRACE(0);
            // ---- phase 1a: halo rows (neighbours' edge rows of r and p) and own p = r + beta p
            {  // all KC columns' halo values are loaded before any is used (one L2 round trip)
                double tr[KC], tp[KC], br[KC], bp[KC];
#pragma unroll
                for (int k2 = 0; k2 < KC; ++k2) {
                    const int c = tid + kBandThreads * k2;
                    tr[k2] = tp[k2] = br[k2] = bp[k2] = 0.0;
                    if (c >= w) continue;
                    if (!top) {
                        if (k == 1) {
                            tr[k2] = tp[k2] = __ldcg(P.r + (size_t)(y0 - 1) * w + c);
                        } else {
                            const size_t e = ((size_t)(band - 1) * 2 + 1) * w + c;
                            tr[k2] = __ldcg(P.ex_r + e);
                            tp[k2] = __ldcg(P.ex_p + prev_par + e);
                        }
                    }
                    if (!bottom) {
                        if (k == 1) {
                            br[k2] = bp[k2] = __ldcg(P.r + (size_t)(y0 + rows) * w + c);
                        } else {
                            const size_t e = ((size_t)(band + 1) * 2 + 0) * w + c;
                            br[k2] = __ldcg(P.ex_r + e);
                            bp[k2] = __ldcg(P.ex_p + prev_par + e);
                        }
                    }
                }
#pragma unroll
                for (int k2 = 0; k2 < KC; ++k2) {
                    const int c = tid + kBandThreads * k2;
                    if (c >= w) continue;
                    if (!top) sp[c + 1] = tr[k2] + beta * tp[k2];
                    if (!bottom) sp[(rows + 1) * W2 + c + 1] = br[k2] + beta * bp[k2];
                }
            }
#pragma unroll
            for (int k2 = 0; k2 < KC; ++k2) {
                const int c = tid + kBandThreads * k2;
                if (c >= w) continue;
#pragma unroll
                for (int row = 0; row < ROWS; ++row) {
                    if (row >= rows) break;
                    double* q = sp + (row + 1) * W2 + c + 1;
                    const double pn = r[row * KC + k2] + beta * (k == 1 ? 0.0 : *q);
                    *q = pn;
                    if (c == 0) q[-1] = pn;
                    if (c == w - 1) q[1] = pn;
                    if (top && row == 0) q[-W2] = pn;
                    if (bottom && row == rows - 1) q[W2] = pn;
                }
            }
            __syncthreads();
            HIVC_TRACE(1);
            // ---- phase 1b: A p and p.Ap, walking each owned column top to bottom
            double d[1] = {0.0};
#pragma unroll
            for (int k2 = 0; k2 < KC; ++k2) {
                const int c = tid + kBandThreads * k2;
                if (c >= w) continue;
                const double* col = sp + c + 1;
                double up = col[0], cur = col[W2];
#pragma unroll
                for (int row = 0; row < ROWS; ++row) {
                    if (row >= rows) break;
                    const double* q = col + (row + 1) * W2;
                    const double dn = q[W2];
                    const double lap = (((cur * -4.0 + up) + dn) + q[-1]) + q[1];
                    const double api = -lap * (((mbits >> (row * KC + k2)) & 1u) ? 0.0 : 1.0);
                    if (STORE_AP) ap[STORE_AP ? row * KC + k2 : 0] = api;
                    d[0] += cur * api;
                    up = cur;
                    cur = dn;
                }
            }
            for (int c = tid; c < w; c += kBandThreads) {
                P.ex_p[cur_par + ((size_t)band * 2 + 0) * w + c] = sp[W2 + c + 1];
                P.ex_p[cur_par + ((size_t)band * 2 + 1) * w + c] = sp[rows * W2 + c + 1];
            }
            HIVC_TRACE(2);
            if (P.trace && tid == 0 && k < 256) P.trace[2048 + k * 160 + band] = globaltimer_ns();  // arrival spread
            grid_reduce<1>(d, sh, P, red, band, nb);
            HIVC_TRACE(3);
            const double pap = d[0];
            if (pap <= 0.0 || rs < 1e-300) break;
            const double alpha = rs / pap;
            // ---- phase 2: x += alpha p, r -= alpha Ap, r.r; publish r's edge rows
            double e1[1] = {0.0};
#pragma unroll
            for (int k2 = 0; k2 < KC; ++k2) {
                const int c = tid + kBandThreads * k2;
                if (c >= w) continue;
                const double* col = sp + c + 1;
                double up = col[0], cur = col[W2];
#pragma unroll
                for (int row = 0; row < ROWS; ++row) {
                    if (row >= rows) break;
                    const double* q = col + (row + 1) * W2;
                    double api;
                    double dn = 0.0;
                    if (STORE_AP) {
                        api = ap[STORE_AP ? row * KC + k2 : 0];
                    } else {
                        dn = q[W2];
                        const double lap = (((cur * -4.0 + up) + dn) + q[-1]) + q[1];
                        api = -lap * (((mbits >> (row * KC + k2)) & 1u) ? 0.0 : 1.0);
                    }
                    double& rr = r[row * KC + k2];
                    rr = rr - alpha * api;
                    e1[0] += rr * rr;
                    if (row == 0) P.ex_r[((size_t)band * 2 + 0) * w + c] = rr;
                    if (row == rows - 1) P.ex_r[((size_t)band * 2 + 1) * w + c] = rr;
                    if (!STORE_AP) {
                        up = cur;
                        cur = dn;
                    }
                }
            }
            HIVC_TRACE(4);
            grid_reduce_arrive<1>(e1, sh, P, red, band);
            // x += alpha p while the other CTAs arrive (x is not read until the level ends):
            // resident rows in smem; streamed rows kXG values at a time, all loads issued first
#pragma unroll
            for (int k2 = 0; k2 < KC; ++k2) {
                const int c = tid + kBandThreads * k2;
                if (c >= w) continue;
#pragma unroll
                for (int row = 0; row < ROWS; ++row) {
                    if (row >= xr || row >= rows) break;
                    double& xs = sx[row * w + c];
                    xs = xs + alpha * sp[(row + 1) * W2 + c + 1];
                }
            }
            if (xr < rows) {
#pragma unroll
                for (int g = 0; g < ROWS * KC; g += kXG) {
                    if ((g + kXG - 1) / KC < xr) continue;  // group entirely in resident rows
                    double xv[kXG];
#pragma unroll
                    for (int j = 0; j < kXG; ++j) {
                        const int idx = g + j, row = idx / KC, c = tid + kBandThreads * (idx % KC);
                        xv[j] = 0.0;
                        if (idx < ROWS * KC && row >= xr && row < rows && c < w)
                            xv[j] = P.x[(size_t)(y0 + row) * w + c];
                    }
#pragma unroll
                    for (int j = 0; j < kXG; ++j) {
                        const int idx = g + j, row = idx / KC, c = tid + kBandThreads * (idx % KC);
                        if (idx < ROWS * KC && row >= xr && row < rows && c < w)
                            P.x[(size_t)(y0 + row) * w + c] = xv[j] + alpha * sp[(row + 1) * W2 + c + 1];
                    }
                }
            }
            HIVC_TRACE(6);
            grid_reduce_finish<1>(e1, sh, P, red, nb);
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
        for (int c = tid; c < w; c += kBandThreads) {
            const size_t gi = (size_t)(y0 + row) * w + c;
            const bool mi = m[gi] != 0;
            const double xv = row < xr ? sx[row * w + c] : P.x[gi];
            P.u[gi] = all_mask ? __ldg(f + gi) : (mi ? __ldg(f + gi) : 0.0) + xv;
        }
    if (band == 0 && tid == 0) {
        *P.iters = it;
        if (P.margin) *P.margin = margin;
        if (P.stamp) P.stamp[1] = globaltimer_ns();
    }
}
