// On-chip CG level kernel over 2-D tiles (included by inpaint.cu).
//
// The level is cut into tiles of <= kTileRows rows x tile_cols (<= 512)
// columns, one CTA per tile: thread c owns column c of its tile and keeps
// the column's r in registers (one per row) and its mask bits in one word;
// the padded search direction p (one halo row above/below, one halo column
// left/right) and as many x rows as fit live in shared memory.  Compared with
// full-width bands (cg_band2), a tile exchanges ~4x fewer halo values per
// iteration (its perimeter instead of two plane-wide rows) and keeps ~all of
// x on chip, and the tile grid can use every SM (1080x1920: 36 x 4 tiles of
// 30 x 480).  Per iteration: p = r + beta p on the own rows and on the halo
// cells (each halo cell already holds the neighbour's previous p edge, so only
// the neighbours' published r edges are loaded, through a global exchange
// buffer), A p and p.Ap, grid reduction, r -= alpha A p and r.r, grid
// reduction (x += alpha p overlapped with its wait).  Float64 expressions and
// the per-CTA summation order are those of the column walk in every level
// kernel (cg_cluster_col.cuh), so a level solves identically in either.
#pragma once

constexpr int kTileRows = 32;
constexpr int kTileThreads = 512;
constexpr int kTileCols = kTileThreads;  // thread c owns column c of its tile

struct TileBatch {
    CgParams P[kMaxBatch];
    const double* setup[kMaxBatch];
    int nt;                // tiles per solve
    unsigned int* ticket;  // nullable: CTAs take (solve, tile) = divmod(ticket, nt) in start order
};

__global__ void __launch_bounds__(kTileThreads, 1) cg_tile_kernel(const __grid_constant__ TileBatch B) {
    constexpr int ROWS = kTileRows;
    extern __shared__ double sp[];  // (trows + 2) x (tcols + 2), then x_rows x tcols
    __shared__ double sh[2 * 4 * 32 + 8];
    __shared__ int s_ticket;
    int t = blockIdx.x;
    if (B.ticket) {
        if (threadIdx.x == 0) s_ticket = (int)atomicAdd(B.ticket, 1u);
        __syncthreads();
        t = s_ticket;
    }
    const int nt = B.nt, tile = t % nt;
    const CgParams& P = B.P[t / nt];
    const double* __restrict__ setup = B.setup[t / nt];
    RedState red;
    const int h = P.h, w = P.w;
    const int trows = P.band_rows, tcols = P.tile_cols, ntc = P.ntc;
    const int ti = tile / ntc, tj = tile - ti * ntc;
    const int y0 = ti * trows, x0 = tj * tcols;
    const int rows = min(trows, h - y0), cols = min(tcols, w - x0);
    const int W2 = tcols + 2;
    const int tid = threadIdx.x;
    const int c = tid;  // local column
    const bool act = c < cols;
    const int gc = x0 + c;
    const bool top = y0 == 0, bottom = y0 + rows == h, left = x0 == 0, right = x0 + cols == w;
    const size_t E = 2 * (size_t)tcols + 2 * (size_t)trows;  // exchange doubles per tile
    const double* __restrict__ f = P.f;
    const uint8_t* __restrict__ m = P.m;
    const int band = tile;  // (HIVC_TRACE)
    if (P.stamp && tile == 0 && tid == 0) P.stamp[0] = globaltimer_ns();

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

    double* sx = sp + (size_t)(trows + 2) * W2;  // resident x rows
    const int xr = min(P.x_rows, rows);
    // ---- r into registers, mask bits, p = 0, resident x
    double r[ROWS];
    uint32_t mbits = 0;
#pragma unroll
    for (int row = 0; row < ROWS; ++row) {
        r[row] = 0.0;
        if (row < rows && act) {
            const size_t gi = (size_t)(y0 + row) * w + gc;
            r[row] = __ldcg(P.r + gi);
            sp[(row + 1) * W2 + c + 1] = 0.0;
            if (m[gi]) mbits |= 1u << row;
            if (row < xr) sx[row * tcols + c] = __ldcg(P.x + gi);
        }
    }
    double* ex_r = P.ex_r;
    const size_t mine = (size_t)tile * E;
    int it = 0;
    double margin = 1e300;
    if (!all_mask && bn != 0.0) {
        double beta = 0.0;
        for (int k = 1; k <= P.max_iter; ++k) {
            it = k;
            HIVC_TRACE(0);
            // ---- phase 1a: own p = r + beta p, then the halo rows / columns.  A halo
            // cell already holds the neighbour's previous p edge (it was computed here
            // last iteration with the neighbour's own operands and expression), so only
            // the neighbours' r edges are loaded; the loads are in flight while the
            // own rows are updated.
            {
                double tr = 0, br = 0, lr = 0, rr_ = 0;
                const bool hc = tid < rows;  // this thread also rebuilds row tid of the side halos
                if (act && !top)
                    tr = k == 1 ? __ldcg(P.r + (size_t)(y0 - 1) * w + gc)
                                : __ldcg(ex_r + (size_t)(tile - ntc) * E + tcols + c);  // upper tile's bottom row
                if (act && !bottom)
                    br = k == 1 ? __ldcg(P.r + (size_t)(y0 + rows) * w + gc)
                                : __ldcg(ex_r + (size_t)(tile + ntc) * E + c);  // lower tile's top row
                if (hc && !left)
                    lr = k == 1 ? __ldcg(P.r + (size_t)(y0 + tid) * w + x0 - 1)
                                : __ldcg(ex_r + (size_t)(tile - 1) * E + 2 * tcols + trows + tid);  // left tile's right column
                if (hc && !right)
                    rr_ = k == 1 ? __ldcg(P.r + (size_t)(y0 + tid) * w + x0 + cols)
                                 : __ldcg(ex_r + (size_t)(tile + 1) * E + 2 * tcols + tid);  // right tile's left column
                if (act) {
#pragma unroll
                    for (int row = 0; row < ROWS; ++row) {
                        if (row >= rows) break;
                        double* q = sp + (row + 1) * W2 + c + 1;
                        const double pn = r[row] + beta * (k == 1 ? 0.0 : *q);
                        *q = pn;
                        if (left && c == 0) q[-1] = pn;  // reflecting plane edges
                        if (right && c == cols - 1) q[1] = pn;
                        if (top && row == 0) q[-W2] = pn;
                        if (bottom && row == rows - 1) q[W2] = pn;
                    }
                }
                HIVC_TRACE(7);
                if (act && !top) {
                    double* q = sp + c + 1;
                    *q = tr + beta * (k == 1 ? 0.0 : *q);
                }
                if (act && !bottom) {
                    double* q = sp + (rows + 1) * W2 + c + 1;
                    *q = br + beta * (k == 1 ? 0.0 : *q);
                }
                if (hc && !left) {
                    double* q = sp + (tid + 1) * W2;
                    *q = lr + beta * (k == 1 ? 0.0 : *q);
                }
                if (hc && !right) {
                    double* q = sp + (tid + 1) * W2 + cols + 1;
                    *q = rr_ + beta * (k == 1 ? 0.0 : *q);
                }
            }
            __syncthreads();
            HIVC_TRACE(1);
            // ---- phase 1b: A p and p.Ap walking the own column top to bottom
            double d[1] = {0.0};
            if (act) {
                const double* col = sp + c + 1;
                double up = col[0], cur = col[W2];
#pragma unroll
                for (int row = 0; row < ROWS; ++row) {
                    if (row >= rows) break;
                    const double* q = col + (row + 1) * W2;
                    const double dn = q[W2];
                    const double lap = (((cur * -4.0 + up) + dn) + q[-1]) + q[1];
                    const double api = -lap * (((mbits >> row) & 1u) ? 0.0 : 1.0);
                    d[0] += cur * api;
                    up = cur;
                    cur = dn;
                }
            }
            HIVC_TRACE(2);
            if (P.trace && tid == 0 && k < 256) P.trace[2048 + k * 160 + (tile < 160 ? tile : 159)] = globaltimer_ns();
            grid_reduce<1>(d, sh, P, red, tile, nt);
            HIVC_TRACE(3);
            const double pap = d[0];
            if (pap <= 0.0 || rs < 1e-300) break;
            const double alpha = rs / pap;
            // ---- phase 2: r -= alpha A p, r.r; publish r's edges
            double e1[1] = {0.0};
            if (act) {
                const double* col = sp + c + 1;
                double up = col[0], cur = col[W2];
#pragma unroll
                for (int row = 0; row < ROWS; ++row) {
                    if (row >= rows) break;
                    const double* q = col + (row + 1) * W2;
                    const double dn = q[W2];
                    const double lap = (((cur * -4.0 + up) + dn) + q[-1]) + q[1];
                    const double api = -lap * (((mbits >> row) & 1u) ? 0.0 : 1.0);
                    double& rr = r[row];
                    rr = rr - alpha * api;
                    e1[0] += rr * rr;
                    up = cur;
                    cur = dn;
                }
                ex_r[mine + c] = r[0];
#pragma unroll
                for (int row = 0; row < ROWS; ++row)
                    if (row == rows - 1) ex_r[mine + tcols + c] = r[row];
                if (c == 0)
#pragma unroll
                    for (int row = 0; row < ROWS; ++row)
                        if (row < rows) ex_r[mine + 2 * tcols + row] = r[row];
                if (c == cols - 1)
#pragma unroll
                    for (int row = 0; row < ROWS; ++row)
                        if (row < rows) ex_r[mine + 2 * tcols + trows + row] = r[row];
            }
            HIVC_TRACE(4);
            grid_reduce_arrive<1>(e1, sh, P, red, tile);
            // x += alpha p while the other CTAs arrive (x is not read until the level ends);
            // the first streamed rows' loads go out before the resident rows are updated
            if (act) {
                constexpr int kPre = 4;
                double xv[kPre];
#pragma unroll
                for (int j = 0; j < kPre; ++j) {
                    const int row = xr + j;
                    xv[j] = row < rows ? P.x[(size_t)(y0 + row) * w + gc] : 0.0;
                }
#pragma unroll
                for (int row = 0; row < ROWS; ++row) {
                    if (row >= xr || row >= rows) break;
                    double& xs = sx[row * tcols + c];
                    xs = xs + alpha * sp[(row + 1) * W2 + c + 1];
                }
#pragma unroll
                for (int j = 0; j < kPre; ++j) {
                    const int row = xr + j;
                    if (row < rows) P.x[(size_t)(y0 + row) * w + gc] = xv[j] + alpha * sp[(row + 1) * W2 + c + 1];
                }
                // further streamed rows, 8 at a time with the loads issued first
#pragma unroll 1
                for (int g = xr + kPre; g < rows; g += 8) {
                    double xw[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int row = g + j;
                        xw[j] = row < rows ? P.x[(size_t)(y0 + row) * w + gc] : 0.0;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int row = g + j;
                        if (row < rows) P.x[(size_t)(y0 + row) * w + gc] = xw[j] + alpha * sp[(row + 1) * W2 + c + 1];
                    }
                }
            }
            HIVC_TRACE(6);
            grid_reduce_finish<1>(e1, sh, P, red, nt);
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
    if (act)
        for (int row = 0; row < rows; ++row) {
            const size_t gi = (size_t)(y0 + row) * w + gc;
            const bool mi = m[gi] != 0;
            const double xv = row < xr ? sx[row * tcols + c] : P.x[gi];
            P.u[gi] = all_mask ? __ldg(f + gi) : (mi ? __ldg(f + gi) : 0.0) + xv;
        }
    if (tile == 0 && tid == 0) {
        *P.iters = it;
        if (P.margin) *P.margin = margin;
        if (P.stamp) P.stamp[1] = globaltimer_ns();
    }
}
