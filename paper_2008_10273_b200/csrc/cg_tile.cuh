// On-chip CG level kernel over 2-D tiles (included by inpaint.cu).
//
// The level is cut into tiles of trows (<= kTileRows) rows x tile_cols (<= 512)
// columns, one CTA per tile: thread c owns column c of its tile and keeps
// the column's r in registers (one per row) and its mask bits in one word;
// the padded search direction p (one halo row above/below, one halo column
// left/right) and as many x rows as fit live in shared memory.  Compared with
// full-width bands, a tile exchanges ~4x fewer halo values per iteration (its
// perimeter instead of two plane-wide rows) and keeps ~all of x on chip, and
// the tile grid can use every SM (1080x1920: 36 x 4 tiles of 30 x 480).  Per
// iteration: p = r + beta p on the own rows and on the halo cells (each halo
// cell already holds the neighbour's previous p edge, so only the
// neighbours' published r edges are loaded, through a global exchange
// buffer), A p and p.Ap, grid reduction, r -= alpha A p and r.r, grid
// reduction (x += alpha p overlapped with its wait).  Float64 expressions and
// the per-CTA summation order are those of the column walk in every level
// kernel (cg_cluster_col.cuh), so a level solves identically in either.
//
// Instantiations (cg_tile_kernel<ROWS, TC>):
//  * TC > 0, "exact": every tile is ROWS x TC (the plan's trows / tcols) except
//    the plane's last tile row / column, which may be shorter.  The row walks
//    are straight-line code with compile-time shared-memory offsets; the
//    missing rows of a short last tile row are inert padding (r = 0, masked,
//    so A p = 0 there and they add exact zeros to the dot products: the sums
//    equal the unpadded ones).
//  * TC == 0, generic: ROWS = kTileRows, runtime tile shape, every row guarded.
// A masked pixel's A p is the constant 0 (a select, not -lap * 0: the two
// differ only in the sign of a zero, which no sum or product here turns into
// a different non-zero value), and -lap is evaluated as the negated sum
// (((4 c - N) - S) - W) - E, which rounds to exactly -lap.
#pragma once

constexpr int kTileRows = 32;
// rows of A p kept in registers between the two stencil phases, per exact tile height
// (as many as the register file takes without spills at 512 threads x 128 registers)
#ifndef HIVC_CG_KEEP30
#define HIVC_CG_KEEP30 14
#endif
#ifndef HIVC_CG_KEEP23
#define HIVC_CG_KEEP23 16
#endif
#ifndef HIVC_CG_KEEP15
#define HIVC_CG_KEEP15 15
#endif
constexpr int kTileThreads = 512;
constexpr int kTileCols = kTileThreads;  // thread c owns column c of its tile

struct TileBatch {
    CgParams P[kMaxBatch];
    const double* setup[kMaxBatch];
    int nt;                // tiles per solve
    unsigned int* ticket;  // nullable: CTAs take (solve, tile) = divmod(ticket, nt) in start order
};

template <int ROWS, int TC>
__global__ void __launch_bounds__(kTileThreads, 1) cg_tile_kernel(const __grid_constant__ TileBatch B) {
    constexpr bool kExact = TC > 0;
    // exact tiles of <= 480 columns leave the last warp without a column: it runs the
    // second grid sum of each iteration
    constexpr bool kSyncWarp = kExact && TC <= kTileThreads - 32;
    // A p of the first kKeep rows stays in registers from the p.Ap walk to the r update
    // (the registers that hold the p loads of phase 1a are free then); the r update
    // recomputes it only for the rows below.  Same values either way.
    constexpr int kKeep = !kExact ? 0 : ROWS == 30 ? HIVC_CG_KEEP30 : ROWS == 23 ? HIVC_CG_KEEP23 : HIVC_CG_KEEP15;
    static_assert(kKeep >= 0 && kKeep <= ROWS, "kept rows");
    constexpr int kSyncWid = kTileThreads / 32 - 1;
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
    const int trows = kExact ? ROWS : P.band_rows;
    const int tcols = kExact ? TC : P.tile_cols;
    const int ntc = P.ntc;
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
    const int xr = min(P.x_rows, rows);  // x rows [0, xr) in shared memory, the rest stream through L2
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // own column, row 0 (padded coordinates (1, c + 1)); row k is col[k * W2]
    double* const col = sp + W2 + c + 1;
    // ---- r into registers, mask bits (rows past the plane: r = 0, masked), p = 0, resident x
    double r[ROWS];
    uint32_t mbits = rows < 32 ? ~((1u << rows) - 1u) : 0u;
    if (!act) mbits = ~0u;
#pragma unroll
    for (int row = 0; row < ROWS; ++row) {
        r[row] = 0.0;
        if (act && (kExact || row < rows)) col[row * W2] = 0.0;
        if (row < rows && act) {
            const size_t gi = (size_t)(y0 + row) * w + gc;
            r[row] = __ldcg(P.r + gi);
            if (m[gi]) mbits |= 1u << row;
            if (row < xr) sx[row * tcols + c] = __ldcg(P.x + gi);
        }
    }
    if (kExact && act) col[ROWS * W2] = 0.0;  // the row below the walk (halo / reflection / padding)
    double* ex_r = P.ex_r;
    const size_t mine = (size_t)tile * E;
    const bool hc = tid < rows;  // this thread also rebuilds row tid of the side halos
    // neighbours' published r edges (ex_r layout per tile: top row, bottom row, left column, right column)
    const double* ex_up = ex_r + (size_t)(tile - ntc) * E + tcols + c;             // upper tile's bottom row
    const double* ex_dn = ex_r + (size_t)(tile + ntc) * E + c;                     // lower tile's top row
    const double* ex_lf = ex_r + (size_t)(tile - 1) * E + 2 * tcols + trows + tid;  // left tile's right column
    const double* ex_rt = ex_r + (size_t)(tile + 1) * E + 2 * tcols + tid;          // right tile's left column
    int it = 0;
    double margin = 1e300;
    if (!all_mask && bn != 0.0) {
        double beta = 0.0;
        // the neighbours' r edges for phase 1a: the first iteration's from r itself, later
        // ones loaded as soon as the previous iteration's second grid sum is complete (in
        // flight while the CTA sums the partials)
        double tr = 0, br = 0, lr = 0, rr_ = 0;
        if (act && !top) tr = __ldcg(P.r + (size_t)(y0 - 1) * w + gc);
        if (act && !bottom) br = __ldcg(P.r + (size_t)(y0 + rows) * w + gc);
        if (hc && !left) lr = __ldcg(P.r + (size_t)(y0 + tid) * w + x0 - 1);
        if (hc && !right) rr_ = __ldcg(P.r + (size_t)(y0 + tid) * w + x0 + cols);
        for (int k = 1; k <= P.max_iter; ++k) {
            it = k;
            HIVC_TRACE(0);
            // ---- phase 1a: own p = r + beta p, then the halo rows / columns.  A halo
            // cell already holds the neighbour's previous p edge (it was computed here
            // last iteration with the neighbour's own operands and expression), so only
            // the neighbours' r edges are needed.  (First iteration: p = r.)
            {
                const bool first = k == 1;
                if (act) {
                    if (first) {
#pragma unroll
                        for (int row = 0; row < ROWS; ++row)
                            if (kExact || row < rows) col[row * W2] = r[row];
                    } else {
                        // every row's p load in flight before the first update (measured: chunks of
                        // 8 / 15 / 20 rows were slower in the later phases of the iteration)
                        constexpr int kChunk = kExact ? ROWS : 1;  // (the generic 32-row kernel spills with chunks)
#pragma unroll
                        for (int r0 = 0; r0 < ROWS; r0 += kChunk) {
                            double pv[kChunk];
#pragma unroll
                            for (int j = 0; j < kChunk; ++j)
                                if (r0 + j < ROWS && (kExact || r0 + j < rows)) pv[j] = col[(r0 + j) * W2];
#pragma unroll
                            for (int j = 0; j < kChunk; ++j)
                                if (r0 + j < ROWS && (kExact || r0 + j < rows))
                                    col[(r0 + j) * W2] = r[r0 + j] + beta * pv[j];
                        }
                    }
                    // reflecting plane edges (own values, re-read: only the edge threads)
                    if (top) col[-W2] = col[0];
                    if (bottom) col[rows * W2] = col[(rows - 1) * W2];
                    const bool rl = left && c == 0, rrf = right && c == cols - 1;
                    if (rl || rrf) {
#pragma unroll 1
                        for (int r0 = 0; r0 < rows; r0 += 8) {  // 8 loads in flight, then the stores
                            double v[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) v[j] = r0 + j < rows ? col[(r0 + j) * W2] : 0.0;
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                if (r0 + j < rows) {
                                    if (rl) col[(r0 + j) * W2 - 1] = v[j];
                                    if (rrf) col[(r0 + j) * W2 + 1] = v[j];
                                }
                        }
                    }
                }
                HIVC_TRACE(7);
                if (act && !top) {
                    double* q = col - W2;
                    *q = first ? tr : tr + beta * *q;
                }
                if (act && !bottom) {
                    double* q = col + rows * W2;
                    *q = first ? br : br + beta * *q;
                }
                if (hc && !left) {
                    double* q = sp + (tid + 1) * W2;
                    *q = first ? lr : lr + beta * *q;
                }
                if (hc && !right) {
                    double* q = sp + (tid + 1) * W2 + cols + 1;
                    *q = first ? rr_ : rr_ + beta * *q;
                }
            }
            __syncthreads();
            HIVC_TRACE(1);
            // ---- phase 1b: A p and p.Ap walking the own column top to bottom
            double d[1] = {0.0};
            double ap[kKeep > 0 ? kKeep : 1];
            if (act) {
                double up = col[-W2], cur = col[0];
#pragma unroll
                for (int row = 0; row < ROWS; ++row) {
                    if (!kExact && row >= rows) break;
                    const double* q = col + row * W2;
                    const double dn = q[W2];
                    // -lap, (((-4 c + N) + S) + W) + E negated term by term (exact: round-to-nearest is symmetric)
                    const double nlap = (((cur * 4.0 - up) - dn) - q[-1]) - q[1];
                    const double api = ((mbits >> row) & 1u) ? 0.0 : nlap;
                    if (row < kKeep) ap[row] = api;
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
#pragma unroll
                for (int row = 0; row < kKeep; ++row) {
                    double& rr = r[row];
                    rr = rr - alpha * ap[row];
                    e1[0] += rr * rr;
                }
                double up = 0.0, cur = 0.0;
                if (kKeep < ROWS) {
                    up = col[(kKeep - 1) * W2];
                    cur = col[kKeep * W2];
                }
#pragma unroll
                for (int row = kKeep; row < ROWS; ++row) {
                    if (!kExact && row >= rows) break;
                    const double* q = col + row * W2;
                    const double dn = q[W2];
                    // -lap, (((-4 c + N) + S) + W) + E negated term by term (exact: round-to-nearest is symmetric)
                    const double nlap = (((cur * 4.0 - up) - dn) - q[-1]) - q[1];
                    const double api = ((mbits >> row) & 1u) ? 0.0 : nlap;
                    double& rr = r[row];
                    rr = rr - alpha * api;
                    e1[0] += rr * rr;
                    up = cur;
                    cur = dn;
                }
                double* ex = ex_r + mine;
                if (!top) ex[c] = r[0];
                if (!bottom) {
                    if (kExact) {
                        ex[tcols + c] = r[ROWS - 1];  // a tile with a lower neighbour is full
                    } else {
#pragma unroll
                        for (int row = 0; row < ROWS; ++row)
                            if (row == rows - 1) ex[tcols + c] = r[row];
                    }
                }
                if (c == 0 && !left)
#pragma unroll
                    for (int row = 0; row < ROWS; ++row)
                        if (row < rows) ex[2 * tcols + row] = r[row];
                if (c == cols - 1 && !right)
#pragma unroll
                    for (int row = 0; row < ROWS; ++row)
                        if (row < rows) ex[2 * tcols + trows + row] = r[row];
            }
            HIVC_TRACE(4);
            // x += alpha p while the other CTAs arrive (x is not read until the level ends);
            // the first streamed rows' loads go out before the resident rows are updated
            auto x_update = [&]() {
                if (!act) return;
                constexpr int kPre = 4;
                double xv[kPre];
#pragma unroll
                for (int j = 0; j < kPre; ++j) {
                    const int row = xr + j;
                    xv[j] = row < rows ? P.x[(size_t)(y0 + row) * w + gc] : 0.0;
                }
#pragma unroll
                for (int row = 0; row < ROWS; ++row) {
                    if (row < xr) {
                        double& xs = sx[row * tcols + c];
                        xs = xs + alpha * col[row * W2];
                    }
                }
#pragma unroll
                for (int j = 0; j < kPre; ++j) {
                    const int row = xr + j;
                    if (row < rows) P.x[(size_t)(y0 + row) * w + gc] = xv[j] + alpha * col[row * W2];
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
                        if (row < rows) P.x[(size_t)(y0 + row) * w + gc] = xw[j] + alpha * col[row * W2];
                    }
                }
            };
            double* bc = sh + 2 * 4 * 32 + red.bpar * 4;
            red.bpar ^= 1;
            if (kSyncWarp) {
                // The idle last warp runs the whole second grid sum (CTA partial, release
                // arrival, poll, fixed-order sum of the CTA partials) while the column
                // warps update x: neither waits for the other until the CTA barrier.
                // Same sums in the same order as cta_partial / sum_partials.
                const double v = warp_sum(e1[0]);
                double* buf = sh + red.par * 4 * 32;
                red.par ^= 1;
                if (lane == 0) buf[wid] = v;
                double* part = P.partials + ((red.epoch + 1) & 1) * kPartialBank;
                ++red.epoch;
                __syncthreads();
                if (wid == kSyncWid) {
                    if (lane == 0) {
                        double s = 0.0;
                        for (int i = 0; i < kTileThreads / 32; ++i) s += buf[i];
                        part[tile * 4] = s;
                        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.bar) : "memory");
                        const unsigned int target = red.epoch * (unsigned)nt;
                        wait_geq_acquire(P.bar, target);
                    }
                    __syncwarp();
                    double sum = 0.0;
                    if (nt <= 32 * kSumPer) {
                        double vals[kSumPer];
#pragma unroll
                        for (int j = 0; j < kSumPer; ++j) {
                            const int g = lane + 32 * j;
                            vals[j] = g < nt ? __ldcg(part + g * 4) : 0.0;
                        }
#pragma unroll
                        for (int j = 0; j < kSumPer; ++j)
                            if (lane + 32 * j < nt) sum += vals[j];
                    } else {
                        for (int g = lane; g < nt; g += 32) sum += __ldcg(part + g * 4);
                    }
                    sum = warp_sum(sum);
                    if (lane == 0) bc[0] = sum;
                } else {
                    x_update();
                }
                HIVC_TRACE(6);
                __syncthreads();
                // every tile's r edges are visible: the next iteration's halo loads go out
                if (act && !top) tr = __ldcg(ex_up);
                if (act && !bottom) br = __ldcg(ex_dn);
                if (hc && !left) lr = __ldcg(ex_lf);
                if (hc && !right) rr_ = __ldcg(ex_rt);
                e1[0] = bc[0];
            } else {
                grid_reduce_arrive<1>(e1, sh, P, red, tile);
                x_update();
                HIVC_TRACE(6);
                // once every CTA has arrived (so every tile's r edges are visible) the
                // next iteration's halo loads go out, then the partials are summed
                grid_wait(P.bar, nt, red.epoch);
                if (act && !top) tr = __ldcg(ex_up);
                if (act && !bottom) br = __ldcg(ex_dn);
                if (hc && !left) lr = __ldcg(ex_lf);
                if (hc && !right) rr_ = __ldcg(ex_rt);
                sum_partials<1>(P.partials + (red.epoch & 1) * kPartialBank, nt, bc);
                __syncthreads();
                e1[0] = bc[0];
            }
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

// The instantiation for a tile plan: exact shapes of the benchmark pyramids
// (1080x1920: 30x480; 540x960: 30x480, 23x480, 15x480), else the generic one.
using TileKernelFn = void (*)(TileBatch);
inline TileKernelFn tile_kernel_for(int trows, int tcols) {
    if (tcols == 480) {
        if (trows == 30) return cg_tile_kernel<30, 480>;
        if (trows == 23) return cg_tile_kernel<23, 480>;
        if (trows == 15) return cg_tile_kernel<15, 480>;
    }
    return cg_tile_kernel<kTileRows, 0>;
}
