// Column-walk variant of cg_cluster_kernel (included by inpaint.cu) for
// cluster level sets whose bands are at most kColRows rows of at most
// kClThreads columns (every level of a 1080p / 540p pyramid up to 270x480).
//
// Same data placement as cg_cluster_kernel (one 16-CTA cluster per solve;
// DSMEM reductions and halo rows; x and the padded p in shared memory; only
// the r edge rows are exchanged, see phase 1), but thread c owns column c of its band for every row: r and A p
// stay in registers (phase 2 reuses the stencil of phase 1), the mask is one
// bit word per thread, and the 5-point stencil walks the column reading 3
// shared values per pixel.  Per-pixel float64 expressions are those of
// cg_cluster_kernel; the per-thread summation order of the dot products
// follows the column (fixed, deterministic).
#pragma once

constexpr int kColRows = 17;  // 16 x 17 rows >= 270 (the 270x480 level of a 1080p pyramid)

__global__ void __launch_bounds__(kClThreads, 1) cg_cluster_col_kernel(const __grid_constant__ ClusterBatch CB) {
    const ClusterLevels& S = CB.S[blockIdx.x / kClusterSize];
    extern __shared__ double smem_cl[];
    __shared__ double sh[2 * 4 * 32];
    __shared__ double red[2][4];
    __shared__ double bcast[2][4];
    __shared__ double s_vals[kCoarsest * kCoarsest];
    __shared__ int s_wcount[kCoarsest * kCoarsest / 32];
    __shared__ double s_mean;
    cgc::cluster_group cluster = cgc::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x;
    int par = 0, rpar = 0;

    auto creduce = [&](double* v, int nv) {  // fixed-order cluster-wide sum (as cg_cluster_kernel)
        {  // this CTA's sums: warp sums, then lane k of warp 0 adds value k's warp sums in warp order
            const int lane = tid & 31, wid = tid >> 5, nw = kClThreads >> 5;
            double* buf = sh + par * 4 * 32;
            par ^= 1;
            for (int k = 0; k < nv; ++k) v[k] = warp_sum(v[k]);
            if (lane == 0)
                for (int k = 0; k < nv; ++k) buf[k * 32 + wid] = v[k];
            __syncthreads();
            if (tid < nv) {
                double s = 0.0;
                for (int i = 0; i < nw; ++i) s += buf[tid * 32 + i];
                red[rpar][tid] = s;
            }
        }
        cluster.sync();
        if (tid < 32) {
            double s[4] = {0, 0, 0, 0};
            if (tid < kClusterSize) {
                const double* rr = cluster.map_shared_rank(&red[rpar][0], tid);
                for (int k = 0; k < nv; ++k) s[k] = rr[k];
            }
            for (int k = 0; k < nv; ++k) {
                double t = s[k];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (tid == 0) bcast[rpar][k] = t;
            }
        }
        __syncthreads();
        for (int k = 0; k < nv; ++k) v[k] = bcast[rpar][k];
        rpar ^= 1;
    };

    for (int li = 0; li < S.nlev; ++li) {
        const int h = S.h[li], w = S.w[li], W2 = w + 2;
        const double* __restrict__ f = S.f[li];
        const uint8_t* __restrict__ m = S.m[li];
        const bool coarsest = li == 0 && S.uc0 == nullptr;
        const bool finest = S.last_is_finest && li == S.nlev - 1;
        const double tol = finest ? S.tol : fmax(kLevelTol, S.tol);
        const double* uc = li == 0 ? S.uc0 : S.u[li - 1];
        const int hc = li == 0 ? S.hc0 : S.h[li - 1], wc = li == 0 ? S.wc0 : S.w[li - 1];
        const int band_rows = (h + kClusterSize - 1) / kClusterSize;
        const int y0 = min(rank * band_rows, h);
        const int rows = min(band_rows, h - y0);
        const bool top = y0 == 0, bottom = y0 + rows == h;
        const int c = tid;
        const bool act = c < w && rows > 0;
        // shared layout: padded p (band_rows+2) x (w+2) | x (band_rows*w) | ex_r 2w
        double* sp = smem_cl;
        double* sx = sp + (size_t)(band_rows + 2) * W2;
        double* exr = sx + (size_t)band_rows * w;

        if (coarsest) {  // x0 = mean(f[mask]), numpy pairwise order; every CTA computes it
            const bool in = tid < h * w;
            const bool mi = in && m[tid] != 0;
            const double fv = in ? f[tid] : 0.0;
            const unsigned bal = __ballot_sync(0xffffffffu, mi);
            const int lane = tid & 31, wid = tid >> 5;
            if (tid < kCoarsest * kCoarsest && lane == 0) s_wcount[wid] = __popc(bal);
            __syncthreads();
            if (mi) {
                int off = 0;
                for (int i = 0; i < wid; ++i) off += s_wcount[i];
                s_vals[off + __popc(bal & ((1u << lane) - 1u))] = fv;
            }
            __syncthreads();
            if (tid == 0) {
                int cnt = 0;
                for (int i = 0; i < (h * w + 31) / 32; ++i) cnt += s_wcount[i];
                s_mean = np_pairwise_sum(s_vals, cnt) / (double)cnt;
            }
            __syncthreads();
        }
        const double mean0 = coarsest ? s_mean : 0.0;
        auto x0_at = [&](int yy, int xx) -> double {  // homogeneous.py:133-154 / 188
            if (coarsest) return mean0;
            double ys = ((double)yy + 0.5) * ((double)hc / (double)h) - 0.5;
            double xs = ((double)xx + 0.5) * ((double)wc / (double)w) - 0.5;
            ys = fmin(fmax(ys, 0.0), (double)(hc - 1));
            xs = fmin(fmax(xs, 0.0), (double)(wc - 1));
            int ya = (int)floor(ys), xa = (int)floor(xs);
            int yb = min(ya + 1, hc - 1), xb = min(xa + 1, wc - 1);
            double wy = ys - (double)ya, wx = xs - (double)xa;
            double c00 = uc[ya * wc + xa], c01 = uc[ya * wc + xb], c10 = uc[yb * wc + xa], c11 = uc[yb * wc + xb];
            return (1 - wy) * ((1 - wx) * c00 + wx * c01) + wy * ((1 - wx) * c10 + wx * c11);
        };
        auto put = [&](int row, double v) {  // own value + the pad cells reflecting it
            double* q = sp + (row + 1) * W2 + c + 1;
            *q = v;
            if (c == 0) q[-1] = v;
            if (c == w - 1) q[1] = v;
            if (top && row == 0) q[-W2] = v;
            if (bottom && row == rows - 1) q[W2] = v;
        };
        // ---- setup A: x = x0 * interior on the own column and the halo rows
        uint32_t mbits = 0;
        if (act) {
#pragma unroll
            for (int row = 0; row < kColRows; ++row) {
                if (row >= rows) break;
                const int gi = (y0 + row) * w + c;
                const bool mi = m[gi] != 0;
                if (mi) mbits |= 1u << row;
                const double xv = x0_at(y0 + row, c) * (mi ? 0.0 : 1.0);
                sx[row * w + c] = xv;
                put(row, xv);
            }
            if (!top) sp[c + 1] = x0_at(y0 - 1, c) * (m[(y0 - 1) * w + c] ? 0.0 : 1.0);
            if (!bottom) sp[(rows + 1) * W2 + c + 1] = x0_at(y0 + rows, c) * (m[(y0 + rows) * w + c] ? 0.0 : 1.0);
        }
        __syncthreads();
        // ---- setup B: b = L(u_D) * interior, r = b - A x
        double r[kColRows], ap[kColRows];
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int row = 0; row < kColRows; ++row) {
            r[row] = 0.0;
            ap[row] = 0.0;
            if (!act || row >= rows) continue;
            const int yy = y0 + row, gi = yy * w + c;
            const bool mi = (mbits >> row) & 1u;
            const double interior = mi ? 0.0 : 1.0;
            auto ud = [&](int a, int b) -> double {
                const int k = a * w + b;
                return m[k] ? f[k] : 0.0;
            };
            const double udi = mi ? f[gi] : 0.0;
            const double b = lap_at(yy, c, h, w, udi, ud) * interior;
            const double* q = sp + (row + 1) * W2 + c + 1;
            const double ax = -((((q[0] * -4.0 + q[-W2]) + q[W2]) + q[-1]) + q[1]) * interior;
            r[row] = b - ax;
            acc[0] += r[row] * r[row];
            acc[1] += b * b;
            acc[2] += mi ? udi * udi : 0.0;
            acc[3] += interior;
        }
        creduce(acc, 4);  // (its barriers also end every read of the x halo in sp)
        double rs = acc[0];
        const bool all_mask = acc[3] == 0.0;
        const double bn = (finest && acc[2] != 0.0) ? sqrt(acc[2]) : sqrt(acc[1]);
        int it = 0;
        if (!all_mask && bn != 0.0) {
            // p0 = r on the band; publish edge rows of r and p0 for the neighbours
            if (act) {
#pragma unroll
                for (int row = 0; row < kColRows; ++row) {
                    if (row >= rows) break;
                    put(row, r[row]);
                }
                exr[c] = r[0];
#pragma unroll
                for (int row = 0; row < kColRows; ++row)
                    if (row == rows - 1) exr[w + c] = r[row];
            }
            cluster.sync();
            double beta = 0.0;
            for (int k = 1; k <= S.max_iter; ++k) {
                it = k;
                const bool tr = S.trace && li == S.nlev - 1 && rank == 0 && tid == 0 && k < 256;
                if (tr) S.trace[k * 8 + 0] = globaltimer_ns();
                // ---- phase 1: own p = r + beta p, then the halo rows: a halo cell already
                // holds the neighbour's previous p edge (computed here with the
                // neighbour's operands), so only its r edge row is read (DSMEM)
                if (act) {
                    const double hr_up = top ? 0.0 : cluster.map_shared_rank(exr, rank - 1)[w + c];
                    const double hr_dn = bottom ? 0.0 : cluster.map_shared_rank(exr, rank + 1)[c];
                    if (k > 1) {
#pragma unroll
                        for (int row = 0; row < kColRows; ++row) {
                            if (row >= rows) break;
                            put(row, r[row] + beta * sp[(row + 1) * W2 + c + 1]);
                        }
                    }
                    if (!top) sp[c + 1] = hr_up + beta * (k == 1 ? 0.0 : sp[c + 1]);
                    if (!bottom) sp[(rows + 1) * W2 + c + 1] = hr_dn + beta * (k == 1 ? 0.0 : sp[(rows + 1) * W2 + c + 1]);
                }
                __syncthreads();
                if (tr) S.trace[k * 8 + 1] = globaltimer_ns();
                double d[4] = {0.0, 0.0, 0.0, 0.0};
                if (act) {
                    const double* col = sp + c + 1;
                    double up = col[0], cur = col[W2];
#pragma unroll
                    for (int row = 0; row < kColRows; ++row) {
                        if (row >= rows) break;
                        const double* q = col + (row + 1) * W2;
                        const double dn = q[W2];
                        const double lap = (((cur * -4.0 + up) + dn) + q[-1]) + q[1];
                        ap[row] = -lap * (((mbits >> row) & 1u) ? 0.0 : 1.0);
                        d[0] += cur * ap[row];
                        up = cur;
                        cur = dn;
                    }
                }
                if (tr) S.trace[k * 8 + 2] = globaltimer_ns();
                creduce(d, 1);
                if (tr) S.trace[k * 8 + 3] = globaltimer_ns();
                const double pap = d[0];
                if (pap <= 0.0 || rs < 1e-300) break;
                const double alpha = rs / pap;
                double e[4] = {0.0, 0.0, 0.0, 0.0};
                if (act) {
#pragma unroll
                    for (int row = 0; row < kColRows; ++row) {
                        if (row >= rows) break;
                        const double pi = sp[(row + 1) * W2 + c + 1];
                        sx[row * w + c] = sx[row * w + c] + alpha * pi;
                        r[row] = r[row] - alpha * ap[row];
                        e[0] += r[row] * r[row];
                    }
                    exr[c] = r[0];
#pragma unroll
                    for (int row = 0; row < kColRows; ++row)
                        if (row == rows - 1) exr[w + c] = r[row];
                }
                if (tr) S.trace[k * 8 + 4] = globaltimer_ns();
                creduce(e, 1);
                if (tr) S.trace[k * 8 + 5] = globaltimer_ns();
                const double rs1 = e[0];
                if (sqrt(rs1) <= tol * bn) break;
                beta = rs1 / rs;
                rs = rs1;
            }
        }
        // ---- level solution u = u_D + x (f when the mask is full)
        if (act)
            for (int row = 0; row < rows; ++row) {
                const int gi = (y0 + row) * w + c;
                const bool mi = (mbits >> row) & 1u;
                S.u[li][gi] = all_mask ? f[gi] : (mi ? f[gi] : 0.0) + sx[row * w + c];
            }
        if (rank == 0 && tid == 0) *S.iters[li] = it;
        // the next level prolongs u from global memory written by every CTA of the cluster
        __threadfence();
        cluster.sync();
    }
}
