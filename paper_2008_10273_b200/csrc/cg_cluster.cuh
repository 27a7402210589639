// Coarse and mid pyramid levels (<= 16 x 8192 px) of one cascadic solve in
// ONE thread-block-cluster launch (included by inpaint.cu).
//
// A cluster of kClusterSize CTAs (one per SM) owns the level; CTA c holds a
// band of rows entirely on chip — r in registers, x and the padded search
// direction p in shared memory.  The two dot products per CG iteration are
// reduced through distributed shared memory (each CTA's partial in its own
// smem, read by every CTA in rank order after barrier.cluster), and the band
// halos are rebuilt from the neighbours' published edge rows of r and p
// (read through DSMEM) — so an iteration needs two hardware cluster barriers
// and no global-memory traffic at all.  Different solves' clusters run
// concurrently on different SMs.  Per-pixel float64 expressions are those of
// cg_level_kernel; reductions are fixed-order and identical in every CTA.
#pragma once
// (inpaint.cu includes <cooperative_groups.h> at global scope)

constexpr int kClusterSize = 16;
constexpr int kClThreads = 512;
constexpr int kClPx = 16;   // band pixels per thread: r in registers (8192 per CTA)
constexpr int kClMaxW = 4096;
constexpr int kClMaxLevels = 16;

struct ClusterLevels {
    int nlev;  // coarse -> fine
    int h[kClMaxLevels], w[kClMaxLevels];
    const double* f[kClMaxLevels];
    const uint8_t* m[kClMaxLevels];
    double* u[kClMaxLevels];
    int* iters[kClMaxLevels];
    const double* uc0;  // coarser solution prolonged into level 0 (nullptr: level 0 is the coarsest)
    int hc0, wc0;
    int last_is_finest;
    double tol;
    int max_iter;
    unsigned long long* trace;  // HIVC_CG_TRACE diagnostics (finest cluster level, rank 0)
};

struct ClusterBatch {  // one cluster per solve (blockIdx.x / kClusterSize)
    ClusterLevels S[kMaxBatch];
};

namespace cgc = cooperative_groups;

__global__ void __launch_bounds__(kClThreads, 1) cg_cluster_kernel(const __grid_constant__ ClusterBatch CB) {
    const ClusterLevels& S = CB.S[blockIdx.x / kClusterSize];
    extern __shared__ double smem_cl[];
    __shared__ double sh[2 * 4 * 32];
    __shared__ double red[2][4];     // this CTA's partials (double-buffered)
    __shared__ double bcast[2][4];
    __shared__ double s_vals[kCoarsest * kCoarsest];
    __shared__ int s_wcount[kCoarsest * kCoarsest / 32];
    __shared__ double s_mean;
    cgc::cluster_group cluster = cgc::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x;
    int par = 0, rpar = 0;

    // fixed-order cluster-wide sum of NV values (identical in every CTA)
    auto creduce = [&](double* v, int nv) {
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
        // shared layout: padded p (band_rows+2) x (w+2) | x (band_rows*w) | ex_r 2w | ex_p 2x2w | mask
        double* sp = smem_cl;
        double* sx = sp + (size_t)(band_rows + 2) * W2;
        double* exr = sx + (size_t)band_rows * w;
        double* exp_ = exr + 2 * w;
        uint8_t* smask = reinterpret_cast<uint8_t*>(exp_ + 4 * w);

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
                int c = 0;
                for (int i = 0; i < (h * w + 31) / 32; ++i) c += s_wcount[i];
                s_mean = np_pairwise_sum(s_vals, c) / (double)c;
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
        auto put = [&](int row, int col, double v) {  // own value + the pad cells reflecting it
            double* q = sp + (row + 1) * W2 + col + 1;
            *q = v;
            if (col == 0) q[-1] = v;
            if (col == w - 1) q[1] = v;
            if (top && row == 0) q[-W2] = v;
            if (bottom && row == rows - 1) q[W2] = v;
        };
        auto lapp = [&](int row, int col) -> double {
            const double* q = sp + (row + 1) * W2 + col + 1;
            return (((q[0] * -4.0 + q[-W2]) + q[W2]) + q[-1]) + q[1];
        };
        // thread t owns band pixels q = t + 512 j (row, col packed; -1 when past the band)
        int rc[kClPx];
#pragma unroll
        for (int j = 0; j < kClPx; ++j) {
            const int q = tid + kClThreads * j;
            rc[j] = q < rows * w ? ((q / w) << 16) | (q % w) : -1;
        }
        // ---- setup A: x = x0 * interior on the band and on its halo rows
#pragma unroll
        for (int j = 0; j < kClPx; ++j) {
            if (rc[j] < 0) continue;
            const int row = rc[j] >> 16, col = rc[j] & 0xFFFF;
            const int gi = (y0 + row) * w + col;
            const bool mi = m[gi] != 0;
            smask[row * w + col] = mi;
            const double xv = x0_at(y0 + row, col) * (mi ? 0.0 : 1.0);
            sx[row * w + col] = xv;
            put(row, col, xv);
        }
        for (int col = tid; col < w && rows > 0; col += kClThreads) {
            if (!top) sp[col + 1] = x0_at(y0 - 1, col) * (m[(y0 - 1) * w + col] ? 0.0 : 1.0);
            if (!bottom) sp[(rows + 1) * W2 + col + 1] = x0_at(y0 + rows, col) * (m[(y0 + rows) * w + col] ? 0.0 : 1.0);
        }
        __syncthreads();
        // ---- setup B: b = L(u_D) * interior, r = b - A x
        double r[kClPx];
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < kClPx; ++j) {
            r[j] = 0.0;
            if (rc[j] < 0) continue;
            const int row = rc[j] >> 16, col = rc[j] & 0xFFFF;
            const int yy = y0 + row, gi = yy * w + col;
            const bool mi = smask[row * w + col] != 0;
            const double interior = mi ? 0.0 : 1.0;
            auto ud = [&](int a, int b) -> double {
                const int k = a * w + b;
                return m[k] ? f[k] : 0.0;
            };
            const double udi = mi ? f[gi] : 0.0;
            const double b = lap_at(yy, col, h, w, udi, ud) * interior;
            const double ax = -lapp(row, col) * interior;
            r[j] = b - ax;
            acc[0] += r[j] * r[j];
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
#pragma unroll
            for (int j = 0; j < kClPx; ++j) {
                if (rc[j] < 0) continue;
                const int row = rc[j] >> 16, col = rc[j] & 0xFFFF;
                put(row, col, r[j]);
                if (row == 0) exr[col] = exp_[col] = r[j];
                if (row == rows - 1) exr[w + col] = exp_[w + col] = r[j];
            }
            cluster.sync();
            double beta = 0.0;
            for (int k = 1; k <= S.max_iter; ++k) {
                it = k;
                const int pp = (k - 1) & 1, cp = k & 1;  // ex_p parity read / written this iteration
                // ---- phase 1: halo p = r + beta p from the neighbours' edge rows (DSMEM), own p update
                const bool tr = S.trace && li == S.nlev - 1 && rank == 0 && tid == 0 && k < 256;
                if (tr) S.trace[k * 8 + 0] = globaltimer_ns();
                if (rows > 0) {
                    const double* up_r = top ? nullptr : cluster.map_shared_rank(exr, rank - 1);
                    const double* up_p = top ? nullptr : cluster.map_shared_rank(exp_, rank - 1);
                    const double* dn_r = bottom ? nullptr : cluster.map_shared_rank(exr, rank + 1);
                    const double* dn_p = bottom ? nullptr : cluster.map_shared_rank(exp_, rank + 1);
                    for (int col = tid; col < w; col += kClThreads) {
                        if (!top) sp[col + 1] = up_r[w + col] + beta * up_p[pp * 2 * w + w + col];
                        if (!bottom) sp[(rows + 1) * W2 + col + 1] = dn_r[col] + beta * dn_p[pp * 2 * w + col];
                    }
                }
                if (k > 1) {
#pragma unroll
                    for (int j = 0; j < kClPx; ++j) {
                        if (rc[j] < 0) continue;
                        const int row = rc[j] >> 16, col = rc[j] & 0xFFFF;
                        put(row, col, r[j] + beta * sp[(row + 1) * W2 + col + 1]);
                    }
                }
                __syncthreads();
                if (tr) S.trace[k * 8 + 1] = globaltimer_ns();
                double d[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int j = 0; j < kClPx; ++j) {
                    if (rc[j] < 0) continue;
                    const int row = rc[j] >> 16, col = rc[j] & 0xFFFF;
                    const double api = -lapp(row, col) * (smask[row * w + col] ? 0.0 : 1.0);
                    d[0] += sp[(row + 1) * W2 + col + 1] * api;
                }
                for (int col = tid; col < w && rows > 0; col += kClThreads) {  // publish p edge rows
                    exp_[cp * 2 * w + col] = sp[W2 + col + 1];
                    exp_[cp * 2 * w + w + col] = sp[rows * W2 + col + 1];
                }
                if (tr) S.trace[k * 8 + 2] = globaltimer_ns();
                creduce(d, 1);
                if (tr) S.trace[k * 8 + 3] = globaltimer_ns();
                const double pap = d[0];
                if (pap <= 0.0 || rs < 1e-300) break;
                const double alpha = rs / pap;
                double e[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int j = 0; j < kClPx; ++j) {
                    if (rc[j] < 0) continue;
                    const int row = rc[j] >> 16, col = rc[j] & 0xFFFF;
                    const double pi = sp[(row + 1) * W2 + col + 1];
                    const double api = -lapp(row, col) * (smask[row * w + col] ? 0.0 : 1.0);
                    sx[row * w + col] = sx[row * w + col] + alpha * pi;
                    r[j] = r[j] - alpha * api;
                    e[0] += r[j] * r[j];
                    if (row == 0) exr[col] = r[j];
                    if (row == rows - 1) exr[w + col] = r[j];
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
        for (int row = 0; row < rows; ++row)
            for (int col = tid; col < w; col += kClThreads) {
                const int gi = (y0 + row) * w + col;
                const bool mi = smask[row * w + col] != 0;
                S.u[li][gi] = all_mask ? f[gi] : (mi ? f[gi] : 0.0) + sx[row * w + col];
            }
        if (rank == 0 && tid == 0) *S.iters[li] = it;
        // the next level prolongs u from global memory written by every CTA of the cluster
        __threadfence();
        cluster.sync();
    }
}
