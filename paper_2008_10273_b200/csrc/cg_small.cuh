// All coarse pyramid levels (<= 8192 px each) of one cascadic solve in ONE
// single-CTA launch (included by inpaint.cu).  Per level the search direction
// p lives in shared memory with a one-pixel pad ring holding the reflected
// edge values (so the 5-point stencil is branch-free), x in shared memory,
// r in registers; the level's solution u is written to global memory, where
// the next (finer) level prolongs it from.  Barriers are __syncthreads and
// the reductions are the same fixed-order block sums as the other CG
// kernels.  Per-pixel float64 expressions are those of cg_level_kernel.
#pragma once

constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxPx = 8192;
constexpr int kSmallPxT = kSmallMaxPx / kSmallThreads;  // pixels per thread
constexpr int kSmallMaxLevels = 16;

struct SmallLevels {
    int nlev;  // levels ordered coarse -> fine
    int h[kSmallMaxLevels], w[kSmallMaxLevels];
    const double* f[kSmallMaxLevels];
    const uint8_t* m[kSmallMaxLevels];
    double* u[kSmallMaxLevels];
    int* iters[kSmallMaxLevels];
    int last_is_finest;  // the finest level of this set is the pyramid's finest level
    double tol;
    int max_iter;
};

__global__ void __launch_bounds__(kSmallThreads, 1) cg_small_kernel(SmallLevels S) {
    extern __shared__ double smem_small[];
    __shared__ double sh[2 * 4 * 32];
    __shared__ double s_vals[kCoarsest * kCoarsest];
    __shared__ int s_wcount[kCoarsest * kCoarsest / 32];
    __shared__ double s_mean;
    const int tid = threadIdx.x;
    int par = 0;
    for (int li = 0; li < S.nlev; ++li) {
        const int h = S.h[li], w = S.w[li], n = h * w, W2 = w + 2;
        const double* __restrict__ f = S.f[li];
        const uint8_t* __restrict__ m = S.m[li];
        const bool coarsest = li == 0;
        const bool finest = S.last_is_finest && li == S.nlev - 1;
        const double tol = finest ? S.tol : fmax(kLevelTol, S.tol);
        const double* uc = coarsest ? nullptr : S.u[li - 1];
        const int hc = coarsest ? 0 : S.h[li - 1], wc = coarsest ? 0 : S.w[li - 1];
        double* sp = smem_small;                       // (h+2) x (w+2), padded p (and x0 during setup)
        double* sx = smem_small + (size_t)(h + 2) * W2;  // n
        uint8_t* smask = reinterpret_cast<uint8_t*>(sx + n);
        if (coarsest) {  // x0 = mean(f[mask]) with numpy's pairwise sum (homogeneous.py:188)
            // compact f[mask] in raster order (ballot + per-warp offsets), then one thread sums
            const bool in = tid < n;
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
                for (int i = 0; i < (n + 31) / 32; ++i) c += s_wcount[i];
                s_mean = np_pairwise_sum(s_vals, c) / (double)c;
            }
            __syncthreads();
        }
        const double mean0 = coarsest ? s_mean : 0.0;
        // stores v at (row, col) of the padded plane, plus the pad cells it reflects into
        auto put = [&](int row, int col, double v) {
            double* q = sp + (row + 1) * W2 + col + 1;
            *q = v;
            if (col == 0) q[-1] = v;
            if (col == w - 1) q[1] = v;
            if (row == 0) q[-W2] = v;
            if (row == h - 1) q[W2] = v;
        };
        auto lapp = [&](int row, int col) -> double {  // 5-point reflecting Laplacian from the padded plane
            const double* q = sp + (row + 1) * W2 + col + 1;
            return (((q[0] * -4.0 + q[-W2]) + q[W2]) + q[-1]) + q[1];
        };
        // ---- setup A: x = x0 * interior (homogeneous.py:71)
#pragma unroll
        for (int j = 0; j < kSmallPxT; ++j) {
            const int q = tid + j * kSmallThreads;
            if (q >= n) continue;
            const int row = q / w, col = q - (q / w) * w;
            const bool mi = m[q] != 0;
            smask[q] = mi;
            double x0;
            if (coarsest) {
                x0 = mean0;
            } else {  // homogeneous.py:133-154 at (row, col)
                double ys = ((double)row + 0.5) * ((double)hc / (double)h) - 0.5;
                double xs = ((double)col + 0.5) * ((double)wc / (double)w) - 0.5;
                ys = fmin(fmax(ys, 0.0), (double)(hc - 1));
                xs = fmin(fmax(xs, 0.0), (double)(wc - 1));
                int y0 = (int)floor(ys), xa = (int)floor(xs);
                int y1 = min(y0 + 1, hc - 1), xb = min(xa + 1, wc - 1);
                double wy = ys - (double)y0, wx = xs - (double)xa;
                double c00 = uc[y0 * wc + xa], c01 = uc[y0 * wc + xb], c10 = uc[y1 * wc + xa], c11 = uc[y1 * wc + xb];
                x0 = (1 - wy) * ((1 - wx) * c00 + wx * c01) + wy * ((1 - wx) * c10 + wx * c11);
            }
            const double xv = x0 * (mi ? 0.0 : 1.0);
            sx[q] = xv;
            put(row, col, xv);
        }
        __syncthreads();
        // ---- setup B: b = L(u_D) * interior, r = b - A x (homogeneous.py:65-72)
        double r[kSmallPxT];
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < kSmallPxT; ++j) {
            const int q = tid + j * kSmallThreads;
            r[j] = 0.0;
            if (q >= n) continue;
            const int row = q / w, col = q - (q / w) * w;
            const bool mi = smask[q] != 0;
            const double interior = mi ? 0.0 : 1.0;
            auto ud = [&](int yy, int xq) -> double {
                const int k = yy * w + xq;
                return m[k] ? f[k] : 0.0;
            };
            const double udi = mi ? f[q] : 0.0;
            const double b = lap_at(row, col, h, w, udi, ud) * interior;
            const double ax = -lapp(row, col) * interior;
            r[j] = b - ax;
            acc[0] += r[j] * r[j];
            acc[1] += b * b;
            acc[2] += mi ? udi * udi : 0.0;
            acc[3] += interior;
        }
        block_sum1<4>(acc, sh, par);  // (its barrier also ends every read of sp above)
        double rs = acc[0];
        const bool all_mask = acc[3] == 0.0;
        const double bn = (finest && acc[2] != 0.0) ? sqrt(acc[2]) : sqrt(acc[1]);
        int it = 0;
        if (!all_mask && bn != 0.0) {
#pragma unroll
            for (int j = 0; j < kSmallPxT; ++j) {  // p = r
                const int q = tid + j * kSmallThreads;
                if (q < n) put(q / w, q - (q / w) * w, r[j]);
            }
            __syncthreads();
            double beta = 0.0;
            for (int k = 1; k <= S.max_iter; ++k) {
                it = k;
                if (k > 1) {  // p = r + beta p
#pragma unroll
                    for (int j = 0; j < kSmallPxT; ++j) {
                        const int q = tid + j * kSmallThreads;
                        if (q >= n) continue;
                        const int row = q / w, col = q - (q / w) * w;
                        put(row, col, r[j] + beta * sp[(row + 1) * W2 + col + 1]);
                    }
                    __syncthreads();
                }
                double d[1] = {0.0};
#pragma unroll
                for (int j = 0; j < kSmallPxT; ++j) {
                    const int q = tid + j * kSmallThreads;
                    if (q >= n) continue;
                    const int row = q / w, col = q - (q / w) * w;
                    const double api = -lapp(row, col) * (smask[q] ? 0.0 : 1.0);
                    d[0] += sp[(row + 1) * W2 + col + 1] * api;
                }
                block_sum1<1>(d, sh, par);
                const double pap = d[0];
                if (pap <= 0.0 || rs < 1e-300) break;
                const double alpha = rs / pap;
                double e[1] = {0.0};
#pragma unroll
                for (int j = 0; j < kSmallPxT; ++j) {
                    const int q = tid + j * kSmallThreads;
                    if (q >= n) continue;
                    const int row = q / w, col = q - (q / w) * w;
                    const double pi = sp[(row + 1) * W2 + col + 1];
                    const double api = -lapp(row, col) * (smask[q] ? 0.0 : 1.0);
                    sx[q] = sx[q] + alpha * pi;
                    r[j] = r[j] - alpha * api;
                    e[0] += r[j] * r[j];
                }
                block_sum1<1>(e, sh, par);
                const double rs1 = e[0];
                if (sqrt(rs1) <= tol * bn) break;
                beta = rs1 / rs;
                rs = rs1;
            }
        }
        // level solution u = u_D + x (f when the mask is full); read by the next level's prolongation
        for (int q = tid; q < n; q += kSmallThreads) {
            const bool mi = smask[q] != 0;
            S.u[li][q] = all_mask ? f[q] : (mi ? f[q] : 0.0) + sx[q];
        }
        if (tid == 0) *S.iters[li] = it;
        __syncthreads();
    }
}
