// Brox-style variational backward flow (encoder side), reference flow.py:187-278.
//
// Float64 replay of the reference: scipy's Gaussian (separable 1-D
// correlations along y then x, reflect boundaries, symmetric accumulation
// centre-first then outermost pair inwards), the pixel-centre bilinear
// pyramid, clamped bilinear warp, one-sided/central differences, the lagged
// nonlinearity (psi_d, psi_g, psi_s), half-point diffusivities with zero
// border flux, damped Jacobi on the 2x2 systems, [-1, 1] increment clip and
// the 3x3 'nearest' median.  Every expression keeps numpy's association and
// FMA contraction is off, so the GPU flow matches the reference to rounding
// of ~1 ulp (tests/test_gpu_parity.py).
//
// Structure-of-arrays float64 planes; one launch per stage (the 30 Jacobi
// sweeps are 30 launches of one small kernel).  The whole launch sequence
// (~500 kernels per pyramid level) is captured once per shape / parameter set
// into a CUDA graph and replayed (HIVC_BROX_GRAPH=0: direct launches).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include <map>
#include <mutex>
#include <tuple>

#include "brox.h"
#include "func_attr.h"
#include "inpaint.h"

namespace hivc {

namespace {

constexpr int kT = 256;

inline int nblk(size_t n) { return (int)std::min<size_t>((n + kT - 1) / kT, 148 * 32); }

#define GRID_LOOP(i, n) for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (n); i += (size_t)gridDim.x * blockDim.x)

// Gaussian taps travel as a kernel parameter (not a __constant__ symbol):
// several contexts may run flows concurrently on their own streams.
struct Taps {
    double t[64];
};

// scipy.ndimage.correlate1d, mode 'reflect' (symmetric weights path)
__global__ void gauss_axis_kernel(const double* __restrict__ src, double* __restrict__ dst, int h, int w, int r,
                                  int axis, const __grid_constant__ Taps T) {
    const double* c_taps = T.t;
    const size_t n = (size_t)h * w;
    GRID_LOOP(i, n) {
        const int y = (int)(i / w), x = (int)(i % w);
        const int len = axis == 0 ? h : w;
        const int pos = axis == 0 ? y : x;
        auto at = [&](int p) -> double {  // 'reflect' (d c b a | a b c d | d c b a), any number of periods
            const int period = 2 * len;
            p %= period;
            if (p < 0) p += period;
            if (p >= len) p = period - 1 - p;
            return axis == 0 ? src[(size_t)p * w + x] : src[(size_t)y * w + p];
        };
        double acc = at(pos) * c_taps[r];
        for (int j = -r; j < 0; ++j) acc = acc + (at(pos + j) + at(pos - j)) * c_taps[r + j];
        dst[i] = acc;
    }
}

// bilinear_resize (flow.py:69-86), optionally * scale (flow upsampling, flow.py:239-240)
__global__ void resize_kernel(const double* __restrict__ src, int ih, int iw, double* __restrict__ dst, int h, int w,
                              double scale, int use_scale) {
    const size_t n = (size_t)h * w;
    GRID_LOOP(i, n) {
        const int y = (int)(i / w), x = (int)(i % w);
        double v;
        if (ih == h && iw == w) {
            v = src[i];
        } else {
            double ys = ((double)y + 0.5) * ((double)ih / (double)h) - 0.5;
            double xs = ((double)x + 0.5) * ((double)iw / (double)w) - 0.5;
            ys = fmin(fmax(ys, 0.0), (double)(ih - 1));
            xs = fmin(fmax(xs, 0.0), (double)(iw - 1));
            int y0 = (int)floor(ys), x0 = (int)floor(xs);
            int y1 = min(y0 + 1, ih - 1), x1 = min(x0 + 1, iw - 1);
            double fy = ys - (double)y0, fx = xs - (double)x0;
            double top = (1 - fx) * src[(size_t)y0 * iw + x0] + fx * src[(size_t)y0 * iw + x1];
            double bot = (1 - fx) * src[(size_t)y1 * iw + x0] + fx * src[(size_t)y1 * iw + x1];
            v = (1 - fy) * top + fy * bot;
        }
        dst[i] = use_scale ? v * scale : v;
    }
}

__device__ __forceinline__ double ddx_at(const double* a, int y, int x, int w) {  // flow.py:135-140
    const double* r = a + (size_t)y * w;
    if (x == 0) return r[1] - r[0];
    if (x == w - 1) return r[w - 1] - r[w - 2];
    return 0.5 * (r[x + 1] - r[x - 1]);
}
__device__ __forceinline__ double ddy_at(const double* a, int y, int x, int h, int w) {  // flow.py:143-148
    if (y == 0) return a[(size_t)w + x] - a[x];
    if (y == h - 1) return a[(size_t)(h - 1) * w + x] - a[(size_t)(h - 2) * w + x];
    return 0.5 * (a[(size_t)(y + 1) * w + x] - a[(size_t)(y - 1) * w + x]);
}

// clamped bilinear warp of tgt along (u, v) (flow.py:94-127)
__global__ void warp1_kernel(const double* __restrict__ tgt, const double* __restrict__ u, const double* __restrict__ v,
                             double* __restrict__ out, int h, int w) {
    const size_t n = (size_t)h * w;
    GRID_LOOP(k, n) {
        const int y = (int)(k / w), x = (int)(k % w);
        double sx = fmin(fmax((double)x + u[k], 0.0), (double)(w - 1));
        double sy = fmin(fmax((double)y + v[k], 0.0), (double)(h - 1));
        int x0 = (int)floor(sx), y0 = (int)floor(sy);
        int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
        double fx = sx - (double)x0, fy = sy - (double)y0;
        double w00 = (1 - fy) * (1 - fx), w01 = (1 - fy) * fx, w10 = fy * (1 - fx), w11 = fy * fx;
        out[k] = ((w00 * tgt[(size_t)y0 * w + x0] + w01 * tgt[(size_t)y0 * w + x1]) + w10 * tgt[(size_t)y1 * w + x0]) +
                 w11 * tgt[(size_t)y1 * w + x1];
    }
}

struct Lin {  // linearisation at the current warp (flow.py:222-230)
    double *ix, *iy, *iz, *ixx, *ixy, *iyy, *ixz, *iyz;
};

__global__ void deriv1_kernel(const double* __restrict__ wp, const double* __restrict__ ref, Lin L, int h, int w) {
    const size_t n = (size_t)h * w;
    GRID_LOOP(k, n) {
        const int y = (int)(k / w), x = (int)(k % w);
        double dxw = ddx_at(wp, y, x, w), dxr = ddx_at(ref, y, x, w);
        double dyw = ddy_at(wp, y, x, h, w), dyr = ddy_at(ref, y, x, h, w);
        L.ix[k] = 0.5 * (dxw + dxr);
        L.iy[k] = 0.5 * (dyw + dyr);
        L.iz[k] = wp[k] - ref[k];
        L.ixz[k] = dxw - dxr;
        L.iyz[k] = dyw - dyr;
    }
}

__global__ void deriv2_kernel(Lin L, int h, int w) {
    const size_t n = (size_t)h * w;
    GRID_LOOP(k, n) {
        const int y = (int)(k / w), x = (int)(k % w);
        L.ixx[k] = ddx_at(L.ix, y, x, w);
        L.ixy[k] = ddy_at(L.ix, y, x, h, w);
        L.iyy[k] = ddy_at(L.iy, y, x, h, w);
    }
}

struct Sys {  // per fixed-point step: 2x2 systems + diffusivity (flow.py:233-250)
    double *psi_d, *psi_g, *psi_s, *a11, *a12, *a22, *b1f, *b2f, *su, *sv;
};

// psi_d, psi_g (pointwise) and psi_s (needs neighbours of u+du, v+dv)
__global__ void robust_kernel(Lin L, Sys S, const double* __restrict__ u, const double* __restrict__ v,
                              const double* __restrict__ du, const double* __restrict__ dv, int h, int w, double gamma,
                              double eps2) {
    const size_t n = (size_t)h * w;
    GRID_LOOP(k, n) {
        const int y = (int)(k / w), x = (int)(k % w);
        double rb = (L.iz[k] + L.ix[k] * du[k]) + L.iy[k] * dv[k];
        S.psi_d[k] = 1.0 / sqrt(rb * rb + eps2);
        double rgx = (L.ixz[k] + L.ixx[k] * du[k]) + L.ixy[k] * dv[k];
        double rgy = (L.iyz[k] + L.ixy[k] * du[k]) + L.iyy[k] * dv[k];
        S.psi_g[k] = gamma / sqrt((rgx * rgx + rgy * rgy) + eps2);
        // ut = u + du, vt = v + dv evaluated at the stencil points
        auto ut = [&](int yy, int xx) { size_t q = (size_t)yy * w + xx; return u[q] + du[q]; };
        auto vt = [&](int yy, int xx) { size_t q = (size_t)yy * w + xx; return v[q] + dv[q]; };
        auto dx = [&](auto f) {
            if (x == 0) return f(y, 1) - f(y, 0);
            if (x == w - 1) return f(y, w - 1) - f(y, w - 2);
            return 0.5 * (f(y, x + 1) - f(y, x - 1));
        };
        auto dy = [&](auto f) {
            if (y == 0) return f(1, x) - f(0, x);
            if (y == h - 1) return f(h - 1, x) - f(h - 2, x);
            return 0.5 * (f(y + 1, x) - f(y - 1, x));
        };
        double gux = dx(ut), guy = dy(ut), gvx = dx(vt), gvy = dy(vt);
        double g2 = ((gux * gux + guy * guy) + gvx * gvx) + gvy * gvy;
        S.psi_s[k] = fmax(1.0 / sqrt(g2 + eps2), 0.05);
    }
}

// half-point weights with zero border flux (flow.py:173-184), edge-padded neighbours
struct W4 {
    double n, s, w, e;
};
__device__ __forceinline__ W4 weights_at(const double* __restrict__ psi, int y, int x, int h, int w) {
    const size_t k = (size_t)y * w + x;
    const double c = psi[k];
    W4 r;
    r.n = y == 0 ? 0.0 : 0.5 * (c + psi[k - w]);
    r.s = y == h - 1 ? 0.0 : 0.5 * (c + psi[k + w]);
    r.w = x == 0 ? 0.0 : 0.5 * (c + psi[k - 1]);
    r.e = x == w - 1 ? 0.0 : 0.5 * (c + psi[k + 1]);
    return r;
}
// _neighbor_sums with edge padding (flow.py:162-170)
__device__ __forceinline__ double nsum(const double* __restrict__ f, const W4& W, int y, int x, int h, int w) {
    const size_t k = (size_t)y * w + x;
    double fn = y == 0 ? f[k] : f[k - w];
    double fs = y == h - 1 ? f[k] : f[k + w];
    double fw = x == 0 ? f[k] : f[k - 1];
    double fe = x == w - 1 ? f[k] : f[k + 1];
    return ((W.n * fn + W.s * fs) + W.w * fw) + W.e * fe;
}

__global__ void system_kernel(Lin L, Sys S, const double* __restrict__ u, const double* __restrict__ v, int h, int w,
                              double alpha) {
    const size_t n = (size_t)h * w;
    GRID_LOOP(k, n) {
        const int y = (int)(k / w), x = (int)(k % w);
        W4 W = weights_at(S.psi_s, y, x, h, w);
        double wsum = ((W.n + W.s) + W.w) + W.e;
        double pd = S.psi_d[k], pg = S.psi_g[k];
        double ix = L.ix[k], iy = L.iy[k], iz = L.iz[k], ixx = L.ixx[k], ixy = L.ixy[k], iyy = L.iyy[k];
        double ixz = L.ixz[k], iyz = L.iyz[k];
        S.a11[k] = ((pd * ix) * ix + pg * (ixx * ixx + ixy * ixy)) + alpha * wsum;
        S.a12[k] = (pd * ix) * iy + pg * (ixx * ixy + ixy * iyy);
        S.a22[k] = ((pd * iy) * iy + pg * (ixy * ixy + iyy * iyy)) + alpha * wsum;
        S.b1f[k] = ((-pd) * ix) * iz - pg * (ixx * ixz + ixy * iyz);
        S.b2f[k] = ((-pd) * iy) * iz - pg * (ixy * ixz + iyy * iyz);
        S.su[k] = nsum(u, W, y, x, h, w) - wsum * u[k];
        S.sv[k] = nsum(v, W, y, x, h, w) - wsum * v[k];
    }
}

// one damped Jacobi sweep of the coupled 2x2 systems (flow.py:251-262); the
// last sweep also applies the [-1, 1] clip (flow.py:265-266)
__global__ void jacobi_kernel(Sys S, const double* __restrict__ du, const double* __restrict__ dv,
                              double* __restrict__ du_out, double* __restrict__ dv_out, int h, int w, double alpha,
                              int clip) {
    const size_t n = (size_t)h * w;
    GRID_LOOP(k, n) {
        const int y = (int)(k / w), x = (int)(k % w);
        W4 W = weights_at(S.psi_s, y, x, h, w);
        double b1 = S.b1f[k] + alpha * (S.su[k] + nsum(du, W, y, x, h, w));
        double b2 = S.b2f[k] + alpha * (S.sv[k] + nsum(dv, W, y, x, h, w));
        double a11 = S.a11[k], a12 = S.a12[k], a22 = S.a22[k];
        double det = a11 * a22 - a12 * a12;
        det = fabs(det) < 1e-12 ? 1e-12 : det;
        double dun = (a22 * b1 - a12 * b2) / det;
        double dvn = (a11 * b2 - a12 * b1) / det;
        double a = 0.5 * du[k] + 0.5 * dun;
        double b = 0.5 * dv[k] + 0.5 * dvn;
        if (clip) {
            a = fmin(fmax(a, -1.0), 1.0);
            b = fmin(fmax(b, -1.0), 1.0);
        }
        du_out[k] = a;
        dv_out[k] = b;
    }
}

// Two damped Jacobi sweeps per launch: du, dv of a 32x16 tile plus a 2-pixel
// halo in shared memory; the 2x2 systems are re-read from global memory in the
// second sweep, where they hit L1 (the tile's ~40 KB were just read), so the
// HBM-bound large levels move ~1.7x fewer bytes per sweep.  The halo ring is
// computed redundantly in sweep 1; sweep s is exact on the tile shrunk by s+1
// on interior sides, so the inner tile equals two jacobi_kernel launches bit
// for bit.
constexpr int kJ2TX = 32, kJ2TY = 16, kJ2H = 2, kJ2NT = 256;
constexpr int kJ2HX = kJ2TX + 2 * kJ2H, kJ2HY = kJ2TY + 2 * kJ2H, kJ2HN = kJ2HX * kJ2HY;

__global__ void __launch_bounds__(kJ2NT) jacobi2_kernel(Sys S, const double* __restrict__ du_in,
                                                       const double* __restrict__ dv_in, double* __restrict__ du_out,
                                                       double* __restrict__ dv_out, int h, int w, double alpha,
                                                       int nsweeps, int clip_last) {
    __shared__ double sm[4 * kJ2HN];
    double* cu = sm;
    double* cv = sm + kJ2HN;
    double* nu = sm + 2 * kJ2HN;
    double* nv = sm + 3 * kJ2HN;
    const int tid = threadIdx.x;
    const int gx0 = blockIdx.x * kJ2TX - kJ2H, gy0 = blockIdx.y * kJ2TY - kJ2H;
    for (int i = tid; i < kJ2HN; i += kJ2NT) {
        const int gx = gx0 + i % kJ2HX, gy = gy0 + i / kJ2HX;
        if (gx >= 0 && gx < w && gy >= 0 && gy < h) {
            const size_t g = (size_t)gy * w + gx;
            cu[i] = du_in[g];
            cv[i] = dv_in[g];
        }
    }
    __syncthreads();
    for (int sw = 0; sw < nsweeps; ++sw) {
        const bool clip = clip_last && sw == nsweeps - 1;
        for (int i = tid; i < kJ2HN; i += kJ2NT) {
            const int lx = i % kJ2HX, ly = i / kJ2HX, gx = gx0 + lx, gy = gy0 + ly;
            // exact region of this sweep: inside the image, sw+1 away from interior halo edges
            const int m = sw + 1;
            if (gx < 0 || gx >= w || gy < 0 || gy >= h) continue;
            if ((gy != 0 && ly < m) || (gy != h - 1 && ly > kJ2HY - 1 - m) || (gx != 0 && lx < m) ||
                (gx != w - 1 && lx > kJ2HX - 1 - m))
                continue;
            const size_t g = (size_t)gy * w + gx;
            const W4 W = weights_at(S.psi_s, gy, gx, h, w);
            const int in = gy == 0 ? i : i - kJ2HX, is = gy == h - 1 ? i : i + kJ2HX;
            const int iw = gx == 0 ? i : i - 1, ie = gx == w - 1 ? i : i + 1;
            const double nsu = ((W.n * cu[in] + W.s * cu[is]) + W.w * cu[iw]) + W.e * cu[ie];
            const double nsv = ((W.n * cv[in] + W.s * cv[is]) + W.w * cv[iw]) + W.e * cv[ie];
            const double b1 = S.b1f[g] + alpha * (S.su[g] + nsu);
            const double b2 = S.b2f[g] + alpha * (S.sv[g] + nsv);
            const double a11 = S.a11[g], a12 = S.a12[g], a22 = S.a22[g];
            double det = a11 * a22 - a12 * a12;
            det = fabs(det) < 1e-12 ? 1e-12 : det;
            const double dun = (a22 * b1 - a12 * b2) / det;
            const double dvn = (a11 * b2 - a12 * b1) / det;
            double a = 0.5 * cu[i] + 0.5 * dun;
            double b = 0.5 * cv[i] + 0.5 * dvn;
            if (clip) {
                a = fmin(fmax(a, -1.0), 1.0);
                b = fmin(fmax(b, -1.0), 1.0);
            }
            nu[i] = a;
            nv[i] = b;
        }
        __syncthreads();
        double* t = cu;
        cu = nu;
        nu = t;
        t = cv;
        cv = nv;
        nv = t;
    }
    for (int k = tid; k < kJ2TX * kJ2TY; k += kJ2NT) {
        const int lx = kJ2H + k % kJ2TX, ly = kJ2H + k / kJ2TX, gx = gx0 + lx, gy = gy0 + ly;
        if (gx < w && gy < h) {
            const size_t g = (size_t)gy * w + gx;
            du_out[g] = cu[ly * kJ2HX + lx];
            dv_out[g] = cv[ly * kJ2HX + lx];
        }
    }
}

// All sweeps of a small level (<= kJCMaxPx px) in ONE launch: one thread-block
// cluster of up to 16 CTAs, CTA c owning a band of rows.  Each thread keeps
// the 2x2 systems of its kJCPx pixels in registers (a11, a12, a22, the clamped
// determinant, b1f, b2f, su, sv) and their half-point weights in shared
// memory; du, dv live in shared memory (two buffers), and the band's halo
// rows are copied from the neighbouring CTAs' buffers over DSMEM at the start
// of every sweep, one cluster barrier per sweep.  Replaces 30 launches that
// are launch-latency bound below ~128 kpx; every expression is jacobi_kernel's,
// so the result is bit-identical.
constexpr int kJCNT = 512, kJCPx = 4, kJCMaxCtas = 16;
constexpr int kJCBand = kJCNT * kJCPx;  // px per CTA

__global__ void __launch_bounds__(kJCNT, 1) jacobi_cluster_kernel(Sys S, const double* __restrict__ du_in,
                                                                 const double* __restrict__ dv_in,
                                                                 double* __restrict__ du_out,
                                                                 double* __restrict__ dv_out, int h, int w, int rpc,
                                                                 double alpha, int iters, int clip_last) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ double jsm[];
    const int rank = (int)cluster.block_rank(), nct = (int)cluster.num_blocks();
    const int y0 = rank * rpc, rows = min(rpc, h - y0), np = rows * w;
    const int H = (rpc + 2) * w;  // band + halo rows
    double* Wn = jsm;             // [kJCBand] x 4 weights
    double* Ws = Wn + kJCBand;
    double* Ww = Ws + kJCBand;
    double* We = Ww + kJCBand;
    double* buf = We + kJCBand;  // [2][du, dv][H]
    const int tid = threadIdx.x;
    double a11[kJCPx], a12[kJCPx], a22[kJCPx], det[kJCPx], b1f[kJCPx], b2f[kJCPx], su[kJCPx], sv[kJCPx];
#pragma unroll
    for (int j = 0; j < kJCPx; ++j) {
        const int q = tid + j * kJCNT;
        if (q < np) {
            const int y = y0 + q / w, x = q % w;
            const size_t g = (size_t)y * w + x;
            const W4 W = weights_at(S.psi_s, y, x, h, w);
            Wn[q] = W.n;
            Ws[q] = W.s;
            Ww[q] = W.w;
            We[q] = W.e;
            a11[j] = S.a11[g];
            a12[j] = S.a12[g];
            a22[j] = S.a22[g];
            double d = a11[j] * a22[j] - a12[j] * a12[j];
            det[j] = fabs(d) < 1e-12 ? 1e-12 : d;
            b1f[j] = S.b1f[g];
            b2f[j] = S.b2f[g];
            su[j] = S.su[g];
            sv[j] = S.sv[g];
            buf[w + q] = du_in[g];
            buf[H + w + q] = dv_in[g];
        }
    }
    cluster.sync();
    for (int it = 0; it < iters; ++it) {
        double* cu = buf + (it & 1) * 2 * H;
        double* cv = cu + H;
        double* nu = buf + ((it + 1) & 1) * 2 * H;
        double* nv = nu + H;
        // halo rows: the upper CTA's last band row, the lower CTA's first
        if (rank > 0) {
            const double* pu = cluster.map_shared_rank(cu, rank - 1);
            const double* pv = cluster.map_shared_rank(cv, rank - 1);
            for (int x = tid; x < w; x += kJCNT) {
                cu[x] = pu[rpc * w + x];
                cv[x] = pv[rpc * w + x];
            }
        }
        if (rank < nct - 1) {
            const double* pu = cluster.map_shared_rank(cu, rank + 1);
            const double* pv = cluster.map_shared_rank(cv, rank + 1);
            for (int x = tid; x < w; x += kJCNT) {
                cu[(rows + 1) * w + x] = pu[w + x];
                cv[(rows + 1) * w + x] = pv[w + x];
            }
        }
        __syncthreads();
        const bool clip = clip_last && it == iters - 1;
#pragma unroll
        for (int j = 0; j < kJCPx; ++j) {
            const int q = tid + j * kJCNT;
            if (q < np) {
                const int y = y0 + q / w, x = q % w;
                const int i = w + q;
                const int in = y == 0 ? i : i - w, is = y == h - 1 ? i : i + w;
                const int iw = x == 0 ? i : i - 1, ie = x == w - 1 ? i : i + 1;
                const double wn = Wn[q], ws = Ws[q], ww = Ww[q], we = We[q];
                const double nsu = ((wn * cu[in] + ws * cu[is]) + ww * cu[iw]) + we * cu[ie];
                const double nsv = ((wn * cv[in] + ws * cv[is]) + ww * cv[iw]) + we * cv[ie];
                const double b1 = b1f[j] + alpha * (su[j] + nsu);
                const double b2 = b2f[j] + alpha * (sv[j] + nsv);
                const double dun = (a22[j] * b1 - a12[j] * b2) / det[j];
                const double dvn = (a11[j] * b2 - a12[j] * b1) / det[j];
                double a = 0.5 * cu[i] + 0.5 * dun;
                double b = 0.5 * cv[i] + 0.5 * dvn;
                if (clip) {
                    a = fmin(fmax(a, -1.0), 1.0);
                    b = fmin(fmax(b, -1.0), 1.0);
                }
                nu[i] = a;
                nv[i] = b;
            }
        }
        cluster.sync();
    }
    const double* fu = buf + (iters & 1) * 2 * H;
    const double* fv = fu + H;
#pragma unroll
    for (int j = 0; j < kJCPx; ++j) {
        const int q = tid + j * kJCNT;
        if (q < np) {
            const size_t g = (size_t)y0 * w + q;
            du_out[g] = fu[w + q];
            dv_out[g] = fv[w + q];
        }
    }
}

// Cluster layout of a level for jacobi_cluster_kernel (rows per CTA, CTAs), or
// {0, 0} when the level does not fit (then the per-sweep launches run).
struct JcPlan {
    int rpc = 0, ctas = 0;
    size_t smem = 0;
};
// Whether one cluster of `ctas` CTAs with `smem` bytes each can be resident
// on this device (cudaOccupancyMaxActiveClusters), cached per device.
static bool jc_cluster_fits(int ctas, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, size_t>, bool> cache;
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(dev, ctas, smem);
    auto f = cache.find(key);
    if (f != cache.end()) return f->second;
    ensure_func_attr((const void*)jacobi_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    ensure_func_attr((const void*)jacobi_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kJCNT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ctas;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    const bool ok = cudaOccupancyMaxActiveClusters(&n, jacobi_cluster_kernel, &cfg) == cudaSuccess && n > 0;
    cudaGetLastError();  // (a rejected query leaves no sticky error)
    cache[key] = ok;
    return ok;
}

static JcPlan jc_plan(int h, int w) {
    JcPlan p;
    static const int max_px = [] {
        const char* e = debug_opt("brox_jc_max");
        return e ? std::atoi(e) : kJCMaxCtas * kJCBand;
    }();
    if ((long long)h * w > max_px || w > kJCBand) return p;
    const int ctas = std::min(kJCMaxCtas, h);
    const int rpc = (h + ctas - 1) / ctas;
    if ((long long)rpc * w > kJCBand) return p;
    const size_t smem = (size_t)(4 * kJCBand + 4 * (rpc + 2) * w) * sizeof(double);
    if (smem > 200 * 1024) return p;
    const int nctas = (h + rpc - 1) / rpc;
    if (!jc_cluster_fits(nctas, smem)) return p;  // then the per-sweep launches run
    p.rpc = rpc;
    p.ctas = nctas;
    p.smem = smem;
    return p;
}

static void launch_jacobi_cluster(const JcPlan& jp, const Sys& S, const double* du, const double* dv, double* du2,
                                  double* dv2, int h, int w, double alpha, int iters, cudaStream_t s) {
    ensure_func_attr((const void*)jacobi_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    ensure_func_attr((const void*)jacobi_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(jp.ctas);
    cfg.blockDim = dim3(kJCNT);
    cfg.dynamicSmemBytes = jp.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = jp.ctas;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel, S, du, dv, du2, dv2, h, w, jp.rpc, alpha, iters, 1));
}

__device__ __forceinline__ void cswap(double& a, double& b) {
    double lo = fmin(a, b), hi = fmax(a, b);
    a = lo;
    b = hi;
}

// u = median3(u + du) with 'nearest' boundaries (flow.py:269-276)
__global__ void median_update_kernel(const double* __restrict__ u, const double* __restrict__ du,
                                     double* __restrict__ out, int h, int w) {
    const size_t n = (size_t)h * w;
    GRID_LOOP(k, n) {
        const int y = (int)(k / w), x = (int)(k % w);
        double a[9];
        int t = 0;
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int yy = min(max(y + dy, 0), h - 1), xx = min(max(x + dx, 0), w - 1);
                size_t q = (size_t)yy * w + xx;
                a[t++] = u[q] + du[q];
            }
        // median of 9 (Paeth's network)
        cswap(a[1], a[2]); cswap(a[4], a[5]); cswap(a[7], a[8]);
        cswap(a[0], a[1]); cswap(a[3], a[4]); cswap(a[6], a[7]);
        cswap(a[1], a[2]); cswap(a[4], a[5]); cswap(a[7], a[8]);
        cswap(a[0], a[3]); cswap(a[5], a[8]); cswap(a[4], a[7]);
        cswap(a[3], a[6]); cswap(a[1], a[4]); cswap(a[2], a[5]);
        cswap(a[4], a[7]); cswap(a[4], a[2]); cswap(a[6], a[4]);
        cswap(a[4], a[2]);
        out[k] = a[4];
    }
}

__global__ void clip_kernel(double* __restrict__ a, size_t n, double bound) {
    GRID_LOOP(k, n) a[k] = fmin(fmax(a[k], -bound), bound);
}

}  // namespace

// ---------------------------------------------------------------- host driver

std::vector<std::pair<int, int>> brox_shapes(int h, int w, double scale, int min_size) {
    std::vector<std::pair<int, int>> out{{h, w}};
    while (std::min(out.back().first, out.back().second) > min_size) {  // flow.py:151-159
        int nh = std::max((int)std::nearbyint(out.back().first * scale), min_size);
        int nw = std::max((int)std::nearbyint(out.back().second * scale), min_size);
        if (nh == out.back().first && nw == out.back().second) break;
        out.push_back({nh, nw});
    }
    return out;
}

void BroxWorkspace::reserve(int h, int w, int levels_px) {
    size_t n = (size_t)h * w;
    if (n <= cap && (size_t)levels_px <= cap_pyr) return;
    release();
    size_t total = (size_t)kPlanes * n + 2 * (size_t)levels_px + 4 * n;  // + graph I/O planes
    CUDA_CHECK(cudaMalloc(&base, total * sizeof(double)));
    cap = n;
    cap_pyr = levels_px;
}

void BroxWorkspace::release() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    key.clear();
    if (base) cudaFree(base);
    base = nullptr;
    cap = cap_pyr = 0;
}

static void set_taps(Taps& T, int& radius, const double* host_taps, int ntaps) {
    radius = (ntaps - 1) / 2;
    for (int i = 0; i < ntaps && i < 64; ++i) T.t[i] = host_taps[i];
}

// levels of at least HIVC_BROX_J2_MIN pixels (default 1 Mpx: the HBM-bound
// ones) run two Jacobi sweeps per launch; 0 disables (measured at 1080p /
// pyramid 0.95: 242 ms per pair -> 234 ms; on smaller levels it does not pay)
static int jacobi2_min_px() {
    static const int v = [] {
        const char* e = debug_opt("brox_j2_min");
        return e ? std::atoi(e) : (1 << 20);
    }();
    return v;
}

// The whole estimator as a launch sequence on stream s (captured once per
// shape/parameter set into a CUDA graph by brox_flow).
static void enqueue_brox(BroxWorkspace& ws, cudaStream_t s, const std::vector<std::pair<int, int>>& shapes,
                         const std::vector<size_t>& lofs, int levels_px, const double* frame_t,
                         const double* frame_prev, int h, int w, const BroxParamsC& P, const double* taps_pre,
                         int ntaps_pre, const double* taps_aa, int ntaps_aa, double* u_out, double* v_out,
                         int64_t* launches) {
    const int L = (int)shapes.size();
    const size_t N = (size_t)h * w;
    double* pl = ws.base;
    auto plane = [&](int i) { return pl + (size_t)i * N; };
    double* refs = pl + (size_t)BroxWorkspace::kPlanes * N;
    double* tgts = refs + levels_px;
    double *tmp = plane(0), *tmp2 = plane(1);
    double *u = plane(2), *v = plane(3), *u2 = plane(4), *v2 = plane(5);
    double *du = plane(6), *dv = plane(7), *du2 = plane(8), *dv2 = plane(9), *wp = plane(10);
    Lin Lz{plane(11), plane(12), plane(13), plane(14), plane(15), plane(16), plane(17), plane(18)};
    Sys Sz{plane(19), plane(20), plane(21), plane(22), plane(23), plane(24), plane(25), plane(26), plane(27), plane(28)};
    int r = 0;
    Taps taps{};
    auto gauss = [&](const double* src, double* dst, int hh, int ww) {
        gauss_axis_kernel<<<nblk((size_t)hh * ww), kT, 0, s>>>(src, tmp2, hh, ww, r, 0, taps);
        gauss_axis_kernel<<<nblk((size_t)hh * ww), kT, 0, s>>>(tmp2, dst, hh, ww, r, 1, taps);
        *launches += 2;
    };
    // presmoothing (flow.py:197-199) into pyramid level 0
    if (P.presmooth_sigma > 0) {
        set_taps(taps, r, taps_pre, ntaps_pre);
        gauss(frame_t, refs, h, w);
        gauss(frame_prev, tgts, h, w);
    } else {
        CUDA_CHECK(cudaMemcpyAsync(refs, frame_t, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(tgts, frame_prev, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    // recursive pyramid (flow.py:201-208): smooth the previous level, then resample
    set_taps(taps, r, taps_aa, ntaps_aa);
    for (int l = 1; l < L; ++l) {
        const int ph = shapes[l - 1].first, pw = shapes[l - 1].second, hh = shapes[l].first, ww = shapes[l].second;
        for (double* pyr : {refs, tgts}) {
            gauss(pyr + lofs[l - 1], tmp, ph, pw);
            resize_kernel<<<nblk((size_t)hh * ww), kT, 0, s>>>(tmp, ph, pw, pyr + lofs[l], hh, ww, 1.0, 0);
            ++*launches;
        }
    }
    const double eps2 = P.eps * P.eps;
    for (int l = L - 1; l >= 0; --l) {
        const int hh = shapes[l].first, ww = shapes[l].second;
        const size_t n = (size_t)hh * ww;
        const int nb = nblk(n);
        const double* ref = refs + lofs[l];
        const double* tgt = tgts + lofs[l];
        if (l == L - 1) {
            CUDA_CHECK(cudaMemsetAsync(u, 0, n * sizeof(double), s));
            CUDA_CHECK(cudaMemsetAsync(v, 0, n * sizeof(double), s));
        } else {
            const int ph = shapes[l + 1].first, pw = shapes[l + 1].second;
            resize_kernel<<<nb, kT, 0, s>>>(u, ph, pw, u2, hh, ww, (double)ww / (double)pw, 1);
            resize_kernel<<<nb, kT, 0, s>>>(v, ph, pw, v2, hh, ww, (double)hh / (double)ph, 1);
            *launches += 2;
            std::swap(u, u2);
            std::swap(v, v2);
        }
        for (int wi = 0; wi < P.warps; ++wi) {
            warp1_kernel<<<nb, kT, 0, s>>>(tgt, u, v, wp, hh, ww);
            deriv1_kernel<<<nb, kT, 0, s>>>(wp, ref, Lz, hh, ww);
            deriv2_kernel<<<nb, kT, 0, s>>>(Lz, hh, ww);
            *launches += 3;
            CUDA_CHECK(cudaMemsetAsync(du, 0, n * sizeof(double), s));
            CUDA_CHECK(cudaMemsetAsync(dv, 0, n * sizeof(double), s));
            for (int fp = 0; fp < P.fixed_point_iters; ++fp) {
                robust_kernel<<<nb, kT, 0, s>>>(Lz, Sz, u, v, du, dv, hh, ww, P.gamma, eps2);
                system_kernel<<<nb, kT, 0, s>>>(Lz, Sz, u, v, hh, ww, P.alpha);
                *launches += 2;
                const JcPlan jp = P.solver_iters > 0 ? jc_plan(hh, ww) : JcPlan{};
                if (jp.ctas > 0) {  // all sweeps in one cluster launch
                    launch_jacobi_cluster(jp, Sz, du, dv, du2, dv2, hh, ww, P.alpha, P.solver_iters, s);
                    ++*launches;
                    std::swap(du, du2);
                    std::swap(dv, dv2);
                    continue;
                }
                const bool two = jacobi2_min_px() > 0 && n >= (size_t)jacobi2_min_px();
                const dim3 g2((ww + kJ2TX - 1) / kJ2TX, (hh + kJ2TY - 1) / kJ2TY);
                for (int it = 0; it < P.solver_iters;) {
                    const int k = two ? std::min(2, P.solver_iters - it) : 1;
                    const bool last = it + k == P.solver_iters;
                    if (two)
                        jacobi2_kernel<<<g2, kJ2NT, 0, s>>>(Sz, du, dv, du2, dv2, hh, ww, P.alpha, k, last);
                    else
                        jacobi_kernel<<<nb, kT, 0, s>>>(Sz, du, dv, du2, dv2, hh, ww, P.alpha, last);
                    ++*launches;
                    std::swap(du, du2);
                    std::swap(dv, dv2);
                    it += k;
                }
                if (P.solver_iters == 0) {  // clip still applies
                    clip_kernel<<<nb, kT, 0, s>>>(du, n, 1.0);
                    clip_kernel<<<nb, kT, 0, s>>>(dv, n, 1.0);
                    *launches += 2;
                }
            }
            median_update_kernel<<<nb, kT, 0, s>>>(u, du, u2, hh, ww);
            median_update_kernel<<<nb, kT, 0, s>>>(v, dv, v2, hh, ww);
            *launches += 2;
            std::swap(u, u2);
            std::swap(v, v2);
        }
    }
    const double bound = (double)std::max(h, w);  // flow.py:277-278
    clip_kernel<<<nblk(N), kT, 0, s>>>(u, N, bound);
    clip_kernel<<<nblk(N), kT, 0, s>>>(v, N, bound);
    *launches += 2;
    CUDA_CHECK(cudaMemcpyAsync(u_out, u, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(v_out, v, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CUDA_CHECK(cudaGetLastError());
}

void brox_flow(BroxWorkspace& ws, cudaStream_t s, const double* frame_t, const double* frame_prev, int h, int w,
               const BroxParamsC& P, const double* taps_pre, int ntaps_pre, const double* taps_aa, int ntaps_aa,
               double* u_out, double* v_out, int64_t* launches) {
    auto shapes = brox_shapes(h, w, P.pyramid_scale, P.min_size);
    const int L = (int)shapes.size();
    int levels_px = 0;
    std::vector<size_t> lofs(L);
    for (int l = 0; l < L; ++l) {
        lofs[l] = levels_px;
        levels_px += shapes[l].first * shapes[l].second;
    }
    ws.reserve(h, w, levels_px);
    static const bool use_graph = [] {
        const char* e = debug_opt("brox_graph");
        return !(e && e[0] == '0');
    }();
    if (!use_graph) {
        enqueue_brox(ws, s, shapes, lofs, levels_px, frame_t, frame_prev, h, w, P, taps_pre, ntaps_pre, taps_aa,
                     ntaps_aa, u_out, v_out, launches);
        return;
    }
    // ~500 launches per pyramid level (84 levels at pyramid_scale 0.95): replay a
    // captured graph over fixed workspace planes instead of launching each kernel
    const size_t N = (size_t)h * w;
    double* io = ws.base + (size_t)BroxWorkspace::kPlanes * N + 2 * (size_t)levels_px;  // in_t, in_p, out_u, out_v
    std::vector<double> key{(double)h, (double)w, P.alpha, P.gamma, P.pyramid_scale, (double)P.min_size,
                            (double)P.warps, (double)P.fixed_point_iters, (double)P.solver_iters, P.eps,
                            P.presmooth_sigma, (double)ntaps_pre, (double)ntaps_aa, (double)(uintptr_t)ws.base};
    key.insert(key.end(), taps_pre, taps_pre + ntaps_pre);
    key.insert(key.end(), taps_aa, taps_aa + ntaps_aa);
    if (!ws.exec || ws.key != key) {
        if (ws.exec) cudaGraphExecDestroy(ws.exec);
        ws.exec = nullptr;
        int64_t n = 0;
        cudaGraph_t g;
        CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_brox(ws, s, shapes, lofs, levels_px, io, io + N, h, w, P, taps_pre, ntaps_pre, taps_aa, ntaps_aa,
                         io + 2 * N, io + 3 * N, &n);
        } catch (...) {  // leave the stream out of capture mode before reporting the error
            cudaGraph_t bad = nullptr;
            cudaStreamEndCapture(s, &bad);
            if (bad) cudaGraphDestroy(bad);
            cudaGetLastError();
            throw;
        }
        CUDA_CHECK(cudaStreamEndCapture(s, &g));
        CUDA_CHECK(cudaGraphInstantiate(&ws.exec, g, 0));
        CUDA_CHECK(cudaGraphDestroy(g));
        ws.key = key;
        ws.graph_launches = n;
    }
    CUDA_CHECK(cudaMemcpyAsync(io, frame_t, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(io + N, frame_prev, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CUDA_CHECK(cudaGraphLaunch(ws.exec, s));
    CUDA_CHECK(cudaMemcpyAsync(u_out, io + 2 * N, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(v_out, io + 3 * N, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    *launches += ws.graph_launches;
}

// ---------------------------------------------------------------- Horn-Schunck (flow.py:281-316)

namespace {

// fx = 0.5 (dx(im1) + dx(im2)), fy likewise, ft = im2 - im1, denom = alpha^2 + fx^2 + fy^2
__global__ void hs_deriv_kernel(const double* __restrict__ im1, const double* __restrict__ im2, double* __restrict__ fx,
                                double* __restrict__ fy, double* __restrict__ ft, double* __restrict__ den, int h,
                                int w, double alpha) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)h * w) return;
    const int y = (int)(i / w), x = (int)(i % w);
    // _dx: interior 0.5 (a[x+1] - a[x-1]); x = 0: a[1] - a[0]; x = w-1: a[w-1] - a[w-2]
    const bool ix = x > 0 && x < w - 1;
    const size_t xl = ix ? i - 1 : (x == 0 ? i : i - 1), xr = ix ? i + 1 : (x == 0 ? i + 1 : i);
    const bool iy = y > 0 && y < h - 1;
    const size_t yu = iy ? i - w : (y == 0 ? i : i - w), yd = iy ? i + w : (y == 0 ? i + w : i);
    auto dx = [&](const double* a) { return ix ? 0.5 * (a[xr] - a[xl]) : a[xr] - a[xl]; };
    auto dy = [&](const double* a) { return iy ? 0.5 * (a[yd] - a[yu]) : a[yd] - a[yu]; };
    const double gx = 0.5 * (dx(im1) + dx(im2)), gy = 0.5 * (dy(im1) + dy(im2));
    fx[i] = gx;
    fy[i] = gy;
    ft[i] = im2[i] - im1[i];
    den[i] = alpha * alpha + gx * gx + gy * gy;
}

// one Jacobi sweep: 8-neighbour average (edge padding, taps in the reference's
// (dy, dx) order), then u = ua - fx c, v = va - fy c, c = (fx ua + fy va + ft) / denom
__global__ void hs_iter_kernel(const double* __restrict__ u, const double* __restrict__ v,
                               const double* __restrict__ fx, const double* __restrict__ fy,
                               const double* __restrict__ ft, const double* __restrict__ den, double* __restrict__ u2,
                               double* __restrict__ v2, int h, int w) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)h * w) return;
    const int y = (int)(i / w), x = (int)(i % w);
    const double k1 = 1.0 / 12.0, k2 = 1.0 / 6.0;
    const int ys[3] = {max(y - 1, 0), y, min(y + 1, h - 1)};
    const int xs[3] = {max(x - 1, 0), x, min(x + 1, w - 1)};
    const double kk[3][3] = {{k1, k2, k1}, {k2, 0.0, k2}, {k1, k2, k1}};
    double ua = 0.0, va = 0.0;
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
            if (dy == 1 && dx == 1) continue;
            const size_t j = (size_t)ys[dy] * w + xs[dx];
            ua = ua + kk[dy][dx] * u[j];
            va = va + kk[dy][dx] * v[j];
        }
    const double gx = fx[i], gy = fy[i];
    const double c = (gx * ua + gy * va + ft[i]) / den[i];
    u2[i] = ua - gx * c;
    v2[i] = va - gy * c;
}

}  // namespace

void horn_schunck_flow(BroxWorkspace& ws, cudaStream_t s, const double* frame_t, const double* frame_prev, int h,
                       int w, double alpha, int iterations, double* u_out, double* v_out, int64_t* launches) {
    ws.reserve(h, w, 0);
    const size_t N = (size_t)h * w;
    double* fx = ws.base;
    double *fy = fx + N, *ft = fy + N, *den = ft + N, *ua = den + N, *va = ua + N;
    const int nb = (int)((N + 255) / 256);
    hs_deriv_kernel<<<nb, 256, 0, s>>>(frame_t, frame_prev, fx, fy, ft, den, h, w, alpha);
    // ping-pong so that the last sweep writes u_out / v_out
    double *a_u = (iterations % 2 == 0) ? u_out : ua, *a_v = (iterations % 2 == 0) ? v_out : va;
    double *b_u = (iterations % 2 == 0) ? ua : u_out, *b_v = (iterations % 2 == 0) ? va : v_out;
    CUDA_CHECK(cudaMemsetAsync(a_u, 0, N * sizeof(double), s));
    CUDA_CHECK(cudaMemsetAsync(a_v, 0, N * sizeof(double), s));
    for (int it = 0; it < iterations; ++it) {
        hs_iter_kernel<<<nb, 256, 0, s>>>(a_u, a_v, fx, fy, ft, den, b_u, b_v, h, w);
        std::swap(a_u, b_u);
        std::swap(a_v, b_v);
    }
    *launches += 1 + iterations;
    CUDA_CHECK(cudaGetLastError());
}

}  // namespace hivc
