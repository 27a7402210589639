// Device-side building blocks shared by the HIVC kernels.
//
// All float work is IEEE float64 with FMA contraction disabled (-fmad=false)
// so every expression rounds exactly as the numpy reference does; the
// association of each sum is spelled out to match the reference's order.
#pragma once

#include <cstdint>

#include "aan_constants.h"

namespace hivc {

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------- reductions
// Deterministic block-wide sum: fixed shuffle tree inside each warp, then the
// warp partials summed in warp order by warp 0.  `sh` needs blockDim/32 doubles.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sh /* [NV][32] */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) sh[k * 32 + wid] = v[k];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double t = lane < nw ? sh[k * 32 + lane] : 0.0;
            v[k] = warp_sum(t);
        }
    }
    __syncthreads();
    if (wid == 0 && lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) sh[k * 32] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = sh[k * 32];
    __syncthreads();
}

// Same fixed-order block sum with ONE __syncthreads: warp partials go to one
// of two shared buffers (alternating per call, `par`), and every thread sums
// the warp partials itself in warp order.  Reusing a buffer two calls later is
// safe because every thread passed the intermediate call's barrier after its
// reads.  `sh` needs 2 * NV * 32 doubles.
template <int NV>
__device__ __forceinline__ void block_sum1(double (&v)[NV], double* sh, int& par) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* buf = sh + par * NV * 32;
    par ^= 1;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) buf[k * 32 + wid] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double s = 0.0;
        for (int i = 0; i < nw; ++i) s += buf[k * 32 + i];
        v[k] = s;
    }
}

// Software grid barrier for cooperative launches (all CTAs co-resident).
// bar[0] is a monotonically increasing arrival counter (zeroed before the
// launch); barrier number e completes when it reaches e * nblocks.  One
// acq_rel atomic per CTA plus acquire polling: ~1.7 us per barrier on B200
// (tools/barrier_bench.cu), vs ~2.6 us for reset/generation + __threadfence.
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_relaxed_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Wait until *bar >= target.  The spin uses relaxed loads: an acquire load
// invalidates the SM's L1 (CCTL.IVALL) every time, which stalls the other
// warps' shared-memory traffic for as long as the poll runs; one acquire
// load of the final value then orders the caller's later reads.
__device__ __forceinline__ void wait_geq_acquire(const unsigned int* bar, unsigned int target) {
    while (ld_relaxed_gpu(bar) < target) {
    }
    (void)ld_acquire_gpu(bar);
}
// Barrier tail for callers that already synchronised the CTA after their last
// global writes (e.g. through block_sum1): thread 0 arrives and waits, then
// the CTA is released.
__device__ __forceinline__ void grid_arrive_wait(unsigned int* bar, unsigned int nblocks, unsigned int& epoch) {
    ++epoch;
    if (threadIdx.x == 0) {
        unsigned int old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        const unsigned int target = epoch * nblocks;
        if (old + 1 != target)  // the last arrival knows from its own atomic (no poll round trip)
            wait_geq_acquire(bar, target);
    }
    __syncthreads();
}

// Split form: arrive (after a CTA barrier that ordered the CTA's global
// writes), independent work, then wait.
// The arrival is a release reduction: nothing waits for its round trip, so
// the work between arrive and wait (its loads included) starts at once.
__device__ __forceinline__ void grid_arrive(unsigned int* bar, unsigned int& epoch) {
    ++epoch;
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void grid_wait(const unsigned int* bar, unsigned int nblocks, unsigned int epoch) {
    if (threadIdx.x == 0) {
        const unsigned int target = epoch * nblocks;
        wait_geq_acquire(bar, target);
    }
    __syncthreads();
}

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks, unsigned int& epoch) {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        unsigned int old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        const unsigned int target = epoch * nblocks;
        wait_geq_acquire(bar, target);
    }
    __syncthreads();
}

// numpy's pairwise summation (np.add.reduce on a contiguous float64 array):
// < 8 terms sequential from 0.0; <= 128 terms 8 strided accumulators; else
// recursive halves split at a multiple of 8.  Serial; small arrays only.
__device__ inline double np_pairwise_sum(const double* a, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// ---------------------------------------------------------------- AAN butterflies (pseudodiff.py:47-117)
__device__ __forceinline__ void aan_fwd(double (&v)[8]) {
    double s07 = v[0] + v[7], d07 = v[0] - v[7];
    double s16 = v[1] + v[6], d16 = v[1] - v[6];
    double s25 = v[2] + v[5], d25 = v[2] - v[5];
    double s34 = v[3] + v[4], d34 = v[3] - v[4];
    double e0 = s07 + s34, e3 = s07 - s34;
    double e1 = s16 + s25, e2 = s16 - s25;
    v[0] = e0 + e1;
    v[4] = e0 - e1;
    double rot = (e2 + e3) * kF_C4;
    v[2] = e3 + rot;
    v[6] = e3 - rot;
    double o0 = d34 + d25, o1 = d25 + d16, o2 = d16 + d07;
    double q = (o0 - o2) * kF_C6;
    double ra = kF_C6R2 * o0 + q;
    double rb = kF_C2R2 * o2 + q;
    double rc = o1 * kF_C4;
    double lo = d07 + rc, hi = d07 - rc;
    v[5] = hi + ra;
    v[3] = hi - ra;
    v[1] = lo + rb;
    v[7] = lo - rb;
}

__device__ __forceinline__ void aan_inv(double (&v)[8]) {
    double p0 = v[0] + v[4], p1 = v[0] - v[4];
    double q13 = v[2] + v[6];
    double q12 = (v[2] - v[6]) * kI_R2 - q13;
    double e0 = p0 + q13, e3 = p0 - q13, e1 = p1 + q12, e2 = p1 - q12;
    double m13 = v[5] + v[3], m10 = v[5] - v[3], m11 = v[1] + v[7], m12 = v[1] - v[7];
    double o7 = m11 + m13;
    double o11 = (m11 - m13) * kI_R2;
    double z = (m10 + m12) * kI_2C2;
    double o10 = kI_K3 * m12 - z;
    double o12 = (-kI_K4) * m10 + z;
    double o6 = o12 - o7, o5 = o11 - o6, o4 = o10 + o5;
    v[0] = e0 + o7;
    v[1] = e1 + o6;
    v[2] = e2 + o5;
    v[3] = e3 - o4;
    v[4] = e3 + o4;
    v[5] = e2 - o5;
    v[6] = e1 - o6;
    v[7] = e0 - o7;
}

// One 8x8 block reconstruction u = IDCT(eig * DCT(mc)) + a, computed by the
// 8 lanes [lane0, lane0+8) of a warp on the shared tile `t` (row-major, row
// stride LD doubles: 8, or 9 so the row passes of 8 lanes hit 8 different
// bank pairs instead of 4-way conflicts).  On entry t holds mc; on exit the reconstruction.
// Mirrors dct2_aan_8x8 / idct2_aan_8x8 / reconstruct_blocks operation by
// operation (pseudodiff.py:141-152, 275-279).
template <int LD = 8>
__device__ __forceinline__ void block_reconstruct_8lanes(double* t, int j, const double* eig, double a,
                                                         unsigned mask8) {
    double v[8];
    // forward pass along x for row j
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = t[j * LD + i];
    aan_fwd(v);
#pragma unroll
    for (int i = 0; i < 8; ++i) t[j * LD + i] = v[i];
    __syncwarp(mask8);
    // forward pass along y for column j, scale, eigenvalues, inverse scale
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = t[i * LD + j];
    aan_fwd(v);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        // (lane-indexed tables: global memory through L1, see aan_constants.h)
        double c = v[i] * __ldg(kFwdScale2 + i * 8 + j);  // dct2: * _FSCALE2
        c = __ldg(eig + i * 8 + j) * c;                   // eig * dct2(mc)
        v[i] = c * __ldg(kInvScale2 + i * 8 + j);         // idct2: coef * _ISCALE2
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) t[i * LD + j] = v[i];
    __syncwarp(mask8);
    // inverse pass along x for row j
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = t[j * LD + i];
    aan_inv(v);
#pragma unroll
    for (int i = 0; i < 8; ++i) t[j * LD + i] = v[i];
    __syncwarp(mask8);
    // inverse pass along y for column j, + a
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = t[i * LD + j];
    aan_inv(v);
#pragma unroll
    for (int i = 0; i < 8; ++i) t[i * LD + j] = v[i] + a;
    __syncwarp(mask8);
}

}  // namespace hivc
