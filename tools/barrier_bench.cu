// Microbenchmark: cost of a grid-wide barrier (+ deterministic reduction) on
// B200 for the persistent CG kernels.  Build & run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/barrier_bench.cu -o /tmp/bb && /tmp/bb
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_v0(unsigned* bar, unsigned nb) {  // current: atomics + volatile spin + nanosleep
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = bar + 1;
        unsigned gen = *vgen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nb - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*vgen == gen) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// v1: monotonically increasing counter, no reset: target = (epoch+1) * nb
__device__ __forceinline__ void bar_v1(unsigned* bar, unsigned nb, unsigned& epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned target = (epoch + 1) * nb;
        atom_add_acqrel(bar, 1u);
        while (ld_acquire(bar) < target) {
        }
    }
    ++epoch;
    __syncthreads();
}

// v2: cluster-hierarchical: hardware cluster barrier, then one atomic per cluster
__device__ __forceinline__ void bar_v2(unsigned* bar, unsigned nclusters, unsigned& epoch) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
        unsigned target = (epoch + 1) * nclusters;
        atom_add_acqrel(bar, 1u);
        while (ld_acquire(bar) < target) {
        }
    }
    ++epoch;
    cl.sync();
}

template <int V>
__global__ void bench(unsigned* bar, int iters, double* partials, double* out) {
    __shared__ double s;
    unsigned epoch = 0;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) partials[blockIdx.x] = (double)(i + blockIdx.x);
        if (V == 0) bar_v0(bar, gridDim.x);
        if (V == 1) bar_v1(bar, gridDim.x, epoch);
        if (V == 2) bar_v2(bar, gridDim.x / 8, epoch);
        if (V == 3) cg::this_grid().sync();
        // deterministic reduction of the partials by warp 0, broadcast
        if (threadIdx.x < 32) {
            double t = 0;
            for (int g = threadIdx.x; g < (int)gridDim.x; g += 32) t += __ldcg(partials + g);
            for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (threadIdx.x == 0) s = t;
        }
        __syncthreads();
        acc += s;
        __syncthreads();
        if (V == 0) bar_v0(bar, gridDim.x);
        if (V == 1) bar_v1(bar, gridDim.x, epoch);
        if (V == 2) bar_v2(bar, gridDim.x / 8, epoch);
        if (V == 3) cg::this_grid().sync();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

template <int V>
float run(int nblocks, int threads, int iters, bool cluster) {
    unsigned* bar;
    double *partials, *out;
    cudaMalloc(&bar, 64);
    cudaMemset(bar, 0, 64);
    cudaMalloc(&partials, 4096 * 8);
    cudaMalloc(&out, 8);
    void* args[] = {&bar, &iters, &partials, &out};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
    if (cluster) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 8;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaLaunchKernelExC(&cfg, (const void*)bench<V>, args);
    cudaDeviceSynchronize();
    cudaMemset(bar, 0, 64);
    cudaEventRecord(a);
    cudaLaunchKernelExC(&cfg, (const void*)bench<V>, args);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
    cudaFree(bar);
    cudaFree(partials);
    cudaFree(out);
    return ms * 1e3f / iters;  // us per (2 barriers + 1 reduction)
}

int main() {
    int iters = 2000;
    for (int threads : {512, 1024}) {
        printf("threads %d: v0 (atomics+nanosleep) %.2f us | v1 (acq/rel counter) %.2f us | v3 (cg grid.sync) %.2f us | "
               "v2 (cluster8 hierarchical, 144 CTAs) %.2f us   [per 2 barriers + 1 reduction]\n",
               threads, run<0>(148, threads, iters, false), run<1>(148, threads, iters, false),
               run<3>(148, threads, iters, false), run<2>(144, threads, iters, true));
    }
    printf("v1 with 135 CTAs x 512: %.2f us\n", run<1>(135, 512, iters, false));
    return 0;
}
