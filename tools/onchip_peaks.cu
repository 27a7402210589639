// On-chip peaks of this B200, for the roofline denominators of the kernels
// whose working set never reaches HBM:
//   * shared-memory load bandwidth (LDS.128, all SMs, conflict free);
//   * L2 read bandwidth (a 32 MiB buffer resident in L2, ld.global.cg);
//   * HBM read bandwidth (a 2 GiB buffer, streaming);
//   * FP64 add / mul issue rate (DADD, DMUL: the CG and Brox kernels run with
//     FMA contraction off, so these are their arithmetic ceilings);
//   * software grid-barrier round trip (one acq_rel atomic per CTA + acquire
//     polling, as the CG level kernels use) at one CTA per SM, and a
//     thread-block-cluster barrier (barrier.cluster arrive/wait).
// Built and run by tools/onchip_peaks.py on the GPU box; prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/onchip_peaks.cu -o /tmp/onchip_peaks
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

constexpr int kSmemDoubles = 16384;  // 128 KiB
constexpr int kSmemIters = 4096;

__global__ void __launch_bounds__(1024) k_smem(double* out) {
    extern __shared__ double2 s2[];
    for (int i = threadIdx.x; i < kSmemDoubles / 2; i += blockDim.x) s2[i] = make_double2(i, i + 1);
    __syncthreads();
    double a0 = 0, a1 = 0, b0 = 0, b1 = 0;
    unsigned base = (unsigned)__cvta_generic_to_shared(s2);
    // lane-consecutive 16-byte words: conflict-free LDS.128; 4 independent loads per step
    unsigned idx = threadIdx.x;
    const unsigned mask = kSmemDoubles / 2 - 1;
#pragma unroll 4
    for (int i = 0; i < kSmemIters; i += 2) {
        double x0, x1, y0, y1;
        unsigned p0 = base + ((idx) & mask) * 16, p1 = base + ((idx + 1024) & mask) * 16;
        asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x0), "=d"(x1) : "r"(p0) : "memory");
        asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(y0), "=d"(y1) : "r"(p1) : "memory");
        a0 += x0;
        a1 += x1;
        b0 += y0;
        b1 += y1;
        idx += 2048;
    }
    if (a0 + a1 + b0 + b1 == -1.0) out[threadIdx.x] = a0;
}

__global__ void k_l2(const double2* __restrict__ buf, size_t n2, int reps, double* out) {
    double a = 0, b = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
            double2 v = __ldcg(buf + i);
            a += v.x;
            b += v.y;
        }
    if (a + b == -1.0) out[0] = a;
}

constexpr int kFpIters = 8192;
__global__ void k_dadd(double* out, double s) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < kFpIters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = x[j] + s;
    double t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += x[j];
    if (t == -1.0) out[0] = t;
}
__global__ void k_dmul(double* out, double s) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j + 1;
    for (int i = 0; i < kFpIters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = x[j] * s;
    double t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += x[j];
    if (t == -1.0) out[0] = t;
}

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__global__ void k_gridbar(unsigned* bar, int rounds) {
    unsigned epoch = 0;
    for (int r = 0; r < rounds; ++r) {
        __syncthreads();
        ++epoch;
        if (threadIdx.x == 0) {
            asm volatile("red.add.release.gpu.global.u32 [%0], 1;" : : "l"(bar) : "memory");
            while (ld_acq(bar) < epoch * gridDim.x) {
            }
        }
        __syncthreads();
    }
}
// two-level barrier: cluster barrier, then one arrival per cluster on the grid counter
__global__ void k_gridbar2(unsigned* bar, int rounds) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned ncl = gridDim.x / cl.num_blocks();
    const bool leader = cl.block_rank() == 0;
    unsigned epoch = 0;
    for (int r = 0; r < rounds; ++r) {
        cl.sync();
        ++epoch;
        if (threadIdx.x == 0) {
            if (leader) asm volatile("red.add.release.gpu.global.u32 [%0], 1;" : : "l"(bar) : "memory");
            while (ld_acq(bar) < epoch * ncl) {
            }
        }
        __syncthreads();
    }
}
// A full fixed-order grid sum of one double per thread, as the CG level kernel
// does it twice per iteration.  v1: every CTA publishes its partial and arrives
// on one counter, then a warp loads all CTA partials.  v2: CTA partials are
// summed per cluster over DSMEM, the cluster leader publishes and arrives, then
// a warp loads the cluster partials.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__global__ void __launch_bounds__(512) k_gridred1(unsigned* bar, double* part, int rounds, double* out) {
    __shared__ double buf[2][16];
    __shared__ double bc[2];
    unsigned epoch = 0;
    double v = threadIdx.x * 1e-3, acc = 0;
    for (int r = 0; r < rounds; ++r) {
        const int pb = r & 1;
        double s = warp_sum(v + acc * 1e-300);
        if ((threadIdx.x & 31) == 0) buf[pb][threadIdx.x >> 5] = s;
        __syncthreads();
        double* pp = part + pb * 2048;
        if (threadIdx.x == 0) {
            double t = 0;
            for (int i = 0; i < 16; ++i) t += buf[pb][i];
            pp[blockIdx.x] = t;
            ++epoch;
            asm volatile("red.add.release.gpu.global.u32 [%0], 1;" : : "l"(bar) : "memory");
            while (ld_acq(bar) < epoch * gridDim.x) {
            }
        } else {
            ++epoch;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            double vals[5], t = 0;
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const int g = threadIdx.x + 32 * j;
                vals[j] = g < (int)gridDim.x ? __ldcg(pp + g) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 5; ++j) t += vals[j];
            t = warp_sum(t);
            if (threadIdx.x == 0) bc[pb] = t;
        }
        __syncthreads();
        acc += bc[pb];
    }
    if (acc == -1.0) out[0] = acc;
}
__global__ void __launch_bounds__(512) k_gridred2(unsigned* bar, double* part, int rounds, double* out) {
    __shared__ double buf[2][16];
    __shared__ double cpart[2];
    __shared__ double bc[2];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned csz = cl.num_blocks(), ncl = gridDim.x / csz, crank = cl.block_rank();
    unsigned epoch = 0;
    double v = threadIdx.x * 1e-3, acc = 0;
    for (int r = 0; r < rounds; ++r) {
        const int pb = r & 1;
        double s = warp_sum(v + acc * 1e-300);
        if ((threadIdx.x & 31) == 0) buf[pb][threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0;
            for (int i = 0; i < 16; ++i) t += buf[pb][i];
            cpart[pb] = t;
        }
        cl.sync();
        double* pp = part + pb * 2048;
        ++epoch;
        if (crank == 0 && threadIdx.x < 32) {
            double t = (unsigned)threadIdx.x < csz ? *cl.map_shared_rank(&cpart[pb], threadIdx.x) : 0.0;
            t = warp_sum(t);
            if (threadIdx.x == 0) {
                pp[blockIdx.x / csz] = t;
                asm volatile("red.add.release.gpu.global.u32 [%0], 1;" : : "l"(bar) : "memory");
            }
        }
        if (threadIdx.x == 0)
            while (ld_acq(bar) < epoch * ncl) {
            }
        __syncthreads();
        if (threadIdx.x < 32) {
            double t = (unsigned)threadIdx.x < ncl ? __ldcg(pp + threadIdx.x) : 0.0;
            t = warp_sum(t);
            if (threadIdx.x == 0) bc[pb] = t;
        }
        __syncthreads();
        acc += bc[pb];
    }
    if (acc == -1.0) out[0] = acc;
}
__global__ void k_clusterbar(int rounds, double* out) {
    cg::cluster_group cl = cg::this_cluster();
    for (int r = 0; r < rounds; ++r) cl.sync();
    if (threadIdx.x == 0 && rounds < 0) out[0] = 1;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    double* out;
    CK(cudaMalloc(&out, 1 << 20));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto best = [&](auto launch, int reps) {
        float b = 1e30f;
        for (int i = 0; i < reps; ++i) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            b = std::min(b, time_ms(e0, e1));
        }
        return b;
    };

    // ---- shared memory
    const size_t smem = kSmemDoubles * sizeof(double);
    CK(cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int smem_ctas = sms;
    float ms = best([&] { k_smem<<<smem_ctas, 1024, smem>>>(out); }, 5);
    CK(cudaGetLastError());
    const double smem_bytes = (double)smem_ctas * 1024 * kSmemIters * 16;  // kSmemIters 16-byte loads per thread
    const double smem_gbs = smem_bytes / (ms * 1e-3) / 1e9;

    // ---- L2 (resident 32 MiB) and HBM (2 GiB streamed)
    const size_t l2_bytes = (size_t)32 << 20, hbm_bytes = (size_t)2 << 30;
    double2* buf;
    CK(cudaMalloc(&buf, hbm_bytes));
    CK(cudaMemset(buf, 0, hbm_bytes));
    const int l2_reps = 20;
    k_l2<<<sms * 4, 512>>>(buf, l2_bytes / 16, 1, out);  // warm
    ms = best([&] { k_l2<<<sms * 4, 512>>>(buf, l2_bytes / 16, l2_reps, out); }, 5);
    const double l2_gbs = (double)l2_bytes * l2_reps / (ms * 1e-3) / 1e9;
    ms = best([&] { k_l2<<<sms * 4, 512>>>(buf, hbm_bytes / 16, 1, out); }, 5);
    const double hbm_read_gbs = (double)hbm_bytes / (ms * 1e-3) / 1e9;
    CK(cudaGetLastError());

    // ---- FP64 issue rate (ops per clock per SM at the observed clock)
    ms = best([&] { k_dadd<<<sms * 8, 256>>>(out, 1e-9); }, 5);
    const double dadd_ops = (double)sms * 8 * 256 * kFpIters * 8;
    const double dadd_tflops = dadd_ops / (ms * 1e-3) / 1e12;
    ms = best([&] { k_dmul<<<sms * 8, 256>>>(out, 1.0000001); }, 5);
    const double dmul_tflops = dadd_ops / (ms * 1e-3) / 1e12;
    CK(cudaGetLastError());

    // ---- grid barrier (one CTA per SM, 512 threads) and cluster barrier (16 CTAs)
    unsigned* bar;
    CK(cudaMalloc(&bar, 64));
    const int rounds = 2000;
    int nb = sms - sms % 16;  // the CG tile kernel runs 144 CTAs
    std::vector<float> gb;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(bar, 0, 64);
        void* args[] = {&bar, (void*)&rounds};
        cudaEventRecord(e0);
        CK(cudaLaunchCooperativeKernel((const void*)k_gridbar, dim3(nb), dim3(512), args, 0, 0));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        gb.push_back(time_ms(e0, e1));
    }
    float gbest = 1e30f;
    for (float v : gb) gbest = std::min(gbest, v);
    const double gridbar_us = gbest * 1e3 / rounds;
    double clbar_us = -1;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nb);
        cfg.blockDim = dim3(512);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 16;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaFuncSetAttribute(k_clusterbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
            float b = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                if (cudaLaunchKernelEx(&cfg, k_clusterbar, rounds, out) != cudaSuccess) break;
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                b = std::min(b, time_ms(e0, e1));
            }
            if (b < 1e29f) clbar_us = b * 1e3 / rounds;
        }
        cudaGetLastError();
    }
    double bar2_us[2] = {-1, -1};
    CK(cudaFuncSetAttribute(k_gridbar2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int v = 0; v < 2; ++v) {
        const int csz = v == 0 ? 16 : 8;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nb);
        cfg.blockDim = dim3(512);
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csz;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeCooperative;
        attr[1].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        float b = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(bar, 0, 64);
            cudaEventRecord(e0);
            if (cudaLaunchKernelEx(&cfg, k_gridbar2, bar, rounds) != cudaSuccess) break;
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            b = std::min(b, time_ms(e0, e1));
        }
        if (b < 1e29f) bar2_us[v] = b * 1e3 / rounds;
        cudaGetLastError();
    }
    double red_us[3] = {-1, -1, -1};
    double* part;
    CK(cudaMalloc(&part, 4096 * sizeof(double)));
    {
        float b = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(bar, 0, 64);
            void* args[] = {&bar, &part, (void*)&rounds, &out};
            cudaEventRecord(e0);
            CK(cudaLaunchCooperativeKernel((const void*)k_gridred1, dim3(nb), dim3(512), args, 0, 0));
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            b = std::min(b, time_ms(e0, e1));
        }
        red_us[0] = b * 1e3 / rounds;
    }
    CK(cudaFuncSetAttribute(k_gridred2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int v = 0; v < 2; ++v) {
        const int csz = v == 0 ? 16 : 8;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nb);
        cfg.blockDim = dim3(512);
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csz;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeCooperative;
        attr[1].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        float b = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(bar, 0, 64);
            cudaEventRecord(e0);
            if (cudaLaunchKernelEx(&cfg, k_gridred2, bar, part, rounds, out) != cudaSuccess) break;
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            b = std::min(b, time_ms(e0, e1));
        }
        if (b < 1e29f) red_us[1 + v] = b * 1e3 / rounds;
        cudaGetLastError();
    }
    std::printf("{\"grid_sum_1level_us\": %.3f, \"grid_sum_2level_c16_us\": %.3f, \"grid_sum_2level_c8_us\": %.3f, ",
                red_us[0], red_us[1], red_us[2]);
    std::printf(
        "\"grid_barrier_2level_c16_us\": %.3f, \"grid_barrier_2level_c8_us\": %.3f, ", bar2_us[0], bar2_us[1]);
    std::printf(
        "\"sms\": %d, \"clock_mhz_attr\": %.0f, \"l2_bytes\": %d, \"smem_per_sm_bytes\": %zu, "
        "\"smem_load_GBps\": %.1f, \"l2_read_GBps\": %.1f, \"l2_probe_bytes\": %zu, \"hbm_read_GBps\": %.1f, "
        "\"dadd_TFLOPs\": %.3f, \"dmul_TFLOPs\": %.3f, \"grid_barrier_us\": %.3f, \"grid_barrier_ctas\": %d, "
        "\"cluster16_barrier_us\": %.3f}\n",
        sms, clk_khz / 1e3, prop.l2CacheSize, prop.sharedMemPerMultiprocessor, smem_gbs, l2_gbs, l2_bytes,
        hbm_read_gbs, dadd_tflops, dmul_tflops, gridbar_us, nb, clbar_us);
    return 0;
}
