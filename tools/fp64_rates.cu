// Throughput of FP64 arithmetic vs FP64 conversions on one GPU (ops per clock per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_rates.cu -o tools/fp64_rates.bin
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_dadd(double* out, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    for (int i = 0; i < kIters; ++i) {
        x0 = x0 + a; x1 = x1 + a; x2 = x2 + a; x3 = x3 + a;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void k_i2f(double* out, int a) {
    int n = threadIdx.x;
    double s0 = 0, s1 = 0;
    for (int i = 0; i < kIters; ++i) {
        s0 += (double)(n + i);           // I2F.F64 + DADD
        s1 += (double)(unsigned)(n ^ i); // I2F.F64.U32 + DADD
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1;
}
__global__ void k_magic(double* out, int a) {
    int n = threadIdx.x;
    double s0 = 0, s1 = 0;
    for (int i = 0; i < kIters; ++i) {
        s0 += __hiloint2double(0x43300000, n + i) - 4503599627370496.0;
        s1 += __hiloint2double(0x43300000, n ^ i) - 4503599627370496.0;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1;
}
__global__ void k_frnd(double* out, double a) {
    double x0 = threadIdx.x * 0.37, x1 = x0 + 0.5;
    double s0 = 0, s1 = 0;
    for (int i = 0; i < kIters; ++i) {
        s0 += floor(x0 + s0 * 1e-300);
        s1 += rint(x1 + s1 * 1e-300);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1;
}
__global__ void k_f2i(double* out, double a) {
    double x0 = threadIdx.x * 0.37;
    int s0 = 0, s1 = 0;
    for (int i = 0; i < kIters; ++i) {
        s0 += (int)(x0 + (double)(s0 & 1));
        s1 += __double2int_rd(x0 + (double)(s1 & 1));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1;
}

template <class K, class A>
float time_kernel(K k, A a, double* out, int blocks, int threads) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<blocks, threads>>>(out, a);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    double* out;
    cudaMalloc(&out, (size_t)blocks * threads * sizeof(double));
    const double threads_total = (double)blocks * threads;
    auto rate = [&](float ms, double ops_per_thread) {
        return threads_total * ops_per_thread / (ms * 1e-3) / (sms * clk * 1e3);
    };
    float t;
    t = time_kernel(k_dadd, 1.0, out, blocks, threads);
    printf("DADD          %.1f ops/clk/SM\n", rate(t, 4.0 * kIters));
    t = time_kernel(k_i2f, 1, out, blocks, threads);
    printf("I2F.F64+DADD  %.1f (conv+add pairs)/clk/SM\n", rate(t, 2.0 * kIters));
    t = time_kernel(k_magic, 1, out, blocks, threads);
    printf("magic+DADD    %.1f (conv+add pairs)/clk/SM\n", rate(t, 2.0 * kIters));
    t = time_kernel(k_frnd, 1.0, out, blocks, threads);
    printf("FRND chain    %.1f ops/clk/SM\n", rate(t, 2.0 * kIters));
    t = time_kernel(k_f2i, 1.0, out, blocks, threads);
    printf("F2I chain     %.1f ops/clk/SM\n", rate(t, 2.0 * kIters));
    return 0;
}
