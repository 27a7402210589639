// Host interface of the cascadic-CG inpainting kernels (inpaint.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "common.h"

#define CUDA_CHECK(expr)                                                                                  \
    do {                                                                                                  \
        cudaError_t _e = (expr);                                                                          \
        if (_e != cudaSuccess)                                                                            \
            ::hivc::fail(HIVC_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));                \
    } while (0)

namespace hivc {

// Device scratch for one solve at a time (per stream): finest-level CG
// vectors x, r, p (two buffers), A p, plus every coarser level's f, mask, u.
struct InpaintWorkspace {
    int device = -1;
    int num_sms = 0;
    int grid_ctas = 0;  // CTAs of the cooperative (grid-barrier) CG kernel
    size_t cap_px = 0, cap_coarse = 0;
    double* dbl = nullptr;
    uint8_t* bytes = nullptr;
    double* partials = nullptr;
    unsigned int* bar = nullptr;
    int* iters = nullptr;      // device: per level (coarse -> fine) CG iterations
    double* margins = nullptr; // device: per level min relative stop-test margin
    void reserve(int h, int w, int dev);
    void release();
    ~InpaintWorkspace() { release(); }
};

void pyramid_shapes(int h, int w, std::vector<std::pair<int, int>>& shapes);

// Queue the full cascadic solve of (f, m) on stream s; u_out receives the
// finest-level solution.  Returns the number of pyramid levels; per-level
// iteration counts land in ws.iters (coarse -> fine) on the device.
int solve_homogeneous_async(InpaintWorkspace& ws, cudaStream_t s, const double* f, const uint8_t* m, int h, int w,
                            double tol, int max_iter, double* u_out, int64_t* launches);

// Relative residual of the inpainting equation (homogeneous.py:206-211);
// synchronises the stream.  Returns -1 when ||f|mask|| == 0.
double strict_relative_residual(InpaintWorkspace& ws, cudaStream_t s, const double* u, const double* f,
                                const uint8_t* m, int h, int w, int64_t* launches);

}  // namespace hivc
