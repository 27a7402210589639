// Host interface of the Brox flow kernels (brox.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <vector>

namespace hivc {

struct BroxParamsC {  // flow.BroxParams (flow.py:56-66)
    double alpha = 40.0, gamma = 40.0, pyramid_scale = 0.5;
    int min_size = 16, warps = 3, fixed_point_iters = 5, solver_iters = 30;
    double eps = 1e-3, presmooth_sigma = 0.8;
};

struct BroxWorkspace {
    static constexpr int kPlanes = 29;  // full-resolution float64 scratch planes
    double* base = nullptr;
    size_t cap = 0, cap_pyr = 0;
    cudaGraphExec_t exec = nullptr;  // captured launch sequence (brox_flow)
    std::vector<double> key;         // shape, parameters, taps, workspace base of `exec`
    int64_t graph_launches = 0;
    void reserve(int h, int w, int levels_px);
    void release();
    ~BroxWorkspace() { release(); }
};

std::vector<std::pair<int, int>> brox_shapes(int h, int w, double scale, int min_size);

// Queue the whole flow computation on stream s.  frame_t / frame_prev / u / v:
// device float64 planes (h*w).  taps_*: host arrays of scipy's normalised
// Gaussian taps (presmoothing sigma and the anti-alias sigma 0.5/scale).
void brox_flow(BroxWorkspace& ws, cudaStream_t s, const double* frame_t, const double* frame_prev, int h, int w,
               const BroxParamsC& P, const double* taps_pre, int ntaps_pre, const double* taps_aa, int ntaps_aa,
               double* u_out, double* v_out, int64_t* launches);

// flow.flow_horn_schunck (flow.py:281-316): `iterations` Jacobi sweeps, float64, on stream s.
void horn_schunck_flow(BroxWorkspace& ws, cudaStream_t s, const double* frame_t, const double* frame_prev, int h,
                       int w, double alpha, int iterations, double* u_out, double* v_out, int64_t* launches);

}  // namespace hivc
