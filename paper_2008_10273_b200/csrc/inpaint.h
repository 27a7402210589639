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

constexpr int kMaxBatch = 16;  // solves per batched launch
constexpr int kTraceLen = 2048 + 256 * 160;  // HIVC_CG_TRACE: phase stamps + per-CTA arrival stamps

// Device scratch for one solve at a time (per stream): finest-level CG
// vectors x, r, p (two buffers), A p, plus every coarser level's f, mask, u.
struct InpaintWorkspace {
    int device = -1;
    int num_sms = 0;
    int grid_ctas = 0;  // CTAs of the cooperative (grid-barrier) CG kernel
    size_t cap_px = 0, cap_coarse = 0, cap_w = 0;
    double* ex = nullptr;       // tile-kernel edge exchange buffers
    unsigned long long* trace = nullptr;  // HIVC_CG_TRACE diagnostics (finest level phase timestamps)
    bool cluster_ok = false;    // 16-CTA cluster kernels for the coarse/mid levels (device can host one)
    // throughput mode (decode lanes): solves of a batch run side by side on the
    // tile kernel, sharing the SMs; latency mode spreads a level over every SM
    bool pack_bands = false;
    size_t ex_cap = 0;         // doubles in ex
    double* dbl = nullptr;
    uint8_t* bytes = nullptr;
    double* partials = nullptr;
    unsigned int* bar = nullptr;
    int* iters = nullptr;      // device: per level (coarse -> fine) CG iterations
    double* margins = nullptr; // device: per level min relative stop-test margin
    cudaEvent_t pre_done = nullptr;  // solve_batch_async: side-stream levels done
    void reserve(int h, int w, int dev);
    void release();
    ~InpaintWorkspace() {
        release();
        if (pre_done) cudaEventDestroy(pre_done);
    }
};

void pyramid_shapes(int h, int w, std::vector<std::pair<int, int>>& shapes);

// Accumulated CG statistics (algorithmic-byte accounting for the roofline).
struct CgTotals {
    int64_t solves = 0;
    int64_t pixel_iters = 0;       // sum over solves and levels of N_l * it_l
    int64_t pixel_levels = 0;      // sum of N_l (per-level setup passes)
    int64_t grid_launches = 0;     // cooperative (multi-CTA) level kernels
    double grid_seconds = 0;       // their summed device time (CUDA events)
    int64_t grid_pixel_iters = 0;  // N_l * it_l of those launches
    int64_t grid_pixels = 0;       // N_l of those launches
};

// Optional per-solve probe: CUDA events around every cooperative level
// kernel and an async copy of the per-level iteration counts to pinned memory.
struct CgProbe {
    struct Launch {  // one level launch covering solves [first_solve, first_solve + nsolves)
        cudaEvent_t start = nullptr, stop = nullptr;
        int64_t pixels = 0;  // per solve
        int first_solve = 0, nsolves = 1, level = 0;
        int stamp_base = 0;  // stamp slots stamp_base + j (entry/exit of solve j's band 0)
    };
    struct Solve {
        int nlevels = 0;
        int64_t pixels[32] = {};
        int* host_iters = nullptr;
    };
    static constexpr int kCap = 512;
    static constexpr int kStampCap = 4096;
    std::vector<Launch> launches;
    std::vector<Solve> solves;
    int* host = nullptr;
    int used = 0;
    int next_stamp = 0;
    // HIVC_BATCH_TRACE: labelled event pairs around each phase of a batched
    // solve, printed (stderr) by harvest
    struct Mark {
        std::string label;
        cudaEvent_t a, b;
    };
    std::vector<Mark> marks;
    void mark_begin(cudaStream_t s, const std::string& label);
    void mark_end(cudaStream_t s);
    unsigned long long* stamps_dev = nullptr;  // [kStampCap][2] globaltimer entry/exit per launch
    int* alloc_iters();
    unsigned long long* stamp_slot(int i);
    void harvest(CgTotals& t);  // call after the stream synchronised
    void reset();
    ~CgProbe();
};

// Queue the full cascadic solve of (f, m) on stream s; u_out receives the
// finest-level solution.  Returns the number of pyramid levels; per-level
// iteration counts land in ws.iters (coarse -> fine) on the device.
int solve_homogeneous_async(InpaintWorkspace& ws, cudaStream_t s, const double* f, const uint8_t* m, int h, int w,
                            double tol, int max_iter, double* u_out, int64_t* launches, CgProbe* probe = nullptr);

// K (<= 16) same-shape solves in one set of launches on stream s: batched
// pyramid, one thread-block cluster per solve for the coarse levels, and for
// the large levels either one ticketed launch running the solves side by side
// (throughput mode, w <= 1024) or one cooperative launch per solve.  Every
// job needs its own workspace.  Spinning (grid-barrier) launches must not run
// concurrently with another batch's: issue all batches on one stream.
struct SolveJob {
    InpaintWorkspace* ws;
    const double* f;
    const uint8_t* m;
    double* u;
    cudaEvent_t done = nullptr;  // optional: recorded on s as soon as this job's solution is complete
};
// s_pre (optional): stream for the pyramid and the cluster/single-CTA levels;
// the finest levels (grid barriers) follow on s.  Either way the solution is
// complete in stream order on s.
int solve_batch_async(const SolveJob* jobs, int K, int h, int w, double tol, int max_iter, cudaStream_t s,
                      int64_t* launches, CgProbe* probe = nullptr, cudaStream_t s_pre = nullptr);

// L_II z_I = rhs_I with z = 0 held on the mask (the interior rows of the
// transpose inpainting system, for the LSQR adjoint of
// prediction.optimize_mask_values): CG from 0 until ||r|| <= tol ||rhs_I||.
// z_out receives the full plane (zeros on the mask).  Returns the iterations.
int solve_poisson_interior(InpaintWorkspace& ws, cudaStream_t s, const double* rhs, const uint8_t* m, int h, int w,
                           double tol, int max_iter, double* z_out, int64_t* launches);
// out[k] = w[pts[k]] - (sum of z over pts[k]'s existing 4-neighbours)
void launch_mask_adjoint(const double* w_full, const double* z, const int32_t* pts, int npts, int h, int w, double* out,
                         cudaStream_t s);

// Relative residual of the inpainting equation (homogeneous.py:206-211);
// synchronises the stream.  Returns -1 when ||f|mask|| == 0.
double strict_relative_residual(InpaintWorkspace& ws, cudaStream_t s, const double* u, const double* f,
                                const uint8_t* m, int h, int w, int64_t* launches);

}  // namespace hivc
